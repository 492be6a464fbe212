"""Encoder-dominated pass (cap 1: one decoder step per bucket) for ncu launch lists."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model
wl = W.WORKLOADS["cfg2"]; sents = wl.corpus()
dm = _lib.device_model(random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED), 0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    out = _lib.decode([dm], sents, 5, 0, 1, False, 1, max_batch=64)
print(f"device {out.device_ms:.1f} ms")
