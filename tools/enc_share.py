import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model
wl = W.WORKLOADS["cfg2"]; sents = wl.corpus()
model = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
dm = _lib.device_model(model, 0)
for f, o in ((0, 1), (0, 2), (2, 10)):
    for _ in range(2): out = _lib.decode([dm], sents, 5, f, o, False, 1, max_batch=64)
    print(f"cap {f}J+{o}: device {out.device_ms:.1f} ms, steps {out.decoder_steps}", flush=True)
out = _lib.decode([dm], sents, 5, 0, 1, False, 1, max_batch=64, profile=0xFF)
print({k: round(v, 1) for k, v in out.kernel_ms.items()})
