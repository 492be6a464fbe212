"""Shortlist decode throughput (profiling aid): cfg2 with a per-sentence
shortlist of 1250 target ids (</s> + 1249 random), fused tensor-core logits
with vocabulary masks, device time from the library's CUDA events."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model

wl = W.WORKLOADS["cfg2"]
sents = wl.corpus()
model = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
dm = _lib.device_model(model, 0)
rng = np.random.default_rng(0)
sls = [np.unique(np.concatenate([[0], rng.choice(np.arange(2, W.V_TRG), 1249, replace=False)])).astype(np.int32)
       for _ in sents]
for it in range(3):
    out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, shortlists=sls,
                      max_batch=wl.batch)
    toks = sum(len(out.hyps(i)[0][0]) - (1 if out.hyps(i)[0][2] else 0) for i in range(len(sents)))
    print(f"shortlist 1250: {toks / (out.device_ms / 1e3):.0f} target words/s ({out.device_ms:.1f} ms device)",
          flush=True)
