"""Shortlist decode throughput: a workload (env SL_CFG,
default cfg2) decoded with and without the build_shortlist lists of the
synthetic lexical table (workload.shortlists, K = K' = 75); device time
from the library's CUDA events."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model

import os
wl = W.WORKLOADS[os.environ.get("SL_CFG", "cfg2")]
sents = wl.corpus()
model = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
dm = _lib.device_model(model, 0)
sls = W.shortlists(sents)
print(f"{wl.name}: mean shortlist {np.mean([len(x) for x in sls]):.0f} ids", flush=True)
for it in range(3):
    for tag, sl in (("full vocabulary", None), ("shortlists", sls)):
        out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, shortlists=sl,
                          max_batch=wl.batch)
        toks = sum(len(out.hyps(i)[0][0]) - (1 if out.hyps(i)[0][2] else 0) for i in range(len(sents)))
        print(f"{wl.name} {tag}: {toks / (out.device_ms / 1e3):.0f} target words/s ({out.device_ms:.1f} ms device)",
              flush=True)
