"""Shortlist decode throughput in steady state (profiling aid): the same
configuration decoded repeatedly (no graph re-instantiation between the
timed calls), full vocabulary first, then with shortlists."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model

wl = W.WORKLOADS[os.environ.get("SL_CFG", "cfg2")]
sents = wl.corpus()
dm = _lib.device_model(random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED), 0)
sls = W.shortlists(sents)
for tag, sl in (("full vocabulary", None), ("shortlists", sls)):
    for it in range(3):
        out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, shortlists=sl,
                          max_batch=wl.batch)
        toks = sum(len(out.hyps(i)[0][0]) - (1 if out.hyps(i)[0][2] else 0) for i in range(len(sents)))
        print(f"{wl.name} {tag} rep {it}: {toks / (out.device_ms / 1e3):.0f} target words/s "
              f"({out.device_ms:.1f} ms device, host setup {out.host_setup_ms:.1f} ms)", flush=True)
