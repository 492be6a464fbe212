"""Ensemble decode throughput: the cfg2 workload
(env ENS_CFG) decoded by 1, 2 and 3 members (random_model seeds 1, 2, 3)
on the fused tensor-core logit path, and by 2 members on the CUDA-core
full-logit path (force_full_logits) for comparison; device time from the
library's CUDA events."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_01108_b200 import _lib, workload as W  # noqa: E402
from paper_1610_01108_b200.model import ModelConfig, random_model  # noqa: E402

wl = W.WORKLOADS[os.environ.get("ENS_CFG", "cfg2")]
sents = wl.corpus()
cfg = ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT)
dms = [_lib.device_model(random_model(cfg, s), 0) for s in (W.MODEL_SEED, 2, 3)]
runs = [("1 member", dms[:1], False), ("2 members fused", dms[:2], False), ("3 members fused", dms[:3], False),
        ("2 members full-logit", dms[:2], True)]
for it in range(2):
    for tag, ms, full in runs:
        out = _lib.decode(ms, sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, max_batch=wl.batch,
                          force_full_logits=full)
        toks = sum(len(out.hyps(i)[0][0]) - (1 if out.hyps(i)[0][2] else 0) for i in range(len(sents)))
        print(f"{wl.name} {tag}: {toks / (out.device_ms / 1e3):.0f} target words/s ({out.device_ms:.1f} ms device)",
              flush=True)
