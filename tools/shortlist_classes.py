"""Per-class in-situ CTA time (AMUN_PROFILE_CTA_TIME) of a workload decoded
with and without shortlists (profiling aid)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model

wl = W.WORKLOADS[os.environ.get("SL_CFG", "cfg2")]
sents = wl.corpus()
dm = _lib.device_model(random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED), 0)
sls = W.shortlists(sents)
for tag, sl in (("full", None), ("shortlists", sls)):
    for it in range(2):
        out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, shortlists=sl,
                          max_batch=wl.batch, profile=_lib.PROFILE_CTA_TIME)
    print(tag, f"{out.device_ms:.1f} ms", {k: round(v, 1) for k, v in out.kernel_ms.items()},
          {k: int(v) for k, v in out.kernel_ctas.items()}, flush=True)
