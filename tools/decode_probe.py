"""Decode a workload a few times through _lib.decode and print device ms /
target words/s (development probe; env knobs such as AMUN_DEBUG_AHEAD,
AMUN_DEBUG_SCHED, AMUN_ABLATE_CLASSES are read by the library)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1610_01108_b200 import _lib, workload as W  # noqa: E402
from paper_1610_01108_b200.model import ModelConfig, random_model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = W.WORKLOADS[name]
sents = wl.corpus()
dm = _lib.device_model(random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED))
for r in range(reps):
    t0 = time.perf_counter()
    out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, max_batch=wl.batch)
    wall = time.perf_counter() - t0
    toks = sum(len(out.hyps(i)[0][0]) - (1 if out.hyps(i)[0][2] else 0) for i in range(len(sents)))
    print(f"{name} rep {r}: device {out.device_ms:.1f} ms, wall {wall * 1e3:.1f} ms, "
          f"{toks / out.device_ms * 1e3:,.0f} target words/s ({toks} tokens)", flush=True)
