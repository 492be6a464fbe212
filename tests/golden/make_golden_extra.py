"""Extra full-size reference goldens for the less common decode paths,
produced by the REAL reference (dev container only; committed as
tests/golden/extra_sets.npz):

  ens2_sl   random_model(FULL, 1) + random_model(FULL, 2) with the reference's
            build_shortlist lists (ensemble + shortlist masks on the fused
            tensor-core logit kernel)
  beam16    one model at beam 16 (largest top-k list of the rows-layout kernel)
  beam9     one model at beam 9 (KK = 10 instantiations)

Sentences: short stratified cfg2 samples; per-step gaps recorded like
make_golden_fullset.py.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_extra.py --procs 8
"""

from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden_ensemble as E  # noqa: E402
import make_golden_fullset as F  # noqa: E402

from paper_1610_01108_b200 import workload as W  # noqa: E402

FULL = F.FULL
SETS = {  # name: (members, sentences, max source length, opts, shortlists?)
    "ens2_sl": ([(FULL, 1), (FULL, 2)], 24, 40, (5, 2, 10, False, 1), True),
    "beam16": ([(FULL, 1)], 8, 16, (16, 2, 10, False, 1), False),
    "beam9": ([(FULL, 1)], 8, 24, (9, 2, 10, False, 1), False),
}


def _decode(job):
    j, src, members, opts, sl = job
    F._init()
    F._GAPS.clear()
    from beamnmt.shortlist import ShortList

    models = [E._member(c, s) for c, s in members]
    h = F.ref_search.beam_search(models, src, F.ref_search.DecodeOptions(*opts),
                                 None if sl is None else ShortList(np.asarray(sl)))[0]
    return j, np.asarray(h.tokens, np.int32), float(h.score), bool(h.finished), np.asarray(F._GAPS, np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    F._init()
    corpus = W.WORKLOADS["cfg2"].corpus()
    out = {}
    for name, (members, n, jmax, opts, use_sl) in SETS.items():
        for c, s in members:
            E._member(c, s)
        pool_idx = [i for i in range(len(corpus)) if len(corpus[i]) <= jmax]
        idx = [pool_idx[k] for k in E.sample([corpus[i] for i in pool_idx], n)]
        sents = [corpus[i] for i in idx]
        sls = W.shortlists(sents) if use_sl else [None] * len(sents)
        jobs = sorted(((j, sents[j], members, opts, None if sls[j] is None else sls[j].tolist())
                       for j in range(len(sents))), key=lambda x: -len(x[1]))
        res = [None] * len(sents)
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(args.procs) as pool:
            for j, toks, score, fin, gaps in pool.imap_unordered(_decode, jobs, chunksize=1):
                res[j] = (toks, score, fin, gaps)
        print(f"{name}: {len(sents)} sentences in {time.perf_counter() - t0:.0f}s", flush=True)
        out[f"{name}_idx"] = np.asarray(idx, np.int32)
        out[f"{name}_members"] = np.asarray([[c["d_emb"], c["d_h"], c["d_att"], s] for c, s in members], np.int64)
        out[f"{name}_shortlists"] = np.asarray(int(use_sl))
        out[f"{name}_tokens"] = np.concatenate([r[0] for r in res]).astype(np.int32)
        out[f"{name}_tok_off"] = np.cumsum([0] + [r[0].size for r in res]).astype(np.int64)
        out[f"{name}_score"] = np.asarray([r[1] for r in res], np.float64)
        out[f"{name}_finished"] = np.asarray([r[2] for r in res], np.bool_)
        out[f"{name}_gap"] = np.concatenate([r[3] for r in res])
        out[f"{name}_gap_off"] = np.cumsum([0] + [r[3].size for r in res]).astype(np.int64)
        out[f"{name}_opts"] = np.asarray([int(x) for x in opts], np.int64)
    np.savez_compressed(HERE / "extra_sets.npz", **out)


if __name__ == "__main__":
    main()
