"""Reference goldens for full-size ENSEMBLE decoding,
produced by the REAL reference (dev container only; committed as
tests/golden/ensemble_sets.npz).

The reference averages the members' log-softmax outputs about the first
member (`pkg/src/beamnmt/search.py:56-72`) and runs one Forward per member
(`search.py:150-152`), so members may differ in d_emb / d_h / d_att as long
as the vocabularies match.  Sets (stratified samples of the cfg2 workload,
beam 5, cap 2J+10):

  ens2   members random_model(FULL, 1), random_model(FULL, 2)
  ens3   members seeds 1, 2, 3 (FULL)
  mixed  random_model(FULL, 1) + random_model(v 30000/30000, d_emb 256,
         d_h 512, d_att 512, seed 5)

Per sentence: 1-best tokens (ragged), f64 score, finished flag, and the
per-step k-th vs (k+1)-th candidate gap (make_golden_fullset.py's recorder
around the reference's own _select_top).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_ensemble.py --procs 8
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
import make_golden_fullset as F  # noqa: E402  (reference import, recorder)

from beamnmt.model import ModelConfig, random_model  # noqa: E402
from beamnmt.nnet import Forward  # noqa: E402

from paper_1610_01108_b200 import workload as W  # noqa: E402

FULL = F.FULL
MIXED_B = dict(v_src=30000, v_trg=30000, d_emb=256, d_h=512, d_att=512)
SETS = {  # name: (member (config, seed) list, sentences, decode options)
    "ens2": ([(FULL, 1), (FULL, 2)], 160, (5, 2, 10, False, 1)),
    "ens3": ([(FULL, 1), (FULL, 2), (FULL, 3)], 48, (5, 2, 10, False, 1)),
    "mixed": ([(FULL, 1), (MIXED_B, 5)], 64, (5, 2, 10, False, 1)),
}

_MODELS: dict = {}


def _member(cfg: dict, seed: int):
    key = (tuple(sorted(cfg.items())), seed)
    if key not in _MODELS:
        m = random_model(ModelConfig(**cfg), seed)
        Forward.for_params(m)
        _MODELS[key] = m
    return _MODELS[key]


def sample(corpus, n):
    order = sorted(range(len(corpus)), key=lambda i: (len(corpus[i]), i))
    stride = max(1, len(order) // n)
    return [order[j] for j in range(stride // 2, len(order), stride)][:n]


def _decode(job):
    j, src, members, opts = job
    F._init()  # installs the gap recorder
    F._GAPS.clear()
    models = [_member(c, s) for c, s in members]
    h = F.ref_search.beam_search(models, src, F.ref_search.DecodeOptions(*opts))[0]
    return j, np.asarray(h.tokens, np.int32), float(h.score), bool(h.finished), np.asarray(F._GAPS, np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    F._init()
    corpus = W.WORKLOADS["cfg2"].corpus()
    out = {}
    for name, (members, n, opts) in SETS.items():
        for c, s in members:  # f64 working copies once, before fork
            _member(c, s)
        idx = sample(corpus, n)
        jobs = sorted(((j, corpus[i], members, opts) for j, i in enumerate(idx)), key=lambda x: -len(x[1]))
        res = [None] * len(idx)
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(args.procs) as pool:
            for j, toks, score, fin, gaps in pool.imap_unordered(_decode, jobs, chunksize=1):
                res[j] = (toks, score, fin, gaps)
        print(f"{name}: {len(idx)} sentences in {time.perf_counter() - t0:.0f}s", flush=True)
        tok_off = np.cumsum([0] + [r[0].size for r in res])
        gap_off = np.cumsum([0] + [r[3].size for r in res])
        out[f"{name}_idx"] = np.asarray(idx, np.int32)
        out[f"{name}_members"] = np.asarray([[c["d_emb"], c["d_h"], c["d_att"], s] for c, s in members], np.int64)
        out[f"{name}_tokens"] = np.concatenate([r[0] for r in res]).astype(np.int32)
        out[f"{name}_tok_off"] = tok_off.astype(np.int64)
        out[f"{name}_score"] = np.asarray([r[1] for r in res], np.float64)
        out[f"{name}_finished"] = np.asarray([r[2] for r in res], np.bool_)
        out[f"{name}_gap"] = np.concatenate([r[3] for r in res])
        out[f"{name}_gap_off"] = gap_off.astype(np.int64)
        out[f"{name}_opts"] = np.asarray([int(x) for x in opts], np.int64)
    np.savez_compressed(HERE / "ensemble_sets.npz", **out)


if __name__ == "__main__":
    main()
