"""Full-set golden decodes of the headline workloads, produced by the REAL
reference package (dev container only; /root/reference is absent on the GPU
box, so the outputs are committed as compact npz fixtures):

  tests/golden/fullset_cfg2.npz   4000 sentences, beam 5, cap 2J+10
  tests/golden/fullset_cfg4.npz   512 sentences, J=100, beam 12, cap 100
  tests/golden/fullset_cfg5.npz   the cfg2 set at beam 1

Each file holds, per sentence: the 1-best tokens (ragged: `tok_off`,
`tokens`), the f64 score, the finished flag, and per search step the gap
between the k-th and (k+1)-th best candidate score (ragged: `gap_off`,
`gap`; float32) -- the near-tie adjudication input (SURVEY §8(d) gates).

The gap is traced by wrapping the reference's own `_select_top`
(`pkg/src/beamnmt/search.py:75-91`, called at `search.py:169`) with a
recorder that calls the original and notes np.partition's k-th / (k+1)-th
values of the same `flat` array; the search itself is untouched.  The
sources are regenerated from the seeds (`workload.py`) and a
sha256 of the id lists is stored so a test can check it decodes the same
input.  Bit-identity of the oracle restatement with the reference is pinned
separately (`make_golden.py`, 234 full-size sentences).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_fullset.py --procs 7 [--sets cfg4,cfg2,cfg5]
"""

from __future__ import annotations

import argparse
import hashlib
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import beamnmt.search as ref_search  # noqa: E402  (the reference)
from beamnmt.model import ModelConfig, random_model  # noqa: E402
from beamnmt.nnet import Forward  # noqa: E402

from paper_1610_01108_b200 import workload  # noqa: E402

FULL = dict(v_src=30000, v_trg=30000, d_emb=500, d_h=1024, d_att=1024)
SETS = {
    # name: (corpus builder, (beam, factor, offset, normalize, n_best))
    "cfg2": (workload.WORKLOADS["cfg2"].corpus, (5, 2, 10, False, 1)),
    "cfg4": (workload.WORKLOADS["cfg4"].corpus, (12, 1, 0, False, 1)),
    "cfg5": (workload.WORKLOADS["cfg5"].corpus, (1, 2, 10, False, 1)),
}

_MODEL = None
_GAPS: list[float] = []
_ORIG_SELECT = ref_search._select_top


def _recording_select(flat, k, n_cols=None):
    chosen = _ORIG_SELECT(flat, k, n_cols) if n_cols is not None else _ORIG_SELECT(flat, k)
    if flat.size > k:
        part = -np.partition(-flat, (k - 1, k))
        _GAPS.append(float(part[k - 1] - part[k]))
    return chosen


def _init():
    global _MODEL
    if _MODEL is None:
        _MODEL = random_model(ModelConfig(**FULL), 1)
        Forward.for_params(_MODEL)
        ref_search._select_top = _recording_select


def _decode(job):
    i, src, opts = job
    _init()
    _GAPS.clear()
    hyps = ref_search.beam_search([_MODEL], src, ref_search.DecodeOptions(*opts))
    h = hyps[0]
    return i, np.asarray(h.tokens, np.int32), float(h.score), bool(h.finished), np.asarray(_GAPS, np.float32)


def src_sha(corpus) -> str:
    hs = hashlib.sha256()
    for s in corpus:
        hs.update(np.asarray(s, np.int32).tobytes())
        hs.update(b"|")
    return hs.hexdigest()


def run_set(name: str, procs: int) -> None:
    build, opts = SETS[name]
    corpus = build()
    n = len(corpus)
    jobs = sorted(((i, corpus[i], opts) for i in range(n)), key=lambda j: -len(j[1]))
    out: list = [None] * n
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        for done, (i, toks, score, fin, gaps) in enumerate(pool.imap_unordered(_decode, jobs, chunksize=1), 1):
            out[i] = (toks, score, fin, gaps)
            if done % 250 == 0:
                print(f"{name}: {done}/{n} in {time.perf_counter() - t0:.0f}s", flush=True)
    tok_off = np.zeros(n + 1, np.int64)
    gap_off = np.zeros(n + 1, np.int64)
    for i, (toks, _, _, gaps) in enumerate(out):
        tok_off[i + 1] = tok_off[i] + toks.size
        gap_off[i + 1] = gap_off[i] + gaps.size
    np.savez_compressed(
        HERE / f"fullset_{name}.npz",
        tokens=np.concatenate([o[0] for o in out]).astype(np.int16 if FULL["v_trg"] < 32768 else np.int32),
        tok_off=tok_off,
        score=np.asarray([o[1] for o in out], np.float64),
        finished=np.asarray([o[2] for o in out], np.bool_),
        gap=np.concatenate([o[3] for o in out]),
        gap_off=gap_off,
        opts=np.asarray([int(x) for x in opts], np.int64),
        src_sha256=np.asarray(src_sha(corpus)),
        src_len=np.asarray([len(s) for s in corpus], np.int32),
    )
    early = [i for i, o in enumerate(out) if o[2]]
    print(f"{name}: {n} sentences in {time.perf_counter() - t0:.0f}s; {int(tok_off[-1])} tokens; "
          f"finished (EOS) sentences: {early[:20]}{'...' if len(early) > 20 else ''}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--sets", default="cfg4,cfg2,cfg5")
    args = ap.parse_args()
    _init()  # build the f64 working copies once, before fork (shared copy-on-write)
    for name in args.sets.split(","):
        run_set(name, args.procs)


if __name__ == "__main__":
    main()
