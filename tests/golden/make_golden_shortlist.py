"""Reference goldens for shortlist decoding, produced
by the REAL reference (dev container only; committed as
tests/golden/shortlist_sets.npz).

Shortlists come from the reference's own build_shortlist
(pkg/src/beamnmt/shortlist.py:128-147) over a LexicalTable holding the
synthetic translation entries of paper_1610_01108_b200.workload (only the
source tokens the sentences use), with the workload's frequency list and
K = K' = 75; the script asserts they equal workload.shortlists() (the ids
the GPU tests and the bench pass to the decoder).  Decodes are the
reference's beam_search(models, src, opts, shortlist) with the per-step
k-th vs (k+1)-th candidate gap recorded (make_golden_fullset.py).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_shortlist.py --procs 7
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
import make_golden_fullset as F  # noqa: E402  (reference import, recorder, model)

from beamnmt.model import Vocabulary  # noqa: E402
from beamnmt.shortlist import LexicalTable, build_shortlist  # noqa: E402

from paper_1610_01108_b200 import workload as W  # noqa: E402

SETS = {  # name: (workload, sentences in the sample, decode options)
    "cfg1": ("cfg1", 32, (5, 2, 10, False, 1)),
    "cfg2": ("cfg2", 32, (5, 2, 10, False, 1)),
}


def sample(corpus, n):
    order = sorted(range(len(corpus)), key=lambda i: (len(corpus[i]), i))
    stride = max(1, len(order) // n)
    return [order[j] for j in range(stride // 2, len(order), stride)][:n]


_SL = {}


def _decode(job):
    i, src, sl_ids, opts = job
    F._init()
    F._GAPS.clear()
    from beamnmt.shortlist import ShortList

    hyps = F.ref_search.beam_search([F._MODEL], src, F.ref_search.DecodeOptions(*opts), ShortList(np.asarray(sl_ids)))
    h = hyps[0]
    return i, np.asarray(h.tokens, np.int32), float(h.score), bool(h.finished), np.asarray(F._GAPS, np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    F._init()
    vocab = Vocabulary.from_tokens([f"w{i}" for i in range(2, W.V_TRG)])
    by_rank = W.target_by_rank()
    freq_ids = [int(i) for i in by_rank]
    out = {}
    for name, (wl_name, n, opts) in SETS.items():
        corpus = W.WORKLOADS[wl_name].corpus()
        idx = sample(corpus, n)
        sents = [corpus[i] for i in idx]
        srcs = sorted({t for s in sents for t in s})
        table = LexicalTable({f"w{s}": [(f"w{int(t)}", 1.0 / (j + 2))
                                        for j, t in enumerate(W.lex_translations(s, by_rank=by_rank))]
                              for s in srcs})
        ref_sl = [build_shortlist(table, freq_ids, [f"w{t}" for t in s], W.SL_K, W.SL_KPRIME, vocab).global_ids
                  for s in sents]
        mine = W.shortlists(sents)
        for a, b in zip(ref_sl, mine):
            assert np.array_equal(np.asarray(a), b.astype(np.int64)), "workload.shortlists != reference build_shortlist"
        jobs = [(j, sents[j], mine[j], opts) for j in range(len(sents))]
        t0 = time.perf_counter()
        res = [None] * len(sents)
        with mp.get_context("fork").Pool(args.procs) as pool:
            for j, toks, score, fin, gaps in pool.imap_unordered(_decode, jobs, chunksize=1):
                res[j] = (toks, score, fin, gaps)
        print(f"{name}: {len(sents)} sentences in {time.perf_counter() - t0:.0f}s, mean |shortlist| "
              f"{np.mean([len(x) for x in mine]):.0f}", flush=True)
        tok_off = np.cumsum([0] + [r[0].size for r in res])
        gap_off = np.cumsum([0] + [r[3].size for r in res])
        out[f"{name}_idx"] = np.asarray(idx, np.int32)
        out[f"{name}_tokens"] = np.concatenate([r[0] for r in res]).astype(np.int32)
        out[f"{name}_tok_off"] = tok_off.astype(np.int64)
        out[f"{name}_score"] = np.asarray([r[1] for r in res], np.float64)
        out[f"{name}_finished"] = np.asarray([r[2] for r in res], np.bool_)
        out[f"{name}_gap"] = np.concatenate([r[3] for r in res])
        out[f"{name}_gap_off"] = gap_off.astype(np.int64)
        out[f"{name}_opts"] = np.asarray([int(x) for x in opts], np.int64)
    np.savez_compressed(HERE / "shortlist_sets.npz", **out)


if __name__ == "__main__":
    main()
