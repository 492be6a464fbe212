"""Generate the golden fixtures that pin `oracle/beamnmt_oracle.py` (and,
through it, the CUDA path) to the REAL reference package.

Runs only in the dev container, where the read-only reference lives at
/root/reference/pkg/src.  Outputs (committed):

  tests/golden/tiny.json      tiny-model decodes, exhaustive oracles, KATs
  tests/golden/tiny.npz       tiny-model encoder / decoder_step arrays
  tests/golden/full.json      full-size (emb500/hid1024/30k, seed 1) decodes
                              for cfg1 (100 sentences), a cfg2 bucket, a cfg4
                              sample and a cfg5 sample: reference tokens and
                              scores, plus per-step k-th/(k+1)-th candidate
                              scores traced by the oracle (for near-tie
                              adjudication); per-tensor sha256 of the
                              reference random_model.

Every full-size decode is run by BOTH the reference and the oracle and the
script asserts they agree bit-for-bit before writing anything.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--skip-full]
"""

from __future__ import annotations

import argparse
import hashlib
import json
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

import beamnmt  # noqa: E402  (the reference)
from beamnmt.model import ModelConfig, ModelParams, random_model, schema  # noqa: E402
from beamnmt.nnet import Forward, decoder_step, encode, init_decoder_state  # noqa: E402
from beamnmt.search import DecodeOptions, _select_top, beam_search, exhaustive_search  # noqa: E402
from beamnmt.shortlist import ShortList  # noqa: E402

from oracle import beamnmt_oracle as orc  # noqa: E402

FULL = dict(v_src=30000, v_trg=30000, d_emb=500, d_h=1024, d_att=1024)


def tiny_model(seed, v_src=5, v_trg=5, d=4):
    return random_model(ModelConfig(v_src=v_src, v_trg=v_trg, d_emb=d, d_h=d, d_att=d), seed)


def hyp_json(h):
    return {"tokens": [int(t) for t in h.tokens], "score": float(h.score), "finished": bool(h.finished)}


def tiny_fixtures():
    cases = []
    arrays = {}
    # (a) beam decodes over many tiny models, several beams / n_best / normalize
    rng = np.random.default_rng(123)
    for i in range(60):
        v_src = int(rng.integers(3, 9))
        v_trg = int(rng.integers(2, 9))
        d = int(rng.integers(2, 9))
        seed = 50_000 + i
        m = tiny_model(seed, v_src, v_trg, d)
        src = [int(x) for x in rng.integers(0, v_src, size=int(rng.integers(1, 5)))]
        beam = int(rng.choice([1, 2, 3, 5, 8, 12]))
        nb = int(rng.integers(1, 5))
        norm = bool(rng.integers(0, 2))
        opts = DecodeOptions(beam_size=beam, max_len_factor=int(rng.integers(0, 3)),
                             max_len_offset=int(rng.integers(1, 6)), length_normalize=norm, n_best=nb)
        hyps = beam_search([m], src, opts)
        cases.append({"kind": "beam", "seed": seed, "v_src": v_src, "v_trg": v_trg, "d": d, "src": src,
                      "opts": [beam, opts.max_len_factor, opts.max_len_offset, int(norm), nb],
                      "hyps": [hyp_json(h) for h in hyps]})
    # (b) exhaustive oracle + full-width beam (acceptance c01 pattern)
    for i in range(24):
        v_trg = 3 + i % 3
        src = [2] * (1 + i % 3)
        seed = 10_000 + i
        m = tiny_model(seed, 5, v_trg, 4)
        ex = exhaustive_search([m], src, 4)
        fw = beam_search([m], src, DecodeOptions(beam_size=v_trg**4, max_len_factor=0, max_len_offset=4))[0]
        cases.append({"kind": "exhaustive", "seed": seed, "v_src": 5, "v_trg": v_trg, "d": 4, "src": src,
                      "cap": 4, "exhaustive": hyp_json(ex), "full_width": hyp_json(fw)})
    # (c) ensembles (4 copies, and 2 different models)
    for i in range(6):
        ma, mb = tiny_model(700 + i, 6, 6, 5), tiny_model(800 + i, 6, 6, 5)
        src = [2, 3, 4][: 1 + i % 3]
        opts = DecodeOptions(beam_size=3, max_len_factor=1, max_len_offset=3, n_best=3)
        cases.append({"kind": "ensemble", "seeds": [700 + i, 800 + i], "v_src": 6, "v_trg": 6, "d": 5,
                      "src": src, "opts": [3, 1, 3, 0, 3],
                      "copies": [hyp_json(h) for h in beam_search([ma] * 4, src, opts)],
                      "pair": [hyp_json(h) for h in beam_search([ma, mb], src, opts)]})
    # (c2) ensembles of members with different d_emb / d_h / d_att (the
    # reference runs one Forward per member, search.py:150-152)
    for i in range(4):
        ma = random_model(ModelConfig(v_src=6, v_trg=7, d_emb=5, d_h=4, d_att=3), 1700 + i)
        mb = random_model(ModelConfig(v_src=6, v_trg=7, d_emb=3, d_h=6, d_att=5), 1800 + i)
        src = [2, 3, 4, 5][: 1 + i % 4]
        opts = DecodeOptions(beam_size=3, max_len_factor=1, max_len_offset=3, n_best=2)
        cases.append({"kind": "ensemble_mixed", "seeds": [1700 + i, 1800 + i], "dims": [[6, 7, 5, 4, 3], [6, 7, 3, 6, 5]],
                      "src": src, "opts": [3, 1, 3, 0, 2],
                      "hyps": [hyp_json(h) for h in beam_search([ma, mb], src, opts)],
                      "states": [[[float(x) for x in st.s] for st in h.states] for h in beam_search([ma, mb], src, opts)]})
    # (d) shortlist decodes
    for i in range(6):
        m = tiny_model(900 + i, 7, 9, 4)
        ids = [0, 1] + sorted(set(int(x) for x in np.random.default_rng(i).integers(2, 9, size=4)))
        src = [2, 5, 3][: 1 + i % 3]
        opts = DecodeOptions(beam_size=3, max_len_factor=1, max_len_offset=3, n_best=2)
        cases.append({"kind": "shortlist", "seed": 900 + i, "v_src": 7, "v_trg": 9, "d": 4, "src": src,
                      "shortlist": ids, "opts": [3, 1, 3, 0, 2],
                      "hyps": [hyp_json(h) for h in beam_search([m], src, opts, shortlist=ShortList(np.array(ids)))]})
    # (e) per-step arrays: encoder, init state, decoder_step (with and without shortlist)
    for i in range(8):
        d = 3 + i
        m = tiny_model(300 + i, 9, 11, d)
        src = [2, 7, 4, 8, 3][: 1 + i % 5]
        a = encode(m, src)
        s0 = init_decoder_state(m, a)
        s1, lp1, al1 = decoder_step(m, s0, 0, a)
        s2, lp2, al2 = decoder_step(m, s1, 5, a, ShortList(np.array([0, 1, 3, 5, 6])))
        for k, v in dict(h=a.h, p=a.precomp_att, s0=s0.s, s1=s1.s, lp1=lp1, al1=al1, s2=s2.s, lp2=lp2,
                         al2=al2).items():
            arrays[f"step{i}_{k}"] = v
        cases.append({"kind": "step", "seed": 300 + i, "v_src": 9, "v_trg": 11, "d": d, "src": src,
                      "y1": 0, "y2": 5, "shortlist2": [0, 1, 3, 5, 6], "key": f"step{i}"})
    # (f) tie-break KATs (test_search.py:160-177 pattern)
    kats = {
        "select_zero_10_4_5": [int(x) for x in _select_top(np.zeros(10), 4, n_cols=5)],
        "select_small": [int(x) for x in _select_top(np.array([-1.0, -0.5, -0.5, -2.0, -0.5, -3.0]), 3, n_cols=3)],
    }
    cfg = ModelConfig(v_src=5, v_trg=5, d_emb=4, d_h=4, d_att=4)
    zeros = ModelParams.from_tensors(cfg, {n: np.zeros((r, c), np.float32) for n, r, c in schema(cfg)})
    kats["all_zero_model"] = [hyp_json(h) for h in beam_search(
        [zeros], [2], DecodeOptions(beam_size=3, max_len_factor=0, max_len_offset=2, n_best=3))]
    return {"cases": cases, "kats": kats}, arrays


# ------------------------------------------------------------------ full size

_REF = None
_ORC = None


def _init_full():
    global _REF, _ORC
    if _REF is None:
        _REF = random_model(ModelConfig(**FULL), 1)
        Forward.for_params(_REF)
        t = {name: arr for name, arr in _REF.tensor_items()}
        _ORC = orc.Net(t)


def _decode_one(job):
    src, opts = job
    _init_full()
    o = DecodeOptions(*opts)
    t0 = time.perf_counter()
    ref = beam_search([_REF], src, o)
    t_ref = time.perf_counter() - t0
    trace = orc.StepTrace()
    mine = orc.beam_search([_ORC], src, orc.Opts(*opts), trace=trace)
    same = [(h.tokens, h.score, h.finished) for h in ref] == [(h.tokens, h.score, h.finished) for h in mine]
    return {"hyps": [hyp_json(h) for h in ref], "oracle_bitexact": bool(same), "kth": trace.kth,
            "next": trace.next_, "ref_seconds": t_ref}


def full_fixtures(procs: int):
    _init_full()
    sha = {name: hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
           for name, arr in _REF.tensor_items()}
    cfg1 = orc.synthetic_corpus(100, 2017, 50)
    cfg2 = orc.synthetic_corpus(4000, 2016, 100)
    order = np.argsort([len(s) for s in cfg2], kind="stable")
    bucket_idx = [int(i) for i in order[::62][:64]]  # stratified 64-sentence sample across lengths
    cfg4 = orc.synthetic_corpus(512, 2018, 100, fixed_len=100)[:6]
    sets = {
        "cfg1": ([(s, (5, 2, 10, False, 1)) for s in cfg1], list(range(100))),
        "cfg2_strat64": ([(cfg2[i], (5, 2, 10, False, 1)) for i in bucket_idx], bucket_idx),
        "cfg4_6": ([(s, (12, 1, 0, False, 1)) for s in cfg4], list(range(6))),
        "cfg5_strat64": ([(cfg2[i], (1, 2, 10, False, 1)) for i in bucket_idx], bucket_idx),
    }
    out = {"model": {"dims": FULL, "seed": 1, "sha256": sha}, "sets": {}}
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for name, (jobs, idx) in sets.items():
            t0 = time.perf_counter()
            res = pool.map(_decode_one, jobs, chunksize=1)
            bad = [i for i, r in enumerate(res) if not r["oracle_bitexact"]]
            print(f"{name}: {len(jobs)} sentences in {time.perf_counter() - t0:.1f}s, oracle mismatches {bad}",
                  flush=True)
            assert not bad, f"oracle differs from reference on {name}: {bad}"
            out["sets"][name] = {"indices": idx, "src": [j[0] for j in jobs], "opts": list(jobs[0][1]),
                                 "results": res}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    tiny, arrays = tiny_fixtures()
    (HERE / "tiny.json").write_text(json.dumps(tiny, indent=0))
    np.savez_compressed(HERE / "tiny.npz", **arrays)
    print("tiny fixtures written", flush=True)
    if not args.skip_full:
        full = full_fixtures(args.procs)
        (HERE / "full.json").write_text(json.dumps(full))
        print("full fixtures written", flush=True)


if __name__ == "__main__":
    main()
