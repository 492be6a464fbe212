"""CPU oracle for the beam-search decode path — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
`beamnmt` (read-only at /root/reference/pkg/src/beamnmt) for exactly the
hot path this repository accelerates: random-model generation, the
bidirectional GRU encoder, MLP attention, the decoder GRU step, the deep
output + logits + log-softmax, ensemble averaging, top-k selection with the
reference tie-break, and the beam-search loop.  Every function cites the
reference file:line it restates.

Who may use it: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` — as the checker or
the timed CPU baseline, never as the product path.  The product
(`paper_1610_01108_b200`) must never import this file.

Pinning: `tests/golden/make_golden.py` imports the real reference in the
dev container, runs both on identical inputs and records the outputs in
`tests/golden/*.npz|json`; `tests/test_oracle_golden.py` checks this module
reproduces those fixtures bit-for-bit (same numpy calls, same shapes, same
order of operations => same OpenBLAS results).

The numpy operation order below is deliberately the reference's, because
bit-identity with the reference is what pins the oracle.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

EOS_ID = 0  # model.py:39
UNK_ID = 1  # model.py:40
EXHAUSTIVE_GUARD = 10**6  # search.py:26

GRU_PARTS = ("W_z", "W_r", "W_h", "U_z", "U_r", "U_h", "b_z", "b_r", "b_h")  # model.py:42


# ---------------------------------------------------------------- model.py

def schema(v_src: int, v_trg: int, d_emb: int, d_h: int, d_att: int) -> list[tuple[str, int, int]]:
    """Canonical tensor list (name, rows, cols) — restates model.py:89-117."""
    out = [("E_src", v_src, d_emb), ("E_trg", v_trg, d_emb)]
    for prefix, d_in in (("enc_fwd", d_emb), ("enc_bwd", d_emb), ("dec", d_emb + 2 * d_h)):
        for part in GRU_PARTS:
            shape = {"W": (d_in, d_h), "U": (d_h, d_h), "b": (1, d_h)}[part[0]]
            out.append((f"{prefix}.{part}", *shape))
    out += [
        ("W_init", 2 * d_h, d_h), ("b_init", 1, d_h),
        ("W_att_s", d_h, d_att), ("W_att_h", 2 * d_h, d_att), ("v_att", 1, d_att),
        ("W_out_s", d_h, d_emb), ("W_out_y", d_emb, d_emb), ("W_out_c", 2 * d_h, d_emb),
        ("b_out", 1, d_emb),
        ("W_logit", d_emb, v_trg), ("b_logit", 1, v_trg),
    ]
    return out


def is_vector(name: str) -> bool:
    """model.py:120-122: biases and v_att are stored as 1-D vectors."""
    base = name.rsplit(".", 1)[-1]
    return base.startswith("b_") or base == "v_att"


def random_tensors(dims: tuple[int, int, int, int, int], seed: int) -> dict[str, np.ndarray]:
    """model.py:328-338: PCG64(seed); weights U[-0.1,0.1) f64->f32 drawn in
    schema order; biases zero with no draws; v_att drawn."""
    rng = np.random.default_rng(seed)
    out: dict[str, np.ndarray] = {}
    for name, rows, cols in schema(*dims):
        if is_vector(name) and name != "v_att":
            arr = np.zeros((rows, cols), dtype=np.float32)
        else:
            arr = rng.uniform(-0.1, 0.1, size=(rows, cols)).astype(np.float32)
        out[name] = arr.reshape(cols) if is_vector(name) else arr
    return out


# ---------------------------------------------------------------- tensor.py

def sigmoid(x: np.ndarray) -> np.ndarray:
    """tensor.py:44-50 (overflow of exp(-x) is the benign saturated limit)."""
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def log_softmax_rows(mat: np.ndarray) -> np.ndarray:
    """tensor.py:79-92: max-shift, then log of summed exponentials, in f64."""
    mat = np.asarray(mat, dtype=np.float64)
    shifted = mat - mat.max(axis=1, keepdims=True)
    return shifted - np.log(np.exp(shifted).sum(axis=1, keepdims=True))


# ---------------------------------------------------------------- nnet.py

class Gru:
    """nnet.py:59-70 — reset-before-matmul GRU on f64 working copies."""

    def __init__(self, t: dict[str, np.ndarray], prefix: str):
        for part in GRU_PARTS:
            setattr(self, part, np.ascontiguousarray(t[f"{prefix}.{part}"], dtype=np.float64))

    def rows(self, x: np.ndarray, h: np.ndarray) -> np.ndarray:
        z = sigmoid(x @ self.W_z + h @ self.U_z + self.b_z)
        r = sigmoid(x @ self.W_r + h @ self.U_r + self.b_r)
        cand = np.tanh(x @ self.W_h + (r * h) @ self.U_h + self.b_h)
        return (1.0 - z) * h + z * cand


@dataclass(eq=False)
class Ann:
    """nnet.py:36-49: annotations h [J, 2 d_h] and precomp_att = h W_att_h."""

    h: np.ndarray
    precomp: np.ndarray


class Net:
    """f64 forward pass — restates nnet.py:73-164 (Forward)."""

    def __init__(self, t: dict[str, np.ndarray]):
        f8 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        self.v_src, self.d_emb = t["E_src"].shape
        self.v_trg = t["E_trg"].shape[0]
        self.d_h = t["W_init"].shape[1]
        self.E_src, self.E_trg = f8(t["E_src"]), f8(t["E_trg"])
        self.fwd, self.bwd, self.dec = Gru(t, "enc_fwd"), Gru(t, "enc_bwd"), Gru(t, "dec")
        self.W_init, self.b_init = f8(t["W_init"]), f8(t["b_init"])
        self.W_att_s, self.W_att_h, self.v_att = f8(t["W_att_s"]), f8(t["W_att_h"]), f8(t["v_att"])
        self.W_out_s, self.W_out_y, self.W_out_c = f8(t["W_out_s"]), f8(t["W_out_y"]), f8(t["W_out_c"])
        self.b_out = f8(t["b_out"])
        # nnet.py:99 — output projection cached as one row per target word
        self.logit_rows = np.ascontiguousarray(t["W_logit"].T, dtype=np.float64)
        self.b_logit = f8(t["b_logit"])

    def encode(self, ids: Sequence[int]) -> Ann:
        """nnet.py:110-126: forward GRU left->right, backward right->left,
        both from zero state; h = [fwd ; bwd]; precomp = h W_att_h."""
        emb = self.E_src[np.asarray(list(ids), dtype=np.int64)]
        J = emb.shape[0]
        halves = []
        for cell, order in ((self.fwd, range(J)), (self.bwd, range(J - 1, -1, -1))):
            out = np.empty((J, self.d_h))
            state = np.zeros((1, self.d_h))
            for j in order:
                state = cell.rows(emb[j : j + 1], state)
                out[j] = state[0]
            halves.append(out)
        h = np.concatenate(halves, axis=1)
        return Ann(h=h, precomp=h @ self.W_att_h)

    def init_state(self, a: Ann) -> np.ndarray:
        """nnet.py:128-130: tanh(mean_j h_j W_init + b_init), shape [1, d_h]."""
        return np.tanh(a.h.mean(axis=0, keepdims=True) @ self.W_init + self.b_init)

    def attention(self, s: np.ndarray, a: Ann) -> tuple[np.ndarray, np.ndarray]:
        """nnet.py:132-141: e = v . tanh(P_j + s W_att_s); softmax over j."""
        B, J = s.shape[0], a.h.shape[0]
        act = np.tanh(a.precomp[None, :, :] + (s @ self.W_att_s)[:, None, :])
        e = (act.reshape(B * J, -1) @ self.v_att).reshape(B, J)
        e -= e.max(axis=1, keepdims=True)
        w = np.exp(e)
        alpha = w / w.sum(axis=1, keepdims=True)
        return alpha, alpha @ a.h

    def step(self, s: np.ndarray, y_prev: np.ndarray, a: Ann,
             sl_ids: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """nnet.py:143-164: one decoder step -> (s', log-probs, alpha)."""
        y = self.E_trg[np.asarray(y_prev, dtype=np.int64)]
        alpha, ctx = self.attention(s, a)
        s_next = self.dec.rows(np.concatenate([y, ctx], axis=1), s)
        t = np.tanh(s_next @ self.W_out_s + y @ self.W_out_y + ctx @ self.W_out_c + self.b_out)
        if sl_ids is None:
            logits = t @ self.logit_rows.T + self.b_logit
        else:
            logits = t @ self.logit_rows[sl_ids].T + self.b_logit[sl_ids]
        return s_next, log_softmax_rows(logits), alpha


# ---------------------------------------------------------------- search.py

@dataclass(frozen=True)
class Opts:
    """search.py:44-53 (DecodeOptions)."""

    beam_size: int = 5
    max_len_factor: int = 2
    max_len_offset: int = 10
    length_normalize: bool = False
    n_best: int = 1

    def cap(self, src_len: int) -> int:
        return self.max_len_factor * src_len + self.max_len_offset


@dataclass(eq=False)
class Hyp:
    """search.py:29-41 (Hypothesis)."""

    tokens: list[int]
    score: float
    states: list[np.ndarray]
    finished: bool

    def rank_score(self, normalize: bool) -> float:
        if normalize and self.tokens:
            return self.score / len(self.tokens)
        return self.score


def mean_about_first(stack: np.ndarray) -> np.ndarray:
    """search.py:67-72: first + mean(stack - first)."""
    first = stack[0]
    return first + (stack - first[None]).mean(axis=0)


def select_top(flat: np.ndarray, k: int, n_cols: int) -> np.ndarray:
    """search.py:75-91: k best flat candidates; ties -> lower token, then
    lower parent; result ordered by (score desc, token asc, parent asc)."""
    if flat.size > k:
        kth = np.partition(flat, flat.size - k)[flat.size - k]
        above = np.nonzero(flat > kth)[0]
        tied = np.nonzero(flat == kth)[0]
        tied = tied[np.lexsort((tied // n_cols, tied % n_cols))]
        idx = np.concatenate([above, tied[: k - above.size]])
    else:
        idx = np.arange(flat.size)
    return idx[np.lexsort((idx // n_cols, idx % n_cols, -flat[idx]))]


@dataclass(eq=False)
class StepTrace:
    """Per-step instrumentation (not in the reference): the k-th and
    (k+1)-th best candidate scores, used to adjudicate near-tie divergences."""

    kth: list[float] = field(default_factory=list)
    next_: list[float] = field(default_factory=list)


def beam_search(nets: Sequence[Net], src: Sequence[int], opts: Opts = Opts(),
                sl_ids: np.ndarray | None = None, trace: StepTrace | None = None) -> list[Hyp]:
    """search.py:116-216: beam search over an ensemble of models."""
    if len(src) == 0:
        raise ValueError("cannot decode an empty source sentence")
    if opts.beam_size < 1:
        raise ValueError(f"beam_size must be >= 1, got {opts.beam_size}")
    if opts.n_best < 1:
        raise ValueError(f"n_best must be >= 1, got {opts.n_best}")
    cap = opts.cap(len(src))
    if cap < 1:
        raise ValueError(f"length cap {cap} must be >= 1")
    if sl_ids is not None:
        sl_ids = np.asarray(sl_ids, dtype=np.int64)
    anns = [n.encode(src) for n in nets]
    seqs: list[list[int]] = [[]]
    scores = np.zeros(1)
    states = [n.init_state(a) for n, a in zip(nets, anns)]
    prev = np.array([EOS_ID], dtype=np.int64)
    done: list[tuple[float, list[int], list[np.ndarray]]] = []
    for _ in range(cap):
        outs = [n.step(s, prev, a, sl_ids) for n, s, a in zip(nets, states, anns)]
        nxt = [o[0] for o in outs]
        lp = mean_about_first(np.stack([o[1] for o in outs]))
        n_cols = lp.shape[1]
        flat = (scores[:, None] + lp).ravel()
        chosen = select_top(flat, opts.beam_size, n_cols)
        if trace is not None and flat.size > opts.beam_size:
            srt = np.sort(flat)[::-1]
            trace.kth.append(float(srt[opts.beam_size - 1]))
            trace.next_.append(float(srt[opts.beam_size]))
        parents = chosen // n_cols
        toks = chosen % n_cols
        gids = toks if sl_ids is None else sl_ids[toks]
        new_scores = flat[chosen]
        keep, kept_seqs = [], []
        for i, (p, g) in enumerate(zip(parents, gids)):
            seq = seqs[p] + [int(g)]
            if int(g) == EOS_ID:
                done.append((float(new_scores[i]), seq, [x[p].copy() for x in nxt]))
            else:
                keep.append(i)
                kept_seqs.append(seq)
        if not keep:
            break
        ki = np.asarray(keep, dtype=np.int64)
        seqs = kept_seqs
        scores = new_scores[ki]
        states = [x[parents[ki]] for x in nxt]
        prev = gids[ki].astype(np.int64)
        if done and float(scores.max()) <= max(d[0] for d in done):
            break
    if done:
        hyps = [Hyp(list(q), sc, st, True) for sc, q, st in done]
    else:
        hyps = [Hyp(seqs[i], float(scores[i]), [x[i] for x in states], False) for i in range(len(seqs))]
    hyps.sort(key=lambda h: (-h.rank_score(opts.length_normalize), h.tokens))
    return hyps[: opts.n_best]


def exhaustive_search(nets: Sequence[Net], src: Sequence[int], cap: int) -> Hyp:
    """search.py:219-277: best sequence by full enumeration (tiny models)."""
    v = nets[0].v_trg
    if v**cap > EXHAUSTIVE_GUARD:
        raise ValueError(f"search space v_trg^cap = {v}^{cap} exceeds the guard")
    anns = [n.encode(src) for n in nets]
    best: list = [None, None]

    def consider(slot, score, seq, st):
        cur = best[slot]
        if cur is None or score > cur[0] or (score == cur[0] and seq < cur[1]):
            best[slot] = (score, seq, st)

    def expand(prefix, score, prev, st):
        outs = [n.step(s, np.array([prev], dtype=np.int64), a) for n, s, a in zip(nets, st, anns)]
        nst = [o[0] for o in outs]
        row = mean_about_first(np.stack([o[1][0] for o in outs]))
        consider(0, score + float(row[EOS_ID]), prefix + [EOS_ID], nst)
        for tok in range(1, v):
            if len(prefix) + 1 < cap:
                expand(prefix + [tok], score + float(row[tok]), tok, nst)
            else:
                consider(1, score + float(row[tok]), prefix + [tok], nst)

    expand([], 0.0, EOS_ID, [n.init_state(a) for n, a in zip(nets, anns)])
    slot = 0 if best[0] is not None else 1
    score, seq, st = best[slot]
    return Hyp(seq, score, [s[0] for s in st], slot == 0)


# ---------------------------------------------------------------- engine.py

def decode_corpus(nets: Sequence[Net], sentences: Sequence[Sequence[int]], opts: Opts,
                  threads: int | None = None) -> list[list[Hyp]]:
    """engine.py:181-221: order-preserving sentence-parallel pool of worker
    threads with BLAS pinned to one thread each (the reference CPU decoder's
    only parallelism)."""
    from threadpoolctl import threadpool_limits

    threads = threads or os.cpu_count() or 1
    results: list = [None] * len(sentences)
    with threadpool_limits(limits=1):
        if threads <= 1 or len(sentences) <= 1:
            return [beam_search(nets, s, opts) for s in sentences]
        nxt = iter(range(len(sentences)))
        lock = threading.Lock()
        errors: list[BaseException] = []

        def worker():
            while True:
                with lock:
                    i = next(nxt, None)
                if i is None:
                    return
                try:
                    results[i] = beam_search(nets, sentences[i], opts)
                except BaseException as e:  # surfaced after join
                    errors.append(e)
                    return

        pool = [threading.Thread(target=worker) for _ in range(threads)]
        for t in pool:
            t.start()
        for t in pool:
            t.join()
        if errors:
            raise errors[0]
    return results


# ---------------------------------------------------------------- workloads

def synthetic_lengths(n: int, seed: int, max_len: int) -> np.ndarray:
    """J = clip(rint(lognormal(ln 26, 0.6)), 1, max_len)."""
    rng = np.random.default_rng(seed)
    return np.clip(np.rint(rng.lognormal(np.log(26.0), 0.6, size=n)), 1, max_len).astype(np.int64)


def synthetic_corpus(n: int, seed: int, max_len: int, v_src: int = 30000,
                     fixed_len: int | None = None) -> list[list[int]]:
    """Sentences of ids uniform in [2, v_src) (tests/conftest.py:44 style)."""
    rng = np.random.default_rng(seed)
    if fixed_len is None:
        lens = np.clip(np.rint(rng.lognormal(np.log(26.0), 0.6, size=n)), 1, max_len).astype(np.int64)
    else:
        lens = np.full(n, fixed_len, dtype=np.int64)
    return [[int(i) for i in rng.integers(2, v_src, size=int(L))] for L in lens]
