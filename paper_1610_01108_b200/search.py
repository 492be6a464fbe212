"""Beam search API (reference: beamnmt/search.py) on the device decoder.

`beam_search` keeps the reference signature and semantics (search.py:116-216):
priming with "</s>", global top-`beam_size` over active x vocabulary with the
(score desc, token asc, parent asc) tie-break, EOS candidates retired to an
unbounded finished list, refill to `beam_size`, stop on empty beam / best
active <= best finished / length cap, final ranking by (-rank_score, tokens).
All of it runs inside libamun_b200.so (`amun_decode`); this module validates
arguments with the reference's messages and converts the result.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import TYPE_CHECKING, Sequence

import numpy as np

from . import _lib
from .model import EOS_ID, ModelParams
from .nnet import DecoderState, Forward

if TYPE_CHECKING:
    from .shortlist import ShortList

EXHAUSTIVE_GUARD = 10**6


@dataclass(eq=False)
class Hypothesis:
    tokens: list[int]
    score: float
    states: list[DecoderState]
    finished: bool

    def rank_score(self, length_normalize: bool) -> float:
        if length_normalize and self.tokens:
            return self.score / len(self.tokens)
        return self.score


@dataclass(frozen=True)
class DecodeOptions:
    beam_size: int = 5
    max_len_factor: int = 2
    max_len_offset: int = 10
    length_normalize: bool = False
    n_best: int = 1

    def max_target_len(self, src_len: int) -> int:
        return self.max_len_factor * src_len + self.max_len_offset


def ensemble_logprobs(per_model: Sequence[np.ndarray]) -> np.ndarray:
    """Mean of log-prob arrays taken about the first member (search.py:56-72):
    k identical inputs return that input bitwise."""
    if len(per_model) == 0:
        raise ValueError("ensemble requires at least one model output")
    arrays = [np.asarray(a, dtype=np.float64) for a in per_model]
    shapes = {a.shape for a in arrays}
    if len(shapes) != 1:
        raise ValueError(f"mismatched log-prob array shapes: {sorted(shapes)}")
    stack = np.stack(arrays)
    return stack[0] + (stack - stack[0][None]).mean(axis=0)


def validate_models(models: Sequence[ModelParams]) -> None:
    if len(models) == 0:
        raise ValueError("at least one model is required")
    head = (models[0].config.v_src, models[0].config.v_trg)
    for m in models[1:]:
        this = (m.config.v_src, m.config.v_trg)
        if this != head:
            raise ValueError(f"model vocabulary mismatch: {this} vs {head}")


def validate_request(models: Sequence[ModelParams], src_ids: Sequence[int], opts: DecodeOptions,
                     shortlist: "ShortList | None") -> np.ndarray | None:
    """Reference argument checks (search.py:132-149, nnet.py:167-174)."""
    validate_models(models)
    if len(src_ids) == 0:
        raise ValueError("cannot decode an empty source sentence")
    if opts.beam_size < 1:
        raise ValueError(f"beam_size must be >= 1, got {opts.beam_size}")
    if opts.n_best < 1:
        raise ValueError(f"n_best must be >= 1, got {opts.n_best}")
    cap = opts.max_target_len(len(src_ids))
    if cap < 1:
        raise ValueError(f"length cap {cap} must be >= 1")
    v_src = models[0].config.v_src
    for pos, i in enumerate(src_ids):
        if not 0 <= i < v_src:
            raise ValueError(f"token id {i} at position {pos} out of range for table with {v_src} rows")
    if shortlist is None:
        return None
    sl = np.asarray(shortlist.global_ids, dtype=np.int64)
    v_trg = models[0].config.v_trg
    if int(sl[-1]) >= v_trg:
        raise ValueError(f"shortlist id {int(sl[-1])} out of range for v_trg={v_trg}")
    return sl


def to_hypotheses(raw) -> list[Hypothesis]:
    return [Hypothesis(tokens=toks, score=score,
                       states=[] if st is None else [DecoderState(np.asarray(x, np.float64)) for x in st],
                       finished=fin) for toks, score, fin, st in raw]


def beam_search(models: Sequence[ModelParams], src_ids: Sequence[int], opts: DecodeOptions = DecodeOptions(),
                shortlist: "ShortList | None" = None, device: int = 0) -> list[Hypothesis]:
    """Decode one sentence on the device, returning up to n_best hypotheses."""
    sl = validate_request(models, src_ids, opts, shortlist)
    dms = [_lib.device_model(m, device) for m in models]
    out = _lib.decode(dms, [list(src_ids)], opts.beam_size, opts.max_len_factor, opts.max_len_offset,
                      opts.length_normalize, opts.n_best, shortlists=None if sl is None else [sl],
                      want_states=True, max_batch=1)
    return to_hypotheses(out.hyps(0))


def exhaustive_search(models: Sequence[ModelParams], src_ids: Sequence[int], cap: int) -> Hypothesis:
    """Full enumeration over the device step hook (search.py:219-277);
    verification oracle for tiny models only."""
    validate_models(models)
    if len(src_ids) == 0:
        raise ValueError("cannot decode an empty source sentence")
    if cap < 1:
        raise ValueError(f"length cap {cap} must be >= 1")
    v_trg = models[0].config.v_trg
    space = v_trg**cap
    if space > EXHAUSTIVE_GUARD:
        raise ValueError(f"search space v_trg^cap = {v_trg}^{cap} = {space} exceeds the "
                         f"{EXHAUSTIVE_GUARD} guard")
    fwds = [Forward.for_params(m) for m in models]
    anns = [f.encode(list(src_ids)) for f in fwds]
    best: list = [None, None]  # finished, unfinished

    def offer(slot, score, seq, states):
        cur = best[slot]
        if cur is None or score > cur[0] or (score == cur[0] and seq < cur[1]):
            best[slot] = (score, seq, states)

    def grow(prefix, score, prev, states):
        outs = [f.step_rows(s, np.array([prev]), a) for f, s, a in zip(fwds, states, anns)]
        nxt = [o[0] for o in outs]
        row = ensemble_logprobs([o[1][0] for o in outs])
        offer(0, score + float(row[EOS_ID]), prefix + [EOS_ID], nxt)
        last = len(prefix) + 1 >= cap
        for tok in range(1, v_trg):
            if last:
                offer(1, score + float(row[tok]), prefix + [tok], nxt)
            else:
                grow(prefix + [tok], score + float(row[tok]), tok, nxt)

    grow([], 0.0, EOS_ID, [f.init_state_row(a) for f, a in zip(fwds, anns)])
    slot = 0 if best[0] is not None else 1
    score, seq, states = best[slot]
    return Hypothesis(tokens=seq, score=score, states=[DecoderState(s[0]) for s in states], finished=slot == 0)
