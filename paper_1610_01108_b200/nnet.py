"""Per-step forward-pass API (reference: beamnmt/nnet.py) backed by the
device kernels.  Same names, argument meaning and validation messages as
the reference; every number is computed by libamun_b200.so on the GPU and
returned as float64 arrays like the reference's.

  embed(table, ids)                      nnet.py:167-174 (host row gather + range check)
  gru_step(g, x, h)                      nnet.py:177-185
  encode(m, src_ids) -> Annotations      nnet.py:188-193
  init_decoder_state(m, a)               nnet.py:196-197
  attention(m, s, a)                     nnet.py:200-203
  decoder_step(m, s, y_prev, a, sl)      nnet.py:206-231
  Forward.for_params(params)             nnet.py:102-108 (device handle)
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import TYPE_CHECKING

import numpy as np

from . import _lib
from .errors import ShapeError
from .model import GruParams, ModelParams

if TYPE_CHECKING:
    from .shortlist import ShortList


@dataclass(eq=False)
class Annotations:
    """Encoder output: h [J, 2 d_h] = [fwd ; bwd], precomp_att = h W_att_h."""

    h: np.ndarray
    precomp_att: np.ndarray
    _s0: np.ndarray | None = field(default=None, repr=False)

    @property
    def length(self) -> int:
        return self.h.shape[0]


@dataclass(eq=False)
class DecoderState:
    s: np.ndarray


def _f64(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


class Forward:
    """Device-resident working copy of one model (replaces the reference's
    float64 `Forward`); cached per (ModelParams, device)."""

    def __init__(self, params: ModelParams, device: int = 0):
        self.config = params.config
        self.dev = _lib.device_model(params, device)

    @classmethod
    def for_params(cls, params: ModelParams, device: int = 0) -> "Forward":
        key = ("forward", device)
        fw = params._device_cache.get(key)
        if fw is None:
            fw = cls(params, device)
            params._device_cache[key] = fw
        return fw

    def encode(self, src_ids: list[int]) -> Annotations:
        if len(src_ids) == 0:
            raise ValueError("cannot encode an empty source sentence")
        h, p, s0 = self.dev.encode(src_ids)
        return Annotations(h=_f64(h), precomp_att=_f64(p), _s0=s0)

    def init_state_row(self, a: Annotations) -> np.ndarray:
        s0 = a._s0 if a._s0 is not None else self.dev.init_state(a.h)
        return _f64(s0).reshape(1, -1)

    def attention_rows(self, s_rows: np.ndarray, a: Annotations) -> tuple[np.ndarray, np.ndarray]:
        alpha, ctx = self.dev.attention(s_rows, a.h, a.precomp_att)
        return _f64(alpha), _f64(ctx)

    def step_rows(self, s_rows: np.ndarray, y_prev: np.ndarray, a: Annotations,
                  shortlist_ids: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        s_next, logp, alpha = self.dev.step(s_rows, y_prev, a.h, a.precomp_att, shortlist_ids)
        return _f64(s_next), logp, _f64(alpha)


def embed(table: np.ndarray, ids) -> np.ndarray:
    """Row gather with the reference's range check (API utility; the device
    path fuses this gather into the encoder / decoder GEMM A-loads)."""
    table = np.asarray(table)
    ids = list(ids)
    n = table.shape[0]
    for pos, i in enumerate(ids):
        if not 0 <= i < n:
            raise ValueError(f"token id {i} at position {pos} out of range for table with {n} rows")
    return table[np.asarray(ids, dtype=np.int64)]


def gru_step(g: GruParams, x: np.ndarray, h: np.ndarray, device: int = 0) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    if x.shape != (g.d_in,):
        raise ShapeError(f"input has shape {x.shape}, cell expects ({g.d_in},)")
    if h.shape != (g.d_h,):
        raise ShapeError(f"state has shape {h.shape}, cell expects ({g.d_h},)")
    return _f64(_lib.gru_cell(g, x.reshape(1, -1), h.reshape(1, -1), device)[0])


def encode(m: ModelParams, src_ids: list[int]) -> Annotations:
    for pos, i in enumerate(src_ids):
        if not 0 <= i < m.config.v_src:
            raise ValueError(f"source id {i} at position {pos} out of range for v_src={m.config.v_src}")
    return Forward.for_params(m).encode(list(src_ids))


def init_decoder_state(m: ModelParams, a: Annotations) -> DecoderState:
    return DecoderState(s=Forward.for_params(m).init_state_row(a)[0])


def attention(m: ModelParams, s: DecoderState, a: Annotations) -> tuple[np.ndarray, np.ndarray]:
    alpha, ctx = Forward.for_params(m).attention_rows(np.asarray(s.s).reshape(1, -1), a)
    return alpha[0], ctx[0]


def decoder_step(m: ModelParams, s: DecoderState, y_prev: int, a: Annotations,
                 shortlist: "ShortList | None" = None) -> tuple[DecoderState, np.ndarray, np.ndarray]:
    v_trg = m.config.v_trg
    if not 0 <= y_prev < v_trg:
        raise ValueError(f"previous token id {y_prev} out of range for v_trg={v_trg}")
    ids = None
    if shortlist is not None:
        ids = shortlist.global_ids
        if len(ids) and int(ids[-1]) >= v_trg:
            raise ValueError(f"shortlist id {int(ids[-1])} out of range for v_trg={v_trg}")
    s_rows, logp, alpha = Forward.for_params(m).step_rows(np.asarray(s.s).reshape(1, -1),
                                                          np.array([y_prev]), a, ids)
    return DecoderState(s=s_rows[0]), logp[0], alpha[0]
