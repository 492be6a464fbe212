"""ctypes binding of the C ABI in include/amun_b200.h (libamun_b200.so).

This is the only way the package reaches the device: there is no CPU
fallback.  If the shared library is missing or no CUDA device is visible the
calls raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import queue
import threading
import time
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import ShapeError

LIB_NAME = "libamun_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

AMUN_OK, AMUN_ERR_INVALID, AMUN_ERR_CUDA, AMUN_ERR_OOM, AMUN_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

# Every symbol include/amun_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "amun_last_error", "amun_version", "amun_device_count", "amun_model_create", "amun_model_destroy",
    "amun_model_device_bytes", "amun_decode", "amun_result_free", "amun_encode", "amun_attention",
    "amun_decoder_step", "amun_init_state", "amun_gru_cell", "amun_decode_stream", "amun_encode_batch",
    "amun_decoder_step_fused", "amun_vocab_create", "amun_vocab_destroy", "amun_vocab_encode",
)

_i32, _i64, _f32p, _f64p, _i32p = ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_float), \
    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)


class Dims(ctypes.Structure):
    _fields_ = [("v_src", _i32), ("v_trg", _i32), ("d_emb", _i32), ("d_h", _i32), ("d_att", _i32)]


class DecodeOpts(ctypes.Structure):
    _fields_ = [("beam_size", _i32), ("max_len_factor", _i32), ("max_len_offset", _i32),
                ("length_normalize", _i32), ("n_best", _i32), ("want_states", _i32), ("max_batch", _i32),
                ("force_full_logits", _i32), ("profile", _i32)]


class Result(ctypes.Structure):
    _fields_ = [("n_sent", _i32), ("n_models", _i32), ("d_h", _i32), ("n_hyp", _i64),
                ("hyp_offsets", _i32p), ("scores", _f64p), ("finished", _i32p),
                ("tok_offsets", ctypes.POINTER(ctypes.c_int64)), ("tokens", _i32p), ("states", _f32p),
                ("decoder_steps", _i64), ("kernel_launches", _i64), ("device_ms", ctypes.c_double),
                ("h2d_bytes", _i64), ("d2h_bytes", _i64), ("kernel_ms", ctypes.c_double * 8),
                ("kernel_count", _i64 * 8), ("host_setup_ms", ctypes.c_double), ("host_post_ms", ctypes.c_double),
                ("kernel_ctas", _i64 * 8)]

# void (*)(void *user, const amun_result *partial, const int32_t *idx)
BUCKET_DONE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(Result), _i32p)

KERNEL_CLASSES = ("encoder", "query", "attention", "gru_a", "gru_b", "deep_out", "logits", "select")
# DecodeOpts.profile flag (include/amun_b200.h AMUN_PROFILE_CTA_TIME): device
# CTA-lifetime accounting per kernel class in the normal multi-lane graph mode
PROFILE_CTA_TIME = 0x40000000


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("AMUN_B200_LIB", LIB_PATH))
        if not path.exists():
            raise RuntimeError(f"{path} not found: build the CUDA extension first "
                               "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(str(path))
        lib.amun_last_error.restype = ctypes.c_char_p
        lib.amun_version.restype = ctypes.c_int
        lib.amun_device_count.argtypes = [_i32p]
        lib.amun_model_create.argtypes = [_i32, ctypes.POINTER(Dims), ctypes.POINTER(_f32p), _i32,
                                          ctypes.POINTER(ctypes.c_void_p)]
        lib.amun_model_destroy.argtypes = [ctypes.c_void_p]
        lib.amun_model_device_bytes.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        lib.amun_decode.argtypes = [ctypes.POINTER(ctypes.c_void_p), _i32, _i32p, _i32p, _i32, _i32p, _i32p,
                                    ctypes.POINTER(DecodeOpts), ctypes.POINTER(ctypes.POINTER(Result))]
        lib.amun_result_free.argtypes = [ctypes.POINTER(Result)]
        lib.amun_decode_stream.argtypes = [ctypes.POINTER(ctypes.c_void_p), _i32, _i32p, _i32p, _i32, _i32p, _i32p,
                                           ctypes.POINTER(DecodeOpts), BUCKET_DONE, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.POINTER(Result))]
        lib.amun_encode.argtypes = [ctypes.c_void_p, _i32p, _i32, _f32p, _f32p, _f32p]
        lib.amun_attention.argtypes = [ctypes.c_void_p, _f32p, _i32, _f32p, _f32p, _i32, _f32p, _f32p]
        lib.amun_decoder_step.argtypes = [ctypes.c_void_p, _f32p, _i32p, _i32, _f32p, _f32p, _i32, _i32p, _i32,
                                          _f32p, _f64p, _f32p]
        lib.amun_init_state.argtypes = [ctypes.c_void_p, _f32p, _i32, _f32p]
        lib.amun_gru_cell.argtypes = [_i32, _i32, _i32, ctypes.POINTER(_f32p), ctypes.POINTER(_f32p),
                                      ctypes.POINTER(_f32p), _i32, _f32p, _f32p, _f32p]
        lib.amun_encode_batch.argtypes = [ctypes.c_void_p, _i32p, _i32p, _i32, _i32, _i32, _f32p, _f32p, _f32p]
        lib.amun_decoder_step_fused.argtypes = [ctypes.c_void_p, _i32, _i32, _f32p, _i32p, _f32p, _f32p, _i32p,
                                                _i32, _i32, _f32p, _f32p, _f32p, _f32p, _i32p, _f32p]
        for name in EXPORTS:
            if name not in ("amun_last_error", "amun_version", "amun_model_destroy", "amun_result_free",
                            "amun_vocab_destroy"):
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == AMUN_OK:
        return
    msg = load().amun_last_error().decode("utf-8", "replace")
    if status == AMUN_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"amun_b200 error {status}: {msg}")


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(load().amun_device_count(ctypes.byref(n)))
    return n.value


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray, ty):
    return a.ctypes.data_as(ty)


class DeviceModel:
    """A model uploaded to one device (replaces Forward.for_params)."""

    def __init__(self, params, device: int = 0):
        lib = load()
        cfg = params.config
        self.config = cfg
        self.device = device
        arrays = [_f32(a) for _, a in params.tensor_items()]
        ptrs = (_f32p * len(arrays))(*[_ptr(a, _f32p) for a in arrays])
        dims = Dims(*cfg.dims)
        h = ctypes.c_void_p()
        check(lib.amun_model_create(device, ctypes.byref(dims), ptrs, len(arrays), ctypes.byref(h)))
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None):
            load().amun_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_bytes(self) -> int:
        n = ctypes.c_int64(0)
        check(load().amun_model_device_bytes(self.handle, ctypes.byref(n)))
        return n.value

    # ---- per-step hooks
    def encode(self, ids: Sequence[int]) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        cfg = self.config
        ids_a = np.ascontiguousarray(ids, dtype=np.int32)
        J = ids_a.size
        h = np.empty((J, 2 * cfg.d_h), np.float32)
        p = np.empty((J, cfg.d_att), np.float32)
        s0 = np.empty(cfg.d_h, np.float32)
        check(load().amun_encode(self.handle, _ptr(ids_a, _i32p), J, _ptr(h, _f32p), _ptr(p, _f32p),
                                 _ptr(s0, _f32p)))
        return h, p, s0

    def init_state(self, h: np.ndarray) -> np.ndarray:
        h = _f32(h)
        if h.ndim != 2 or h.shape[1] != 2 * self.config.d_h:
            raise ShapeError(f"annotations have shape {h.shape}, expected (J, {2 * self.config.d_h})")
        s0 = np.empty(self.config.d_h, np.float32)
        check(load().amun_init_state(self.handle, _ptr(h, _f32p), h.shape[0], _ptr(s0, _f32p)))
        return s0

    def attention(self, s: np.ndarray, h: np.ndarray, p: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        s, h, p = _f32(np.atleast_2d(s)), _f32(h), _f32(p)
        R, J = s.shape[0], h.shape[0]
        self._check_rows(s, h, p)
        alpha = np.empty((R, J), np.float32)
        ctx = np.empty((R, 2 * self.config.d_h), np.float32)
        check(load().amun_attention(self.handle, _ptr(s, _f32p), R, _ptr(h, _f32p), _ptr(p, _f32p), J,
                                    _ptr(alpha, _f32p), _ptr(ctx, _f32p)))
        return alpha, ctx

    def step(self, s: np.ndarray, y_prev: Sequence[int], h: np.ndarray, p: np.ndarray,
             shortlist: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        s, h, p = _f32(np.atleast_2d(s)), _f32(h), _f32(p)
        y = np.ascontiguousarray(y_prev, dtype=np.int32).reshape(-1)
        R, J = s.shape[0], h.shape[0]
        self._check_rows(s, h, p)
        if y.size != R:
            raise ShapeError(f"{y.size} previous tokens for {R} state rows")
        sl = None if shortlist is None else np.ascontiguousarray(shortlist, dtype=np.int32)
        n = self.config.v_trg if sl is None else sl.size
        s_out = np.empty((R, self.config.d_h), np.float32)
        logp = np.empty((R, n), np.float64)
        alpha = np.empty((R, J), np.float32)
        check(load().amun_decoder_step(self.handle, _ptr(s, _f32p), _ptr(y, _i32p), R, _ptr(h, _f32p),
                                       _ptr(p, _f32p), J, None if sl is None else _ptr(sl, _i32p),
                                       0 if sl is None else sl.size, _ptr(s_out, _f32p), _ptr(logp, _f64p),
                                       _ptr(alpha, _f32p)))
        return s_out, logp, alpha

    # ---- production-kernel hooks (the tensor-core kernels amun_decode runs)
    def encode_batch(self, sentences: Sequence[Sequence[int]], production: bool = True):
        """Encoder + initial state of B sentences as one padded bucket:
        returns h [B, jmax, 2 d_h], p [B, jmax, d_att], s0 [B, d_h]."""
        cfg = self.config
        lens = np.asarray([len(s) for s in sentences], np.int32)
        B, jmax = lens.size, int(lens.max())
        ids = np.zeros((B, jmax), np.int32)
        for b, s in enumerate(sentences):
            ids[b, :len(s)] = s
        h = np.empty((B, jmax, 2 * cfg.d_h), np.float32)
        p = np.empty((B, jmax, cfg.d_att), np.float32)
        s0 = np.empty((B, cfg.d_h), np.float32)
        check(load().amun_encode_batch(self.handle, _ptr(ids, _i32p), _ptr(lens, _i32p), B, jmax, int(production),
                                       _ptr(h, _f32p), _ptr(p, _f32p), _ptr(s0, _f32p)))
        return h, p, s0

    def step_fused(self, s: np.ndarray, y_prev: Sequence[int], h: np.ndarray, p: np.ndarray,
                   lens: Sequence[int], k: int, kk: int):
        """One decoder step of B sentences x k rows on the production kernels.
        Returns s' [R, d_h], the per-row log-normaliser lse [R] (f64, merged
        from the logit kernel's per-tile partials the way the select kernel
        merges them) and the row's kk best candidates (tokens [R, kk],
        log-probs [R, kk], ordered by (log-prob desc, token asc))."""
        cfg = self.config
        s, h, p = _f32(np.atleast_2d(s)), _f32(h), _f32(p)
        y = np.ascontiguousarray(y_prev, dtype=np.int32).reshape(-1)
        lens_a = np.ascontiguousarray(lens, dtype=np.int32)
        B, jmax = h.shape[0], h.shape[1]
        R = B * k
        if s.shape != (R, cfg.d_h) or y.size != R or lens_a.size != B:
            raise ShapeError(f"{s.shape} states / {y.size} tokens for {B} sentences x {k} rows")
        if h.shape != (B, jmax, 2 * cfg.d_h) or p.shape != (B, jmax, cfg.d_att):
            raise ShapeError(f"annotations have shapes {h.shape} / {p.shape}")
        nt = -(-cfg.v_trg // 128)
        s_out = np.empty((R, cfg.d_h), np.float32)
        pmax = np.empty((R, nt), np.float32)
        psum = np.empty((R, nt), np.float32)
        cval = np.empty((R, nt, kk), np.float32)
        ctok = np.empty((R, nt, kk), np.int32)
        check(load().amun_decoder_step_fused(self.handle, B, k, _ptr(s, _f32p), _ptr(y, _i32p), _ptr(h, _f32p),
                                             _ptr(p, _f32p), _ptr(lens_a, _i32p), jmax, kk, _ptr(s_out, _f32p),
                                             _ptr(pmax, _f32p), _ptr(psum, _f32p), _ptr(cval, _f32p),
                                             _ptr(ctok, _i32p), None))
        # select-kernel merge (kernels.cu select phase 1): M = max_t pmax_t,
        # lse = M + log sum_t psum_t exp(pmax_t - M), summed in f64
        mx = pmax.max(axis=1)
        lse = mx.astype(np.float64) + np.log((psum * np.exp(pmax - mx[:, None])).astype(np.float64).sum(axis=1))
        flat_v = cval.reshape(R, -1).astype(np.float64)
        flat_t = ctok.reshape(R, -1)
        tok = np.empty((R, kk), np.int64)
        lp = np.empty((R, kk), np.float64)
        for r in range(R):
            ok = flat_t[r] >= 0
            order = np.lexsort((flat_t[r][ok], -flat_v[r][ok]))[:kk]
            tok[r] = flat_t[r][ok][order]
            lp[r] = flat_v[r][ok][order] - lse[r]
        return s_out, lse, tok, lp

    def _check_rows(self, s, h, p):
        cfg = self.config
        if s.shape[1] != cfg.d_h:
            raise ShapeError(f"state has shape {s.shape}, expected (*, {cfg.d_h})")
        if h.ndim != 2 or h.shape[1] != 2 * cfg.d_h or p.shape != (h.shape[0], cfg.d_att):
            raise ShapeError(f"annotations have shapes {h.shape} / {p.shape}")


def gru_cell(g, x: np.ndarray, h: np.ndarray, device: int = 0) -> np.ndarray:
    """One GRU update for rows x [R, d_in], h [R, d_h] on the device."""
    x, h = _f32(np.atleast_2d(x)), _f32(np.atleast_2d(h))
    W = [_f32(g.W_z), _f32(g.W_r), _f32(g.W_h)]
    U = [_f32(g.U_z), _f32(g.U_r), _f32(g.U_h)]
    b = [_f32(g.b_z).reshape(-1), _f32(g.b_r).reshape(-1), _f32(g.b_h).reshape(-1)]
    arr = lambda xs: (_f32p * 3)(*[_ptr(a, _f32p) for a in xs])
    out = np.empty_like(h)
    check(load().amun_gru_cell(device, g.d_in, g.d_h, arr(W), arr(U), arr(b), x.shape[0], _ptr(x, _f32p),
                               _ptr(h, _f32p), _ptr(out, _f32p)))
    return out


def device_model(params, device: int = 0) -> DeviceModel:
    """Per-(model, device) handle cached on the ModelParams object."""
    cache = params._device_cache
    dm = cache.get(device)
    if dm is None:
        dm = DeviceModel(params, device)
        cache[device] = dm
    return dm


class DecodeOut:
    """Flat copy of an amun_result: per sentence, ranked hypotheses."""

    def __init__(self, res: Result, want_states: bool, state_widths: Sequence[int] = ()):
        # states: per hypothesis the ensemble members' final state rows
        # concatenated (member m has width state_widths[m] = its d_h)
        widths = list(state_widths) or [res.d_h] * res.n_models
        self.state_splits = np.cumsum(widths)[:-1]
        nh = res.n_hyp
        self.n_sent = res.n_sent
        self.hyp_offsets = np.ctypeslib.as_array(res.hyp_offsets, shape=(res.n_sent + 1,)).copy()
        if nh:
            self.scores = np.ctypeslib.as_array(res.scores, shape=(nh,)).copy()
            self.finished = np.ctypeslib.as_array(res.finished, shape=(nh,)).astype(bool)
            self.tok_offsets = np.ctypeslib.as_array(res.tok_offsets, shape=(nh + 1,)).copy()
            nt = int(self.tok_offsets[-1])
            self.tokens = np.ctypeslib.as_array(res.tokens, shape=(max(nt, 1),))[:nt].copy()
            self.states = (np.ctypeslib.as_array(res.states, shape=(nh, int(sum(widths)))).copy()
                           if want_states else None)
        else:
            self.scores = np.zeros(0)
            self.finished = np.zeros(0, bool)
            self.tok_offsets = np.zeros(1, np.int64)
            self.tokens = np.zeros(0, np.int32)
            self.states = None
        self.decoder_steps = res.decoder_steps
        self.kernel_launches = res.kernel_launches
        self.device_ms = res.device_ms
        self.host_setup_ms = res.host_setup_ms
        self.host_post_ms = res.host_post_ms
        self.h2d_bytes = res.h2d_bytes
        self.d2h_bytes = res.d2h_bytes
        self.kernel_ms = {k: res.kernel_ms[i] for i, k in enumerate(KERNEL_CLASSES)}
        self.kernel_count = {k: res.kernel_count[i] for i, k in enumerate(KERNEL_CLASSES)}
        self.kernel_ctas = {k: res.kernel_ctas[i] for i, k in enumerate(KERNEL_CLASSES)}

    def hyps(self, i: int):
        """[(tokens list, score, finished, states or None)] for sentence i."""
        out = []
        tok = self.tokens
        for h in range(self.hyp_offsets[i], self.hyp_offsets[i + 1]):
            a, b = self.tok_offsets[h], self.tok_offsets[h + 1]
            out.append((tok[a:b].tolist(), float(self.scores[h]), bool(self.finished[h]),
                        None if self.states is None else np.split(self.states[h], self.state_splits)))
        return out


def decode(models: Sequence[DeviceModel], sentences: Sequence[Sequence[int]], beam_size: int,
           max_len_factor: int, max_len_offset: int, length_normalize: bool, n_best: int,
           shortlists: Sequence[np.ndarray] | None = None, want_states: bool = False, max_batch: int = 64,
           force_full_logits: bool = False, profile: bool = False, on_bucket=None,
           flat: tuple[np.ndarray, np.ndarray] | None = None) -> DecodeOut:
    """Decode a batch of sentences (lists of source ids), or with `flat` =
    (ids, lens) the already concatenated ids and per-sentence lengths."""
    lib = load()
    if flat is not None:
        ids = np.ascontiguousarray(flat[0], dtype=np.int32)
        lens = np.ascontiguousarray(flat[1], dtype=np.int32)
    else:
        lens = np.asarray([len(s) for s in sentences], dtype=np.int32)
        ids = (np.concatenate([np.asarray(s, dtype=np.int32) for s in sentences]) if len(sentences)
               else np.zeros(0, np.int32))
        ids = np.ascontiguousarray(ids, dtype=np.int32)
    sl_ids = sl_len = None
    if shortlists is not None:
        sl_len = np.asarray([len(s) for s in shortlists], dtype=np.int32)
        sl_ids = np.ascontiguousarray(np.concatenate([np.asarray(s, np.int32) for s in shortlists]), np.int32)
    handles = (ctypes.c_void_p * len(models))(*[m.handle for m in models])
    widths = [m.config.d_h for m in models]
    opts = DecodeOpts(beam_size, max_len_factor, max_len_offset, int(length_normalize), n_best, int(want_states),
                      max_batch, int(force_full_logits), int(profile))
    res = ctypes.POINTER(Result)()
    t_call = time.perf_counter()
    sl_p = None if sl_ids is None else _ptr(sl_ids, _i32p)
    sl_l = None if sl_len is None else _ptr(sl_len, _i32p)
    if on_bucket is None:
        check(lib.amun_decode(handles, len(models), _ptr(ids, _i32p), _ptr(lens, _i32p), len(lens), sl_p, sl_l,
                              ctypes.byref(opts), ctypes.byref(res)))
    else:
        # finished buckets are handed to on_bucket(sentence indices, DecodeOut)
        # while later buckets still decode.  The library's callback only
        # copies the bucket's results and queues them: on_bucket runs on a
        # consumer thread, so the native decode loop (which feeds every lane
        # its next steps) is never held up by the caller's post-processing.
        # An exception inside on_bucket is re-raised after the call (ctypes
        # cannot propagate it through C).
        errors: list[BaseException] = []
        done_q: queue.SimpleQueue = queue.SimpleQueue()

        def _cb(_user, part, idx):
            if errors:
                return
            try:
                out = DecodeOut(part.contents, want_states, widths)
                done_q.put((np.ctypeslib.as_array(idx, shape=(out.n_sent,)).copy(), out))
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errors.append(e)

        def _consume():
            while True:
                item = done_q.get()
                if item is None:
                    return
                if errors:
                    continue
                try:
                    on_bucket(*item)
                except BaseException as e:  # noqa: BLE001 - re-raised below
                    errors.append(e)

        consumer = threading.Thread(target=_consume, name="amun-bucket-consumer", daemon=True)
        consumer.start()
        cb = BUCKET_DONE(_cb)
        try:
            check(lib.amun_decode_stream(handles, len(models), _ptr(ids, _i32p), _ptr(lens, _i32p), len(lens),
                                         sl_p, sl_l, ctypes.byref(opts), cb, None, ctypes.byref(res)))
        finally:
            done_q.put(None)
            consumer.join()
        if errors:
            lib.amun_result_free(res)
            raise errors[0]
    t_ret = time.perf_counter()
    try:
        out = DecodeOut(res.contents, want_states, widths)
    finally:
        lib.amun_result_free(res)
    out.call_ms = 1e3 * (t_ret - t_call)  # the C call, wall (vs device_ms inside it)
    return out


class NativeVocab:
    """Host vocabulary handle of the native text front-end (text.cu): maps
    whole corpora of lines to source ids in one call."""

    def __init__(self, tokens: Sequence[str]):
        lib = load()
        enc = [t.encode("utf-8", "surrogatepass") for t in tokens]
        offs = np.zeros(len(enc) + 1, dtype=np.int64)
        np.cumsum([len(b) for b in enc], out=offs[1:])
        buf = b"".join(enc)
        self.handle = ctypes.c_void_p()
        check(lib.amun_vocab_create(buf, _ptr(offs, ctypes.POINTER(ctypes.c_int64)), len(enc),
                                    ctypes.byref(self.handle)))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.amun_vocab_destroy(h)
            self.handle = None

    def encode(self, lines: Sequence[str], lowercase: bool, unk_id: int):
        """(ids int32 [sum lens], lens int32 [n], oov int32 [n]) of the lines,
        split like preprocess() (str.lower() first when lowercase)."""
        enc = [(ln.lower() if lowercase else ln).encode("utf-8", "surrogatepass") for ln in lines]
        offs = np.zeros(len(enc) + 1, dtype=np.int64)
        np.cumsum([len(b) for b in enc], out=offs[1:])
        buf = b"".join(enc)
        ids = np.empty(int(offs[-1]) + 1, dtype=np.int32)  # a token has >= 1 byte
        lens = np.empty(len(enc), dtype=np.int32)
        oov = np.empty(len(enc), dtype=np.int32)
        n = ctypes.c_int64()
        check(load().amun_vocab_encode(self.handle, buf, _ptr(offs, ctypes.POINTER(ctypes.c_int64)), len(enc), unk_id,
                                       _ptr(ids, _i32p), ids.size, _ptr(lens, _i32p), _ptr(oov, _i32p),
                                       ctypes.byref(n)))
        return ids[:n.value], lens, oov
