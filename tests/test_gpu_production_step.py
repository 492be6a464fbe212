"""Per-step gates on the PRODUCTION kernels (north_star: per-step
log-probabilities within 1e-3 relative at fp32 accumulation).

`amun_decoder_step_fused` / `amun_encode_batch(production=1)` run exactly
the kernels `amun_decode` runs — tcgen05 3xFP16 GEMMs (query, GRU phase
A/B, deep output; encoder input projection, bi-GRU recurrence,
precomp_att), the fused attention kernel and the fused tensor-core logit
kernel with its per-tile (max, sum exp, top-kk) partials — at the bench's
bucket shapes: 64 sentences x beam 5 (R = 320, cfg2 lengths) and 64 x
beam 12 (R = 768, cfg4's J = 100).  The f64 oracle (oracle/, pinned to the
reference's fixtures) is the checker: reference nnet.py:143-164 (step),
tensor.py:79-92 (log-softmax), search.py:169 (per-row candidates).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import full_model

pytestmark = pytest.mark.gpu

LOGP_RTOL = 1e-3   # north_star gate
TAU = 1e-4         # near-tie threshold for candidate-order differences


@pytest.fixture(scope="module")
def full():
    return full_model()


@pytest.fixture(scope="module")
def net():
    from oracle import beamnmt_oracle as orc

    return orc.Net({n: a for n, a in full_model().tensor_items()})


def _sample(name: str, n: int):
    from paper_1610_01108_b200 import workload as W

    corpus = W.WORKLOADS[name].corpus()
    order = sorted(range(len(corpus)), key=lambda i: (len(corpus[i]), i))
    stride = max(1, len(order) // n)
    return [corpus[i] for i in order[stride // 2::stride][:n]]


def _pad(anns, jmax, width, attr):
    out = np.zeros((len(anns), jmax, width), np.float32)
    for b, a in enumerate(anns):
        v = getattr(a, attr)
        out[b, : v.shape[0]] = v
    return out


def _topk_ref(lp_row: np.ndarray, kk: int):
    order = np.lexsort((np.arange(lp_row.size), -lp_row))[: kk + 1]
    return order[:kk], lp_row[order]


@pytest.mark.parametrize("cfg,k,n_sent", [("cfg2", 5, 64), ("cfg4", 12, 64), ("cfg2", 9, 8), ("cfg2", 9, 1)])
def test_production_step_logprobs(gpu, full, net, cfg, k, n_sent):
    """>= 2 x n_sent x k full-size decoder states (two consecutive steps of
    beam-like rows per sentence) through the production step kernels."""
    from paper_1610_01108_b200 import _lib

    sents = _sample(cfg, n_sent)
    anns = [net.encode(s) for s in sents]
    lens = [len(s) for s in sents]
    jmax = max(lens)
    H = _pad(anns, jmax, 2 * net.d_h, "h")
    P = _pad(anns, jmax, net.W_att_h.shape[1], "precomp")
    # step-1 states (all k rows from s0 after </s>), then k distinct
    # continuations per sentence: the rows of a real beam after one step
    s_rows, y_rows = [], []
    for a in anns:
        s1, lp1, _ = net.step(net.init_state(a), np.array([0]), a)
        top, _ = _topk_ref(lp1[0], k)
        s_rows.append(np.repeat(s1, k, axis=0))
        y_rows.append(top)
    s = np.concatenate(s_rows)
    y = np.concatenate(y_rows)
    dm = _lib.device_model(full)
    worst_lp = worst_s = 0.0
    n_rows = n_tie = 0
    for step in range(2):
        ref_s, ref_lp = [], []
        for b, a in enumerate(anns):
            sn, lp, _ = net.step(s[b * k:(b + 1) * k], y[b * k:(b + 1) * k], a)
            ref_s.append(sn)
            ref_lp.append(lp)
        ref_s = np.concatenate(ref_s)
        ref_lp = np.concatenate(ref_lp)
        s_gpu, lse, tok, lp = dm.step_fused(s.astype(np.float32), y, H, P, lens, k, k)
        worst_s = max(worst_s, float(np.max(np.abs(s_gpu - ref_s))))
        np.testing.assert_allclose(s_gpu, ref_s, atol=1e-5)
        for r in range(s.shape[0]):
            want_tok, want_lp = _topk_ref(ref_lp[r], k)
            got_ref = ref_lp[r][tok[r]]  # the reference's log-prob of every token the kernel chose
            rel = np.max(np.abs(lp[r] - got_ref) / np.abs(got_ref))
            worst_lp = max(worst_lp, float(rel))
            assert rel < LOGP_RTOL, (cfg, step, r, rel)
            if not np.array_equal(tok[r], want_tok):
                # only a near tie at the boundary or inside the list may reorder
                gaps = np.abs(np.diff(want_lp))
                assert gaps.min() < TAU, (cfg, step, r, tok[r], want_tok, want_lp)
                n_tie += 1
            n_rows += 1
        # next step: every row continues with its own best token
        s = ref_s
        y = np.array([int(_topk_ref(ref_lp[r], 1)[0][0]) for r in range(ref_lp.shape[0])])
    print(f"\n{cfg}: {n_rows} full-size states at R={n_sent * k}: candidate log-prob max rel err "
          f"{worst_lp:.2e}, state max abs err {worst_s:.2e}, {n_tie} near-tie reorderings")
    assert worst_lp < 1e-5  # FP32-equivalent, far inside the 1e-3 gate


def test_production_encoder_matches_oracle(gpu, full, net):
    """Tensor-core encoder (input projection, bi-GRU recurrence with the
    block-row layout, precomp_att) on a 64-sentence bucket of mixed lengths
    vs the f64 oracle; the FP32 CUDA-core encoder alongside."""
    from paper_1610_01108_b200 import _lib

    sents = _sample("cfg2", 64)
    dm = _lib.device_model(full)
    h, p, s0 = dm.encode_batch(sents, production=True)
    hf, pf, s0f = dm.encode_batch(sents, production=False)
    worst = {"h": 0.0, "p": 0.0, "s0": 0.0}
    for b, src in enumerate(sents):
        a = net.encode(src)
        J = len(src)
        worst["h"] = max(worst["h"], float(np.max(np.abs(h[b, :J] - a.h))))
        worst["p"] = max(worst["p"], float(np.max(np.abs(p[b, :J] - a.precomp))))
        worst["s0"] = max(worst["s0"], float(np.max(np.abs(s0[b] - net.init_state(a)[0]))))
        assert not np.any(h[b, J:]), "padded positions must stay zero"
        np.testing.assert_allclose(hf[b, :J], a.h, atol=5e-5)
    print(f"\ntensor-core encoder vs f64 oracle, max abs err: {worst}")
    assert worst["h"] < 5e-5 and worst["p"] < 5e-5 and worst["s0"] < 5e-5, worst
