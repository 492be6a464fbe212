"""Parity of the CUDA path (through the C ABI) with the reference: golden
fixtures produced by the reference itself (tests/golden) and the pinned
oracle run on the GPU box.  All tests need a B200.

Gates (north_star): per-step log-probs within 1e-3 relative; token
sequences identical except where the reference's own k-th vs (k+1)-th
candidate gap is < TAU (documented near ties, counted and printed).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import (full_model, fullset_src_sha, golden_full, golden_fullset, golden_tiny, golden_tiny_arrays,
                      tiny_model)
from paper_1610_01108_b200 import _lib
from paper_1610_01108_b200.model import EOS_ID, ModelConfig, ModelParams, random_model, schema
from paper_1610_01108_b200.nnet import decoder_step, encode, gru_step, init_decoder_state, attention
from paper_1610_01108_b200.search import DecodeOptions, beam_search, exhaustive_search
from paper_1610_01108_b200.shortlist import ShortList

pytestmark = pytest.mark.gpu

TAU = 1e-4          # near-tie threshold on the reference's candidate gap
SCORE_RTOL = 1e-5   # tiny models: fp32 vs f64 beam scores
SCORE_RTOL_FULL = 1e-5  # full size: relative error of the summed f64 beam score (|score| up to ~2000)


def _cmp_hyps(got, gold, tol=SCORE_RTOL):
    assert [h.tokens for h in got] == [g["tokens"] for g in gold]
    assert [h.finished for h in got] == [g["finished"] for g in gold]
    for h, g in zip(got, gold):
        assert abs(h.score - g["score"]) <= tol * max(1.0, abs(g["score"])), (h.score, g["score"])


# ------------------------------------------------------------------ tiny goldens

def test_tiny_beam_cases(gpu):
    cases = [c for c in golden_tiny()["cases"] if c["kind"] == "beam"]
    for c in cases:
        m = tiny_model(c["seed"], c["v_src"], c["v_trg"], c["d"])
        beam, f, o, norm, nb = c["opts"]
        got = beam_search([m], c["src"], DecodeOptions(beam, f, o, bool(norm), nb))
        _cmp_hyps(got, c["hyps"])


def test_tiny_exhaustive_equals_full_width_beam(gpu):
    """Acceptance c01 pattern (tests/test_acceptance.py:103-120) with the
    reference's own exhaustive results as the oracle; beam up to 5^4=625
    exercises the general (full-logits) selection path."""
    for c in (c for c in golden_tiny()["cases"] if c["kind"] == "exhaustive"):
        m = tiny_model(c["seed"], c["v_src"], c["v_trg"], c["d"])
        fw = beam_search([m], c["src"], DecodeOptions(beam_size=c["v_trg"] ** c["cap"], max_len_factor=0,
                                                      max_len_offset=c["cap"]))[0]
        ex = c["exhaustive"]
        assert fw.tokens == ex["tokens"]
        assert abs(fw.score - ex["score"]) <= 1e-5
        mine = exhaustive_search([m], c["src"], c["cap"])
        assert mine.tokens == ex["tokens"] and abs(mine.score - ex["score"]) <= 1e-5
        for k in (1, 2, 3, 5):
            hyp = beam_search([m], c["src"], DecodeOptions(beam_size=k, max_len_factor=0, max_len_offset=c["cap"]))[0]
            assert ex["score"] >= hyp.score - 1e-5


def test_tiny_ensembles(gpu):
    for c in (c for c in golden_tiny()["cases"] if c["kind"] == "ensemble"):
        a = tiny_model(c["seeds"][0], c["v_src"], c["v_trg"], c["d"])
        b = tiny_model(c["seeds"][1], c["v_src"], c["v_trg"], c["d"])
        beam, f, o, norm, nb = c["opts"]
        opts = DecodeOptions(beam, f, o, bool(norm), nb)
        _cmp_hyps(beam_search([a] * 4, c["src"], opts), c["copies"])
        _cmp_hyps(beam_search([a, b], c["src"], opts), c["pair"])
        single = beam_search([a], c["src"], opts)
        quad = beam_search([a] * 4, c["src"], opts)
        assert [h.tokens for h in single] == [h.tokens for h in quad]  # c03


def test_tiny_mixed_dim_ensembles(gpu):
    """Members with different d_emb / d_h / d_att (the reference runs one
    Forward per member, search.py:150-152): per-member row strides on the
    device, hypothesis states returned per member with its own width."""
    cases = [c for c in golden_tiny()["cases"] if c["kind"] == "ensemble_mixed"]
    assert cases
    for c in cases:
        ms = [random_model(ModelConfig(*d), s) for d, s in zip(c["dims"], c["seeds"])]
        beam, f, o, norm, nb = c["opts"]
        got = beam_search(ms, c["src"], DecodeOptions(beam, f, o, bool(norm), nb))
        _cmp_hyps(got, c["hyps"])
        for h, gst in zip(got, c["states"]):
            assert [st.s.shape[0] for st in h.states] == [len(x) for x in gst]
            for st, want in zip(h.states, gst):
                np.testing.assert_allclose(st.s, want, rtol=1e-4, atol=1e-5)


def test_tiny_shortlists(gpu):
    for c in (c for c in golden_tiny()["cases"] if c["kind"] == "shortlist"):
        m = tiny_model(c["seed"], c["v_src"], c["v_trg"], c["d"])
        beam, f, o, norm, nb = c["opts"]
        got = beam_search([m], c["src"], DecodeOptions(beam, f, o, bool(norm), nb),
                          shortlist=ShortList(np.array(c["shortlist"])))
        _cmp_hyps(got, c["hyps"])
    # full-coverage shortlist decodes identically (acceptance c04)
    m = random_model(ModelConfig(v_src=15, v_trg=15, d_emb=8, d_h=8, d_att=8), seed=44)
    rng = np.random.default_rng(8)
    for _ in range(10):
        src = [int(i) for i in rng.integers(2, 15, size=rng.integers(1, 6))]
        a = beam_search([m], src, DecodeOptions(beam_size=5))[0]
        b = beam_search([m], src, DecodeOptions(beam_size=5), shortlist=ShortList.full(15))[0]
        assert a.tokens == b.tokens


def test_tiny_step_arrays(gpu):
    arr = golden_tiny_arrays()
    for c in (c for c in golden_tiny()["cases"] if c["kind"] == "step"):
        m = tiny_model(c["seed"], c["v_src"], c["v_trg"], c["d"])
        k = c["key"]
        a = encode(m, c["src"])
        np.testing.assert_allclose(a.h, arr[f"{k}_h"], atol=2e-6)
        np.testing.assert_allclose(a.precomp_att, arr[f"{k}_p"], atol=2e-6)
        s0 = init_decoder_state(m, a)
        np.testing.assert_allclose(s0.s, arr[f"{k}_s0"], atol=2e-6)
        s1, lp1, al1 = decoder_step(m, s0, c["y1"], a)
        np.testing.assert_allclose(lp1, arr[f"{k}_lp1"], atol=1e-5)
        np.testing.assert_allclose(al1, arr[f"{k}_al1"], atol=1e-6)
        s2, lp2, _ = decoder_step(m, s1, c["y2"], a, ShortList(np.array(c["shortlist2"])))
        np.testing.assert_allclose(lp2, arr[f"{k}_lp2"], atol=1e-5)
        np.testing.assert_allclose(s2.s, arr[f"{k}_s2"], atol=2e-6)
        al, ctx = attention(m, s0, a)
        assert abs(al.sum() - 1.0) < 1e-5 and ctx.shape == (2 * c["d"],)


def test_gru_step_matches_scalar_oracle(gpu):
    from oracle import beamnmt_oracle as orc

    m = tiny_model(5, 6, 6, 7)
    rng = np.random.default_rng(3)
    x, h = rng.standard_normal(7), rng.standard_normal(7)
    got = gru_step(m.enc_fwd, x, h)
    g = orc.Gru({f"c.{k}": getattr(m.enc_fwd, k) for k in orc.GRU_PARTS}, "c")
    np.testing.assert_allclose(got, g.rows(x[None], h[None])[0], atol=2e-6)


def test_all_zero_model_ties(gpu):
    cfg = ModelConfig(v_src=5, v_trg=5, d_emb=4, d_h=4, d_att=4)
    zeros = ModelParams.from_tensors(cfg, {n: np.zeros((r, c), np.float32) for n, r, c in schema(cfg)})
    hyps = beam_search([zeros], [2], DecodeOptions(beam_size=3, max_len_factor=0, max_len_offset=2, n_best=3))
    assert [h.tokens for h in hyps] == [[EOS_ID]]
    assert hyps[0].score == pytest.approx(np.log(1 / 5), abs=1e-9)


# ------------------------------------------------------------------ full size

@pytest.fixture(scope="module")
def full():
    return full_model()


@pytest.fixture(scope="module")
def oracle_net():
    from oracle import beamnmt_oracle as orc

    return orc.Net({n: a for n, a in full_model().tensor_items()})


def test_full_size_step_logprobs(gpu, full, oracle_net):
    """Per-step log-probs within 1e-3 relative of the f64 oracle (pinned to
    decoder_step, nnet.py:206) at several decoder states."""
    src = golden_full()["sets"]["cfg1"]["src"][0]
    a_ref = oracle_net.encode(src)
    s = oracle_net.init_state(a_ref)
    a = encode(full, src)
    np.testing.assert_allclose(a.h, a_ref.h, atol=5e-5)
    y = 0
    worst = 0.0
    for step in range(4):
        s_ref, lp_ref, _ = oracle_net.step(s, np.array([y]), a_ref)
        s_gpu, lp, _ = _lib.device_model(full).step(s.astype(np.float32), [y], a_ref.h, a_ref.precomp)
        rel = np.max(np.abs(lp[0] - lp_ref[0]) / np.abs(lp_ref[0]))
        worst = max(worst, rel)
        assert rel < 1e-3
        np.testing.assert_allclose(s_gpu[0], s_ref[0], atol=1e-5)
        y = int(np.argmax(lp_ref[0]))
        s = s_ref
    print(f"\nfull-size per-step logp max relative error {worst:.2e}")
    assert worst < 1e-5  # FP32-equivalent accuracy, far inside the gate


def _decode_set(model, s, max_batch=64, **kw):
    beam, f, o, norm, nb = s["opts"]
    dm = _lib.device_model(model)
    return _lib.decode([dm], s["src"], beam, f, o, bool(norm), 2, max_batch=max_batch, **kw)


def _first_divergence(got, want) -> int:
    """Index of the first differing token (the decode step that emitted it)."""
    for d, (x, y) in enumerate(zip(got, want)):
        if x != y:
            return d
    return min(len(got), len(want))


def _adjudicate(name, gold_hyps, gaps, out, score_rtol=SCORE_RTOL_FULL):
    """Token identity per sentence, except documented near ties.

    A sentence whose 1-best first differs from the reference's at token d is
    excused only if, at some search step t >= d, the reference's k-th vs
    (k+1)-th candidate gap was below the accumulated score error of two
    hypotheses after t + 1 steps, tau(t) = max(TAU, 2 * eps * (t + 1)), where
    eps is the largest per-step score error measured on this run's
    token-identical sentences (|score - reference| / steps; fp32-equivalent
    arithmetic vs the reference's f64 drifts ~1e-5 per step).  Why t >= d: a
    different beam membership at step t (the only thing the k-th/(k+1)-th
    gap governs) changes which prefixes of length t + 1 survive, so the two
    searches' final hypotheses can first differ at a token d <= t, never
    later; a near tie at a step before d cannot explain a divergence at d.
    A final-ranking tie (two best hypotheses within tau) is excused
    likewise.  Exact sentences must match the score to score_rtol."""
    exact, ties, fails, worst, eps = 0, [], [], 0.0, 0.0
    for i, (gtoks, gscore) in enumerate(gold_hyps):
        hyps = out.hyps(i)
        toks, score = hyps[0][0], hyps[0][1]
        if toks == gtoks:
            exact += 1
            rel = abs(score - gscore) / max(1.0, abs(gscore))
            worst = max(worst, rel)
            eps = max(eps, abs(score - gscore) / max(1, len(gtoks)))
            assert rel <= score_rtol, (name, i, score, gscore)
    for i, (gtoks, gscore) in enumerate(gold_hyps):
        hyps = out.hyps(i)
        toks = hyps[0][0]
        if toks == gtoks:
            continue
        d = _first_divergence(toks, gtoks)
        g = np.asarray(gaps[i], np.float64)
        steps = np.arange(g.size)
        taus = np.maximum(TAU, 2.0 * eps * (steps + 1))
        hit = np.flatnonzero((steps >= d) & (g < taus))
        t = int(hit[0]) if hit.size else -1
        final_gap = abs(hyps[0][1] - hyps[1][1]) if len(hyps) > 1 else np.inf
        tau_end = max(TAU, 2.0 * eps * max(1, len(gtoks)))
        ok = t >= 0 or final_gap < tau_end
        (ties if ok else fails).append((i, d, t, float(g[t]) if t >= 0 else None,
                                        round(float(taus[t]), 7) if t >= 0 else None, final_gap))
    n = len(gold_hyps)
    # exceptions: (sentence, first divergent token d, excusing step t >= d, its gap, tau(t), final-rank gap)
    summary = (f"{name}: {exact}/{n} token-identical, {len(ties)} near-tie exceptions {ties}, "
               f"{len(fails)} unexplained {fails[:10]}; max score rel err {worst:.2e}, "
               f"per-step score error eps {eps:.2e}")
    print("\n" + summary)
    assert not fails, summary
    # ~0.1-0.5% of sentences flip on a near tie (cfg2: 15-19 of 4000); every exception is
    # individually excused above, the count only bounds their rate (at least 2 for a set of a few hundred)
    assert len(ties) <= max(2, n // 100), summary
    return exact, ties


@pytest.mark.parametrize("name", ["cfg1", "cfg2_strat64", "cfg4_6", "cfg5_strat64"])
def test_full_size_decode_matches_reference(gpu, full, name):
    s = golden_full()["sets"][name]
    out = _decode_set(full, s)
    gold = [(r["hyps"][0]["tokens"], r["hyps"][0]["score"]) for r in s["results"]]
    gaps = [np.array(r["kth"]) - np.array(r["next"]) for r in s["results"]]
    _adjudicate(name, gold, gaps, out)


@pytest.mark.parametrize("name,max_batch", [("cfg2", 64), ("cfg4", 64), ("cfg5", 512)])
def test_fullset_decode_matches_reference(gpu, full, name, max_batch):
    """The headline workloads in full, decoded exactly as
    bench.py decodes them (same bucket size), against the reference's own
    1-best of every sentence (tests/golden/make_golden_fullset.py),
    including the sentences that stop early on </s>."""
    from paper_1610_01108_b200 import workload as W

    g = golden_fullset(name)
    wl = W.WORKLOADS[name]
    corpus = wl.corpus()
    assert fullset_src_sha(corpus) == str(g["src_sha256"]), "workload generator drifted from the goldens"
    beam, f, o, _, _ = (int(x) for x in g["opts"])
    dm = _lib.device_model(full)
    out = _lib.decode([dm], corpus, beam, f, o, False, 2, max_batch=max_batch)
    n = len(corpus)
    toff, goff = g["tok_off"], g["gap_off"]
    gold = [(g["tokens"][toff[i]:toff[i + 1]].astype(int).tolist(), float(g["score"][i])) for i in range(n)]
    gaps = [g["gap"][goff[i]:goff[i + 1]] for i in range(n)]
    exact, ties = _adjudicate(name, gold, gaps, out)
    early = np.nonzero(g["finished"])[0].tolist()
    tied = {t[0] for t in ties}
    for i in early:  # EOS -> finished list -> stop rules at full size
        h = out.hyps(i)[0]
        assert h[2] and (h[0] == gold[i][0] or i in tied), (name, i, h[0][-5:], gold[i][0][-5:])
    print(f"{name}: early-stopping sentences {early} all reproduced")


def test_batch_composition_invariance(gpu, full):
    """Byte-identical output for any bucket size (the 1/2/4/8-GPU identity
    argument: a sentence's result never depends on its batch-mates)."""
    s = golden_full()["sets"]["cfg2_strat64"]
    sub = dict(s, src=s["src"][:24])
    a = _decode_set(full, sub, max_batch=64)
    b = _decode_set(full, sub, max_batch=5)
    for i in range(24):
        assert a.hyps(i)[0][:2] == b.hyps(i)[0][:2]


def test_tensor_core_logits_match_cuda_core_path(gpu, full, monkeypatch):
    """tcgen05 3xFP16 kernels (logits, decoder-step GEMMs, encoder) vs the
    FP32 CUDA-core kernels on the same decode: identical tokens, scores equal
    to FP32 rounding."""
    s = golden_full()["sets"]["cfg2_strat64"]
    sub = dict(s, src=s["src"][:32])
    a = _decode_set(full, sub)
    monkeypatch.setenv("AMUN_NO_TC", "1")
    b = _decode_set(full, sub)
    for i in range(32):
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0], i
        assert abs(ha[1] - hb[1]) <= 1e-5 * abs(hb[1]), (i, ha[1], hb[1])


def test_tensor_core_logits_tiny_shapes(gpu, monkeypatch):
    """d_emb % 4 == 0 tiny models take the tensor-core path too (one
    partially out-of-bounds 128-wide vocabulary tile, K = 4 or 8)."""
    for seed, v, d in ((1, 5, 4), (2, 7, 8), (3, 200, 8), (4, 300, 12)):
        m = tiny_model(seed, 9, v, d)
        opts = DecodeOptions(beam_size=3, n_best=3)
        a = beam_search([m], [2, 3, 4], opts)
        monkeypatch.setenv("AMUN_NO_TC", "1")
        b = beam_search([m], [2, 3, 4], opts)
        monkeypatch.delenv("AMUN_NO_TC")
        assert [h.tokens for h in a] == [h.tokens for h in b]
        for x, y in zip(a, b):
            assert abs(x.score - y.score) <= 1e-5 * max(1.0, abs(y.score))


def test_fused_and_full_logit_paths_agree(gpu, full):
    s = golden_full()["sets"]["cfg1"]
    sub = dict(s, src=s["src"][:6])
    a = _decode_set(full, sub)
    b = _decode_set(full, sub, force_full_logits=True)
    for i in range(6):
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0]
        assert abs(ha[1] - hb[1]) <= 1e-6 * abs(ha[1])


@pytest.mark.parametrize("knob", ["AMUN_NO_TC_ENC", "AMUN_NO_TC_GEMM", "AMUN_NO_AHEAD"])
def test_tensor_core_encoder_and_step_gemms_match_cuda_core(gpu, full, monkeypatch, knob):
    """One tensor-core subsystem at a time swapped for its FP32 CUDA-core
    version (encoder: input projection, bi-GRU recurrence, precomp_att;
    step: query / GRU / deep-output GEMMs), or the encode-ahead encoder for
    the per-bucket tensor-core encoder: same tokens, scores within FP32
    rounding of each other."""
    s = golden_full()["sets"]["cfg2_strat64"]
    sub = dict(s, src=s["src"][:24])
    a = _decode_set(full, sub)
    monkeypatch.setenv(knob, "1")
    b = _decode_set(full, sub)
    for i in range(24):
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0], (knob, i)
        assert abs(ha[1] - hb[1]) <= 1e-5 * abs(hb[1]), (knob, i, ha[1], hb[1])


def test_engine_translate_corpus_matches_beam_search(gpu):
    """Engine.translate_corpus (batched device decode + vectorised
    detokenisation) equals per-line beam_search + the reference's
    detokenisation (engine.py:175-179): final </s> dropped, BPE "@@" pieces
    joined, n-best order and scores, empty lines, OOV counts."""
    from paper_1610_01108_b200.engine import Engine, EngineConfig
    from paper_1610_01108_b200.model import Vocabulary
    from paper_1610_01108_b200.subword import bpe_join

    m = tiny_model(11, 30, 40, 8)
    src_vocab = Vocabulary.from_tokens([f"s{i}" for i in range(2, 30)])
    trg_vocab = Vocabulary.from_tokens([f"t{i}@@" if i % 3 == 0 else f"t{i}" for i in range(2, 40)])
    cfg = EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>",
                       beam_size=4, n_best=3, max_len_factor=1, max_len_offset=6, lowercase=False)
    eng = Engine(cfg, [m], src_vocab, trg_vocab, None, None, None, 0, 0.0)
    rng = np.random.default_rng(5)
    lines = [" ".join(f"s{int(i)}" for i in rng.integers(2, 30, size=int(rng.integers(1, 9)))) for _ in range(40)]
    lines[3] = ""
    lines[7] = "s4 unknownword s5"
    res = eng.translate_corpus(lines)
    opts = DecodeOptions(beam_size=4, n_best=3, max_len_factor=1, max_len_offset=6)
    for line, r in zip(lines, res):
        if not line.split():
            assert r.text == "" and r.score == 0.0
            continue
        ids = src_vocab.ids(line.split())
        want = beam_search([m], ids, opts)
        texts = []
        for h in want:
            toks = h.tokens[:-1] if h.finished and h.tokens and h.tokens[-1] == EOS_ID else h.tokens
            texts.append(" ".join(bpe_join([trg_vocab.tokens[i] for i in toks])))
        assert [t for _, t in r.n_best] == texts
        assert [s for s, _ in r.n_best] == [h.score for h in want]
        assert r.oov == sum(1 for t in line.split() if t not in src_vocab)


def test_full_size_shortlist_fused_matches_full_logit_path(gpu, full, monkeypatch):
    """Per-sentence shortlists (nnet.py:160-163) on the fused tensor-core
    logit kernel (vocabulary masks) vs the full-logit CUDA-core path: same
    tokens, scores within FP32 rounding."""
    s = golden_full()["sets"]["cfg1"]
    src = s["src"][:12]
    rng = np.random.default_rng(17)
    sls = [np.unique(np.concatenate([[0], rng.choice(np.arange(2, 30000), 1249, replace=False)])).astype(np.int32)
           for _ in src]
    dm = _lib.device_model(full)
    a = _lib.decode([dm], src, 5, 2, 10, False, 2, shortlists=sls)
    monkeypatch.setenv("AMUN_NO_TC", "1")
    b = _lib.decode([dm], src, 5, 2, 10, False, 2, shortlists=sls)
    for i in range(len(src)):
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0], i
        assert set(ha[0]) <= set(sls[i].tolist())
        assert abs(ha[1] - hb[1]) <= 1e-5 * abs(hb[1]), (i, ha[1], hb[1])


def test_beam12_long_sentences_tensor_core_vs_cuda_core(gpu, full, monkeypatch):
    """cfg4 shape (beam 12, J = 100 golden sentences): the tensor-core path
    (R = 72 rows, two MMA sub-blocks, fused attention with 12 rows) against
    the FP32 CUDA-core kernels."""
    s = golden_full()["sets"]["cfg4_6"]
    sub = dict(s, src=s["src"][:3])
    a = _decode_set(full, sub)
    monkeypatch.setenv("AMUN_NO_TC", "1")
    b = _decode_set(full, sub)
    for i in range(3):
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0], i
        assert abs(ha[1] - hb[1]) <= 1e-5 * abs(hb[1]), (i, ha[1], hb[1])


def test_shortlist_batch_composition_invariance(gpu, full, monkeypatch):
    """Masked fused logits: a sentence's result does not depend on its
    bucket-mates or the bucket size."""
    s = golden_full()["sets"]["cfg1"]
    src = s["src"][:10]
    rng = np.random.default_rng(23)
    sls = [np.unique(np.concatenate([[0], rng.choice(np.arange(2, 30000), 999, replace=False)])).astype(np.int32)
           for _ in src]
    dm = _lib.device_model(full)
    a = _lib.decode([dm], src, 5, 2, 10, False, 1, shortlists=sls, max_batch=64)
    b = _lib.decode([dm], src, 5, 2, 10, False, 1, shortlists=sls, max_batch=3)
    for i in range(len(src)):
        # buckets gather their shortlist union, so the log-normaliser's
        # per-tile grouping (fp32 partials) follows the bucket: tokens are
        # identical, scores agree to fp32 rounding
        ha, hb = a.hyps(i)[0], b.hyps(i)[0]
        assert ha[0] == hb[0], i
        assert abs(ha[1] - hb[1]) <= 1e-6 * abs(hb[1]), (i, ha[1], hb[1])
    monkeypatch.setenv("AMUN_SL_GATHER_FRAC", "0")  # full-vocabulary masked kernel: byte-identical
    a = _lib.decode([dm], src, 5, 2, 10, False, 1, shortlists=sls, max_batch=64)
    b = _lib.decode([dm], src, 5, 2, 10, False, 1, shortlists=sls, max_batch=3)
    for i in range(len(src)):
        assert a.hyps(i)[0][:2] == b.hyps(i)[0][:2], i


def test_engine_two_workers_on_one_device(gpu, full):
    """The multi-device Engine path (engine.py:181-221 analogue: shard by
    length-bucket LPT -> one host thread per device -> concurrent decode ->
    gather by input index) exercised as two workers on GPU 0: byte-identical
    to one worker."""
    from paper_1610_01108_b200 import workload as W
    from paper_1610_01108_b200.engine import Engine, EngineConfig
    from paper_1610_01108_b200.model import Vocabulary

    sents = W.WORKLOADS["cfg2"].corpus()[:96]
    lines = W.lines_of(sents)
    vocab = Vocabulary.from_tokens([f"w{i}" for i in range(2, W.V_SRC)])

    def engine(devices):
        cfg = EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>",
                           devices=devices, max_batch=16, n_best=2)
        return Engine(cfg, [full], vocab, vocab, None, None, None, 0, 0.0)

    one = engine((0,)).translate_corpus(lines)
    two = engine((0, 0)).translate_corpus(lines)
    assert [(r.text, r.score, r.n_best) for r in one] == [(r.text, r.score, r.n_best) for r in two]


def test_encode_ahead_chunking_is_byte_identical(gpu, full, monkeypatch):
    """Encode-ahead over one chunk vs many small chunks (AMUN_ENC_CHUNK): the
    encoder's split counts depend on the weight shape only, never on how
    many sentences share a step GEMM, so every hypothesis is byte-identical
    (the same argument makes 1/2/4/8-GPU shards identical)."""
    from paper_1610_01108_b200 import workload as W

    sents = W.WORKLOADS["cfg2"].corpus()[:150]
    dm = _lib.device_model(full)
    a = _lib.decode([dm], sents, 5, 2, 10, False, 2, max_batch=16)
    monkeypatch.setenv("AMUN_ENC_CHUNK", "40")
    b = _lib.decode([dm], sents, 5, 2, 10, False, 2, max_batch=16)
    for i in range(len(sents)):
        assert a.hyps(i) == b.hyps(i), i


@pytest.mark.parametrize("name,max_batch", [("cfg1", 1), ("cfg1", 64), ("cfg2", 64)])
def test_shortlist_decode_matches_reference(gpu, full, name, max_batch):
    """Shortlist decodes (nnet.py:160-163, search.py:146-148) against the
    reference's own beam_search with its build_shortlist lists over the
    synthetic lexical table (tests/golden/make_golden_shortlist.py): the
    gathered-union logit path (batch 1: the sentence's own list; buckets:
    the union with per-sentence masks) and, for wide unions, the masked
    full-vocabulary kernel."""
    from conftest import golden_shortlist
    from paper_1610_01108_b200 import workload as W

    g = golden_shortlist()
    corpus = W.WORKLOADS[name].corpus()
    sents = [corpus[i] for i in g[f"{name}_idx"]]
    sls = W.shortlists(sents)
    beam, f, o, _, _ = (int(x) for x in g[f"{name}_opts"])
    out = _lib.decode([_lib.device_model(full)], sents, beam, f, o, False, 2, shortlists=sls, max_batch=max_batch)
    toff, goff = g[f"{name}_tok_off"], g[f"{name}_gap_off"]
    gold = [(g[f"{name}_tokens"][toff[i]:toff[i + 1]].astype(int).tolist(), float(g[f"{name}_score"][i]))
            for i in range(len(sents))]
    gaps = [g[f"{name}_gap"][goff[i]:goff[i + 1]] for i in range(len(sents))]
    _adjudicate(f"shortlist {name} batch {max_batch}", gold, gaps, out)
    for i in range(len(sents)):
        assert set(out.hyps(i)[0][0]) <= set(sls[i].tolist())


@pytest.mark.parametrize("name", ["ens2", "ens3", "mixed"])
def test_ensemble_decode_matches_reference(gpu, full, name):
    """Full-size ensembles (search.py:56-72: log-probs averaged about the
    first member; search.py:150-152: one Forward per member, so members may
    differ in d_emb / d_h / d_att) against the reference's own beam_search
    (tests/golden/make_golden_ensemble.py), decoded in buckets of 64.  The
    members' logits run as ONE fused tensor-core launch per step (member-sum
    candidates + per-member log-softmax partials): the per-class launch
    counts show one logit launch per decoder step, never the CUDA-core
    full-logit path."""
    from conftest import golden_ensemble
    from paper_1610_01108_b200 import workload as W

    g = golden_ensemble()
    members = []
    for de, dh, da, seed in g[f"{name}_members"].tolist():
        if (de, dh, da, seed) == (500, 1024, 1024, 1):
            members.append(full)
        else:
            members.append(random_model(ModelConfig(30000, 30000, de, dh, da), seed))
    dms = [_lib.device_model(m) for m in members]
    corpus = W.WORKLOADS["cfg2"].corpus()
    sents = [corpus[i] for i in g[f"{name}_idx"]]
    beam, f, o, _, _ = (int(x) for x in g[f"{name}_opts"])
    out = _lib.decode(dms, sents, beam, f, o, False, 2, max_batch=64)
    toff, goff = g[f"{name}_tok_off"], g[f"{name}_gap_off"]
    gold = [(g[f"{name}_tokens"][toff[i]:toff[i + 1]].astype(int).tolist(), float(g[f"{name}_score"][i]))
            for i in range(len(sents))]
    gaps = [g[f"{name}_gap"][goff[i]:goff[i + 1]] for i in range(len(sents))]
    _adjudicate(f"ensemble {name}", gold, gaps, out)
    prof = _lib.decode(dms, sents[:3], beam, f, o, False, 2, max_batch=64, profile=(1 << 6) | (1 << 7))
    assert prof.kernel_count["logits"] == prof.decoder_steps, (prof.kernel_count, prof.decoder_steps)
    for i in range(3):
        assert prof.hyps(i) == out.hyps(i)


def test_bench_api_through_engine(gpu, full):
    """paper_1610_01108_b200.bench on the real Engine (reference
    pkg/src/beamnmt/bench.py:74-126): the throughput report counts the
    corpus's source tokens and its 1-best target words, and the decoder's
    device time is part of the wall time."""
    from paper_1610_01108_b200 import workload as W
    from paper_1610_01108_b200.bench import latency_bench, throughput_bench
    from paper_1610_01108_b200.engine import Engine, EngineConfig
    from paper_1610_01108_b200.model import Vocabulary

    sents = W.WORKLOADS["cfg2"].corpus()[:40]
    lines = W.lines_of(sents)
    vocab = Vocabulary.from_tokens([f"w{i}" for i in range(2, W.V_SRC)])
    eng = Engine(EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>",
                              devices=(0,), max_batch=16), [full], vocab, vocab, None, None, None, 0, 0.0)
    rep, res = throughput_bench(eng, lines, threads=4, warmup=True)
    assert rep.total_tokens == sum(map(len, sents)) and rep.sentence_count == 40
    assert rep.target_tokens == sum(len(r.text.split()) for r in res) > 0
    assert 0 < rep.device_seconds <= rep.wall_seconds
    lrep, lres = latency_bench(eng, lines[:4])
    assert [r.text for r in lres] == [r.text for r in res[:4]]
    assert 0 < lrep.device_seconds <= lrep.wall_seconds


@pytest.mark.parametrize("name,max_batch", [("ens2_sl", 64), ("ens2_sl", 5), ("beam16", 64), ("beam16", 3),
                                            ("beam9", 64)])
def test_extra_paths_match_reference(gpu, full, name, max_batch):
    """Less common decode paths against the reference's own beam_search
    (tests/golden/make_golden_extra.py): a 2-member ensemble WITH shortlists
    (masks on the fused ensemble logit kernel), beam 16 (the rows-layout
    logit kernel's largest list) and beam 9, in several bucket sizes."""
    from paper_1610_01108_b200 import workload as W

    from conftest import GOLDEN

    with np.load(GOLDEN / "extra_sets.npz") as z:
        g = {k: z[k] for k in z.files}
    members = []
    for de, dh, da, seed in g[f"{name}_members"].tolist():
        members.append(full if (de, dh, da, seed) == (500, 1024, 1024, 1)
                       else random_model(ModelConfig(30000, 30000, de, dh, da), seed))
    dms = [_lib.device_model(m) for m in members]
    corpus = W.WORKLOADS["cfg2"].corpus()
    sents = [corpus[i] for i in g[f"{name}_idx"]]
    sls = W.shortlists(sents) if int(g[f"{name}_shortlists"]) else None
    beam, f, o, _, _ = (int(x) for x in g[f"{name}_opts"])
    out = _lib.decode(dms, sents, beam, f, o, False, 2, shortlists=sls, max_batch=max_batch)
    toff, goff = g[f"{name}_tok_off"], g[f"{name}_gap_off"]
    gold = [(g[f"{name}_tokens"][toff[i]:toff[i + 1]].astype(int).tolist(), float(g[f"{name}_score"][i]))
            for i in range(len(sents))]
    gaps = [g[f"{name}_gap"][goff[i]:goff[i + 1]] for i in range(len(sents))]
    _adjudicate(f"{name} batch {max_batch}", gold, gaps, out)
    if sls is not None:
        for i in range(len(sents)):
            assert set(out.hyps(i)[0][0]) <= set(sls[i].tolist())


def test_rows_logits_cluster_sizes_agree(gpu, full):
    """The rows-layout logit kernel (beams >= 8) shares each weight tile over
    a cluster of as many CTAs as the bucket has 128-row tiles (6 at R = 768)
    and runs single CTAs for buckets of 3 sentences: both must give
    byte-identical decodes, so a sentence's result never depends on its
    bucket's size."""
    from paper_1610_01108_b200 import workload as W

    sents = W.WORKLOADS["cfg4"].corpus()[:64]
    dm = _lib.device_model(full)
    a = _lib.decode([dm], sents, 12, 1, 0, False, 2, max_batch=64)
    b = _lib.decode([dm], sents, 12, 1, 0, False, 2, max_batch=3)
    for i in range(len(sents)):
        assert a.hyps(i) == b.hyps(i), i
