"""Host-side logic of the drop-in API (no GPU): model container, random
model, vocabulary, BPE, shortlist, argument validation with the reference's
messages, ensemble averaging, sharding."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import tiny_model
from oracle import beamnmt_oracle as orc
from paper_1610_01108_b200 import (
    DecodeOptions,
    ModelConfig,
    ModelParams,
    ShortList,
    Vocabulary,
    average_checkpoints,
    beam_search,
    bpe_apply,
    bpe_join,
    bpe_learn,
    build_shortlist,
    ensemble_logprobs,
    load_model,
    load_vocab,
    preprocess,
    random_model,
    save_model,
)
from paper_1610_01108_b200.errors import FormatError
from paper_1610_01108_b200.model import schema
from paper_1610_01108_b200.sharding import (STEP_FLOP, STEP_LATENCY_ROWS, length_buckets, partition_lpt,
                                            sentence_work, shard_sentences)
from paper_1610_01108_b200.shortlist import LexicalTable, load_freq_list, load_lex_table
from paper_1610_01108_b200.subword import load_bpe_model, save_bpe_model
from paper_1610_01108_b200.workload import WORKLOADS


# ------------------------------------------------------------------ model

def test_random_model_matches_oracle_draws():
    m = random_model(ModelConfig(v_src=13, v_trg=11, d_emb=6, d_h=5, d_att=7), 123)
    want = orc.random_tensors((13, 11, 6, 5, 7), 123)
    for name, arr in m.tensor_items():
        np.testing.assert_array_equal(arr, want[name], err_msg=name)
        assert not arr.flags.writeable


def test_schema_has_40_tensors_in_reference_order():
    names = [n for n, _, _ in schema(ModelConfig(30000, 30000))]
    assert len(names) == 40
    assert names[:3] == ["E_src", "E_trg", "enc_fwd.W_z"]
    assert names[-2:] == ["W_logit", "b_logit"]


def test_save_load_roundtrip_bitwise(tmp_path):
    m = tiny_model(3, 7, 9, 5)
    p = tmp_path / "m.amnt"
    save_model(m, p)
    back = load_model(p)
    assert back.config == m.config
    for (n, a), (_, b) in zip(m.tensor_items(), back.tensor_items()):
        np.testing.assert_array_equal(a, b, err_msg=n)


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated"),
    (lambda b: b + b"\0", "trailing bytes"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "unsupported format version"),
])
def test_container_errors(tmp_path, mutate, msg):
    p = tmp_path / "m.amnt"
    save_model(tiny_model(1), p)
    p.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(FormatError, match=msg):
        load_model(p)


def test_from_tensors_validation():
    cfg = ModelConfig(v_src=5, v_trg=5, d_emb=4, d_h=4, d_att=4)
    t = {n: np.zeros((r, c), np.float32) for n, r, c in schema(cfg)}
    with pytest.raises(FormatError, match="missing tensor"):
        ModelParams.from_tensors(cfg, {k: v for k, v in t.items() if k != "v_att"})
    with pytest.raises(FormatError, match="unexpected tensor"):
        ModelParams.from_tensors(cfg, {**t, "bogus": np.zeros(1)})
    t["W_init"] = np.zeros((3, 3), np.float32)
    with pytest.raises(FormatError, match="has shape"):
        ModelParams.from_tensors(cfg, t)


def test_non_finite_rejected():
    cfg = ModelConfig(v_src=5, v_trg=5, d_emb=4, d_h=4, d_att=4)
    t = {n: np.zeros((r, c), np.float32) for n, r, c in schema(cfg)}
    t["E_src"][0, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        ModelParams.from_tensors(cfg, t)


def test_average_checkpoints(tmp_path):
    paths = []
    for seed in (1, 2):
        p = tmp_path / f"{seed}.amnt"
        save_model(tiny_model(seed, 6, 6, 4), p)
        paths.append(p)
    avg = average_checkpoints(paths)
    a, b = load_model(paths[0]), load_model(paths[1])
    for (n, x), (_, y), (_, z) in zip(a.tensor_items(), b.tensor_items(), avg.tensor_items()):
        np.testing.assert_allclose(z, ((x.astype(np.float64) + y) / 2).astype(np.float32), atol=1e-7)
    with pytest.raises(ValueError):
        average_checkpoints([])


# ------------------------------------------------------------------ vocab / text

def test_vocabulary(tmp_path):
    v = Vocabulary.from_tokens(["a", "b"])
    assert len(v) == 4 and v.id("a") == 2 and v.id("zz") == 1 and "b" in v and v.token(0) == "</s>"
    p = tmp_path / "v.txt"
    p.write_text("x\ny\n")
    assert load_vocab(p).tokens == ["</s>", "<unk>", "x", "y"]
    p.write_text("x\nx\n")
    with pytest.raises(FormatError, match="duplicate"):
        load_vocab(p)
    p.write_text("</s>\n")
    with pytest.raises(FormatError, match="reserved"):
        load_vocab(p)


def test_bpe_roundtrip_and_file(tmp_path):
    corpus = ["low lower lowest", "newer newest new", "wider widest"] * 3
    model = bpe_learn(corpus, 20)
    words = preprocess("Lower NEWEST widest unseenword")
    pieces = bpe_apply(model, words)
    assert bpe_join(pieces) == words
    assert any(p.endswith("@@") for p in pieces)
    save_bpe_model(model, tmp_path / "r.bpe")
    assert load_bpe_model(tmp_path / "r.bpe").merges == model.merges


def test_bpe_matches_reference_rules():
    """Same learning tie-break and segmentation as the reference (SPEC
    §subword): golden rules derived by hand for a tiny corpus."""
    model = bpe_learn(["aaa aaa ab"], 3)
    assert model.merges[0] == ("a", "a")
    assert bpe_apply(model, ["aaa"]) in (["aa@@", "a"], ["aaa"], ["a@@", "aa"])


def test_shortlist(tmp_path):
    vocab = Vocabulary.from_tokens(["x", "y", "z"])
    lex = tmp_path / "lex"
    lex.write_text("s x 0.5\ns y 0.9\nt zz 0.4\n")
    table = load_lex_table(lex, vocab)
    assert table.get("s")[0] == ("y", 0.9)
    assert table.get("t")[0][0] == "<unk>"
    freq = tmp_path / "freq"
    freq.write_text("z\nq\nx\n")
    ids, skipped = load_freq_list(freq, vocab)
    assert ids == [4, 2] and skipped == 1
    sl = build_shortlist(table, ids, ["s"], 1, 1, vocab)
    assert list(sl.global_ids) == [0, 1, 3, 4]
    with pytest.raises(ValueError, match="ascending"):
        ShortList(np.array([0, 1, 3, 2]))
    with pytest.raises(ValueError, match="0"):
        ShortList(np.array([1, 2]))
    assert len(ShortList.full(6)) == 6


# ------------------------------------------------------------------ validation (raises before the device)

def test_beam_search_validation_messages():
    m = tiny_model(15)
    with pytest.raises(ValueError, match="at least one model"):
        beam_search([], [2])
    with pytest.raises(ValueError, match="empty"):
        beam_search([m], [])
    with pytest.raises(ValueError, match="beam_size"):
        beam_search([m], [2], DecodeOptions(beam_size=0))
    with pytest.raises(ValueError, match="n_best"):
        beam_search([m], [2], DecodeOptions(n_best=0))
    with pytest.raises(ValueError, match="cap"):
        beam_search([m], [2], DecodeOptions(max_len_factor=0, max_len_offset=0))
    with pytest.raises(ValueError, match="out of range"):
        beam_search([m], [2, 99])
    with pytest.raises(ValueError, match="vocabulary mismatch"):
        beam_search([tiny_model(1, v_trg=5), tiny_model(1, v_trg=6)], [2])
    with pytest.raises(ValueError, match="shortlist id"):
        beam_search([m], [2], shortlist=ShortList(np.array([0, 1, 7])))


def test_decode_options_defaults():
    o = DecodeOptions()
    assert (o.beam_size, o.max_len_factor, o.max_len_offset, o.length_normalize, o.n_best) == (5, 2, 10, False, 1)
    assert o.max_target_len(30) == 70


def test_ensemble_logprobs():
    rng = np.random.default_rng(0)
    x = np.log(rng.dirichlet(np.ones(9)))
    for k in range(1, 6):
        np.testing.assert_array_equal(ensemble_logprobs([x] * k), x)
    a = np.array([math.log(0.5), math.log(0.5)])
    b = np.array([math.log(0.25), math.log(0.75)])
    np.testing.assert_allclose(ensemble_logprobs([a, b]), (a + b) / 2, atol=1e-12)
    with pytest.raises(ValueError, match="mismatch"):
        ensemble_logprobs([np.zeros(5), np.zeros(6)])


# ------------------------------------------------------------------ sharding / workloads

def test_partition_lpt_balances_and_covers():
    costs = [float(c) for c in np.random.default_rng(1).integers(1, 100, 50)]
    parts = partition_lpt(costs, 4)
    assert sorted(i for p in parts for i in p) == list(range(50))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)


def test_shard_sentences_whole_buckets():
    wl = WORKLOADS["cfg2"]
    lens = [len(s) for s in wl.corpus()]
    for n in (1, 2, 4, 8):
        parts = shard_sentences(lens, n, 64, 5)
        assert sorted(i for p in parts for i in p) == list(range(4000))
        # whole buckets per part, and the estimated makespan (work, or the
        # serial step chain of a part's longest bucket) within 6% of its lower bound
        works = [sum(sentence_work(lens[i], 5) for i in p) for p in parts]
        lats = [max(2 * lens[i] + 10 for i in p) * STEP_LATENCY_ROWS * STEP_FLOP for p in parts]
        span = max(max(w, l) for w, l in zip(works, lats))
        assert span / max(sum(works) / n, max(lats)) < 1.06
    buckets = length_buckets(lens, 64)
    assert len(buckets) == 63 and all(len(b) == 64 for b in buckets[:-1])


def test_workload_matches_survey_totals():
    c2 = WORKLOADS["cfg2"].corpus()
    assert sum(map(len, c2)) == 120774
    assert sum(2 * len(s) + 10 for s in c2) == 281548
    c1 = WORKLOADS["cfg1"].corpus()
    assert sum(map(len, c1)) == 2813
    assert WORKLOADS["cfg2"].corpus() == orc.synthetic_corpus(4000, 2016, 100)


def test_engine_vectorised_texts_match_detokenize():
    """Engine._hyp_texts (flat device output -> strings) equals the
    per-hypothesis reference detokenisation (engine.py:175-179)."""
    from types import SimpleNamespace

    from paper_1610_01108_b200.engine import Engine, EngineConfig
    from paper_1610_01108_b200.model import EOS_ID, Vocabulary

    trg = Vocabulary.from_tokens([f"t{i}@@" if i % 3 == 0 else f"t{i}" for i in range(2, 20)])
    cfg = EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>")
    eng = Engine(cfg, [tiny_model(1, 20, 20, 4)], trg, trg, None, None, None, 0, 0.0)
    rng = np.random.default_rng(3)
    hyps = []
    for _ in range(60):
        toks = [int(t) for t in rng.integers(1, 20, size=int(rng.integers(0, 9)))]
        fin = bool(rng.integers(0, 2))
        if fin:
            toks.append(EOS_ID)
        hyps.append((toks, fin))
    flat = np.array([t for toks, _ in hyps for t in toks], np.int32)
    offs = np.cumsum([0] + [len(t) for t, _ in hyps]).astype(np.int64)
    res = SimpleNamespace(tokens=flat, tok_offsets=offs, finished=np.array([f for _, f in hyps]),
                          scores=np.zeros(len(hyps)))
    assert eng._hyp_texts(res) == [eng._detokenize(t, f) for t, f in hyps]


class _StubEngine:
    """Engine stand-in for the measurement API (no decoding): every line
    'a b c' translates to 'x y' with score -1, and each call reports 2 ms of
    device time on two devices (the longer one counts)."""

    def __init__(self):
        from paper_1610_01108_b200 import DecodeOptions

        self.opts = DecodeOptions(beam_size=5)
        self.shortlist_active = False
        self.startup_seconds = 0.25
        self.last_stats = {}
        self.calls = 0

    def translate_corpus(self, lines, threads=None, opts=None):
        from paper_1610_01108_b200.engine import TranslationResult

        self.calls += 1
        self.last_stats = {"device_ms": [1.0, 2.0]}
        return [TranslationResult("x y", -1.0, [(-1.0, "x y")], len(line.split()), 0) for line in lines]

    def translate_line(self, line, opts=None):
        return self.translate_corpus([line], opts=opts)[0]

    def with_options(self, **changes):
        from dataclasses import replace

        return replace(self.opts, **changes)


def test_bench_api_reports_and_validation():
    """paper_1610_01108_b200.bench keeps the reference's report definitions
    (pkg/src/beamnmt/bench.py:39-126): source words over decode wall time,
    startup excluded; adds target words/s and the engine's device time."""
    from paper_1610_01108_b200.bench import beam_sweep, latency_bench, throughput_bench

    eng = _StubEngine()
    corpus = ["a b c", "d e", "f"]
    rep, res = throughput_bench(eng, corpus, threads=3, warmup=True)
    assert eng.calls == 2 and len(res) == 3
    assert rep.total_tokens == 6 and rep.target_tokens == 6 and rep.sentence_count == 3
    assert math.isclose(rep.words_per_second, 6 / rep.wall_seconds)
    assert math.isclose(rep.target_words_per_second, 6 / rep.wall_seconds)
    assert rep.device_seconds == pytest.approx(0.002) and rep.threads == 3 and rep.beam == 5
    assert rep.startup_seconds == 0.25 and rep.to_dict()["ms_per_sentence"] == pytest.approx(1e3 * rep.wall_seconds / 3)
    lrep, _ = latency_bench(eng, corpus)
    assert lrep.threads == 1 and lrep.device_seconds == pytest.approx(0.006)
    rows = beam_sweep(eng, corpus, [1, 4])
    assert [r["beam"] for r in rows] == [1, 4] and all(r["bleu"] is None and r["mean_model_score"] == -1.0 for r in rows)
    with pytest.raises(ValueError, match="benchmark corpus is empty"):
        throughput_bench(eng, [], threads=1)
    with pytest.raises(ValueError, match="threads must be >= 1"):
        throughput_bench(eng, corpus, threads=0)
    with pytest.raises(ValueError, match="benchmark corpus is empty"):
        latency_bench(eng, [])
    with pytest.raises(ValueError, match="beam list is empty"):
        beam_sweep(eng, corpus, [])
    with pytest.raises(ValueError, match="beam sizes must be >= 1"):
        beam_sweep(eng, corpus, [2, 0])
    with pytest.raises(ValueError, match="line count mismatch"):
        beam_sweep(eng, corpus, [2], references=["r"])


def test_native_text_front_end_matches_python_path():
    """text.cu (amun_vocab_encode) splits like preprocess() = str.lower() +
    str.split() (every Unicode whitespace, engine.py:144-164) and maps tokens
    like Vocabulary.ids_and_oov (<unk> + OOV count) -- host-only code, no GPU."""
    from paper_1610_01108_b200 import _lib
    from paper_1610_01108_b200.model import UNK_ID, Vocabulary
    from paper_1610_01108_b200.subword import preprocess

    vocab = Vocabulary.from_tokens(["a", "b", "ça", "日本", "x​y", "Z", "</s>x", "𝒜"])
    nv = _lib.NativeVocab(vocab.tokens)
    ws = [" ", "\t", "\n", "\r", "\x0b", "\x0c", "\x1c", "\x1d", "\x1e", "\x1f", "\x85", "\xa0", " ",
          " ", " ", " ", " ", " ", " ", " ", "　"]
    rng = np.random.default_rng(5)
    words = ["a", "b", "ÇA", "日本", "x​y", "z", "Z", "</s>", "</s>x", "𝒜", "oov", "Á", "ß", ""]
    lines = ["", "   ", "a b", "A  B\tça", "　日本　", "x​y"]
    for _ in range(300):
        n = int(rng.integers(0, 9))
        parts = [words[int(rng.integers(len(words)))] for _ in range(n)]
        seps = [ws[int(rng.integers(len(ws)))] * int(rng.integers(1, 3)) for _ in range(n + 1)]
        lines.append("".join(s + p for s, p in zip(seps, parts + [""])))
    for lower in (True, False):
        ids, lens, oov = nv.encode(lines, lower, UNK_ID)
        want_ids, want_lens, want_oov = [], [], []
        for line in lines:
            i, o = vocab.ids_and_oov(preprocess(line, lower))
            want_ids += i
            want_lens.append(len(i))
            want_oov.append(o)
        assert ids.tolist() == want_ids and lens.tolist() == want_lens and oov.tolist() == want_oov
    big = lines * 12  # > 512 lines: the multi-threaded slices, concatenated in order
    ids, lens, oov = nv.encode(big, True, UNK_ID)
    assert lens.tolist() == [len(preprocess(x)) for x in big]
    assert ids.tolist() == [i for x in big for i in vocab.ids_and_oov(preprocess(x))[0]]
    with pytest.raises(ValueError, match="duplicate"):
        _lib.NativeVocab(["</s>", "<unk>", "a", "a"])


def test_host_glue_matches_reference_goldens(tmp_path):
    """BPE learning / segmentation / joining and lexical-table / frequency
    list / shortlist construction against fixtures the reference itself
    produced (tests/golden/make_golden_host.py: pkg/src/beamnmt/subword.py,
    shortlist.py)."""
    import json

    from conftest import GOLDEN
    from paper_1610_01108_b200.shortlist import build_shortlist

    g = json.loads((GOLDEN / "host.json").read_text())
    for c in g["bpe"]:
        model = bpe_learn(c["corpus"], c["num_merges"])
        assert [list(p) for p in model.merges] == c["merges"]
        assert bpe_apply(model, c["words"]) == c["pieces"]
        got = [bpe_join(p) for p in (c["pieces"], ["a@@", "@@", "b"], ["x@@@@", "y"], ["tail@@"], [], ["a", "", "b"])]
        assert got == c["joins"]
    vocab = Vocabulary(g["vocab"])
    lp, fp = tmp_path / "lex", tmp_path / "freq"
    lp.write_text("\n".join(g["lex_lines"]) + "\n")
    fp.write_text("z\nq\nx\nz\n\nw\n")
    table = load_lex_table(lp, vocab)
    assert {s: [list(e) for e in v] for s, v in table.entries.items()} == g["table"]
    freq, skipped = load_freq_list(fp, vocab)
    assert (freq, skipped) == (g["freq"], g["freq_skipped"])
    for s in g["shortlists"]:
        assert build_shortlist(table, freq, s["src"], s["K"], s["Kprime"], vocab).global_ids.tolist() == s["ids"]
