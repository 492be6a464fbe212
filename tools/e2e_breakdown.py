"""Where the end-to-end time goes (profiling aid, not part of the product):
host text front-end, amun_decode wall vs its device-timed region, and the
host result assembly, for the bench's cfg2 workload on one GPU."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.engine import Engine, EngineConfig
from paper_1610_01108_b200.model import ModelConfig, Vocabulary, random_model

wl = W.WORKLOADS["cfg2"]
sents = wl.corpus()
model = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
dm = _lib.device_model(model, 0)
vocab = Vocabulary.from_tokens([f"w{i}" for i in range(2, W.V_SRC)])
eng = Engine(EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>",
                          beam_size=wl.beam, max_len_factor=wl.max_len_factor, max_len_offset=wl.max_len_offset,
                          devices=(0,), max_batch=wl.batch), [model], vocab, vocab, None, None, None, 0, 0.0)
lines = W.lines_of(sents)
for _ in range(2):
    out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, max_batch=wl.batch)
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    out = _lib.decode([dm], sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, max_batch=wl.batch)
    t1 = time.perf_counter()
    hy = [out.hyps(i) for i in range(len(sents))]
    t2 = time.perf_counter()
    res = eng.translate_corpus(lines)
    t3 = time.perf_counter()
    print(f"decode wall {1e3*(t1-t0):.1f} ms (C call {out.call_ms:.1f}, device {out.device_ms:.1f}, host setup {out.host_setup_ms:.1f}, "
          f"post {out.host_post_ms:.1f}), hyps {1e3*(t2-t1):.1f} ms, "
          f"translate_corpus wall {1e3*(t3-t2):.1f} ms, d2h {out.d2h_bytes/1e6:.1f} MB", flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "profile":
    _orig = eng._decode
    _t = {}

    def _timed(*a, **k):
        t0 = time.perf_counter()
        r = _orig(*a, **k)
        _t["dec"] = 1e3 * (time.perf_counter() - t0)
        return r

    eng._decode = _timed
    import gc
    for _ in range(6):
        t0 = time.perf_counter()
        eng.translate_corpus(lines)
        print(f"translate_corpus {1e3 * (time.perf_counter() - t0):.1f} ms: _decode {_t['dec']:.1f} "
              f"(device {eng.last_stats['device_ms'][0]:.1f}); gc counts {gc.get_count()}", flush=True)
    import cProfile, pstats
    for _ in range(5):
        t0 = time.perf_counter()
        eng.translate_corpus(lines)
        print(f"translate_corpus {1e3 * (time.perf_counter() - t0):.1f} ms (device {eng.last_stats['device_ms']})",
              flush=True)
    pr = cProfile.Profile()
    pr.enable()
    eng.translate_corpus(lines)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
