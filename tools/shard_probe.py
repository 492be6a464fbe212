"""One rank's LPT shard of cfg2 decoded on one GPU (profiling aid for the
N-GPU strong-scaling tail): device time vs 1/N of the full pass."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, random_model
from paper_1610_01108_b200.sharding import shard_sentences

wl = W.WORKLOADS["cfg2"]
sents = wl.corpus()
dm = _lib.device_model(random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED), 0)
for n in [1] + [int(a) for a in sys.argv[1:]]:
    shards = shard_sentences([len(s) for s in sents], n, wl.batch, wl.beam, wl.max_len_factor, wl.max_len_offset)
    worst = 0.0
    for r in (range(n) if n <= 2 else [0, n - 1]):
        sub = [sents[i] for i in shards[r]]
        for _ in range(2):
            out = _lib.decode([dm], sub, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1, max_batch=wl.batch)
        worst = max(worst, out.device_ms)
        print(f"N={n} rank {r}: {len(sub)} sentences, {out.device_ms:.1f} ms", flush=True)
    print(f"N={n}: slowest rank {worst:.1f} ms", flush=True)
