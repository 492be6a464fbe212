"""Debug: beam-9 sentence 3 of extra_sets through several device paths."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from conftest import GOLDEN, full_model
from paper_1610_01108_b200 import _lib, workload as W

z = np.load(GOLDEN / "extra_sets.npz")
corpus = W.WORKLOADS["cfg2"].corpus()
sents = [corpus[i] for i in z["beam9_idx"]]
toff = z["beam9_tok_off"]
i = 3
gold = z["beam9_tokens"][toff[i]:toff[i + 1]].tolist()
print("gold", z["beam9_score"][i], gold[:30])
dm = _lib.device_model(full_model())
for tag, kw in (("fused", {}), ("full-logit", {"force_full_logits": True})):
    for beam in (9, 10, 11):
        out = _lib.decode([dm], [sents[i]], beam, 2, 10, False, 3, **kw)
        h = out.hyps(0)
        print(tag, beam, [(round(s, 6), t[:20] == gold[:20], next((k for k, (a, b) in enumerate(zip(t, gold)) if a != b), None)) for t, s, _, _ in h])
