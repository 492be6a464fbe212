"""Host-glue goldens from the REAL reference (dev container only; committed
as tests/golden/host.json): BPE learning / segmentation / joining
(pkg/src/beamnmt/subword.py) and lexical-table / frequency-list /
shortlist construction (pkg/src/beamnmt/shortlist.py) on small synthetic
inputs with ties, unknown targets, duplicates and repeated tokens.

    python tests/golden/make_golden_host.py
"""

from __future__ import annotations

import json
import random
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from beamnmt import shortlist as S  # noqa: E402
from beamnmt import subword as B  # noqa: E402
from beamnmt.model import Vocabulary  # noqa: E402


def corpus(rng: random.Random, n: int) -> list[str]:
    stems = ["low", "new", "wid", "aa", "ab", "ba", "x", "höh", "日本", "ing", "er", "est"]
    out = []
    for _ in range(n):
        words = ["".join(rng.choice(stems) for _ in range(rng.randint(1, 3))) for _ in range(rng.randint(1, 9))]
        out.append(" ".join(words))
    return out


def main() -> None:
    rng = random.Random(1610)
    bpe_cases = []
    for n_lines, merges in ((5, 10), (40, 60), (200, 150), (3, 0), (30, 500)):
        lines = corpus(rng, n_lines)
        model = B.bpe_learn(lines, merges)
        words = [w for ln in corpus(rng, 20) for w in ln.split()] + ["a", "unseen", "ab", "q"]
        pieces = B.bpe_apply(model, words)
        joins = [B.bpe_join(p) for p in (pieces, ["a@@", "@@", "b"], ["x@@@@", "y"], ["tail@@"], [], ["a", "", "b"])]
        bpe_cases.append({"corpus": lines, "num_merges": merges, "merges": [list(p) for p in model.merges],
                          "words": words, "pieces": pieces, "joins": joins})
    vocab = Vocabulary.from_tokens(["x", "y", "z", "u", "v", "w"])
    lex_lines = ["s x 0.5", "s y 0.9", "s x 0.7", "t zz 0.4", "t qq 0.6", "t u 0.6", "r v 1.0", "", "r w 0.25",
                 "r u 0.25", "p x 0.1", "p y 0.1", "p z 0.1"]
    with tempfile.TemporaryDirectory() as d:
        lp, fp = Path(d) / "lex", Path(d) / "freq"
        lp.write_text("\n".join(lex_lines) + "\n")
        fp.write_text("z\nq\nx\nz\n\nw\n")
        table = S.load_lex_table(lp, vocab)
        freq, skipped = S.load_freq_list(fp, vocab)
    sls = []
    for src, k, kp in ((["s", "t"], 1, 1), (["r", "r", "p", "zz"], 2, 2), ([], 0, 0), (["p"], 3, 3), (["t", "s"], 9, 9)):
        sls.append({"src": src, "K": k, "Kprime": kp,
                    "ids": S.build_shortlist(table, freq, src, k, kp, vocab).global_ids.tolist()})
    out = {"bpe": bpe_cases, "vocab": vocab.tokens, "lex_lines": lex_lines,
           "table": {s: [list(e) for e in v] for s, v in table.entries.items()}, "freq": freq,
           "freq_skipped": skipped, "shortlists": sls}
    (HERE / "host.json").write_text(json.dumps(out, ensure_ascii=False, indent=0))


if __name__ == "__main__":
    main()
