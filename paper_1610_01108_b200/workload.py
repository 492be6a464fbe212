"""Synthetic benchmark workloads (SURVEY §8(d) / BASELINE.md §4).

All configs use random_model(ModelConfig(30000, 30000, 500, 1024, 1024),
seed=1).  Source lengths J = clip(rint(lognormal(ln 26, 0.6)), 1, max_len),
drawn for all sentences first, then ids uniform in [2, v_src) per sentence
(the tests/conftest.py:44 convention); text lines are "w<id>" tokens.

  cfg1  100 sentences, seed 2017, J <= 50,  beam 5,  batch 1
  cfg2  4000 sentences, seed 2016, J <= 100, beam 5, length buckets of 64
  cfg3  cfg2 sharded over 2/4/8 GPUs
  cfg4  512 sentences, J = 100, beam 12, cap = 1 * J + 0 = 100
  cfg5  cfg2 set, beam 1, buckets of 512

Shortlist workloads use a synthetic lexical table:
target frequency ranks are a fixed permutation of [2, v_trg); each source
id's translations, best first, are distinct ranks drawn log-uniformly (so
frequent targets recur across sources, as in a real table), probabilities
1/(j + 2) for the j-th.  A sentence's shortlist is the reference's
build_shortlist set (shortlist.py:128-147): {0, 1} U the K most frequent
targets U the K' best translations of each source token, K = K' = 75 (the
EngineConfig defaults, engine.py:40-41).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

V_SRC = V_TRG = 30000
D_EMB, D_H, D_ATT = 500, 1024, 1024
MODEL_SEED = 1


def corpus(n: int, seed: int, max_len: int, v_src: int = V_SRC, fixed_len: int | None = None) -> list[list[int]]:
    rng = np.random.default_rng(seed)
    if fixed_len is None:
        lens = np.clip(np.rint(rng.lognormal(np.log(26.0), 0.6, size=n)), 1, max_len).astype(np.int64)
    else:
        lens = np.full(n, fixed_len, dtype=np.int64)
    return [[int(i) for i in rng.integers(2, v_src, size=int(L))] for L in lens]


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    sentences: int
    seed: int
    max_len: int
    fixed_len: int | None
    beam: int
    max_len_factor: int
    max_len_offset: int
    batch: int

    def corpus(self) -> list[list[int]]:
        return corpus(self.sentences, self.seed, self.max_len, fixed_len=self.fixed_len)


WORKLOADS = {
    "cfg1": Workload("cfg1", "100 synthetic sentences <=50 tokens, beam 5, batch 1", 100, 2017, 50, None, 5, 2, 10, 1),
    "cfg2": Workload("cfg2", "4000-sentence UN-test-shaped synthetic set, beam 5, length buckets of 64", 4000, 2016,
                     100, None, 5, 2, 10, 64),
    "cfg4": Workload("cfg4", "512 sentences of length 100, beam 12, target cap 100", 512, 2018, 100, 100, 12, 1, 0, 64),
    "cfg5": Workload("cfg5", "cfg2 set, greedy (beam 1), buckets of 512", 4000, 2016, 100, None, 1, 2, 10, 512),
}


def lines_of(sentences: list[list[int]]) -> list[str]:
    return [" ".join(f"w{i}" for i in s) for s in sentences]


# ---------------------------------------------------------------- shortlists

LEX_SEED = 1610
SL_K = SL_KPRIME = 75
LEX_ENTRIES = 100  # translations per source id in the synthetic table


def target_by_rank(v_trg: int = V_TRG) -> np.ndarray:
    """Target ids in descending frequency (the frequency list)."""
    return np.random.default_rng(LEX_SEED).permutation(np.arange(2, v_trg))


def lex_translations(src_id: int, v_trg: int = V_TRG, n: int = LEX_ENTRIES,
                     by_rank: np.ndarray | None = None) -> np.ndarray:
    """Target ids of source id `src_id`'s table entries, best first."""
    if by_rank is None:
        by_rank = target_by_rank(v_trg)
    rng = np.random.default_rng((LEX_SEED, int(src_id)))
    ranks: list[int] = []
    seen: set[int] = set()
    while len(ranks) < n:
        for r in (np.exp(rng.random(2 * n) * np.log(v_trg - 2)).astype(np.int64) - 1):
            r = int(min(max(r, 0), v_trg - 3))
            if r not in seen:
                seen.add(r)
                ranks.append(r)
                if len(ranks) == n:
                    break
    return by_rank[np.asarray(ranks)]


def shortlists(sentences: list[list[int]], K: int = SL_K, Kprime: int = SL_KPRIME,
               v_trg: int = V_TRG) -> list[np.ndarray]:
    """Per-sentence ascending shortlist ids (int32), build_shortlist semantics."""
    by_rank = target_by_rank(v_trg)
    base = set(int(i) for i in by_rank[:K]) | {0, 1}
    cache: dict[int, np.ndarray] = {}
    out = []
    for s in sentences:
        ids = set(base)
        for tok in s:
            tr = cache.get(tok)
            if tr is None:
                tr = cache[tok] = lex_translations(tok, v_trg, by_rank=by_rank)[:Kprime]
            ids.update(int(i) for i in tr)
        out.append(np.array(sorted(ids), dtype=np.int32))
    return out
