"""Sentence sharding across GPUs.

Sentences are independent units (engine.py:181-221 decodes them in any
order), so multi-GPU decoding is data parallel with no collective: sort by
source length, cut length buckets, and give buckets to devices by greedy
longest-processing-time on the estimated decode work.  Results are gathered
on the host by original index.  A sentence's result does not depend on its
batch-mates (rows are independent in every kernel), so output is identical
for any device count.
"""

from __future__ import annotations

from typing import Sequence

# Algorithmic FLOP per decoder row-step and per source token at
# emb500/hid1024/30k; only their ratio matters here.
STEP_FLOP = 57.83e6
SRC_FLOP = 22.92e6


def sentence_work(src_len: int, beam: int, max_len_factor: int = 2, max_len_offset: int = 10) -> float:
    cap = max_len_factor * src_len + max_len_offset
    return cap * beam * STEP_FLOP + src_len * SRC_FLOP


def length_buckets(lengths: Sequence[int], bucket: int) -> list[list[int]]:
    """Indices sorted by length (stable), cut every `bucket` sentences —
    the same bucketing amun_decode applies internally."""
    order = sorted(range(len(lengths)), key=lambda i: lengths[i])
    return [order[i:i + bucket] for i in range(0, len(order), bucket)]


def partition_lpt(costs: Sequence[float], n_parts: int) -> list[list[int]]:
    """Greedy LPT: largest cost first onto the least-loaded part (ties to
    the lowest part index).  Deterministic."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    parts: list[list[int]] = [[] for _ in range(n_parts)]
    load = [0.0] * n_parts
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        p = min(range(n_parts), key=lambda q: (load[q], q))
        parts[p].append(i)
        load[p] += costs[i]
    return parts


def shard_sentences(lengths: Sequence[int], n_parts: int, bucket: int, beam: int, max_len_factor: int = 2,
                    max_len_offset: int = 10) -> list[list[int]]:
    """Sentence indices per part: whole length buckets assigned by LPT."""
    buckets = length_buckets(lengths, bucket)
    costs = [sum(sentence_work(lengths[i], beam, max_len_factor, max_len_offset) for i in b) for b in buckets]
    out = []
    for part in partition_lpt(costs, n_parts):
        out.append(sorted((i for b in part for i in buckets[b]), key=lambda i: (lengths[i], i)))
    return out
