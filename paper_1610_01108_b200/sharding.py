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
# A bucket's decoder steps are serial: on a lightly loaded GPU one step of a
# 320-row bucket takes ~0.31 ms, as long as the saturated GPU needs for
# ~1200 row-steps of throughput work (cfg2: 0.26 us per row-step).  So a
# bucket of S steps bounds its device's time from below by S x 1200 row-steps
# of work, whatever else runs there.
STEP_LATENCY_ROWS = 1200


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


def partition_makespan(costs: Sequence[float], latencies: Sequence[float], n_parts: int) -> list[list[int]]:
    """Greedy LPT on the estimated finish time of a part, max(sum of its
    costs, its largest latency bound): largest cost first onto the part whose
    estimate grows least (ties: lower load, then lower index).  A long
    serial item then shares its part only with the work that fits under its
    own latency, instead of also getting a full share of the rest."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    parts: list[list[int]] = [[] for _ in range(n_parts)]
    load = [0.0] * n_parts
    lat = [0.0] * n_parts
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        def after(q):
            return max(load[q] + costs[i], lat[q], latencies[i])
        p = min(range(n_parts), key=lambda q: (after(q), load[q], q))
        parts[p].append(i)
        load[p] += costs[i]
        lat[p] = max(lat[p], latencies[i])
    return parts


def shard_sentences(lengths: Sequence[int], n_parts: int, bucket: int, beam: int, max_len_factor: int = 2,
                    max_len_offset: int = 10) -> list[list[int]]:
    """Sentence indices per part: whole length buckets, assigned by LPT on
    the estimated finish time (work, and the serial step chain of a part's
    longest bucket)."""
    buckets = length_buckets(lengths, bucket)
    costs = [sum(sentence_work(lengths[i], beam, max_len_factor, max_len_offset) for i in b) for b in buckets]
    lats = [max(max_len_factor * lengths[i] + max_len_offset for i in b) * STEP_LATENCY_ROWS * STEP_FLOP
            for b in buckets]
    out = []
    for part in partition_makespan(costs, lats, n_parts):
        out.append(sorted((i for b in part for i in buckets[b]), key=lambda i: (lengths[i], i)))
    return out
