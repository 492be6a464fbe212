"""Throughput / latency measurement API (reference: beamnmt/bench.py:23-140).

Same report fields and definitions: words_per_second counts post-BPE SOURCE
tokens over decode wall time, model load excluded (bench.py:46-51, :73-77).
`target_words_per_second` (1-best target tokens, final </s> excluded) is
added because the B200 headline metric is target words/s.
"""

from __future__ import annotations

import time
from dataclasses import asdict, dataclass
from typing import Sequence

from .engine import Engine, TranslationResult


@dataclass(frozen=True)
class BenchReport:
    total_tokens: int
    wall_seconds: float
    words_per_second: float
    ms_per_sentence: float
    sentence_count: int
    threads: int
    beam: int
    shortlist_active: bool
    startup_seconds: float
    target_tokens: int = 0
    target_words_per_second: float = 0.0

    def to_dict(self) -> dict:
        return asdict(self)


def _report(engine: Engine, results: Sequence[TranslationResult], wall: float, threads: int,
            beam: int) -> BenchReport:
    src = sum(r.src_tokens for r in results)
    trg = sum(len(r.text.split()) for r in results)
    wall = max(wall, 1e-9)
    return BenchReport(total_tokens=src, wall_seconds=wall, words_per_second=src / wall,
                       ms_per_sentence=1000.0 * wall / len(results), sentence_count=len(results),
                       threads=threads, beam=beam, shortlist_active=engine.shortlist_active,
                       startup_seconds=engine.startup_seconds, target_tokens=trg,
                       target_words_per_second=trg / wall)


def throughput_bench(engine: Engine, corpus: Sequence[str], threads: int,
                     warmup: bool = False) -> tuple[BenchReport, list[TranslationResult]]:
    if len(corpus) == 0:
        raise ValueError("benchmark corpus is empty")
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    if warmup:
        engine.translate_corpus(corpus, threads=threads)
    t0 = time.perf_counter()
    results = engine.translate_corpus(corpus, threads=threads)
    wall = time.perf_counter() - t0
    return _report(engine, results, wall, threads, engine.opts.beam_size), results


def latency_bench(engine: Engine, corpus: Sequence[str],
                  warmup: bool = False) -> tuple[BenchReport, list[TranslationResult]]:
    """Sentences strictly one at a time (batch of one per call)."""
    if len(corpus) == 0:
        raise ValueError("benchmark corpus is empty")
    if warmup:
        for line in corpus:
            engine.translate_line(line)
    t0 = time.perf_counter()
    results = [engine.translate_line(line) for line in corpus]
    wall = time.perf_counter() - t0
    return _report(engine, results, wall, 1, engine.opts.beam_size), results


SWEEP_HEADER = ["beam", "words_per_second", "bleu", "mean_model_score"]


def beam_sweep(engine: Engine, corpus: Sequence[str], beams: Sequence[int], references=None,
               threads: int | None = None) -> list[dict]:
    """Throughput per beam size (bleu is not computed by this package)."""
    if len(beams) == 0:
        raise ValueError("beam list is empty")
    if any(b < 1 for b in beams):
        raise ValueError(f"beam sizes must be >= 1, got {list(beams)}")
    if references is not None and len(references) != len(corpus):
        raise ValueError(f"line count mismatch: {len(corpus)} corpus vs {len(references)} references")
    rows = []
    for beam in beams:
        opts = engine.with_options(beam_size=beam)
        t0 = time.perf_counter()
        results = engine.translate_corpus(corpus, opts=opts)
        wall = max(time.perf_counter() - t0, 1e-9)
        rows.append({"beam": beam, "words_per_second": sum(r.src_tokens for r in results) / wall, "bleu": None,
                     "mean_model_score": sum(r.score for r in results) / len(results)})
    return rows
