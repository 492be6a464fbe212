"""Measurement API of the package: throughput, latency and beam sweeps over an
Engine (drop-in for beamnmt.bench, reference pkg/src/beamnmt/bench.py:23-140).

Definitions kept from the reference so reports compare one to one:
`words_per_second` is post-BPE SOURCE tokens per second of decode wall time
(bench.py:46-51), model loading is excluded and reported as
`startup_seconds`, latency decodes strictly one sentence per call.  Added for
the GPU decoder: `target_words_per_second` (1-best target tokens, final
`</s>` excluded -- the B200 headline metric) and `device_seconds`, the
decoder's own CUDA-event time over the engine calls of the measurement
(the part of the wall time spent on the device).
"""

from __future__ import annotations

import time
from dataclasses import asdict, dataclass
from typing import Callable, Sequence

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
    device_seconds: float = 0.0

    def to_dict(self) -> dict:
        return asdict(self)


class _Measured:
    """Runs `fn` (returning the results and the device milliseconds of its
    engine calls) once, after an optional untimed warm-up call."""

    def __init__(self, fn: Callable[[], tuple[list[TranslationResult], float]], warmup: bool):
        if warmup:
            fn()
        t0 = time.perf_counter()
        self.results, self.device_ms = fn()
        self.wall = max(time.perf_counter() - t0, 1e-9)

    def report(self, engine: Engine, threads: int, beam: int) -> BenchReport:
        res = self.results
        src = sum(r.src_tokens for r in res)
        trg = sum(len(r.text.split()) for r in res)
        return BenchReport(total_tokens=src, wall_seconds=self.wall, words_per_second=src / self.wall,
                           ms_per_sentence=1e3 * self.wall / len(res), sentence_count=len(res), threads=threads,
                           beam=beam, shortlist_active=engine.shortlist_active,
                           startup_seconds=engine.startup_seconds, target_tokens=trg,
                           target_words_per_second=trg / self.wall, device_seconds=self.device_ms / 1e3)


def _device_ms(engine: Engine) -> float:
    """Device time of the engine's last call: its devices decode concurrently,
    so the longest one (empty calls decode nothing)."""
    return max(engine.last_stats.get("device_ms") or [0.0])


def _check_corpus(corpus: Sequence[str]) -> None:
    if len(corpus) == 0:
        raise ValueError("benchmark corpus is empty")


def throughput_bench(engine: Engine, corpus: Sequence[str], threads: int,
                     warmup: bool = False) -> tuple[BenchReport, list[TranslationResult]]:
    """The whole corpus through one translate_corpus call (the GPU engine
    batches it into length buckets; `threads` is kept for the reference's
    signature and report)."""
    _check_corpus(corpus)
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")

    def once():
        res = engine.translate_corpus(corpus, threads=threads)
        return res, _device_ms(engine)

    m = _Measured(once, warmup)
    return m.report(engine, threads, engine.opts.beam_size), m.results


def latency_bench(engine: Engine, corpus: Sequence[str],
                  warmup: bool = False) -> tuple[BenchReport, list[TranslationResult]]:
    """One sentence per translate_line call, in corpus order."""
    _check_corpus(corpus)

    def serial():
        out, dev = [], 0.0
        for line in corpus:
            out.append(engine.translate_line(line))
            dev += _device_ms(engine)
        return out, dev

    m = _Measured(serial, warmup)
    return m.report(engine, 1, engine.opts.beam_size), m.results


SWEEP_HEADER = ["beam", "words_per_second", "bleu", "mean_model_score"]


def beam_sweep(engine: Engine, corpus: Sequence[str], beams: Sequence[int], references=None,
               threads: int | None = None) -> list[dict]:
    """Source words/s and mean model score per beam size.  BLEU is outside
    the decoder's scope: the column is kept and left empty."""
    if not len(beams):
        raise ValueError("beam list is empty")
    bad = [b for b in beams if b < 1]
    if bad:
        raise ValueError(f"beam sizes must be >= 1, got {list(beams)}")
    if references is not None and len(references) != len(corpus):
        raise ValueError(f"line count mismatch: {len(corpus)} corpus vs {len(references)} references")
    table = []
    for beam in beams:
        opts = engine.with_options(beam_size=beam)
        m = _Measured(lambda: (engine.translate_corpus(corpus, opts=opts), 0.0), False)
        res = m.results
        table.append(dict(zip(SWEEP_HEADER, (beam, sum(r.src_tokens for r in res) / m.wall, None,
                                             sum(r.score for r in res) / len(res)))))
    return table
