"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libamun_b200.so; everything else runs on the CPU-only dev container."""

from __future__ import annotations

import os

# Oracle bit-identity with the reference assumes single-threaded OpenBLAS
# (the goldens were generated that way, like engine.py:190 pins it).
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

# numpy may already have been imported (by a pytest plugin) before the env
# vars above took effect: pin BLAS to one thread at runtime as well.
_BLAS_LIMIT = threadpool_limits(limits=1)

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))

from paper_1610_01108_b200.model import ModelConfig, random_model  # noqa: E402

FULL = ModelConfig(v_src=30000, v_trg=30000, d_emb=500, d_h=1024, d_att=1024)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libamun_b200.so")


def tiny_model(seed: int, v_src: int = 5, v_trg: int = 5, d: int = 4):
    return random_model(ModelConfig(v_src=v_src, v_trg=v_trg, d_emb=d, d_h=d, d_att=d), seed)


@lru_cache(maxsize=1)
def golden_tiny() -> dict:
    return json.loads((GOLDEN / "tiny.json").read_text())


@lru_cache(maxsize=1)
def golden_tiny_arrays() -> dict:
    with np.load(GOLDEN / "tiny.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def golden_full() -> dict:
    return json.loads((GOLDEN / "full.json").read_text())


@lru_cache(maxsize=None)
def golden_fullset(name: str) -> dict:
    """Reference 1-best of a whole headline workload (make_golden_fullset.py)."""
    with np.load(GOLDEN / f"fullset_{name}.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def golden_shortlist() -> dict:
    """Reference shortlist decodes (make_golden_shortlist.py)."""
    with np.load(GOLDEN / "shortlist_sets.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def golden_ensemble() -> dict:
    """Reference full-size ensemble decodes (make_golden_ensemble.py)."""
    with np.load(GOLDEN / "ensemble_sets.npz") as z:
        return {k: z[k] for k in z.files}


def fullset_src_sha(corpus) -> str:
    import hashlib

    hs = hashlib.sha256()
    for s in corpus:
        hs.update(np.asarray(s, np.int32).tobytes())
        hs.update(b"|")
    return hs.hexdigest()


@lru_cache(maxsize=1)
def full_model():
    """random_model(emb500/hid1024/30k, seed 1) — the model every full-size
    golden fixture was produced with."""
    return random_model(FULL, 1)


@pytest.fixture(scope="session")
def gpu():
    from paper_1610_01108_b200 import _lib

    try:
        n = _lib.device_count()
    except RuntimeError as e:  # pragma: no cover - only on a box without a GPU
        pytest.fail(f"GPU test selected but no CUDA device: {e}")
    assert n >= 1
    return 0
