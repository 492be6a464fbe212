"""The C-ABI library: builds, loads, exports exactly what include/amun_b200.h
declares, and fails loudly (no CPU fallback) without a GPU.  CPU only."""

from __future__ import annotations

import re
import subprocess

import pytest

from conftest import REPO
from paper_1610_01108_b200 import _lib

HEADER = REPO / "include" / "amun_b200.h"


def declared_functions() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(amun_\w+)\s*\(", text, flags=re.M))


def test_header_and_binding_agree():
    assert declared_functions() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(amun_\w+)\b", out))
    assert declared_functions() <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version():
    assert _lib.load().amun_version() == 1


def test_no_device_raises_instead_of_falling_back():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        _lib.device_count()


def test_invalid_arguments_map_to_value_error():
    lib = _lib.load()
    st = lib.amun_model_create(0, None, None, 0, None)
    assert st == _lib.AMUN_ERR_INVALID
    with pytest.raises(ValueError, match="null argument"):
        _lib.check(st)
