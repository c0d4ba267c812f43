"""The C-ABI library builds, loads without a GPU and exports every symbol that
include/optimus_b200.h declares; argument validation runs host-side."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_24832_b200 import _lib
from paper_2605_24832_b200.errors import ConfigError

HEADER = Path(__file__).resolve().parents[1] / "include" / "optimus_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(optimus_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared_symbols()
    for n in ("optimus_kv_append", "optimus_attn_plan", "optimus_paged_attn",
              "optimus_unmask_partials", "optimus_unmask_finalize"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version_and_validation_without_gpu():
    lib = _lib.load()
    assert lib.optimus_version() == 100
    # bad head_dim is rejected before any device work
    st = lib.optimus_paged_attn(None, 0, 1, None, None, 1, None, None, None, None, None, None, 1,
                                None, None, 1, None, 0, 32, 8, 8, 96, 16, 1.0, None, 0, None, None, 1, None)
    assert st == _lib.OPTIMUS_EINVAL
    assert "head_dim" in _lib.last_error()
    with pytest.raises(ConfigError):
        _lib.check(st, "optimus_paged_attn")
    # empty append is a no-op that needs no device
    assert lib.optimus_kv_append(None, None, 1024, None, None, None, None, 1, 0, 8, 128, 16,
                                 None, None, 1, None, 1, None) == 0
