"""CPU: the C-ABI library is built in-tree, loads, and exports every entry point the header
declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "agile_b200.h")


def _declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(agile_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("agile_create", "agile_destroy", "agile_store_attach", "agile_run_seq", "agile_run_reads",
                 "agile_run_loop", "agile_embbag", "agile_embbag_host", "agile_stats", "agile_event_log",
                 "agile_last_error", "agile_sync"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as g
    g.build()
    lib = ctypes.CDLL(g.LIB)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2504_19365_b200 import _lib
    assert set(_declared()) <= set(_lib.SIGNATURES)


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2504_19365_b200 import AgileSystem
    from paper_2504_19365_b200.errors import AgileError
    with pytest.raises(AgileError, match="no CUDA device"):
        AgileSystem(device=0)
