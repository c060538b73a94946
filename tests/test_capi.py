"""The C-ABI library loads, exports every symbol include/hetbridge.h declares,
and follows the status convention (ErrorCode ordinal + 1). No compute calls."""
import ctypes
import os
import re

from helpers import ROOT
from paper_2605_27678_b200 import _lib


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hetbridge.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == syms


def test_status_convention_matches_reference_error_codes():
    L = _lib.lib()
    names = ["RankOutOfModule", "CoordOutOfBounds", "IndivisibleBatch", "PartialOverlap", "NonIntegerFan",
             "PlanInfeasible", "ShardIntervalMismatch", "MissingSourceShard", "GradIntervalMismatch",
             "UnknownMicrobatch"]
    for i, n in enumerate(names):
        assert L.hb_error_name(i + 1).decode() == n
    assert L.hb_error_name(0).decode() == "OK"
    assert L.hb_error_name(25).decode() == "CudaError"
    assert L.hb_abi_version() == 7


def test_error_message_and_no_exception_across_abi():
    L = _lib.lib()
    lay = _lib.Layout(b"enc", 4, 1, 1, 2, 8)
    c = (ctypes.c_int * 4)()
    st = L.hb_coord_of_rank(ctypes.byref(lay), 7, c)
    assert st == 1
    assert "outside module 'enc'" in _lib.last_error()
    assert L.hb_coord_of_rank(None, 0, c) == 24  # null layout -> InvalidArgument


def test_exec_create_validates_before_touching_cuda():
    L = _lib.lib()
    e = _lib.Edge(_lib.Layout(b"a", 1, 1, 1, 2, 0), _lib.Layout(b"b", 1, 1, 1, 2, 0), 2, 4)
    p = ctypes.c_void_p()
    assert L.hb_plan_create(ctypes.byref(e), ctypes.byref(p)) == 0
    x = ctypes.c_void_p()
    m = (ctypes.c_int * 2)(0, 0)
    st = L.hb_exec_create(p, None, 0, 0, m, 2, None, ctypes.byref(x))  # n_gpus = 0
    assert st == 24 and not x.value
    L.hb_plan_destroy(p)


def test_header_has_no_cxx_or_torch_types():
    with open(os.path.join(ROOT, "include", "hetbridge.h")) as f:
        text = f.read()
    assert 'extern "C"' in text
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    for bad in ("std::", "torch", "at::", "c10", "template", "class "):
        assert bad not in text
