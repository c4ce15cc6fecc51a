"""C-ABI checks that need no GPU (-m "not gpu"): the in-tree library loads,
exports every symbol include/qtt.h declares, and validates arguments before
touching the device.  No compute calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    from paper_1511_06029_b200 import build
    build.build()
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


def header_functions():
    src = open(os.path.join(ROOT, "include", "qtt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qtt_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(q):
    declared = header_functions()
    assert len(declared) >= 10
    assert sorted(q.SYMBOLS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", q.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (qtt_[a-z_]+)", out))
    for name in declared:
        assert name in exported, name
        assert hasattr(q._lib.load(), name)


def test_library_is_sm100a(q):
    out = subprocess.run(["cuobjdump", "--list-elf", q.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", q.library_path()], capture_output=True, text=True).stdout
    assert "DMMA" in sass          # FP64 tensor-core MMA
    assert "UBLKCP" in sass        # TMA bulk copy


def test_status_strings(q):
    assert q.qtt_status_string(0) == "QTT_SUCCESS"
    assert q.qtt_status_string(1) == "QTT_ERROR_INVALID_VALUE"
    assert q.qtt_status_string(4) == "QTT_ERROR_CUDA"
    assert q.qtt_status_string(99) == "QTT_ERROR_UNKNOWN"


def test_create_validation_without_device(q):
    lib = q._lib.load()
    h = C.c_void_p()
    core = np.zeros((1, 2, 2, 1))
    ptrs = (C.c_void_p * 1)(core.ctypes.data)
    # d = 0, bad ranks, null cores: rejected before any device call
    assert lib.qtt_create(C.byref(h), 0, (C.c_int64 * 1)(1), ptrs) == 1
    assert lib.qtt_create(C.byref(h), 1, (C.c_int64 * 2)(2, 1), ptrs) == 1
    assert lib.qtt_create(C.byref(h), 1, (C.c_int64 * 2)(1, 1), None) == 1
    assert lib.qtt_create(C.byref(h), 31, (C.c_int64 * 32)(*([1] * 32)), ptrs) == 1
    assert lib.qtt_create(None, 1, (C.c_int64 * 2)(1, 1), ptrs) == 1
    assert h.value is None
    # null handle
    assert lib.qtt_apply(None, None, None, 1, None) == 1
    assert lib.qtt_destroy(None) == 0
    import torch
    if not torch.cuda.is_available():
        # valid arguments, but no CUDA device: fails loudly, no CPU fallback
        st = lib.qtt_create(C.byref(h), 1, (C.c_int64 * 2)(1, 1), ptrs)
        assert st in (2, 4) and h.value is None


def test_python_validation(q):
    with pytest.raises(ValueError):
        q.qtt_create([np.zeros((1, 2, 2, 3))], ranks=[1, 1])
    with pytest.raises(ValueError):
        q.qtt_create([])
