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


def _build_c_example(tmp_path, q):
    """Compile examples/qtt_c_example.c as plain C99 against include/qtt.h."""
    import shutil
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "qtt_c_example")
    libdir = os.path.dirname(q.library_path())
    cmd = [gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(root, "include"),
           "-I/usr/local/cuda/include", os.path.join(root, "examples", "qtt_c_example.c"),
           "-L" + libdir, "-lqtt_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    env = dict(os.environ, LD_LIBRARY_PATH=libdir + ":/usr/local/cuda/lib64:" + os.environ.get("LD_LIBRARY_PATH", ""))
    return exe, env


def test_c_example_compiles_and_plans(tmp_path, q):
    """The header is valid C99 and the library links from plain C; the host-only
    planner runs without a GPU."""
    exe, env = _build_c_example(tmp_path, q)
    r = subprocess.run([exe, "--plan"], capture_output=True, text=True, env=env)
    assert r.returncode == 0 and "QTT_SUCCESS" in r.stdout, r.stdout + r.stderr


def test_bounds_checked_build_compiles(tmp_path):
    """The -DQTT_BOUNDS_CHECK debug build (the stand-in for compute-sanitizer,
    DESIGN.md §10) still compiles and carries trap instructions; the production
    library carries none."""
    import shutil
    import sys
    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        pytest.skip("no nvcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = str(tmp_path / "libqtt_checked.so")
    env = dict(os.environ, QTT_EXTRA_NVFLAGS="-DQTT_BOUNDS_CHECK", QTT_LIB_OUT=lib,
               QTT_OBJ_DIR=str(tmp_path / "obj"))
    r = subprocess.run([sys.executable, "-m", "paper_1511_06029_b200.build", "--force"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert sass.count("BPT.TRAP") > 100
