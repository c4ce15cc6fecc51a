"""B200-native QTT apply: y = A x for a matrix A in Quantized Tensor-Train form.

Thin Python binding over the C ABI in ``include/qtt.h`` (``libqtt_b200.so``):
argument marshalling only -- every step of PAPER.md Alg. 2 runs
in the library's CUDA kernels.  PyTorch provides device memory and streams.
There is no CPU fallback: without the built library, or without an sm_100
device, calls raise.

Layout (readings R1, R2, R8): ``cores[k]`` has shape
``(r_k, 2, 2, r_{k+1})`` = ``[alpha_{k-1}][i_k][j_k][alpha_k]`` with i_k the row
digit; digits are LSB-first.  A batch of right-hand sides is a tensor of
shape ``(nrhs, N)`` (row s = RHS s), whose memory image is the column-major
``N x nrhs`` matrix of the ABI.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import QttError, SYMBOLS

__all__ = [
    "QttOperator", "QttError", "qtt_create", "qtt_create_ex", "qtt_plan_stages", "plan_stages", "qtt_apply", "qtt_apply_ws", "qtt_apply_host",
    "qtt_workspace_size", "qtt_get_info", "qtt_get_stage", "qtt_get_stage_split", "qtt_get_apply_plan", "qtt_set_stage_timing",
    "qtt_stage_times", "qtt_destroy", "qtt_status_string", "library_path", "SYMBOLS",
    "morton_pack", "morton_unpack", "QttProduct",
]

VARIANT_NAMES = {0: "generic", 1: "dmma", 2: "merged", 3: "wide", 4: "small", 5: "diag", 6: "fused"}
MAX_STAGE_LEVELS = 10


def library_path() -> str:
    return _lib.LIB_PATH


def _ptr(t) -> int:
    return int(t.data_ptr())


_TORCH = None


def _torch():
    """torch, imported on first use (the binding's import does not need it)."""
    global _TORCH
    if _TORCH is None:
        import torch
        _TORCH = torch
    return _TORCH


def _stream_handle(stream) -> int | None:
    if stream is None:
        return int(_torch().cuda.current_stream().cuda_stream) or None
    if isinstance(stream, int):
        return stream or None
    return int(stream.cuda_stream) or None


# ----------------------------------------------------------------- C names
def qtt_status_string(code: int) -> str:
    return _lib.load().qtt_status_string(code).decode()


def _marshal_cores(cores, ranks):
    d = len(cores)
    if d < 1:
        raise ValueError("need at least one core")
    arrs = [np.ascontiguousarray(np.asarray(G, dtype=np.float64)) for G in cores]
    if ranks is None:
        ranks = [arrs[0].shape[0]] + [a.shape[3] for a in arrs]
    ranks = [int(r) for r in ranks]
    if len(ranks) != d + 1:
        raise ValueError("ranks must have d+1 entries")
    for k, a in enumerate(arrs):
        if a.shape != (ranks[k], 2, 2, ranks[k + 1]):
            raise ValueError(f"core {k + 1} has shape {a.shape}, expected {(ranks[k], 2, 2, ranks[k + 1])}")
    return arrs, ranks


def qtt_create_ex(cores, ranks=None, max_stage_levels: int = MAX_STAGE_LEVELS) -> int:
    """cores: list of d float64 arrays (r_{k-1}, 2, 2, r_k). Returns a handle (int)."""
    lib = _lib.load()
    arrs, ranks = _marshal_cores(cores, ranks)
    d = len(arrs)
    r_arr = (C.c_int64 * (d + 1))(*ranks)
    p_arr = (C.c_void_p * d)(*[a.ctypes.data for a in arrs])
    h = C.c_void_p()
    _lib.check("qtt_create_ex", lib.qtt_create_ex(C.byref(h), d, r_arr, p_arr, int(max_stage_levels)))
    return int(h.value)


def qtt_create(cores, ranks=None) -> int:
    """cores: list of d float64 arrays (r_{k-1}, 2, 2, r_k). Returns a handle (int)."""
    lib = _lib.load()
    arrs, ranks = _marshal_cores(cores, ranks)
    d = len(arrs)
    r_arr = (C.c_int64 * (d + 1))(*ranks)
    p_arr = (C.c_void_p * d)(*[a.ctypes.data for a in arrs])
    h = C.c_void_p()
    _lib.check("qtt_create", lib.qtt_create(C.byref(h), d, r_arr, p_arr))
    return int(h.value)


def qtt_plan_stages(ranks, smem_optin: int = 0, max_stage_levels: int = MAX_STAGE_LEVELS):
    """Host-only: the stage schedule for a rank profile, as [(k_first, k_last, variant_code)]."""
    lib = _lib.load()
    ranks = [int(r) for r in ranks]
    d = len(ranks) - 1
    if d < 1:
        raise ValueError("need d >= 1")
    r_arr = (C.c_int64 * (d + 1))(*ranks)
    n = C.c_int()
    a, b, v = (C.c_int * d)(), (C.c_int * d)(), (C.c_int * d)()
    _lib.check("qtt_plan_stages", lib.qtt_plan_stages(d, r_arr, int(smem_optin), int(max_stage_levels),
                                                      C.byref(n), a, b, v))
    return [(a[i], b[i], v[i]) for i in range(n.value)]


def stage_super_core(cores, k_first: int, k_last: int) -> np.ndarray:
    """Host-only: the super-core W[a][ii][jj][b] of levels k_first..k_last (1-based)."""
    arrs, ranks = _marshal_cores(cores, None)
    d = len(arrs)
    L = k_last - k_first + 1
    W = np.empty((ranks[k_first - 1], 1 << L, 1 << L, ranks[k_last]), dtype=np.float64)
    _lib.check("qtt_stage_super_core", _lib.load().qtt_stage_super_core(
        d, (C.c_int64 * (d + 1))(*ranks), (C.c_void_p * d)(*[a.ctypes.data for a in arrs]),
        int(k_first), int(k_last), W.ctypes.data))
    return W


def plan_stages(ranks, max_stage_levels: int = MAX_STAGE_LEVELS):
    """Like qtt_plan_stages with variant names and split-K factors:
    [{'k_first', 'k_last', 'variant', 'ksplit'}] (host only)."""
    lib = _lib.load()
    ranks = [int(r) for r in ranks]
    d = len(ranks) - 1
    if d < 1:
        raise ValueError("need d >= 1")
    n = C.c_int()
    a, b, v, k = (C.c_int * d)(), (C.c_int * d)(), (C.c_int * d)(), (C.c_int * d)()
    _lib.check("qtt_plan_stages_split", lib.qtt_plan_stages_split(
        d, (C.c_int64 * (d + 1))(*ranks), 0, int(max_stage_levels), C.byref(n), a, b, v, k))
    return [dict(k_first=a[i], k_last=b[i], variant=VARIANT_NAMES.get(v[i], str(v[i])), ksplit=k[i])
            for i in range(n.value)]


def qtt_apply(h: int, x, y, nrhs: int, stream=None) -> None:
    _lib.check("qtt_apply", _lib.load().qtt_apply(h, _ptr(x), _ptr(y), int(nrhs), _stream_handle(stream)))


def qtt_apply_ws(h: int, x, y, nrhs: int, ws, ws_bytes: int, stream=None) -> None:
    _lib.check("qtt_apply_ws", _lib.load().qtt_apply_ws(
        h, _ptr(x), _ptr(y), int(nrhs), _ptr(ws) if ws is not None else None, int(ws_bytes),
        _stream_handle(stream)))


def qtt_apply_host(h: int, x: np.ndarray, y: np.ndarray, nrhs: int, stream=None) -> None:
    _lib.check("qtt_apply_host", _lib.load().qtt_apply_host(
        h, x.ctypes.data, y.ctypes.data, int(nrhs), _stream_handle(stream)))


def qtt_workspace_size(h: int, nrhs: int) -> int:
    b = C.c_size_t()
    _lib.check("qtt_workspace_size", _lib.load().qtt_workspace_size(h, int(nrhs), C.byref(b)))
    return int(b.value)


def qtt_get_info(h: int) -> dict:
    d, N, mr, fl, nl = C.c_int(), C.c_int64(), C.c_int64(), C.c_double(), C.c_int()
    _lib.check("qtt_get_info", _lib.load().qtt_get_info(
        h, C.byref(d), C.byref(N), C.byref(mr), C.byref(fl), C.byref(nl)))
    return dict(d=d.value, N=N.value, max_rank=mr.value, flops_per_rhs=fl.value, launches_per_apply=nl.value)


def qtt_get_stage(h: int, s: int) -> dict:
    a, b, v = C.c_int(), C.c_int(), C.c_int()
    _lib.check("qtt_get_stage", _lib.load().qtt_get_stage(h, int(s), C.byref(a), C.byref(b), C.byref(v)))
    return dict(k_first=a.value, k_last=b.value, variant=VARIANT_NAMES.get(v.value, str(v.value)))


def qtt_get_apply_plan(h: int, nrhs: int = 1):
    """(launches, [{'k_first', 'k_last', 'variant'}]) of an apply with nrhs RHS (host only)."""
    info = qtt_get_info(h)
    n = max(info["d"], 1)
    launches, ns = C.c_int(), C.c_int()
    a, b, v = (C.c_int * n)(), (C.c_int * n)(), (C.c_int * n)()
    _lib.check("qtt_get_apply_plan", _lib.load().qtt_get_apply_plan(
        h, int(nrhs), C.byref(launches), C.byref(ns), C.cast(a, C.c_void_p), C.cast(b, C.c_void_p),
        C.cast(v, C.c_void_p)))
    return launches.value, [dict(k_first=a[i], k_last=b[i], variant=VARIANT_NAMES.get(v[i], str(v[i])))
                            for i in range(ns.value)]


def qtt_get_stage_split(h: int, s: int, nrhs: int = 1) -> int:
    k = C.c_int()
    _lib.check("qtt_get_stage_split", _lib.load().qtt_get_stage_split(h, int(s), int(nrhs), C.byref(k)))
    return k.value


def qtt_set_stage_timing(h: int, enable: bool) -> None:
    _lib.check("qtt_set_stage_timing", _lib.load().qtt_set_stage_timing(h, int(bool(enable))))


def qtt_stage_times(h: int, n_stages: int):
    ms = (C.c_float * n_stages)()
    n = C.c_int()
    _lib.check("qtt_stage_times", _lib.load().qtt_stage_times(h, ms, int(n_stages), C.byref(n)))
    return [float(v) for v in ms], int(n.value)


def qtt_destroy(h: int) -> None:
    _lib.check("qtt_destroy", _lib.load().qtt_destroy(h))


def _grid_args(t, dim: int, levels: int):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous float64 CUDA tensor")
    N = 1 << (dim * levels)
    if t.numel() % N or t.numel() == 0:
        raise ValueError(f"tensor size {t.numel()} is not a multiple of N = {N}")
    return t.numel() // N


def morton_pack(grid, dim: int, levels: int, out=None, stream=None):
    """Natural-order grid(s) (C order [z][y][x], nrhs blocks) -> QTT-order vectors (nrhs, N)."""
    import torch
    nrhs = _grid_args(grid, dim, levels)
    N = 1 << (dim * levels)
    y = torch.empty((nrhs, N), dtype=torch.float64, device=grid.device) if out is None else out
    _grid_args(y, dim, levels)
    if y.numel() != grid.numel():
        raise ValueError("out must have as many elements as grid")
    _lib.check("qtt_morton_pack", _lib.load().qtt_morton_pack(
        _ptr(grid), _ptr(y), int(dim), int(levels), int(nrhs), _stream_handle(stream)))
    return y


def morton_unpack(x, dim: int, levels: int, out=None, stream=None):
    """QTT-order vectors (nrhs, N) -> natural-order grids, same shape as x unless out is given."""
    import torch
    nrhs = _grid_args(x, dim, levels)
    y = torch.empty_like(x) if out is None else out
    _grid_args(y, dim, levels)
    if y.numel() != x.numel():
        raise ValueError("out must have as many elements as x")
    _lib.check("qtt_morton_unpack", _lib.load().qtt_morton_unpack(
        _ptr(x), _ptr(y), int(dim), int(levels), int(nrhs), _stream_handle(stream)))
    return y


# ----------------------------------------------------------------- object API
class QttOperator:
    """A QTT matrix resident on the current CUDA device; ``apply`` computes y = A x."""

    def __init__(self, cores, ranks=None, max_stage_levels: int | None = None, fused: bool = True):
        self._h = None
        self._apply_fn = _lib.load().qtt_apply          # the C entry point (argtypes set by _lib)
        if max_stage_levels is None:
            self._h = qtt_create(cores, ranks)
        else:
            self._h = qtt_create_ex(cores, ranks, max_stage_levels)
        if not fused:
            self.set_fused(False)
        info = qtt_get_info(self._h)
        import torch
        self.device = torch.device("cuda", torch.cuda.current_device())   # where qtt_create put the cores
        self.d = info["d"]
        self.N = info["N"]
        self.max_rank = info["max_rank"]
        self.flops_per_rhs = info["flops_per_rhs"]
        self.launches_per_apply = info["launches_per_apply"]
        self.ranks = [int(np.shape(cores[0])[0])] + [int(np.shape(G)[3]) for G in cores]

    @classmethod
    def transpose_of(cls, cores, max_stage_levels: int | None = None) -> "QttOperator":
        """The operator A^T for A given by `cores`: the row and column digits of
        every core swapped, G^T_k[a][j][i][b] = G_k[a][i][j][b] (the QTT
        definition P:953-962 read with i and j exchanged).  Host-side reshuffle
        of the cores; the apply is the ordinary one."""
        arrs, ranks = _marshal_cores(cores, None)
        return cls([np.ascontiguousarray(np.transpose(G, (0, 2, 1, 3))) for G in arrs], ranks,
                   max_stage_levels)

    @classmethod
    def from_ttb1(cls, path, max_stage_levels: int | None = None) -> "QttOperator":
        """Operator from a TTB1 core file (``ttb1.load_operator``)."""
        from . import ttb1
        ranks, cores = ttb1.load_operator(path)
        return cls(cores, ranks, max_stage_levels)

    @property
    def handle(self) -> int:
        if self._h is None:
            raise ValueError("operator is closed")
        return self._h

    def _check_x(self, x):
        torch = _torch()
        if not isinstance(x, torch.Tensor):
            raise ValueError("x must be a torch.Tensor on a CUDA device")
        if x.dtype != torch.float64:
            raise ValueError(f"x must be float64, got {x.dtype}")
        if not x.is_cuda:
            raise ValueError("x must be on a CUDA device")
        if x.dim() not in (1, 2) or x.shape[-1] != self.N:
            raise ValueError(f"x must have shape (N,) or (nrhs, N) with N={self.N}, got {tuple(x.shape)}")
        if not x.is_contiguous():
            raise ValueError("x must be contiguous")
        return 1 if x.dim() == 1 else int(x.shape[0])

    def apply(self, x, out=None, stream=None, workspace=None):
        torch = _torch()
        # the common call (a float64 CUDA tensor, out given, no workspace) takes a
        # lean path: every torch attribute access costs ~0.1-0.2 us, and at the
        # latency-bound sizes the host call is as long as the apply itself
        if (workspace is None and out is not None and type(x) is torch.Tensor and type(out) is torch.Tensor
                and x.dtype is torch.float64 and out.dtype is torch.float64 and x.is_cuda and out.is_cuda):
            shape = x.shape
            if (shape == out.shape and 1 <= len(shape) <= 2 and shape[-1] == self.N and x.is_contiguous()
                    and out.is_contiguous() and self._h is not None):
                nrhs = shape[0] if len(shape) == 2 else 1
                if nrhs >= 1:
                    code = self._apply_fn(self._h, x.data_ptr(), out.data_ptr(), nrhs, _stream_handle(stream))
                    if code:
                        raise QttError("qtt_apply", code)
                    return out
        nrhs = self._check_x(x)
        if nrhs < 1:
            raise ValueError("nrhs must be >= 1")
        y = torch.empty_like(x) if out is None else out
        if out is not None:
            if out.shape != x.shape or out.dtype != torch.float64 or not out.is_contiguous() or not out.is_cuda:
                raise ValueError("out must be a contiguous float64 CUDA tensor shaped like x")
        if workspace is None:
            qtt_apply(self.handle, x, y, nrhs, stream)
        else:
            qtt_apply_ws(self.handle, x, y, nrhs, workspace, workspace.numel() * workspace.element_size(), stream)
        return y

    __matmul__ = apply

    def compressed_matvec(self, b_cores, out=None, stream=None, cores_only: bool = False):
        """c = A b for b in QTT form (PAPER section 4.2).  b_cores: d arrays (r_{k-1}, 2, r_k).

        Returns the dense c (torch float64 tensor of N entries on the current device), or with
        cores_only=True the list of product cores (R_{k-1}, 2, R_k) as device tensors."""
        import torch
        bs = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in b_cores]
        if len(bs) != self.d:
            raise ValueError(f"need {self.d} cores, got {len(bs)}")
        br = [bs[0].shape[0]] + [v.shape[2] for v in bs]
        for k, v in enumerate(bs):
            if v.ndim != 3 or v.shape != (br[k], 2, br[k + 1]):
                raise ValueError(f"b core {k + 1} has shape {v.shape}")
        rb = (C.c_int64 * (self.d + 1))(*br)
        ptrs = (C.c_void_p * self.d)(*[v.ctypes.data for v in bs])
        cr = (C.c_int64 * (self.d + 1))()
        lib = _lib.load()
        if cores_only:
            R = [a * b for a, b in zip(self.ranks, br)]
            sizes = [R[k] * 2 * R[k + 1] for k in range(self.d)]
            buf = torch.empty(sum(sizes), dtype=torch.float64, device=self.device)
            _lib.check("qtt_compressed_matvec_cores", lib.qtt_compressed_matvec_cores(
                self.handle, rb, ptrs, _ptr(buf), buf.numel() * 8, cr, _stream_handle(stream)))
            out_cores, off = [], 0
            for k in range(self.d):
                out_cores.append(buf[off:off + sizes[k]].view(R[k], 2, R[k + 1]))
                off += sizes[k]
            return out_cores
        y = torch.empty(self.N, dtype=torch.float64, device=self.device) if out is None else out
        if y.numel() != self.N or y.dtype != torch.float64 or not y.is_cuda or not y.is_contiguous():
            raise ValueError("out must be a contiguous float64 CUDA tensor of N entries")
        _lib.check("qtt_compressed_matvec", lib.qtt_compressed_matvec(
            self.handle, rb, ptrs, _ptr(y), cr, _stream_handle(stream)))
        return y

    def apply_grid(self, grid, dim: int, out=None, stream=None):
        """y = A x with x, y natural-order grids (Morton pack / apply / unpack)."""
        import torch
        if self.d % dim:
            raise ValueError(f"dim={dim} does not divide d={self.d}")
        nrhs = _grid_args(grid, dim, self.d // dim)
        y = torch.empty_like(grid) if out is None else out
        _grid_args(y, dim, self.d // dim)
        if y.numel() != grid.numel():
            raise ValueError("out must have as many elements as grid")
        _lib.check("qtt_apply_grid", _lib.load().qtt_apply_grid(
            self.handle, _ptr(grid), _ptr(y), int(dim), int(nrhs), _stream_handle(stream)))
        return y

    def apply_host(self, x: np.ndarray, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if x.ndim not in (1, 2) or x.shape[-1] != self.N:
            raise ValueError(f"x must have shape (N,) or (nrhs, N) with N={self.N}")
        nrhs = 1 if x.ndim == 1 else x.shape[0]
        if out is None:
            y = np.empty_like(x)
        else:
            # the C side writes N * nrhs doubles at out's data pointer
            if (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != x.shape
                    or not out.flags.c_contiguous or not out.flags.writeable):
                raise ValueError(f"out must be a writeable C-contiguous float64 array of shape {x.shape}")
            y = out
        qtt_apply_host(self.handle, x, y, nrhs, stream)
        return y

    def workspace_size(self, nrhs: int = 1) -> int:
        return qtt_workspace_size(self.handle, nrhs)

    def stages(self, nrhs: int = 1):
        """The stages an apply with `nrhs` RHS runs: {'k_first', 'k_last', 'variant',
        'ksplit'} each (variant 'fused': all of them in one persistent launch)."""
        _, st = qtt_get_apply_plan(self.handle, nrhs)
        if st and st[0]["variant"] == "fused":
            return [dict(s_, ksplit=1) for s_ in st]
        return [dict(qtt_get_stage(self.handle, s), ksplit=qtt_get_stage_split(self.handle, s, nrhs))
                for s in range(self.launches_per_apply)]

    def set_fused(self, enable: bool = True):
        """Allow (default) or forbid the fused one-launch apply on this handle."""
        _lib.check("qtt_set_fused", _lib.load().qtt_set_fused(self.handle, 1 if enable else 0))

    def launches(self, nrhs: int = 1) -> int:
        """Kernel launches of one apply with `nrhs` RHS (1 for a fused apply)."""
        return qtt_get_apply_plan(self.handle, nrhs)[0]

    def stage_splits(self, nrhs: int = 1):
        """Split-K factor of every stage at `nrhs` (1 = unsplit)."""
        return [qtt_get_stage_split(self.handle, s, nrhs) for s in range(self.launches_per_apply)]

    def set_stage_timing(self, enable: bool = True):
        qtt_set_stage_timing(self.handle, enable)

    def stage_times(self):
        return qtt_stage_times(self.handle, self.launches_per_apply)

    def close(self):
        if self._h is not None:
            h, self._h = self._h, None
            qtt_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class QttProduct:
    """y = F_0 F_1 ... F_{n-1} x for QttOperator factors (applied right to left).

    The factors are referenced, not owned: keep them open while the product is used."""

    def __init__(self, factors):
        self._h = None
        if not factors:
            raise ValueError("need at least one factor")
        self.factors = list(factors)
        hs = (C.c_void_p * len(self.factors))(*[f.handle for f in self.factors])
        h = C.c_void_p()
        _lib.check("qtt_product_create", _lib.load().qtt_product_create(C.byref(h), len(self.factors), hs))
        self._h = int(h.value)
        self.N = self.factors[0].N
        self.flops_per_rhs = sum(f.flops_per_rhs for f in self.factors)

    def workspace_size(self, nrhs: int = 1) -> int:
        b = C.c_size_t()
        _lib.check("qtt_product_workspace_size", _lib.load().qtt_product_workspace_size(self._h, int(nrhs), C.byref(b)))
        return int(b.value)

    def apply(self, x, out=None, stream=None, workspace=None):
        import torch
        nrhs = self.factors[0]._check_x(x)
        y = torch.empty_like(x) if out is None else out
        if out is not None and (out.shape != x.shape or out.dtype != torch.float64 or not out.is_cuda
                                or not out.is_contiguous()):
            raise ValueError("out must be a contiguous float64 CUDA tensor shaped like x")
        if workspace is None:
            _lib.check("qtt_product_apply", _lib.load().qtt_product_apply(
                self._h, _ptr(x), _ptr(y), nrhs, _stream_handle(stream)))
        else:
            _lib.check("qtt_product_apply_ws", _lib.load().qtt_product_apply_ws(
                self._h, _ptr(x), _ptr(y), nrhs, _ptr(workspace),
                workspace.numel() * workspace.element_size(), _stream_handle(stream)))
        return y

    __matmul__ = apply

    def close(self):
        if self._h is not None:
            h, self._h = self._h, None
            _lib.load().qtt_product_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
