"""Multi-GPU QTT apply by top-bit sharding (NEXT-4).

One process per GPU.  With P = 2^s ranks, x and y are split into P contiguous
blocks of n = N/P entries by the top s index bits (Morton order: octree
subdomains).  Rank g runs its shard plan (``qtt_create_shard``): Alg. 2's
levels 1..d-s on its own block (they never pair bits across blocks,
PAPER.md P:1487-1496) and a projection of the result onto all P output
blocks with the top s cores, all in the library's kernels.  The one exchange
is a sum ReduceScatter of the [P][n] send buffers (NCCL over NVLink through
torch.distributed; plumbing only) -- or, with ``fused=True``, the projection
kernel stores each block straight into its owner's receive buffer (CUDA IPC
peer memory) and the owner sums the P slots in fixed order, ordered across
processes by interprocess CUDA events.

This module holds argument marshalling and the collective call; every flop
runs in libqtt_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from . import _marshal_cores, _ptr, _stream_handle, QttOperator

__all__ = ["ShardedQttOperator", "QttShard", "shard_projection", "exchange", "block_of"]


def shard_projection(cores, log2_parts: int, part: int) -> np.ndarray:
    """Host-only: c_{h,part} for every output block h, shape (P, r_{d-s})
    (``qtt_shard_projection``; no GPU needed)."""
    arrs, ranks = _marshal_cores(cores, None)
    d = len(arrs)
    P = 1 << log2_parts
    r = ranks[d - log2_parts]
    out = np.empty((P, r), dtype=np.float64)
    _lib.check("qtt_shard_projection", _lib.load().qtt_shard_projection(
        d, (C.c_int64 * (d + 1))(*ranks), (C.c_void_p * d)(*[a.ctypes.data for a in arrs]),
        int(log2_parts), int(part), out.ctypes.data))
    return out


def block_of(x, part: int, parts: int):
    """Rank `part`'s block of a full (nrhs, N) array: the entries whose top
    log2(parts) index bits equal `part` (a contiguous slice)."""
    n = x.shape[-1] // parts
    return x[..., part * n:(part + 1) * n]


def exchange(send, out, group=None):
    """Sum-ReduceScatter of send [nrhs][P][n] into out [nrhs][n] (block = this rank).

    NCCL: one reduce_scatter_tensor per RHS (block h of RHS s is contiguous).
    Backends without reduce_scatter (gloo) fall back to all_reduce + slice."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    for s in range(send.shape[0]):
        if backend == "nccl":
            dist.reduce_scatter_tensor(out[s], send[s].reshape(-1), op=dist.ReduceOp.SUM, group=group)
        else:
            buf = send[s].clone()
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
            out[s].copy_(buf[rank])
    return out


class QttShard:
    """Part `part` of 2^log2_parts of a QTT operator (``qtt_create_shard``): maps the
    part's block of x to its [nrhs][P][n] send buffer.  No collective here."""

    def __init__(self, cores, log2_parts: int, part: int):
        self._h = None
        arrs, ranks = _marshal_cores(cores, None)
        self.d = len(arrs)
        self.s = int(log2_parts)
        self.part = int(part)
        self.P = 1 << self.s
        self.N = 1 << self.d
        self.n = self.N >> self.s
        self.ranks = ranks
        h = C.c_void_p()
        _lib.check("qtt_create_shard", _lib.load().qtt_create_shard(
            C.byref(h), self.d, (C.c_int64 * (self.d + 1))(*ranks),
            (C.c_void_p * self.d)(*[a.ctypes.data for a in arrs]), self.s, self.part))
        self._h = int(h.value)

    def workspace_size(self, nrhs: int = 1) -> int:
        b = C.c_size_t()
        _lib.check("qtt_workspace_size", _lib.load().qtt_workspace_size(self._h, int(nrhs), C.byref(b)))
        return int(b.value)

    def stages(self, nrhs: int = 1):
        """Per launch: {'k_first', 'k_last', 'variant', 'ksplit'} (the last stage
        is the projection)."""
        from . import qtt_get_info, qtt_get_stage, qtt_get_stage_split
        n = qtt_get_info(self._h)["launches_per_apply"]
        return [dict(qtt_get_stage(self._h, i), ksplit=qtt_get_stage_split(self._h, i, nrhs)) for i in range(n)]

    def apply(self, x_local, send=None, stream=None, workspace=None):
        import torch
        xl = x_local if x_local.dim() == 2 else x_local.view(1, -1)
        if xl.dtype != torch.float64 or not xl.is_cuda or not xl.is_contiguous() or xl.shape[-1] != self.n:
            raise ValueError(f"x_local must be a contiguous float64 CUDA tensor with {self.n} columns")
        nrhs = xl.shape[0]
        if send is None:
            send = torch.empty((nrhs, self.P, self.n), dtype=torch.float64, device=xl.device)
        if workspace is None:
            _lib.check("qtt_shard_apply", _lib.load().qtt_shard_apply(
                self._h, _ptr(xl), _ptr(send), nrhs, _stream_handle(stream)))
        else:
            _lib.check("qtt_shard_apply_ws", _lib.load().qtt_shard_apply_ws(
                self._h, _ptr(xl), _ptr(send), nrhs, _ptr(workspace),
                workspace.numel() * workspace.element_size(), _stream_handle(stream)))
        return send

    # ---- fused exchange: projection stores straight into the parts' receive buffers
    def set_peers(self, recv_ptrs):
        """recv_ptrs[h]: device pointer (this process's mapping) of part h's receive
        buffer, [P][nrhs][n] doubles."""
        if len(recv_ptrs) != self.P:
            raise ValueError(f"need {self.P} receive buffers")
        arr = (C.c_void_p * self.P)(*[int(p) for p in recv_ptrs])
        _lib.check("qtt_shard_set_peers", _lib.load().qtt_shard_set_peers(self._h, arr, self.P))

    def apply_fused(self, x_local, stream=None):
        import torch
        xl = x_local if x_local.dim() == 2 else x_local.view(1, -1)
        if xl.dtype != torch.float64 or not xl.is_cuda or not xl.is_contiguous() or xl.shape[-1] != self.n:
            raise ValueError(f"x_local must be a contiguous float64 CUDA tensor with {self.n} columns")
        _lib.check("qtt_shard_apply_fused", _lib.load().qtt_shard_apply_fused(
            self._h, _ptr(xl), xl.shape[0], _stream_handle(stream)))

    @staticmethod
    def reduce(recv, out, stream=None, parts=None):
        """out = sum over the P slots of recv ([P][nrhs][n] tensor, or a raw device
        pointer with `parts` given), fixed order."""
        P = recv.shape[0] if parts is None else int(parts)
        src = _ptr(recv) if parts is None else int(recv)
        _lib.check("qtt_shard_reduce", _lib.load().qtt_shard_reduce(
            src, _ptr(out), P, int(out.numel()), _stream_handle(stream)))
        return out

    def close(self):
        if self._h is not None:
            h, self._h = self._h, None
            _lib.load().qtt_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def ipc_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    _lib.check("qtt_ipc_alloc", _lib.load().qtt_ipc_alloc(int(nbytes), C.byref(p)))
    return int(p.value)


def ipc_handle(ptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    _lib.check("qtt_ipc_get_handle", _lib.load().qtt_ipc_get_handle(int(ptr), C.addressof(buf)))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    buf = C.create_string_buffer(bytes(handle), 64)
    p = C.c_void_p()
    _lib.check("qtt_ipc_open", _lib.load().qtt_ipc_open(C.addressof(buf), C.byref(p)))
    return int(p.value)


class ShardedQttOperator:
    """y = A x with x, y sharded by the top index bits over the ranks of `group`.

    ``apply(x_local)`` takes this rank's block (shape (n,) or (nrhs, n)) and
    returns this rank's block of y.  World size must be a power of two; with
    one rank it is a plain QttOperator."""

    def __init__(self, cores, group=None, fused: bool = False, max_nrhs: int = 1):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world & (self.world - 1):
            raise ValueError(f"world size {self.world} is not a power of two")
        self.s = self.world.bit_length() - 1
        arrs, ranks = _marshal_cores(cores, None)
        self.d = len(arrs)
        self.N = 1 << self.d
        self.n = self.N >> self.s
        self.flops_per_rhs = 4.0 * sum(ranks[k] * ranks[k + 1] for k in range(self.d)) * self.N
        self._op = None
        self._shard = None
        self.fused = bool(fused) and self.s > 0
        self.max_nrhs = int(max_nrhs)
        self._recv = None
        self._peers = []
        self._ev_proj = self._ev_red = None
        self._peer_proj, self._peer_red = [], []
        self._hgroup = None
        if self.s == 0:
            self._op = QttOperator(arrs)
        else:
            self._shard = QttShard(arrs, self.s, self.rank)
        if self.fused:
            # every part's receive buffer [P][max_nrhs][n], mapped into every process (CUDA IPC)
            self._recv = ipc_alloc(self.world * self.max_nrhs * self.n * 8)
            handles = [None] * self.world
            dist.all_gather_object(handles, ipc_handle(self._recv), group=group)
            ptrs = []
            for r, hd in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self._recv)
                else:
                    p = ipc_open(hd)
                    self._peers.append(p)
                    ptrs.append(p)
            self._shard.set_peers(ptrs)
            # stream-ordered cross-process sync: interprocess CUDA events, one
            # "projection stored" and one "reduction done" per part
            import torch
            self._ev_proj = torch.cuda.Event(interprocess=True)
            self._ev_red = torch.cuda.Event(interprocess=True)
            evh = [None] * self.world
            dist.all_gather_object(evh, (self._ev_proj.ipc_handle(), self._ev_red.ipc_handle()), group=group)
            dev = torch.cuda.current_device()
            for r, (hp, hr) in enumerate(evh):
                if r != self.rank:
                    self._peer_proj.append(torch.cuda.Event.from_ipc_handle(dev, hp))
                    self._peer_red.append(torch.cuda.Event.from_ipc_handle(dev, hr))
            # host-only barriers (they order event records before the peers' waits)
            if dist.get_backend(group) == "gloo":
                self._hgroup = group
            else:
                ranks = list(range(dist.get_world_size())) if group is None else dist.get_process_group_ranks(group)
                self._hgroup = dist.new_group(ranks=ranks, backend="gloo")

    def workspace_size(self, nrhs: int = 1) -> int:
        return (self._op or self._shard).workspace_size(nrhs)

    def local_apply(self, x_local, send=None, stream=None, workspace=None):
        """The kernel part only: this rank's [nrhs][P][n] send buffer."""
        return self._shard.apply(x_local, send=send, stream=stream, workspace=workspace)

    def apply(self, x_local, out=None, stream=None, workspace=None, send=None):
        import torch
        if out is not None:
            nr = 1 if x_local.dim() == 1 else x_local.shape[0]
            if (not isinstance(out, torch.Tensor) or out.dtype != torch.float64 or not out.is_cuda
                    or not out.is_contiguous() or out.numel() != nr * self.n):
                raise ValueError(f"out must be a contiguous float64 CUDA tensor of {nr} x {self.n} entries")
        if self._op is not None:
            return self._op.apply(x_local, out=out, stream=stream, workspace=workspace)
        if self.fused:
            return self._apply_fused(x_local, out, stream)
        send = self.local_apply(x_local, send=send, stream=stream, workspace=workspace)
        y = torch.empty((send.shape[0], self.n), dtype=torch.float64, device=send.device) if out is None else out
        # the collective runs on the stream the shard kernels were enqueued on
        # (torch.distributed issues NCCL work on the current stream)
        st = torch.cuda.current_stream(send.device) if stream is None else stream
        with torch.cuda.stream(st):
            exchange(send, y.view(send.shape[0], self.n), self.group)
        return y if x_local.dim() == 2 else y.view(-1)

    def _apply_fused(self, x_local, out, stream):
        """Projection stores into every part's receive slot (peer memory), then
        each part sums its P slots in fixed order -- all stream-ordered, no
        device synchronisation:

          host barrier (every peer has recorded its previous "reduced" event)
          wait on the peers' "reduced" events (their previous reduction has
            read the slots this projection overwrites)
          fused local stages + projection; record "projected"
          host barrier (every peer has recorded "projected" for this apply)
          wait on the peers' "projected" events; reduce; record "reduced"

        The barriers are host-only (gloo): a stream wait captures an event's
        latest record at call time, so each wait must follow the peer's record
        call.  No kernel waits on another process's kernel."""
        import torch
        import torch.distributed as dist
        xl = x_local if x_local.dim() == 2 else x_local.view(1, -1)
        nrhs = xl.shape[0]
        if nrhs > self.max_nrhs:
            raise ValueError(f"nrhs {nrhs} > max_nrhs {self.max_nrhs} given at construction")
        st = torch.cuda.current_stream(xl.device) if stream is None else stream
        y = torch.empty((nrhs, self.n), dtype=torch.float64, device=xl.device) if out is None else out
        dist.barrier(group=self._hgroup)
        for ev in self._peer_red:
            st.wait_event(ev)
        self._shard.apply_fused(xl, stream=st)
        self._ev_proj.record(st)
        dist.barrier(group=self._hgroup)
        for ev in self._peer_proj:
            st.wait_event(ev)
        QttShard.reduce(self._recv, y.view(nrhs, self.n), stream=st, parts=self.world)
        self._ev_red.record(st)
        return y if x_local.dim() == 2 else y.view(-1)

    def close(self, sync: bool = True):
        """Free the shard and the exchange buffers.  With fused exchange, every
        part must call close() (collective: a device sync and a host barrier,
        so no peer still stores into our buffer).  The finaliser passes
        sync=False: it must not block on peers that may already be gone."""
        if self._ev_red is not None:
            if sync:
                import torch
                import torch.distributed as dist
                torch.cuda.synchronize()
                dist.barrier(group=self._hgroup)
            self._ev_proj = self._ev_red = None
            self._peer_proj, self._peer_red = [], []
        for o in (self._op, self._shard):
            if o is not None:
                o.close()
        self._op = self._shard = None
        lib = _lib.load()
        for p in self._peers:
            lib.qtt_ipc_close(p)
        self._peers = []
        if self._recv:
            lib.qtt_ipc_free(self._recv)
            self._recv = None

    def __del__(self):
        try:
            self.close(sync=False)
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
