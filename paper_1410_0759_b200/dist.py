"""Batch-sharded data parallelism for the convolution path.

The minibatch N is split across ranks (one process per GPU); forward and
backward-data need no communication; backward-filter produces a partial dW
over the rank's N/G * P * Q reduction slice and ends in ONE allreduce(sum) of
dW over NCCL (NVLink / NVSwitch).  With `accumulate`, the reduced gradient is
added to the prior df after the allreduce (otherwise G copies of the prior df
would be summed).

Two ways to run the reduction: the library's own NCCL communicator
(`NativeComm`: libdnnp loads libnccl at run time, the reduction is enqueued
by the C ABI on the library's stream -- no torch needed by a C caller, and it
is captured into CUDA graphs like the kernels), or torch.distributed (any
backend: nccl on GPUs, gloo for the CPU tests).  The convolution math is
libdnnp.so either way.
"""
from __future__ import annotations

import ctypes

from . import _lib
from .conv import ConvDesc, FilterView, _plan, conv_backward_filter
from .tensor import TensorView, bind_stream, make_desc


def batch_shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """(first image, image count) of `rank`'s contiguous batch slice; the
    first n_total % world ranks take one extra image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def shard_view(view: TensorView, rank: int, world: int) -> TensorView:
    """The rank's batch slice of a strided 4-D view (same strides, buffer
    offset by start * stride_n; works for NCHW, NHWC and sub-tensor views)."""
    d = view.desc
    start, count = batch_shard(d.n, rank, world)
    if count == 0:
        raise ValueError("empty shard")
    desc = make_desc(count, d.c, d.h, d.w, layout="custom", strides=d.strides, elem_type=d.dtype)
    return TensorView(desc, view.buf[start * d.stride_n:])


def allreduce_filter_grad(df_local, group=None):
    """Sum the per-rank partial filter gradients in place (torch tensor)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(df_local, op=dist.ReduceOp.SUM, group=group)
    return df_local


class OverlappedAllreduce:
    """dW allreduces off the compute stream (issue each layer's
    allreduce as soon as its backward-filter finishes, overlapped with the
    remaining backward work).  `submit(t)` records an event on the current
    (compute) stream and enqueues the allreduce of `t` on a dedicated
    communication stream behind it; `wait()` makes the compute stream wait
    for every submitted reduction (call it before the gradients are read or
    rewritten).  On CPU tensors (gloo) the reduction runs synchronously."""

    def __init__(self, group=None):
        import torch
        self.group = group
        self.cuda = torch.cuda.is_available() and torch.cuda.is_initialized()
        self.stream = torch.cuda.Stream() if self.cuda else None
        self.pending = 0

    def submit(self, t):
        import torch
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()
                and dist.get_world_size(self.group) > 1):
            return t
        if not (self.cuda and t.is_cuda):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            return t
        ev = torch.cuda.Event()
        ev.record()  # the producing kernels, on the compute stream
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            t.record_stream(self.stream)
        self.pending += 1
        return t

    def wait(self):
        import torch
        if self.cuda and self.pending:
            torch.cuda.current_stream().wait_stream(self.stream)
        self.pending = 0


def conv_backward_filter_dp(dy: TensorView, x: TensorView, conv: ConvDesc, engine,
                            df: FilterView, group=None) -> None:
    """Data-parallel backward-filter on this rank's shard (dy, x are the
    rank's slices): local partial dW, one allreduce, then accumulate."""
    import torch
    if not conv.accumulate:
        conv_backward_filter(dy, x, conv, engine, df)
        allreduce_filter_grad(df.buf, group)
        return
    part = torch.empty_like(df.buf)
    pv = FilterView(df.desc, part)
    conv_backward_filter(dy, x, ConvDesc(conv.u, conv.v, conv.pad_h, conv.pad_w, conv.mode, False),
                         engine, pv)
    allreduce_filter_grad(part, group)
    df.buf.add_(part)


class NativeComm:
    """The library's NCCL communicator on this thread's handle.

    `NativeComm.unique_id()` on one rank (128 bytes), shipped to every rank by
    any means (torch.distributed broadcast, a file, MPI), then
    `NativeComm(uid, world, rank)` on each; `from_torch(group)` does both over
    an initialised torch.distributed group.  The handle owns the
    communicator.
    """

    def __init__(self, uid: bytes, world: int, rank: int):
        if len(uid) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        self.world, self.rank = world, rank
        buf = ctypes.create_string_buffer(uid, 128)
        _lib.check(_lib.lib().dnnp_nccl_comm_create(_lib.handle(), buf, world, rank),
                   "dnnp_nccl_comm_create")

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().dnnp_nccl_unique_id(buf, 128), "dnnp_nccl_unique_id")
        return buf.raw

    @classmethod
    def from_torch(cls, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world, rank)

    def allreduce(self, t):
        """In-place sum of a CUDA tensor over the communicator, on torch's
        current stream."""
        import torch
        bind_stream(TensorView(make_desc(1, 1, 1, t.numel(), elem_type=(
            "f64" if t.dtype == torch.float64 else "f32")), t))
        _lib.check(_lib.lib().dnnp_allreduce_sum(_lib.handle(), t.data_ptr(), t.numel(),
                                                 1 if t.dtype == torch.float64 else 0),
                   "dnnp_allreduce_sum")
        return t


def conv_backward_filter_allreduce(dy: TensorView, x: TensorView, conv: ConvDesc, engine,
                                   df: FilterView) -> None:
    """Backward-filter of this rank's shard plus ONE allreduce(sum) of dW over
    the library's NCCL communicator (NativeComm), in a single C call
    (dnnp_convolution_backward_filter_allreduce); accumulate adds the reduced
    gradient after the reduction.  CUDA tensors only."""
    xd, fd, cd, dyd, ecode = _plan(2, x.desc, df.desc, conv, dy.desc, engine, 4 << 30)
    bind_stream(dy, x, df)
    _lib.check(_lib.lib().dnnp_convolution_backward_filter_allreduce(
        _lib.handle(), xd, x.ptr, dyd, dy.ptr, cd, ecode, fd, df.ptr),
        "convolution_backward_filter_allreduce")


class NativeOverlappedAllreduce:
    """dW allreduces over the library's NCCL communicator on a dedicated
    communication stream (each layer's reduction overlaps the
    remaining backward work).  A second library handle owns the stream and
    the communicator; `submit(t)` orders the reduction of `t` after the
    kernels queued so far on the compute stream, `wait()` makes the compute
    stream wait for every submitted reduction.  Capturable into a CUDA graph
    (the cross-stream dependencies are events)."""

    def __init__(self, uid: bytes, world: int, rank: int):
        import torch
        L = _lib.lib()
        self.h = ctypes.c_void_p()
        _lib.check(L.dnnp_create(ctypes.byref(self.h)), "dnnp_create")
        self.stream = torch.cuda.Stream()
        _lib.check(L.dnnp_set_stream(self.h, ctypes.c_void_p(self.stream.cuda_stream)),
                   "dnnp_set_stream")
        buf = ctypes.create_string_buffer(uid, 128)
        _lib.check(L.dnnp_nccl_comm_create(self.h, buf, world, rank), "dnnp_nccl_comm_create")
        self.pending = 0

    @classmethod
    def from_torch(cls, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [NativeComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world, rank)

    def submit(self, t):
        import torch
        ev = torch.cuda.Event()
        ev.record()  # the producing kernels, on the compute stream
        self.stream.wait_event(ev)
        _lib.check(_lib.lib().dnnp_allreduce_sum(self.h, t.data_ptr(), t.numel(),
                                                 1 if t.dtype == torch.float64 else 0),
                   "dnnp_allreduce_sum")
        self.pending += 1
        return t

    def wait(self):
        import torch
        if self.pending:
            torch.cuda.current_stream().wait_stream(self.stream)
        self.pending = 0

    def close(self):
        if self.h:
            _lib.lib().dnnp_destroy(self.h)
            self.h = None
