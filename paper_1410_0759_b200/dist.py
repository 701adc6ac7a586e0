"""Batch-sharded data parallelism for the convolution path.

The minibatch N is split across ranks (one process per GPU); forward and
backward-data need no communication; backward-filter produces a partial dW
over the rank's N/G * P * Q reduction slice and ends in ONE allreduce(sum) of
dW over NCCL (NVLink / NVSwitch).  With `accumulate`, the reduced gradient is
added to the prior df after the allreduce (otherwise G copies of the prior df
would be summed).

torch.distributed is the plumbing (any backend: nccl on GPUs, gloo for the
CPU tests); the convolution math is libdnnp.so.
"""
from __future__ import annotations

from .conv import ConvDesc, FilterView, conv_backward_filter
from .tensor import TensorView, make_desc


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
