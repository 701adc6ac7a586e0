"""Multi-process host logic of the batch-sharded path on CPU:
world_size 2 over gloo.  The per-rank partial dW is computed by the C oracle
(test infrastructure) on the rank's shard; the allreduce must reproduce the
unsharded dW, and shard views must address the right images."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
import paper_1410_0759_b200 as dp
from paper_1410_0759_b200 import dist as dpd


def test_batch_shard_partition():
    for n in (1, 5, 16, 1024):
        for world in (1, 2, 3, 8):
            spans = [dpd.batch_shard(n, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == n
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_shard_view_layouts():
    for layout in ("nchw", "nhwc"):
        a = np.arange(6 * 3 * 4 * 5, dtype=np.float32).reshape(6, 3, 4, 5)
        v = dp.TensorView.from_array(a, layout=layout)
        for r in range(4):
            s = dpd.shard_view(v, r, 4)
            start, count = dpd.batch_shard(6, r, 4)
            assert np.array_equal(s.numpy(), a[start:start + count])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    N, C, H, W, K, R, S = 4, 3, 7, 6, 5, 3, 3
    x = rng.uniform(-0.5, 0.5, (N, C, H, W)).astype(np.float64)
    dy = rng.uniform(-0.5, 0.5, (N, K, H, W)).astype(np.float64)
    start, count = dpd.batch_shard(N, rank, world)
    xs, dys = np.ascontiguousarray(x[start:start + count]), np.ascontiguousarray(dy[start:start + count])
    part = np.zeros(K * C * R * S)
    cg = [1, 1, 1, 1, 0, 0]
    orc.conv_backward_filter([count, C, H, W, C * H * W, H * W, W, 1], xs.reshape(-1),
                             [count, K, H, W, K * H * W, H * W, W, 1], dys.reshape(-1), cg,
                             [K, C, R, S], part)
    t = torch.from_numpy(part)
    dpd.allreduce_filter_grad(t)
    results[rank] = t.numpy().copy()
    dist.destroy_process_group()


def test_allreduce_matches_unsharded():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    rng = np.random.default_rng(11)
    N, C, H, W, K, R, S = 4, 3, 7, 6, 5, 3, 3
    x = rng.uniform(-0.5, 0.5, (N, C, H, W)).astype(np.float64)
    dy = rng.uniform(-0.5, 0.5, (N, K, H, W)).astype(np.float64)
    full = np.zeros(K * C * R * S)
    orc.conv_backward_filter([N, C, H, W, C * H * W, H * W, W, 1], x.reshape(-1),
                             [N, K, H, W, K * H * W, H * W, W, 1], dy.reshape(-1),
                             [1, 1, 1, 1, 0, 0], [K, C, R, S], full)
    for r in range(world):
        assert orc.rel_err(results[r], full) <= 1e-12
    assert np.array_equal(results[0], results[1])


@pytest.mark.gpu
def test_dp_backward_filter_single_rank_gpu():
    """On one GPU (world 1) the DP entry equals the plain call."""
    rng = np.random.default_rng(5)
    x = dp.TensorView.from_array(rng.uniform(-1, 1, (4, 8, 9, 9)).astype(np.float32), device="cuda")
    dy = dp.TensorView.from_array(rng.uniform(-1, 1, (4, 16, 9, 9)).astype(np.float32), device="cuda")
    cd = dp.ConvDesc(1, 1, 1, 1)
    df1 = dp.FilterView.from_array(np.zeros((16, 8, 3, 3), np.float32), device="cuda")
    df2 = dp.FilterView.from_array(np.zeros((16, 8, 3, 3), np.float32), device="cuda")
    dp.conv_backward_filter(dy, x, cd, "implicit", df1)
    dpd.conv_backward_filter_dp(dy, x, cd, "implicit", df2)
    assert torch.equal(df1.buf, df2.buf)


def _overlap_worker(rank, world, port, results, use_cuda):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if use_cuda:
        torch.cuda.set_device(0)
        torch.zeros(1, device="cuda")  # initialise the context before the helper
    ov = dpd.OverlappedAllreduce()
    rng = np.random.default_rng(21)
    layers = []
    for li in range(3):
        N, C, H, K = 4, 3 + li, 9, 4 + 2 * li
        x = rng.uniform(-0.5, 0.5, (N, C, H, H)).astype(np.float32)
        dy = rng.uniform(-0.5, 0.5, (N, K, H, H)).astype(np.float32)
        layers.append((x, dy, K, C))
    outs = []
    for x, dy, K, C in layers:
        dev = "cuda" if use_cuda else None
        xv = dpd.shard_view(dp.TensorView.from_array(x, device=dev), rank, world)
        dyv = dpd.shard_view(dp.TensorView.from_array(dy, device=dev), rank, world)
        if use_cuda:
            df = dp.FilterView(dp.make_filter_desc(K, C, 3, 3), torch.zeros(K * C * 9, device="cuda"))
            dp.conv_backward_filter(dyv, xv, dp.ConvDesc(1, 1, 1, 1), "implicit", df)
            ov.submit(df.buf)
            outs.append(df.buf)
        else:
            t = torch.from_numpy(np.full(K * C * 9, float(rank + 1), dtype=np.float32))
            ov.submit(t)
            outs.append(t)
    ov.wait()
    if use_cuda:
        torch.cuda.synchronize()
    results[rank] = [o.cpu().numpy().copy() for o in outs]
    dist.destroy_process_group()


def test_overlapped_allreduce_cpu():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_overlap_worker, args=(2, _free_port(), results, False), nprocs=2, join=True)
    for r in range(2):
        for o in results[r]:
            assert np.all(o == 3.0)


@pytest.mark.gpu
def test_overlapped_allreduce_two_ranks_one_gpu():
    """Two gloo ranks sharing cuda:0: per-rank partial dW from the library,
    allreduces on the communication stream, equal to the unsharded dW."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_overlap_worker, args=(2, _free_port(), results, True), nprocs=2, join=True)
    rng = np.random.default_rng(21)
    for li in range(3):
        N, C, H, K = 4, 3 + li, 9, 4 + 2 * li
        x = rng.uniform(-0.5, 0.5, (N, C, H, H)).astype(np.float32)
        dy = rng.uniform(-0.5, 0.5, (N, K, H, H)).astype(np.float32)
        full = np.zeros(K * C * 9)
        orc.conv_backward_filter([N, C, H, H, C * H * H, H * H, H, 1], x.astype(np.float64).reshape(-1),
                                 [N, K, H, H, K * H * H, H * H, H, 1],
                                 dy.astype(np.float64).reshape(-1), [1, 1, 1, 1, 0, 0],
                                 [K, C, 3, 3], full)
        for r in range(2):
            assert orc.rel_err(results[r][li], full) <= 1e-4
        assert np.array_equal(results[0][li], results[1][li])
