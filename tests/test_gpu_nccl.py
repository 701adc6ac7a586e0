"""Native NCCL path of the batch-sharded backward-filter (
include/dnnp.h dnnp_nccl_* / dnnp_convolution_backward_filter_allreduce).
One GPU is available in this run, so the communicator has one rank: the
allreduce is the identity and the fused call must equal backward-filter bit
for bit (plain and accumulate), through the C ABI and the overlapped
comm-stream helper, eagerly and inside a captured CUDA graph.  The sharding
arithmetic and the reduction order across ranks are covered by the gloo
world-size-2 tests (tests/test_dist.py)."""
import numpy as np
import pytest

import paper_1410_0759_b200 as dp
from paper_1410_0759_b200 import dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    uid = dist.NativeComm.unique_id()
    assert len(uid) == 128 and any(uid)
    return dist.NativeComm(uid, 1, 0)


def _problem(acc, seed=0):
    import torch
    rng = np.random.default_rng(seed)
    n, c, h, k, r = 4, 32, 13, 64, 3
    cd = dp.ConvDesc(1, 1, 1, 1, "convolution", acc)
    mk = lambda cnt: torch.from_numpy(rng.uniform(-0.5, 0.5, cnt).astype(np.float32)).cuda()  # noqa: E731
    x = dp.TensorView(dp.make_desc(n, c, h, h), mk(n * c * h * h))
    dy = dp.TensorView(dp.make_desc(n, k, h, h), mk(n * k * h * h))
    df0 = mk(k * c * r * r)
    return x, dy, cd, df0, dp.make_filter_desc(k, c, r, r)


@pytest.mark.parametrize("acc", [False, True])
def test_backward_filter_allreduce_one_rank(comm, acc):
    import torch
    x, dy, cd, df0, fd = _problem(acc)
    a = dp.FilterView(fd, df0.clone())
    b = dp.FilterView(fd, df0.clone())
    dist.conv_backward_filter_allreduce(dy, x, cd, "implicit", a)
    dp.conv_backward_filter(dy, x, cd, "implicit", b)
    torch.cuda.synchronize()
    assert torch.equal(a.buf, b.buf)


def test_overlapped_native_allreduce_in_graph():
    import torch
    uid = dist.NativeComm.unique_id()
    ov = dist.NativeOverlappedAllreduce(uid, 1, 0)
    x, dy, cd, df0, fd = _problem(False, seed=1)
    df = dp.FilterView(fd, torch.zeros_like(df0))
    ref = dp.FilterView(fd, torch.zeros_like(df0))
    dp.conv_backward_filter(dy, x, cd, "implicit", ref)

    def step():
        dp.conv_backward_filter(dy, x, cd, "implicit", df)
        ov.submit(df.buf)
        ov.wait()

    step()
    torch.cuda.synchronize()
    assert torch.equal(df.buf, ref.buf)
    df.buf.zero_()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(df.buf, ref.buf)
    ov.close()


def test_allreduce_requires_communicator_and_device_buffer():
    import ctypes
    from paper_1410_0759_b200 import _lib
    L = _lib.lib()
    h = ctypes.c_void_p()
    assert L.dnnp_create(ctypes.byref(h)) == 0
    buf = (ctypes.c_float * 4)()
    assert L.dnnp_allreduce_sum(h, ctypes.cast(buf, ctypes.c_void_p), 4, 0) == _lib.BAD_PARAM
    assert L.dnnp_destroy(h) == 0
