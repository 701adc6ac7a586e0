"""Caller-supplied workspace (additive dnnp_get_convolution_workspace_size +
*_ex entries; SURVEY 8(b) "minimal-workspace contract"): the queried size is
enough (the _ex call succeeds and matches the plain call bit for bit), one
half of it is refused with ALLOC_FAILED (AllocTooLarge), and the pass does
not touch the library's own arena."""
import numpy as np
import pytest

import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

SHAPES = [(4, 16, 20, 20, 32, 3, 3, 1, 1, 1, 1),
          (2, 3, 40, 44, 64, 11, 11, 4, 4, 2, 2),     # space-to-depth
          (2, 3, 40, 44, 96, 11, 11, 1, 1, 0, 0),     # tap folding / wide blocking
          (8, 64, 13, 13, 192, 3, 3, 1, 1, 1, 1)]     # pairs, stream-K


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("pas", ["fwd", "bwd_data", "bwd_filter"])
def test_workspace_query_and_ex(shape, pas):
    import torch
    n, c, h, w, k, r, s, u, v, ph, pw = shape
    rng = np.random.default_rng(5)
    cd = dp.ConvDesc(u, v, ph, pw)
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    xd, yd = dp.make_desc(n, c, h, w), dp.make_desc(n, k, p, q)
    fd = dp.make_filter_desc(k, c, r, s)
    t = lambda cnt: torch.from_numpy(rng.uniform(-0.5, 0.5, cnt).astype(np.float32)).cuda()
    x, dy, f = t(n * c * h * w), t(n * k * p * q), t(k * c * r * s)
    launches = dp.kernel_launch_count()
    need = dp.convolution_workspace_size(pas, xd, fd, cd, yd)
    assert need > 0
    assert dp.kernel_launch_count() == launches  # the query plans, it does not run the pass

    def run(ws):
        xv, dyv = dp.TensorView(xd, x), dp.TensorView(yd, dy)
        fv = dp.FilterView(fd, f)
        if pas == "fwd":
            out = dp.TensorView(yd, torch.zeros(n * k * p * q, device="cuda"))
            dp.conv_forward(xv, fv, cd, "implicit", out, workspace=ws)
        elif pas == "bwd_data":
            out = dp.TensorView(xd, torch.zeros(n * c * h * w, device="cuda"))
            dp.conv_backward_data(dyv, fv, cd, "implicit", out, workspace=ws)
        else:
            out = dp.FilterView(fd, torch.zeros(k * c * r * s, device="cuda"))
            dp.conv_backward_filter(dyv, xv, cd, "implicit", out, workspace=ws)
        torch.cuda.synchronize()
        return out.buf.clone()

    ref = run(None)
    # exactly the queried bytes, at a base only 256-byte aligned (the size
    # includes the slack of the 1024-byte carve-out alignment)
    raw = torch.empty(need + 2048, dtype=torch.uint8, device="cuda")
    off = (1024 - raw.data_ptr() % 1024) % 1024 + 256
    ws = raw[off:off + need]
    assert ws.numel() == need and ws.data_ptr() % 1024 == 256
    torch.cuda.synchronize()
    dp.scratch_high_water(reset=True)
    got = run(ws)
    assert dp.scratch_high_water() == 0  # nothing from the library arena
    assert torch.equal(got, ref)
    small = torch.empty(max(need // 2, 1), dtype=torch.uint8, device="cuda")
    with pytest.raises(dp.AllocTooLarge):
        run(small)
