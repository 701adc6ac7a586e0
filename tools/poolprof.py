import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_1410_0759_b200 as dp
x = dp.TensorView(dp.make_desc(128, 64, 55, 55), torch.rand(128*64*55*55, device="cuda"))
for pk in ("max", "average"):
    pd = dp.PoolingDesc(pk, 3, 3, 2, 2, 0, 0)
    y = dp.empty_view(dp.make_desc(128, 64, 27, 27), device="cuda")
    dy = dp.TensorView(dp.make_desc(128, 64, 27, 27), torch.rand(128*64*27*27, device="cuda"))
    dx = dp.empty_view(dp.make_desc(128, 64, 55, 55), device="cuda")
    am = torch.empty((128, 64, 27, 27), dtype=torch.int64, device="cuda") if pk == "max" else None
    for _ in range(2):
        dp.pool_forward(pd, x, y, am)
        dp.pool_backward(pd, y, dy, x, dx, am)
torch.cuda.synchronize()
