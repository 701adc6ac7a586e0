import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1410_0759_b200 as dp
from paper_1410_0759_b200 import bench_cli as bc
def times(op, n=8):
    out=[]
    for _ in range(n):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); op(); b.record(); torch.cuda.synchronize(); out.append(round(a.elapsed_time(b)*1e3,1))
    return out
lay = bc.Layer("c512k7", 32, 512, 14, 14, 512, 7, 7, 1, 1, 3, 3)
prob = bc._Problem(lay, "f32", 2014, 0)
for ch in ("1000000000", "16384"):
    os.environ["DNNP_TC_CHAIN"] = ch
    print("c512k7 fwd chain", ch, times(prob.op("fwd", "implicit")), flush=True)
os.environ.pop("DNNP_TC_CHAIN")
lay = bc.load_suite("alexnet")[1]
prob = bc._Problem(lay, "f32", 2014, 0)
bias = dp.TensorView(dp.make_desc(1, lay.k, 1, 1), torch.rand(lay.k, device="cuda") - 0.5)
print("conv2 fwd plain", times(prob.op("fwd", "implicit")), flush=True)
print("conv2 fwd alpha=.5", times(lambda: dp.conv_forward(prob.x, prob.f, prob.cd, "implicit", prob.y, alpha=0.5)), flush=True)
print("conv2 fwd beta=1", times(lambda: dp.conv_forward(prob.x, prob.f, prob.cd, "implicit", prob.y, beta=1.0)), flush=True)
print("conv2 fused bias", times(lambda: dp.conv_bias_activation_forward(prob.x, prob.f, prob.cd, "implicit", prob.y, bias=bias)), flush=True)
print("conv2 fused relu", times(lambda: dp.conv_bias_activation_forward(prob.x, prob.f, prob.cd, "implicit", prob.y, activation="relu")), flush=True)
