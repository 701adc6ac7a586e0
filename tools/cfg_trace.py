import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1410_0759_b200 import bench_cli as bc
lay = bc.load_suite("alexnet")[0]
prob = bc._Problem(lay, "f32", 2014, 0)
for var in ("", "1"):
    if var: os.environ["DNNP_TC_BLOCK_S2D"] = var
    os.environ["DNNP_TC_TRACE"] = "1"
    for pas in ("fwd", "bwd_data"):
        print("===", var, pas, flush=True)
        prob.op(pas, "implicit")(); torch.cuda.synchronize()
    os.environ.pop("DNNP_TC_TRACE")
