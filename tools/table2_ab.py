import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1410_0759_b200 as dp
from paper_1410_0759_b200 import bench_cli as bc
for name in ("layer4", "layer5"):
    lay = {l.name: l for l in bc.load_suite("table2")}[name]
    prob = bc._Problem(lay, "f32", 2014, 0)
    for var in ("", "DNNP_TC_SK=1", "DNNP_TC_NO_PAIRS=1", "DNNP_TC_BN=128"):
        for k in ("DNNP_TC_SK", "DNNP_TC_NO_PAIRS", "DNNP_TC_BN"): os.environ.pop(k, None)
        if var: k, v = var.split("="); os.environ[k] = v
        res = []
        for pas in ("fwd", "bwd_data"):
            t = bc._time(prob.op(pas, "implicit"), 9)
            res.append(f"{pas} {lay.flops()/t/1e12:6.1f}")
        print(name, f"[{var or 'default':<20}]", "  ".join(res), flush=True)
