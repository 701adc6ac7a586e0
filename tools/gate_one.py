import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1410_0759_b200 as dp
from paper_1410_0759_b200 import bench_cli as bc
lay = {l.name: l for l in bc.load_suite("alexnet")}["conv3"]
prob = bc._Problem(lay, "f32", 2014, 0)
g = dp.TensorView(prob.x.desc, prob.x.buf.clamp(min=0))
dp.conv_backward_data_activation(prob.dy, prob.f, prob.cd, "implicit", prob.dx, "relu", g)
torch.cuda.synchronize()
