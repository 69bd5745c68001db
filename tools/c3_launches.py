"""One C3 image (AMF + 100 restore iterations) for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/c3_launches.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench_workloads as W
import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import amf_detect, restore_regularize

img = torch.from_numpy(W._c3_input()).cuda()
g = sk.Grid.from_tensor(img)
mask = amf_detect(g)
out, rep = restore_regularize(g, mask)
torch.cuda.synchronize()
print("iterations", rep.iterations)
