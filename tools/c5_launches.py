"""One C5 batch (32 distinct 1080p frames at 10%: batched AMF + restore_frames)
for an ncu launch list:  ncu --metrics gpu__time_duration.sum --csv python tools/c5_launches.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench_workloads as W
from paper_1609_04567_b200.apps import amf_frames, restore_frames

batch = torch.from_numpy(np.stack(W._c5_frames(32))).cuda()
for _ in range(2):
    masks, _ = amf_frames(batch)
    _, reps = restore_frames(batch, masks)
torch.cuda.synchronize()
print("iterations", [r.iterations for r in reps][:8])
