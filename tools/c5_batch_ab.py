"""C5 device rate vs frames per restore_frames launch (128 distinct 1080p
frames at 10% noise) -- A/B tool, not the bench."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench_workloads as W
from paper_1609_04567_b200.apps import amf_frames, restore_frames

n = 128
dev = torch.from_numpy(np.stack(W._c5_frames(n))).cuda()
for B in (16, 32, 48, 64, 32, 64):
    def run():
        for b0 in range(0, n, B):
            batch = dev[b0:min(n, b0 + B)]
            masks, _ = amf_frames(batch)
            restore_frames(batch, masks)
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        run()
    e.record()
    torch.cuda.synchronize()
    print(f"B={B}: {3 * n / (s.elapsed_time(e) / 1e3):.0f} frames/s", flush=True)
