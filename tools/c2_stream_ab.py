"""C2 stream-mode e2e (sobel_stream over 512 pinned 2048^2 frames) across
batch widths and batches in flight -- A/B tool, not the bench."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import sobel_stream

F, H, W = 512, 2048, 2048
hin = torch.randint(0, 256, (F, H, W), dtype=torch.uint8).pin_memory()
grids = [sk.Grid.from_tensor(hin[i]) for i in range(F)]
n = [0]


def writer(g):
    n[0] += 1


for width in (16, 32, 64):
    for wpd in (2, 3, 4):
        for _ in range(2):
            sobel_stream(grids, writer=writer, width=width, host_buffers=True, workers_per_device=wpd)
        ps = []
        for _ in range(3):
            t0 = time.perf_counter()
            sobel_stream(grids, writer=writer, width=width, host_buffers=True, workers_per_device=wpd)
            ps.append(time.perf_counter() - t0)
        print(f"width {width} workers {wpd}: {F / statistics.median(ps):.0f} frames/s", flush=True)
