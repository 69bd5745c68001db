"""Host-side cost breakdown of small device runs (cProfile over N C1 solves)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

u0 = torch.zeros((1024, 1024), dtype=torch.float32, device="cuda")
f = torch.ones((1024, 1024), dtype=torch.float32, device="cuda")
kern = helmholtz_kernel(HelmholtzConfig(1024, 1024))
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)


def c1():
    return sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                    sk.Condition.below(1e-4), g0, env=gf)


for _ in range(20):
    c1()
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    c1()
torch.cuda.synchronize()
print(f"wall per C1 solve: {(time.perf_counter() - t0) / n * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    c1()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
