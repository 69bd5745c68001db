"""Host-side cost of one C1 solve through loop_stencil_reduce_d (cProfile
over 100 solves + wall/kernel split) -- A/B tool, not the bench."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

n = 1024
kern = helmholtz_kernel(HelmholtzConfig(n, n))
u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
f = torch.ones((n, n), dtype=torch.float32, device="cuda")
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
ex = sk.DeviceExecutor(1)


def solve():
    return sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                    sk.Condition.below(1e-4), g0, env=gf, executor=ex)


for _ in range(50):
    solve()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    solve()
torch.cuda.synchronize()
print(f"wall per solve {(time.perf_counter() - t0) * 1e4:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    solve()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(45)
