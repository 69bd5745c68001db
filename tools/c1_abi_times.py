"""Per-call wall time of the C-ABI entry points during C1 solves (the
library functions wrapped with timers) -- A/B tool."""
import collections
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import _native as N
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

lib = N.load()
times = collections.defaultdict(list)


class Timed:
    def __init__(self, name, fn):
        self.name, self.fn = name, fn

    def __call__(self, *a):
        t = time.perf_counter()
        r = self.fn(*a)
        times[self.name].append((time.perf_counter() - t) * 1e6)
        return r


for name in ("sk_run_begin", "sk_run_loop", "sk_run_result", "sk_run_launches", "sk_run_destroy"):
    setattr(lib, name, Timed(name, getattr(lib, name)))

n = 1024
kern = helmholtz_kernel(HelmholtzConfig(n, n))
u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
f = torch.ones((n, n), dtype=torch.float32, device="cuda")
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
ex = sk.DeviceExecutor(1)
for i in range(300):
    if i == 100:
        times.clear()
    t = time.perf_counter()
    sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0), sk.Condition.below(1e-4),
                             g0, env=gf, executor=ex)
    times["solve"].append((time.perf_counter() - t) * 1e6)
print({k: round(statistics.median(v), 1) for k, v in times.items()})
