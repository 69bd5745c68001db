"""Host-side phases of one C1 solve through the DeviceExecutor protocol
(begin / run_loop / finish), wall-clock medians over 200 solves -- A/B tool."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel
from paper_1609_04567_b200.loop import _as_plan

n = 1024
kern = helmholtz_kernel(HelmholtzConfig(n, n))
u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
f = torch.ones((n, n), dtype=torch.float32, device="cuda")
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
ex = sk.DeviceExecutor(1)
cond = sk.Condition.below(1e-4)
ph = {"plan": [], "begin": [], "run_loop": [], "finish": [], "total": []}
for i in range(260):
    t0 = time.perf_counter()
    plan = _as_plan(kern, 1, sk.max_combinator(0.0), gf, indexed=False, delta=sk.abs_change())
    t1 = time.perf_counter()
    run = ex.begin(plan, g0)
    t2 = time.perf_counter()
    it, v, exh = ex.run_loop(run, cond)
    t3 = time.perf_counter()
    out, led = ex.finish(run)
    t4 = time.perf_counter()
    if i >= 60:
        for k, a, b in (("plan", t0, t1), ("begin", t1, t2), ("run_loop", t2, t3), ("finish", t3, t4),
                        ("total", t0, t4)):
            ph[k].append((b - a) * 1e6)
print({k: round(statistics.median(v), 1) for k, v in ph.items()}, "us; iterations", it)
