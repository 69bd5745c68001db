"""One or more Helmholtz solves for profiling (ncu) -- not a benchmark."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--timing", type=int, default=1)
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
u0 = torch.zeros((a.n, a.n), dtype=dt, device="cuda")
f = torch.ones((a.n, a.n), dtype=dt, device="cuda")
ex = sk.DeviceExecutor(1, timing=bool(a.timing))
for _ in range(a.solves):
    out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(HelmholtzConfig(a.n, a.n)),
                                        sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), sk.Grid.from_tensor(u0),
                                        env=sk.Grid.from_tensor(f), executor=ex)
torch.cuda.synchronize()
print(rep.iterations, rep.final_reduce, ex.last_kernel_time)
