"""Sweep time of run-time compiled user elementals vs the hand-written
Helmholtz kernel on the same grid (not the bench; prints JSON lines)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel
from paper_1609_04567_b200.grid import ABSENT

AX, AY, B = 1.0, 1.0, 5.0


def jacobi(nb, env):
    c = nb.center
    l = nb.at(0, -1)
    r = nb.at(0, 1)
    u = nb.at(-1, 0)
    d = nb.at(1, 0)
    l = 0.0 if l is ABSENT else l
    r = 0.0 if r is ABSENT else r
    u = 0.0 if u is ABSENT else u
    d = 0.0 if d is ABSENT else d
    f = env.at(*nb.center_index)
    return 0.0 * c + 1.0 * (f + AX * (l + r) + AY * (u + d)) / B


def run(n, dtype, which, sweeps=10):
    u0 = torch.zeros((n, n), dtype=dtype, device="cuda")
    f = torch.ones((n, n), dtype=dtype, device="cuda")
    ex = sk.DeviceExecutor(1, timing=True)
    kern = sk.ElementalFn(jacobi, 1) if which == "jit" else helmholtz_kernel(HelmholtzConfig(n, n))
    for _ in range(2):
        out, rep = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                            sk.stop_after(sweeps), sk.Grid.from_tensor(u0),
                                            env=sk.Grid.from_tensor(f), executor=ex)
    ms, k = ex.last_kernel_time
    per = ms / k
    esz = torch.tensor([], dtype=dtype).element_size()
    gbs = 3 * esz * n * n / (per / 1e3) / 1e9
    return {"kernel": which, "n": n, "dtype": str(dtype), "ms_per_sweep": per, "GB/s": gbs,
            "final": rep.final_reduce}


if __name__ == "__main__":
  for n in (8192, 16384):
    for dt in (torch.float32, torch.float64):
        for w in ("builtin", "jit"):
            print(json.dumps(run(n, dt, w)))
