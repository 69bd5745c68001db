"""Per-sweep times of the product Helmholtz sweep (CUDA events inside the
library, SK_FLAG_TIMING) for the fp32 C4 route and the fp64 routes -- A/B
tool, not the bench."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel


def one(n, dt, delta, comb, cond, name, solves=2):
    u0 = torch.zeros((n, n), dtype=dt, device="cuda")
    f = torch.ones((n, n), dtype=dt, device="cuda")
    ex = sk.DeviceExecutor(1, timing=True)
    best = None
    for _ in range(solves):
        out, rep = sk.loop_stencil_reduce_d(1, helmholtz_kernel(HelmholtzConfig(n, n)), delta, comb,
                                            cond, sk.Grid.from_tensor(u0), env=sk.Grid.from_tensor(f),
                                            executor=ex)
        ms, cnt = ex.last_kernel_time
        per = ms / cnt
        best = per if best is None else min(best, per)
    torch.cuda.synchronize()
    alg = 3 * n * n * (4 if dt == torch.float32 else 8)
    print(f"{name:28s} n={n} its={rep.iterations} {best:.4f} ms/sweep {alg / best / 1e6:.0f} GB/s "
          f"frac {alg / best / 1e6 / 6555.5:.3f}", flush=True)
    del u0, f, out


n64 = int(sys.argv[1]) if len(sys.argv) > 1 else 23170
one(32768, torch.float32, sk.abs_change(), sk.max_combinator(0.0), sk.Condition.below(1e-4), "f32 abs/max")
one(n64, torch.float64, sk.abs_change(), sk.max_combinator(0.0), sk.Condition.below(1e-4), "f64 abs/max")
one(n64, torch.float64, sk.sq_change(), sk.sum_combinator(0.0), sk.Condition.below(1e-4 * n64 * n64),
    "f64 sq/sum")
