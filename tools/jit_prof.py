"""One JIT Jacobi solve for ncu (not a benchmark)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1609_04567_b200 as sk
from tools.jit_perf import jacobi  # noqa: F401  (same function as the perf script)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dt = torch.float32 if (len(sys.argv) < 3 or sys.argv[2] == "f32") else torch.float64
u0 = torch.zeros((n, n), dtype=dt, device="cuda")
f = torch.ones((n, n), dtype=dt, device="cuda")
out, rep = sk.loop_stencil_reduce_d(1, sk.ElementalFn(jacobi, 1), sk.abs_change(),
                                    sk.max_combinator(0.0), sk.stop_after(3),
                                    sk.Grid.from_tensor(u0), env=sk.Grid.from_tensor(f),
                                    executor=sk.DeviceExecutor(1, timing=True))
torch.cuda.synchronize()
print(rep.iterations)
