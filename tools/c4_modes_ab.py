"""C4 solve time in the timing (batched, per-launch events) and production (graph WHILE) loop forms -- A/B tool."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel
n = 32768
kern = helmholtz_kernel(HelmholtzConfig(n, n))
u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
f = torch.ones((n, n), dtype=torch.float32, device="cuda")
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
for timing in (True, False, True, False):
    ex = sk.DeviceExecutor(1, timing=timing)
    for _ in range(2):
        out, rep = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0), sk.Condition.below(1e-4), g0, env=gf, executor=ex)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(5):
        out, rep = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0), sk.Condition.below(1e-4), g0, env=gf, executor=ex)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print("timing" if timing else "graph ", f"{ms:.2f} ms/solve  {36*n*n/ms/1e6:.1f} Gcell/s  per sweep {ms/36:.4f} ms", rep.iterations, ex.launches)
