"""Wall time of a repeated drop-in loop call with a user elemental (Python
Jacobi, 1024^2 fp32, stop_after(36)) with and without the JIT translation
cache -- A/B tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import jit
from jit_perf import jacobi

n = 1024
u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
f = torch.ones((n, n), dtype=torch.float32, device="cuda")
g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
ex = sk.DeviceExecutor(1)


def call():
    return sk.loop_stencil_reduce_d(1, sk.ElementalFn(jacobi, 1), sk.abs_change(), sk.max_combinator(0.0),
                                    sk.stop_after(36), g0, env=gf, executor=ex)


for label in ("cached", "uncached"):
    if label == "uncached":
        jit._program_key = lambda *a: None
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per 36-sweep call", flush=True)
