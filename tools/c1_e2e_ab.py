"""C1 end-to-end pipeline variants (per-solve wall ms over 50 solves):
as in the bench (upload k+1 / solve k / read back k), without the read-back,
without the upload -- A/B tool, not the bench."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel

n = 1024
kern = helmholtz_kernel(HelmholtzConfig(n, n))
h0 = torch.zeros((n, n), dtype=torch.float32).pin_memory()
hf = torch.ones((n, n), dtype=torch.float32).pin_memory()
houts = [torch.empty((n, n), dtype=torch.float32).pin_memory() for _ in range(2)]
cur = torch.cuda.current_stream()
up_s, down_s = torch.cuda.Stream(), torch.cuda.Stream()
ex = sk.DeviceExecutor(1)
d0, df0 = h0.cuda(), hf.cuda()


def upload():
    with torch.cuda.stream(up_s):
        du, df = h0.to("cuda", non_blocking=True), hf.to("cuda", non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(up_s)
    return du, df, ev


def run(count, do_up=True, do_down=True):
    nxt = upload() if do_up else (d0, df0, None)
    for k in range(count):
        du, df, ev = nxt
        if ev is not None:
            cur.wait_event(ev)
            du.record_stream(cur)
            df.record_stream(cur)
        if k + 1 < count:
            nxt = upload() if do_up else (d0, df0, None)
        o, _ = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), sk.Grid.from_tensor(du),
                                        env=sk.Grid.from_tensor(df), executor=ex)
        if do_down:
            ot = o.tensor()
            down_s.wait_stream(cur)
            with torch.cuda.stream(down_s):
                houts[k % 2].copy_(ot, non_blocking=True)
            ot.record_stream(down_s)
    torch.cuda.synchronize()


def run_api(count):
    """the C4 form: Grid.prefetch_device / prefetch_host(out=) (the public API)"""
    def host_inputs():
        return sk.Grid.from_tensor(h0), sk.Grid.from_tensor(hf)

    nxt = tuple(g.prefetch_device() for g in host_inputs())
    prev = None
    for k in range(count):
        gu, gf = nxt
        if k + 1 < count:
            nxt = tuple(g.prefetch_device() for g in host_inputs())
        o, _ = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), gu, env=gf, executor=ex)
        o.prefetch_host(out=houts[k % 2].numpy())
        if prev is not None:
            prev.to_array()
        prev = o
    prev.to_array()


run_api(8)
t0 = time.perf_counter()
run_api(50)
print(f"{'grid api':14s} {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per solve", flush=True)

for name, u, d in (("bench form", True, True), ("no read-back", True, False), ("no upload", False, True),
                   ("neither", False, False)):
    run(8, u, d)
    t0 = time.perf_counter()
    run(50, u, d)
    print(f"{name:14s} {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per solve", flush=True)
