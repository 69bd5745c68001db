"""Host cost of the pieces of one drop-in loop call on a device grid (begin /
finish internals), per call -- A/B tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200 import _native as N
from paper_1609_04567_b200.partition import model_ledger

u0 = torch.zeros((1024, 1024), device="cuda")
g = sk.Grid.from_tensor(u0)
cur = torch.cuda.current_stream()


def t(name, fn, n=5000):
    for _ in range(100):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:44s} {(time.perf_counter() - t0) / n * 1e6:6.2f} us")


t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("torch.device('cuda', current_device())", lambda: torch.device("cuda", torch.cuda.current_device()))
t("stream.device", lambda: cur.device)
dev = torch.device("cuda", 0)
t("grid.tensor(device=dev)", lambda: g.tensor(device=dev))
t("grid.storage_dtype()", lambda: g.storage_dtype())
t("torch.empty x2", lambda: [torch.empty((1024, 1024), device=dev) for _ in range(2)])


def plan():
    p = N.sk_plan()
    p.kernel = 1
    p.dtype = 1
    p.rows, p.cols = 1024, 1024
    p.partitions = 1
    p.reduce_op = 2
    p.delta_op = 1
    p.halo_top = p.halo_bottom = 0
    p.flags = 0
    p.identity = 0.0
    for i, v in enumerate((1.0, 1.0, 5.0, 0.0, 1.0)):
        p.params[i] = v
    return p


t("sk_plan build", plan)
t("Grid.from_tensor", lambda: sk.Grid.from_tensor(u0))
t("model_ledger", lambda: model_ledger((1024, 1024), 1, 1, 36))
t("N.stream_handle", lambda: N.stream_handle(cur))
