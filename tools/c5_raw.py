"""C5 without the stream farm: batches of B frames uploaded from pinned host
memory, detected + restored (amf_frames + restore_frames) and read back into
pinned host memory, copies on their own streams overlapping the next batch's
compute.  The ceiling the pipeline's host side is measured against."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench_workloads import _c5_frames_range  # noqa: E402
from paper_1609_04567_b200.apps import amf_frames, restore_frames  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
host = torch.from_numpy(np.stack(_c5_frames_range(0, nf))).pin_memory()
outs = [torch.empty((B, 1080, 1920), dtype=torch.float64, pin_memory=True) for _ in range(2)]
comp, up, down = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run():
    ev_free = [None, None]
    for k, b0 in enumerate(range(0, nf, B)):
        n = min(B, nf - b0)
        with torch.cuda.stream(up):
            d = host[b0:b0 + n].to("cuda", non_blocking=True)
            e_up = torch.cuda.Event()
            e_up.record(up)
        comp.wait_event(e_up)
        with torch.cuda.stream(comp):
            m, _ = amf_frames(d, stream=comp)
            res, _ = restore_frames(d, m, stream=comp)
            e_c = torch.cuda.Event()
            e_c.record(comp)
        slot = k & 1
        if ev_free[slot] is not None:
            ev_free[slot].synchronize()
        down.wait_event(e_c)
        with torch.cuda.stream(down):
            for i in range(n):
                outs[slot][i].copy_(res[i], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(down)
            ev_free[slot] = ev
    torch.cuda.synchronize()


run()
for _ in range(3):
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    print(json.dumps({"frames": nf, "batch": B, "frames_per_s": round(nf / dt, 1)}), flush=True)
