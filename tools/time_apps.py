"""Stable timings of the secondary workloads: warm the GPU (clocks ramp from
idle), then median of several timed repetitions.  Not the bench."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import stencil_oracle as O
import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.apps import amf_frames, restore_regularize, sobel_frames


def warm(sec=1.0):
    x = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while True:
        for _ in range(20):
            x.add_(1)
        e.record()
        torch.cuda.synchronize()
        if s.elapsed_time(e) > sec * 1e3:
            break


def med(fn, reps=7):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["sobel", "amf", "restore", "c5", "c1"]
warm()
if "c1" in which:
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel, helmholtz_solve
    u0 = torch.zeros((1024, 1024), dtype=torch.float32, device="cuda")
    f = torch.ones((1024, 1024), dtype=torch.float32, device="cuda")
    kern = helmholtz_kernel(HelmholtzConfig(1024, 1024))

    def c1():
        return sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), sk.Grid.from_tensor(u0),
                                        env=sk.Grid.from_tensor(f))
    c1()
    ms = med(c1, reps=9)
    print(json.dumps({"workload": "C1 1024^2 fp32 36 sweeps (graph loop, incl. begin/finish)",
                      "ms": ms, "us_per_iteration": ms * 1e3 / 36,
                      "cell_updates_per_s": 36 * 1024 * 1024 / ms * 1e3}))
if "sobel" in which:
    F, H, W = 128, 2048, 2048
    fr = torch.randint(0, 256, (F, H, W), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(fr)
    sobel_frames(fr, out=out)
    ms = med(lambda: sobel_frames(fr, out=out))
    print(json.dumps({"workload": f"sobel_frames {F}x{H}x{W}", "ms": ms,
                      "frames_per_s": F / ms * 1e3, "GB/s": 2.0 * F * H * W / ms / 1e6}))
if "amf" in which or "restore" in which:
    noisy, _ = O.salt_pepper(O.gradient_image(4096, 4096), 0.5, seed=42)
    t = torch.from_numpy(noisy.astype(np.uint8)).cuda()
    if "amf" in which:
        ms = med(lambda: amf_frames(t[None]))
        print(json.dumps({"workload": "amf 4096^2 50%", "ms": ms}))
    if "restore" in which:
        mask, _ = amf_frames(t[None])
        gi, gm = sk.Grid.from_tensor(t), sk.Grid.from_tensor(mask[0])
        ms = med(lambda: restore_regularize(gi, gm), reps=3)
        print(json.dumps({"workload": "restore 4096^2 50% (100 it)", "ms": ms}))
if "c5" in which:
    frames = [O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]
              for i in range(8)]
    ft = torch.from_numpy(np.stack(frames).astype(np.uint8)).cuda()

    def run():
        masks, _ = amf_frames(ft)
        for i in range(ft.shape[0]):
            restore_regularize(sk.Grid.from_tensor(ft[i]), sk.Grid.from_tensor(masks[i]))

    ms = med(run, reps=3)
    print(json.dumps({"workload": "C5 8 frames serial", "ms": ms, "frames_per_s": 8e3 / ms}))
