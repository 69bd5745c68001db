"""Time (and, under ncu, profile) the non-Helmholtz workloads at config sizes.

    python tools/prof_apps.py [--which sobel,amf,restore,c5] [--reps 3]
Prints one JSON line per workload.  Not the bench (see bench.py)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1609_04567_b200 as sk
from oracle import stencil_oracle as O
from paper_1609_04567_b200.apps import amf_detect, amf_frames, restore_regularize, sobel_frames

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="sobel,amf,restore,c5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=4096)
a = ap.parse_args()
which = a.which.split(",")


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        r = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, r


if "sobel" in which:
    F, H, W = 64, 2048, 2048
    fr = torch.randint(0, 256, (F, H, W), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(fr)
    ms, _ = timed(lambda: sobel_frames(fr, out=out), a.reps)
    gbs = 2.0 * F * H * W / (ms / 1e3) / 1e9
    print(json.dumps({"workload": "sobel_frames", "frames": F, "ms": ms,
                      "frames_per_s": F / (ms / 1e3), "GB/s": gbs}))

if "amf" in which or "restore" in which:
    n = a.n
    noisy, truth = O.salt_pepper(O.gradient_image(n, n), 0.5, seed=42)
    t = torch.from_numpy(noisy.astype(np.uint8)).cuda()
    if "amf" in which:
        ms, (m, cnt) = timed(lambda: amf_frames(t[None]), a.reps)
        print(json.dumps({"workload": f"amf {n}^2 50%", "ms": ms, "flagged": int(cnt[0]),
                          "Mpix_per_s": n * n / (ms / 1e3) / 1e6}))
    if "restore" in which:
        mask, _ = amf_frames(t[None])
        g_img = sk.Grid.from_tensor(t)
        g_mask = sk.Grid.from_tensor(mask[0])
        ms, (out, rep) = timed(lambda: restore_regularize(g_img, g_mask), 1)
        flagged = int(mask.sum())
        print(json.dumps({"workload": f"restore {n}^2 50%", "ms": ms, "iterations": rep.iterations,
                          "exhausted": rep.exhausted, "flagged": flagged,
                          "ms_per_iteration": ms / rep.iterations,
                          "flagged_updates_per_s": flagged * rep.iterations / (ms / 1e3)}))

if "c5" in which:
    frames = [O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]
              for i in range(8)]
    ft = torch.from_numpy(np.stack(frames).astype(np.uint8)).cuda()

    def run():
        masks, _ = amf_frames(ft)
        outs = []
        for i in range(ft.shape[0]):
            o, r = restore_regularize(sk.Grid.from_tensor(ft[i]), sk.Grid.from_tensor(masks[i]))
            outs.append(r.iterations)
        return outs

    ms, its = timed(run, 1)
    print(json.dumps({"workload": "C5 8 frames 1080p 10% (serial, one stream)", "ms": ms,
                      "frames_per_s": 8 / (ms / 1e3), "iterations": its}))
