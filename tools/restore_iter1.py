"""Run one restore iteration 1 alone (every flagged pixel active), for an
ncu capture of that launch and the per-pixel instruction counts the bench
roofline uses (profiles/restore_counts.json):

    ncu --set full -k regex:restore_sweep -c 1 ... python tools/restore_iter1.py [--c5]

default: C3 (4096^2, 50% noise); --c5: the C5 farm batch (32 distinct
1080x1920 frames at 10% noise stacked into one grid, as bench_workloads.c5).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench_workloads as W  # noqa: E402
import paper_1609_04567_b200 as sk  # noqa: E402
from paper_1609_04567_b200.apps import amf_detect, amf_frames  # noqa: E402

if "--c5" in sys.argv:
    import numpy as np

    sub = torch.from_numpy(np.stack(W._c5_frames(32))).cuda()
    masks, counts = amf_frames(sub)
    F, H, Wd = sub.shape
    img, mask = sub.reshape(F * H, Wd), masks.reshape(F * H, Wd)
else:
    img = torch.from_numpy(W._c3_input()).cuda()
    mask = amf_detect(sk.Grid.from_tensor(img)).tensor()
print("flagged", int(mask.sum().item()), "iter1_ms", W._restore_iter1_ms(sk, img, mask))
