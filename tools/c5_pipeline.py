"""C5 stream: video_restore_pipeline frames/s vs farm width (host frames in,
device-backed restored frames out).  Not the bench; exploration tool."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1609_04567_b200 as sk
from oracle import stencil_oracle as O
from paper_1609_04567_b200.apps import video_restore_pipeline

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
base = [sk.Grid.from_array(O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0].astype(np.uint8))
        for i in range(16)]
frames = [base[i % 16] for i in range(nf)]
video_restore_pipeline(frames[:4], width=2)  # warm up (library, clocks)
for width in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8", "32"])]:
    got = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = video_restore_pipeline(frames, width=width, writer=lambda g: got.append(g.to_array()))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"width": width, "frames": nf, "s": dt, "frames_per_s": nf / dt,
                      "stages": {s.name: round(s.busy_s, 3) for s in rep.stages
                                 if not s.name.startswith("restore-")}}), flush=True)
