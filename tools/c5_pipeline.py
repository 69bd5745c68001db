"""C5 stream: video_restore_pipeline frames/s vs farm width and batch cap
(pinned host uint8 frames in, fp64 frames out into recycled pinned host
frames).  Exploration tool, not the bench.

    python tools/c5_pipeline.py [frames] [width,width,...]
    SK_BATCH_CAP=<n> caps the per-GPU restore batch (default: half the lanes)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_04567_b200 as sk  # noqa: E402
from bench_workloads import _c5_frames_range  # noqa: E402
from paper_1609_04567_b200.apps import video_restore_pipeline  # noqa: E402

if os.environ.get("SWITCH"):
    sys.setswitchinterval(float(os.environ["SWITCH"]))
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 256
host = torch.from_numpy(np.stack(_c5_frames_range(0, nf))).pin_memory()
frames = [sk.Grid.from_tensor(host[i]) for i in range(nf)]
video_restore_pipeline(frames[:16], width=4, writer=lambda g: None, host_buffers=True)
for width in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "64"])]:
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = video_restore_pipeline(frames, width=width, writer=lambda g: None, host_buffers=True)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"width": width, "frames": nf, "cap": os.environ.get("SK_BATCH_CAP"), "switch": sys.getswitchinterval(),
                      "frames_per_s": [round(nf / t, 1) for t in ts],
                      "median": round(nf / statistics.median(ts), 1)}), flush=True)
