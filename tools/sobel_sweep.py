"""Time the batched Sobel (`sobel_frames`) on the C2 stack (512 x 2048^2 u8,
resident in HBM) with CUDA events: one line of JSON per run.  Used to A/B the
TMA ring configurations (SK_TMA_CFG / SK_TMA_HINT / SK_SOBEL_TMA=0 env)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04567_b200.apps import sobel_frames  # noqa: E402

F = int(os.environ.get("FRAMES", "512"))
frames = torch.randint(0, 256, (F, 2048, 2048), dtype=torch.uint8, device="cuda")
out = torch.empty_like(frames)
for _ in range(3):
    sobel_frames(frames, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    sobel_frames(frames, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts)[len(ts) // 2]
print(json.dumps({"cfg": os.environ.get("SK_TMA_CFG", "0"), "hint": os.environ.get("SK_TMA_HINT", "0"),
                  "tma": os.environ.get("SK_SOBEL_TMA", "1"), "ms": round(ms, 4),
                  "min_ms": round(min(ts), 4), "GBps": round(2 * F * 2048 * 2048 / ms / 1e6, 1)}))
