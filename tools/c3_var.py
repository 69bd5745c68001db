"""Per-step timing spread of C3 (AMF + restore) to chase run-to-run variance."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1609_04567_b200 as sk
from bench_workloads import _c3_input
from paper_1609_04567_b200.apps import amf_detect, restore_regularize

img = torch.from_numpy(_c3_input()).cuda()
g = sk.Grid.from_tensor(img)
for k in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = amf_detect(g)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    o, r = restore_regularize(g, m)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"step {k}: amf {1e3*(t1-t0):.1f} ms  restore {1e3*(t2-t1):.1f} ms  it={r.iterations}",
          flush=True)
