"""C3 at its BASELINE size, from the REAL reference (slow: ~10-20 min on 8 cores).

    python tests/golden/make_golden_c3.py   -> tests/golden/golden_c3.json

4096x4096 gradient image, 50% salt-and-pepper (seed 42), amf_detect(wmax=7)
then restore_regularize(RestoreConfig()), both 1:n over 8 partitions.
Records SHA-256 of the mask and of the fp64 / rint-uint8 outputs, the
iteration count, exhaustion and the final reduce.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from stencilkit import Grid  # noqa: E402
from stencilkit.apps import amf_detect, restore_regularize, salt_pepper  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
r = np.arange(n)[:, None]
c = np.arange(n)[None, :]
clean = Grid.from_array(((r * 3 + c * 2) % 200 + 20).astype(np.int64))
t0 = time.perf_counter()
noisy, _ = salt_pepper(clean, 0.5, seed=42)
mask = amf_detect(noisy, partitions=8)
t1 = time.perf_counter()
out, rep = restore_regularize(noisy, mask, partitions=8)
t2 = time.perf_counter()
a = out.to_array().astype(np.float64)
m = mask.to_array().astype(np.uint8)
res = {f"C3_denoise_{n}": dict(
    rows=n, cols=n, P=8, flagged=int(m.sum()), sha_mask=sha(m), iterations=rep.iterations,
    exhausted=rep.exhausted, final_reduce=rep.final_reduce, sha=sha(a),
    sha_u8=sha(np.clip(np.rint(a), 0, 255).astype(np.uint8)), detect_s=t1 - t0,
    restore_s=t2 - t1)}
with open(os.path.join(HERE, f"golden_c3_{n}.json"), "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res))
