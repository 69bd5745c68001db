"""BASELINE C5 at its stated size: all 1000 frames of the synthetic video
(frame i = salt_pepper(_synthetic_frame(1080, 1920, i), 0.1, seed=42+i),
reference cli.py:187-191, apps/denoise.py:295-304) detected and restored on
the device in batches of 32 (amf_frames + restore_frames, the farm the bench
times), each frame against the REAL reference's run of it
(tests/golden/golden_c5.json, tests/golden/make_golden_c5.py): the noise
mask's SHA-256, the iteration count, the exhausted flag and the SHA-256 of
the fp64 restored frame, bit for bit ("pin all 1000 frames'
SHA-256 and iteration counts")."""

import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_c5.json")


def _frame(i):
    from oracle import stencil_oracle as O

    return O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0].astype(np.uint8)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_c5_every_frame_matches_the_reference():
    import torch

    from paper_1609_04567_b200.apps import amf_frames, restore_frames

    gold = json.load(open(GOLD))["frames"]
    n = len(gold)
    assert n >= 64
    pool = ThreadPoolExecutor(max(4, os.cpu_count() or 4))
    B = 32
    checked = 0
    for b0 in range(0, n, B):
        ids = list(range(b0, min(n, b0 + B)))
        host = np.stack(list(pool.map(_frame, ids)))
        dev = torch.from_numpy(host).cuda()
        masks, counts = amf_frames(dev)
        outs, reps = restore_frames(dev, masks)
        m_host = masks.cpu().numpy()
        o_host = [o.cpu().numpy() for o in outs]
        shas = list(pool.map(_sha, o_host))
        msha = list(pool.map(lambda a: _sha(np.ascontiguousarray(a)), m_host))
        for k, i in enumerate(ids):
            g = gold[str(i)]
            assert int(counts[k]) == g["flagged"], i
            assert msha[k] == g["sha_mask"], i
            assert reps[k].iterations == g["iterations"] and reps[k].exhausted == g["exhausted"], i
            assert shas[k] == g["sha"], i
            checked += 1
    assert checked == n
