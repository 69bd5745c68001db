"""The stream tier on the GPU: lanes (device + CUDA stream per farm
replica), stream-ordered hand-off, and the multi-device video pipeline
pinned to the reference's C5 frames (tests/golden/golden_c5.json, produced
by the real reference, make_golden_c5.py).

Reference: streams.py:215-376 (ordered farm, run_stream),
apps/denoise.py:307-368 (video_restore_pipeline), cli.py:187-191 (frames).
"""

import hashlib
import json
import os
import threading

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
from paper_1609_04567_b200.streams import Stage, current_lane, ordered_farm, pipeline, run_stream

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_c5.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def c5_frame(i):
    from oracle import stencil_oracle as O

    return O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]


def test_lanes_get_their_own_streams_and_devices():
    import torch

    seen = []
    lock = threading.Lock()

    def factory():
        lane = current_lane()
        with lock:
            seen.append((lane.index, lane.device, lane.stream))

        def fn(x):
            assert torch.cuda.current_stream() == current_lane().stream
            return x

        return fn

    out = []
    run_stream(range(10), ordered_farm(Stage(factory=factory), 3, devices=[0, 0, 0]), out.append)
    assert out == list(range(10))
    assert sorted(s[0] for s in seen) == [0, 1, 2]
    assert all(s[1] == 0 for s in seen)
    assert len({s[2].cuda_stream for s in seen}) == 3


def test_async_stages_hand_off_by_events():
    """Stages return as soon as their work is enqueued; the next stage's
    lane waits on the item's event, the sink sees completed results, in
    order, although the lanes finish their GPU work out of order."""
    import torch

    n = 1 << 20

    def produce(x):
        t = torch.full((n,), float(x), device="cuda")
        torch.cuda._sleep(int(2_000_000 * ((x * 7) % 5)))  # uneven GPU time per item
        t.add_(1.0)
        return t  # not synchronised

    def scale(t):
        return t * 2.0  # runs on another lane's stream after the event

    got = []
    rep = run_stream(range(24), pipeline(ordered_farm(Stage(produce), 4),
                                         ordered_farm(Stage(scale), 2)),
                     lambda t: got.append(float(t[0].item()) + float(t[-1].item())))
    assert rep.items_out == 24 and rep.failures == []
    assert got == [4.0 * (x + 1) for x in range(24)]


def test_video_pipeline_frames_match_reference_c5():
    """video_restore_pipeline over C5 frames with the farm spread over a
    device list (here the box's one GPU, twice): every frame's restored
    image bit-identical to the reference's, in stream order."""
    meta = json.load(open(GOLD))["frames"]
    from paper_1609_04567_b200.apps import video_restore_pipeline

    k = 12
    frames = [sk.Grid.from_array(c5_frame(i)) for i in range(k)]
    for width, devices in ((4, [0, 0]), (3, None)):
        got = []
        rep = video_restore_pipeline(frames, width=width, devices=devices,
                                     writer=lambda g: got.append(g.to_array()))
        assert rep.items_in == rep.items_out == k and rep.failures == []
        for i, a in enumerate(got):
            assert sha(a) == meta[str(i)]["sha"], (width, i)
            assert sha(np.clip(np.rint(a), 0, 255).astype(np.uint8)) == meta[str(i)]["sha_u8"]


def test_video_pipeline_mask_writer_and_1n():
    meta = json.load(open(GOLD))["frames"]
    from paper_1609_04567_b200.apps import video_restore_pipeline

    frames = [sk.Grid.from_array(c5_frame(i)) for i in range(4)]
    masks, got = [], []
    video_restore_pipeline(frames, width=2, devices=[0], mask_writer=lambda m: masks.append(
        m.to_array()), writer=lambda g: got.append(g.to_array()))
    for i in range(4):
        assert int(masks[i].sum()) == meta[str(i)]["flagged"]
        assert sha(masks[i].astype(np.uint8)) == meta[str(i)]["sha_mask"]
        assert sha(got[i]) == meta[str(i)]["sha"]
    got = []
    video_restore_pipeline(frames[:2], width=2, partitions=3, mode="1:n",
                           writer=lambda g: got.append(g.to_array()))
    for i in range(2):
        assert sha(got[i]) == meta[str(i)]["sha"]
