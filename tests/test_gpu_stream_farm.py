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


def test_video_pipeline_host_buffers_recycle_pinned_frames():
    """host_buffers=True: results arrive by DMA in recycled pinned host frames
    (pinned uint8 frames in); each frame, copied by the writer while it owns
    the buffer, is the reference's (golden_c5 SHA-256), in stream order."""
    import torch

    meta = json.load(open(GOLD))["frames"]
    from paper_1609_04567_b200.apps import video_restore_pipeline

    k = 12
    host = torch.from_numpy(np.stack([c5_frame(i).astype(np.uint8) for i in range(k)])).pin_memory()
    frames = [sk.Grid.from_tensor(host[i]) for i in range(k)]
    got, ptrs = [], set()

    def writer(g):
        t = g.tensor()
        assert t.is_pinned() and not t.is_cuda
        ptrs.add(t.data_ptr())
        got.append(g.to_array())

    video_restore_pipeline(frames, width=3, writer=writer, host_buffers=True)
    assert len(got) == k
    for i in range(k):
        assert sha(got[i]) == meta[str(i)]["sha"], i
    assert len(ptrs) < k  # buffers were reused


def test_video_pipeline_batched_farm_failures_shapes_loader(monkeypatch):
    """The batch-granular farm (default for 1:1 with fused detection) keeps
    the stream contract of the lane farm (SK_LANE_FARM=1): stream order,
    a bad frame (pixel out of range), a failing loader call and a failing
    write poison only their own item, shape changes split batches, and
    items_in == items_out + len(failures)."""
    from paper_1609_04567_b200.apps import salt_pepper, video_restore_pipeline

    def frame(i, h, w):
        r = np.arange(h)[:, None]
        c = np.arange(w)[None, :]
        return salt_pepper(sk.Grid.from_array(((r * 3 + c * 2 + i) % 200 + 20).astype(np.int64)),
                           0.2, seed=70 + i)[0]

    src = [frame(0, 40, 50), frame(1, 40, 50), "bad-load", frame(3, 30, 20),
           sk.Grid.from_array(np.full((40, 50), 300, dtype=np.int64)), frame(5, 40, 50),
           frame(6, 40, 50), frame(7, 30, 20)]

    def loader(x):
        if isinstance(x, str):
            raise ValueError("cannot load")
        return x

    results = {}
    for lane_farm in ("", "1"):
        if lane_farm:
            monkeypatch.setenv("SK_LANE_FARM", "1")
        else:
            monkeypatch.delenv("SK_LANE_FARM", raising=False)
        got = []

        def writer(g):
            if len(got) == 3:
                got.append(None)
                raise RuntimeError("disk full")
            got.append(g.to_array())

        rep = video_restore_pipeline(src, width=4, loader=loader, writer=writer)
        assert rep.items_in == 8 and rep.items_in == rep.items_out + len(rep.failures)
        results[lane_farm] = (got, sorted(s for s, _e in rep.failures))
    (g0, f0), (g1, f1) = results[""], results["1"]
    assert f0 == f1 == [2, 4, 5]  # the load, the out-of-range frame, the failed write
    assert len(g0) == len(g1)
    for a, b in zip(g0, g1):
        assert (a is None and b is None) or np.array_equal(a, b)


def test_sobel_stream_order_failures_and_host_buffers():
    """sobel_stream (C2 stream mode): frames in stream order through the
    batched TMA Sobel, every output the oracle's, a bad frame failing alone,
    pinned host buffers recycled."""
    import torch

    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import sobel_stream

    rng = np.random.default_rng(21)
    imgs = [rng.integers(0, 256, (97, 333)).astype(np.uint8) for _ in range(9)]
    imgs.insert(4, rng.integers(0, 256, (40, 2049)).astype(np.uint8))  # shape change mid-stream
    src = [sk.Grid(a.shape, a) for a in imgs]
    src.insert(6, sk.Grid.from_array(np.full((97, 333), 300, dtype=np.int64)))  # out of range
    for hb in (False, True):
        got, ptrs = [], set()

        def writer(g):
            if hb:
                t = g.tensor()
                assert t.is_pinned() and t.dtype == torch.uint8
                ptrs.add(t.untyped_storage().data_ptr())
            got.append(np.asarray(g.to_array()).astype(np.uint8))

        rep = sobel_stream(src, writer=writer, width=4, host_buffers=hb)
        assert rep.items_in == 11 and rep.items_out == 10 and [s for s, _ in rep.failures] == [6]
        want = [O.sobel(a) for a in imgs]
        assert len(got) == 10
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
        if hb:
            assert len(ptrs) < 10
