"""Sobel, adaptive-median detection, restoration and Life on the device vs
the reference's own outputs (golden fixtures from tests/golden/make_golden.py).

Bar: bit-exact output images/masks, bit-exact fp64 restored grids, identical
iteration counts and exhaustion flags; integer reduce values equal; the
restore SUM reduce within rel 1e-12 (deterministic fp64 sum in a different
order than numpy's pairwise sum).
"""

import numpy as np
import pytest

import paper_1609_04567_b200 as sk
import paper_1609_04567_b200.apps
from paper_1609_04567_b200.apps import (GolConfig, RestoreConfig, amf_detect, amf_frames,
                                        game_of_life, restore_regularize, sobel_filter,
                                        sobel_frames)

pytestmark = pytest.mark.gpu


def _P(m):
    return m.get("P", 1)


def test_sobel_cases(golden):
    for name in golden.cases("sobel"):
        m = golden.meta[name]
        img = golden[name + "/in"]
        P = _P(m)
        out, rep = sobel_filter(sk.Grid.from_array(img.astype(np.int64)), partitions=P,
                                mode="1:n" if P > 1 else "1:1", with_report=True)
        a = out.to_array()
        assert a.dtype == np.int64
        assert np.array_equal(a.astype(np.uint8), golden[name + "/out"]), name
        assert rep.final_reduce == m["final_reduce"] and isinstance(rep.final_reduce, int), name
        assert rep.iterations == 1
        assert vars(rep.copies) == m["ledger"], name


def test_sobel_frames_batched(golden):
    import torch

    names = ["sobel_130x259", "sobel_64x48_P3"]
    for name in names:
        img = golden[name + "/in"]
        H, W = img.shape
        Wp = -(-W // 8) * 8
        frames = torch.zeros((3, H, Wp), dtype=torch.uint8, device="cuda")
        for f in range(3):
            frames[f, :, :W] = torch.from_numpy(np.roll(img, f, axis=0))
        out = torch.zeros_like(frames)
        # the kernel works on [H, W] inside a pitched [H, Wp] buffer
        view = frames[:, :, :W]
        edges, sums = sobel_frames(view, out=out[:, :, :W])
        for f in range(3):
            ref = golden[name + "/out"] if f == 0 else None
            got = edges[f].cpu().numpy()
            if ref is not None:
                assert np.array_equal(got, ref), name
            assert int(sums[f]) == int(got.astype(np.int64).sum())


def test_amf_cases(golden):
    for name in golden.cases("amf"):
        m = golden.meta[name]
        img = golden[name + "/in"]
        P = _P(m)
        mask = amf_detect(sk.Grid.from_array(img.astype(np.int64)), wmax=m["wmax"], partitions=P,
                          mode="1:n" if P > 1 else "1:1")
        a = mask.to_array()
        assert np.array_equal(a.astype(np.uint8), golden[name + "/out"]), name
        assert int(a.sum()) == m["flagged"]


def test_amf_frames_batched(golden):
    import torch

    name = "amf_grad50_96"
    img = torch.from_numpy(golden[name + "/in"]).cuda()
    frames = torch.stack([img, img.flip(0), img.flip(1)])
    masks, counts = amf_frames(frames)
    assert np.array_equal(masks[0].cpu().numpy(), golden[name + "/out"])
    assert np.array_equal(masks[1].cpu().numpy(), golden[name + "/out"][::-1])
    assert int(counts[0]) == golden.meta[name]["flagged"]


def test_restore_cases(golden):
    for name in golden.cases("restore"):
        m = golden.meta[name]
        if not golden.has(name + "/in"):
            continue
        P = _P(m)
        cfg = RestoreConfig(max_iterations=m["max_iterations"])
        out, rep = restore_regularize(sk.Grid.from_array(golden[name + "/in"].astype(np.int64)),
                                      sk.Grid.from_array(golden[name + "/mask"].astype(np.int64)),
                                      cfg, partitions=P, mode="1:n" if P > 1 else "1:1")
        assert rep.iterations == m["iterations"], name
        assert rep.exhausted == m["exhausted"], name
        assert np.array_equal(out.to_array(), golden[name + "/out"]), name
        assert rep.final_reduce == pytest.approx(m["final_reduce"], rel=1e-12), name
        assert vars(rep.copies) == m["ledger"], name


def test_restore_empty_mask_one_iteration():
    img = sk.Grid.from_array(np.arange(64, dtype=np.int64).reshape(8, 8))
    out, rep = restore_regularize(img, sk.Grid.filled((8, 8), 0))
    assert rep.iterations == 1 and rep.final_reduce == 0.0
    assert out.data == [float(v) for v in range(64)]


def test_life_cases(golden):
    for name in golden.cases("life"):
        m = golden.meta[name]
        P = _P(m)
        out, rep = game_of_life(sk.Grid.from_array(golden[name + "/in"].astype(np.int64)),
                                config=GolConfig(m["rows"], m["cols"], steps=m["steps"]),
                                partitions=P, mode="1:n" if P > 1 else "1:1")
        assert np.array_equal(out.to_array().astype(np.uint8), golden[name + "/out"]), name
        assert rep.final_reduce == m["final_reduce"]


def test_life_blinker_and_glider():
    blinker = [[0, 0, 0, 0, 0], [0, 0, 1, 0, 0], [0, 0, 1, 0, 0], [0, 0, 1, 0, 0], [0] * 5]
    flipped = [[0] * 5, [0] * 5, [0, 1, 1, 1, 0], [0] * 5, [0] * 5]
    one = game_of_life(sk.Grid.from_rows(blinker), config=GolConfig(5, 5, steps=1))[0]
    two = game_of_life(one, config=GolConfig(5, 5, steps=1))[0]
    assert one.to_rows() == flipped and two.to_rows() == blinker


def test_video_pipeline_order_and_identity(golden):
    from paper_1609_04567_b200.apps import salt_pepper, video_restore_pipeline

    r = np.arange(12)[:, None]
    c = np.arange(12)[None, :]
    base = sk.Grid.from_array(((r * 3 + c * 2) % 200 + 20).astype(np.int64))
    frames = [salt_pepper(base, 0.2, seed=60 + i)[0] for i in range(6)]
    outs = {}
    for width in (1, 3):
        got = []
        rep = video_restore_pipeline(frames, width=width, writer=lambda g: got.append(g))
        assert rep.items_out == 6 and rep.failures == []
        outs[width] = got
    for a, b in zip(outs[1], outs[3]):
        assert a == b
    # each frame equals a standalone restore of that frame
    for f, o in zip(frames, outs[1]):
        mask = amf_detect(f)
        ref, _ = restore_regularize(f, mask)
        assert o == ref


def test_sobel_max_combinator_and_odd_shapes():
    """MAX reduce and widths/heights that exercise partial vectors, border
    fix-ups and tail rows of the SWAR kernel."""
    from oracle import stencil_oracle as O

    rng = np.random.default_rng(99)
    for shape in ((3, 3), (7, 9), (13, 250), (61, 257), (258, 263), (2, 520)):
        img = rng.integers(0, 256, shape)
        ref = O.sobel(img)
        out, rep = sk.parallel_loop("1:1", 1, 1, sk.apps.sobel_kernel, sk.max_combinator(-1),
                                    sk.stop_after(1), sk.Grid.from_array(img))
        assert np.array_equal(out.to_array().astype(np.uint8), ref), shape
        assert rep.final_reduce == int(ref.max())
        out2 = sobel_filter(sk.Grid.from_array(img))
        assert np.array_equal(out2.to_array().astype(np.uint8), ref), shape


def test_sobel_iterated_twice():
    from oracle import stencil_oracle as O

    img = np.random.default_rng(7).integers(0, 256, (40, 72))
    out, rep = sk.parallel_loop("1:1", 1, 1, sk.apps.sobel_kernel, sk.sum_combinator(0),
                                sk.stop_after(2), sk.Grid.from_array(img))
    ref = O.sobel(O.sobel(img))
    assert np.array_equal(out.to_array().astype(np.uint8), ref)
    assert rep.final_reduce == int(ref.astype(np.int64).sum())


def test_restore_frames_batch_matches_single_frame_runs(golden_large):
    """A batch of frames in one persistent launch: every frame bit-identical to
    its own restore_regularize run (and to the reference's C5 fixtures)."""
    import hashlib

    import torch

    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import amf_frames, restore_frames

    frames = [O.salt_pepper(O.synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]
              for i in range(4)]
    ft = torch.from_numpy(np.stack(frames).astype(np.uint8)).cuda()
    masks, _ = amf_frames(ft)
    outs, reps = restore_frames(ft, masks)
    for i in range(4):
        m = golden_large.meta[f"C5_restore_frame{i}_P8"]
        a = outs[i].cpu().numpy()
        assert reps[i].iterations == m["iterations"], i
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == m["sha"], i
        single, rep1 = restore_regularize(sk.Grid.from_array(frames[i]),
                                          sk.Grid.from_tensor(masks[i]))
        assert rep1.final_reduce == reps[i].final_reduce
    # a mixed batch: frames that stop early stay untouched while others run
    small = [O.salt_pepper(O.gradient_image(40, 48), lvl, seed=s)[0]
             for lvl, s in ((0.1, 1), (0.5, 2), (0.0, 3), (0.3, 4))]
    st = torch.from_numpy(np.stack(small).astype(np.uint8)).cuda()
    mk, _ = amf_frames(st)
    outs, reps = restore_frames(st, mk)
    for i in range(4):
        ref, ri, rv, rex = O.restore_loop(small[i], mk[i].cpu().numpy())
        assert reps[i].iterations == ri and reps[i].exhausted == rex, i
        assert np.array_equal(outs[i].cpu().numpy(), ref), i


def test_batched_launches_reuse_stream_counters():
    """Batched Sobel / AMF launches take chunks from a per-stream counter that
    each launch resets on exit: many launches over several streams (and
    interleaved Sobel / AMF on one stream) give the single-launch results."""
    import torch

    from paper_1609_04567_b200.apps import amf_frames

    gen = torch.Generator(device="cuda").manual_seed(5)
    frames = torch.randint(0, 256, (6, 257, 300), dtype=torch.uint8, device="cuda", generator=gen)
    fr16 = torch.zeros((6, 257, 304), dtype=torch.uint8, device="cuda")
    fr16[:, :, :300] = frames
    view = fr16[:, :, :300]  # 16-byte pitch: the ring kernel

    def o16():  # output with the same 304-byte pitch
        return torch.empty_like(fr16)[:, :, :300]

    ref_e, ref_s = sobel_frames(view, out=o16())
    ref_m, ref_c = amf_frames(view, out=o16())
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for rep in range(4):
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                outs.append(sobel_frames(view, out=o16(), stream=st))
                outs.append(amf_frames(view, out=o16()))
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        if k % 2 == 0:
            assert torch.equal(o[0], ref_e) and torch.equal(o[1], ref_s)
        else:
            assert torch.equal(o[0], ref_m) and torch.equal(o[1], ref_c)
