"""The TMA row-ring Sobel (csrc/sk_sobel_tma.cu) behind `sobel_frames`, the
stream-mode entry point, against the oracle's restatement of the reference
block kernel (oracle.stencil_oracle.sobel; apps/sobel.py:47-66) and its
per-frame pixel sum (apps/sobel.py:73-74), pixel for pixel.

Geometries cover: each inner TMA box width (256/128/64/32/16-byte blocks),
pitches wider than the row, a CTA run that crosses frame boundaries (many
small frames), single-row / single-column / two-row frames (every pixel a
border pixel), widths that are not a multiple of 8 (masked lanes), and a
width over 2048 (the generic batched sweep takes over)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(F, H, W, pitch, seed):
    import torch

    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import sobel_frames

    rng = np.random.default_rng(seed)
    imgs = rng.integers(0, 256, (F, H, W)).astype(np.uint8)
    if seed % 2:  # smooth content too: small gradients exercise the rounding
        r = np.arange(H)[:, None]
        c = np.arange(W)[None, :]
        imgs[0] = ((r * 3 + c * 5) % 256).astype(np.uint8)
    buf = torch.full((F, H, pitch), 77, dtype=torch.uint8, device="cuda")
    buf[:, :, :W] = torch.from_numpy(imgs).cuda()
    outp = -(-W // 16) * 16
    out = torch.full((F, H, outp), 5, dtype=torch.uint8, device="cuda")
    edges, sums = sobel_frames(buf[:, :, :W], out=out[:, :, :W])
    torch.cuda.synchronize()
    got = edges.cpu().numpy()
    s = sums.cpu().numpy()
    for f in range(F):
        want = O.sobel(imgs[f])
        assert np.array_equal(got[f], want), (F, H, W, pitch, f)
        assert int(s[f]) == int(want.astype(np.int64).sum()), (F, H, W, pitch, f)


@pytest.mark.parametrize("F,H,W,pitch", [
    (1, 2048, 2048, 2048),   # C2 frame, 256-byte blocks
    (5, 37, 1920, 1920),     # 1080p width: 128-byte blocks, a half-used last warp
    (3, 130, 259, 272),      # 16-byte blocks, masked lanes, pitch > width
    (4, 64, 2000, 2048),     # 256-byte blocks reaching into the pitch
    (9, 3, 96, 96),          # 32-byte blocks; every run crosses frames
    (40, 7, 64, 64),         # many tiny frames: segments of 1..7 rows
    (3, 1, 16, 16),          # one row: every pixel on the border
    (2, 2, 17, 32),          # two rows, odd width
    (6, 50, 1, 16),          # one column
    (2, 33, 2064, 2064),     # wider than 2048: the generic batched sweep
])
def test_sobel_frames_tma_geometries(F, H, W, pitch):
    _case(F, H, W, pitch, seed=F * 1000 + H + W)


def test_sobel_frames_tma_repeat_and_streams():
    """Back-to-back launches on two streams reuse nothing stale."""
    import torch

    from oracle import stencil_oracle as O
    from paper_1609_04567_b200.apps import sobel_frames

    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 256, (6, 300, 1024)).astype(np.uint8)
    frames = torch.from_numpy(imgs).cuda()
    want = [O.sobel(i) for i in imgs]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    res = []
    for k in range(4):
        st = sts[k % 2]
        with torch.cuda.stream(st):
            res.append(sobel_frames(frames[k % 3: k % 3 + 3], stream=st))
    torch.cuda.synchronize()
    for k, (e, s) in enumerate(res):
        for i in range(3):
            assert np.array_equal(e[i].cpu().numpy(), want[k % 3 + i])
            assert int(s[i]) == int(want[k % 3 + i].astype(np.int64).sum())
