"""The non-default bench workloads (BASELINE.json configs C1, C2, C3, C5).

Used by `bench.py --workload c1|c2|c3|c5`; each returns the contract's JSON
line (same keys as the C4 line in bench.py).  The CPU legs time the numpy
restatement in oracle/ (bit-identical to the reference) on bounded samples.
"""

from __future__ import annotations

import json
import os
import statistics
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))


def fp64_peak():
    """Measured FP64 rates (tools/fp64_peak.cu on this pool's B200)."""
    p = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["dfma_per_s"]), float(d["dsqrt_per_s"]), "measured (profiles/r01_fp64_peak.json)"
    return 18.5e12, 1.25e12, "fallback (nominal)"


# Per active flagged pixel and iteration the reference's search does 18 steps
# x 2 evaluations of F, each 8 ring terms of (sub, mul, add, sqrt, mul, add)
# plus beta*s, plus the step bookkeeping: ~1550 DP add/mul + 288 IEEE sqrt
# (SURVEY.md 8(d)).  In DFMA-equivalents (one IEEE DSQRT costs
# dfma_rate / dsqrt_rate of them):
RESTORE_DP_OPS = 1550
RESTORE_SQRT = 288
SM_MAX_HZ = 1.965e9  # B200 boost clock (the bench's clocks line reports the live one)


def restore_roofline(flagged, t_iter1_ms, workload):
    """Roofline of restore iteration 1 (every flagged pixel active).

    The kernel certifies most ternary-search comparisons with an exact fp32
    bracket and evaluates only the rest in fp64 (sk_restore.cu), so it no
    longer executes the reference's fp64 work: its limiter is instruction
    issue.  Reported: the issue roofline (warp instructions per flagged
    pixel from the committed ncu capture, profiles/restore_counts.json, over
    the live CUDA-event time of the launch) as the headline; beside it the
    fp64 pipe fraction the kernel executes and the reference-equivalent fp64
    rate (the reference's per-pixel work over the same time: > 1 means the
    exact filter saved more fp64 work than the pipe could have done)."""
    dfma, dsq, src = fp64_peak()
    eq = RESTORE_DP_OPS + RESTORE_SQRT * dfma / dsq
    cnt = json.load(open(os.path.join(ROOT, "profiles", "restore_counts.json")))[workload]
    t = t_iter1_ms / 1e3
    issue_peak = 148 * 4 * SM_MAX_HZ  # warp instructions / s (one per scheduler per clock)
    issued = flagged * cnt["warp_inst_per_pixel"] / t
    return {"bound": "issue", "achieved": issued / 1e9, "peak": issue_peak / 1e9,
            "unit": "Gwarp-inst/s", "frac": issued / issue_peak, "traffic": None,
            "kernel": "restore_sweep (iteration 1: every flagged pixel active)",
            "work_per_unit": f"{cnt['warp_inst_per_pixel']} warp instructions per flagged "
                             f"pixel-iteration (ncu, profiles/restore_counts.json)",
            "avg_kernel_ms": t_iter1_ms,
            "peak_source": "148 SMs x 4 schedulers x 1 warp-instruction/clock at 1965 MHz",
            "issue_active_ncu": cnt["issue_active"],
            "fp64_executed": {"dp_inst_per_pixel": cnt["dp_inst_per_pixel"],
                              "frac": flagged * cnt["dp_inst_per_pixel"] / t / dfma,
                              "pipe_active_ncu": cnt["fp64_pipe_active"]},
            "fp64_reference_equivalent": {
                "work_per_unit": f"{eq:.0f} DFMA-eq per flagged pixel-iteration "
                                 f"({RESTORE_DP_OPS} DP add/mul + {RESTORE_SQRT} DSQRT, the "
                                 f"reference's search)",
                "achieved": flagged * eq / t / 1e12, "peak": dfma / 1e12, "unit": "TDFMA-eq/s",
                "frac": flagged * eq / t / dfma, "peak_source": src}}


def _traffic(key, units=1):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    v = json.load(open(p)).get(key)
    return None if v is None else v * units


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _base(args, metric, unit, value, ms, dtype, workload, extra=None):
    d = {"metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps,
         "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
         "vs_baseline": None, "dtype": dtype, "data": "synthetic",
         "config": {"workload": workload}}
    if extra:
        d["config"].update(extra)
    return d


# ----------------------------------------------------------------------------- C1


def c1(args, ClockSampler, measured_peaks, local=0):
    """1024^2 fp32 Helmholtz, MAX|delta| < 1e-4 (36 sweeps): the reference's
    own CPU-scale config.  L2-resident and latency-bound: the whole loop is
    one persistent cooperative launch."""
    import torch

    import paper_1609_04567_b200 as sk
    from paper_1609_04567_b200.apps import HelmholtzConfig, helmholtz_kernel
    from oracle import stencil_oracle as O

    n, per_step = 1024, 50
    kern = helmholtz_kernel(HelmholtzConfig(n, n))
    u0 = torch.zeros((n, n), dtype=torch.float32, device="cuda")
    f = torch.ones((n, n), dtype=torch.float32, device="cuda")
    g0, gf = sk.Grid.from_tensor(u0), sk.Grid.from_tensor(f)
    ex = sk.DeviceExecutor(1)

    def solve():
        return sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                        sk.Condition.below(1e-4), g0, env=gf, executor=ex)

    for _ in range(args.warmup * per_step):
        out, rep = solve()
    assert rep.iterations == 36
    ex.launches = 0
    s, e = _events()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        s.record()
        for _ in range(args.steps * per_step):
            out, rep = solve()
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    cells = 36.0 * n * n * per_step
    # e2e through the public API from pinned host buffers, pipelined like a
    # stream of solves (as C4): solve k+1's inputs upload on a copy stream
    # while solve k runs, and solve k's result downloads on another; every
    # solve still uploads u0 and f and reads its result back
    h0 = torch.zeros((n, n), dtype=torch.float32).pin_memory()
    hf = torch.ones((n, n), dtype=torch.float32).pin_memory()
    houts = [torch.empty((n, n), dtype=torch.float32).pin_memory() for _ in range(2)]
    cur = torch.cuda.current_stream()
    up_s, down_s = torch.cuda.Stream(), torch.cuda.Stream()
    ex_e = sk.DeviceExecutor(1)

    def upload():
        with torch.cuda.stream(up_s):
            du, df = h0.to("cuda", non_blocking=True), hf.to("cuda", non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up_s)
        return du, df, ev

    def e2e_pass(count):
        nxt = upload()
        for k in range(count):
            du, df, ev = nxt
            cur.wait_event(ev)
            du.record_stream(cur)
            df.record_stream(cur)
            if k + 1 < count:
                nxt = upload()
            o, _ = sk.loop_stencil_reduce_d(1, kern, sk.abs_change(), sk.max_combinator(0.0),
                                            sk.Condition.below(1e-4), sk.Grid.from_tensor(du),
                                            env=sk.Grid.from_tensor(df), executor=ex_e)
            ot = o.tensor()
            down_s.wait_stream(cur)
            with torch.cuda.stream(down_s):
                houts[k % 2].copy_(ot, non_blocking=True)
            ot.record_stream(down_s)
        torch.cuda.synchronize()

    e2e_pass(4)  # warm
    t0 = time.perf_counter()
    e2e_pass(per_step)
    e2e_s = (time.perf_counter() - t0) / per_step
    # roofline: the persistent loop's time per sweep (barrier + fold included)
    peak, pk = measured_peaks()
    sweep_ms = ms / per_step / 36
    ach = 12.0 * n * n / (sweep_ms / 1e3) / 1e9
    t0 = time.perf_counter()
    O.helmholtz_loop(np.zeros((n, n), np.float32), np.ones((n, n), np.float32),
                     O.helmholtz_consts(), delta="abs", op="max", cond=lambda v, it: v < 1e-4,
                     P=os.cpu_count() or 1, threads=os.cpu_count() or 1)
    cpu = 36.0 * n * n / (time.perf_counter() - t0)
    line = _base(args, "stencil cell-updates/s", "cell-updates/s", cells / (ms / 1e3), ms, "f32",
                 "C1 Helmholtz 1024x1024 fp32, MAX|delta|<1e-4 (36 sweeps), "
                 f"{per_step} solves per step", {"l2": "12.6 MB working set is L2-resident "
                                                       "by design (the config's own size)"})
    line.update({
        "gpu_launches": ex.launches,
        "e2e": {"value": 36.0 * n * n / e2e_s, "unit": "cell-updates/s",
                "h2d_bytes_per_step": 8 * n * n * per_step,
                "d2h_bytes_per_step": 4 * n * n * per_step, "ms_per_solve": e2e_s * 1e3,
                "mode": f"{per_step} solves through loop_stencil_reduce_d from pinned host "
                        "buffers, pipelined: solve k+1's H2D overlaps solve k and its D2H"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": None, "avg_kernel_ms": sweep_ms,
                     "kernel": "helm_resident<float> (grid held in registers/smem for the whole loop; one cooperative launch per solve): time per sweep incl. grid barrier",
                     "note": "latency-bound (L2-resident); one cooperative launch per solve",
                     "peak_source": pk},
        "cpu_baseline": {"value": cpu, "unit": "cell-updates/s", "cores": os.cpu_count(),
                         "kind": "port", "sample": "the full C1 solve (36 sweeps) with the "
                                                   "numpy restatement, P=cores threads"},
        "clocks": clk.summary(),
    })
    return line


# ----------------------------------------------------------------------------- C2


def _sobel_cpu(frames=8):
    from oracle import stencil_oracle as O

    rng = np.random.default_rng(0)
    imgs = [rng.integers(0, 256, (2048, 2048)).astype(np.uint8) for _ in range(frames)]
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as pool:
        list(pool.map(O.sobel, imgs))
    dt = time.perf_counter() - t0
    return frames / dt, cores, f"{frames} random 2048x2048 frames, oracle Sobel on {cores} threads"


def c2(args, ClockSampler, measured_peaks, local=0, world=1, rank=0):
    """Sobel over a stream of 512 synthetic 2048x2048 uint8 frames.
    value: frames resident in HBM, batched launches of 64 frames;
    e2e: frames from pinned host memory, H2D / kernel / D2H overlapped over
    3 CUDA streams (the stream mode)."""
    import torch

    from paper_1609_04567_b200.apps import sobel_frames

    F_all, B, H, W = 512, 512, 2048, 2048
    F = F_all // world
    gen = torch.Generator(device="cuda").manual_seed(rank)
    frames = torch.randint(0, 256, (F, H, W), dtype=torch.uint8, device="cuda", generator=gen)
    out = torch.empty_like(frames)

    def step(timed=None):
        for b in range(0, F, B):
            if timed is not None:
                a, z = _events()
                a.record()
            sobel_frames(frames[b:b + B], out=out[b:b + B])
            if timed is not None:
                z.record()
                timed.append((a, z))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = []
    s, e = _events()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        # GPU-side gate (outside the timed region): the host enqueues all K
        # steps while the GPU spins ~20 ms, so a host-side hiccup (page
        # faults, GC, the clock sampler's fork) cannot open gaps between the
        # timed launches; the events still bracket exactly the K steps
        torch.cuda._sleep(40_000_000)
        s.record()
        for _ in range(args.steps):
            step(ev)
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    kms = statistics.mean(a.elapsed_time(z) for a, z in ev)
    peak, pk = measured_peaks()
    ach = 2.0 * B * H * W / (kms / 1e3) / 1e9
    # e2e: the stream mode through the public API -- sobel_stream over pinned
    # host uint8 frames, edges DMA'd back into recycled pinned host frames
    # handed to the writer in stream order (median of 3 passes)
    import paper_1609_04567_b200 as sk
    from paper_1609_04567_b200.apps import sobel_stream

    hin = torch.randint(0, 256, (F, H, W), dtype=torch.uint8).pin_memory()
    grids = [sk.Grid.from_tensor(hin[i]) for i in range(F)]
    seen = []

    def writer(g):
        seen.append(int(g.tensor()[1024, 1024]))

    width = 32
    for _ in range(2):  # warm: the process-wide pinned result pool reaches its steady size
        sobel_stream(grids, writer=writer, width=width, host_buffers=True)
    passes = []
    for _ in range(3):
        seen.clear()
        t0 = time.perf_counter()
        sobel_stream(grids, writer=writer, width=width, host_buffers=True)
        passes.append(time.perf_counter() - t0)
        assert len(seen) == F
    e2e_s = statistics.median(passes)
    cpu, cores, sample = _sobel_cpu() if rank == 0 else (None, None, None)
    line = _base(args, "frames/s", "frames/s", F * world / (ms / 1e3), ms, "u8",
                 f"C2 Sobel over {F_all} synthetic 2048x2048 uint8 frames (batches of {B})",
                 {"frames": F_all, "parallelism": f"frames split over {world} GPU(s)",
                  "l2": f"{F * H * W * 2 / 1e9:.1f} GB per step > L2"})
    line["n_gpus"] = world
    line.update({
        "gpu_launches": args.steps * (F // B),
        "e2e": {"value": F * world / e2e_s, "unit": "frames/s",
                "h2d_bytes_per_step": F * H * W, "d2h_bytes_per_step": F * H * W,
                "passes_frames_per_s": [round(F / x, 1) for x in passes],
                "mode": f"median of 3 passes of sobel_stream(width={width}, host_buffers=True) "
                        f"over {F} pinned host frames: batches of {width // 2} through the TMA "
                        "Sobel, two in flight per GPU (upload / launch / read-back overlap), "
                        "edges DMA'd into recycled pinned frames"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": _traffic("sobel_2048_per_frame", B),
                     "avg_kernel_ms": kms,
                     "kernel": f"sobel_tma_kernel ({B} frames/launch; TMA row ring), 2 B/pixel",
                     "note": "issue-bound (79% issue-active; FMA 57%, XU 60%, ALU 54%): exact "
                             "f16-subnormal features, fp32 magnitude, per-pixel sqrt/round "
                             "(profiles/r02_ncu_sobel_tma.json; the same ring as a pure copy "
                             "streams 5.9 TB/s)",
                     "peak_source": pk},
        "cpu_baseline": None if cpu is None else
        {"value": cpu, "unit": "frames/s", "cores": cores, "kind": "port", "sample": sample},
        "clocks": clk.summary(),
    })
    return line


# ----------------------------------------------------------------------------- C3


def _c3_input(n=4096):
    """C3 input: a smooth gradient image (values 20..219) with 50% salt and
    pepper noise (PCG64 seed 42), via the package's host-side synthesis."""
    from paper_1609_04567_b200.apps.denoise import salt_pepper_array

    r = np.arange(n, dtype=np.int64)[:, None]
    c = np.arange(n, dtype=np.int64)[None, :]
    noisy, _ = salt_pepper_array((r * 3 + c * 2) % 200 + 20, 0.5, seed=42)
    return noisy.astype(np.uint8)


def _restore_iter1_ms(sk, img_t, mask_t):
    """Duration of restore iteration 1 (every flagged pixel active): CUDA events
    around that launch (timing executor, same kernels)."""
    from paper_1609_04567_b200.apps.denoise import RestoreConfig, _float_sum, restore_kernel

    ex = sk.DeviceExecutor(1, timing=True)
    mk = sk.Grid.from_tensor(mask_t)
    mk.value_range = (0, 1)
    sk.loop_stencil_reduce_d(1, restore_kernel(RestoreConfig()), sk.abs_change(), _float_sum(),
                             sk.stop_after(1), sk.Grid.from_tensor(img_t), env=mk, executor=ex,
                             indexed=True)
    return ex.last_kernel_time[0] / max(ex.last_kernel_time[1], 1)


def c3(args, ClockSampler, measured_peaks, local=0):
    """Two-phase restoration of one 4096^2 image with 50% salt-and-pepper
    noise: AMF detection + 100 restore iterations (the cap; bit-exact)."""
    import torch

    import paper_1609_04567_b200 as sk
    from paper_1609_04567_b200.apps import amf_detect, restore_regularize
    from oracle import stencil_oracle as O

    noisy = _c3_input()
    img = torch.from_numpy(noisy).cuda()
    g = sk.Grid.from_tensor(img)

    def step():
        mask = amf_detect(g)
        out, rep = restore_regularize(g, mask)
        return out, rep, mask

    for _ in range(args.warmup):
        out, rep, mask = step()
    assert rep.iterations == 100 and rep.exhausted
    s, e = _events()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        s.record()
        for _ in range(args.steps):
            out, rep, mask = step()
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    flagged = int(mask.tensor().sum().item())
    t1 = _restore_iter1_ms(sk, img, mask.tensor())
    # e2e: host uint8 image in, host fp64 restored image out, through the
    # public API.  Headline: the image in pinned host memory (one DMA up)
    # and the result read into a pinned host array with prefetch_host(out=)
    # (one DMA down); drop_in: numpy in, a fresh numpy array out (pageable
    # copies; the fresh 134 MB array's first-touch page faults dominate)
    hin = torch.from_numpy(noisy).pin_memory()
    hout = torch.empty(noisy.shape, dtype=torch.float64).pin_memory().numpy()

    def e2e():
        gh = sk.Grid.from_tensor(hin)
        m2 = amf_detect(gh)
        o2, _ = restore_regularize(gh, m2)
        o2.prefetch_host(out=hout)
        return o2.to_array()

    def e2e_drop_in():
        gh = sk.Grid.from_array(noisy)
        m2 = amf_detect(gh)
        o2, _ = restore_regularize(gh, m2)
        return o2.to_array()

    assert np.array_equal(e2e(), e2e_drop_in())
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        e2e()
        ts.append(time.perf_counter() - t0)
    e2e_s = sorted(ts)[1]
    t0 = time.perf_counter()
    e2e_drop_in()
    drop_s = time.perf_counter() - t0
    # CPU: the port on a 1024^2 crop of the same image family, extrapolated x16
    small = _c3_input(1024)
    t0 = time.perf_counter()
    m = O.amf_detect(small)
    t_amf = time.perf_counter() - t0
    work = small.astype(np.float64)
    t0 = time.perf_counter()
    for _ in range(3):
        work = O.restore_sweep(work, m)
    t_it = (time.perf_counter() - t0) / 3
    cpu_s = 16 * (t_amf + 100 * t_it)
    line = _base(args, "frames/s (denoise)", "images/s", 1e3 / ms, ms, "f64",
                 "C3 two-phase denoise 4096x4096 uint8, 50% noise: AMF + 100 restore iterations",
                 {"flagged": flagged, "iterations": rep.iterations})
    line.update({
        "gpu_launches": None,
        "e2e": {"value": 1.0 / e2e_s, "unit": "images/s", "h2d_bytes_per_step": noisy.size,
                "d2h_bytes_per_step": 8 * noisy.size,
                "mode": "median of 3: amf_detect + restore_regularize on a host grid over pinned "
                        "memory, the fp64 result read into a pinned host array "
                        "(prefetch_host(out=)); one image at a time",
                "drop_in": {"value": 1.0 / drop_s, "mode": "numpy image in (Grid.from_array), "
                                                          "fresh numpy array out (to_array)"}},
        "roofline": restore_roofline(flagged, t1, "c3"),
        "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "images/s", "cores": 1, "kind": "port",
                         "sample": "oracle AMF + 3 restore sweeps on a 1024^2 image "
                                   "(same generator), extrapolated to 4096^2 x 100 iterations "
                                   "(x16 pixels)"},
        "clocks": clk.summary(),
    })
    # per image: one persistent launch per phase (AMF, restore) + the
    # flagged-list build (count, scan, scatter, bounds)
    line["gpu_launches"] = 6 * args.steps
    return line


# ----------------------------------------------------------------------------- C5


def _c5_frame(i, rows=1080, cols=1920, level=0.1):
    """C5 input frame i: the CLI's synthetic frame (reference cli.py:187-191)
    with salt-and-pepper noise from numpy's PCG64 seeded 42 + i (reference
    apps/denoise.py:295-304), via the package's host-side input synthesis."""
    from paper_1609_04567_b200.apps.denoise import salt_pepper_array

    r = np.arange(rows, dtype=np.int64)[:, None]
    c = np.arange(cols, dtype=np.int64)[None, :]
    noisy, _ = salt_pepper_array((3 * r + 2 * c + 5 * i) % 256, level, seed=42 + i)
    return noisy.astype(np.uint8)


def _c5_frames_range(first, n):
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as ex:
        return list(ex.map(_c5_frame, range(first, first + n)))


def _c5_frames(n):
    """n distinct C5 frames, generated on all host cores (numpy releases the
    GIL in the PCG64 fills); not timed."""
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as ex:
        return list(ex.map(_c5_frame, range(n)))


def c5(args, ClockSampler, measured_peaks, local=0, world=1, rank=0, width=32):
    """Streaming video denoise: 1000 synthetic 1920x1080 frames (10% noise), a
    farm of stencil-reduce loops.
    value: frames resident in HBM; per batch of 32 frames one batched AMF
    launch + one persistent restore launch in which every frame runs its own
    loop to its own stop (restore_frames);
    e2e: video_restore_pipeline (read -> detect -> ordered_farm(restore, W) ->
    write) from host uint8 frames to host fp64 frames."""
    import torch

    import paper_1609_04567_b200 as sk
    from paper_1609_04567_b200.apps import (amf_frames, restore_regularize,
                                            video_restore_pipeline)
    from oracle import stencil_oracle as O

    total = 1000 // world
    # every frame of this rank's share of the 1000 is distinct (frame index
    # rank * total + i), generated on the host once, resident in HBM for
    # `value` and in pinned host memory for `e2e`
    host = np.stack(_c5_frames_range(rank * total, total))
    dev = torch.from_numpy(host).cuda()
    B = 32  # frames per persistent launch (the device-side farm of loops)
    from paper_1609_04567_b200.apps import restore_frames

    def step(n=total):
        its = []
        for b0 in range(0, n, B):
            batch = dev[b0:min(n, b0 + B)]
            masks, _ = amf_frames(batch)
            _, reps = restore_frames(batch, masks)
            its += [r.iterations for r in reps]
        return its

    for _ in range(args.warmup):
        step(64)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            its = step()
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / args.steps
    # the frames with committed reference results (tests/golden/golden_c5.json,
    # frames 0..63 run by the reference) must have taken the same iterations
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_c5.json")))["frames"]
    for i, k in enumerate(its):
        g = gold.get(str(rank * total + i))
        assert g is None or g["iterations"] == k, f"C5 frame {rank * total + i}: {k} iterations"
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([sec], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    # roofline: restore iteration 1 (every flagged pixel active) at the farm's
    # batch scale -- B frames stacked into one grid, the work of one
    # device-side batch of B loops
    sub = dev[:B]
    masks, counts = amf_frames(sub)
    F, H, W = sub.shape
    t1 = _restore_iter1_ms(sk, sub.reshape(F * H, W), masks.reshape(F * H, W))
    # e2e: the reference's pipeline shape over this rank's frames, host uint8
    # frames in (pinned), restored fp64 frames out by one DMA each into
    # recycled pinned host frames handed to the writer (host_buffers=True)
    hin = torch.from_numpy(host).pin_memory()
    frames = [sk.Grid.from_tensor(hin[i]) for i in range(total)]
    seen = []

    def writer(g):
        seen.append(float(g.tensor()[540, 960]))

    # warm: device batches and the pinned result frames reach their steady-state pools
    video_restore_pipeline(frames[:256], width=width, writer=writer, host_buffers=True)
    passes = []
    for _ in range(3):
        seen.clear()
        t0 = time.perf_counter()
        video_restore_pipeline(frames, width=width, writer=writer, host_buffers=True)
        passes.append(time.perf_counter() - t0)
        assert len(seen) == total
    e2e_s = statistics.median(passes)
    line = _base(args, "frames/s (denoise)", "frames/s", total * world / sec, sec * 1e3, "f64",
                 f"C5 video denoise 1000 synthetic 1920x1080 frames, 10% noise "
                 f"(all distinct), device farm batches of {B}",
                 {"mean_iterations": float(np.mean(its)), "pipeline_farm_width": width,
                  "parallelism": f"frames split over {world} GPU(s)"})
    line["n_gpus"] = world
    cpu_line = None
    if rank == 0:
        t0 = time.perf_counter()
        m = O.amf_detect(host[0])
        O.restore_loop(host[0], m)
        cpu_line = {"value": 1.0 / (time.perf_counter() - t0), "unit": "frames/s", "cores": 1,
                    "kind": "port", "sample": "one 1920x1080 frame: oracle AMF + restore loop "
                                              "to convergence, single thread"}
    line.update({
        "gpu_launches": None,
        "e2e": {"value": len(frames) / e2e_s, "unit": "frames/s",
                "passes_frames_per_s": [round(len(frames) / x, 1) for x in passes],
                "h2d_bytes_per_step": len(frames) * 1080 * 1920,
                "d2h_bytes_per_step": len(frames) * 1080 * 1920 * 8,
                "mode": f"median of 3 passes of video_restore_pipeline(width={width}, "
                        f"host_buffers=True) over {len(frames)} pinned host uint8 frames: the "
                        f"ordered farm at batch granularity (2 workers per GPU, batches of "
                        f"{max(1, width // 2)}), fp64 results DMA'd into recycled pinned host "
                        f"frames handed to the writer in stream order"},
        "roofline": restore_roofline(int(counts.sum()), t1, "c5"),
        "cpu_baseline": cpu_line,
        "clocks": clk.summary(),
    })
    # per batch: batched AMF + one persistent restore launch + the
    # flagged-list build (count, scan, scatter, bounds)
    line["gpu_launches"] = args.steps * 6 * (-(-total // B))
    return line
