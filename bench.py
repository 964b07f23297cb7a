"""Benchmark: Mrays/s and FPS of 1080p VOctree HH rendering (BASELINE.json configs[1]).

Workload (config 2): depth-9 spherical-shell VOctree
(3,557,912 leaves, n_max = 2 -> 104 f32 per leaf, 1.48 GB payload), T = 30
frames, 1920x1080 camera look_at((1.6,1.3,0.9) -> (0.5,0.5,0.5)), uncached
render (the fused ray-gen + traversal + HH shading + compositing +
finalize kernel).  One step = one full 1080p frame; steps sweep frames
0..29.  Synthetic data generated in-process (deterministic seeds).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun as batched playback (the north star's "by frame
for batched playback"): every rank holds a full tree replica and renders
frames f = rank, rank + N, ... of the sweep -- one full frame per rank per
step, no data-path collective (weak scaling; the timed region is the max
over ranks).  The single-frame tile path (64x64 tiles interleaved over the
ranks, one NCCL all-gather, unpack) is timed as well and reported under
"tile_frame".  The reference arm (--impl reference) times the reference's own CPU
renderer (voxvid from baseline/_ref, numba, all host threads) or, if that
is not installed, the C oracle port (OpenMP, all host threads).
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mrays/s and FPS at 1080p (VOctree HH render) at 1/2/4/8 B200 vs CPU ref"
UNIT = "Mrays/s"
WIDTH, HEIGHT, FRAMES = 1920, 1080, 30
WORKLOAD = ("cfg2: depth-9 shell VOctree (3,557,912 leaves, n_max 2, T 30), 1920x1080, uncached render "
            "(ray gen + traversal + HH shading + compositing + finalize), frame sweep")
C_COEF, K_HH = 31, 14
L2_BYTES = 126 * 2**20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- helpers
def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def ncu_traffic():
    """DRAM bytes per launch of the render kernel from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "render_camera_ncu.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def make_tree(config: int):
    from paper_2202_06088_b200 import synthetic

    t0 = time.time()
    if config == 3:
        tree = synthetic.motion_tree(depth=9, n_max=2, frames=60, seed=0)
    else:
        tree = synthetic.shell_tree(depth=9, n_max=2, frames=FRAMES, seed=0)
    log(f"[bench] tree: {tree.n_leaves} leaves, {tree.n_internal} internal, "
        f"{tree.leaf_data.nbytes / 1e9:.3f} GB payload, built in {time.time() - t0:.1f}s")
    return tree


def algorithmic_bytes(tree, cam, frames, device):
    """Reference-defined bytes per frame:
    sum_rays 32 P + 4C V + 4(C+3K) S + 20, with P/V/S the internal-node pops,
    visited leaves and shaded leaves of the reference traversal (early stop
    1e-4), counted by the instrumented kernel on host-generated rays (bit-
    exact with the reference's counts)."""
    import torch

    import paper_2202_06088_b200 as vv

    o, d = cam.rays()
    ot = torch.from_numpy(o).to(device)
    dt = torch.from_numpy(d).to(device)
    out = {}
    c = tree.coeff_count
    k = tree.basis_count
    for f in frames:
        _, _, _, st = vv.render_rays(tree, ot, dt, f, stats=True)
        P = st["node_pops"].to(torch.int64).sum().item()
        V = st["sample_count"].to(torch.int64).sum().item()
        S = st["shaded"].to(torch.int64).sum().item()
        n = o.shape[0]
        s_sh = (tree.n_max + 1) ** 2
        out[f] = dict(
            P=P, V=V, S=S,
            # uncached path (render_kernel decoding every visited leaf)
            bytes=32 * P + 4 * c * V + 4 * (c + 3 * k) * S + 20 * n,
            # sliced path actually executed: render kernel reads a node row per
            # pop, the f64 sigma per visited leaf and the 3S fp32 sliced SH
            # coefficients per shaded leaf, writes 20 B per pixel ...
            render_bytes=32 * P + 8 * V + 12 * s_sh * S + 20 * n,
            # ... after the per-frame slice pass read, per leaf, the w_sigma /
            # w_gamma chunks the frame's A / B rows do not zero out (16 B
            # each), w_hh, and wrote sigma + q
            slice_bytes=tree.n_leaves * (16 * (_nz_chunks(tree.bases.a[f], c) + _nz_chunks(tree.bases.b[f], c))
                                         + 12 * k + 8 + 12 * s_sh),
            # the reference's formula (every payload column)
            slice_formula_bytes=tree.n_leaves * (4 * (2 * c + 3 * k) + 8 + 12 * s_sh),
        )
    return out


def _nz_chunks(row, c):
    """float4 chunks (4 columns) of an fp32 basis row holding a nonzero entry."""
    r = np.asarray(row, dtype=np.float32)[:c]
    return int(np.count_nonzero(np.pad(r != 0, (0, -c % 4)).reshape(-1, 4).any(axis=1)))


# --------------------------------------------------------------------------- CPU baselines
def cpu_reference_render(tree, cam, frames, warm=()):
    """Time the reference's own render() (voxvid numba) if installed in baseline/_ref.

    ``warm`` frames are rendered untimed first (the W warm-up steps)."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "voxvid").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", str(ref_dir / ".numba_cache"))
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
    sys.path.insert(0, str(ref_dir))
    import numba
    from voxvid import render as rr
    from voxvid.octree import VOctree as RV
    from voxvid.temporal import TemporalBases as RTB

    rtree = RV(tree.depth, tree.node_child, tree.leaf_coords, tree.leaf_data, RTB(tree.bases.a, tree.bases.b),
               tree.n_max, tree.bbox_lo, tree.side)
    rcam = rr.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w)
    small = rr.Camera(64, 36, cam.fx / 30, cam.fy / 30, 32.0, 18.0, cam.c2w)
    t0 = time.time()
    rr.render(rtree, small, frames[0])  # JIT warm-up
    log(f"[bench] reference JIT warm-up {time.time() - t0:.1f}s, numba threads {numba.get_num_threads()}")
    for f in warm:
        rr.render(rtree, rcam, f)
    times = []
    for f in frames:
        t0 = time.perf_counter()
        rr.render(rtree, rcam, f)
        times.append(time.perf_counter() - t0)
    return dict(times=times, cores=int(numba.get_num_threads()), kind="reference",
                impl="voxvid.render.render (numba, baseline/_ref), uncached")


def cpu_port_render(tree, cam, frames, warm=()):
    """Time the C oracle port (OpenMP, all host threads): ray gen + render_kernel + finalize.

    ``warm`` frames are rendered untimed first (the W warm-up steps)."""
    from oracle import oracle

    nt = oracle.num_procs()
    for f in warm:
        o, d = cam.rays()
        out = oracle.render_rays(tree, o, d, f, nthreads=nt)
        oracle.finalize(out["premult"], out["alpha"], out["tbar"])
    times = []
    for f in frames:
        t0 = time.perf_counter()
        o, d = cam.rays()
        out = oracle.render_rays(tree, o, d, f, nthreads=nt)
        oracle.finalize(out["premult"], out["alpha"], out["tbar"])
        times.append(time.perf_counter() - t0)
    return dict(times=times, cores=nt, kind="port", impl="oracle/vv_oracle.c (OpenMP), uncached")


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    cam_mod = __import__("paper_2202_06088_b200.synthetic", fromlist=["bench_camera"])
    tree = make_tree(args.config)
    cam = cam_mod.bench_camera(WIDTH, HEIGHT)
    warm = [i % FRAMES for i in range(args.warmup)]
    frames = [i % FRAMES for i in range(args.warmup, args.warmup + args.steps)]
    res = cpu_reference_render(tree, cam, frames, warm) if not args.port else None
    if res is None:
        res = cpu_port_render(tree, cam, frames, warm)
    n_rays = WIDTH * HEIGHT
    ms = 1e3 * sum(res["times"]) / len(res["times"])
    value = n_rays * len(res["times"]) / sum(res["times"]) / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "fps": round(1e3 / ms, 4),
        "config": {"workload": WORKLOAD, "rays_per_step": n_rays, "frames": frames,
                   "warmup_frames": warm},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
                         "sample": f"{len(frames)} full 1080p frames {frames}", "impl": res["impl"]},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2202_06088_b200 as vv
    from paper_2202_06088_b200 import synthetic
    from paper_2202_06088_b200.device import replica, stream_ptr
    from paper_2202_06088_b200.distributed import TileRenderer

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    tree = make_tree(args.config)
    cam = synthetic.bench_camera(WIDTH, HEIGHT)
    n_rays = WIDTH * HEIGHT
    t0 = time.time()
    rep = replica(tree, dev)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: upload {time.time() - t0:.2f}s, {rep.device_bytes / 1e9:.3f} GB on device")

    # batched playback: frame f is rendered by rank f mod world (full replica
    # per GPU, frames independent -> no data-path collective, weak scaling)
    frames_total = FRAMES if args.config != 3 else 60
    step_frames = [(args.warmup * world + i * world + rank) % frames_total for i in range(args.steps)]
    warm_frames = [(i * world + rank) % frames_total for i in range(args.warmup)]

    rgb = torch.empty((HEIGHT, WIDTH, 3), dtype=torch.float32, device=dev)
    alpha = torch.empty((HEIGHT, WIDTH), dtype=torch.float32, device=dev)
    depth = torch.empty((HEIGHT, WIDTH), dtype=torch.float32, device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)

    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    cur = {"mid": None}

    def step(f):
        # identical work to render(tree, cam, f): per-frame slice pass, then the
        # fused ray-gen/traversal/shading/finalize kernel -- split here so the
        # dominant kernel's own duration is measured (roofline)
        fs = vv.build_frame_cache(tree, f)
        if cur["mid"] is not None:
            cur["mid"].record(stream)
        vv.render_into(tree, cam, f, rgb, alpha, depth, cache=fs)
        del fs

    for f in warm_frames:
        step(f)
    torch.cuda.synchronize()

    # device-timed region: K steps, L2 flushed between steps (outside the events)
    stream = torch.cuda.current_stream(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local_rank) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    wall0 = time.perf_counter()
    for i, f in enumerate(step_frames):
        flush.zero_()
        starts[i].record(stream)
        cur["mid"] = mids[i]
        step(f)
        ends[i].record(stream)
    cur["mid"] = None
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    render_ms = sum(m.elapsed_time(e) for m, e in zip(mids, ends))
    slice_ms = sum(s.elapsed_time(m) for s, m in zip(starts, mids))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())

    # playback on the device: groups of playback_group(tree) frames of the same
    # camera share one octree walk (render_frames_into; images bitwise equal
    # to render()), every frame with its own slice pass; L2 flushed between
    # groups outside the events
    from paper_2202_06088_b200.render import playback_group

    G = playback_group(tree)

    pb_outs = [(torch.empty((HEIGHT, WIDTH, 3), dtype=torch.float32, device=dev),
                torch.empty((HEIGHT, WIDTH), dtype=torch.float32, device=dev),
                torch.empty((HEIGHT, WIDTH), dtype=torch.float32, device=dev)) for _ in range(G)]
    groups = [step_frames[i:i + G] for i in range(0, len(step_frames) - G + 1, G)] or [step_frames[:G]]
    warm_group = [warm_frames[i % len(warm_frames)] for i in range(G)]  # a full group: loads its kernels
    for gr in [warm_group] * 2:
        vv.render_frames_into(tree, cam, gr, pb_outs[:len(gr)])
    torch.cuda.synchronize()
    gs = [torch.cuda.Event(enable_timing=True) for _ in groups]
    ge = [torch.cuda.Event(enable_timing=True) for _ in groups]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i, gr in enumerate(groups):
        flush.zero_()
        gs[i].record(stream)
        vv.render_frames_into(tree, cam, gr, pb_outs[:len(gr)])
        ge[i].record(stream)
    torch.cuda.synchronize()
    pb_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(gs, ge))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(pb_ms, op=dist.ReduceOp.MAX)
    pb_frames = sum(len(g) for g in groups)
    pb_ms_frame = float(pb_ms.item()) / pb_frames
    playback = {"value": round(world * n_rays / pb_ms_frame / 1e3, 3), "unit": UNIT,
                "ms_per_frame": round(pb_ms_frame, 4), "fps": round(world * 1e3 / pb_ms_frame, 2),
                "frames_per_walk": G, "frames": pb_frames,
                "what": f"groups of {G} frames of the fixed bench camera share one octree walk "
                        "(vv_render_camera_multi); each frame has its own slice pass, accumulators and "
                        "early termination; images bitwise equal to render() per frame"}

    # end-to-end through the public API: every frame complete on the host
    for f in warm_frames[:3]:  # two results alive at once in the loop below: warm both pinned buffers
        layer = vv.render(tree, cam, f)
    torch.cuda.synchronize()
    # single-call latency: render() -> numpy, one frame at a time
    te = time.perf_counter()
    for f in step_frames[:10]:
        layer = vv.render(tree, cam, f)
    single_ms = (time.perf_counter() - te) / len(step_frames[:10]) * 1e3
    assert layer.rgb.shape == (HEIGHT, WIDTH, 3)
    del layer
    # steady-state playback: pinned result pool and render streams warm
    # (a 41 MB cudaHostAlloc costs 25-100 ms; none may land in the timed run)
    for _ in range(2):
        collections.deque(vv.render_sequence(tree, cam, warm_group * 2), maxlen=0)  # full groups; holds no frame
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    got = 0
    for layer in vv.render_sequence(tree, cam, step_frames):  # this rank's frames, to this rank's host
        got += 1
    e2e_s = time.perf_counter() - te
    assert got == len(step_frames) and layer.rgb.shape == (HEIGHT, WIDTH, 3)
    del layer
    if world > 1:
        et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_s = float(et.item())
    e2e = {"value": round(world * n_rays * len(step_frames) / e2e_s / 1e6, 3), "unit": UNIT,
           "h2d_bytes_per_step": (168 + 48) * world, "d2h_bytes_per_step": 5 * 4 * n_rays * world,
           "api": "paper_2202_06088_b200.render_sequence(tree, cam, frames) -> numpy LayerImages (fp32) "
                  "per frame on every rank; frames rendered in groups of 3 sharing one walk (see playback), "
                  "group g rendered while group g-1 copies to pinned host memory",
           "single_render_call_ms": round(single_ms, 3)}

    # single-frame latency across the ranks: 64x64 tiles interleaved over the
    # GPUs, one NCCL all-gather of the packed slabs, unpack on rank 0
    tile_frame = None
    if world > 1:
        tiles = TileRenderer(WIDTH, HEIGHT, 64, rank, world, dev)

        def tile_step(f):
            tiles.render_slab(tree, cam, f)
            tiles.gather()
            if rank == 0:
                tiles.unpack(rgb, alpha, depth)

        for f in warm_frames:
            tile_step(f)
        torch.cuda.synchronize()
        nt = min(10, len(step_frames))
        ts = [torch.cuda.Event(enable_timing=True) for _ in range(nt)]
        tend = [torch.cuda.Event(enable_timing=True) for _ in range(nt)]
        dist.barrier()
        torch.cuda.synchronize()
        for i, f in enumerate(step_frames[:nt]):
            flush.zero_()  # L2 flush outside the per-frame events
            ts[i].record(stream)
            tile_step(f)
            tend[i].record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ts, tend)) / nt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tile_frame = {"ms_per_frame": round(float(tt.item()), 4),
                      "mrays": round(n_rays / float(tt.item()) / 1e3, 3),
                      "parallelism": f"64x64 tiles interleaved over {world} GPUs + NCCL all_gather + unpack",
                      "note": "one frame split across all GPUs (strong scaling); L2 flushed between frames "
                              "outside the per-frame events; the all-gather is inside them"}
        # fused form: every rank stores its tiles straight into rank 0's
        # frame over NVLink (CUDA IPC), one stream-ordered barrier per frame
        p2p = TileRenderer(WIDTH, HEIGHT, 64, rank, world, dev, mode="p2p")
        for f in warm_frames:
            p2p.render_frame(tree, cam, f)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        for i, f in enumerate(step_frames[:nt]):
            flush.zero_()
            ts[i].record(stream)
            p2p.render_frame(tree, cam, f)
            tend[i].record(stream)
        torch.cuda.synchronize()
        tp = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(ts, tend)) / nt], dtype=torch.float64, device=dev)
        dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        dist.barrier()
        p2p.close()
        tile_frame["p2p"] = {"ms_per_frame": round(float(tp.item()), 4),
                             "mrays": round(n_rays / float(tp.item()) / 1e3, 3),
                             "parallelism": f"64x64 tiles interleaved over {world} GPUs, each rank's tile kernel "
                                            "storing into rank 0's frame through CUDA IPC (NVLink/NVSwitch), "
                                            "one all-reduce barrier; no slab, no all-gather, no unpack"}

    if rank != 0:
        return

    # roofline of the dominant kernel (k_render_camera), reference-defined bytes
    ab = algorithmic_bytes(tree, cam, sorted(set(step_frames)), dev)
    bytes_per_step = [ab[f]["bytes"] for f in step_frames]
    peak, peak_kind = measured_peak()
    # per GPU (rank 0's kernels; every rank does the same per-frame work)
    rbytes = sum(ab[f]["render_bytes"] for f in step_frames)
    sbytes = sum(ab[f]["slice_bytes"] for f in step_frames)
    achieved = rbytes / (render_ms / 1e3) / 1e9
    slice_gbs = sbytes / (slice_ms / 1e3) / 1e9
    frame_gbs = (rbytes + sbytes) / (total_ms / 1e3) / 1e9
    uncached_gbs = sum(bytes_per_step) / (total_ms / 1e3) / 1e9
    mean_ab = {k: float(np.mean([ab[f][k] for f in step_frames]) / n_rays) for k in ("P", "V", "S")}

    # CPU baseline: oracle port on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        sample_frames = [step_frames[0]]
        res = cpu_port_render(tree, cam, sample_frames)
        cpu = {"value": round(n_rays * len(res["times"]) / sum(res["times"]) / 1e6, 4), "unit": UNIT,
               "cores": res["cores"], "kind": res["kind"],
               "sample": f"{len(sample_frames)} full 1080p frame(s) {sample_frames}, host ray gen + render + finalize"}

    ms = total_ms / len(step_frames)
    value = world * n_rays * len(step_frames) / (total_ms / 1e3) / 1e6  # whole job
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "fps": round(world * 1e3 / ms, 2),
        "config": {
            "workload": WORKLOAD,
            "rays_per_step": n_rays * world, "frames_rank0": step_frames[:8] + (["..."] if len(step_frames) > 8 else []),
            "l2": "inputs larger than L2 (1.54 GB tree) and L2 flushed between steps (252 MiB memset outside "
                  "the per-step CUDA events)",
            "parallelism": f"frames x {world} GPUs (frame f on rank f mod {world}, full replica each)"
                           if world > 1 else "single",
            "per_ray": mean_ab, "wall_ms_timed_region": round(wall * 1e3, 3),
            "dtype_note": "f64 traversal/sigma/compositing, fp32 HH colour",
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(),
                     "peak_kind": peak_kind, "kernel": "k_render_camera",
                     "kernel_ms": round(render_ms / len(step_frames), 4),
                     "bytes_per_launch": float(np.mean([ab[f]["render_bytes"] for f in step_frames])),
                     "bytes_formula": "sum_rays 32 P + 8 V + 12 S_sh S + 20 (sliced path; P/V/S reference counts)",
                     "slice_pass": {"kernel": "k_build_slice",
                                    "ms": round(slice_ms / len(step_frames), 4),
                                    "achieved": round(slice_gbs, 1) if slice_gbs else None,
                                    "frac": round(slice_gbs / peak, 4) if slice_gbs else None,
                                    "bytes_per_launch": float(np.mean([ab[f]["slice_bytes"] for f in step_frames])),
                                    "bytes_formula": "per leaf 16 B per w_sigma / w_gamma float4 chunk the "
                                                     "frame's A / B row does not zero out + 12 K (w_hh) + 8 + "
                                                     "12 S_sh (record); the reference formula 4(2C + 3K) + 8 + "
                                                     "12 S_sh reads every column",
                                    "reference_formula_bytes": float(ab[step_frames[0]]["slice_formula_bytes"])},
                     "frame_achieved": round(frame_gbs, 1) if frame_gbs else None,
                     "uncached_formula_achieved": round(uncached_gbs, 1) if uncached_gbs else None,
                     "uncached_bytes_per_frame": float(np.mean(bytes_per_step))},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "playback": playback,
        "gpu_launches": len(step_frames) * 2 * world,
        "tile_frame": tile_frame,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--port", action="store_true", help="reference arm: force the C oracle port")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("VV_BENCH_FUNCTIONAL_GLOO"):
            # functional check of the N > 1 code on a box with fewer GPUs:
            # ranks share devices, gloo carries the host-side collectives; the
            # printed numbers are NOT measurements (GPUs are shared)
            local_rank = local_rank % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
