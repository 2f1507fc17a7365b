"""Benchmark: 1080p FPS on the 23M-Gaussian LoD city (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1, one rank per GPU)

Workload (BASELINE.json configs[2]): synthetic 23M-Gaussian MatrixCity-scale
city (extent 1600 m, 3000 buildings), 6x6 blocks, 3 LoD levels built from the
training views (rates 0.5/0.34/0.25, SH 3/2/1, intervals 0/200/400 m), 1080p
flythrough over camera heights {150, 300, 500} m (cmd_bench's orbit sweep,
cli.py:203-218).  One step = one frame: LoD selection + assembly + projection +
depth sort + binning + blend (rasterize_stats after assemble_render_set).
N > 1: the flythrough is view-split across ranks (BASELINE configs[4]), each
rank renders K frames of its own share (weak scaling), no collective on the
data path.  Scene inputs (>= 600 MB per frame) exceed the 126 MB L2, so no
flush is needed between frames.

Keys beyond the base contract: roofline (dominant kernel, live CUDA-event
stage times), cpu_baseline (the C oracle port, all host cores, bounded
sample), e2e (through the C ABI with the image read back to pinned host
memory every frame), stages_ms, clocks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LOD_BUILD = None
# stage marks of cs_render; since K5+K6 were fused (k_bin_pairs + k_emit_heavy) all
# pair emission is timed under "gather_scan" and "duplicate" is an empty slot kept
# so the JSON schema stays comparable across rounds
STAGES = ("select", "project", "depth_sort", "gather_scan", "duplicate", "tile_sort", "ranges", "blend")
SCENES = {
    # name: (gaussians, extent, buildings, blocks, intervals, altitudes, W, H)
    "c3": (23_000_000, 1600.0, 3000, (6, 6), ((0.0, 200.0), (200.0, 400.0), (400.0, math.inf)),
           (150.0, 300.0, 500.0), 1920, 1080),
    "c3-small": (2_000_000, 1600.0, 3000, (6, 6), ((0.0, 200.0), (200.0, 400.0), (400.0, math.inf)),
                 (150.0, 300.0, 500.0), 1920, 1080),
    "tiny": (200_000, 200.0, 100, (2, 2), ((0.0, 40.0), (40.0, 80.0), (80.0, math.inf)),
             (20.0, 40.0, 80.0), 640, 360),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)  # the whole 3-altitude flythrough
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--scene", choices=tuple(SCENES), default="c3")
    ap.add_argument("--frames-per-altitude", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train", action="store_true", help="skip the block-training leg (C4)")
    ap.add_argument("--no-assign", action="store_true", help="skip the data-assignment leg (f2)")
    ap.add_argument("--assign-poses", type=int, default=4)
    ap.add_argument("--no-c5", action="store_true", help="skip the 740-test-view batch render (C5)")
    ap.add_argument("--train-steps", type=int, default=72, help="timed block iterations per rank")
    ap.add_argument("--train-warmup", type=int, default=36)
    ap.add_argument("--train-views", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# scene


def build_scene(name: str, seed: int, dev, keep_raw: bool = False, build_lod: bool = True):
    import torch
    from paper_2404_01133_b200 import lodgen
    from paper_2404_01133_b200.synth import city_cameras, generate_city_torch, orbit_cameras
    n, extent, nb, dims, ints, alts, W, H = SCENES[name]
    t0 = time.perf_counter()
    pos, op, sc, q, sh = generate_city_torch(seed, extent, nb, n, device=dev)
    pmin, pmax = lodgen.central_third(pos)
    mem = lodgen.block_membership(pos, pmin, pmax, dims)
    cams = city_cameras(64, extent, W, H, seed=seed)
    train = [c for i, c in enumerate(cams) if i % 8 != 0]   # every 8th is test (colmap.py:152-156)
    torch.cuda.synchronize()
    t_lod = time.perf_counter()
    scene = lodgen.build_lod_device(pos, op, sc, q, sh, mem, int(np.prod(dims)), train,
                                    distance_intervals=ints) if build_lod else None
    torch.cuda.synchronize()
    global LOD_BUILD
    LOD_BUILD = None if not build_lod else {"s": round(time.perf_counter() - t_lod, 3), "gaussians": int(pos.shape[0]),
                 "views": len(train), "blocks": int(np.prod(dims)),
                 "what": "significance (K15) + priority sort + level rows + MAD bounds + gather "
                         "(lodgen.build_lod_device, build_lod lod.py:211-248), wall clock after sync"}
    lo = pos.double().min(dim=0).values.cpu().numpy()
    hi = pos.double().max(dim=0).values.cpu().numpy()
    center = 0.5 * (lo + hi)
    radius = 0.5 * max(hi[0] - lo[0], hi[1] - lo[1])
    raw = (pos, op, sc, q, sh, mem, int(np.prod(dims))) if keep_raw else None
    del pos, op, sc, q, sh, mem
    torch.cuda.empty_cache()
    return scene, center, radius, alts, (W, H), time.perf_counter() - t0, raw


def _profiler(env: str):
    """cudaProfilerStart now and return the stop callable when `env` is set (for
    ncu --profile-from-start off captures of exactly the timed region); a
    no-op otherwise.  Never set during a measured run."""
    import torch
    if not os.environ.get(env):
        return lambda: None
    torch.cuda.cudart().cudaProfilerStart()
    return lambda: torch.cuda.cudart().cudaProfilerStop()


def flythrough(center, radius, alts, wh, per_alt):
    from paper_2404_01133_b200.synth import orbit_cameras
    cams = []
    for a in alts:
        cams += orbit_cameras(center, radius, a, per_alt, wh[0], wh[1])
    return cams


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = Path(f"/tmp/cs_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [l.split(",") for l in self.path.read_text().splitlines() if l.strip()]
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for name, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        self.path.unlink(missing_ok=True)
        busy = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic work per stage


def stage_bytes(st: dict) -> dict:
    """Algorithmic HBM bytes of each stage summed over the measured frames
    (every array read or written once per pass)."""
    na, m, p = st["assembled"], st["visible"], st["pairs"]
    return {
        # per assembled: 3 fp32 quads (48 B) + depth keys (8 + 4) + id (4);
        # per visible: its SH row (level width) + HotRec 64 + rect 8 + cull box 8
        "project": na * (48 + 16) + st["sh_bytes_visible"] + m * (64 + 8 + 8),
        # 4 LSD passes over (u32 key, u32 id) + one histogram read + run check
        "depth_sort": na * 4 + 4 * 2 * na * 8 + m * 4,
        # fused K5+K6: per visible id + rect gather (8); per pair (tile, id) written
        "gather_scan": m * (4 + 8) + p * 8,
        # (folded into gather_scan: the stage boundary remains, ~0 ms)
        "duplicate": 0,
        # 2 LSD passes over (u32 tile, u32 id) + one histogram read
        "tile_sort": p * 4 + 2 * 2 * p * 8,
        # per pair: key + id read, cull box gathered (8) and written pair-major (8)
        "ranges": p * (4 + 4 + 8 + 8),
    }


def blend_flops(st: dict) -> float:
    """Algorithmic float64 flops of the blend: per
    evaluated (pixel, splat) the quadratic form (2 sub + 7 mul + 2 add = 11);
    per accepted fragment exp (3 mul/add + 9 FMA = 21) and alpha/T/colour
    (4 mul/add + 3 FMA = 10)."""
    return 11.0 * st["evals"] + 31.0 * st["fragments"]


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/*_frame_traffic.json, newest), or None."""
    # capture tags run r1a .. r1z, r1aa ..: newest = longest, then greatest
    tag = lambda f: f.name[: -len("_frame_traffic.json")]
    files = sorted((ROOT / "profiles").glob("*_frame_traffic.json"), key=lambda f: (len(tag(f)), tag(f)))
    if not files:
        return None, None
    data = json.loads(files[-1].read_text())
    hits = [v for k, v in data.items() if k.startswith(kernel)]
    if not hits:
        return None, files[-1].name
    launches = [x for lst in hits for x in lst]
    return sum(x["dram_bytes"] for x in launches) / len(launches), files[-1].name


def ncu_pipes(kernel: str):
    """Issue-slot / FP64 / FMA pipe / shared-memory utilisation of `kernel` from
    the same committed capture (percent), or None."""
    tag = lambda f: f.name[: -len("_frame_traffic.json")]
    files = sorted((ROOT / "profiles").glob("*_frame_traffic.json"), key=lambda f: (len(tag(f)), tag(f)))
    if not files:
        return None
    data = json.loads(files[-1].read_text())
    hits = [x for k, v in data.items() if k.startswith(kernel) for x in v]
    keys = ("issue_active_pct", "fp64_pipe_pct", "fma_pipe_pct", "smem_pct", "threads_per_inst")
    if not hits or any(k not in hits[0] for k in keys):
        return None
    return {k: round(sum(x[k] or 0.0 for x in hits) / len(hits), 1) for k in keys}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    import torch.distributed as dist
    # CS_BENCH_SHARED_GPU=1 (testing only): every rank on the visible GPU(s) modulo
    # their count, with gloo carrying the collectives -- exercises the N > 1
    # code path (view split, LoD broadcast, LPT training, fusion all-gather) on
    # a one-GPU box.  Never set for a measured run.
    shared = os.environ.get("CS_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import ctypes

    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200._lib import CsFrameStats, CsSource

    # N > 1: rank 0 runs the LoD build, the levels and table reach the other
    # ranks by NCCL broadcast (fusion.broadcast_device_lod_scene)
    scene, center, radius, alts, wh, build_s, raw = build_scene(args.scene, args.seed, dev,
                                                                keep_raw=not (args.no_train and args.no_assign),
                                                                build_lod=(rank == 0))
    lod_bcast_ms = None
    if world > 1:
        from paper_2404_01133_b200 import fusion
        torch.cuda.synchronize()
        dist.barrier()
        tb = time.perf_counter()
        scene = fusion.broadcast_device_lod_scene(scene if rank == 0 else None, src=0)
        torch.cuda.synchronize()
        lod_bcast_ms = 1000.0 * (time.perf_counter() - tb)
    cams_all = flythrough(center, radius, alts, wh, args.frames_per_altitude)
    # view split: rank r renders its contiguous share of the flythrough, cycling
    share = [cams_all[i] for i in range(len(cams_all)) if i * world // len(cams_all) == rank] or cams_all
    settings = cs.RenderSettings()
    lib = _lib.load()
    ctx = device.context(local)
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    src = CsSource()
    src.kind = _lib.CS_SRC_LOD_BLOCK
    src.force_level = -1
    src.lod = scene.handle
    cset = device.settings_struct(settings)
    W, H = wh
    out = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    ccams = [device.camera_struct(c) for c in share]

    def frame(i, flags=0, stats=None):
        rc = lib.cs_render(ctx, ctypes.byref(src), ctypes.byref(ccams[i % len(ccams)]), ctypes.byref(cset),
                           out.data_ptr(), flags, ctypes.byref(stats) if stats is not None else None, sh)
        _lib.check(rc, "cs_render")

    # sizing pass (synchronous, grows pair buffers) + per-frame counts for the roofline
    K = args.steps
    counts = dict(assembled=0, visible=0, pairs=0, evals=0, fragments=0, sh_bytes_visible=0, warp_hits=0,
                  warp_hits_empty=0)
    for i in range(min(len(ccams), max(K, 1))):
        s = CsFrameStats()
        frame(i, _lib.CS_RENDER_SYNC, s)
    from paper_2404_01133_b200.device import sh_stride
    row_bytes = [4 * sh_stride(lc.sh_coeffs) for lc in scene.level_clouds]
    seg_idx = (ctypes.c_int32 * 4096)()
    seg_cnt = (ctypes.c_int64 * 4096)()
    n_seg = ctypes.c_int32(0)
    blend_item_max = []  # longest blend work item per frame, SM clocks (DIAG)
    blend_item_sum = []  # sum over the frame's blend work items
    for i in range(K):
        s = CsFrameStats()
        frame(i, _lib.CS_RENDER_SYNC | _lib.CS_RENDER_DIAG, s)
        counts["assembled"] += s.assembled
        counts["visible"] += s.visible
        counts["pairs"] += s.pairs
        counts["evals"] += s.evals
        counts["fragments"] += s.fragments
        counts["warp_hits"] += s.warp_hits
        counts["warp_hits_empty"] += s.warp_hits_empty
        blend_item_max.append(s.blend_max_item_cycles)
        blend_item_sum.append(s.blend_item_cycles)
        # SH rows are read for visible splats; their width depends on the level
        # (C = 16/9/4 -> 192/112/48 B): weight by this frame's assembled level mix
        _lib.check(lib.cs_dump_segments(ctx, seg_idx, seg_cnt, 4096, ctypes.byref(n_seg), sh))
        sh_assembled = sum(seg_cnt[q] * row_bytes[seg_idx[q] // scene.n_blocks] for q in range(n_seg.value))
        counts["sh_bytes_visible"] += sh_assembled * (s.visible / max(s.assembled, 1))
    for i in range(args.warmup):
        frame(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        prof = _profiler("CS_PROFILE_FRAMES")  # ncu --profile-from-start off: the timed frames only
        for i in range(K):
            frame(i)
        e1.record(stream)
        torch.cuda.synchronize()
        prof()
    ms = e0.elapsed_time(e1)
    # per-stage breakdown from a second, untimed pass with CUDA-event marks
    # between the stages (the timed frames above run as replayed frame graphs,
    # cs_render's asynchronous fast path; marked frames take the direct path)
    lib.cs_timing_begin(ctx, K)
    for i in range(K):
        frame(i)
    torch.cuda.synchronize()
    stage = (ctypes.c_double * 8)()
    nfr = ctypes.c_int32(0)
    _lib.check(lib.cs_timing_end(ctx, stage, ctypes.byref(nfr)))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(t.item())
    stages_ms = {k: stage[i] / max(nfr.value, 1) for i, k in enumerate(STAGES)}

    # e2e: same frames through the C ABI, image copied to pinned host memory each frame
    e2e = None
    if not args.no_e2e:
        host = [torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        outs = [out, torch.empty_like(out)]
        copy_stream = torch.cuda.Stream(dev)
        done = [torch.cuda.Event(), torch.cuda.Event()]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(K):
            b = i & 1
            done[b].synchronize()  # host buffer b free again
            rc = lib.cs_render(ctx, ctypes.byref(src), ctypes.byref(ccams[i % len(ccams)]),
                               ctypes.byref(cset), outs[b].data_ptr(), 0, None, sh)
            _lib.check(rc)
            ready = torch.cuda.Event()
            ready.record(stream)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ready)
                host[b].copy_(outs[b], non_blocking=True)
                done[b].record(copy_stream)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": world * K / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": ctypes.sizeof(_lib.CsCamera) + ctypes.sizeof(_lib.CsSettings),
               "d2h_bytes_per_step": H * W * 3 * 4,
               "path": "cs_render (C ABI) + D2H of the float32 image into pinned host memory"}

    clocks = clk.summary()
    value = world * K / (ms_max / 1000.0)
    # roofline of the dominant kernel (+ every HBM-bound stage)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6450.0)
    bytes_ = stage_bytes(counts)
    dom = max(STAGES, key=lambda k: stages_ms[k])
    stage_roof = {k: {"bytes_per_frame": v / K, "ms": stages_ms[k],
                      "achieved_gbs": (v / K) / (stages_ms[k] / 1000.0) / 1e9 if stages_ms[k] else None}
                  for k, v in bytes_.items()}
    for v in stage_roof.values():
        v["frac"] = v["achieved_gbs"] / hbm_peak if v["achieved_gbs"] else None
    if dom in bytes_:
        achieved = stage_roof[dom]["achieved_gbs"]
        traffic, tsrc = ncu_traffic({"project": "k_project", "depth_sort": "k_onesweep",
                                     "tile_sort": "k_onesweep", "duplicate": "k_bin_pairs",
                                     "gather_scan": "k_bin_pairs", "ranges": "k_tile_ranges"}[dom])
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "B200_PROFILING.md fallback"}
    else:  # blend: float64-pipe bound (quadratic form per evaluation, exp + alpha/T per fragment)
        # measured on this box: DFMA chains on every SM (cs_measure_fp64_peak)
        pk = ctypes.c_double(0.0)
        _lib.check(lib.cs_measure_fp64_peak(ctx, ctypes.byref(pk), sh), "cs_measure_fp64_peak")
        fp64_peak = pk.value
        achieved = blend_flops(counts) / K / (stages_ms[dom] / 1000.0) / 1e12
        traffic, tsrc = ncu_traffic("k_blend")
        roof = {"kernel": "k_blend", "bound": "fp64", "achieved": achieved, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic,
                "peak_source": "measured in this run: dense DFMA chains on every SM, CUDA events "
                               "(cs_measure_fp64_peak; MEASURED_PEAKS.json has no FP64 entry)",
                "flops_per_frame": blend_flops(counts) / K}
    roof["traffic_source"] = f"profiles/{tsrc} (ncu --set full, dram__bytes_read+write per launch)" if tsrc else None
    # the blend is issue-bound (divergent per-pixel termination), not FP64-pipe-bound:
    # the ncu pipe utilisations of the same capture explain the flop fraction
    roof["ncu_pipes_pct"] = ncu_pipes("k_blend")
    roof["stages_hbm"] = stage_roof

    # C5: batch render of the 740 test views of a 5920-camera set (every 8th,
    # colmap.py:152-156) on the same LoD scene, view-split across ranks
    c5 = None
    if not args.no_c5:
        from paper_2404_01133_b200.synth import city_cameras
        all5 = city_cameras(5920, SCENES[args.scene][1], wh[0], wh[1], seed=args.seed)
        test5 = [c for i, c in enumerate(all5) if i % 8 == 0]
        mine = [test5[i] for i in range(len(test5)) if i * world // len(test5) == rank]
        c5cams = [device.camera_struct(c) for c in mine]

        def frame5(c, flags=0):
            _lib.check(lib.cs_render(ctx, ctypes.byref(src), ctypes.byref(c), ctypes.byref(cset),
                                     out.data_ptr(), flags, None, sh), "cs_render")

        vis5, pairs5 = [], []
        for c in c5cams:  # sizing pass (synchronous: pair buffers grow to the largest view)
            s5 = CsFrameStats()
            _lib.check(lib.cs_render(ctx, ctypes.byref(src), ctypes.byref(c), ctypes.byref(cset),
                                     out.data_ptr(), _lib.CS_RENDER_SYNC, ctypes.byref(s5), sh),
                       "cs_render")
            vis5.append(s5.visible)
            pairs5.append(s5.pairs)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for c in c5cams:
            frame5(c)
        f1.record(stream)
        torch.cuda.synchronize()
        t5 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        # untimed second pass with the per-stage event marks
        lib.cs_timing_begin(ctx, len(c5cams))
        for c in c5cams:
            frame5(c)
        torch.cuda.synchronize()
        st5 = (ctypes.c_double * 8)()
        n5 = ctypes.c_int32(0)
        _lib.check(lib.cs_timing_end(ctx, st5, ctypes.byref(n5)))
        c5 = {"metric": "C5 batch render FPS (740 test views, 1080p, LoD, view-split)",
              "value": len(test5) / (float(t5.item()) / 1000.0), "unit": "frames/s",
              "views": len(test5), "views_this_rank": len(mine), "n_gpus": world,
              "ms_max_rank": float(t5.item()), "scaling": "weak in views per rank" if world > 1 else "n/a",
              "visible_M_min_med_max": [round(float(x) / 1e6, 3) for x in
                                        (min(vis5), float(np.median(vis5)), max(vis5))] if vis5 else None,
              "pairs_M_min_med_max": [round(float(x) / 1e6, 3) for x in
                                      (min(pairs5), float(np.median(pairs5)), max(pairs5))] if pairs5 else None,
              "stages_ms": {k: round(st5[i] / max(n5.value, 1), 4) for i, k in enumerate(STAGES)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(scene, cams_all, settings, n_frames=1)

    assign = None
    if raw is not None and not args.no_assign and rank == 0:
        del scene
        scene = None
        torch.cuda.empty_cache()
        assign = assign_leg(args, raw, wh, dev)
    train = None
    if not args.no_train:
        scene = None
        torch.cuda.empty_cache()
        train = train_leg(args, raw, wh, rank, world, dev)
        raw = None

    if rank == 0:
        line = {
            "metric": "1080p FPS on 23M-Gaussian LoD city" if args.scene == "c3" else f"FPS ({args.scene})",
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_city_torch, reference distributions), random-init scene",
            "config": {"workload": f"{args.scene}: {SCENES[args.scene][0]} Gaussians, "
                                   f"{SCENES[args.scene][3][0]}x{SCENES[args.scene][3][1]} blocks, 3 LoD levels, "
                                   f"{wh[0]}x{wh[1]} flythrough at {list(alts)} m",
                       "frames_in_flythrough": len(cams_all), "view_split": world > 1,
                       "l2": "per-frame inputs (>600 MB) exceed L2; no flush",
                       "scene_build_s": round(build_s, 1)},
            "stages_ms": stages_ms,
            "counts_per_frame": {k: v / K for k, v in counts.items()},
            "blend_longest_item_us": (round(float(np.median(blend_item_max)) / ((clocks or {}).get("sm_mhz") or 1965.0), 1)
                                      if blend_item_max else None),
            "blend_item_us_sum_per_warp_slot": (round(float(np.median(blend_item_sum)) / ((clocks or {}).get("sm_mhz") or 1965.0)
                                                      / lib_blend_slots(), 1) if blend_item_sum else None),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "train": train,
            "lod_build": LOD_BUILD,
            "c5": c5,
            "lod_broadcast_ms": lod_bcast_ms,
            "assign": assign,
            "gpu_launches": K * launches_per_frame(),
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def assign_leg(args, raw, wh, dev):
    """f2: training-data assignment contribution tests (assign_b1, partition.py:318-334)
    on the full 23M-Gaussian cloud: per (pose, block) one masked render at the
    assignment scale (0.25) + SSIM, as partition.assign runs them."""
    import torch
    from paper_2404_01133_b200 import device, partition
    from paper_2404_01133_b200.synth import city_cameras
    pos, op, sc, q, sh, mem, n_blocks = raw
    full = device.DeviceCloud.from_torch(pos, op, sc, q, sh)
    extent = SCENES[args.scene][1]
    cams = city_cameras(64, extent, wh[0], wh[1], seed=args.seed)
    poses = [c for i, c in enumerate(cams) if i % 8 != 0][:: max(1, 56 // max(args.assign_poses, 1))]
    poses = poses[:args.assign_poses]
    scaled = [partition._scaled_camera(c, 0.25) for c in poses]
    r = partition._Renderer(full, None)
    counts = torch.bincount(mem.long(), minlength=n_blocks).cpu().numpy()
    blocks = [j for j in range(n_blocks) if counts[j] > 0]
    masks = {j: (mem == j).to(torch.uint8) for j in blocks}
    acc = torch.zeros((len(poses), n_blocks, 4), dtype=torch.float64, device=dev)
    fulls = [r(c) for c in scaled]  # warm-up + the full images
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, c in enumerate(scaled):
        for j in blocks:
            partition._ssim_into(fulls[i], r(c, masks[j]), acc[i, j])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    l = 1.0 - acc[:, blocks, 3].cpu().numpy()
    del full, masks, fulls
    torch.cuda.empty_cache()
    n = len(poses) * len(blocks)
    return {"metric": "assign_b1 contribution tests/s (f2)", "value": n / dt, "unit": "tests/s",
            "tests": n, "s": round(dt, 3), "poses": len(poses), "blocks": len(blocks),
            "resolution": f"{scaled[0].width}x{scaled[0].height}", "gaussians": int(pos.shape[0]),
            "l_ssim_min_med_max": [float(l.min()), float(np.median(l)), float(l.max())],
            "what": "masked cs_render (exclude = block j) + cs_ssim per (pose, block), synchronous "
                    "renders as partition.assign issues them; wall clock after sync"}


def train_leg(args, raw, wh, rank, world, dev):
    """C4: block-parallel training iterations/s (+ the NCCL fusion all-gather).

    Every rank builds the same scene, takes its LPT share of the 36 blocks and
    runs them round-robin; one step = one block iteration (fwd + loss + bwd +
    Adam on one 1080p view).  value = all ranks' iterations / max rank time.
    """
    import torch
    import torch.distributed as dist
    from paper_2404_01133_b200 import blocktrain, fusion
    from paper_2404_01133_b200.lodgen import central_third
    pos, op, sc, q, sh, mem, n_blocks = raw
    counts = blocktrain.block_counts(mem, n_blocks)
    owner = blocktrain.assign_blocks(mem, n_blocks, world)
    owned = [j for j in range(n_blocks) if owner[j] == rank and counts[j] > 0]
    t0 = time.perf_counter()
    jobs = blocktrain.setup_blocks(pos, op, sc, q, sh, mem, owned, wh[0], wh[1],
                                   n_views=args.train_views, seed=args.seed)
    pmin, pmax = central_third(pos)
    dims = SCENES[args.scene][3]
    del pos, op, sc, q, sh
    torch.cuda.empty_cache()
    setup_s = time.perf_counter() - t0
    order = [jobs[j] for j in owned if j in jobs]
    stream = torch.cuda.current_stream(dev)
    per_block = {jb.j: [] for jb in order}
    for i in range(args.train_warmup):
        jb = order[i % len(order)]
        per_block[jb.j].append(jb.step().clone())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = args.train_steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    losses = []
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    prof = _profiler("CS_PROFILE_TRAIN")
    for i in range(K):
        job = order[i % len(order)]
        v = job.iters % len(job.cams)
        job.iters += 1
        losses.append(job.trainer.step(job.cams[v], job.targets[v], events=ev[i]).clone())
        per_block[job.j].append(losses[-1])
    e1.record(stream)
    torch.cuda.synchronize()
    prof()
    ms = e0.elapsed_time(e1)
    phases = {"forward": 0.0, "loss": 0.0, "backward": 0.0, "adam": 0.0}
    for e in ev:
        for k, (a, b) in zip(phases, ((0, 1), (1, 2), (2, 3), (3, 4))):
            phases[k] += e[a].elapsed_time(e[b]) / K
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # fusion: every rank filters its blocks; NCCL all-gather-v in block order
    local = {j: jb.fusion_inputs() for j, jb in jobs.items()}
    fuse_ms = None
    fused_n = None
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        f0 = time.perf_counter()
        fused = fusion.fuse_all_gather(local, n_blocks, owner, pmin, pmax, dims, sh_coeffs=16)
        torch.cuda.synchronize()
        fuse_ms = 1000 * (time.perf_counter() - f0)
        fused_n = int(fused.shape[0])
    sizes = [jobs[j].count for j in jobs]
    return {
        "metric": "block-train iters/s (C4)", "value": world * K / (ms_max / 1000.0), "unit": "iters/s",
        "ms_per_iter": ms_max / K, "steps": K, "warmup": args.train_warmup, "n_gpus": world,
        "scaling": "weak", "phases_ms": phases,
        # mean over blocks of each block's first / last training loss (same view cycle)
        "loss_first_last_mean": [float(np.mean([float(v[0]) for v in per_block.values() if v])),
                                 float(np.mean([float(v[-1]) for v in per_block.values() if v]))],
        "iters_per_block": float(np.mean([len(v) for v in per_block.values()])),
        "config": {"workload": f"{n_blocks} blocks of the {args.scene} scene (LPT over ranks), "
                               f"{args.train_views} orbit views/block at {wh[0]}x{wh[1]}",
                   "blocks_this_rank": len(order),
                   "gaussians_per_block_min_med_max": [min(sizes), int(np.median(sizes)), max(sizes)]
                   if sizes else None,
                   "setup_s": round(setup_s, 1)},
        "fusion_all_gather_ms": fuse_ms, "fused_gaussians": fused_n,
    }


def lib_blend_slots() -> int:
    """Resident blend warps on the GPU (148 SMs x CTAs/SM x 8 warps)."""
    import torch
    return torch.cuda.get_device_properties(0).multi_processor_count * 3 * 8


def launches_per_frame() -> int:
    """Kernels of one C3 frame (memsets excluded), as listed by the ncu launch
    capture: k_lod_select, k_project, depth sort [k_radix_hist,
    k_radix_hist_scan, 4 x k_onesweep], k_fix_short_runs, k_fix_long_runs,
    (fused) k_bin_pairs (also counts the tile-sort digits), k_emit_heavy
    (pairs of chunks above kBinHeavy), tile sort [k_radix_hist_scan,
    2 x k_onesweep], k_tile_ranges, k_tile_order, k_blend."""
    return 1 + 1 + (1 + 1 + 4) + 2 + 2 + (1 + 2) + 1 + 1 + 1


def host_scene(scene):
    """Materialise the device LoD scene as float32 host arrays for the oracle."""
    from types import SimpleNamespace
    levels = []
    for L in range(scene.n_levels):
        lc = scene.level_clouds[L]
        pos_op = lc.pos_op.float().cpu().numpy()
        scl = lc.scale.float().cpu().numpy()
        quat = lc.quat.float().cpu().numpy()
        C = lc.sh_coeffs
        sh = lc.sh[:, :3 * C].cpu().numpy().reshape(-1, 3, C)
        blocks = []
        for j in range(scene.n_blocks):
            o = int(scene.block_offsets[L][j])
            n = int(scene.counts[L, j])
            blocks.append(SimpleNamespace(positions=pos_op[o:o + n, :3], opacities=pos_op[o:o + n, 3],
                                          scales=scl[o:o + n, :3], rotations=quat[o:o + n], sh=sh[o:o + n],
                                          count=n))
        levels.append(tuple(blocks))
    return SimpleNamespace(levels=tuple(levels), bounds_min=scene.bounds_min, bounds_max=scene.bounds_max,
                           distance_intervals=scene.distance_intervals)


def cpu_baseline(scene, cams, settings, n_frames=1):
    """The C oracle port (oracle/), all host threads, on a bounded sample."""
    from oracle import oracle as O
    hs = host_scene(scene)
    pick = [cams[len(cams) // 2 + i] for i in range(n_frames)]   # 300 m altitude frames
    O.lib()
    t0 = time.perf_counter()
    outs = []
    for cam in pick:
        cloud, _ = O.assemble(hs, cam)
        outs.append(O.rasterize_frame_c(cloud, cam, settings, nthreads=os.cpu_count() or 1))
    dt = time.perf_counter() - t0
    # full-size parity of the same frame(s) (checker only, outside every timed region):
    # the compatibility tier (assemble_render_set + rasterize_stats) vs the oracle
    import paper_2404_01133_b200 as cs
    parity = []
    for cam, (ref_img, ref_st) in zip(pick, outs):
        a = cs.assemble_render_set(scene, cam)
        img, st = cs.rasterize_stats(a.cloud, cam, settings)
        parity.append({"visible": [st.visible_splats, ref_st["visible_splats"]],
                       "fragments": [st.blended_fragments, ref_st["blended_fragments"]],
                       "image_max_abs_err": float(np.abs(img.pixels - ref_img).max())})
    return {"value": n_frames / dt, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{n_frames} frame(s) of the 300 m orbit (assemble + project + sort + bin + blend)",
            "parity": {"frames": parity, "bar": "visible and fragment counts equal, image max-abs <= 1e-4",
                       "ok": all(q["visible"][0] == q["visible"][1] and q["fragments"][0] == q["fragments"][1]
                                 and q["image_max_abs_err"] <= 1e-4 for q in parity)}}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores (the C oracle
    port, oracle/; the reference package itself is Python and does not travel)."""
    if rank != 0:
        return 0
    import torch
    torch.cuda.set_device(0)
    import paper_2404_01133_b200 as cs
    scene, center, radius, alts, wh, build_s, _ = build_scene(args.scene, args.seed, torch.device("cuda", 0))
    cams = flythrough(center, radius, alts, wh, args.frames_per_altitude)
    from oracle import oracle as O
    hs = host_scene(scene)
    settings = cs.RenderSettings()
    nthreads = os.cpu_count() or 1
    steps = max(1, min(args.steps, 4))
    warm = min(args.warmup, 1)
    for i in range(warm):
        cloud, _ = O.assemble(hs, cams[i])
        O.rasterize_frame_c(cloud, cams[i], settings, nthreads=nthreads)
    t0 = time.perf_counter()
    for i in range(steps):
        cam = cams[(i * len(cams)) // steps]
        cloud, _ = O.assemble(hs, cam)
        O.rasterize_frame_c(cloud, cam, settings, nthreads=nthreads)
    dt = time.perf_counter() - t0
    v = steps / dt
    print(json.dumps({
        "impl": "reference", "metric": "1080p FPS on 23M-Gaussian LoD city", "value": v,
        "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": 1000 * dt / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.scene} flythrough, {steps} frames spread over "
                                                    f"altitudes {list(alts)} m"},
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": nthreads, "kind": "port",
                         "sample": f"{steps} of {len(cams)} flythrough frames (requested steps={args.steps})"},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
