"""Benchmark: 1080p FPS on the 23M-Gaussian LoD city (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1, one rank per GPU)

Workload (BASELINE.json configs[2], C3): synthetic 23M-Gaussian
MatrixCity-scale city (extent 1600 m, 3000 buildings; generated on the HOST
with a seeded CPU torch generator, so both arms render identical inputs), 6x6
blocks, 3 LoD levels built from the training views (rates 0.5/0.34/0.25, SH
3/2/1, intervals 0/200/400 m), 1080p flythrough over camera heights
{150, 300, 500} m, 20 frames per altitude (cmd_bench's orbit sweep,
cli.py:203-218).  One step = one frame: LoD selection + assembly +
projection + depth sort + binning + blend.  The K timed frames are strided
over the whole 60-frame flythrough (frame (i * 60) // K, ``timed_frames``),
so every altitude is in the headline.  N > 1: the flythrough is view-split
across ranks (BASELINE configs[4]), each rank renders the strided frames of
its own share (weak scaling), no collective on the data path.  Scene inputs
(>= 600 MB per frame) exceed the 126 MB L2, so no flush is needed between
frames.

cmd_bench's protocol (cli.py:236-294) rides along as ``altitudes``: per
altitude and mode (lod / finest / full = no LoD) the mean FPS (1000 n / sum
ms) and min FPS (1000 / max ms) over all 20 frames, each frame timed with
CUDA events.  Extra legs: C1 and C2 lines (BASELINE configs[0], [1]) with
their own roofline and CPU baseline, C5 (740 test views), C4 block training
with per-phase rooflines, LoD build, data assignment.

--impl reference (the reference arm): the reference algorithm on the box's
host cores -- the scene is generated on the host by the same seeded
generator, its detail levels built by the C/numpy restatement of build_lod
(oracle.build_lod), and the SAME strided frames rendered by the oracle
(assemble + project + sort + bin + blend, all host threads).  It never loads
libcsgpu.so.  Both arms print the same ``config`` (incl. a SHA-256 of the
levels' positions, counts and bounds) so the configurations can be compared.
"""

from __future__ import annotations

import argparse
import hashlib
import importlib
import json
import math
import os
import statistics
import subprocess
import sys
import time
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PKG = "paper_2404_01133_b200"
LOD_BUILD = None
# stage marks of cs_render; since K5+K6 were fused (k_bin_pairs + k_emit_heavy) all
# pair emission is timed under "gather_scan" and "duplicate" is an empty slot kept
# so the JSON schema stays comparable across rounds
STAGES = ("select", "project", "depth_sort", "gather_scan", "duplicate", "tile_sort", "ranges", "blend")
INF = math.inf
SCENES = {
    # name: (gaussians, extent, buildings, blocks, intervals, altitudes, W, H)
    "c3": (23_000_000, 1600.0, 3000, (6, 6), ((0.0, 200.0), (200.0, 400.0), (400.0, INF)),
           (150.0, 300.0, 500.0), 1920, 1080),
    "c3-small": (2_000_000, 1600.0, 3000, (6, 6), ((0.0, 200.0), (200.0, 400.0), (400.0, INF)),
                 (150.0, 300.0, 500.0), 1920, 1080),
    "tiny": (200_000, 200.0, 100, (2, 2), ((0.0, 40.0), (40.0, 80.0), (80.0, INF)),
             (20.0, 40.0, 80.0), 640, 360),
}
FRAMES_PER_ALT = 20
RATES = (0.5, 0.34, 0.25)      # config.py:103, finest first
SH_DEGREES = (3, 2, 1)         # config.py:105, finest first
N_MAD = 4.0                    # config.py:104


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)  # the whole 3-altitude flythrough
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--scene", choices=tuple(SCENES), default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-modes", action="store_true", help="skip cmd_bench's per-altitude lod/finest/full pass")
    ap.add_argument("--no-train", action="store_true", help="skip the block-training leg (C4)")
    ap.add_argument("--no-assign", action="store_true", help="skip the data-assignment leg (f2)")
    ap.add_argument("--no-c12", action="store_true", help="skip the C1 / C2 lines")
    ap.add_argument("--assign-poses", type=int, default=4)
    ap.add_argument("--no-c5", action="store_true", help="skip the 740-test-view batch render (C5)")
    ap.add_argument("--train-steps", type=int, default=72, help="timed block iterations per rank")
    ap.add_argument("--train-warmup", type=int, default=36)
    ap.add_argument("--train-views", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


def timed_frames(n_frames: int, k: int):
    """The K timed frames, strided over the whole flythrough (every altitude)."""
    return [(i * n_frames) // k for i in range(k)]


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# scene (identical inputs for both arms)


def host_modules():
    """paper_2404_01133_b200.synth (and .core) WITHOUT the package __init__,
    which loads libcsgpu.so: the reference arm uses the same host generator
    but must not load the CUDA library.  In the GPU arm the real package is
    imported first and this simply returns its synth module."""
    if PKG not in sys.modules:
        stub = types.ModuleType(PKG)
        stub.__path__ = [str(ROOT / PKG)]
        sys.modules[PKG] = stub
    return importlib.import_module(PKG + ".synth")


def generate_host(name: str, seed: int):
    """The scene's Gaussians as float32 CPU torch tensors (seeded CPU generator)."""
    n, extent, nb = SCENES[name][:3]
    return host_modules().generate_city_torch(seed, extent, nb, n, device="cpu")


def train_cameras(name: str, seed: int):
    synth = host_modules()
    extent, W, H = SCENES[name][1], SCENES[name][6], SCENES[name][7]
    cams = synth.city_cameras(64, extent, W, H, seed=seed)
    return [c for i, c in enumerate(cams) if i % 8 != 0]   # every 8th is test (colmap.py:152-156)


def flythrough_of(pos_min, pos_max, name: str):
    synth = host_modules()
    alts, W, H = SCENES[name][5], SCENES[name][6], SCENES[name][7]
    center = 0.5 * (pos_min + pos_max)
    radius = 0.5 * max(pos_max[0] - pos_min[0], pos_max[1] - pos_min[1])
    cams = []
    for a in alts:
        cams += synth.orbit_cameras(center, radius, a, FRAMES_PER_ALT, W, H)
    return cams


def flythrough(center, radius, alts, wh, per_alt):
    from paper_2404_01133_b200.synth import orbit_cameras
    cams = []
    for a in alts:
        cams += orbit_cameras(center, radius, a, per_alt, wh[0], wh[1])
    return cams


def fingerprint(level_positions, counts, bmin, bmax) -> str:
    """SHA-256 (16 hex) of the detail levels: per level the float32 positions in
    assembled (block) order, then the (level, block) counts and the bounds."""
    h = hashlib.sha256()
    for p in level_positions:
        h.update(np.ascontiguousarray(p, dtype=np.float32).tobytes())
    h.update(np.ascontiguousarray(counts, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(bmin, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(bmax, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def run_config(name: str, K: int, cams_all, sha: str) -> dict:
    """The config object both arms print (must be identical between them)."""
    n, extent, nb, dims, ints, alts, W, H = SCENES[name]
    return {"workload": f"{name}: {n} Gaussians, {dims[0]}x{dims[1]} blocks, 3 LoD levels, "
                        f"{W}x{H} orbit flythrough at {list(alts)} m ({FRAMES_PER_ALT} frames each)",
            "timed_frames": timed_frames(len(cams_all), K), "frames_in_flythrough": len(cams_all),
            "scene_sha256": sha, "l2": "per-frame inputs (>600 MB) exceed L2; no flush"}


def build_scene(name: str, seed: int, dev, keep_raw: bool = True, build_lod: bool = True):
    """GPU arm: host generation -> HBM, membership + LoD build on the device."""
    import torch
    from paper_2404_01133_b200 import lodgen
    n, extent, nb, dims, ints, alts, W, H = SCENES[name]
    t0 = time.perf_counter()
    host = generate_host(name, seed)
    pos, op, sc, q, sh = (t.to(dev) for t in host)
    del host
    pmin, pmax = lodgen.central_third(pos)
    mem = lodgen.block_membership(pos, pmin, pmax, dims)
    train = train_cameras(name, seed)
    torch.cuda.synchronize()
    t_lod = time.perf_counter()
    scene = lodgen.build_lod_device(pos, op, sc, q, sh, mem, int(np.prod(dims)), train,
                                    distance_intervals=ints, compression_rates=RATES,
                                    lod_sh_degrees=SH_DEGREES, n_mad=N_MAD) if build_lod else None
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


def device_fingerprint(scene) -> str:
    pos = [lc.pos_op[:, :3].float().cpu().numpy() for lc in scene.level_clouds]
    return fingerprint(pos, scene.counts, scene.bounds_min, scene.bounds_max)


def _profiler(env: str):
    """cudaProfilerStart now and return the stop callable when `env` is set (for
    ncu --profile-from-start off captures of exactly the timed region); a
    no-op otherwise.  Never set during a measured run."""
    import torch
    if not os.environ.get(env):
        return lambda: None
    torch.cuda.cudart().cudaProfilerStart()
    return lambda: torch.cuda.cudart().cudaProfilerStop()


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
        # per assembled: 3 fp32 quads (48 B) + depth keys (8 + 4); per visible:
        # its SH row (level width) + HotRec 64 + FastRec 64 + rect 8 + cull box 8
        "project": na * (48 + 12) + st["sh_bytes_visible"] + m * (64 + 64 + 8 + 8),
        # 4 LSD passes over (u32 key, u32 id) -- the first pass reads no ids --
        # + one histogram read + run check
        "depth_sort": na * 4 + 4 * 2 * na * 8 - na * 4 + m * 4,
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
    """Algorithmic float64 flops of the reference blend:
    per evaluated (pixel, splat) the quadratic form (2 sub + 7 mul + 2 add =
    11); per accepted fragment exp (3 mul/add + 9 FMA = 21) and alpha/T/colour
    (4 mul/add + 3 FMA = 10)."""
    return 11.0 * st["evals"] + 31.0 * st["fragments"]


def blend_flops32(st: dict) -> float:
    """Float32 flops the certified blend (K9f) executes for the same work: per
    evaluation the offsets (4) and the log2-domain quadratic form with log2(o)
    folded in (3 FMA + 2 mul = 8); per accepted fragment the error bound (3),
    1 - alpha (1), T (1), the transmittance bound (3 + band 2) and the colour
    weight and sums (1 + 3 FMA = 7): 12 E + 17 F (MUFU ex2/rcp not counted)."""
    return 12.0 * st["evals"] + 17.0 * st["fragments"]


def _traffic_files():
    """profiles/*_frame_traffic.json oldest first: tags are r<round><suffix>,
    suffixes a..z then aa..zz inside a round."""
    import re

    def key(f):
        tag = f.name[: -len("_frame_traffic.json")]
        m = re.match(r"r(\d+)([a-z]*)", tag)
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (-1, 0, tag)
    return sorted((ROOT / "profiles").glob("*_frame_traffic.json"), key=key)


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/*_frame_traffic.json, newest), or None."""
    files = _traffic_files()
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
    files = _traffic_files()
    if not files:
        return None
    data = json.loads(files[-1].read_text())
    hits = [x for k, v in data.items() if k.startswith(kernel) for x in v]
    keys = ("issue_active_pct", "fp64_pipe_pct", "fma_pipe_pct", "smem_pct", "threads_per_inst")
    if not hits or any(k not in hits[0] for k in keys):
        return None
    return {k: round(sum(x[k] or 0.0 for x in hits) / len(hits), 1) for k in keys}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


# ---------------------------------------------------------------------------
# the frame driver (C ABI)


class Frames:
    """cs_render through the C ABI for one source (lod / finest / full / cloud)."""

    def __init__(self, ctx, stream_handle, settings, out, kind, lod=None, force_level=-1, cloud=None):
        import ctypes
        from paper_2404_01133_b200 import _lib, device
        self.lib, self.ctx, self.sh, self.out = _lib.load(), ctx, stream_handle, out
        self.src = _lib.CsSource()
        self.src.kind = kind
        self.src.force_level = force_level
        if lod is not None:
            self.src.lod = lod.handle
        if cloud is not None:
            self.src.cloud = cloud.desc()
        self.keep = (lod, cloud)
        self.cset = device.settings_struct(settings)
        self.ctypes = ctypes
        self._lib = _lib

    def __call__(self, ccam, flags=0, stats=None, out=None):
        c = self.ctypes
        rc = self.lib.cs_render(self.ctx, c.byref(self.src), c.byref(ccam), c.byref(self.cset),
                                (out if out is not None else self.out).data_ptr(), flags,
                                c.byref(stats) if stats is not None else None, self.sh)
        self._lib.check(rc, "cs_render")


def per_frame_ms(fr: Frames, ccams, stream):
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(ccams) + 1)]
    ev[0].record(stream)
    for i, c in enumerate(ccams):
        fr(c)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ccams))]


def size_pass(fr: Frames, ccams):
    """Synchronous renders: grow the pair buffers to the largest frame."""
    from paper_2404_01133_b200._lib import CS_RENDER_SYNC, CsFrameStats
    out = []
    for c in ccams:
        s = CsFrameStats()
        fr(c, CS_RENDER_SYNC, s)
        out.append(s)
    return out


def frame_counts(fr: "Frames", ccams, ctx, sh, lod_scene=None, sh_coeffs_full=16):
    """Per-frame counts summed over `ccams` (CS_RENDER_DIAG renders): assembled,
    visible, pairs, evaluations, fragments, warp hits, and the SH bytes the
    projection reads for visible splats (their width depends on the level:
    C = 16/9/4 -> 192/112/48 B, weighted by the frame's assembled level mix)."""
    import ctypes
    from paper_2404_01133_b200 import _lib
    from paper_2404_01133_b200._lib import CsFrameStats
    from paper_2404_01133_b200.device import sh_stride
    lib = _lib.load()
    counts = dict(assembled=0, visible=0, pairs=0, evals=0, fragments=0, sh_bytes_visible=0, warp_hits=0,
                  warp_hits_empty=0, blend_exact_hits=0, blend_floor_resolved=0, blend_replays=0)
    seg_idx = (ctypes.c_int32 * 4096)()
    seg_cnt = (ctypes.c_int64 * 4096)()
    n_seg = ctypes.c_int32(0)
    item_max, item_sum = [], []
    for c in ccams:
        s = CsFrameStats()
        fr(c, _lib.CS_RENDER_SYNC | _lib.CS_RENDER_DIAG, s)
        for k_ in ("assembled", "visible", "pairs", "evals", "fragments", "warp_hits", "warp_hits_empty",
                   "blend_exact_hits", "blend_floor_resolved", "blend_replays"):
            counts[k_] += getattr(s, k_)
        item_max.append(s.blend_max_item_cycles)
        item_sum.append(s.blend_item_cycles)
        if lod_scene is not None:
            row_bytes = [4 * sh_stride(lc.sh_coeffs) for lc in lod_scene.level_clouds]
            _lib.check(lib.cs_dump_segments(ctx, seg_idx, seg_cnt, 4096, ctypes.byref(n_seg), sh))
            sh_assembled = sum(seg_cnt[q] * row_bytes[seg_idx[q] // lod_scene.n_blocks] for q in range(n_seg.value))
            counts["sh_bytes_visible"] += sh_assembled * (s.visible / max(s.assembled, 1))
        else:
            counts["sh_bytes_visible"] += s.visible * 4 * sh_stride(sh_coeffs_full)
    return counts, item_max, item_sum


def fps_summary(ms):
    return {"mean_fps": round(1000.0 * len(ms) / sum(ms), 1), "min_fps": round(1000.0 / max(ms), 1),
            "mean_ms": round(sum(ms) / len(ms), 4), "max_ms": round(max(ms), 4)}


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
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # rank count / NVLS visible in the log
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200._lib import CsFrameStats

    # N > 1: rank 0 runs the LoD build, the levels and table reach the other
    # ranks by NCCL broadcast (fusion.broadcast_device_lod_scene)
    scene, center, radius, alts, wh, build_s, raw = build_scene(args.scene, args.seed, dev,
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
    sha = device_fingerprint(scene)
    cams_all = flythrough(center, radius, alts, wh, FRAMES_PER_ALT)
    K = args.steps
    # view split: rank r renders its contiguous share of the flythrough
    share = [i for i in range(len(cams_all)) if i * world // len(cams_all) == rank] or list(range(len(cams_all)))
    mine = [share[i] for i in timed_frames(len(share), K)]       # strided over the share
    settings = cs.RenderSettings()
    ctx = device.context(local)
    stream = torch.cuda.current_stream(dev)
    sh = device.stream_handle(dev)
    W, H = wh
    out = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    ccam = [device.camera_struct(c) for c in cams_all]
    lod = Frames(ctx, sh, settings, out, _lib.CS_SRC_LOD_BLOCK, lod=scene)
    lib = _lib.load()
    import ctypes

    # sizing pass (synchronous, grows pair buffers) + per-frame counts for the roofline
    size_pass(lod, [ccam[i] for i in mine])
    counts, blend_item_max, blend_item_sum = frame_counts(lod, [ccam[i] for i in mine], ctx, sh, scene)
    for i in range(args.warmup):
        lod(ccam[mine[i % len(mine)]])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        prof = _profiler("CS_PROFILE_FRAMES")  # ncu --profile-from-start off: the timed frames only
        for i in mine:
            lod(ccam[i])
        e1.record(stream)
        torch.cuda.synchronize()
        prof()
    ms = e0.elapsed_time(e1)
    # per-stage breakdown from a second, untimed pass with CUDA-event marks
    # between the stages (the timed frames above run as replayed frame graphs,
    # cs_render's asynchronous fast path; marked frames take the direct path)
    lib.cs_timing_begin(ctx, K)
    for i in mine:
        lod(ccam[i])
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
        for n_, i in enumerate(mine):
            b = n_ & 1
            done[b].synchronize()  # host buffer b free again
            lod(ccam[i], out=outs[b])
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
               "path": "cs_render (C ABI) + D2H of the float32 image into pinned host memory, "
                       "host wall clock over the same strided frames"}

    clocks = clk.summary()
    value = world * K / (ms_max / 1000.0)
    roof = frame_roofline(lib, ctx, sh, stages_ms, counts, K)

    # cmd_bench's protocol (cli.py:236-294): per altitude x mode mean and min FPS
    altitudes = None
    if not args.no_modes:
        altitudes = modes_pass(args, scene, raw, cams_all, ccam, alts, ctx, sh, settings, out, stream, share)

    c5 = None
    if not args.no_c5:
        c5 = c5_leg(args, scene, ctx, sh, settings, out, stream, wh, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(scene, cams_all, mine, settings)

    c12 = None
    if rank == 0 and world == 1 and not args.no_c12:
        c12 = {"c1": small_config_leg("c1", ctx, sh, dev, not args.no_cpu_baseline),
               "c2": small_config_leg("c2", ctx, sh, dev, not args.no_cpu_baseline)}

    assign = None
    if raw is not None and not args.no_assign and rank == 0:
        del scene
        scene = None
        lod = None
        torch.cuda.empty_cache()
        assign = assign_leg(args, raw, wh, dev)
    train = None
    if not args.no_train and raw is not None:
        scene = None
        lod = None
        torch.cuda.empty_cache()
        train = train_leg(args, raw, wh, rank, world, dev)
        raw = None

    if rank == 0:
        line = {
            "metric": "1080p FPS on 23M-Gaussian LoD city" if args.scene == "c3" else f"FPS ({args.scene})",
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_city_torch on the host, seeded CPU generator; reference "
                    "distributions), random-init scene",
            "config": run_config(args.scene, K, cams_all, sha),
            "view_split": world > 1,
            "scene_build_s": round(build_s, 1),
            "stages_ms": stages_ms,
            "counts_per_frame": {k: v / K for k, v in counts.items()},
            "blend_longest_item_us": (round(float(np.median(blend_item_max)) / ((clocks or {}).get("sm_mhz") or 1965.0), 1)
                                      if blend_item_max else None),
            "blend_item_us_sum_per_warp_slot": (round(float(np.median(blend_item_sum)) / ((clocks or {}).get("sm_mhz") or 1965.0)
                                                      / lib_blend_slots(), 1) if blend_item_sum else None),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "altitudes": altitudes,
            "c1": (c12 or {}).get("c1"),
            "c2": (c12 or {}).get("c2"),
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


def frame_roofline(lib, ctx, sh, stages_ms, counts, K, tag=""):
    """roofline object of the dominant stage (+ every HBM-bound stage)."""
    import ctypes
    from paper_2404_01133_b200 import _lib
    pk_json = peaks()
    hbm_peak = pk_json.get("hbm_gbs", 6450.0)
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
                "frac": achieved / hbm_peak, "traffic": traffic if not tag else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk_json else "B200_PROFILING.md fallback"}
    else:  # blend
        # The reference's blend is float64 arithmetic (_kernels.py:52-72): its
        # algorithmic work is blend_flops (FP64 flops).  K9f takes the same
        # decisions from certified float32 evaluations,
        # so the primary figure is the reference's FP64 work per second against
        # the FP64 peak measured here; the FP32 work the kernel actually issues
        # is reported beside it against the FP32 peak.
        pk = ctypes.c_double(0.0)
        _lib.check(lib.cs_measure_fp64_peak(ctx, ctypes.byref(pk), sh), "cs_measure_fp64_peak")
        fp64_peak = pk.value
        sec = stages_ms[dom] / 1000.0
        achieved = blend_flops(counts) / K / sec / 1e12
        fp32_peak = 148 * 128 * 2 * pk_json.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        a32 = blend_flops32(counts) / K / sec / 1e12
        traffic, tsrc = ncu_traffic("k_blend_fast")
        roof = {"kernel": "k_blend_fast", "bound": "fp64", "achieved": achieved, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic if not tag else None,
                "peak_source": "measured in this run: dense DFMA chains on every SM, CUDA events "
                               "(cs_measure_fp64_peak; MEASURED_PEAKS.json has no FP64 entry)",
                "flops_per_frame": blend_flops(counts) / K,
                "work": "reference float64 blend flops (11 per evaluation, 31 per fragment); "
                        "executed as certified float32 (fp32 below) with float64 re-decisions",
                "fp32": {"achieved": a32, "peak": fp32_peak, "frac": a32 / fp32_peak,
                         "flops_per_frame": blend_flops32(counts) / K,
                         "peak_source": "148 SMs x 128 FP32 lanes x 2 x max SM clock (B200_PROFILING.md)"}}
    roof["traffic_source"] = (f"profiles/{tsrc} (ncu --set full, dram__bytes_read+write per launch)"
                              if tsrc and not tag else None)
    # the blend is issue-bound (divergent per-pixel termination), not FP64-pipe-bound:
    # the ncu pipe utilisations of the same capture explain the flop fraction
    if not tag:
        roof["ncu_pipes_pct"] = ncu_pipes("k_blend_fast")
    roof["stages_hbm"] = stage_roof
    return roof


def modes_pass(args, scene, raw, cams_all, ccam, alts, ctx, sh, settings, out, stream, share):
    """cmd_bench (cli.py:236-294): every frame of this rank's share per mode,
    timed individually with CUDA events; per altitude mean FPS = 1000 n / sum
    ms and min FPS = 1000 / max ms (cli.py:267-279).  Modes: lod (block LoD),
    finest (every visible block at the finest level), full (the whole cloud,
    no LoD: the paper's ablation)."""
    from paper_2404_01133_b200 import _lib, device
    modes = {"lod": Frames(ctx, sh, settings, out, _lib.CS_SRC_LOD_BLOCK, lod=scene),
             "finest": Frames(ctx, sh, settings, out, _lib.CS_SRC_LOD_BLOCK, lod=scene,
                              force_level=scene.n_levels - 1)}
    full = None
    if raw is not None:
        pos, op, sc, q, shc = raw[:5]
        full = device.DeviceCloud.from_torch(pos, op, sc, q, shc)
        modes["full"] = Frames(ctx, sh, settings, out, _lib.CS_SRC_CLOUD, cloud=full)
    res = {}
    for name, fr in modes.items():
        cams = [ccam[i] for i in share]
        st = size_pass(fr, cams)
        per_frame_ms(fr, cams[:4], stream)      # warm (captures the frame graph)
        ms = per_frame_ms(fr, cams, stream)
        for a_i, alt in enumerate(alts):
            sel = [k for k, i in enumerate(share) if i // FRAMES_PER_ALT == a_i]
            if not sel:
                continue
            d = res.setdefault(f"{int(alt)}m", {})
            d[name] = fps_summary([ms[k] for k in sel])
            d[name]["pairs_M_max"] = round(max(st[k].pairs for k in sel) / 1e6, 2)
            d[name]["visible_M_mean"] = round(sum(st[k].visible for k in sel) / len(sel) / 1e6, 3)
    del full
    res["what"] = ("per altitude x mode: all frames of the orbit, each timed with CUDA events "
                   "(frame graphs replayed), mean_fps = 1000 n / sum ms, min_fps = 1000 / max ms "
                   "(cmd_bench, cli.py:267-279)")
    return res


def c5_leg(args, scene, ctx, sh, settings, out, stream, wh, rank, world):
    """C5: batch render of the 740 test views of a 5920-camera set (every 8th,
    colmap.py:152-156) on the same LoD scene, view-split across ranks."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200.synth import city_cameras
    lib = _lib.load()
    all5 = city_cameras(5920, SCENES[args.scene][1], wh[0], wh[1], seed=args.seed)
    test5 = [c for i, c in enumerate(all5) if i % 8 == 0]
    mine = [test5[i] for i in range(len(test5)) if i * world // len(test5) == rank]
    c5cams = [device.camera_struct(c) for c in mine]
    fr = Frames(ctx, sh, settings, out, _lib.CS_SRC_LOD_BLOCK, lod=scene)
    st5 = size_pass(fr, c5cams)
    vis5 = [s.visible for s in st5]
    pairs5 = [s.pairs for s in st5]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for c in c5cams:
        fr(c)
    f1.record(stream)
    torch.cuda.synchronize()
    t5 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=out.device)
    if world > 1:
        dist.all_reduce(t5, op=dist.ReduceOp.MAX)
    # untimed second pass with the per-stage event marks
    lib.cs_timing_begin(ctx, len(c5cams))
    for c in c5cams:
        fr(c)
    torch.cuda.synchronize()
    st = (ctypes.c_double * 8)()
    n5 = ctypes.c_int32(0)
    _lib.check(lib.cs_timing_end(ctx, st, ctypes.byref(n5)))
    return {"metric": "C5 batch render FPS (740 test views, 1080p, LoD, view-split)",
            "value": len(test5) / (float(t5.item()) / 1000.0), "unit": "frames/s",
            "views": len(test5), "views_this_rank": len(mine), "n_gpus": world,
            "ms_max_rank": float(t5.item()), "scaling": "weak in views per rank" if world > 1 else "n/a",
            "visible_M_min_med_max": [round(float(x) / 1e6, 3) for x in
                                      (min(vis5), float(np.median(vis5)), max(vis5))] if vis5 else None,
            "pairs_M_min_med_max": [round(float(x) / 1e6, 3) for x in
                                    (min(pairs5), float(np.median(pairs5)), max(pairs5))] if pairs5 else None,
            "stages_ms": {k: round(st[i] / max(n5.value, 1), 4) for i, k in enumerate(STAGES)}}


def small_config_leg(name, ctx, sh, dev, with_cpu: bool):
    """C1 (configs[0]: 100k city, one block, 3 LoD levels, 256x256, the 16
    generated views) and C2 (configs[1]: 1.1M city, 1080p, no LoD, the 16
    generated views + 4 look_at altitude views {0.15, 0.5, 1.5, 4.0} x extent):
    device-timed FPS over all views, stage breakdown + roofline, and the C
    oracle on the same frames (C1: all 16; C2: 2 views) with parity counts."""
    import ctypes
    import torch
    from paper_2404_01133_b200 import _lib, device, lodgen
    from paper_2404_01133_b200.synth import city_cameras, generate_city_torch, look_at
    lib = _lib.load()
    from paper_2404_01133_b200.render import RenderSettings
    settings = RenderSettings()
    stream = torch.cuda.current_stream(dev)
    if name == "c1":
        n, extent, nb, W, H = 100_000, 100.0, 40, 256, 256
    else:
        n, extent, nb, W, H = 1_100_000, 100.0, 40, 1920, 1080
    pos, op, sc, q, shc = (t.to(dev) for t in generate_city_torch(0, extent, nb, n, device="cpu"))
    cams = city_cameras(16, extent, W, H, seed=0)
    out = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    if name == "c1":
        pmin, pmax = lodgen.central_third(pos)
        mem = lodgen.block_membership(pos, pmin, pmax, (1, 1))
        train = [c for i, c in enumerate(cams) if i % 8 != 0]
        scene = lodgen.build_lod_device(pos, op, sc, q, shc, mem, 1, train,
                                        distance_intervals=((0.0, 40.0), (40.0, 80.0), (80.0, INF)))
        fr = Frames(ctx, sh, settings, out, _lib.CS_SRC_LOD_BLOCK, lod=scene)
        what = "100k city, 1 block, 3 LoD levels (intervals 0/40/80 m), 256x256, 16 views, LoD block mode"
    else:
        center = pos.double().mean(dim=0).cpu().numpy()
        for f in (0.15, 0.5, 1.5, 4.0):
            cams.append(look_at(center + np.array([f * extent, 0.0, f * extent]), center, W, H, 0.85 * W))
        scene = device.DeviceCloud.from_torch(pos, op, sc, q, shc)
        fr = Frames(ctx, sh, settings, out, _lib.CS_SRC_CLOUD, cloud=scene)
        what = "1.1M city, no LoD, 1920x1080, 16 generated views + 4 altitude views"
    ccams = [device.camera_struct(c) for c in cams]
    stats = size_pass(fr, ccams)
    counts, _, _ = frame_counts(fr, ccams, ctx, sh, scene if name == "c1" else None)
    reps = 8 if name == "c1" else 2
    per_frame_ms(fr, ccams, stream)   # warm + frame graphs
    ms = []
    for _ in range(reps):
        ms += per_frame_ms(fr, ccams, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        for c in ccams:
            fr(c)
    e1.record(stream)
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    nf = reps * len(ccams)
    lib.cs_timing_begin(ctx, len(ccams))
    for c in ccams:
        fr(c)
    torch.cuda.synchronize()
    st = (ctypes.c_double * 8)()
    nst = ctypes.c_int32(0)
    _lib.check(lib.cs_timing_end(ctx, st, ctypes.byref(nst)))
    stages_ms = {k: st[i] / max(nst.value, 1) for i, k in enumerate(STAGES)}
    leg = {"metric": f"{name.upper()} FPS", "value": nf / (total_ms / 1000.0), "unit": "frames/s",
           "frames": nf, "views": len(cams), "what": what, **fps_summary(ms),
           "stages_ms": {k: round(v, 4) for k, v in stages_ms.items()},
           "visible_M_min_max": [round(min(s.visible for s in stats) / 1e6, 3),
                                 round(max(s.visible for s in stats) / 1e6, 3)],
           "pairs_M_min_max": [round(min(s.pairs for s in stats) / 1e6, 3),
                               round(max(s.pairs for s in stats) / 1e6, 3)],
           "roofline": frame_roofline(lib, ctx, sh, stages_ms, counts, len(ccams), tag=name)}
    if with_cpu:
        leg["cpu_baseline"] = small_cpu_baseline(name, scene, pos, op, sc, q, shc, cams, settings)
    return leg


def small_cpu_baseline(name, scene, pos, op, sc, q, shc, cams, settings):
    from types import SimpleNamespace
    from oracle import oracle as O
    import paper_2404_01133_b200 as cs
    nthreads = os.cpu_count() or 1
    if name == "c1":
        hs = host_scene(scene)
        pick = list(range(len(cams)))
    else:
        host = SimpleNamespace(positions=pos.cpu().numpy(), opacities=op.cpu().numpy(),
                               scales=sc.cpu().numpy(), rotations=q.cpu().numpy(), sh=shc.cpu().numpy())
        pick = [1, len(cams) - 2]   # an orbit view and the 1.5 x extent altitude view
    O.lib()
    t0 = time.perf_counter()
    outs = []
    for i in pick:
        cloud = O.assemble(hs, cams[i])[0] if name == "c1" else host
        outs.append(O.rasterize_frame_c(cloud, cams[i], settings, nthreads=nthreads))
    dt = time.perf_counter() - t0
    parity = []
    for i, (rimg, rst) in zip(pick, outs):
        src = cs.assemble_render_set(scene, cams[i]).cloud if name == "c1" else scene
        img, st = cs.rasterize_stats(src, cams[i], settings)
        parity.append(st.visible_splats == rst["visible_splats"] and
                      st.blended_fragments == rst["blended_fragments"] and
                      float(np.abs(img.pixels - rimg).max()) <= 1e-4)
    return {"value": len(pick) / dt, "unit": "frames/s", "cores": nthreads, "kind": "port",
            "cpu_model": cpu_model(), "sample": f"{len(pick)} of the leg's views (C oracle, all stages)",
            "parity_ok": all(parity), "parity_frames": len(parity)}


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
    Per-phase rooflines: forward (the frame's dominant stage), loss (FP32
    flops of the SSIM/L1 forward + gradient), backward (float64 decision
    replay + float32 partials, per evaluation / accepted fragment), Adam (HBM
    bytes of the update).
    """
    import torch
    import torch.distributed as dist
    from paper_2404_01133_b200 import _lib, blocktrain, fusion
    from paper_2404_01133_b200._lib import CsFrameStats
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
    schedule = []
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    prof = _profiler("CS_PROFILE_TRAIN")
    for i in range(K):
        job = order[i % len(order)]
        v = job.iters % len(job.cams)
        job.iters += 1
        schedule.append((job, v))
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
    # algorithmic work of the same K iterations (untimed DIAG renders of the
    # same views: evaluations E, fragments F, visible M; block sizes)
    E = F = M = G = 0
    for job, v in schedule:
        s = CsFrameStats()
        tr = job.trainer
        from paper_2404_01133_b200 import device as _dev
        import ctypes
        out = torch.empty((wh[1], wh[0], 3), dtype=torch.float32, device=dev)
        _lib.check(_lib.load().cs_render(tr.h, ctypes.byref(tr.src), ctypes.byref(_dev.camera_struct(job.cams[v])),
                                         ctypes.byref(tr.cset), out.data_ptr(),
                                         _lib.CS_RENDER_SYNC | _lib.CS_RENDER_DIAG, ctypes.byref(s),
                                         _dev.stream_handle(dev)))
        E += s.evals
        F += s.fragments
        M += s.visible
        G += tr.K
        C = tr.C
    px = wh[0] * wh[1]
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6450.0)
    fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12   # TFLOP/s at the max SM clock (B200_PROFILING.md)
    # loss (K13): 5 windowed moments (separable 11-tap: 44 flops each) + SSIM map per
    # pixel and channel, gradient: 3 partial maps correlated back (132) + combine
    loss_flops = (5 * 44 + 20 + 3 * 44 + 15) * 3 * px
    # Adam (K14): geom 11 floats x (param, m, v read+write, grad read) + SH 3C floats x
    # the same + 48 B of activated quads written, per Gaussian
    adam_bytes = (11 * 4 * 7 + 3 * C * 4 * 7 + 48) * G / K
    # backward (K10 + K11): float64 decision replay per evaluation (11) and per
    # accepted fragment (31) as the forward, per fragment ~40 float32 flops of
    # partials (not counted against the FP64 pipe)
    bwd_flops64 = (11.0 * E + 31.0 * F) / K
    roof = {
        "forward": {"ms": phases["forward"], "note": "the frame pipeline; see the C3 roofline"},
        "loss": {"bound": "fp32", "achieved": loss_flops / (phases["loss"] / 1e3) / 1e12, "peak": fp32_peak,
                 "unit": "TFLOP/s", "flops_per_iter": loss_flops,
                 "frac": loss_flops / (phases["loss"] / 1e3) / 1e12 / fp32_peak},
        "backward": {"bound": "fp64", "flops64_per_iter": bwd_flops64,
                     "achieved": bwd_flops64 / (phases["backward"] / 1e3) / 1e12, "unit": "TFLOP/s",
                     "evals_per_iter": E / K, "fragments_per_iter": F / K, "visible_per_iter": M / K},
        "adam": {"bound": "hbm", "bytes_per_iter": adam_bytes,
                 "achieved": adam_bytes / (phases["adam"] / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                 "frac": adam_bytes / (phases["adam"] / 1e3) / 1e9 / hbm},
    }
    # fusion: every rank filters its blocks; NCCL all-gather-v in block order
    local = {j: jb.fusion_inputs() for j, jb in jobs.items()}
    fuse_ms = None
    fused_n = None
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        f0 = time.perf_counter()
        fused = fusion.fuse_all_gather(local, n_blocks, owner, pmin, pmax, dims, sh_coeffs=16,
                                       dtype=torch.float32, device=dev)
        torch.cuda.synchronize()
        fuse_ms = 1000 * (time.perf_counter() - f0)
        fused_n = int(fused.shape[0])
    sizes = [jobs[j].count for j in jobs]
    return {
        "metric": "block-train iters/s (C4)", "value": world * K / (ms_max / 1000.0), "unit": "iters/s",
        "ms_per_iter": ms_max / K, "steps": K, "warmup": args.train_warmup, "n_gpus": world,
        "scaling": "weak", "phases_ms": phases, "roofline": roof,
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


def cpu_baseline(scene, cams, timed, settings):
    """The C oracle port (oracle/), all host threads, on a bounded sample: one
    timed frame per altitude.  Then the full-size parity of the same frames
    (checker only, outside every timed region): the compatibility tier
    (assemble_render_set + rasterize_stats, device tile list) vs the oracle's
    decisions, assembled count, sorted tile list, fragments and image."""
    from oracle import oracle as O
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import bin_tiles_last
    hs = host_scene(scene)
    pick = []
    for a in range(len(cams) // FRAMES_PER_ALT):
        on_alt = [i for i in timed if i // FRAMES_PER_ALT == a]
        if on_alt:
            pick.append(on_alt[len(on_alt) // 2])
    nthreads = os.cpu_count() or 1
    O.lib()
    t0 = time.perf_counter()
    outs = []
    for i in pick:
        cloud, _ = O.assemble(hs, cams[i])
        outs.append(O.rasterize_frame_c(cloud, cams[i], settings, nthreads=nthreads))
    dt = time.perf_counter() - t0
    parity = []
    for i, (ref_img, ref_st) in zip(pick, outs):
        cam = cams[i]
        dec = cs.decide_visibility(scene, cam)
        odec = O.decide_visibility(hs, cam)
        dec_ok = [(d.block, d.visible, d.level, d.distance, d.screen_box) for d in dec] == list(odec)
        a = cs.assemble_render_set(scene, cam)
        ocloud, _ = O.assemble(hs, cam)
        img, st = cs.rasterize_stats(a.cloud, cam, settings)
        tid, off = bin_tiles_last(cam, settings.tile_size)
        rp = O.project_cloud(ocloud, cam, settings, nthreads=nthreads)
        rtid, roff, _, _ = O.bin_tiles(rp, cam, settings.tile_size)
        parity.append({"frame": i, "decisions_bit_exact": dec_ok,
                       "assembled": [a.cloud.count, ocloud.count],
                       "visible": [st.visible_splats, ref_st["visible_splats"]],
                       "pairs": [int(tid.shape[0]), int(rtid.shape[0])],
                       "tile_lists_bit_exact": bool(np.array_equal(tid, rtid) and np.array_equal(off, roff)),
                       "fragments": [st.blended_fragments, ref_st["blended_fragments"]],
                       "image_max_abs_err": float(np.abs(img.pixels - ref_img).max())})
        del tid, rtid, rp
    ok = all(q["decisions_bit_exact"] and q["tile_lists_bit_exact"] and q["assembled"][0] == q["assembled"][1]
             and q["visible"][0] == q["visible"][1] and q["fragments"][0] == q["fragments"][1]
             and q["image_max_abs_err"] <= 1e-4 for q in parity)
    return {"value": len(pick) / dt, "unit": "frames/s", "cores": nthreads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"frames {pick} (one timed frame per altitude; assemble + project + sort + bin + blend)",
            "parity": {"frames": parity, "ok": ok,
                       "bar": "decisions and sorted tile lists bit-exact, counts equal, image max-abs <= 1e-4"}}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores, never
    loading libcsgpu.so.  Scene: the same seeded host generator, detail levels
    by oracle.build_lod (lod.py:211-248 restated), membership by
    oracle.block_of_points; frames: the same strided flythrough frames as the
    GPU arm, each assembled (lod.py:360-401) and rendered (render.py:252-280)
    by the C oracle with all host threads."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    name = args.scene
    n, extent, nb, dims, ints, alts, W, H = SCENES[name]
    t0 = time.perf_counter()
    pos, op, sc, q, sh = (t.numpy() for t in generate_host(name, args.seed))
    cloud = O.Arrays(pos, op, sc, q, sh)
    p64 = pos.astype(np.float64)
    lo, hi = p64.min(axis=0), p64.max(axis=0)
    # ContractionMap.central_third (partition.py:84-97), as lodgen.central_third
    center = 0.5 * (lo + hi)
    sixth = np.maximum((hi - lo) / 6.0, 1e-6)
    z1 = hi[2] if hi[2] > lo[2] else lo[2] + 1e-6
    pmin = np.array([center[0] - sixth[0], center[1] - sixth[1], lo[2]])
    pmax = np.array([center[0] + sixth[0], center[1] + sixth[1], z1])
    mem = O.block_of_points(pos, pmin, pmax, dims)
    nthreads = os.cpu_count() or 1
    t_lod = time.perf_counter()
    hs = O.build_lod(cloud, mem, int(np.prod(dims)), train_cameras(name, args.seed), ints, RATES, SH_DEGREES,
                     N_MAD, nthreads=nthreads)
    lod_s = time.perf_counter() - t_lod
    del cloud, pos, op, sc, q, sh, p64
    counts = np.array([[b.count for b in L] for L in hs.levels], dtype=np.int64)
    sha = fingerprint([np.concatenate([np.asarray(b.positions) for b in L]) for L in hs.levels],
                      counts, hs.bounds_min, hs.bounds_max)
    cams = flythrough_of(lo, hi, name)
    build_s = time.perf_counter() - t0
    K = args.steps
    frames = timed_frames(len(cams), K)
    warm = min(args.warmup, 2)
    settings = O.DefaultSettings()
    for i in range(warm):
        c, _ = O.assemble(hs, cams[frames[i % K]])
        O.rasterize_frame_c(c, cams[frames[i % K]], settings, nthreads=nthreads)
    per = []
    t1 = time.perf_counter()
    for i in frames:
        ts = time.perf_counter()
        c, _ = O.assemble(hs, cams[i])
        O.rasterize_frame_c(c, cams[i], settings, nthreads=nthreads)
        per.append(1000.0 * (time.perf_counter() - ts))
    dt = time.perf_counter() - t1
    v = K / dt
    alt = {}
    for a_i, a in enumerate(alts):
        ms = [m for i, m in zip(frames, per) if i // FRAMES_PER_ALT == a_i]
        if ms:
            alt[f"{int(a)}m"] = {"lod": fps_summary(ms)}
    print(json.dumps({
        "impl": "reference", "metric": "1080p FPS on 23M-Gaussian LoD city" if name == "c3" else f"FPS ({name})",
        "value": v, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": warm,
        "ms_per_step": 1000 * dt / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (generate_city_torch on the host, seeded CPU generator)",
        "config": run_config(name, K, cams, sha),
        "altitudes": alt,
        "scene_build_s": round(build_s, 1), "lod_build_host_s": round(lod_s, 1),
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": nthreads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"the {K} strided flythrough frames {frames[:3]}...{frames[-1]} "
                                   f"(requested steps={args.steps}); C oracle: assemble + project + sort "
                                   f"+ bin + blend, {nthreads} threads"},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
