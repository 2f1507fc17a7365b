"""Per-view blend diagnostics on the C3 LoD scene: the 740 C5 test views (and
the C3 flythrough), each rendered once with CS_RENDER_DIAG (counters: float64
hits, floor re-decisions, transmittance replays, longest work item) and timed
per frame (CUDA events).  Run twice -- default and CS_BLEND_EXACT=1 -- and
compare:  python tools/blend_views.py OUT.json"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    out_path = sys.argv[1]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200._lib import CS_RENDER_DIAG, CS_RENDER_SYNC, CsFrameStats
    from paper_2404_01133_b200.render import RenderSettings
    from paper_2404_01133_b200.synth import city_cameras
    scene, center, radius, alts, wh, _, _ = bench.build_scene("c3", 0, dev, keep_raw=False)
    ctx = device.context(0)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    out = torch.empty((wh[1], wh[0], 3), dtype=torch.float32, device=dev)
    fr = bench.Frames(ctx, sh, RenderSettings(), out, _lib.CS_SRC_LOD_BLOCK, lod=scene)
    all5 = city_cameras(5920, bench.SCENES["c3"][1], wh[0], wh[1], seed=0)
    test5 = [device.camera_struct(c) for i, c in enumerate(all5) if i % 8 == 0]
    bench.size_pass(fr, test5)
    ms = bench.per_frame_ms(fr, test5, stream)   # warm
    ms = bench.per_frame_ms(fr, test5, stream)
    rows = []
    for i, c in enumerate(test5):
        s = CsFrameStats()
        fr(c, CS_RENDER_DIAG | CS_RENDER_SYNC, s)
        rows.append({"view": i, "ms": ms[i], "pairs": s.pairs, "visible": s.visible, "evals": s.evals,
                     "frags": s.fragments, "exact": s.blend_exact_hits, "floor": s.blend_floor_resolved,
                     "replays": s.blend_replays, "longest_us": s.blend_max_item_cycles / 1965.0})
    json.dump(rows, open(out_path, "w"))
    t = sum(r["ms"] for r in rows)
    print("total ms", round(t, 2), "FPS", round(1000 * len(rows) / t, 1))
    for k in ("exact", "floor", "replays"):
        print(k, "sum", sum(r[k] for r in rows), "max", max(r[k] for r in rows))
    top = sorted(rows, key=lambda r: -r["ms"])[:12]
    for r in top:
        print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})


if __name__ == "__main__":
    main()
