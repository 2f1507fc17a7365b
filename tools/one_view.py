"""Render one C5 test view of the C3 LoD scene a few times (for ncu captures
of a single frame): python tools/one_view.py VIEW [REPEATS]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    view = int(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200.render import RenderSettings
    from paper_2404_01133_b200.synth import city_cameras
    scene, center, radius, alts, wh, _, _ = bench.build_scene("c3", 0, dev, keep_raw=False)
    ctx = device.context(0)
    sh = torch.cuda.current_stream().cuda_stream
    out = torch.empty((wh[1], wh[0], 3), dtype=torch.float32, device=dev)
    fr = bench.Frames(ctx, sh, RenderSettings(), out, _lib.CS_SRC_LOD_BLOCK, lod=scene)
    all5 = city_cameras(5920, bench.SCENES["c3"][1], wh[0], wh[1], seed=0)
    cam = device.camera_struct([c for i, c in enumerate(all5) if i % 8 == 0][view])
    bench.size_pass(fr, [cam])
    torch.cuda.synchronize()
    stop = bench._profiler("CS_PROFILE_FRAMES")
    for _ in range(reps):
        fr(cam, _lib.CS_RENDER_SYNC)
    torch.cuda.synchronize()
    stop()


if __name__ == "__main__":
    main()
