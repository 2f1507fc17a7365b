"""Launch-gap estimate for one C3 frame: the same camera rendered K times by
direct cs_render calls vs by replaying a CUDA graph captured from one
cs_render call (same kernels and memsets; the graph removes host launch
cost and most inter-kernel gaps).  Diagnostic only."""
import ctypes
import importlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2404_01133_b200 import _lib, device  # noqa: E402
from paper_2404_01133_b200._lib import CsSource  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    scene, center, radius, alts, wh, _, _ = bench.build_scene("c3", 0, dev)
    cam = bench.flythrough(center, radius, alts, wh, 4)[1]
    lib = _lib.load()
    ctx = device.context(0)
    src = CsSource()
    src.kind = _lib.CS_SRC_LOD_BLOCK
    src.force_level = -1
    src.lod = scene.handle
    settings = importlib.import_module("paper_2404_01133_b200.render").RenderSettings()
    c = device.camera_struct(cam)
    s = device.settings_struct(settings)
    out = torch.empty((wh[1], wh[0], 3), dtype=torch.float32, device=dev)
    side = torch.cuda.Stream()

    def frame(stream, flags=0):
        _lib.check(lib.cs_render(ctx, ctypes.byref(src), ctypes.byref(c), ctypes.byref(s), out.data_ptr(),
                                 flags, None, ctypes.c_void_p(stream.cuda_stream)), "cs_render")

    with torch.cuda.stream(side):
        frame(side, _lib.CS_RENDER_SYNC)
        for _ in range(5):
            frame(side)
    torch.cuda.synchronize()
    K = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record(side)
        for _ in range(K):
            frame(side)
        e1.record(side)
    torch.cuda.synchronize()
    direct = e0.elapsed_time(e1) / K
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        frame(side)
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / K
    print(f"direct {direct:.4f} ms/frame  graph {graph:.4f} ms/frame  gap estimate {direct - graph:.4f} ms")


if __name__ == "__main__":
    main()
