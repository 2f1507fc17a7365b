"""Per-tile list-length statistics of the bench's C3 flythrough frames (tile
scheduling diagnostics for the blend): max / percentiles of pairs per tile
and the heaviest tiles' share of all pairs."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import importlib  # noqa: E402
render = importlib.import_module("paper_2404_01133_b200.render")
from paper_2404_01133_b200.lod import AssembledCloud  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    scene, center, radius, alts, wh, _, _ = bench.build_scene("c3", 0, dev)
    cams = bench.flythrough(center, radius, alts, wh, 4)
    for i, cam in enumerate(cams[::3]):
        ac = AssembledCloud(scene, cam, "block", None, 0, [])
        render.render(ac, cam)
        torch.cuda.synchronize()
        _, offs = render.bin_tiles_last(cam, 16)
        n = np.diff(offs)
        q = np.percentile(n, [50, 90, 99, 99.9])
        top = np.sort(n)[::-1]
        print(f"view {i}: pairs {n.sum()/1e6:.2f}M tiles {n.size} max {n.max()} p50/90/99/99.9 "
              f"{q.astype(int).tolist()} top10 {top[:10].tolist()} top1% share {top[:n.size // 100].sum() / n.sum():.3f}")


if __name__ == "__main__":
    main()
