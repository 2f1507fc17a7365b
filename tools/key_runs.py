"""How many depth keys share a sort key (K4b run fix-up load) if the 32-bit
depth key were cut to its top 24 bits (3 radix passes instead of 4): C3
frames, depths from the projection dump (depth order)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    from paper_2404_01133_b200.lod import AssembledCloud
    from paper_2404_01133_b200.render import RenderSettings, project_cloud
    scene, center, radius, alts, wh, _, _ = bench.build_scene("c3", 0, dev, keep_raw=False)
    cams = bench.flythrough(center, radius, alts, wh, 60)
    near = RenderSettings().near_plane
    nb = np.frombuffer(np.float64(near).tobytes(), dtype=np.uint64)[0]
    for i in (0, 10, 30, 50):
        ac = AssembledCloud(scene, cams[i], "block", None, 0, [])
        p = project_cloud(ac, cams[i])
        z = p["depths"]
        zb = z.view(np.uint64)
        k32 = np.minimum((zb - nb) >> np.uint64(24), np.uint64(0xfffffffe))
        for name, k in (("32-bit", k32), ("24-bit", k32 >> np.uint64(8)), ("20-bit", k32 >> np.uint64(12))):
            eq = k[1:] == k[:-1]
            starts = np.flatnonzero(np.diff(np.concatenate([[0], eq.astype(np.int8), [0]])) == 1)
            ends = np.flatnonzero(np.diff(np.concatenate([[0], eq.astype(np.int8), [0]])) == -1)
            lens = ends - starts + 1
            print(f"frame {i} {name}: keys {len(k)} in-runs {int(lens.sum())} runs {len(lens)} "
                  f"max {int(lens.max()) if len(lens) else 0} runs>8 {int((lens > 8).sum())} "
                  f"distinct top bytes {len(np.unique(k >> np.uint64(24 if name == '32-bit' else 16)))}")


if __name__ == "__main__":
    main()
