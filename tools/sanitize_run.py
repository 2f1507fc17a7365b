"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the hot path on small inputs so the instrumented run
stays short --

* one LoD frame of a 200k-Gaussian 2x2-block city at 640x360 (K1, K3, the
  depth sort + run fix-up, K5+K6, the tile sort, K8, K8b, K9) on the direct
  path, then the same frame asynchronously twice (frame-graph capture + replay);
* one pointwise-LoD frame (lod.py:378-390);
* one training step (cs_render_train -> cs_training_loss -> cs_render_backward
  -> cs_block_adam) of a 20k-Gaussian block at 320x240;
* the LoD build kernels (significance, priority sort, level rows, MAD bounds,
  gather) and the fusion filter.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""

import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_01133_b200 as cs  # noqa: E402
from paper_2404_01133_b200 import device, fusion, lodgen  # noqa: E402
from paper_2404_01133_b200.synth import city_cameras, generate_city, generate_city_torch, orbit_cameras  # noqa: E402
from paper_2404_01133_b200.train import DeviceBlockTrainer  # noqa: E402


def main():
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    pos, op, sc, q, sh = (t.to(dev) for t in generate_city_torch(0, 200.0, 100, 200_000, device="cpu"))
    pmin, pmax = lodgen.central_third(pos)
    mem = lodgen.block_membership(pos, pmin, pmax, (2, 2))
    cams = city_cameras(16, 200.0, 640, 360, seed=0)
    scene = lodgen.build_lod_device(pos, op, sc, q, sh, mem, 4, cams[1:8],
                                    distance_intervals=((0.0, 40.0), (40.0, 80.0), (80.0, math.inf)))
    st = cs.RenderSettings()
    cam = orbit_cameras(pos.double().mean(0).cpu().numpy(), 60.0, 40.0, 4, 640, 360)[1]
    a = cs.assemble_render_set(scene, cam)
    img, stats = cs.rasterize_stats(a.cloud, cam, st)
    for _ in range(3):                     # capture + replay of the frame graph
        cs.render(a.cloud, cam, st)
    torch.cuda.synchronize()
    p = cs.assemble_render_set(scene, cam, mode="pointwise")
    cs.rasterize_stats(p.cloud, cam, st)
    kept = fusion.fuse_filter(pos, pmin, pmax, (2, 2), 1)
    # one training step of a 20k-Gaussian block
    c = generate_city(seed=4, extent=40.0, n_buildings=6, n_gaussians=20_000)
    tcam = city_cameras(8, 40.0, 320, 240, seed=4)[2]
    T = lambda x: torch.tensor(np.asarray(x), dtype=torch.float32, device=dev)
    target = cs.render(c, tcam, st).clone()
    tr = DeviceBlockTrainer(T(c.positions) + 0.02, T(c.scales), T(c.rotations), T(c.opacities), T(c.sh))
    loss = tr.step(tcam, target)
    torch.cuda.synchronize()
    print(f"sanitize run ok: visible={stats.visible_splats} fragments={stats.blended_fragments} "
          f"pointwise={p.cloud.count} fuse_kept={int(kept.numel())} loss={float(loss):.5f}")


if __name__ == "__main__":
    main()
