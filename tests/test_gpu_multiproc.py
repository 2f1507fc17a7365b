"""Two ranks on one B200 (gloo carries the CUDA tensors): the LoD scene built
on rank 0 reaches rank 1 through fusion.broadcast_device_lod_scene and renders
bit-identically there (needs a GPU; the NCCL path on an 8-GPU box runs the
same code with backend "nccl")."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2404_01133_b200 as cs
        from paper_2404_01133_b200 import fusion, lodgen
        from paper_2404_01133_b200.synth import city_cameras, generate_city_torch
        dev = torch.device("cuda", 0)
        scene = None
        if rank == 0:
            pos, op, sc, qq, sh = generate_city_torch(3, 200.0, 40, 150_000, device=dev)
            pmin, pmax = lodgen.central_third(pos)
            mem = lodgen.block_membership(pos, pmin, pmax, (3, 3))
            cams = city_cameras(16, 200.0, 320, 240, seed=3)
            scene = lodgen.build_lod_device(pos, op, sc, qq, sh, mem, 9, cams[1:],
                                            distance_intervals=((0.0, 40.0), (40.0, 80.0), (80.0, np.inf)))
        scene = fusion.broadcast_device_lod_scene(scene, src=0)
        cam = city_cameras(16, 200.0, 320, 240, seed=3)[5]
        a = cs.assemble_render_set(scene, cam)
        img, st = cs.rasterize_stats(a.cloud, cam)
        q.put((rank, img.pixels, st.visible_splats, st.blended_fragments, scene.counts.copy()))
    finally:
        dist.destroy_process_group()


def test_lod_broadcast_renders_identically():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, *rest = q.get(timeout=300)
        got[r] = rest
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got[0][3], got[1][3])
    assert got[0][1] == got[1][1] > 0 and got[0][2] == got[1][2]
    assert np.array_equal(got[0][0], got[1][0])
