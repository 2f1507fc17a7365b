"""The multi-GPU exchanges on the NCCL backend, executed on the
one B200 of the test box as a world of one rank: fusion.fuse_all_gather
(all-reduce of the kept counts + one all-gather of the rows) with the CUDA
membership filter, and fusion.broadcast_device_lod_scene, both through
torch.distributed's "nccl" process group on CUDA tensors.  The world-size-2
logic of the same functions is covered on gloo (tests/test_multiproc.py);
this checks that the NCCL calls themselves (CUDA-only tensors, dtype/device
agreement, the padded all-gather) run and give the reference's bytes."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(port, q):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        import paper_2404_01133_b200 as cs
        from paper_2404_01133_b200 import fusion, lodgen
        from paper_2404_01133_b200.synth import city_cameras, generate_city_torch
        out = {"backend": dist.get_backend()}
        # fusion all-gather with the CUDA membership filter (fuse_filter)
        g = np.load(os.path.join(HERE, "golden", "fuse.npz"))
        pmin, pmax, dims = g["p_min"], g["p_max"], tuple(int(d) for d in g["dims"])
        n_blocks = int(np.prod(dims))
        local, C = {}, 0
        for j in range(n_blocks):
            if f"block{j}/positions" not in g:
                continue
            t = lambda k: torch.from_numpy(np.ascontiguousarray(g[f"block{j}/{k}"])).to(dev)
            local[j] = (t("positions"), t("opacities"), t("scales"), t("rotations"), t("sh"))
            C = int(g[f"block{j}/sh"].shape[2])
        fused = fusion.fuse_all_gather(local, n_blocks, [0] * n_blocks, pmin, pmax, dims, sh_coeffs=C,
                                       dtype=torch.float64, device=dev)
        out["fused_device"] = str(fused.device)
        out["fused"] = fused.cpu().numpy()
        # LoD scene broadcast, then a render of the received scene
        pos, op, sc, qq, sh = generate_city_torch(3, 200.0, 40, 60_000, device=dev)
        p0, p1 = lodgen.central_third(pos)
        mem = lodgen.block_membership(pos, p0, p1, (3, 3))
        cams = city_cameras(12, 200.0, 320, 240, seed=5)
        scene = lodgen.build_lod_device(pos, op, sc, qq, sh, mem, 9, cams[1:],
                                        distance_intervals=((0.0, 40.0), (40.0, 80.0), (80.0, np.inf)))
        got = fusion.broadcast_device_lod_scene(scene, src=0)
        imgs = []
        for sc_ in (scene, got):
            a = cs.assemble_render_set(sc_, cams[4])
            img, st = cs.rasterize_stats(a.cloud, cams[4])
            imgs.append((img.pixels, st.visible_splats, st.blended_fragments))
        out["renders"] = imgs
        out["counts"] = (np.asarray(scene.counts).copy(), np.asarray(got.counts).copy())
        q.put(out)
    finally:
        dist.destroy_process_group()


def _expected_fused():
    from oracle import oracle as O
    from paper_2404_01133_b200 import fusion
    from types import SimpleNamespace
    g = np.load(os.path.join(HERE, "golden", "fuse.npz"))
    pmin, pmax, dims = g["p_min"], g["p_max"], tuple(int(d) for d in g["dims"])
    blocks = []
    for j in range(int(np.prod(dims))):
        if f"block{j}/positions" in g:
            blocks.append((SimpleNamespace(**{k: g[f"block{j}/{k}"] for k in
                                              ("positions", "opacities", "scales", "rotations", "sh")}), j))
    ref = O.fuse(blocks, pmin, pmax, dims)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    return fusion.pack_rows(t(ref.positions), t(ref.opacities), t(ref.scales), t(ref.rotations), t(ref.sh)).numpy()


def test_nccl_fusion_all_gather_and_lod_broadcast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert out["backend"] == "nccl"
    assert out["fused_device"].startswith("cuda")
    want = _expected_fused()
    assert out["fused"].shape == want.shape
    assert out["fused"].tobytes() == want.tobytes()
    (a_img, a_vis, a_frag), (b_img, b_vis, b_frag) = out["renders"]
    np.testing.assert_array_equal(out["counts"][0], out["counts"][1])
    assert a_vis == b_vis and a_frag == b_frag and a_vis > 0
    assert np.asarray(a_img).tobytes() == np.asarray(b_img).tobytes()
