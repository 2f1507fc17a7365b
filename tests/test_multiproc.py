"""World-size-2 CPU (gloo) tests of the multi-GPU host logic.

* fusion.fuse_all_gather: each rank filters the blocks it owns (membership
  from the C oracle here, the CUDA kernel on the box), the kept rows are
  exchanged block-ordered; every rank must end with rows byte-identical to
  the CPU fuse() of all blocks (partition.py:570-587), for the golden 9-block
  fusion fixture and LPT and round-robin ownership.
* lpt_assign / the bench's view split: deterministic, balanced, complete.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, owner, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2404_01133_b200 import fusion
        g = np.load(os.path.join(HERE, "golden", "fuse.npz"))
        pmin, pmax, dims = g["p_min"], g["p_max"], tuple(int(d) for d in g["dims"])
        n_blocks = int(np.prod(dims))
        local = {}
        C = 0
        for j in range(n_blocks):
            if owner[j] != rank or f"block{j}/positions" not in g:
                continue
            t = lambda k: torch.from_numpy(np.ascontiguousarray(g[f"block{j}/{k}"]))
            local[j] = (t("positions"), t("opacities"), t("scales"), t("rotations"), t("sh"))
            C = int(g[f"block{j}/sh"].shape[2])
        Cs = [0] * world
        dist.all_gather_object(Cs, C)
        C = max(Cs)
        filt = lambda pos, j: torch.from_numpy(
            np.nonzero(O.block_of_points(pos.numpy(), pmin, pmax, dims) == j)[0])
        fused = fusion.fuse_all_gather(local, n_blocks, owner, pmin, pmax, dims, sh_coeffs=C, filter_fn=filt,
                                       dtype=torch.float64, device="cpu")
        result_q.put((rank, fused.numpy()))
    finally:
        dist.destroy_process_group()


def _expected():
    from oracle import oracle as O
    from paper_2404_01133_b200 import fusion
    g = np.load(os.path.join(HERE, "golden", "fuse.npz"))
    pmin, pmax, dims = g["p_min"], g["p_max"], tuple(int(d) for d in g["dims"])
    from types import SimpleNamespace
    blocks = []
    for j in range(int(np.prod(dims))):
        if f"block{j}/positions" in g:
            blocks.append((SimpleNamespace(**{k: g[f"block{j}/{k}"] for k in
                                              ("positions", "opacities", "scales", "rotations", "sh")}), j))
    ref = O.fuse(blocks, pmin, pmax, dims)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    return fusion.pack_rows(t(ref.positions), t(ref.opacities), t(ref.scales), t(ref.rotations), t(ref.sh)).numpy()


@pytest.mark.parametrize("policy", ["lpt", "round_robin", "idle_rank"])
def test_fuse_all_gather_gloo_world2(policy):
    """LPT and round-robin ownership over 2 ranks; "idle_rank": 3 ranks where
    rank 2 owns no block (it must still join the collectives, with the agreed
    dtype/device, and end with the same bytes)."""
    from paper_2404_01133_b200.train import lpt_assign
    g = np.load(os.path.join(HERE, "golden", "fuse.npz"))
    n_blocks = int(np.prod(g["dims"]))
    sizes = [int(g[f"block{j}/positions"].shape[0]) if f"block{j}/positions" in g else 0 for j in range(n_blocks)]
    world = 3 if policy == "idle_rank" else 2
    owner = lpt_assign(sizes, 2) if policy in ("lpt", "idle_rank") else [j % 2 for j in range(n_blocks)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, owner, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _expected()
    for r in range(world):
        assert got[r].shape == want.shape
        assert got[r].tobytes() == want.tobytes(), r


def test_lpt_assign_balanced_and_deterministic():
    from paper_2404_01133_b200.train import lpt_assign
    rng = np.random.default_rng(0)
    sizes = rng.integers(300_000, 1_000_000, 36).tolist()
    for n in (1, 2, 4, 8):
        own = lpt_assign(sizes, n)
        assert own == lpt_assign(sizes, n) and set(own) <= set(range(n)) and len(own) == 36
        loads = [sum(s for s, o in zip(sizes, own) if o == r) for r in range(n)]
        assert max(loads) <= sum(sizes) / n + max(sizes)   # LPT bound
        if n == 8:
            assert max(loads) / (sum(sizes) / n) < 1.15


def test_view_split_covers_flythrough():
    # bench.py: rank r renders frames i with i * world // n == r (contiguous, complete, disjoint)
    for n_frames in (60, 740):
        for world in (1, 2, 4, 8):
            shares = [[i for i in range(n_frames) if i * world // n_frames == r] for r in range(world)]
            assert sorted(sum(shares, [])) == list(range(n_frames))
            assert max(map(len, shares)) - min(map(len, shares)) <= 1


def _lod_levels_from_golden():
    """(levels, table) of the golden 2x2x3 LoD city in the device layout, on CPU."""
    g = np.load(os.path.join(HERE, "golden", "city.npz"))
    L, J = int(g["n_levels"]), int(g["n_blocks"])
    levels, counts = [], np.zeros((L, J), dtype=np.int64)
    for lvl in range(L):
        pos, op, sc, rot, sh = [], [], [], [], []
        for j in range(J):
            p = f"level{lvl}/block{j}/"
            pos.append(g[p + "positions"]); op.append(g[p + "opacities"]); sc.append(g[p + "scales"])
            rot.append(g[p + "rotations"]); sh.append(g[p + "sh"])
            counts[lvl, j] = g[p + "positions"].shape[0]
        K = int(counts[lvl].sum())
        q = np.zeros((3, K, 4), dtype=np.float32)
        q[0, :, :3] = np.concatenate(pos); q[0, :, 3] = np.concatenate(op)
        q[1, :, :3] = np.concatenate(sc); q[2] = np.concatenate(rot)
        shc = np.concatenate(sh).astype(np.float32)
        C = shc.shape[2]
        stride = (3 * C + 3) // 4 * 4
        rows = np.zeros((K, stride), dtype=np.float32)
        rows[:, :3 * C] = shc.reshape(K, 3 * C)
        levels.append((torch.from_numpy(q), torch.from_numpy(rows), C))
    table = dict(counts=counts, bounds_min=g["bounds_min"], bounds_max=g["bounds_max"],
                 intervals=np.array(g["intervals"], dtype=np.float64), sh_degrees=g["sh_degrees"])
    return levels, table


def _lod_worker(rank, world, port, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_01133_b200 import fusion
        if rank == 0:
            levels, table = _lod_levels_from_golden()
            out = fusion.broadcast_lod(levels, table, src=0, device="cpu")
        else:
            out = fusion.broadcast_lod(None, None, src=0, device="cpu")
        levels, table = out
        result_q.put((rank, [(q.numpy(), sh.numpy(), C) for q, sh, C in levels],
                      {k: np.asarray(v) for k, v in table.items()}))
    finally:
        dist.destroy_process_group()


def test_lod_table_broadcast_gloo_world2():
    """fusion.broadcast_lod: the LoD levels + table built on rank 0 arrive byte-identical on rank 1."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lod_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, lv, tb = q.get(timeout=120)
        got[r] = (lv, tb)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_levels, want_table = _lod_levels_from_golden()
    for r in range(2):
        lv, tb = got[r]
        assert len(lv) == len(want_levels)
        for (q_, sh, C), (wq, wsh, wC) in zip(lv, want_levels):
            assert C == wC and q_.tobytes() == wq.numpy().tobytes() and sh.tobytes() == wsh.numpy().tobytes()
        for k, v in want_table.items():
            assert np.array_equal(tb[k], np.asarray(v)), k
