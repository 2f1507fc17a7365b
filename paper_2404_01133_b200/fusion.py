"""Block fusion (partition.fuse, partition.py:570-587) on the device.

``fuse_device`` keeps, from each fine-tuned block cloud j, the rows whose
contracted position still bins into block j (K12 cs_fuse_filter: the
normalize -> contract -> bin chain in float64 numpy order, stable
compaction), and concatenates the kept rows in ascending block order -- the
same bytes as the CPU ``fuse``.

``fuse_all_gather`` is the multi-GPU form used after block-parallel training
(SURVEY.md section 8e): every rank filters the blocks it owns on its own GPU,
the per-block kept counts are summed with one all-reduce, and the kept rows are
exchanged with one all-gather (padded to the largest rank) and placed in
ascending block order on the device (an all-gather-v), so every rank ends
with the byte-identical fused cloud.
"""

from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np
import torch

from . import _lib, device
from ._lib import check
from .core import pad_sh


def _dims3(dims):
    dims = tuple(int(d) for d in dims)
    return dims + (1,) if len(dims) == 2 else dims


def fuse_filter(positions: torch.Tensor, p_min, p_max, dims, block: int) -> torch.Tensor:
    """Ascending row indices (device int64) of `positions` that bin into `block`."""
    nx, ny, nz = _dims3(dims)
    pos = positions.contiguous()
    f32 = 1 if pos.dtype == torch.float32 else 0
    if not f32:
        pos = pos.double().contiguous()
    n = pos.shape[0]
    kept = torch.empty(max(n, 1), dtype=torch.int64, device=pos.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=pos.device)
    pmin = np.ascontiguousarray(p_min, dtype=np.float64)
    pmax = np.ascontiguousarray(p_max, dtype=np.float64)
    check(_lib.load().cs_fuse_filter(device.context(pos.device.index), n, pos.data_ptr(), f32,
                                     pmin.ctypes.data, pmax.ctypes.data, nx, ny, nz, int(block),
                                     kept.data_ptr(), cnt.data_ptr(),
                                     device.stream_handle(pos.device)), "fuse_filter")
    return kept[: int(cnt.item())]


class FusedArrays:
    def __init__(self, positions, opacities, scales, rotations, sh):
        self.positions, self.opacities, self.scales = positions, opacities, scales
        self.rotations, self.sh = rotations, sh

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


def fuse_device(block_clouds: Sequence, p_min, p_max, dims) -> FusedArrays:
    """partition.fuse with the membership test on the GPU; host arrays out."""
    n_blocks = int(np.prod(_dims3(dims)))
    pieces = []
    dev = torch.device("cuda", device._device_index())
    for cloud, j in sorted(block_clouds, key=lambda item: item[1]):
        if not 0 <= j < n_blocks:
            raise ValueError(f"block index {j} outside the grid")
        pos = np.asarray(cloud.positions, dtype=np.float64)
        if pos.shape[0] == 0:
            continue
        idx = fuse_filter(torch.from_numpy(np.ascontiguousarray(pos)).to(dev), p_min, p_max, dims, j)
        if idx.numel():
            rows = idx.cpu().numpy()
            pieces.append([np.asarray(getattr(cloud, f))[rows]
                           for f in ("positions", "opacities", "scales", "rotations", "sh")])
    if not pieces:
        return FusedArrays(np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros((0, 4)),
                           np.zeros((0, 3, 16)))
    width = max(p[4].shape[2] for p in pieces)
    return FusedArrays(*(np.concatenate([p[i] for p in pieces]) for i in range(4)),
                       np.concatenate([pad_sh(p[4], width) for p in pieces]))


# ---------------------------------------------------------------------------
# multi-GPU fusion: all-gather-v in block order

PARAM_WIDTH_NOSH = 3 + 1 + 3 + 4  # positions, opacity, scales, rotations


def pack_rows(positions, opacities, scales, rotations, sh) -> torch.Tensor:
    """Rows as one contiguous float tensor [n, 11 + 3C] for a single collective."""
    n = positions.shape[0]
    return torch.cat([positions.reshape(n, 3), opacities.reshape(n, 1), scales.reshape(n, 3),
                      rotations.reshape(n, 4), sh.reshape(n, -1)], dim=1).contiguous()


def unpack_rows(rows: torch.Tensor, sh_coeffs: int):
    n = rows.shape[0]
    return (rows[:, 0:3], rows[:, 3], rows[:, 4:7], rows[:, 7:11],
            rows[:, 11:11 + 3 * sh_coeffs].reshape(n, 3, sh_coeffs))


def fuse_all_gather(local_blocks: Dict[int, Tuple[torch.Tensor, ...]], n_blocks: int, owner: List[int],
                    p_min, p_max, dims, sh_coeffs: int, group=None, filter_fn=None,
                    dtype: torch.dtype = None, device=None) -> torch.Tensor:
    """Fuse block clouds trained on different ranks.

    local_blocks: {block j: (positions, opacities, scales, rotations, sh)} for the
    blocks this rank owns (owner[j] == rank).  Returns the fused rows
    [N, 11 + 3C] on every rank, blocks in ascending order, rows within a block
    in ascending index order (partition.py:578-587).  ``filter_fn`` defaults to
    the CUDA membership filter; tests on CPU ranks pass the oracle's.

    The row dtype and device must agree on every rank: pass ``dtype`` and
    ``device`` explicitly (required on a rank that owns no rows -- e.g. more
    ranks than occupied blocks -- otherwise taken from its own blocks).

    Exchange: one all-reduce of the per-block kept counts, then ONE all-gather
    of every rank's kept rows (its blocks in ascending order, padded to the
    largest rank's row count), after which each rank places the blocks in
    ascending block order with one device gather -- the all-gather-v of
    SURVEY.md 8e as a single collective instead of one broadcast per block.
    """
    import torch.distributed as dist
    filter_fn = filter_fn or (lambda pos, j: fuse_filter(pos, p_min, p_max, dims, j))
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    some = next(iter(local_blocks.values()))[0] if local_blocks else None
    if dtype is None or device is None:
        if some is None:
            raise ValueError("fuse_all_gather: a rank without blocks needs explicit dtype and device")
        dtype = dtype or some.dtype
        device = device or some.device
    dev = torch.device(device)
    width = PARAM_WIDTH_NOSH + 3 * sh_coeffs
    counts = torch.zeros(n_blocks, dtype=torch.int64, device=dev)
    pieces = []
    for j in sorted(local_blocks):
        if owner[j] != rank:
            raise ValueError(f"rank {rank} does not own block {j}")
        params = local_blocks[j]
        idx = filter_fn(params[0], j)
        rows = pack_rows(*(p[idx] for p in params)).to(device=dev, dtype=dtype)
        if rows.shape[1] != width:
            raise ValueError(f"block {j}: rows of width {rows.shape[1]}, expected {width} (sh_coeffs)")
        pieces.append(rows)
        counts[j] = rows.shape[0]
    dist.all_reduce(counts, group=group)             # owners fill their slots
    counts_h = counts.cpu().tolist()
    per_rank = [0] * world
    for j in range(n_blocks):
        per_rank[owner[j]] += counts_h[j]
    cap = max(max(per_rank), 1)
    mine = torch.zeros((cap, width), dtype=dtype, device=dev)
    if pieces:
        cat = torch.cat(pieces)
        mine[:cat.shape[0]] = cat
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)     # the one data collective
    flat = torch.cat(gathered)                       # [world * cap, width]
    # row index of every fused row: block j's rows sit in its owner's buffer after
    # the owner's lower-numbered blocks
    cursor = [0] * world
    index = []
    for j in range(n_blocks):
        n = counts_h[j]
        if n == 0:
            continue
        r = owner[j]
        index.append(torch.arange(r * cap + cursor[r], r * cap + cursor[r] + n, device=dev))
        cursor[r] += n
    if not index:
        return torch.empty((0, width), dtype=dtype, device=dev)
    return flat.index_select(0, torch.cat(index))


# ---------------------------------------------------------------------------
# LoD table broadcast (SURVEY.md 8e "LoD table"): the source rank's detail
# levels and table reach every rank through one broadcast per tensor, so a
# single rank runs the LoD build (lodgen.build_lod_cloud) for the whole box.

_HDR = 4  # n_levels, n_blocks, fp64, reserved


def broadcast_lod(levels, table, src: int = 0, group=None, device=None):
    """Broadcast LoD level tensors and table from ``src``.

    levels: on src, a list of (quads (3, K_L, 4), sh rows (K_L, stride_L),
    sh_coeffs) per level; table: on src, dict(counts (L, J) int64,
    bounds_min/bounds_max (J, 3), intervals (L, 2), sh_degrees (L,)).  Other
    ranks pass None and receive both (tensors on ``device``).
    """
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else (
        levels[0][0].device if levels else torch.device("cpu"))
    hdr = torch.zeros(_HDR, dtype=torch.int64, device=dev)
    if rank == src:
        hdr[0], hdr[1] = len(levels), int(np.asarray(table["counts"]).shape[1])
        hdr[2] = 1 if levels[0][0].dtype == torch.float64 else 0
    dist.broadcast(hdr, src=src, group=group)
    L, J, fp64 = int(hdr[0]), int(hdr[1]), bool(hdr[2])
    # the table: per level (count, sh_coeffs, stride) + counts, then the float64 part
    itab = torch.zeros(L * 3 + L * J, dtype=torch.int64, device=dev)
    ftab = torch.zeros(J * 6 + L * 3, dtype=torch.float64, device=dev)
    if rank == src:
        for i, (q, sh, C) in enumerate(levels):
            itab[3 * i], itab[3 * i + 1], itab[3 * i + 2] = q.shape[1], int(C), sh.shape[1]
        itab[3 * L:] = torch.as_tensor(np.asarray(table["counts"], dtype=np.int64).reshape(-1))
        f = np.concatenate([np.asarray(table["bounds_min"], dtype=np.float64).reshape(-1),
                            np.asarray(table["bounds_max"], dtype=np.float64).reshape(-1),
                            np.asarray(table["intervals"], dtype=np.float64).reshape(-1),
                            np.asarray(table["sh_degrees"], dtype=np.float64).reshape(-1)])
        ftab.copy_(torch.as_tensor(f))
    dist.broadcast(itab, src=src, group=group)
    dist.broadcast(ftab, src=src, group=group)
    it = itab.cpu().numpy()
    ft = ftab.cpu().numpy()
    out_levels = []
    for i in range(L):
        K, C, stride = int(it[3 * i]), int(it[3 * i + 1]), int(it[3 * i + 2])
        if rank == src:
            q, sh = levels[i][0].contiguous(), levels[i][1].contiguous()
        else:
            q = torch.empty((3, K, 4), dtype=torch.float64 if fp64 else torch.float32, device=dev)
            sh = torch.empty((K, stride), dtype=torch.float32, device=dev)
        if K:
            dist.broadcast(q, src=src, group=group)
            dist.broadcast(sh, src=src, group=group)
        out_levels.append((q, sh, C))
    out_table = dict(counts=it[3 * L:].reshape(L, J),
                     bounds_min=ft[:3 * J].reshape(J, 3), bounds_max=ft[3 * J:6 * J].reshape(J, 3),
                     intervals=ft[6 * J:6 * J + 2 * L].reshape(L, 2),
                     sh_degrees=ft[6 * J + 2 * L:].astype(np.int64))
    return out_levels, out_table


def broadcast_device_lod_scene(dscene, src: int = 0, group=None):
    """A DeviceLodScene on every rank from the one built on ``src`` (others pass None)."""
    import torch.distributed as dist
    from . import device as _device
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == src:
        levels = [(torch.stack([lc.pos_op, lc.scale, lc.quat]), lc.sh, lc.sh_coeffs)
                  for lc in dscene.level_clouds]
        table = dict(counts=dscene.counts, bounds_min=dscene.bounds_min, bounds_max=dscene.bounds_max,
                     intervals=np.array(dscene.distance_intervals, dtype=np.float64),
                     sh_degrees=np.array(dscene.sh_degrees))
        broadcast_lod(levels, table, src, group, dev)
        return dscene
    levels, table = broadcast_lod(None, None, src, group, dev)
    clouds = [_device.DeviceCloud(q[0], q[1], q[2], sh, C, q.shape[1]) for q, sh, C in levels]
    return _device.DeviceLodScene.from_device_levels(
        clouds, table["counts"], table["bounds_min"], table["bounds_max"],
        [tuple(r) for r in table["intervals"]], tuple(int(d) for d in table["sh_degrees"]), dev.index)
