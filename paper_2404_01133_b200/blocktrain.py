"""Block-parallel training workload (BASELINE.json configs[3]).

The paper's divide-and-conquer fine-tuning: the scene is split
into a 6x6 grid of blocks (grid_partition membership, partition.py:208-231),
every block is optimised independently on its own views, and the trained
blocks are fused back with the membership rule of partition.fuse
(partition.py:570-587).  Here:

* blocks are assigned to ranks by LPT on their sizes (train.lpt_assign); a
  rank runs its blocks round-robin, one block iteration = forward render of
  one 1080p view of that block + loss + backward + Adam (train.BlockTrainer);
* there is no gradient exchange: the only collective is the fused-cloud
  all-gather after training (fusion.fuse_all_gather, NCCL over NVLink);
* ground truth = the device-tier render of the unperturbed full scene from the
  block's views (synthetic data; no dataset on the box), the trained
  parameters start from the block's Gaussians with seeded position noise.
"""

from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np
import torch

from . import device
from .render import RenderSettings, render
from .synth import orbit_cameras
from .train import BlockTrainer, DeviceBlockTrainer, lpt_assign


class BlockJob:
    """One block: its trainer, views and target images (all in HBM)."""

    def __init__(self, j: int, trainer: BlockTrainer, cams, targets: List[torch.Tensor]):
        self.j, self.trainer, self.cams, self.targets = j, trainer, cams, targets
        self.iters = 0

    @property
    def count(self) -> int:
        return int(self.trainer.activated()[0].shape[0])

    def fusion_inputs(self):
        """(positions, opacities, scales, rotations, sh) as fusion.fuse_all_gather takes them."""
        p, s, q, o, sh = (t.detach() for t in self.trainer.activated())
        return p, o, s, q, sh

    def step(self) -> torch.Tensor:
        v = self.iters % len(self.cams)
        self.iters += 1
        return self.trainer.step(self.cams[v], self.targets[v])


def block_views(pos_block: torch.Tensor, n_views: int, width: int, height: int,
                altitude: float = 150.0) -> list:
    """Orbit views around the block's centroid (cmd_bench's sweep shape,
    cli.py:203-218), radius from the block's horizontal spread."""
    p = pos_block.double()
    center = p.mean(dim=0).cpu().numpy()
    spread = float(p[:, :2].std(dim=0).max().item()) if p.shape[0] > 1 else 10.0
    radius = min(max(1.5 * spread, 40.0), 400.0)
    return orbit_cameras(center, radius, altitude, n_views, width, height)


def setup_blocks(pos, op, sc, q, sh, membership: torch.Tensor, owned: Sequence[int], width: int,
                 height: int, n_views: int = 4, noise: float = 0.05, seed: int = 0,
                 settings: RenderSettings = None, trainer_cls=DeviceBlockTrainer) -> Dict[int, BlockJob]:
    """Build the BlockJobs this rank owns from the full scene tensors."""
    settings = settings or RenderSettings()
    full = device.DeviceCloud.from_torch(pos, op, sc, q, sh)
    g = torch.Generator(device=pos.device)
    g.manual_seed(seed)
    jobs = {}
    for j in owned:
        idx = torch.nonzero(membership == j).squeeze(1)
        if idx.numel() == 0:
            continue
        cams = block_views(pos[idx], n_views, width, height)
        targets = [render(full, cam, settings, sync=True).clone() for cam in cams]
        p0 = pos[idx] + noise * torch.randn(pos[idx].shape, generator=g, device=pos.device)
        tr = trainer_cls(p0, sc[idx], q[idx], op[idx], sh[idx], settings=settings)
        jobs[j] = BlockJob(j, tr, cams, targets)
    del full
    return jobs


def assign_blocks(membership: torch.Tensor, n_blocks: int, world: int) -> List[int]:
    counts = torch.bincount(membership.long(), minlength=n_blocks).cpu().tolist()
    return lpt_assign(counts, world)


def block_counts(membership: torch.Tensor, n_blocks: int) -> List[int]:
    return torch.bincount(membership.long(), minlength=n_blocks).cpu().tolist()
