"""LoD generation on the GPU (cs_significance / cs_priority / cs_lod_rows /
cs_mad_bounds / cs_gather_cloud) vs the reference's golden vectors and the
CPU oracle (needs a B200).

Bar: hit counts, priority order, every level's kept rows and the MAD bounds
bit-exact; significance scores within 4 ulp (the score's volume ** 0.1 is
CUDA's pow, <= 2 ulp from glibc's; everything around it is float64 in numpy
order)."""

import math
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import lodgen_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SCORE_RTOL = 4 * 2.0 ** -52


@pytest.fixture(scope="module")
def lg():
    from paper_2404_01133_b200 import device, lodgen
    return SimpleNamespace(device=device, lodgen=lodgen)


def _dcloud(lg, cloud):
    return lg.device.device_cloud(cloud)


def _check_scores(got, want):
    np.testing.assert_allclose(got, want, rtol=SCORE_RTOL, atol=0)
    assert np.array_equal(got == 0, want == 0)


def test_golden_significance_priority_levels(lg, golden_lodgen):
    g = golden_lodgen
    cloud, cams, mem, nb = lodgen_inputs(g)
    dc = _dcloud(lg, cloud)
    scores, hits = lg.lodgen.significance_scores(dc, cams, return_hits=True)
    _, ohits = O.significance_scores(cloud, cams)
    assert np.array_equal(hits.cpu().numpy(), ohits)
    _check_scores(scores.cpu().numpy(), g["scores"])
    order = lg.lodgen.priority(scores)
    assert np.array_equal(order.cpu().numpy(), g["order"])
    # the reference's own scores through the device ranking as well
    order_ref = lg.lodgen.priority(torch.as_tensor(g["scores"], device=dc.device))
    assert np.array_equal(order_ref.cpu().numpy(), g["order"])
    rates = tuple(reversed(tuple(g["rates"])))
    rows, counts = lg.lodgen.level_rows(order, torch.as_tensor(mem, device=dc.device), nb, rates)
    rows = rows.cpu().numpy()
    for L in range(len(rates)):
        off = 0
        for j in range(nb):
            want = g[f"level{L}/block{j}"]
            assert counts[L, j] == want.size, (L, j)
            assert np.array_equal(rows[L, off:off + want.size], want), (L, j)
            off += want.size


def test_golden_mad_bounds(lg, golden_lodgen):
    g = golden_lodgen
    cloud, _, mem, nb = lodgen_inputs(g)
    dc = _dcloud(lg, cloud)
    bmin, bmax = lg.lodgen.block_bounds(dc, torch.as_tensor(mem, device=dc.device), nb, float(g["n_mad"]))
    assert np.array_equal(bmin, g["bounds_min"]) and np.array_equal(bmax, g["bounds_max"])
    from paper_2404_01133_b200 import lod
    sub = SimpleNamespace(positions=g["positions"][mem == 4], opacities=g["opacities"][mem == 4],
                          scales=g["scales"][mem == 4], rotations=g["rotations"][mem == 4],
                          sh=np.zeros((int((mem == 4).sum()), 3, 1), np.float32))
    lo, hi = lod.mad_bounds(sub, math.inf)
    assert np.array_equal(lo, g["block4_inf_lo"]) and np.array_equal(hi, g["block4_inf_hi"])
    with pytest.raises(ValueError):
        lod.mad_bounds(sub, 0.0)


def test_build_lod_api_matches_golden(lg, golden_lodgen):
    """lod.build_lod with the reference signature: level clouds == golden rows."""
    from paper_2404_01133_b200 import lod
    g = golden_lodgen
    cloud, cams, mem, nb = lodgen_inputs(g)
    grid = SimpleNamespace(membership=mem.astype(np.int64), n_blocks=nb)
    config = SimpleNamespace(compression_rates=tuple(g["rates"]), lod_sh_degrees=tuple(g["sh_degrees"]),
                             n_mad=float(g["n_mad"]),
                             distance_intervals=((0.0, 200.0), (200.0, 400.0), (400.0, math.inf)))
    scene = lod.build_lod(cloud, grid, cams, config)
    assert scene.n_levels == 3 and scene.n_blocks == nb
    assert np.array_equal(scene.bounds_min, g["bounds_min"])
    degrees = tuple(reversed(tuple(g["sh_degrees"])))
    for L in range(3):
        C = (degrees[L] + 1) ** 2
        for j in range(nb):
            rows = g[f"level{L}/block{j}"]
            b = scene.levels[L][j]
            assert np.array_equal(b.positions, cloud.positions[rows].astype(np.float64)), (L, j)
            assert np.array_equal(b.opacities, cloud.opacities[rows].astype(np.float64))
            assert np.array_equal(b.rotations, cloud.rotations[rows].astype(np.float64))
            assert b.sh.shape[2] == C
            assert np.array_equal(b.sh, cloud.sh[rows][:, :, :C].astype(np.float64)), (L, j)
    # compress (lod.py:119-127) = sorted top-k of the priority, SH truncated
    c = lod.compress(cloud, 0.34, 2, cams)
    keep = O.keep_count(0.34, cloud.count)
    rows = np.sort(g["order"][:keep])
    assert np.array_equal(c.positions, cloud.positions[rows].astype(np.float64))
    assert c.sh.shape[2] == 9


def test_city_vs_oracle(lg):
    """A 300k-Gaussian city, 40 views: every decision equal to the oracle."""
    from paper_2404_01133_b200.synth import city_cameras, generate_city
    cloud = generate_city(seed=5, extent=300.0, n_buildings=60, n_gaussians=300_000)
    cams = city_cameras(40, 300.0, 640, 480, seed=5)
    dc = _dcloud(lg, cloud)
    scores, hits = lg.lodgen.significance_scores(dc, cams, return_hits=True)
    want, ohits = O.significance_scores(cloud, cams)
    assert np.array_equal(hits.cpu().numpy(), ohits)
    assert ohits.max() > 5
    _check_scores(scores.cpu().numpy(), want)
    order = lg.lodgen.priority(scores).cpu().numpy()
    assert np.array_equal(order, O.priority(want))
    mem = (np.arange(cloud.count) * 7919 % 5).astype(np.int32)   # 5 interleaved blocks
    mem[mem == 3] = 1                                           # block 3 empty
    rates = (0.25, 0.34, 1.0)
    rows, counts = lg.lodgen.level_rows(torch.as_tensor(order, device=dc.device),
                                        torch.as_tensor(mem, device=dc.device), 5, rates)
    want_rows = O.level_rows(order, mem, 5, tuple(reversed(rates)))
    rows = rows.cpu().numpy()
    for L in range(3):
        cat = np.concatenate(want_rows[L])
        assert np.array_equal(rows[L, :cat.size], cat)
        assert [counts[L, j] for j in range(5)] == [w.size for w in want_rows[L]]
    assert counts[2].sum() == cloud.count and counts[:, 3].sum() == 0
    bmin, bmax = lg.lodgen.block_bounds(dc, torch.as_tensor(mem, device=dc.device), 5, 3.0)
    pos = np.asarray(cloud.positions, dtype=np.float64)
    for j in range(5):
        if (mem == j).any():
            lo, hi = O.mad_bounds(pos[mem == j], 3.0)
            assert np.array_equal(bmin[j], lo) and np.array_equal(bmax[j], hi), j
        else:
            assert not bmin[j].any() and not bmax[j].any()


def test_empty_and_errors(lg):
    from paper_2404_01133_b200 import lod
    empty = SimpleNamespace(positions=np.zeros((0, 3)), opacities=np.zeros(0), scales=np.zeros((0, 3)),
                            rotations=np.zeros((0, 4)), sh=np.zeros((0, 3, 16)), count=0)
    assert lod.significance_scores(empty, []).shape == (0,)
    with pytest.raises(ValueError):
        lod.mad_bounds(empty, 3.0)
    with pytest.raises(ValueError):
        lg.lodgen.keep_count(0.0, 10)
