"""CPU oracle for LoD generation pinned against the
reference's own outputs (tests/golden/lodgen.npz, made by
tests/golden/make_golden.py from citysplat.lod under the Sandybridge pin):
significance scores bit-exact, priority order, per-level kept rows and MAD
bounds identical."""

import math

import numpy as np

from conftest import lodgen_inputs
from oracle import oracle as O


def test_oracle_significance_scores_bitexact(golden_lodgen):
    cloud, cams, _, _ = lodgen_inputs(golden_lodgen)
    scores, hits = O.significance_scores(cloud, cams)
    assert np.array_equal(scores, golden_lodgen["scores"])
    assert hits.max() > 0 and (hits == 0).any()


def test_oracle_priority_and_levels(golden_lodgen):
    g = golden_lodgen
    order = O.priority(g["scores"])
    assert np.array_equal(order, g["order"])
    rows = O.level_rows(order, g["membership"], int(g["n_blocks"]), g["rates"])
    for L in range(len(rows)):
        for j in range(int(g["n_blocks"])):
            assert np.array_equal(rows[L][j], g[f"level{L}/block{j}"]), (L, j)
    # duplicated Gaussians (rows 20000+) tie with their originals: the original ranks first
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    dup = np.arange(0, 20_000, 40)
    assert (rank[dup] < rank[20_000 + np.arange(dup.size)]).all()


def test_oracle_mad_bounds(golden_lodgen):
    g = golden_lodgen
    mem = g["membership"]
    pos = g["positions"].astype(np.float64)
    for j in range(int(g["n_blocks"])):
        lo, hi = O.mad_bounds(pos[mem == j], float(g["n_mad"]))
        assert np.array_equal(lo, g["bounds_min"][j]) and np.array_equal(hi, g["bounds_max"][j])
    lo, hi = O.mad_bounds(pos[mem == 4], math.inf)
    assert np.array_equal(lo, g["block4_inf_lo"]) and np.array_equal(hi, g["block4_inf_hi"])


def test_oracle_build_lod_matches_golden(golden_lodgen):
    """oracle.build_lod (the reference arm's host LoD build, lod.py:211-248)
    reproduces the golden level rows and MAD bounds end to end."""
    g = golden_lodgen
    cloud, cams, mem, J = lodgen_inputs(g)
    rates = tuple(float(r) for r in g["rates"])
    degrees = tuple(int(d) for d in g["sh_degrees"])
    scene = O.build_lod(cloud, mem, J, cams, ((0.0, 1.0),) * len(rates), rates, degrees,
                        float(g["n_mad"]))
    pos = np.asarray(cloud.positions)
    for L in range(len(rates)):
        width = min((degrees[::-1][L] + 1) ** 2, 16)
        for j in range(J):
            rows = g[f"level{L}/block{j}"]
            assert np.array_equal(scene.levels[L][j].positions, pos[rows]), (L, j)
            assert scene.levels[L][j].sh.shape == (rows.size, 3, width)
    assert np.array_equal(scene.bounds_min, g["bounds_min"])
    assert np.array_equal(scene.bounds_max, g["bounds_max"])
