"""CPU oracle for training-data assignment pinned against
the reference's own outputs (tests/golden/assign.npz, made by
tests/golden/make_golden.py from citysplat.partition.assign): entries,
provenance and the enlarged bounds identical, contribution l_ssim within 1e-9."""

import numpy as np

from conftest import assign_inputs
from oracle import oracle as O


def test_oracle_contracted_matches_reference(golden_assign):
    g = golden_assign
    c = O.contract_normalized(g["positions"].astype(np.float64), g["p_min"], g["p_max"])
    assert np.array_equal(c, g["contracted"])


def test_oracle_assign_matches_golden(golden_assign):
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    entries, prov, bmin, bmax, l = O.assign(views, grid, cloud, float(g["epsilon"]), st,
                                            float(g["scale"]), int(g["min_count"]))
    fin = np.isfinite(g["l_ssim"])
    assert np.array_equal(fin, np.isfinite(l))
    np.testing.assert_allclose(l[fin], g["l_ssim"][fin], atol=1e-9, rtol=0)
    assert np.array_equal(entries, g["entries"])
    assert np.array_equal(prov, g["provenance"])
    assert np.array_equal(bmin, g["bounds_min_used"]) and np.array_equal(bmax, g["bounds_max_used"])
