"""Bundle / PLY loading vs the reference's own
lod.load_lod of a bundle it wrote (tests/golden/bundle/, bundle.npz): every
array identical.  The device-resident load renders like the host path (GPU)."""

import json
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

FIELDS = ("positions", "opacities", "scales", "rotations", "sh")


def test_load_lod_matches_reference(golden_bundle):
    from paper_2404_01133_b200 import bundle
    g = golden_bundle
    scene = bundle.load_lod(GOLDEN / "bundle")
    assert scene.n_levels == int(g["n_levels"]) and scene.n_blocks == int(g["n_blocks"])
    assert np.array_equal(scene.bounds_min, g["bounds_min"]) and np.array_equal(scene.bounds_max, g["bounds_max"])
    assert scene.distance_intervals == tuple(map(tuple, g["intervals"]))
    assert scene.sh_degrees == tuple(int(d) for d in g["sh_degrees"])
    for f in FIELDS:
        assert np.array_equal(getattr(scene.full, f), g[f"full/{f}"]), f
    for l in range(scene.n_levels):
        for j in range(scene.n_blocks):
            for f in FIELDS:
                assert np.array_equal(getattr(scene.levels[l][j], f), g[f"level{l}/block{j}/{f}"]), (l, j, f)


def test_load_errors(tmp_path):
    from paper_2404_01133_b200 import bundle
    with pytest.raises(bundle.DataError):
        bundle.load_lod(tmp_path)
    bad = tmp_path / "x.ply"
    bad.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 0\nend_header\n")
    with pytest.raises(bundle.PlySchemaError):
        bundle.load_ply(bad)
    src = GOLDEN / "bundle"
    dst = tmp_path / "b"
    shutil.copytree(src, dst)
    (dst / "levels" / "1" / "blocks" / "2.ply").unlink()
    with pytest.raises(bundle.DataError):
        bundle.load_lod(dst)
    blob = (src / "full.ply").read_bytes()
    (tmp_path / "trunc.ply").write_bytes(blob[: len(blob) // 2])
    with pytest.raises(bundle.DataError):
        bundle.load_ply(tmp_path / "trunc.ply")


@pytest.mark.gpu
def test_load_lod_device_renders_like_reference(golden_bundle):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200 import bundle
    g = golden_bundle
    dscene = bundle.load_lod_device(GOLDEN / "bundle")
    cam = g.camera("cam")
    a = cs.assemble_render_set(dscene, cam)
    img, st = cs.rasterize_stats(a.cloud, cam)
    assert st.visible_splats == int(g["render/visible"])
    assert st.blended_fragments == int(g["render/fragments"])
    assert np.abs(img.pixels - g["render/image"]).max() <= 1e-4
