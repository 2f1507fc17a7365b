"""bench.py's algorithmic-work helpers (CPU): the roofline numerators the
bench reports are the per-unit figures DESIGN.md section 4 states, and the
committed ncu capture it cites is the newest one."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_blend_flops_per_unit():
    st = {"evals": 1.0, "fragments": 0.0}
    assert bench.blend_flops(st) == 11.0 and bench.blend_flops32(st) == 12.0
    st = {"evals": 0.0, "fragments": 1.0}
    assert bench.blend_flops(st) == 31.0 and bench.blend_flops32(st) == 17.0


def test_stage_bytes_per_unit():
    one = {"assembled": 1.0, "visible": 0.0, "pairs": 0.0, "sh_bytes_visible": 0.0}
    b = bench.stage_bytes(one)
    assert b["project"] == 60 and b["depth_sort"] == 4 + 64 - 4
    vis = {"assembled": 0.0, "visible": 1.0, "pairs": 0.0, "sh_bytes_visible": 0.0}
    assert bench.stage_bytes(vis)["project"] == 64 + 64 + 8 + 8
    pair = {"assembled": 0.0, "visible": 0.0, "pairs": 1.0, "sh_bytes_visible": 0.0}
    b = bench.stage_bytes(pair)
    assert b["gather_scan"] == 8 and b["tile_sort"] == 4 + 32 and b["ranges"] == 24


def test_newest_traffic_capture_is_cited():
    files = bench._traffic_files()
    assert files, "profiles/*_frame_traffic.json missing"
    tags = [f.name.split("_")[0] for f in files]
    rounds = [int(t[1]) for t in tags]
    assert rounds == sorted(rounds)
    assert tags[-1].startswith("r%d" % max(rounds))
