#!/bin/bash
# The reference's own hot-path tests on the B200 through the drop-in shim, and
# the same files on the reference's CPU path (no shim) for comparison.
# Output: gpurun_out/<tag>_ref_suite_{shim,cpu}.log
tag=${1:-r2}
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
cd "$ROOT"
export PYTHONPATH="$ROOT/baseline/_ref:$ROOT/baseline/_ref/citysplat_tests:$ROOT:$ROOT/tools/ref_suite"
FILES="test_render.py test_lod.py test_acceptance.py"
cd baseline/_ref/citysplat_tests
timeout 1800 python -m pytest -p cs_shim -p no:cacheprovider $FILES -rA -q 2>&1 | tail -150 > "$ROOT/gpurun_out/${tag}_ref_suite_shim.log"
timeout 1800 python -m pytest -p no:cacheprovider $FILES -q 2>&1 | tail -15 > "$ROOT/gpurun_out/${tag}_ref_suite_cpu.log"
tail -3 "$ROOT/gpurun_out/${tag}_ref_suite_shim.log" "$ROOT/gpurun_out/${tag}_ref_suite_cpu.log"
