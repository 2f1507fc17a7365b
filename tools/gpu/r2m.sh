# K3 staged (bulk-copy, persistent) vs direct: parity incl. exclude masks / graphs / full scale, bench-lite
export TESTS="tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_invariance.py tests/test_gpu_assign.py tests/test_gpu_graph.py tests/test_gpu_failures.py"
bash tools/gpu/ab_blend.sh r2m "-DCS_PROJ_STAGED=1" "-DCS_PROJ_STAGED=0"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_c3_fullscale.py -q -x 2>&1 | tail -3
