set -x
python -m pytest tests/test_gpu_failures.py -x -q 2>&1 | tail -30 > gpurun_out/r2b_failures.log
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c3_fullscale.py 2>&1 | tail -30 > gpurun_out/r2b_pytest.log
timeout 1500 python -m pytest tests/test_gpu_c3_fullscale.py -x -q -s 2>&1 | tail -40 > gpurun_out/r2b_c3full.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
tail -3 gpurun_out/r2b_failures.log gpurun_out/r2b_pytest.log gpurun_out/r2b_c3full.log; tail -c 600 gpurun_out/r2b_bench.err
