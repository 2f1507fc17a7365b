# round-2 GPU batch: new parity/failure/invariance/backward tests, full suite, bench, reference arm
python -m pytest tests/test_gpu_failures.py tests/test_gpu_invariance.py tests/test_gpu_backward_scale.py -q -s 2>&1 | tail -40 > gpurun_out/r2c_new.log
python -m pytest tests -m gpu -q --deselect tests/test_gpu_c3_fullscale.py 2>&1 | tail -30 > gpurun_out/r2c_pytest.log
timeout 1500 python -m pytest tests/test_gpu_c3_fullscale.py -q -s -k full_cloud 2>&1 | tail -30 > gpurun_out/r2c_c3full.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
tail -5 gpurun_out/r2c_new.log gpurun_out/r2c_pytest.log gpurun_out/r2c_c3full.log; tail -c 1500 gpurun_out/r2c_bench.err
