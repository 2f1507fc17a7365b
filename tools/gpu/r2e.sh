# blend: exact alpha + bulk-copy staging vs cp.async staging; backward tests; reference suite via shim
bash tools/gpu/ab_blend.sh r2e "-DCS_BLEND_BULK=1" "-DCS_BLEND_BULK=0"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
python -m pytest tests/test_gpu_backward_scale.py tests/test_gpu_backward.py tests/test_gpu_parity.py tests/test_gpu_failures.py -q -s 2>&1 | tail -25 > gpurun_out/r2e_pytest.log
tail -4 gpurun_out/r2e_pytest.log
bash tools/ref_suite/run.sh r2e
