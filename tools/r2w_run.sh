timeout 900 python -m pytest tests/test_gpu_blend_fast.py -q -s -x > gpurun_out/r2w_fast.log 2>&1; grep -E "passed|failed|Error|assert" gpurun_out/r2w_fast.log | head -5
bash tools/blend_sweep.sh r2w "-DCS_FAST_MINB=3 -DCS_FAST_PF=1" "-DCS_FAST_MINB=3 -DCS_FAST_PF=2" "-DCS_FAST_MINB=4 -DCS_FAST_PF=1"
