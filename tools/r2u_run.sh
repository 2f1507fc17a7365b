timeout 900 python -m pytest tests/test_gpu_blend_fast.py -q -s -x > gpurun_out/r2u_fast.log 2>&1; grep -E "fragments|passed|failed|Error|assert" gpurun_out/r2u_fast.log | head -20
bash tools/blend_sweep.sh r2u "-DCS_FAST_MINB=3 -DCS_FAST_PF=1" "-DCS_FAST_MINB=3 -DCS_FAST_PF=2" "-DCS_FAST_MINB=3 -DCS_FAST_PF=3" "-DCS_FAST_MINB=4 -DCS_FAST_PF=2" "-DCS_FAST_MINB=2 -DCS_FAST_PF=4"
