# backward 1080p detail; blend v1 vs v2 A/B (parity + bench-lite); racecheck re-run
python -m pytest tests/test_gpu_backward_scale.py -q -s -k 1080p 2>&1 | grep -v "^    \|^$" | tail -30 > gpurun_out/r2k_bwd.log
bash tools/gpu/ab_blend.sh r2k "" "-DCS_BLEND_V2=1" "-DCS_BLEND_V2=1 -DCS_BLEND2_BATCH=16" "-DCS_BLEND_V2=1 -DCS_BLEND2_THREADS=256 -DCS_BLEND2_MINB=2"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2k_sanitize_racecheck.log 2>&1
tail -3 gpurun_out/r2k_sanitize_racecheck.log; tail -12 gpurun_out/r2k_bwd.log
