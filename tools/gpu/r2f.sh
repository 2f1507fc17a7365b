# A/B blend: round-1 kernel file vs current (cp.async / bulk), same scene; backward-at-scale detail; reference suite
cp paper_2404_01133_b200/csrc/cs_blend.cu /tmp/cs_blend_cur.cu
cp tools/gpu/cs_blend_r1.cu paper_2404_01133_b200/csrc/cs_blend.cu
bash tools/gpu/ab_blend.sh r2f_r1 ""
cp /tmp/cs_blend_cur.cu paper_2404_01133_b200/csrc/cs_blend.cu
bash tools/gpu/ab_blend.sh r2f_cur "-DCS_BLEND_BULK=0" "-DCS_BLEND_BULK=1"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
python -m pytest tests/test_gpu_backward_scale.py -q -s -k 1080p 2>&1 | grep -v "^    \|^$" | tail -60 > gpurun_out/r2f_bwd.log
python -m pytest tests/test_gpu_failures.py -q 2>&1 | tail -5
bash tools/ref_suite/run.sh r2f
