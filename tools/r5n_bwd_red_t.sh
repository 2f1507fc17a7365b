#!/bin/bash
# K10 reduction: field-major float rows, 33-float stride (CS_BWD_RED_T=1) vs row-major (=0):
# gradient tests with variant 1, then the training leg A/B twice each
B="--no-cpu-baseline --no-e2e --no-c5 --no-c12 --no-modes --no-assign"
CS_NVCC_EXTRA="-DCS_BWD_RED_T=1" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || echo "build failed"
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_backward_scale.py tests/test_gpu_train.py -q > gpurun_out/r5n_pytest.log 2>&1; tail -1 gpurun_out/r5n_pytest.log
for V in 1 0 1 0; do
  CS_NVCC_EXTRA="-DCS_BWD_RED_T=$V" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r5n_var.log 2>&1
  tail -1 gpurun_out/r5n_var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); t=d['train']
print('RED_T=$V', 'fps', round(d['value'],1), 'train', round(t['value'],1), {k: round(v,4) for k,v in t['phases_ms'].items()})"
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
