#!/bin/bash
# K10 shared-memory transpose of the nine float64 partials (CS_BWD_RED_SMEM): smoke + GPU tests, then the
# training leg A/B (CS_BWD_RED_SMEM=1 / 0, twice each)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5g_smoke.log 2>&1; tail -1 gpurun_out/r5g_smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5g_pytest.log 2>&1; tail -1 gpurun_out/r5g_pytest.log
B="--no-cpu-baseline --no-e2e --no-c5 --no-c12 --no-modes --no-assign"
for V in 1 0 1 0; do
  CS_NVCC_EXTRA="-DCS_BWD_RED_SMEM=$V" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r5g_var.log 2>&1
  tail -1 gpurun_out/r5g_var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); t=d['train']
print('RED_SMEM=$V', 'fps', round(d['value'],1), 'train', round(t['value'],1), {k: round(v,4) for k,v in t['phases_ms'].items()})"
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
