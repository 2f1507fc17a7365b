#!/bin/bash
# GPU tests with the warp-aggregated k_tile_order, then a k_tile_ranges
# cache-hint sweep (CS_RANGES_HINT 0/1/2, twice each; frame-only bench), then
# the block-training ncu capture summarised on the box (the report itself
# stays there: gpurun returns <= 64 MiB).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5b_smoke.log 2>&1; tail -1 gpurun_out/r5b_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r5b_pytest.log 2>&1; tail -1 gpurun_out/r5b_pytest.log
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
for V in 0 1 2 0 1 2; do
  CS_NVCC_EXTRA="-DCS_RANGES_HINT=$V" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r5b_var.log 2>&1
  tail -1 gpurun_out/r5b_var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d['stages_ms']
print('HINT=$V', 'fps', round(d['value'],1), 'ranges', round(s['ranges'],4), 'tile_sort', round(s['tile_sort'],4), 'blend', round(s['blend'],4))"
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
CS_PROFILE_TRAIN=1 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o /tmp/r5b_train python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-assign \
  --train-steps 1 --train-warmup 36 > gpurun_out/r5b_train.log 2>&1
python tools/ncu_summary.py /tmp/r5b_train.ncu-rep gpurun_out/r5b_train_ncu.md gpurun_out/r5b_train_traffic.json > gpurun_out/r5b_summary.log 2>&1
head -40 gpurun_out/r5b_train_ncu.md
