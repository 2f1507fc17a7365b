#!/bin/bash
# One GPU call: build, GPU tests, bench (+ optional ncu capture of one kernel).
#   bash tools/gpu_round.sh TAG [KERNEL_REGEX]
TAG=${1:-run}
KREGEX=${2:-}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-3000
if [ -n "$KREGEX" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" --launch-skip 2 -c 1 \
    -o gpurun_out/${TAG}_kernel python bench.py --steps 3 --warmup 0 --no-cpu-baseline --no-e2e --no-train \
    > gpurun_out/ncu_${TAG}.log 2>&1
  tail -3 gpurun_out/ncu_${TAG}.log
fi
