#!/bin/bash
# One GPU call: build + smoke, GPU tests, bench (+ optional ncu capture of one kernel).
#   BENCH_ARGS="--no-cpu-baseline" bash tools/gpu_round.sh TAG [KERNEL_REGEX]
# Logs: gpurun_out/{smoke,pytest,bench}_TAG.log; the last lines are echoed.
TAG=${1:-run}
KREGEX=${2:-}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1
grep -E "passed|failed|error" gpurun_out/pytest_${TAG}.log | tail -3
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.log 2>&1
tail -1 gpurun_out/bench_${TAG}.log | python -c "
import json, sys
line = sys.stdin.readline()
try:
    d = json.loads(line)
    print('FPS', round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1) if d.get('e2e') else None,
          'stages', {k: round(v, 3) for k, v in d['stages_ms'].items()})
    if d.get('train'):
        print('train', round(d['train']['value'], 1), {k: round(v, 3) for k, v in d['train']['phases_ms'].items()})
except Exception as e:
    print('bench output not JSON:', line[:300])
"
if [ -n "$KREGEX" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" --launch-skip 2 -c 1 \
    -o gpurun_out/${TAG}_kernel python bench.py --steps 3 --warmup 0 --no-cpu-baseline --no-e2e --no-train \
    > gpurun_out/ncu_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}.log
fi
