#!/bin/bash
# NCCL world-of-one test, the whole GPU suite, then two more default bench runs (run-to-run spread)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5f_smoke.log 2>&1; tail -1 gpurun_out/r5f_smoke.log
timeout 600 python -m pytest tests/test_gpu_nccl.py -q -x > gpurun_out/r5f_nccl.log 2>&1; tail -3 gpurun_out/r5f_nccl.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r5f_pytest.log 2>&1; tail -1 gpurun_out/r5f_pytest.log
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/r5f_bench_$i.log 2>&1
  tail -1 gpurun_out/r5f_bench_$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('run $i', 'FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'c5', round(d['c5']['value'],1), 'c2', round(d['c2']['value'],1), 'c1', round(d['c1']['value'],1), 'train', round(d['train']['value'],1), 'clocks', d['clocks'])"
done
