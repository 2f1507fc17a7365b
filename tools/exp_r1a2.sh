#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/sort_bench.cu -o /tmp/sb
/tmp/sb > gpurun_out/a2_sort.log 2>&1; cat gpurun_out/a2_sort.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/a2_pytest.log 2>&1; tail -1 gpurun_out/a2_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e > gpurun_out/a2_bench.log 2>&1
tail -1 gpurun_out/a2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
