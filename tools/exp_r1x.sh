#!/bin/bash
# blend counter change + sort profile
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/x_smoke.log 2>&1; tail -1 gpurun_out/x_smoke.log
timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e > gpurun_out/x_bench.log 2>&1
tail -1 gpurun_out/x_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/sort_bench.cu -o /tmp/sb
/tmp/sb > gpurun_out/x_sort.log 2>&1; cat gpurun_out/x_sort.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_onesweep -c 8 -o gpurun_out/x_sort /tmp/sb prof > gpurun_out/x_sort_ncu.log 2>&1
tail -2 gpurun_out/x_sort_ncu.log
