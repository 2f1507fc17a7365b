bash tools/ncu_kernel.sh r2q k_blend_fast
CS_BLEND_EXACT=1 timeout 600 python bench.py --no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e > gpurun_out/r2q_bench_exact.log 2>&1
tail -1 gpurun_out/r2q_bench_exact.log | cut -c1-300
python -c "
import json
d=json.loads(open('gpurun_out/r2q_bench_exact.log').read().strip().splitlines()[-1])
print('exact kernel:', d['stages_ms'])"
