python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_depth_runs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
for i in 1 2; do
timeout 600 python bench.py $B > gpurun_out/r3p_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/r3p_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
