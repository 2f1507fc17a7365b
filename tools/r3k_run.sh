python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_blend_fast.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python tools/blend_views.py gpurun_out/r3k_views_fast.json 2>&1 | head -5
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-e2e"
timeout 600 python bench.py $B > gpurun_out/r3k_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/r3k_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'c5', round(d['c5']['value'],1), d['c5']['stages_ms']['blend'])"
