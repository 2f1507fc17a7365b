python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-e2e"
timeout 600 python bench.py $B > gpurun_out/r3y_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/r3y_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'c5', round(d['c5']['value'],1), 'c1', round(d['c1']['value'],1), 'c2', round(d['c2']['value'],1), {k: round(v,4) for k,v in d['counts_per_frame'].items() if 'blend_' in k})"
