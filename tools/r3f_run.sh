TAG=${1:-r3f}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${TAG}_pytest.log 2>&1; tail -4 gpurun_out/${TAG}_pytest.log
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, {k: round(v,4) for k,v in d['counts_per_frame'].items() if 'blend_' in k})"
