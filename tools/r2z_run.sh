TAG=${1:-r2z}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/tile_stats.py > gpurun_out/${TAG}_tiles.log 2>&1; tail -22 gpurun_out/${TAG}_tiles.log
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
timeout 300 python -m pytest tests/test_gpu_depth_runs.py -q -x 2>&1 | tail -2
