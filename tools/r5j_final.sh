#!/bin/bash
# final check of HEAD: smoke, all GPU tests, default bench line
TAG=${1:-r5j}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'c5', round(d['c5']['value'],1), 'c2', round(d['c2']['value'],1), 'c1', round(d['c1']['value'],1), 'train', round(d['train']['value'],1), d['train']['phases_ms'], 'clocks', d['clocks'])"
