#!/bin/bash
# quick check: smoke, gpu tests, frame bench (no cpu baseline / train / e2e)
TAG=${1:-q}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-c5 ${BENCH_ARGS:---no-train} > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, {k: round(v/1e6,2) for k,v in d['counts_per_frame'].items()}, d['train'] and (round(d['train']['value'],1), {k: round(v,3) for k,v in d['train']['phases_ms'].items()}))"
