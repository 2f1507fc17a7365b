# fast blend v2: tests, bench (MINB=4), A/B MINB=3
TAG=${1:-r2r}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_blend_fast.py -q -s -x > gpurun_out/${TAG}_fast.log 2>&1; grep -E "fragments|passed|failed|Error|assert" gpurun_out/${TAG}_fast.log | head -20
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench4.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench4.log').read().strip().splitlines()[-1])
print('MINB4 FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, d['counts_per_frame'], d['blend_longest_item_us'])"
CS_NVCC_EXTRA="-DCS_FAST_MINB=3" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench3.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench3.log').read().strip().splitlines()[-1])
print('MINB3 FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, d['blend_longest_item_us'])"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest.log 2>&1; tail -4 gpurun_out/${TAG}_pytest.log
