# certified float32 blend: first GPU pass (ex2 accuracy, new tests, full GPU suite, bench)
TAG=${1:-r2p}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ex2_check tools/ex2_check.cu && /tmp/ex2_check > gpurun_out/${TAG}_ex2_check.txt 2>&1; cat gpurun_out/${TAG}_ex2_check.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_blend_fast.py -q -s -x > gpurun_out/${TAG}_fast.log 2>&1; grep -E "fragments|passed|failed|Error|assert" gpurun_out/${TAG}_fast.log | head -20
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest.log 2>&1; tail -5 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}); print(d.get('counts_per_frame'))"
