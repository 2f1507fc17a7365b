# final check of HEAD: build + smoke, the whole GPU suite, the default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; tail -1 gpurun_out/final_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'gpu_launches', d['gpu_launches'], 'clocks', d['clocks'], 'c5', round(d['c5']['value'],1), 'train', round(d['train']['value'],1))"
