# guarded-alpha blend + bulk-copy staging + float64 backward sums: full GPU suite, bench, blend ncu
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2d_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-c12 --no-assign > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
tail -5 gpurun_out/r2d_pytest.log; tail -c 1500 gpurun_out/r2d_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r2d_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['stages_ms'], d['counts_per_frame'], d.get('train',{}).get('phases_ms'), d['cpu_baseline']['parity']['ok'] if d.get('cpu_baseline') else None, d.get('altitudes'))"
