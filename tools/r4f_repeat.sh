# run-to-run spread of the default bench line on one box (three back-to-back runs)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r4f_bench_$i.log 2>&1
  tail -1 gpurun_out/r4f_bench_$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('run $i FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'blend', round(d['stages_ms']['blend'],3), 'c5', round(d['c5']['value'],1), 'c2', round(d['c2']['value'],1), 'c1', round(d['c1']['value'],1), 'train', round(d['train']['value'],1), 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
