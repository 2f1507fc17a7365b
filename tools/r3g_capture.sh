# round-2 milestone capture: smoke, GPU tests, default bench, reference arm,
# launch list, --set full of the timed frames (summarised on the box)
TAG=${1:-r4z}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
python - <<PY
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'])
print('stages', {k: round(v,3) for k,v in d['stages_ms'].items()})
r=d['roofline']; print('roof', r['kernel'], round(r['frac'],3), round(r['achieved'],2), r.get('fp32'))
print('c1', round(d['c1']['value'],1), 'c2', round(d['c2']['value'],1), 'c5', round(d['c5']['value'],1), 'train', round(d['train']['value'],1), d['train']['phases_ms'])
print('alt', {a: {m: (v['mean_fps'], v['min_fps']) for m, v in x.items()} for a, x in d['altitudes'].items()})
print('parity', [ (f['frame'], f['decisions_bit_exact'], f['tile_lists_bit_exact'], f['image_max_abs_err']) for f in d['cpu_baseline']['parity']['frames']])
PY
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-200
SKIP_TRAIN=1 timeout 1500 bash tools/profile_frame.sh ${TAG} > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_frame.ncu-rep gpurun_out/${TAG}_frame_ncu.md gpurun_out/${TAG}_frame_traffic.json > /dev/null 2>&1
rm -f gpurun_out/${TAG}_frame.ncu-rep
du -sh gpurun_out/${TAG}*
