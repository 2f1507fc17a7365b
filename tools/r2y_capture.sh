# bench (stages), launch list, one-kernel ncu of the fast blend, summaries made on the box
TAG=${1:-r2y}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
python - <<PY
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))
print('stages', {k: round(v,3) for k,v in d['stages_ms'].items()})
print('counts', {k: round(v/1e6,3) for k,v in d['counts_per_frame'].items()})
print('roofline', json.dumps(d['roofline'])[:600])
print('alt', json.dumps(d['altitudes'])[:900])
print('c1', d['c1']['value'], 'c2', d['c2']['value'], 'c5', d['c5']['value'], 'train', d['train']['value'], d['train']['phases_ms'])
PY
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-assign --no-modes --no-c12 --no-c5 > /dev/null 2>&1
bash tools/ncu_kernel.sh ${TAG} k_blend_fast
python tools/ncu_summary.py gpurun_out/${TAG}_kernel.ncu-rep gpurun_out/${TAG}_blend_ncu.md gpurun_out/${TAG}_blend_traffic.json > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_kernel.ncu-rep --page raw --csv > gpurun_out/${TAG}_blend_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_kernel.ncu-rep --page source --csv > gpurun_out/${TAG}_blend_source.csv 2>/dev/null
du -sh gpurun_out/*
