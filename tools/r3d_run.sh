TAG=${1:-r3d}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_tile_local.py tests/test_gpu_parity.py tests/test_gpu_depth_runs.py tests/test_gpu_graph.py tests/test_gpu_failures.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -15 gpurun_out/${TAG}_pytest.log
export CS_TILE_LOCAL=1
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/${TAG}_bench.log
CS_TILE_LOCAL=0 timeout 600 python bench.py $B > gpurun_out/${TAG}_bench_global.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench_global.log').read().strip().splitlines()[-1])
print('global FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 4 --warmup 1 $B > /dev/null 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/${TAG}_launches.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr=rows[h]; iK=hdr.index('Kernel Name'); iV=hdr.index('Metric Value')
d=collections.OrderedDict(); n=collections.Counter()
for r in rows[h+1:]:
    k=r[iK].split('(')[0][:50]; d[k]=d.get(k,0)+float(r[iV].replace(',',''))/1000; n[k]+=1
for k,v in d.items(): print(f"{k:50s} n={n[k]:3d} avg_us={v/n[k]:8.1f}")
PY
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_tl_sort --launch-skip 1 -c 1 -o gpurun_out/${TAG}_tlm \
  python bench.py --steps 2 --warmup 1 $B > gpurun_out/${TAG}_tlm_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_tlm.ncu-rep --page source --csv > gpurun_out/${TAG}_tlm_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_tlm.ncu-rep --page raw --csv > gpurun_out/${TAG}_tlm_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
