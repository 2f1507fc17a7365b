python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--steps 8 --warmup 2 --no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  --csv --log-file gpurun_out/r3n_launches_warm.csv python bench.py $B > gpurun_out/r3n_bench_under_ncu.log 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/r3n_launches_warm.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr=rows[h]; iK=hdr.index('Kernel Name'); iV=hdr.index('Metric Value')
d=collections.OrderedDict(); n=collections.Counter(); tot=0
for r in rows[h+1:]:
    k=r[iK].split('(')[0][:50]; v=float(r[iV].replace(',',''))/1000; d[k]=d.get(k,0)+v; n[k]+=1; tot+=v
frames=n['k_lod_select']
for k,v in d.items(): print(f"{k:50s} n={n[k]:3d} avg_us={v/n[k]:8.1f}")
print('frames', frames, 'sum of kernel us per frame', round(tot/frames,1))
PY
