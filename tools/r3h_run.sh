# training-step profile: launch list of timed training iterations + one k_blend_bwd --set full
TAG=${1:-r3h}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-assign --no-modes --no-c12 --no-c5"
CS_PROFILE_TRAIN=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_train_launches.csv python bench.py $B --train-steps 2 --train-warmup 36 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/${TAG}_train_launches.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr=rows[h]; iK=hdr.index('Kernel Name'); iV=hdr.index('Metric Value')
d=collections.OrderedDict(); n=collections.Counter()
for r in rows[h+1:]:
    k=r[iK].split('(')[0][:50]; d[k]=d.get(k,0)+float(r[iV].replace(',',''))/1000; n[k]+=1
for k,v in d.items(): print(f"{k:50s} n={n[k]:3d} avg_us={v/n[k]:8.1f}")
PY
CS_PROFILE_TRAIN=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_blend_bwd -c 1 -o gpurun_out/${TAG}_bwd python bench.py $B --train-steps 1 --train-warmup 36 > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_bwd.ncu-rep --page source --csv > gpurun_out/${TAG}_bwd_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_bwd.ncu-rep --page raw --csv > gpurun_out/${TAG}_bwd_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_bwd.ncu-rep
ls -la gpurun_out | grep $TAG
