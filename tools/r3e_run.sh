TAG=${1:-r3e}
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1])
print('FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
CS_NVCC_EXTRA="-DCS_EXP_NO_HOT" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
timeout 600 python bench.py $B > gpurun_out/${TAG}_bench_nohot.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench_nohot.log').read().strip().splitlines()[-1])
print('NO-HOT FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
for K in k_onesweep k_bin_pairs k_fix_short_runs k_project_staged; do
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:$K -c 1 -o gpurun_out/${TAG}_$K \
  python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_$K.ncu-rep --page source --csv > gpurun_out/${TAG}_${K}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_$K.ncu-rep
done
ls -la gpurun_out | grep ${TAG}
