# onesweep build-flag sweep on the C3 bench (depth_sort / tile_sort stage times)
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
for v in "" "-DCS_PROJ_MINB=2" "-DCS_PROJ_THREADS=512 -DCS_PROJ_MINB=1"; do
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r4o_sweep.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/r4o_sweep.log').read().strip().splitlines()[-1])
print('[$v]', 'FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items() if k in ('project',)})" || tail -3 gpurun_out/r4o_sweep.log
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
