# onesweep build-flag sweep on the C3 bench (depth_sort / tile_sort stage times)
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
for v in "" "-DCS_FIX_GRID_MULT=16" "-DCS_FIX_GRID_MULT=40" "-DCS_FIX_GRID_MULT=4"; do
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r4n_sweep.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/r4n_sweep.log').read().strip().splitlines()[-1])
print('[$v]', 'FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items() if k in ('depth_sort',)})" || tail -3 gpurun_out/r4n_sweep.log
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
