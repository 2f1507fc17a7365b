# K14 Adam CTA split sweep (training leg, adam phase ms)
B="--no-cpu-baseline --no-assign --no-modes --no-c12 --no-c5 --no-e2e --steps 5 --warmup 3"
for v in "" "-DCS_ADAM_GEOM_DIV=2" "-DCS_ADAM_GEOM_DIV=5" "-DCS_ADAM_GEOM_DIV=8"; do
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py $B > gpurun_out/r4t_sweep.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/r4t_sweep.log').read().strip().splitlines()[-1])
t=d['train']; print('[$v]', 'train', round(t['value'],1), {k: round(v,4) for k,v in t['phases_ms'].items()})" || tail -3 gpurun_out/r4t_sweep.log
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
