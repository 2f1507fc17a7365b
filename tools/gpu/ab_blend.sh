# A/B of blend variants: bench-lite (headline + stages) per CS_NVCC_EXTRA setting
tag=$1; shift
LITE="--steps 20 --warmup 5 --no-modes --no-c5 --no-train --no-assign --no-cpu-baseline --no-e2e --no-c12"
for v in "$@"; do
  name=$(echo "$v" | tr -c 'A-Za-z0-9=_\n' '_')
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  timeout 600 python bench.py $LITE > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/${tag}_$name.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), {k: round(v,4) for k,v in d['stages_ms'].items()})" 2>&1 | tail -1
done
