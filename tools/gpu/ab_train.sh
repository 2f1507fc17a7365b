# A/B of backward precision variants: gradient-at-scale tests + training phases (bench-lite with the train leg)
tag=$1; shift
LITE="--steps 4 --warmup 2 --no-modes --no-c5 --no-assign --no-cpu-baseline --no-e2e --no-c12"
for v in "$@"; do
  name=$(echo "$v" | tr -c 'A-Za-z0-9=_\n' '_')
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  r=$(python -m pytest tests/test_gpu_backward_scale.py -q 2>&1 | grep -E "AssertionError: \(|passed|failed" | tail -2 | tr "\n" " ")
  timeout 600 python bench.py $LITE > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/${tag}_$name.json').read().strip().splitlines()[-1]); t=d['train']; print('$v', '| $r |', round(t['value'],1), {k: round(v,3) for k,v in t['phases_ms'].items()})" 2>&1 | tail -1
done
