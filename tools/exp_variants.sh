#!/bin/bash
# Build-time variant sweep: for each -D setting rebuild cs_<FILE>.cu and run the bench.
#   bash tools/exp_variants.sh TAG FILE "BENCH ARGS" "-DX=1" "-DX=2" ...
TAG=$1; FILE=$2; ARGS=$3; shift 3
for V in "$@"; do
  touch paper_2404_01133_b200/csrc/${FILE}.cu
  CS_NVCC_EXTRA="$V" python paper_2404_01133_b200/_build.py > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --no-e2e $ARGS > gpurun_out/${TAG}_var.log 2>&1
  tail -1 gpurun_out/${TAG}_var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
t=d.get('train'); c5=d.get('c5')
print('$V', 'fps', round(d['value'],1), 'stages', {k: round(v,3) for k,v in d['stages_ms'].items()}, 'train', t and round(t['value'],1), t and {k: round(v,3) for k,v in t['phases_ms'].items()})
if c5: print('   c5', round(c5['value'],1), c5.get('stages_ms'))"
done
touch paper_2404_01133_b200/csrc/${FILE}.cu
python paper_2404_01133_b200/_build.py > /dev/null 2>&1
