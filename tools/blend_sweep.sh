# build variants of the blend and print the C3 blend stage time, longest item and guard counters
#   bash tools/blend_sweep.sh TAG "FLAGS1" "FLAGS2" ...
TAG=$1; shift
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
for v in "$@"; do
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py $B > gpurun_out/${TAG}_sweep.log 2>&1
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[0] if False else 'gpurun_out/' + __import__('os').environ.get('TAG', '') + '_sweep.log').read().strip().splitlines()[-1]) if False else None
PY
  python -c "
import json,sys
d=json.loads(open('gpurun_out/${TAG}_sweep.log').read().strip().splitlines()[-1])
c=d['counts_per_frame']
print('$v', 'FPS', round(d['value'],1), 'blend', round(d['stages_ms']['blend'],3), 'project', round(d['stages_ms']['project'],3), 'longest_us', d['blend_longest_item_us'], 'exact', round(c.get('blend_exact_hits',0)), 'floor', round(c.get('blend_floor_resolved',0)), 'replays', round(c.get('blend_replays',0)))"
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
