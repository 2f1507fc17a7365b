#!/bin/bash
# One --set full capture (with source) of the first launch of kernel KREGEX
# inside the bench's timed frames:  bash tools/ncu_kernel.sh TAG KREGEX [extra bench args]
TAG=$1; KREGEX=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"$KREGEX" -c 1 -o gpurun_out/${TAG}_kernel \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-assign --no-modes --no-c12 --no-c5 "$@" \
  > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
