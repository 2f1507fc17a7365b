#!/bin/bash
# ncu captures for profiles/: (1) launch list with per-launch durations of a
# short bench run, (2) --set full of every kernel of one C3 frame, (3) --set
# full of one block-training iteration.   bash tools/profile_frame.sh TAG
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
FRAME='k_lod_select|k_project|k_radix_hist|k_onesweep|k_pair_count|k_duplicate|k_tile_ranges|k_tile_order|k_blend'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$FRAME" -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-e2e --no-train \
  > gpurun_out/${TAG}_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$FRAME" --launch-skip 22 -c 22 \
  -o gpurun_out/${TAG}_frame python bench.py --steps 2 --warmup 0 --no-cpu-baseline --no-e2e --no-train \
  > gpurun_out/${TAG}_frame.log 2>&1
TRAIN='k_project|k_blend|k_ssim|k_adam|k_project_bwd|k_blend_bwd'
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$TRAIN" --launch-skip 400 -c 9 \
  -o gpurun_out/${TAG}_train python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  --train-steps 2 --train-warmup 40 > gpurun_out/${TAG}_train.log 2>&1
ls -la gpurun_out | grep $TAG
