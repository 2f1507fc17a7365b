#!/bin/bash
# ncu captures for profiles/: (1) launch list with per-launch durations of a
# short bench run, (2) --set full of every kernel of the timed frames, (3)
# --set full of timed block-training iterations.  The bench brackets its timed
# regions with cudaProfilerStart/Stop when CS_PROFILE_FRAMES / CS_PROFILE_TRAIN
# are set, so --profile-from-start off captures exactly those kernels.
#   bash tools/profile_frame.sh TAG     (SKIP_FRAME=1 / SKIP_TRAIN=1: one half only;
#   each --set full report is 20-45 MB and gpurun returns <= 64 MB per call;
#   REP_DIR=/tmp keeps the reports on the box and returns their summaries)
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
[ "${SKIP_FRAME:-0}" = "1" ] || CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-assign \
  > gpurun_out/${TAG}_launches.log 2>&1
[ "${SKIP_FRAME:-0}" = "1" ] || CS_PROFILE_FRAMES=1 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o ${REP_DIR:-gpurun_out}/${TAG}_frame python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-assign \
  > gpurun_out/${TAG}_frame.log 2>&1
[ "${SKIP_TRAIN:-0}" = "1" ] || CS_PROFILE_TRAIN=1 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o ${REP_DIR:-gpurun_out}/${TAG}_train python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-assign \
  --train-steps 1 --train-warmup 36 > gpurun_out/${TAG}_train.log 2>&1
# REP_DIR=/tmp: reports stay on the box, summaries come back (gpurun returns <= 64 MiB)
if [ -n "${REP_DIR:-}" ]; then
  for k in frame train; do
    [ -f ${REP_DIR}/${TAG}_$k.ncu-rep ] && python tools/ncu_summary.py ${REP_DIR}/${TAG}_$k.ncu-rep \
      gpurun_out/${TAG}_${k}_ncu.md gpurun_out/${TAG}_${k}_traffic.json > gpurun_out/${TAG}_${k}_summary.log 2>&1
  done
fi
ls -la gpurun_out | grep $TAG
