# ncu: launch list of the timed frames + --set full (with source) of one timed frame; backward flakiness x3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; tail -1 gpurun_out/r2l_smoke.log
for i in 1 2 3; do python -m pytest tests/test_gpu_backward_scale.py -q 2>&1 | grep -E "Error|passed|failed" | tail -3; done > gpurun_out/r2l_bwd_repeat.log
LITE="--no-cpu-baseline --no-e2e --no-train --no-assign --no-modes --no-c5 --no-c12"
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/r2l_launches.csv python bench.py --steps 20 --warmup 2 $LITE > gpurun_out/r2l_launches.log 2>&1
CS_PROFILE_FRAMES=1 timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o gpurun_out/r2l_frame python bench.py --steps 1 --warmup 1 $LITE > gpurun_out/r2l_frame.log 2>&1
ls -la gpurun_out | grep r2l; cat gpurun_out/r2l_bwd_repeat.log
