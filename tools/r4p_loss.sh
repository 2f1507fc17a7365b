# K13 register-sliding SSIM: parity tests + training leg

timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_metrics.py tests/test_gpu_backward.py tests/test_gpu_backward_scale.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-assign --no-modes --no-c12 --no-c5 --no-e2e > gpurun_out/r4p_bench.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/r4p_bench.log').read().strip().splitlines()[-1])
t=d['train']; print('FPS', round(d['value'],1), 'train', round(t['value'],1), {k: round(v,4) for k,v in t['phases_ms'].items()})"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_project_bwd|k_adam' -c 6 --csv --log-file gpurun_out/r4p_launches.csv python bench.py --no-cpu-baseline --no-assign --no-modes --no-c12 --no-c5 --no-e2e --steps 2 --warmup 1 --train-steps 2 --train-warmup 1 > /dev/null 2>&1
grep -o '"k_[a-z_]*(.*' gpurun_out/r4p_launches.csv | awk -F'","' '{print $1, $NF}' | cut -c1-20,200-
