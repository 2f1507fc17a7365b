# r1 blend + KEEP float64 sums; float64 backward partials; lazy assembly; backward-at-scale detail; suites
python -m pytest tests/test_gpu_backward_scale.py -q -s 2>&1 | grep -v "^    \|^$" | tail -40 > gpurun_out/r2g_bwd.log
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_backward_scale.py 2>&1 | tail -15 > gpurun_out/r2g_pytest.log
bash tools/ref_suite/run.sh r2g
LITE="--steps 20 --warmup 5 --no-modes --no-c5 --no-assign --no-cpu-baseline --no-e2e --no-c12"
timeout 900 python bench.py $LITE > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['stages_ms'], d['train']['phases_ms'], d['train']['value'])"
tail -3 gpurun_out/r2g_bwd.log gpurun_out/r2g_pytest.log
