# full GPU suite, full default bench + reference arm, compute-sanitizer over the sanitize workload
python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2j_pytest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2j_ref.json 2> gpurun_out/r2j_ref.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2j_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2j_sanitize_summary.txt
  tail -3 gpurun_out/r2j_sanitize_$tool.log >> gpurun_out/r2j_sanitize_summary.txt
done
cat gpurun_out/r2j_pytest.log gpurun_out/r2j_sanitize_summary.txt; tail -c 600 gpurun_out/r2j_bench.err
