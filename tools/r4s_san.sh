# compute-sanitizer over the hot path (incl. the certified blend K9f) after the round-2 changes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/r4s_san_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/r4s_san_$t.log
done
