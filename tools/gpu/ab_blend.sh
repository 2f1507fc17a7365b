# A/B of blend variants: parity tests + bench-lite (headline + stages) per CS_NVCC_EXTRA setting
#   bash tools/gpu/ab_blend.sh TAG "<flags A>" "<flags B>" ...   (PARITY=0 skips the tests)
tag=$1; shift
LITE="--steps 20 --warmup 5 --no-modes --no-c5 --no-train --no-assign --no-cpu-baseline --no-e2e --no-c12"
for v in "$@"; do
  name=$(echo "$v" | tr -c 'A-Za-z0-9=_\n' '_')
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  r=""
  if [ "${PARITY:-1}" = "1" ]; then
    r=$(python -m pytest -q ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_invariance.py} 2>&1 | tail -1)
  fi
  timeout 600 python bench.py $LITE > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err
  python - "$v" "$r" "gpurun_out/${tag}_$name.json" <<'PY'
import json, sys
v, r, f = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(v, "|", r, "|", round(d["value"], 1), {k: round(x, 4) for k, x in d["stages_ms"].items()},
          "fragments/frame", round(d["counts_per_frame"]["fragments"]))
except Exception as e:
    print(v, "|", r, "| bench failed", e)
PY
done
