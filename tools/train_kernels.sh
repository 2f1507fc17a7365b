#!/bin/bash
# Per-kernel durations (ncu launch list) of block-training iterations.
TAG=${1:-tk}
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_project_bwd|k_blend_bwd|k_adam|k_ssim|k_blend<float, 1" \
  --launch-skip 100 -c 60 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-assign \
  --train-steps 8 --train-warmup 36 > gpurun_out/${TAG}_train_launches.csv 2>&1
python - "$TAG" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_train_launches.csv")) if len(r) > 10]
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, rows = rows[h], rows[h:]
iN = hdr.index("Kernel Name"); iV = hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    try: d[r[iN].split("(")[0]].append(float(r[iV].replace(",", "")))
    except ValueError: pass
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v)/1000:8.1f} us")
PY
