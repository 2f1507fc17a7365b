# backward box shape (two pixels per lane): C4 train leg
B="--no-cpu-baseline --no-assign --no-modes --no-c12 --no-c5 --no-e2e --steps 5 --warmup 3"
for v in "" "-DCS_BLEND_MINB=2" "-DCS_BLEND_MINB=4" "-DCS_SSIM_TX=32 -DCS_SSIM_TY=16"; do
  CS_NVCC_EXTRA="$v" python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 900 python bench.py $B > gpurun_out/r4l_sweep.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/r4l_sweep.log').read().strip().splitlines()[-1])
t=d['train']; print('[$v]', 'train it/s', round(t['value'],1), {k: round(v,3) for k,v in t['phases_ms'].items()})" || tail -3 gpurun_out/r4l_sweep.log
done
python paper_2404_01133_b200/_build.py --force > /dev/null 2>&1
