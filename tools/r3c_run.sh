TAG=${1:-r3c}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_blend_fast.py tests/test_gpu_tile_local.py tests/test_gpu_parity.py tests/test_gpu_invariance.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -15 gpurun_out/${TAG}_pytest.log
B="--no-cpu-baseline --no-train --no-assign --no-modes --no-c12 --no-c5 --no-e2e"
CS_TILE_LOCAL=0 timeout 600 python bench.py $B > gpurun_out/${TAG}_bench_global.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench_global.log').read().strip().splitlines()[-1])
print('global FPS', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, {k: round(v/1e6,3) for k,v in d['counts_per_frame'].items()}, d['blend_longest_item_us'])"
CS_TILE_LOCAL=0 bash tools/ncu_kernel.sh ${TAG} k_blend_fast
python tools/ncu_summary.py gpurun_out/${TAG}_kernel.ncu-rep gpurun_out/${TAG}_blend_ncu.md > /dev/null 2>&1; cat gpurun_out/${TAG}_blend_ncu.md
ncu -i gpurun_out/${TAG}_kernel.ncu-rep --page source --csv > gpurun_out/${TAG}_blend_source.csv 2>/dev/null
bash tools/ncu_kernel.sh ${TAG}_tlm "k_tl_sort<256"
ncu -i gpurun_out/${TAG}_tlm_kernel.ncu-rep --page source --csv > gpurun_out/${TAG}_tlm_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_tlm_kernel.ncu-rep --page raw --csv > gpurun_out/${TAG}_tlm_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
