#!/bin/bash
# final capture of the round's last kernels: smoke, all GPU tests, default
# bench line, reference arm, training ncu (--set full, summarised on the box)
TAG=r5h
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-200
REP_DIR=/tmp SKIP_FRAME=1 bash tools/profile_frame.sh ${TAG} > /dev/null 2>&1
grep -E "k_blend_bwd|k_blend<|k_adam|k_ssim" gpurun_out/${TAG}_train_ncu.md
