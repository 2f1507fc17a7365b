#!/bin/bash
# End-of-milestone capture: smoke, all GPU tests, default bench line, reference
# arm, ncu launch list and --set full of the timed frames.  Training capture:
#   SKIP_FRAME=1 bash tools/profile_frame.sh TAG   (a separate gpurun call:
#   each report is 20-45 MB and gpurun returns <= 64 MB per call).
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-300
REP_DIR=/tmp SKIP_TRAIN=1 bash tools/profile_frame.sh ${TAG} > /dev/null 2>&1
ls gpurun_out | grep ${TAG}
