#!/bin/bash
# End-of-milestone capture: smoke, all GPU tests, default bench line, ncu launch list,
# --set full captures of one frame and one training iteration.   bash tools/round_capture.sh TAG
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-300
bash tools/profile_frame.sh ${TAG} > /dev/null 2>&1
ls gpurun_out | grep ${TAG}
