python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/blend_views.py gpurun_out/r3i_views_fast.json 2>&1 | tail -20
CS_BLEND_EXACT=1 timeout 900 python tools/blend_views.py gpurun_out/r3i_views_exact.json 2>&1 | tail -20
timeout 300 python -m pytest tests/test_gpu_primitive.py -q 2>&1 | tail -2
