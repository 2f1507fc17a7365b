python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-assign --no-modes --no-c12 --no-c5"
CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_project_staged -c 1 -o gpurun_out/r3z_k3 python bench.py $B > /dev/null 2>&1
ncu -i gpurun_out/r3z_k3.ncu-rep --page source --csv > gpurun_out/r3z_k3_source.csv 2>/dev/null
ncu -i gpurun_out/r3z_k3.ncu-rep --page source --csv --print-source cuda > gpurun_out/r3z_k3_cuda.csv 2>/dev/null
ncu -i gpurun_out/r3z_k3.ncu-rep --page raw --csv > gpurun_out/r3z_k3_raw.csv 2>/dev/null
rm -f gpurun_out/r3z_k3.ncu-rep
ls -la gpurun_out | grep r3z
