K=k_adam
timeout 900 ncu --set full --clock-control none -k regex:"$K" -s 1 -c 1 -o gpurun_out/r4s_$K python bench.py --no-cpu-baseline --no-assign --no-modes --no-c12 --no-c5 --no-e2e --steps 2 --warmup 1 --train-steps 2 --train-warmup 1 > gpurun_out/r4s_$K.log 2>&1
ncu -i gpurun_out/r4s_$K.ncu-rep --page details > gpurun_out/r4s_${K}_details.txt
rm -f gpurun_out/r4s_$K.ncu-rep
grep -E " Duration|DRAM Throughput|Memory Throughput|Issued Instructions  |Achieved Active|L2 Hit|Registers Per" gpurun_out/r4s_${K}_details.txt
