#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/sort_bench.cu -o /tmp/sb
/tmp/sb > gpurun_out/y_sort.log 2>&1; cat gpurun_out/y_sort.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_onesweep -c 8 -o gpurun_out/y_sort /tmp/sb prof > gpurun_out/y_sort_ncu.log 2>&1
tail -1 gpurun_out/y_sort_ncu.log
