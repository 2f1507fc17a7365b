#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/sort_bench.cu -o /tmp/sb
/tmp/sb > gpurun_out/z_sort.log 2>&1; cat gpurun_out/z_sort.log
