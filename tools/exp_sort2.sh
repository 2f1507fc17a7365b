#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/sort_bench.cu -o /tmp/sb
/tmp/sb | grep "v12/3e"
bash tools/exp_quick.sh s2 | tail -2
