# K13 iteration: parity tests, launch times, ncu details of both loss kernels
timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_metrics.py -x -q 2>&1 | tail -2
bash tools/r4q_ncu.sh > /dev/null 2>&1
for K in k_ssim_stats k_ssim_grad; do echo $K; grep -E " Duration|Issued Instructions  |Executed Ipc Active|Achieved Active" gpurun_out/r4q_${K}_details.txt; done
