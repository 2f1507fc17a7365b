for K in k_ssim_stats k_ssim_grad; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o gpurun_out/r4q_$K env PYTHONPATH=. python tools/loss_once.py > gpurun_out/r4q_$K.log 2>&1; tail -5 gpurun_out/r4q_$K.log
ncu -i gpurun_out/r4q_$K.ncu-rep --page raw --csv > gpurun_out/r4q_${K}_raw.csv
ncu -i gpurun_out/r4q_$K.ncu-rep --page details > gpurun_out/r4q_${K}_details.txt
ncu -i gpurun_out/r4q_$K.ncu-rep --page source --csv > gpurun_out/r4q_${K}_source.csv
rm -f gpurun_out/r4q_$K.ncu-rep
done
