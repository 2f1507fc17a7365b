bash tools/ncu_kernel.sh r2v k_blend_fast
CS_BLEND_EXACT=1 bash tools/ncu_kernel.sh r2v_exact "k_blend<"
ls gpurun_out | grep r2v
