bash tools/ncu_kernel.sh r2s k_blend_fast
CS_BLEND_EXACT=1 bash tools/ncu_kernel.sh r2s_exact "k_blend<"
