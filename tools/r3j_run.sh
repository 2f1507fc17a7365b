python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for M in fast exact; do
  if [ $M = exact ]; then export CS_BLEND_EXACT=1; K="k_blend<"; else unset CS_BLEND_EXACT; K=k_blend_fast; fi
  CS_PROFILE_FRAMES=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"$K" --launch-skip 1 -c 1 -o gpurun_out/r3j_$M python tools/one_view.py 565 3 > gpurun_out/r3j_$M.log 2>&1
  ncu -i gpurun_out/r3j_$M.ncu-rep --page source --csv > gpurun_out/r3j_${M}_source.csv 2>/dev/null
  ncu -i gpurun_out/r3j_$M.ncu-rep --page raw --csv > gpurun_out/r3j_${M}_raw.csv 2>/dev/null
  rm -f gpurun_out/r3j_$M.ncu-rep
done
ls -la gpurun_out | grep r3j
