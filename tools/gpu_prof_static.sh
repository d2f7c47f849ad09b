timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_generate" -s 4 -c 1 -o gpurun_out/prof_static python tools/k1_split.py > gpurun_out/ncu_static.log 2>&1
echo rc=$?
