mkdir -p gpurun_out/prof2
ncu --set full --clock-control none --import-source on -k regex:inverse -s 1 -c 1 -o gpurun_out/prof2/inv_c3 python scripts/prof_target.py inverse --reps 2 > gpurun_out/prof2/inv.log 2>&1; tail -1 gpurun_out/prof2/inv.log
