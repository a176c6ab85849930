mkdir -p gpurun_out
python scripts/prof_target.py inverse --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:inverse -s 1 -c 1 -o gpurun_out/prof_inv_c3 python scripts/prof_target.py inverse --reps 2 > gpurun_out/ncu_inv.log 2>&1; tail -1 gpurun_out/ncu_inv.log
python scripts/prof_target.py forward --config 2 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:dwt53_level -s 1 -c 1 -o gpurun_out/prof_fwd_c2 python scripts/prof_target.py forward --config 2 --reps 2 > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log
