V=build/variants/libdwt2_tuning.so
export DWT2_LIB=$V
echo "== correctness (grouped, all levels in the tail)"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -8
echo "== correctness (grouped, gsz 3)"
DWT2_TAIL_GROUPED=1 DWT2_PT_GSZ=3 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 NRAND=10 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -8
mkdir -p gpurun_out/ptail
B="python bench.py --variant-lib $V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0 --config 4"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 40 --csv --log-file gpurun_out/ptail/launches_q18.csv $B > /dev/null 2>&1; echo "launches: $?"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 timeout 900 ncu --clock-control none --set full --import-source on -k regex:ptail -s 2 -c 1 -o gpurun_out/ptail/ptail_q18 $B > /dev/null 2>&1; echo "full: $?"
