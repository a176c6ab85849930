V=build/variants/libdwt2_tuning.so
export DWT2_LIB=$V
echo "== correctness (grouped, all levels in the tail)"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -5
echo "== correctness (grouped, gsz 3, bmax 4)"
DWT2_TAIL_GROUPED=1 DWT2_PT_GSZ=3 DWT2_PT_BMAX=4 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 NRAND=10 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -5
run() { timeout 300 python bench.py --variant-lib $V "$@" --no-e2e --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1))"; }
echo "== timing config 4 (5/3)"
echo "base: $(run --config 4)"
for q in 16384 65536 262144 1048576; do for g in 1 2 3; do
  echo "grouped q=$q gsz=$g: c4 $(DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=$q DWT2_PT_GSZ=$g run --config 4)"
done; done
for t in 296 592; do echo "grouped q=262144 gsz=2 tasks=$t: c4 $(DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 DWT2_PT_GSZ=2 DWT2_PT_TASKS=$t run --config 4)"; done
echo "9/7 base: $(run --config 4 --wavelet cdf97)"
for q in 65536 262144; do for g in 1 2; do
echo "9/7 grouped q=$q g=$g: $(DWT2_TAIL_GROUPED=1 DWT2_K2_TAIL_QUADS=$q DWT2_PT_GSZ=$g run --config 4 --wavelet cdf97)"
done; done
mkdir -p gpurun_out/ptail
B="python bench.py --variant-lib $V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0 --config 4"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 40 --csv --log-file gpurun_out/ptail/launches3_q18.csv $B > /dev/null 2>&1; echo "launches: $?"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 timeout 900 ncu --clock-control none --set full --import-source on -k regex:ptail -s 2 -c 1 -o gpurun_out/ptail/ptail3_q18 $B > /dev/null 2>&1; echo "full: $?"
