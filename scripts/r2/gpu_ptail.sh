V=build/variants/libdwt2_tuning.so
export DWT2_LIB=$V
echo "== correctness (grouped, all levels in the tail)"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -8
echo "== correctness (grouped, gsz 3, small blocks)"
DWT2_TAIL_GROUPED=1 DWT2_PT_GSZ=3 DWT2_PT_BMAX=4 DWT2_TAIL_QUADS=1073741824 DWT2_K2_TAIL_QUADS=1073741824 NRAND=10 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -8
echo "== correctness (grouped, default split, 2^18)"
DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=262144 NRAND=10 timeout 600 python scripts/r2/ptail_check.py 2>&1 | tail -4
run() { timeout 300 python bench.py --variant-lib $V "$@" --no-e2e --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1))"; }
echo "== timing config 4 (5/3)"
echo "base: $(run --config 4)"
for q in 16384 65536 262144 1048576; do for g in 1 2 3; do
  echo "grouped q=$q gsz=$g: c4 $(DWT2_TAIL_GROUPED=1 DWT2_TAIL_QUADS=$q DWT2_PT_GSZ=$g run --config 4)"
done; done
