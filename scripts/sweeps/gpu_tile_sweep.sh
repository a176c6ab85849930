# sweep of the work-queue tile policy (env overrides) on configs 2, 4, 5, 3
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tiny or ragged or config4 or config5" 2>&1 | tail -2
for combo in "32 7 2" "32 7 100000" "32 3 2" "32 11 2" "16 7 2" "64 3 2" "32 3 1" "8 3 1"; do
  set -- $combo
  for c in 2 4 5 3; do
    r=$(DWT2_TPW=$1 DWT2_MIN_TB=$2 DWT2_MIN_TPW=$3 timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
    echo "TPW=$1 MINTB=$2 MINTPW=$3 config=$c : $r"
  done
done
python scripts/level_times.py
