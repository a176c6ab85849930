# guided tile split sweep (percent of rows in one-per-warp tiles, small tiles per warp)
for ga in 50 60 70 80 85; do
  for gb in 2 4 8; do
    c2=$(DWT2_GUIDED_A=$ga DWT2_GUIDED_B=$gb timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
    st=$(DWT2_GUIDED_A=$ga DWT2_GUIDED_B=$gb timeout 300 python scripts/strip_host_cost.py 2>&1 | sed -n 2p | sed 's/.*graph (GPU only) //')
    echo "A=$ga B=$gb  c2: $c2   strip G=8 ALL: $st"
  done
done
