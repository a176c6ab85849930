# 5/3 inverse ring: rows in flight per warp (unroll / code size vs prefetch depth)
b() { timeout 300 python bench.py "$@" --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"; }
echo "default(6): c3 $(b --config 3 --op inverse) c4 $(b --config 4 --op inverse) c2 $(b --config 2 --op inverse)"
for v in inv3 inv4 inv8; do
  export DWT2_LIB=build/variants/libdwt2_$v.so
  echo "$v: c3 $(b --config 3 --op inverse) c4 $(b --config 4 --op inverse) c2 $(b --config 2 --op inverse)"
done
