# K = 2 kernels: rows in flight per warp (the unrolled row loop's code size vs prefetch depth)
b() { timeout 300 python bench.py "$@" --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"; }
echo "default(8): fwd c3 $(b --config 3 --wavelet cdf97) c4 $(b --config 4 --wavelet cdf97) inv c3 $(b --config 3 --wavelet cdf97 --op inverse)"
for v in k2ds6 k2ds4 k2ds2; do
  export DWT2_LIB=build/variants/libdwt2_$v.so
  echo "$v: fwd c3 $(b --config 3 --wavelet cdf97) c4 $(b --config 4 --wavelet cdf97) inv c3 $(b --config 3 --wavelet cdf97 --op inverse)"
done
