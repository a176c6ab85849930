# tiles per warp of the queued inverse and K = 2 kernels
b() { timeout 300 python bench.py "$@" --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"; }
for t in 4 8 16 32; do echo "INV_TPW=$t c3: $(DWT2_INV_TPW=$t b --config 3 --op inverse)  c4: $(DWT2_INV_TPW=$t b --config 4 --op inverse)  c2: $(DWT2_INV_TPW=$t b --config 2 --op inverse)"; done
for t in 2 4 8 16; do echo "K2_TPW=$t c3: $(DWT2_K2_TPW=$t b --config 3 --wavelet cdf97)  c4: $(DWT2_K2_TPW=$t b --config 4 --wavelet cdf97)  inv c3: $(DWT2_K2_TPW=$t b --config 3 --wavelet cdf97 --op inverse)"; done
