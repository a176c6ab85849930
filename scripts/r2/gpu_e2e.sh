# dwt2_forward_host band schedule (tuning build): e2e Gpix/s of config 3 / 4
V=build/variants/libdwt2_tuning.so
for rep in 1 2; do
for tb in "0 16" "3 16" "4 16" "5 16" "4 32" "6 16"; do set -- $tb; out="taper $1 bands $2:"; for c in 3 4; do out="$out $(DWT2_HOST_TAPER=$1 DWT2_HOST_BANDS=$2 timeout 300 python bench.py --variant-lib $V --config $c --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['e2e']['value'],3))")"; done; echo $out; done
done
