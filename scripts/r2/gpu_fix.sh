set -x
B=gpurun_out/r2final
mkdir -p $B
timeout 900 python -m pytest tests/test_gpu_peer_strips.py tests/test_gpu_peer_ipc.py tests/test_gpu_strip_levels.py -q -x 2>&1 | tail -2
for v in product build/variants/libdwt2_old.so; do timeout 600 python scripts/r2/c5_groups.py $v 2>&1 | tail -4; done
timeout 900 python bench.py --config 5 > $B/fwd53_c5.json 2> $B/fwd53_c5.err; tail -c 200 $B/fwd53_c5.json; echo
timeout 900 python bench.py --config 5 --op inverse > $B/inv53_c5.json 2> $B/inv53_c5.err
timeout 900 python bench.py > $B/default_c3.json 2> $B/default_c3.err; tail -c 200 $B/default_c3.json; echo
timeout 900 python bench.py --config 1 > $B/fwd53_c1.json 2> $B/fwd53_c1.err
timeout 900 python bench.py --config 4 > $B/fwd53_c4.json 2> $B/fwd53_c4.err
timeout 900 python bench.py --config 4b > $B/fwd53_c4b.json 2> $B/fwd53_c4b.err
timeout 900 python bench.py --config 2 > $B/fwd53_c2.json 2> $B/fwd53_c2.err
for f in default_c3 fwd53_c1 fwd53_c2 fwd53_c4 fwd53_c4b fwd53_c5 inv53_c5; do python -c "
import json; d=json.loads(open('$B/$f.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f', round(d.get('value',0),2), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'clk', (d.get('clocks') or {}).get('reasons'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $B/launches_default_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 > $B/ncu_default.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dwt53_level -s 3 -c 1 -o $B/c3_level python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 --no-graph > $B/ncu_full.log 2>&1
tail -2 $B/ncu_full.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dwt53_small -s 3 -c 1 -o $B/c1_small python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 --no-graph > $B/ncu_small.log 2>&1
tail -2 $B/ncu_small.log
