# Round-2 final round-style run of this build: smoke, the GPU suite, the default
# bench line, the reference arm, every config and 8f row through bench.py, ncu
# launch lists and one full capture of the headline kernel (-> gpurun_out/r2final/)
set -x
B=gpurun_out/r2final
mkdir -p $B
timeout 300 python __graft_entry__.py smoke
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py > $B/default_c3.json 2> $B/default_c3.err; tail -c 300 $B/default_c3.json
timeout 900 python bench.py --impl reference > $B/reference_c3.json 2>&1; tail -c 300 $B/reference_c3.json
for c in 1 2 4 4b 5; do timeout 900 python bench.py --config $c > $B/fwd53_c$c.json 2> $B/fwd53_c$c.err; done
for c in 2 3 4 4b 5; do timeout 900 python bench.py --config $c --op inverse > $B/inv53_c$c.json 2> $B/inv53_c$c.err; done
for c in 3 4; do
  timeout 900 python bench.py --config $c --wavelet cdf97 > $B/fwd97_c$c.json 2> $B/fwd97_c$c.err
  timeout 900 python bench.py --config $c --wavelet cdf97 --op inverse > $B/inv97_c$c.json 2> $B/inv97_c$c.err
done
for sch in nonsep_naive nonsep_lifting nonsep_adapted sep_conv sep_lifting; do
  timeout 900 python bench.py --config 3 --scheme $sch --no-e2e > $B/scheme_${sch}_c3.json 2> $B/scheme_${sch}_c3.err
done
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), d.get('unit'), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'cpu', round(d['cpu_baseline']['value'],4) if d.get('cpu_baseline') else None, 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
# ncu: launch lists (cold, serialised -- shares, not bench values) and the headline capture
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $B/launches_default_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 > $B/ncu_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $B/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 --no-graph > $B/ncu_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $B/launches_c1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 --no-graph > $B/ncu_c1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dwt53_level_kernel -s 8 -c 1 -o $B/c3_level python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 --no-graph > $B/ncu_full.log 2>&1
ls -la $B | tail -40
