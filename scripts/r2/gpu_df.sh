set -x
mkdir -p gpurun_out/df
timeout 300 python __graft_entry__.py smoke
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python scripts/r2/df_probe.py 2>&1 | tail -6
timeout 600 python scripts/r2/df_probe.py nodf 2>&1 | tail -6
python -c "
import torch,glob
for f in sorted(glob.glob('gpurun_out/df_product_*.pt')):
    g=f.replace('product','nodf'); a=torch.load(f); b=torch.load(g); print(f, 'identical' if torch.equal(a,b) else 'DIFFERENT')
"
for c in 4 4b 5; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/df/fwd53_c$c.json 2>&1; tail -c 200 gpurun_out/df/fwd53_c$c.json; echo; done
