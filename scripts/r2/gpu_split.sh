set -x
for v in product build/variants/libdwt2_smallsplit.so product build/variants/libdwt2_smallsplit.so; do
  timeout 600 python scripts/r2/variant_probe.py $v 2>&1 | grep 'config 4'
  timeout 300 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'scripts')
from paper_1708_07853_b200 import dwt2
if '$v' != 'product': dwt2.use_variant('$v')
import torch
from _timing import time_calls
from paper_1708_07853_b200 import workloads
x=torch.from_numpy(workloads.uniform_int(512,512,1)).cuda(); pairs=[(x.clone(),torch.empty_like(x)) for _ in range(20)]
p=dwt2.Plan(512,512,1); print('$v'.split('/')[-1], 'config 1', round(time_calls(lambda q: p.forward(q[0],q[1]), pairs, 20),2), 'us')
y=p.forward(x).cpu(); import numpy as np, oracle; r=oracle.forward(x.cpu().numpy().astype(np.float64),1,round_f32=True); print('exact', np.array_equal(y.numpy(), r.astype(np.float32)))
"
done
