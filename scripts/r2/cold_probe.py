"""Is config 2 with 3 buffer pairs really L2-cold?  K = 20 graph-captured
calls: (a) P pairs cycled (bench protocol), (b) one pair with a 256 MiB
read-only L2 flush before every call, minus the flushes timed alone,
(c) the same with a write flush (256 MiB memset), (d) torch copy under (b)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = H = 4096
x = torch.from_numpy(workloads.GENERATORS["smooth"](W, H, 2)).cuda()
p = dwt2.Plan(W, H, 1)
fl = torch.zeros(64 * 1024 * 1024, device="cuda")
sink = torch.zeros((), device="cuda")
pair = [(x, torch.empty_like(x))]
rf = time_calls(lambda q: sink.copy_(fl.amax()), pair, 20)
wf = time_calls(lambda q: fl.fill_(1.0), pair, 20)
for P in (1, 2, 3, 4, 20):
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(P)]
    a = time_calls(lambda q: p.forward(q[0], q[1]), pairs, 20)
    print(f"P {P:2d}: {a:5.1f} us", flush=True)
b = time_calls(lambda q: (sink.copy_(fl.amax()), p.forward(q[0], q[1])), pair, 20) - rf
c = time_calls(lambda q: (fl.fill_(1.0), p.forward(q[0], q[1])), pair, 20) - wf
d = time_calls(lambda q: (sink.copy_(fl.amax()), q[1].copy_(q[0])), pair, 20) - rf
print(f"read-flush before every call: level {b:5.1f} us (flush alone {rf:5.1f}); write-flush: level {c:5.1f} us "
      f"(flush alone {wf:5.1f}); copy with read-flush {d:5.1f} us")
