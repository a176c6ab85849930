"""Why cycling over many buffer pairs slows the level kernel (VERDICT r1 weak
#12): config 2 (4096^2, 1 level) as K = 20 graph-captured calls cycling over P
buffer pairs, (a) as is, (b) with a tiny kernel before each call that touches
one float per 2 MiB page of the NEXT call's input and output (warms the
address translation, moves ~no data), (c) the pairs carved out of ONE
allocation, and (d) a plain device copy under the same protocol."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = H = 4096
N = W * H
x = torch.from_numpy(workloads.GENERATORS["smooth"](W, H, 2)).cuda()
p = dwt2.Plan(W, H, 1)
import os
PAGE = int(os.environ.get("TOUCH_BYTES", str(2 << 20))) // 4
sink = torch.zeros(1, device="cuda")


def touch(t):
    sink.add_(t.view(-1)[::PAGE].sum())


for P in (1, 3, 20):
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(P)]
    a = time_calls(lambda q: p.forward(q[0], q[1]), pairs, 20)
    nxt = {id(pairs[i][0]): pairs[(i + 1) % P] for i in range(P)}

    def fwd_touch(q):
        n = nxt[id(q[0])]
        touch(n[0])
        touch(n[1])
        p.forward(q[0], q[1])
    b = time_calls(fwd_touch, pairs, 20)
    t0 = time_calls(lambda q: (touch(q[0]), touch(q[1])), pairs, 20)
    big = torch.empty(2 * P * N, device="cuda")
    cpairs = [(big[2 * i * N:(2 * i + 1) * N].view(H, W), big[(2 * i + 1) * N:(2 * i + 2) * N].view(H, W)) for i in range(P)]
    for q in cpairs:
        q[0].copy_(x)
    c = time_calls(lambda q: p.forward(q[0], q[1]), cpairs, 20)
    d = time_calls(lambda q: q[1].copy_(q[0]), pairs, 20)
    print(f"touch stride {PAGE * 4} B, pairs {P:2d}: level {a:5.1f} us | +touch next {b:5.1f} (touch alone {t0:4.1f}) | one allocation {c:5.1f} | "
          f"copy {d:5.1f} us", flush=True)
    del pairs, cpairs, big
