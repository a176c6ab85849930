"""TMA sensitivity to the number of distinct inputs: is it the tensor-map
descriptors or the pages?  K = 20 graph-captured 5/3 forward calls of
config 2's shape cycling over P inputs that are (a) distinct buffers, (b) the
SAME memory seen through P base pointers 16 bytes apart (P distinct tensor
maps over the same pages), (c) distinct buffers with one shared output."""
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
for P in (1, 3, 8, 20):
    a_pairs = [(x.clone(), torch.empty_like(x)) for _ in range(P)]
    big = torch.empty(N + 4 * P, device="cuda")
    big[:N].copy_(x.view(-1))
    outs = [torch.empty_like(x) for _ in range(P)]
    b_pairs = [(big[4 * i:4 * i + N].view(H, W), outs[i]) for i in range(P)]
    one_out = torch.empty_like(x)
    c_pairs = [(a_pairs[i][0], one_out) for i in range(P)]
    a = time_calls(lambda q: p.forward(q[0], q[1]), a_pairs, 20)
    b = time_calls(lambda q: p.forward(q[0], q[1]), b_pairs, 20)
    c = time_calls(lambda q: p.forward(q[0], q[1]), c_pairs, 20)
    print(f"P {P:2d}: distinct buffers {a:5.1f} | same memory, P tensor maps {b:5.1f} | distinct inputs, one output {c:5.1f} us",
          flush=True)
    del a_pairs, b_pairs, c_pairs, big, outs
