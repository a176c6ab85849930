"""Per-call time of tiny forward calls in a CUDA graph (K = 50 calls, one
buffer pair per call): the launch + dependency-chain floor of one level."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
for W, H, L in [(8, 8, 1), (64, 64, 1), (128, 128, 1), (256, 256, 1), (512, 512, 1), (64, 64, 2), (64, 64, 4)]:
    K = 50
    pairs = [(torch.from_numpy(workloads.uniform_int(W, H, i)).cuda(), torch.empty(H, W, device="cuda")) for i in range(K)]
    p = dwt2.Plan(W, H, L)
    us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, K)
    print(f"{W}x{H} L{L}: {us:6.2f} us per call ({us / L:5.2f} per level)")
    p.close()
# empty-kernel floor for comparison (torch's own tiny kernel)
x = torch.zeros(1, device="cuda")
us = time_calls(lambda q: q[0].add_(1.0), [(x,)], 50)
print(f"torch add_ on 1 element: {us:6.2f} us per call")
