"""Run one forward per size in a subprocess (CUDA_LAUNCH_BLOCKING=1) and
report which sizes fail and the max error against the oracle."""
import os
import subprocess
import sys

SIZES = [(4095, 31), (4095, 32), (4094, 32), (4094, 31), (4093, 64), (8194, 64), (6, 8), (5, 8), (7, 9),
         (8194, 8192), (4095, 3001)]
if len(sys.argv) > 1:
    W, H = int(sys.argv[1]), int(sys.argv[2])
    sys.path.insert(0, ".")
    import numpy as np
    import torch
    import oracle
    from paper_1708_07853_b200 import dwt2, workloads
    x = workloads.uniform_int(W, H, 7)
    p = dwt2.Plan(W, H, 1)
    y = p.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    if W * H <= 1 << 20:
        ref = oracle.forward(x.astype(np.float64), 1, round_f32=True)
        print(f"{W}x{H}: ok, max err {np.abs(y.cpu().numpy() - ref).max()}")
    else:
        print(f"{W}x{H}: ok (no oracle)")
    sys.exit(0)
env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
for W, H in SIZES:
    r = subprocess.run([sys.executable, __file__, str(W), str(H)], capture_output=True, text=True, env=env, timeout=120)
    print(r.stdout.strip() if r.returncode == 0 else f"{W}x{H}: FAILED {r.stderr.strip().splitlines()[-1][:120]}")
