"""Timing helper of the measurement scripts (same protocol as bench.py):
K calls captured as ONE CUDA graph, replayed once between two CUDA events on
the launching stream.  Working sets smaller than 2x the 126 MB L2 get one
input/output pair per call (the caller's make_pair), and the L2 is flushed
once (read-only 256 MB pass) before the timed replay.  CUDA event timestamps
tick every 2.048 us on this driver (scripts/diag_small.py), so single short
calls are never bracketed alone."""
import torch

import _variant  # noqa: F401  (DWT2_LIB: tuning / profiling builds)

L2_BYTES = 126e6
_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.zeros(64 * 1024 * 1024, device="cuda")
    _flush.amax()


def time_calls(call, pairs, K, reps=3):
    """call(pair) enqueues one call; pairs: list of buffers tuples (cycled).
    Returns the median over reps of the per-call time in microseconds."""
    g = torch.cuda.CUDAGraph()
    call(pairs[0])                                   # first-use costs outside the capture
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(K):
            call(pairs[i % len(pairs)])
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush_l2()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / K)
    ts.sort()
    return ts[len(ts) // 2]


def n_pairs(bytes_per_call, K):
    """Buffer pairs cycled so that no timed call finds its input in L2: a pair
    is reused only after more than 2x L2 of other traffic, or (small calls)
    each of the K calls gets its own pair, read once after the flush
    (bench.py's buffer_pairs)."""
    if bytes_per_call >= 2 * L2_BYTES:
        return 1
    return min(K, int(-(-2 * L2_BYTES // bytes_per_call)) + 1)
