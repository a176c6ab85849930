"""Multi-GPU plumbing: row-strip partition with a ghost-row (halo) exchange,
and batch sharding.  One process per GPU, torch.distributed for the process
group (NCCL on GPUs; gloo for the CPU tests of this host logic).

Row strips (BASELINE.json config 3).  Rank g of G owns
pixel rows [r_g, r_{g+1}) with r_g = 2 floor(g ceil(H/2) / G) (balanced quad
rows, even-aligned; the paper's row bands mapped to cores, with
the partition rule of SPEC.md L349-357).  A level-1 output quad row n reads
input rows 2n-2 .. 2n+2 (Eq. (5) with the CDF 5/3 supports P: {0, +1},
U: {-1, 0}), so a strip needs exactly 2 ghost rows from the rank above and 1
from the rank below.  The exchange is one grouped NCCL send/recv per step
(``batch_isend_irecv``); the interior quad rows, which read no ghost row, run
while it is in flight (``DWT2_STRIP_INTERIOR``), then the two boundary quad
rows (``DWT2_STRIP_BOUNDARY``).  The global top/bottom strips use the
whole-sample symmetric mirror instead of ghosts.

Batches (config 5) shard whole images with no communication.
"""
from __future__ import annotations

import numpy as np


def strip_rows(height: int, rank: int, world: int) -> tuple:
    """[r_g, r_{g+1}) of rank g: even-aligned balanced quad-row bands."""
    hq = (height + 1) // 2
    lo = 2 * ((rank * hq) // world)
    hi = height if rank == world - 1 else 2 * (((rank + 1) * hq) // world)
    return lo, hi


def shard(count: int, rank: int, world: int) -> range:
    """Contiguous balanced share of `count` images for `rank` of `world`."""
    return range((count * rank) // world, (count * (rank + 1)) // world)


def ghost_rows(height: int, rank: int, world: int) -> tuple:
    """(ghosts above, ghosts below) in rank's input buffer."""
    lo, hi = strip_rows(height, rank, world)
    return (2 if lo > 0 else 0), (1 if hi < height else 0)


def halo_plan(height: int, rank: int, world: int) -> list:
    """The point-to-point messages of one exchange, as (op, peer, buf_row0, nrows)
    with buffer rows counted in rank's [ghost_top + strip + ghost_bot] buffer.
      recv 2 rows from rank-1 into the top ghost slots;
      recv 1 row  from rank+1 into the bottom ghost slot;
      send its first strip row to rank-1 (their bottom ghost);
      send its last 2 strip rows to rank+1 (their top ghosts)."""
    lo, hi = strip_rows(height, rank, world)
    gt, gb = ghost_rows(height, rank, world)
    n = hi - lo
    if n < 2:
        raise ValueError("row strips need at least 2 rows each (H >= 2 G)")
    msgs = []
    if gt:
        msgs.append(("recv", rank - 1, 0, 2))
        msgs.append(("send", rank - 1, gt, 1))
    if gb:
        msgs.append(("recv", rank + 1, gt + n, 1))
        msgs.append(("send", rank + 1, gt + n - 2, 2))
    return msgs


def place_strip_output(full: np.ndarray, strip_out: np.ndarray, W: int, H: int, r0: int, r1: int) -> None:
    """Copy a strip-local Mallat output (W x (r1-r0)) into the global one (W x H)."""
    Hq = (H + 1) // 2
    qs, qe = r0 // 2, (r1 + 1) // 2
    hq_loc = qe - qs
    full[qs:qe, :] = strip_out[:hq_loc, :]                      # LL | HL rows
    h0, h1 = min(qs, H // 2), min(qe, H // 2)
    if h1 > h0:
        full[Hq + h0:Hq + h1, :] = strip_out[hq_loc:hq_loc + (h1 - h0), :]   # LH | HH rows


def take_strip_output(full: np.ndarray, W: int, H: int, r0: int, r1: int) -> np.ndarray:
    """Inverse of place_strip_output: the strip-local view of a global output."""
    Hq = (H + 1) // 2
    qs, qe = r0 // 2, (r1 + 1) // 2
    h0, h1 = min(qs, H // 2), min(qe, H // 2)
    out = np.empty((r1 - r0, W), dtype=full.dtype)
    out[:qe - qs] = full[qs:qe]
    out[qe - qs:] = full[Hq + h0:Hq + h1]
    return out


class StripExchange:
    """Owns rank's input buffer (ghost rows + strip rows) as a torch tensor and
    runs the ghost-row exchange over the default process group."""

    def __init__(self, width: int, height: int, rank: int, world: int, device=None, dtype=None):
        import torch
        self.width, self.height, self.rank, self.world = width, height, rank, world
        self.r0, self.r1 = strip_rows(height, rank, world)
        self.ghost_top, self.ghost_bot = ghost_rows(height, rank, world)
        rows = self.ghost_top + (self.r1 - self.r0) + self.ghost_bot
        self.buf = torch.empty((rows, width), dtype=dtype or torch.float32, device=device)
        self.msgs = halo_plan(height, rank, world)

    @property
    def strip(self):
        """View of the owned rows (fill it with the strip's pixels)."""
        return self.buf[self.ghost_top:self.ghost_top + (self.r1 - self.r0)]

    def start(self):
        """Post the grouped sends/receives; returns the request list."""
        import torch.distributed as dist
        ops = []
        for op, peer, row0, nrows in self.msgs:
            view = self.buf[row0:row0 + nrows]
            ops.append(dist.P2POp(dist.isend if op == "send" else dist.irecv, view, peer))
        return dist.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def finish(reqs):
        for r in reqs:
            r.wait()


def strip_forward_step(exchange: StripExchange, plan, out, overlap: bool = True, stream=None):
    """One level-1 forward of rank's strip: halo exchange + fused kernel(s).
    With overlap, the interior quad rows run while the ghost rows are in flight."""
    from . import dwt2
    reqs = exchange.start()
    if overlap:
        plan.forward(exchange.buf, out, dwt2.DWT2_STRIP_INTERIOR, stream)
        exchange.finish(reqs)
        plan.forward(exchange.buf, out, dwt2.DWT2_STRIP_BOUNDARY, stream)
    else:
        exchange.finish(reqs)
        plan.forward(exchange.buf, out, dwt2.DWT2_STRIP_ALL, stream)
    return out
