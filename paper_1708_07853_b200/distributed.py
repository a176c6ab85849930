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

Multi-level strips: with L levels the strip bounds are
multiples of 2^L (``strip_rows_levels``), so every level's strip is even-
aligned in that level's LL image; each level exchanges its own ghost rows
(2 above, 1 below) of the previous level's LL before its kernel runs
(``StripPyramid``).  The strip-local output is the Mallat pyramid of the
strip's W x rows sub-image, with every level's subband rows where a Mallat
pyramid puts them.

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


def strip_rows_levels(height: int, rank: int, world: int, levels: int = 1) -> tuple:
    """[r_g, r_{g+1}) of rank g for an L-level pyramid: balanced runs of
    2^L-row units (levels = 1 is ``strip_rows``)."""
    unit = 1 << levels
    nunits = -(-height // unit)
    lo = unit * ((rank * nunits) // world)
    hi = height if rank == world - 1 else unit * (((rank + 1) * nunits) // world)
    return lo, hi


def level_rows(width: int, height: int, lo: int, hi: int, levels: int) -> list:
    """Per level k: (W_k, H_k, rb_k, re_k, ghost_top, ghost_bot) -- the level's
    global input size and the strip's rows of it (rb_k = lo / 2^k,
    re_k = ceil(re_{k-1} / 2)); mirrors dwt2_strip_level_info."""
    out = []
    w, h, rb, re = width, height, lo, hi
    for _ in range(levels):
        out.append((w, h, rb, re, 2 if rb > 0 else 0, 1 if re < h else 0))
        w, h, rb, re = (w + 1) // 2, (h + 1) // 2, rb // 2, (re + 1) // 2
    return out


def halo_messages(rb: int, re: int, height: int, rank: int) -> list:
    """The exchange of one level for rows [rb, re) of a `height`-row level
    image (see ``halo_plan``)."""
    gt, gb = (2 if rb > 0 else 0), (1 if re < height else 0)
    n = re - rb
    if n < 2:
        raise ValueError("row strips need at least 2 rows per level")
    msgs = []
    if gt:
        msgs.append(("recv", rank - 1, 0, 2))
        msgs.append(("send", rank - 1, gt, 1))
    if gb:
        msgs.append(("recv", rank + 1, gt + n, 1))
        msgs.append(("send", rank + 1, gt + n - 2, 2))
    return msgs


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
    return halo_messages(lo, hi, height, rank)


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


def _p2p_ops(msgs, buf):
    """The grouped sends/receives of rows of `buf` (a 2-D tensor)."""
    import torch.distributed as dist
    return [dist.P2POp(dist.isend if op == "send" else dist.irecv, buf[row0:row0 + nrows], peer)
            for op, peer, row0, nrows in msgs]


def _p2p(msgs, buf):
    """Post grouped sends/receives of rows of `buf` (a 2-D tensor)."""
    import torch.distributed as dist
    ops = _p2p_ops(msgs, buf)
    return dist.batch_isend_irecv(ops) if ops else []


class StripPyramid:
    """Rank's buffers of an L-level row-strip transform: one ghost-padded input
    buffer per level (level 0: the image rows; level k >= 1: the LL of level
    k-1, written by the level kernel into its owned rows) and the strip-local
    output pyramid.  Row pitches of levels >= 1 are rounded up to 4 floats
    (16-byte rows: the TMA-staged kernel path)."""

    def __init__(self, width: int, height: int, rank: int, world: int, levels: int = 1, device=None):
        import torch
        self.width, self.height, self.rank, self.world, self.levels = width, height, rank, world, levels
        self.r0, self.r1 = strip_rows_levels(height, rank, world, levels)
        self.geom = level_rows(width, height, self.r0, self.r1, levels)
        self.bufs = []
        for k, (w, h, rb, re, gt, gb) in enumerate(self.geom):
            pitch = width if k == 0 else -(-w // 4) * 4
            full = torch.empty((gt + (re - rb) + gb, pitch), dtype=torch.float32, device=device)
            self.bufs.append(full)
        self.msgs = [halo_messages(rb, re, h, rank) for (w, h, rb, re, gt, gb) in self.geom]
        self.out = torch.empty((self.r1 - self.r0, width), dtype=torch.float32, device=device)
        self.ghost_top, self.ghost_bot = self.geom[0][4], self.geom[0][5]

    @property
    def buf(self):
        return self.bufs[0]

    def owned(self, k: int):
        """Level k's owned rows (a view of its input buffer, level width)."""
        w, h, rb, re, gt, gb = self.geom[k]
        return self.bufs[k][gt:gt + (re - rb), :w]

    @property
    def strip(self):
        return self.owned(0)

    def level_buffer(self, k: int):
        """Level k's whole ghost-padded buffer, level width columns."""
        return self.bufs[k][:, :self.geom[k][0]]

    def start(self, k: int):
        """Post level k's ghost-row exchange over the default process group
        (the P2POp lists are built once: the per-step host cost is the NCCL
        group call only)."""
        import torch.distributed as dist
        if not hasattr(self, "_ops"):
            self._ops = [_p2p_ops(self.msgs[j], self.bufs[j]) for j in range(self.levels)]
        return dist.batch_isend_irecv(self._ops[k]) if self._ops[k] else []

    @staticmethod
    def finish(reqs):
        for r in reqs:
            r.wait()

    def global_rows(self, k: int) -> tuple:
        """Global row range [lo, hi) of level k's buffer (ghosts included)."""
        w, h, rb, re, gt, gb = self.geom[k]
        return rb - gt, re + gb


def strip_pyramid_step(pyr: StripPyramid, plan, overlap: bool = True, stream=None, exchange=None):
    """All levels of rank's strip: per level, the ghost-row exchange and the
    fused level kernel(s); with overlap, the interior quad rows run while the
    ghost rows are in flight, then the two boundary quad rows.  exchange(k)
    may replace the process-group exchange (single-GPU emulation in tests); it
    returns request objects whose wait() orders the current stream after the
    ghost rows have landed, as NCCL's Work.wait() does.

    Measured on one B200 (scripts/strip_host_cost.py, config 3 at G = 8): the
    boundary launch right behind the interior one (programmatic dependent
    launch) costs no GPU time over a single launch of all rows (59 us per
    step either way), and running it on a side stream instead adds ~30 us of
    host enqueue time per level without saving GPU time -- so both parts stay
    on the current stream."""
    import torch
    from . import dwt2
    # raw C-ABI arguments of every level, built once (a step then costs the
    # launches' own host time, not Python tensor bookkeeping)
    key = (id(plan), pyr.out.data_ptr())
    if getattr(pyr, "_launch_key", None) != key:
        args = []
        for k in range(pyr.levels):
            buf = pyr.bufs[k]
            ll = pyr.owned(k + 1) if k + 1 < pyr.levels else None
            args.append((buf.data_ptr(), buf.stride(0), 0 if ll is None else ll.data_ptr(),
                         0 if ll is None else ll.stride(0)))
        pyr._launch_args, pyr._launch_key = args, key
    h = plan.handle
    out = pyr.out.data_ptr()
    if stream is not None:
        sh = stream.cuda_stream
    else:
        sh = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
    launch = getattr(plan, "launch_level", None) or dwt2.dwt2_forward_strip_level
    for k in range(pyr.levels):
        reqs = pyr.start(k) if exchange is None else exchange(k)
        bp, bpitch, lp, lpitch = pyr._launch_args[k]
        if overlap:
            launch(h, k, bp, bpitch, lp, lpitch, out, dwt2.DWT2_STRIP_INTERIOR, sh)
            pyr.finish(reqs)          # NCCL Work.wait(): the current stream waits for the receives
            launch(h, k, bp, bpitch, lp, lpitch, out, dwt2.DWT2_STRIP_BOUNDARY, sh)
        else:
            pyr.finish(reqs)
            launch(h, k, bp, bpitch, lp, lpitch, out, dwt2.DWT2_STRIP_ALL, sh)
    return pyr.out


def place_pyramid_output(full: np.ndarray, strip_out: np.ndarray, W: int, H: int, r0: int, r1: int,
                         levels: int) -> None:
    """Copy a strip-local L-level pyramid (W x (r1-r0)) into the global one."""
    w, h, rb, re, hl = W, H, r0, r1, r1 - r0
    for k in range(levels):
        Hq, Hh, Wq = (h + 1) // 2, h // 2, (w + 1) // 2
        qs, qe = rb // 2, (re + 1) // 2
        hq_loc = qe - qs
        last = k == levels - 1
        c0 = 0 if last else Wq                    # LL of inner levels is not output
        full[qs:qe, c0:w] = strip_out[:hq_loc, c0:w]                          # (LL |) HL
        h0, h1 = min(qs, Hh), min(qe, Hh)
        if h1 > h0:
            full[Hq + h0:Hq + h1, :w] = strip_out[hq_loc:hq_loc + (h1 - h0), :w]   # LH | HH
        w, h, rb, re = Wq, Hq, qs, qe


# ---- peer-memory halo (include/dwt2.h "peer strip context") -----------------
#
# The same row strips as StripPyramid, with the exchange fused into the level
# launch: every rank's level buffers live in one device allocation whose CUDA
# IPC handle the neighbours map; boundary-role CTAs in the level kernel's own
# launch read the 2 rows above / 1 row below from the neighbour's memory over
# NVLink once the neighbour's flag says they are final.  Host side, a step is
# ONE launch per level with no wait, so it can be captured in a CUDA graph.  The descriptors
# (plain bytes) travel once, through all_gather_object on the process group.

def peer_neighbours(descs: list, rank: int) -> tuple:
    """(above, below) descriptor bytes of `rank` from the all-gathered list,
    checked for matching geometry (the C side checks again): the rank above
    must end where this strip begins, the rank below begin where it ends."""
    from . import dwt2
    me = dwt2.PeerDesc.from_bytes(descs[rank])
    above = below = None
    if rank > 0:
        above = dwt2.PeerDesc.from_bytes(descs[rank - 1])
        if above.row_end != me.row_begin:
            raise ValueError(f"rank {rank}: the strip above ends at row {above.row_end}, this one begins at "
                             f"{me.row_begin}")
    if rank + 1 < len(descs):
        below = dwt2.PeerDesc.from_bytes(descs[rank + 1])
        if below.row_begin != me.row_end:
            raise ValueError(f"rank {rank}: the strip below begins at row {below.row_begin}, this one ends at "
                             f"{me.row_end}")
    for d in (above, below):
        if d is not None and (d.width, d.global_height, d.levels) != (me.width, me.global_height, me.levels):
            raise ValueError(f"rank {rank}: neighbour geometry {d.width}x{d.global_height} L{d.levels} differs")
    return above, below


def gather_descriptors(desc_bytes: bytes, group=None) -> list:
    """All ranks' descriptor bytes, in rank order (one all_gather_object)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, desc_bytes, group=group)
    return out


class PeerStripPyramid:
    """Rank's L-level row strip with peer-memory halos.  Fill ``strip`` (the
    level-0 owned rows, inside the C context's allocation), then ``step()``;
    the strip-local Mallat pyramid lands in ``out`` (the layout of
    StripPyramid.out).  ``connect()`` is collective over the process group.
    Emulated ranks (several in one process, tests and 1-GPU measurement) use
    ``connect_local`` and ``sequential_step``."""

    def __init__(self, width: int, height: int, rank: int, world: int, levels: int = 1, device=None,
                 timeout_ms: int = 0):
        import torch
        from . import dwt2
        self.width, self.height, self.rank, self.world, self.levels = width, height, rank, world, levels
        self.r0, self.r1 = strip_rows_levels(height, rank, world, levels)
        self.geom = level_rows(width, height, self.r0, self.r1, levels)
        self.ghost_top, self.ghost_bot = self.geom[0][4], self.geom[0][5]
        self.plan = dwt2.StripPlan(width, height, self.r0, self.r1, levels)
        self.ctx = dwt2.PeerStrip(self.plan, timeout_ms)
        self.out = torch.empty((self.r1 - self.r0, width), dtype=torch.float32, device=device)

    @property
    def strip(self):
        """Level-0 owned rows (write the strip's pixels here before a step)."""
        return self.ctx.owned(0)

    def owned(self, k: int):
        return self.ctx.owned(k)

    def export(self) -> bytes:
        return self.ctx.export().to_bytes()

    def connect(self, group=None):
        from . import dwt2
        above, below = peer_neighbours(gather_descriptors(self.export(), group), self.rank)
        self.ctx.connect(above, below, dwt2.DWT2_PEER_RANKS)

    def connect_descriptors(self, descs: list, mode=None):
        """Connect from the descriptor bytes of every rank (rank order), however
        they were gathered (a process group, a pipe between processes)."""
        from . import dwt2
        above, below = peer_neighbours(descs, self.rank)
        self.ctx.connect(above, below, dwt2.DWT2_PEER_RANKS if mode is None else mode)

    def connect_local(self, ranks: list, mode=None):
        """Ranks of one process (this object is ranks[self.rank])."""
        from . import dwt2
        above, below = peer_neighbours([r.export() for r in ranks], self.rank)
        self.ctx.connect(above, below, dwt2.DWT2_PEER_SEQUENTIAL if mode is None else mode)

    def step(self, stream=None):
        """One step of every level (concurrent ranks, one per GPU)."""
        return self.ctx.forward(self.out, stream)

    def status(self) -> int:
        return self.ctx.status()

    def close(self):
        self.ctx.close()
        self.plan.close()


def sequential_step(ranks: list, stream=None, fused: bool = True):
    """One step of emulated ranks in one stream, level by level: fused, every
    rank's PUBLISH launch, then every rank's ALL launch (the one-launch form a
    rank issues on its own GPU); else every rank's INTERIOR launch (which
    publishes), then every rank's BOUNDARY launch.  Every flag a launch waits
    for was published by an earlier launch."""
    from . import dwt2
    for k in range(ranks[0].levels):
        parts = ((dwt2.DWT2_STRIP_PUBLISH, dwt2.DWT2_STRIP_ALL) if fused
                 else (dwt2.DWT2_STRIP_INTERIOR, dwt2.DWT2_STRIP_BOUNDARY))
        for part in parts:
            for r in ranks:
                r.ctx.level(k, part, r.out, stream)
