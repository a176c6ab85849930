#!/usr/bin/env python
"""Benchmark of the forward 2-D CDF 5/3 DWT (non-separable lifting) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One "step" is one pass of the whole hot path over one batch of the workload:
every level of the forward transform of the config's image(s) (and, for row
strips at N > 1, the ghost-row exchange).  Default workload: BASELINE.json
config 3 (16384 x 16384 fp32, 1 level), the configuration the north-star
target ("70 % of HBM bandwidth per level on 16384 x 16384 fp32") is stated on;
at N > 1 it is split into N row strips whose halo rows the boundary kernels
read from the neighbour GPUs' memory (``--exchange peer``; ``nccl``: grouped
send/recv per level) -- strong scaling: the image is fixed.  Inputs are 1 GiB, larger than the 126 MB L2,
so no L2 flush is needed between steps.

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
and torch.cuda.synchronize() on both sides, CUDA events on the launching
stream, max over ranks (``value``, ``ms_per_step``).  Then, outside the timed
region: the correctness gate on the timed outputs against the CPU oracle
(``gate``; a mismatch exits 3 with no timing printed), and a
second pass of --stat-steps (default 100) steps with an event between steps
for the median / min / p90 per step (the paper's median of 100, PAPER.md
L305-306; ``step_stats``).  Rank 0 prints one JSON line.

``--impl reference`` times the CPU oracle (oracle/, plain fp64 C) on the
host cores instead: each step is a bounded sample of the same workload (one
band per usable core, the bands the cpu_baseline leg times).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "forward 2-D CDF 5/3 DWT Gpixel/s and HBM GB/s vs peak, 1/2/4/8 B200"
UNIT = "Gpixel/s"
BYTES_PER_PX = 8            # algorithmic: 4 B read + 4 B written per pixel per level
# algorithmic bytes per pixel per level of the comparison schemes (each step one HBM pass; the in-place
# separable steps 2-4 read 4 B and write 2 B): see scripts/scheme_compare.py, DESIGN.md 5.3
SCHEME_BYTES = {"fused": 8, "fused_literal": 8, "fused_adapted": 8, "nonsep_naive": 8, "nonsep_lifting": 16,
                "nonsep_adapted": 16, "sep_conv": 16, "sep_lifting": 26}
SCHEME_STEPS = {"fused": 1, "fused_literal": 1, "fused_adapted": 1, "nonsep_naive": 1, "nonsep_lifting": 2,
                "nonsep_adapted": 2, "sep_conv": 2, "sep_lifting": 4}
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def config_dict(args, cfg, world):
    d = describe(cfg, world, args.steps)
    if args.wavelet != "cdf53":
        d["wavelet"] = args.wavelet
    if args.op != "forward":
        d["op"] = args.op
    if args.scheme != "fused":
        d["scheme"] = args.scheme
    return d


def kernel_label(args):
    if args.scheme != "fused":
        return f"{args.scheme} scheme kernels ({SCHEME_STEPS[args.scheme]} per level)"
    if args.op == "inverse":
        return "dwt53_inverse kernel" if args.wavelet == "cdf53" else "dwt_k2_inverse_kernel"
    return "dwt53_level_kernel" if args.wavelet == "cdf53" else "dwt_k2_level_kernel"


def metric_name(args):
    m = METRIC if args.wavelet == "cdf53" else METRIC.replace("CDF 5/3", "CDF 9/7")
    if args.op == "inverse":
        m = m.replace("forward", "inverse", 1)
    if args.scheme != "fused":
        m = m.replace("DWT", f"DWT ({args.scheme} scheme, one kernel per step)", 1)
    return m


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="3", choices=["1", "2", "3", "4", "4b", "5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--op", default="forward", choices=["forward", "inverse"],
                    help="inverse: time the inverse transform (SURVEY 8f N2) of the config's pyramid")
    ap.add_argument("--scheme", default="fused", choices=["fused", "fused_literal", "fused_adapted", "nonsep_naive",
                                                        "nonsep_lifting", "nonsep_adapted", "sep_conv", "sep_lifting"],
                    help="forward with one of the paper's schemes, one kernel per step (SURVEY 8f N1)")
    ap.add_argument("--wavelet", default="cdf53", choices=["cdf53", "cdf97"],
                    help="cdf97: the K = 2 non-separable kernel (SURVEY 8f N4); single-image and batch configs")
    ap.add_argument("--no-overlap", action="store_true", help="strips, --exchange nccl: exchange, then one launch")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="row strips (N > 1): peer = halo rows read from the neighbours' memory inside the "
                         "BOUNDARY kernels (CUDA IPC over NVLink; the step is one CUDA graph); nccl = grouped "
                         "NCCL send/recv of the ghost rows per level, host-launched")
    ap.add_argument("--no-graph", action="store_true", help="launch every step from the host instead of "
                    "replaying a CUDA graph of it")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0, help="oracle sample rows (0 = auto)")
    ap.add_argument("--stat-steps", type=int, default=100,
                    help="steps of the per-step timing pass (median / min / p90; the paper's median of 100)")
    ap.add_argument("--no-gate", action="store_true", help="skip the correctness gate (sweeps only)")
    ap.add_argument("--variant-lib", default=None, help="measurement sweeps: load this build of libdwt2 "
                    "(build/variants/...) instead of the in-tree product library")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------------------
# clocks (NVML polled from a thread during the timed region)
# ----------------------------------------------------------------------------
class ClockSampler:
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
               "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
               "display_clock_setting": 0x100}

    def __init__(self, device_index: int):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed region"
        if not inside:   # region shorter than the poll period: nearest samples
            inside = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:3]
            window = "adjacent to timed region"
        reasons = set()
        for _, _, rs in inside:
            for name, bit in self.REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in inside]) if inside else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(inside),
                "window": window}


# ----------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------
def buffer_pairs(cfg, steps):
    """Input/output pairs the timed steps cycle over (see OursRunner)."""
    if cfg.pixels * 8 >= 2 * 126e6:
        return 1
    return min(max(1, steps), int(-(-2 * 126e6 // (cfg.pixels * 8))) + 1)


def describe(cfg, world, steps=20):
    g0 = cfg.groups[0]
    if cfg.name == "5":
        images = "256x2048^2 + 32x4095x3001"
    else:
        images = f"{g0.width}x{g0.height}"
    return {"workload": f"config {cfg.name}: {cfg.description}", "images": images, "levels": cfg.levels,
            "pixels": cfg.pixels, "input": "fp32, seeded synthetic, resident in HBM",
            "l2": "inputs larger than the 126 MB L2; no flush between steps" if cfg.pixels * 8 >= 2 * 126e6
            else ("timed steps cycle over %d input/output pairs, each reused only after > 2x L2 of other traffic "
                  "(or read once); L2 flushed (256 MB read pass) once before the timed region"
                  % buffer_pairs(cfg, steps)),
            "parallelism": ("row strips x%d, %s halo exchange per level" % (world, OursRunner.exchange_label())
                            if cfg.name in ("1", "2", "3", "4", "4b")
                            and world > 1 else ("image shards x%d, no communication" % world if world > 1
                                                else "single GPU"))}


class OursRunner:
    """Device-resident inputs; step() enqueues one full forward on the current stream."""

    def __init__(self, cfg, rank, world, device):
        import torch
        from paper_1708_07853_b200 import dwt2
        from paper_1708_07853_b200 import distributed as D
        self.cfg, self.rank, self.world = cfg, rank, world
        self.dwt2, self.D = dwt2, D
        self.torch = torch
        self.flush = None
        # inputs + outputs smaller than 2x the 126 MB L2: every timed step gets
        # its own input/output pair (K distinct pairs) and the L2 is flushed
        # once (read-only pass) before the timed region
        self.small = cfg.pixels * 8 < 2 * 126e6
        if self.small:
            self.flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=device)   # 256 MB
            self.flush_sink = torch.zeros((), dtype=torch.float32, device=device)
        # buffer pairs cycled through the K timed steps: enough that a pair is
        # reused only after more than 2x L2 of other traffic (then none of its
        # lines can still be cached), at most K (each pair then read once after
        # the flush).  Touching K distinct pairs when fewer suffice costs a
        # mid-size level ~25 % more time per step for reasons outside the L2
        # (config 2: 26 us with 2-4 pairs, 33 us with 10-20; a plain copy does
        # not show it; scripts/c2_protocol.py) -- not what a stream of images
        # through a few buffers sees.
        self.nbuf = buffer_pairs(cfg, self.steps)
        self.i = 0
        self.launches = 0
        self.algo_bytes = 0           # algorithmic bytes one step moves on this rank
        self.level1_bytes = 0
        self.pixels = 0               # finest-level pixels this rank transforms per step
        self.h2d = self.d2h = 0
        self.sha = hashlib.sha256()     # of every input image this rank transforms, in order
        if cfg.name == "5":
            self.items, self.batch_meta = [], []
            for grp in cfg.groups:
                idx = D.shard(grp.count, rank, world)
                if len(idx) == 0:
                    continue
                xs = np.stack([grp.image(i) for i in idx])
                self.sha.update(xs.tobytes())
                x = torch.from_numpy(xs).to(device)
                out = torch.empty_like(x)
                plan = dwt2.Plan(grp.width, grp.height, cfg.levels, max_count=len(idx), wavelet=self.wavelet)
                info = plan.info()
                if self.op == "inverse":
                    x = plan.forward(x).clone()          # the pyramid is the inverse's input
                self.items.append((plan, x, out))
                self.batch_meta.append((grp, idx))
                self.launches += info.launches_per_forward * SCHEME_STEPS[self.scheme]
                self.algo_bytes += info.algorithmic_bytes * len(idx) * SCHEME_BYTES[self.scheme] // BYTES_PER_PX
                self.level1_bytes += SCHEME_BYTES[self.scheme] * grp.width * grp.height * len(idx)
                self.pixels += grp.width * grp.height * len(idx)
            self.mode = "batch"
        elif world == 1:
            g = cfg.groups[0]
            self.host_img = g.image(0)
            self.sha.update(self.host_img.tobytes())
            x = torch.from_numpy(self.host_img).to(device)
            self.plan = dwt2.Plan(g.width, g.height, cfg.levels, wavelet=self.wavelet)
            if self.op == "inverse":
                x = self.plan.forward(x).clone()           # the pyramid is the inverse's input
            self.xs = [x] + [x.clone() for _ in range(self.nbuf - 1)]
            self.outs = [torch.empty_like(x) for _ in range(self.nbuf)]
            self.x, self.out = x, self.outs[0]
            info = self.plan.info()
            self.launches = info.launches_per_forward * SCHEME_STEPS[self.scheme]
            self.algo_bytes = info.algorithmic_bytes * SCHEME_BYTES[self.scheme] // BYTES_PER_PX
            self.level1_bytes = SCHEME_BYTES[self.scheme] * g.width * g.height
            self.pixels = g.width * g.height
            self.mode = "single"
        else:
            # row strips, one ghost-row exchange per level (levels > 1: SURVEY 8f N3)
            g = cfg.groups[0]
            img = g.image(0)
            self.sha.update(img.tobytes())
            if self.exchange == "peer":
                # flag waits take microseconds; a 2 s bound turns a broken mapping into a
                # quick failure (checked after the warm-up) instead of a long hang
                self.ex = D.PeerStripPyramid(g.width, g.height, rank, world, cfg.levels, device=device,
                                             timeout_ms=2000)
                try:
                    self.ex.connect()          # all_gather of the CUDA IPC descriptors (once)
                    ok = 1
                except dwt2.DWT2Error as e:   # e.g. no CUDA IPC between the processes
                    ok, self.peer_error = 0, str(e)
                import torch.distributed as dist
                flag = torch.tensor([ok], device=device)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                if not int(flag.item()):
                    # every rank switches to the NCCL exchange together (a GPU path too)
                    self.ex.close()
                    OursRunner.exchange = "nccl"
                    self.exchange_note = "peer mapping failed (%s): NCCL exchange" % getattr(self, "peer_error", "another rank")
                self.splan = None
            if self.exchange == "nccl":
                self.ex = D.StripPyramid(g.width, g.height, rank, world, cfg.levels, device=device)
                self.splan = dwt2.StripPlan(g.width, g.height, self.ex.r0, self.ex.r1, cfg.levels)
            r0, r1 = self.ex.r0, self.ex.r1
            self.ex.strip.copy_(torch.from_numpy(np.ascontiguousarray(img[r0:r1])))
            self.out = self.ex.out
            # peer: one launch per level (interior tiles + boundary-role CTAs); nccl: interior + boundary
            self.launches = cfg.levels * (1 if (self.overlap_off or self.exchange == "peer") else 2)
            self.algo_bytes = sum(BYTES_PER_PX * w * (re - rb) for (w, h, rb, re, gt, gb) in self.ex.geom)
            self.level1_bytes = BYTES_PER_PX * g.width * (r1 - r0)
            self.pixels = g.width * (r1 - r0)
            self.mode = "strip"
            self.host_img = img

    overlap_off = False
    exchange = "peer"
    wavelet = "cdf53"

    @classmethod
    def exchange_label(cls):
        return "peer-memory (NVLink loads in the boundary kernels)" if cls.exchange == "peer" else "NCCL send/recv"

    def strip_step(self):
        if self.exchange == "peer":
            self.ex.step()
        else:
            self.D.strip_pyramid_step(self.ex, self.splan, overlap=not self.overlap_off)
    steps = 20
    op = "forward"
    scheme = "fused"

    def call(self, plan, x, out):
        """The timed operation on one buffer pair."""
        if self.op == "inverse":
            plan.inverse(x, out)
        elif self.scheme != "fused":
            plan.forward_scheme(self.scheme, x, out)
        else:
            plan.forward(x, out)

    def flush_l2(self):
        """Evict the L2 with clean lines: a read-only pass over 256 MB (a
        write-based flush would leave ~126 MB of dirty lines whose write-back
        lands in the next timed step)."""
        if self.flush is not None:
            self.flush_sink.copy_(self.flush.amax())

    def step(self):
        if self.mode == "single":
            j = self.i % self.nbuf
            self.i += 1
            self.call(self.plan, self.xs[j], self.outs[j])
        elif self.mode == "batch":
            for plan, x, out in self.items:
                self.call(plan, x, out)
        else:
            self.strip_step()

    def level1_kernel_ms(self, iters):
        """Average duration of the dominant kernel (level 1: 3/4 of the
        algorithmic bytes of a pyramid), CUDA events on its launch stream,
        through level-1-only plans on the same buffers."""
        torch = self.torch
        s = torch.cuda.current_stream()
        if self.mode == "single" and self.cfg.levels == 1:
            return None   # identical to the step: caller uses the step time
        if self.mode == "strip":
            return None
        if self.mode == "single":
            plans = [(self.dwt2.Plan(self.cfg.groups[0].width, self.cfg.groups[0].height, 1, wavelet=self.wavelet),
                       self.x, self.out)]
        else:
            plans = [(self.dwt2.Plan(p.width, p.height, 1, max_count=x.shape[0], wavelet=self.wavelet), x, o)
                     for p, x, o in self.items]
        for p, x, o in plans:          # warm-up (tensor maps, first-launch costs)
            self.call(p, x, o)
        torch.cuda.synchronize()
        # back to back between one event pair (event ticks are 2.048 us);
        # with a flush, K flushes timed alone are subtracted
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            self.flush_l2()
            for p, x, o in plans:
                self.call(p, x, o)
        e1.record(s)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(s)
        for _ in range(iters):
            self.flush_l2()
        f1.record(s)
        torch.cuda.synchronize()
        for p, _, _ in plans:
            p.close()
        return (e0.elapsed_time(e1) - f0.elapsed_time(f1)) / iters

    def e2e(self, steps, warm):
        """Same metric through the public API with HOST buffers: H2D of the
        step's input from pinned memory and D2H of its result are inside the
        timed region (the C-ABI dwt2_forward_host pipelines them by row band)."""
        torch = self.torch
        if self.mode == "single" and (self.op != "forward" or self.scheme != "fused" or self.wavelet != "cdf53"):
            # inverse / schemes / 9/7: H2D of the input, the operation, D2H of the result
            hin = self.x.cpu().pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            s = torch.cuda.current_stream()

            def one():
                self.x.copy_(hin, non_blocking=True)
                self.call(self.plan, self.x, self.out)
                hout.copy_(self.out, non_blocking=True)
            for _ in range(warm):
                one()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(steps):
                one()
            e1.record(s)
            e1.synchronize()
            self.h2d = self.d2h = hin.numel() * 4
            return e0.elapsed_time(e1) / 1e3 / steps
        if self.mode == "single":
            hin = torch.from_numpy(self.host_img).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            for _ in range(warm):
                self.plan.forward_host(hin, hout)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                self.plan.forward_host(hin, hout)
            dt = (time.perf_counter() - t0) / steps
            self.h2d = self.d2h = hin.numel() * 4
            return dt
        if self.mode == "strip":
            hin = torch.from_numpy(np.ascontiguousarray(self.ex.strip.cpu().numpy())).pin_memory()
            hout = torch.empty(self.out.shape, dtype=torch.float32).pin_memory()
            s = torch.cuda.current_stream()
            def one():
                self.ex.strip.copy_(hin, non_blocking=True)
                self.strip_step()
                hout.copy_(self.out, non_blocking=True)
            for _ in range(warm):
                one()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(steps):
                one()
            e1.record(s)
            e1.synchronize()
            self.h2d, self.d2h = hin.numel() * 4, hout.numel() * 4
            return e0.elapsed_time(e1) / 1e3 / steps
        # batch: chunks of images pipelined through three streams -- H2D of
        # chunk i+1 || the batched call on chunk i || D2H of chunk i-1
        hosts = [(torch.empty(x.shape, dtype=torch.float32).pin_memory(),
                  torch.empty(x.shape, dtype=torch.float32).pin_memory()) for _, x, _ in self.items]
        for (hi, _), (_, x, _) in zip(hosts, self.items):
            hi.copy_(x.cpu())
        s = torch.cuda.current_stream()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        CH = 8                                   # images per chunk

        def one():
            up.wait_stream(s)                    # the previous step's calls are done with the inputs
            for (hi, ho), (plan, x, o) in zip(hosts, self.items):
                for i0 in range(0, x.shape[0], CH):
                    i1 = min(x.shape[0], i0 + CH)
                    with torch.cuda.stream(up):
                        x[i0:i1].copy_(hi[i0:i1], non_blocking=True)
                        landed = torch.cuda.Event()
                        landed.record(up)
                    s.wait_event(landed)
                    self.call(plan, x[i0:i1], o[i0:i1])
                    done = torch.cuda.Event()
                    done.record(s)
                    with torch.cuda.stream(down):
                        down.wait_event(done)
                        ho[i0:i1].copy_(o[i0:i1], non_blocking=True)
            s.wait_stream(down)                  # the step ends when its results are on the host
        for _ in range(warm):
            one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            one()
        e1.record(s)
        e1.synchronize()
        self.h2d = sum(h.numel() * 4 for h, _ in hosts)
        self.d2h = self.h2d
        return e0.elapsed_time(e1) / 1e3 / steps


ORACLE_BAND_PX = 1 << 23        # pixels per oracle band (64 MiB of fp64 input: not cache-resident)
MAX_ORACLE_THREADS = 256        # bounds the host memory of the all-cores leg (~64 MiB of output per thread)


def cpu_info():
    """Host facts recorded with every oracle timing."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"nproc": usable, "cpu_count": os.cpu_count(), "cpu_model": model}


def oracle_bands(cfg, wavelet: str = "cdf53", op: str = "forward", rows: int = 0, threads: int = 1):
    """The bounded sample of the workload both oracle legs time (cpu_baseline
    and --impl reference): full-width bands of ``rows`` rows of the config's
    first image (whole images' first rows for config 5), each transformed as a
    standalone image with the config's levels.  Band i is rows [i R, (i+1) R)
    (wrapping inside the image), so ``threads`` threads each own one band.
    Returns (fns, pixels per band, levels, text)."""
    import oracle
    g = cfg.groups[0]
    if rows <= 0:
        rows = max(64, min(g.height, ORACLE_BAND_PX // g.width))
    rows -= rows % 2
    img = g.image(0)
    nb = max(1, g.height // rows)
    w, h, L = g.width, rows, 0          # every level must stay >= 2 x 2
    while L < cfg.levels and w >= 2 and h >= 2:
        w, h, L = (w + 1) // 2, (h + 1) // 2, L + 1
    fns, bands = [], {}
    for i in range(threads):
        b = i % nb
        if b not in bands:                  # read-only inputs are shared by the threads that wrap around
            bands[b] = np.ascontiguousarray(img[b * rows:(b + 1) * rows], dtype=np.float64)
        x64 = bands[b]
        if op == "inverse":
            y64 = oracle.forward(x64, L, round_f32=True, wavelet=wavelet)      # the band's pyramid (untimed)
            fns.append(lambda y64=y64: oracle.inverse(y64, L, round_f32=True, wavelet=wavelet))
        else:
            fns.append(lambda x64=x64: oracle.forward(x64, L, round_f32=True, wavelet=wavelet))
    if op == "inverse":
        alg = "C97 (9/7 inverse lifting" if wavelet == "cdf97" else "C (inverse lifting"
    else:
        alg = "A97 (separable 9/7 lifting" if wavelet == "cdf97" else "A (separable lifting"
    text = (f"{threads} band(s) of {g.width}x{rows} rows of image 0 of config {cfg.name} (band i = rows "
            f"[i*{rows}, (i+1)*{rows}) mod {nb} bands), {L} level(s) each, oracle algorithm {alg}, fp64, "
            f"fp32 storage between levels), one thread per band")
    return fns, g.width * rows, L, text


def run_threads(fns):
    """Run every fn on its own thread (the oracle's ctypes calls release the
    GIL) and return the wall time of the whole set."""
    ts = [threading.Thread(target=f) for f in fns]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return time.perf_counter() - t0


def oracle_baseline(cfg, wavelet, op, rows=0, reps=3):
    """The oracle as it stands on the host cores: one thread on band 0, and
    all usable cores with one band each (median of ``reps`` runs each)."""
    info = cpu_info()
    cores = max(1, min(MAX_ORACLE_THREADS, info["nproc"] or 1))
    fns1, px, L, text1 = oracle_bands(cfg, wavelet, op, rows, 1)
    t1 = statistics.median(run_threads(fns1) for _ in range(reps))
    fnsn, _, _, textn = oracle_bands(cfg, wavelet, op, rows, cores)
    tn = statistics.median(run_threads(fnsn) for _ in range(reps))
    return {"value": cores * px / tn / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": textn,
            "median_of": reps, "one_thread": {"value": px / t1 / 1e9, "cores": 1, "sample": text1},
            "scaling_all_cores": (cores * px / tn) / (px / t1), **info}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(cfg_name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        e = d.get("configs", {}).get(cfg_name)
        return None if e is None else e.get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------
# correctness gate (after the timed region, on the timed outputs; SPEC.md L495:
# no timing of wrong code).  The oracle is test infrastructure: this gate, the
# cpu_baseline leg and --impl reference are the only places bench.py runs it.
# ----------------------------------------------------------------------------
GATE_TOL_I = 1e-4                 # BASELINE.json north_star: max-abs vs the fp64 oracle (i)
GATE_FULL_PX = 150_000_000        # whole-output oracle comparison up to this many (level-weighted) pixels
GATE_RANDOM = 25_000              # random positions per subband in sampled checks (+ every border quad)
GATE_RT97 = 1e-3                  # round trip |inverse(forward(x)) - x| bound (fp32-stored coefficients)


def _bands1(W, H):
    """(row0, col0, rows, cols) of the level-1 LL, HL, LH, HH in the Mallat layout."""
    wl, hl = (W + 1) // 2, (H + 1) // 2
    return [(0, 0, hl, wl), (0, wl, hl, W // 2), (hl, 0, H // 2, wl), (hl, wl, H // 2, W // 2)]


def _positions(W, H, bands, rng, q0=0, q1=None):
    """Every border quad of each listed level-1 subband (first / last 2 rows and
    columns, and the first / last 2 of the quad rows [q0, q1) a strip owns) plus
    GATE_RANDOM random positions, restricted to quad rows [q0, q1)."""
    B, M, N = [], [], []
    for b in bands:
        _, _, rows, cols = _bands1(W, H)[b]
        lo, hi = q0, rows if q1 is None else min(q1, rows)
        if hi <= lo or cols == 0:
            continue
        rs = np.unique(np.clip(np.r_[0, 1, rows - 2, rows - 1, lo, lo + 1, hi - 2, hi - 1], lo, hi - 1))
        cs = np.unique(np.clip(np.r_[0, 1, cols - 2, cols - 1], 0, cols - 1))
        mm, nn = np.meshgrid(np.arange(cols), rs)
        B.append(np.full(mm.size, b)); M.append(mm.ravel()); N.append(nn.ravel())
        mm, nn = np.meshgrid(cs, np.arange(lo, hi))
        B.append(np.full(mm.size, b)); M.append(mm.ravel()); N.append(nn.ravel())
        B.append(np.full(GATE_RANDOM, b)); M.append(rng.integers(0, cols, GATE_RANDOM))
        N.append(rng.integers(lo, hi, GATE_RANDOM))
    return np.concatenate(B), np.concatenate(M), np.concatenate(N)


class Gate:
    """Collects the checks of one rank; fail() records the first mismatch."""

    def __init__(self):
        self.checks, self.n, self.max_i, self.failed = [], 0, 0.0, None

    def compare(self, what, got, ref, exact):
        got = np.asarray(got, dtype=np.float64)
        ref = np.asarray(ref, dtype=np.float64)
        self.n += got.size
        if not np.all(np.isfinite(got)):
            self.failed = self.failed or f"{what}: non-finite output"
            return
        d = np.abs(got - ref)
        if exact:
            bad = int(np.count_nonzero(d))
            if bad:
                self.failed = self.failed or f"{what}: {bad} of {got.size} not bit-exact (max {d.max():.3g})"
        else:
            dm = float(d.max()) if d.size else 0.0
            self.max_i = max(self.max_i, dm)
            if dm > GATE_TOL_I:
                self.failed = self.failed or f"{what}: max abs {dm:.3g} > {GATE_TOL_I}"
        self.checks.append(what)

    def check(self, what, ok):
        self.checks.append(what)
        if not ok:
            self.failed = self.failed or what


def gate(runner, cfg, args):
    """Check the outputs of the timed steps against the oracle (see module notes
    in DESIGN.md 7): whole outputs where the oracle finishes in seconds, else
    level-1 coefficients at every border quad plus random positions (the
    oracle's pointwise convolution, algorithm B) and the exactness grid."""
    import oracle
    from paper_1708_07853_b200 import workloads
    torch = runner.torch
    t0 = time.perf_counter()
    G = Gate()
    rng = np.random.default_rng(20260)
    wav, L, op = args.wavelet, cfg.levels, args.op
    integer = cfg.groups[0].kind == "uniform"
    fused = args.scheme in ("fused", "fused_literal", "fused_adapted")
    # 5/3 with fp64 register math reaches oracle (ii) bit for bit; the kernel-per-step
    # schemes store fp32 between steps, which is exact only on the integer grid (<= 2 levels)
    exact = wav == "cdf53" and (fused or (integer and L <= 2))

    def ref_forward(x64, levels, ex):
        return oracle.forward(x64, levels, round_f32=ex, wavelet=wav)

    def full_forward(what, img, out, levels):
        G.compare(what, out, ref_forward(img.astype(np.float64), levels, exact), exact)

    def full_inverse(what, pyr, out, levels, orig):
        if wav == "cdf53":
            G.compare(what, out, oracle.inverse(pyr.astype(np.float64), levels, round_f32=True), True)
        else:
            G.compare(what, out, oracle.inverse(pyr.astype(np.float64), levels, round_f32=False, wavelet=wav), False)
        rt = float(np.abs(out.astype(np.float64) - orig).max())
        if wav == "cdf53" and integer and levels <= 2:
            G.check(what + " round trip exact", rt == 0.0)
        else:
            G.check(what + f" round trip max abs {rt:.3g} <= {GATE_RT97}", rt <= GATE_RT97)

    def sampled_level1(what, img, out_rows, W, H, bands, q0=0, q1=None):
        """out_rows(band, n) -> output row index of level-1 quad row n of `band`."""
        b, m, n = _positions(W, H, bands, rng, q0, q1)
        ref = oracle.conv_sample(img, b, m, n, wavelet=wav)
        c0 = np.array([c for (_, c, _, _) in _bands1(W, H)])[b]
        got = out_rows(b, n, m + c0)
        G.compare(what, got, ref.astype(np.float32) if exact else ref, exact)

    if runner.mode == "single":
        g = cfg.groups[0]
        W, H = g.width, g.height
        outs = runner.outs[:runner.nbuf]
        ref_out = outs[(runner.i - 1) % runner.nbuf]
        G.check("all timed output buffers identical", all(torch.equal(o, ref_out) for o in outs))
        out = ref_out.cpu().numpy()
        img = runner.host_img
        heavy = workloads.level_pixels(W, H, L) * (3 if wav == "cdf97" else 1)
        if op == "inverse":
            pyr = runner.x.cpu().numpy()
            if heavy <= 2 * GATE_FULL_PX:             # the inverse oracle over the whole pyramid: <= ~30 s
                full_inverse(f"inverse {W}x{H} L{L}: every element vs oracle", pyr, out, L, img)
            elif wav == "cdf53" and integer and L <= 2:
                G.compare(f"inverse {W}x{H} L{L}: round trip, every element (exact)", out, img, True)
            else:
                # no pointwise inverse oracle: the round trip through fp32-stored coefficients
                rt = float(np.abs(out.astype(np.float64) - img).max())
                G.n += out.size
                G.check(f"inverse {W}x{H} L{L}: round trip max abs {rt:.3g} <= {GATE_RT97}", rt <= GATE_RT97)
        elif heavy <= GATE_FULL_PX:
            full_forward(f"forward {W}x{H} L{L}: every element vs oracle", img, out, L)
        else:
            bands = [0, 1, 2, 3] if L == 1 else [1, 2, 3]
            sampled_level1(f"forward {W}x{H}: level-1 border quads + random positions vs oracle B",
                           img, lambda b, n, col: out[np.array([r for (r, _, _, _) in _bands1(W, H)])[b] + n, col],
                           W, H, bands)
            if wav == "cdf53" and integer and L <= 2:
                o = ref_out
                q = 64.0 if L == 1 else 4096.0
                G.check(f"every coefficient on the 1/{int(q)} grid, |c| <= 2295",
                        bool(torch.equal(o * q, torch.round(o * q))) and float(o.abs().max()) <= 2295.0)
    elif runner.mode == "batch":
        for (plan, x, out_t), (grp, idx) in zip(runner.items, runner.batch_meta):
            outs = out_t.cpu().numpy()
            for j in sorted({0, len(idx) - 1}):
                img = grp.image(idx[j])
                what = f"{'inverse' if op == 'inverse' else 'forward'} {grp.width}x{grp.height} image {idx[j]} L{L}"
                if op == "inverse":
                    full_inverse(what + ": every element vs oracle", x[j].cpu().numpy(), outs[j], L, img)
                else:
                    full_forward(what + ": every element vs oracle", img, outs[j], L)
    else:
        # row strip of this rank: level-1 coefficients of its quad rows (strip-local Mallat)
        g = cfg.groups[0]
        W, H = g.width, g.height
        ex = runner.ex
        qs, qe = ex.r0 // 2, (ex.r1 + 1) // 2
        hq_loc, Wq = qe - qs, (W + 1) // 2
        out = runner.out.cpu().numpy()

        def rows(b, n, col):
            r = np.where(b < 2, n - qs, hq_loc + (n - qs))
            return out[r, col]
        bands = [0, 1, 2, 3] if L == 1 else [1, 2, 3]
        sampled_level1(f"rank strip rows [{ex.r0}, {ex.r1}): level-1 border quads + random positions vs oracle B",
                       runner.host_img, rows, W, H, bands, qs, qe)
    return {"status": "fail" if G.failed else "pass", "error": G.failed, "elements_checked": G.n,
            "checks": G.checks, "max_abs_vs_oracle_i": G.max_i if not exact else 0.0,
            "bit_exact_vs_oracle_ii": exact, "seconds": round(time.perf_counter() - t0, 2)}


# ----------------------------------------------------------------------------
def run_reference(args, cfg):
    """The reference arm: the oracle as it stands on the box's host cores (one
    thread per band, all usable cores), each step one bounded sample of the
    workload -- the same bands as the cpu_baseline leg."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    info = cpu_info()
    cores = max(1, min(MAX_ORACLE_THREADS, info["nproc"] or 1))
    fns, px, L, text = oracle_bands(cfg, args.wavelet, args.op, args.cpu_sample_rows, cores)
    for _ in range(args.warmup):
        run_threads(fns)
    times = [run_threads(fns) for _ in range(args.steps)]
    dt = sum(times) / len(times)
    v = cores * px / dt / 1e9
    line = {"impl": "reference", "metric": metric_name(args), "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(args, cfg, 1),
            "step_stats": {"median_ms": statistics.median(times) * 1e3, "min_ms": min(times) * 1e3,
                           "p90_ms": float(np.percentile(times, 90)) * 1e3, "n": len(times)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": text, **info},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def step_stats(runner, args, use_graph, barrier, ms_mean, device, world):
    """Per-step device times of --stat-steps steps: median / min / p90 (max over
    ranks per step), with a CUDA event between consecutive steps."""
    import torch
    n = max(args.steps, args.stat_steps)
    if ms_mean < 0.02:
        return {"note": f"steps of {ms_mean * 1e3:.1f} us are below the 2.048 us event tick x 10: "
                        "only the K-step mean is reported", "n": 0}
    stream = torch.cuda.current_stream()
    if use_graph:
        runner.i = 0
        g = torch.cuda.CUDAGraph()
        evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(n + 1)]
        with torch.cuda.graph(g):
            evs[0].record()
            for i in range(n):
                runner.step()
                evs[i + 1].record()
        g.replay()                     # warm-up replay
        torch.cuda.synchronize()
        if runner.small:
            runner.flush_l2()
        barrier()
        torch.cuda.synchronize()
        g.replay()
    else:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        barrier()
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(n):
            runner.step()
            evs[i + 1].record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([evs[i].elapsed_time(evs[i + 1]) for i in range(n)], device=device, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = t.cpu().numpy()
    return {"median_ms": float(np.median(t)), "min_ms": float(t.min()), "p90_ms": float(np.percentile(t, 90)),
            "max_ms": float(t.max()), "mean_ms": float(t.mean()), "n": int(n),
            "method": ("one CUDA graph replay, external CUDA events between steps (max over ranks per step)"
                       if use_graph else "host-launched steps, CUDA events between steps (max over ranks)")}


def warm_l2(runner, args):
    """Companion number for working sets that fit the L2 (configs 1, 2):
    K steps on ONE buffer pair, no flush (inputs L2-resident after the first)."""
    import torch
    if not runner.small or runner.mode != "single":
        return None
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(args.steps):
            runner.call(runner.plan, runner.xs[0], runner.outs[0])
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    return {"ms_per_step": ms, "value": runner.pixels / (ms * 1e-3) / 1e9, "unit": UNIT,
            "note": "one buffer pair, L2-warm (not the headline)"}


def main():
    args = parse()
    from paper_1708_07853_b200 import workloads
    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    if args.variant_lib:
        from paper_1708_07853_b200 import dwt2
        dwt2.use_variant(args.variant_lib)
    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
        dist.barrier()          # communicator up before the first grouped send/recv (all ranks)

    OursRunner.overlap_off = args.no_overlap
    OursRunner.exchange = args.exchange
    OursRunner.steps = args.steps
    OursRunner.op = args.op
    OursRunner.scheme = args.scheme
    if (args.op != "forward" or args.scheme != "fused") and world > 1 and cfg.name != "5":
        raise SystemExit("row strips run the forward fused kernel only")
    if args.scheme != "fused" and (args.op != "forward" or args.wavelet != "cdf53"):
        raise SystemExit("the comparison schemes are forward CDF 5/3")
    OursRunner.wavelet = args.wavelet
    if args.wavelet != "cdf53" and world > 1 and cfg.name != "5":
        raise SystemExit("row strips run the CDF 5/3 kernel only")
    runner = OursRunner(cfg, rank, world, device)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        runner.step()
    torch.cuda.synchronize()
    if runner.mode == "strip" and OursRunner.exchange == "peer":
        # a timed-out flag wait on any rank (DWT2_ETIMEOUT): no timing of a broken exchange
        bad = torch.tensor([0 if runner.ex.status() == 0 else 1], device=device)
        if world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()):
            if rank == 0:
                print(json.dumps({"metric": metric_name(args), "error": "peer halo exchange timed out during "
                                  "the warm-up (DWT2_ETIMEOUT): no timing is reported"}), flush=True)
            raise SystemExit(3)
    graph = None
    if not args.no_graph and (runner.mode != "strip" or OursRunner.exchange == "peer"):
        # the K timed steps as ONE CUDA graph (the level kernels keep their
        # programmatic dependent-launch edges): no host launch gaps, and the
        # NVML sampler thread cannot gate the GPU
        runner.i = 0
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(args.steps):
                runner.step()
        graph.replay()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    if runner.small:
        runner.flush_l2()
    barrier()
    torch.cuda.synchronize()
    t_host0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        runner.i = 0
        for _ in range(args.steps):
            runner.step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t_host1 = time.perf_counter()
    barrier()
    sampler.stop()

    # correctness gate on the outputs of the timed steps (never inside the timed region)
    gate_res = {"status": "skipped"} if args.no_gate else gate(runner, cfg, args)
    bad = torch.tensor([1.0 if gate_res["status"] == "fail" else 0.0], device=device)
    if world > 1:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    if float(bad.item()) > 0:
        if rank == 0 or gate_res["status"] == "fail":
            print(json.dumps({"metric": metric_name(args), "gate": gate_res, "rank": rank,
                              "error": "correctness gate failed: no timing is reported"}), flush=True)
        raise SystemExit(3)

    # per-step statistics (the paper's protocol: median of 100 measurements,
    # PAPER.md L305-306): one more replay of --stat-steps steps with a CUDA event
    # between consecutive steps, recorded inside the graph (external events, so
    # no host gap between steps); steps shorter than ~20 us are below the
    # 2.048 us event tick and get no per-step numbers
    stats = step_stats(runner, args, graph is not None, barrier, ms, device, world)
    warm = warm_l2(runner, args) if graph is not None else None
    ms_t = torch.tensor([ms], device=device)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_px = cfg.pixels
    value = total_px / (ms_max * 1e-3) / 1e9

    # dominant kernel (level 1) duration
    k_ms = runner.level1_kernel_ms(max(3, args.steps))
    if k_ms is None:
        # one-level configs: the level (all its step kernels for a scheme) is the step;
        # row strips: level 1's share of the step by algorithmic bytes (the exchange included)
        if runner.mode == "strip":
            k_ms = ms * runner.level1_bytes / max(1, runner.algo_bytes)
        else:
            k_ms = ms / max(1, runner.launches // SCHEME_STEPS[args.scheme])
    k_bytes = runner.level1_bytes
    achieved = k_bytes / (k_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    # key of the committed ncu capture: config [+ _cdf97] [+ _inverse]
    tkey = cfg.name + ("" if args.wavelet == "cdf53" else f"_{args.wavelet}") + ("_inverse" if args.op == "inverse" else "")
    traffic = ncu_traffic(tkey) if world == 1 and args.scheme == "fused" else None

    # end to end through the host-buffer API
    e2e = None
    if not args.no_e2e:
        e_steps = max(1, min(args.steps, 10))
        dt = runner.e2e(e_steps, 1)
        dt_t = torch.tensor([dt], device=device)
        if world > 1:
            dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
        e2e = {"value": total_px / float(dt_t.item()) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(runner.h2d) * world, "d2h_bytes_per_step": int(runner.d2h) * world}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(cfg, args.wavelet, args.op, args.cpu_sample_rows)

    if rank == 0:
        clocks = sampler.summary(t_host0, t_host1)
        runner_sha = runner.sha.hexdigest()
        algo_bytes_total = runner.algo_bytes * world if cfg.name != "5" else sum(
            BYTES_PER_PX * workloads.level_pixels(g.width, g.height, cfg.levels) * g.count for g in cfg.groups)
        line = {
            "metric": metric_name(args),
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_dict(args, cfg, world),
                           **({"exchange_note": runner.exchange_note} if getattr(runner, "exchange_note", None) else {})),
            "gate": gate_res,
            "step_stats": stats,
            "warm_l2": warm,
            "hbm_gbs_algorithmic": algo_bytes_total / (ms_max * 1e-3) / 1e9,
            "ns_per_pel": ms_max * 1e6 / total_px,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_label(args) + " (level 1)", "kernel_ms": k_ms,
                         "bytes_per_launch": k_bytes, "peak_source": peak_src,
                         "frac_of_8tbs": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": runner.launches * args.steps,
            "launch": "one CUDA graph of the K timed steps" if graph is not None else "host launches",
            "clocks": clocks,
        }
        line["config"]["input_sha256"] = runner_sha[:16] + (" (rank 0's inputs)" if world > 1 else "")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
