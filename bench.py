"""Benchmark: one GIS build-prune pass of BASELINE config 2 per step.

Workload (BASELINE.json configs[1]): damped pendulum, 1024 x 1024 uniform
grid (V = 1,048,576 cells), 21 inputs, 20 samples per cell (4 corners + 16
seeded-uniform, seed 0), RK4 with 10 substeps over dt = 0.05, bloat 0.1.
A step = grid index + enclosures/graph build (K1+K2) + non-leaving prune
(K3) + retention, i.e. the build and analyze phases of one engine iteration
(cg/engine.py:168-172).  Metric: (cell, control, sample) integrations per
second, I = V * 21 * 20 = 440,401,920 per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--gpus N > 1 started as a plain process re-executes itself under
torch.distributed.run, one rank per GPU (NCCL); under torchrun it runs as the
given rank.  Rows are sharded by contiguous CellId ranges and the prune
exchanges the bitmap per sweep (paper_2202_06111_b200.distributed).

--impl reference times the reference's own CPU implementation: the
unmodified cisgraph package (baseline/_ref) through its public API --
build_graph_parallel over all host cores, non_leaving_mask (Tarjan), retain
-- on a bounded sample of the same workload (a 128 x 128 block of cells at
full resolution, the aligned CellId range around the origin, built and
pruned as its own GIS pass) every step, plus one full config-2 pass as the
same-config anchor (--no-full-pass skips it).  Without baseline/_ref the
numpy port oracle/gis_oracle.py (pinned bit-exact to it) runs instead and
the line says kind "port".  Under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np

CONFIG_ID = 2
SAMPLE_LOG2 = 14          # CPU sample: 2^14 cells = a 128 x 128 block
SAMPLE_BLOCK = 48         # aligned block index containing the origin (path prefix 110000)
METRIC = "(cell,control,sample) integrations/s"
UNIT = "integrations/s"
# algorithmic fp64 flops per integration, pendulum RK4 x10:
# 6 (sample point) + 10 * (13n + 4*F_rhs) = 426 arithmetic + 40 sin calls.
ARITH_FLOPS = 426
SIN_CALLS = 40
# C_sin: SURVEY 8(d) freezes it at the executed DP flops of the sin the kernel
# calls.  K1 calls its own polynomial (gis_math.cuh: 7 DFMA + 2 DMUL = 16
# flops), not CUDA libm's (26), so 426 + 40*16 = 1066 flops per integration,
# which is also what ncu counts as executed (DFMA = 2).
SIN_FLOPS = 16
LIBM_SIN_FLOPS = 26       # reported beside it: the same work priced at CUDA libm's sin
# fp64-pipe instructions per integration in the shipped K1 (cuobjdump of the
# pendulum RK4 instantiation): 58 per RK4 substep (48 DFMA + 8 DMUL + 2 DADD)
# x 10, 6 for the sample point, 4 min/max compares; every one takes one fp64
# issue slot, DFMA or not.  ncu's executed DFMA:DMUL:DADD counts of the r01h
# capture give 480 : 84 : 22 per integration, i.e. the same 586 + 4.
DP_INSTR_PER_INT = 590
L2_FLUSH_BYTES = 512 << 20
NCU_SUMMARY = "ncu_step_r02bo.json"  # tools/make_ncu_summary.py of the committed capture
NCU_PEEL_SUMMARY = "ncu_step_r02bo.json"  # the same capture holds K3


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def host_info() -> dict:
    """the host the CPU figures come from."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:  # pragma: no cover
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": host_cores()}


# ------------------------------------------------- CPU reference / oracle ---
# The reference is pure Python (cisgraph 0.1.0).  Installed unmodified into
# baseline/_ref (pip --no-deps from a copy of /root/reference/pkg: numpy and
# scipy come from the image, shapely is not needed on this path), it travels
# to the GPU box with the snapshot.  Where it is absent, the numpy oracle port
# (oracle/gis_oracle.py, pinned bit-exact to it) stands in: kind "port".

REF_DIRS = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def import_reference():
    """The unmodified cisgraph package, or None."""
    for d in REF_DIRS:
        if (d / "cisgraph" / "__init__.py").exists():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            import cisgraph
            return cisgraph, str(d)
    return None, None


class RefPass:
    """One GIS build + prune pass of config 2 through the reference's public
    API, exactly engine.run's build and analyze phases (cg/engine.py:
    168-172): ``build_graph_parallel`` with BuildPlan(1024, all cores), then
    ``non_leaving_mask`` (Tarjan + reverse closure, single-threaded) and
    ``retain``.  The pendulum enters through the reference's plugin API
    (SystemModel(step=callable), the numpy step a user would write:
    oracle.gis_oracle.make_step); the BASELINE sample table is injected
    through cisgraph.image._unit_grid."""

    def __init__(self, block: bool):
        from oracle import gis_oracle as O
        from paper_2202_06111_b200.configs import config
        from paper_2202_06111_b200.image import sample_fractions

        self.cg, self.where = import_reference()
        cfg = config(CONFIG_ID)
        m = cfg.model
        self.frac = np.asarray(sample_fractions(cfg.image, m.n), dtype=np.float64)
        self.workers = host_cores()
        self.block = block
        if self.cg is None:  # the oracle port of the same pass
            self.kind = "port"
            self.O = O
            cov = O.Cover.root(m.X.lo, m.X.hi)
            for _ in range(cfg.initial_depth):
                cov = cov.subdivide()
            self.step_fn = O.make_step(m.step.spec())
            self.inputs = O.input_grid(m.U.lo, m.U.hi, cfg.input_counts)
        else:
            self.kind = "reference"
            from cisgraph import geometry as G, image as I, system as Sy

            I._unit_grid = lambda n, spd, f=self.frac: f
            self.model = Sy.SystemModel(m.name, m.n, m.m, G.Box(m.X.lo, m.X.hi),
                                        G.Box(m.U.lo, m.U.hi), O.make_step(m.step.spec()))
            cov = G.Covering.initial(self.model.X)
            for _ in range(cfg.initial_depth):
                cov = cov.subdivide(None)
            self.inputs = Sy.sample_inputs(self.model.U, cfg.input_counts)
            self.icfg = I.ImageConfig(2, cfg.image.bloat)
        if block:
            k = 1 << SAMPLE_LOG2
            keep = np.zeros(len(cov), dtype=bool)
            keep[SAMPLE_BLOCK * k:(SAMPLE_BLOCK + 1) * k] = True
            cov = cov.retain(keep)
        self.cov = cov
        self.bloat = cfg.image.bloat
        n_inputs = len(self.inputs) if self.kind == "port" else len(self.inputs.points)
        self.integrations = len(cov) * n_inputs * len(self.frac)

    def run(self):
        """(build_s, prune_s, E, kept) of one pass."""
        t0 = time.perf_counter()
        if self.kind == "port":
            O = self.O
            tree = O.BoxTree(self.cov.lo, self.cov.hi)
            ip, ix = O.build_graph_pool(self.cov.lo, self.cov.hi, self.step_fn, self.inputs,
                                        self.frac, self.bloat, self.workers, batch=1024,
                                        tree=tree)
            t1 = time.perf_counter()
            keep = O.non_leaving_mask(ip, ix, len(self.cov))
            E = len(ix)
        else:
            from cisgraph import analysis as A, graph as Gr

            g = Gr.build_graph_parallel(self.cov, self.cov.build_index(), self.model,
                                        self.inputs, self.icfg,
                                        Gr.BuildPlan(batch_size=1024, workers=self.workers))
            t1 = time.perf_counter()
            keep = A.non_leaving_mask(g)
            E = g.edge_count
        self.cov.retain(keep)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, int(E), int(keep.sum())

    def describe(self):
        what = ("unmodified reference cisgraph 0.1.0 (" + self.where + "): build_graph_parallel"
                f"(BuildPlan(1024, {self.workers})) + non_leaving_mask (Tarjan) + retain"
                if self.kind == "reference" else
                f"oracle/gis_oracle.py port: fork pool x{self.workers} + Tarjan + retain")
        size = ("a 128x128-cell block of config 2 at full resolution (the aligned CellId range "
                "around the origin)" if self.block else "the full config-2 1024x1024 covering")
        return f"{size}, {len(self.cov)} cells, {self.integrations} integrations per pass; {what}"


def cpu_passes(steps: int, warmup: int):
    rp = RefPass(block=True)
    for _ in range(warmup):
        rp.run()
    times, last = [], None
    for _ in range(steps):
        b, p, E, kept = rp.run()
        times.append(b + p)
        last = (b, p, E, kept)
    t = sum(times) / len(times)
    return rp, t, last


def cpu_baseline(steps: int = 4, warmup: int = 1):
    """The reference (or port) on the block sample; the cpu_baseline dict."""
    rp, t, (b, p, E, kept) = cpu_passes(steps, warmup)
    return {"value": rp.integrations / t, "unit": UNIT, "cores": rp.workers, "kind": rp.kind,
            "sample": (f"{rp.describe()}; E={E}, kept={kept}; mean of {steps} passes "
                       f"({t:.2f} s each: build {b:.2f} s, prune {p:.2f} s)"),
            "ms_per_step": t * 1e3, "host": host_info()}


def full_pass():
    """One full config-2 pass through the reference (the same-config anchor
    of the block-sample rate)."""
    rp = RefPass(block=False)
    b, p, E, kept = rp.run()
    return {"full_pass_s": b + p, "build_s": b, "prune_s": p, "cells": len(rp.cov),
            "integrations": rp.integrations, "edges": E, "kept": kept, "cores": rp.workers,
            "kind": rp.kind, "integrations_per_s": rp.integrations / (b + p),
            "what": rp.describe()}


def reference_arm(args):
    rank, world = _env_rank()
    if rank != 0:
        return 0
    rp, t, (b, p, E, kept) = cpu_passes(args.steps, args.warmup)
    value = rp.integrations / t
    full = None
    if not args.no_full_pass:
        try:
            full = full_pass()
        except Exception as exc:  # pragma: no cover - report, do not lose the line
            full = {"failed": f"{type(exc).__name__}: {exc}"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "none",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config 2 definition)",
        "config": {"workload": "pendulum-rk4-1024x1024 (config 2), 128x128 block sample",
                   "cells": len(rp.cov), "inputs": 21, "samples": len(rp.frac),
                   "edges": E, "kept": kept},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rp.workers, "kind": rp.kind,
                         "sample": rp.describe() + f"; build {b:.2f} s + prune {p:.2f} s",
                         "host": host_info(), "full_pass": full},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- clocks ---

class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 10 ms through
    NVML while the timed region runs; falls back to nvidia-smi polling."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index, self.sm, self.reasons, self.max_mhz = index, [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            masks = [(name, getattr(N, attr)) for name, attr in self.REASONS]

            def poll():
                while not self._stop.is_set():
                    self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(name for name, m in masks if r & m)
                    time.sleep(0.01)
            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
        except Exception:  # pragma: no cover - NVML unavailable
            self.th = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.th is not None:
            self.th.join(timeout=2)

    @staticmethod
    def max_clock(index: int):
        try:
            import pynvml as N

            N.nvmlInit()
            return N.nvmlDeviceGetMaxClockInfo(N.nvmlDeviceGetHandleByIndex(index),
                                               N.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML unavailable
            return None

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(self.sm), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, 10 ms polling over the timed region"}


# --------------------------------------------------------------- B200 arm --

def b200_arm(args):
    import torch
    import torch.distributed as dist

    rank, world = _env_rank()
    cpu_line = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # separate process: the oracle forks a pool and must never see CUDA
        r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-baseline-only"],
                           capture_output=True, text=True)
        if r.returncode == 0 and r.stdout.strip():
            cpu_line = json.loads(r.stdout.strip().splitlines()[-1])
        else:
            cpu_line = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "port",
                        "sample": f"failed: {r.stderr.strip()[-300:]}"}

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GIS_DIST_BACKEND=gloo is a test mode only: several ranks may then share
    # one GPU (their kernels never wait on each other; the collectives run on
    # host copies) to exercise the multi-rank path on a one-GPU box
    backend = os.environ.get("GIS_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2202_06111_b200.distributed import all_reduce_

    from paper_2202_06111_b200 import Covering, SpatialIndex, _device as D, sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_dev, non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.distributed import build_and_prune_sharded
    from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows, build_graph_serial
    from paper_2202_06111_b200.image import sample_fractions

    cfg = config(CONFIG_ID)
    m = cfg.model
    inputs = sample_inputs(m.U, cfg.input_counts)
    S = len(sample_fractions(cfg.image, m.n))
    cov = Covering.initial(m.X)
    for _ in range(cfg.initial_depth):
        cov = cov.subdivide(None)
    V = len(cov)
    I = V * len(inputs) * S
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    def device_step():
        index = SpatialIndex._dyadic(cov)
        if world > 1:
            keep, edges, sweeps = build_and_prune_sharded(cov, index, m, inputs, cfg.image)
        else:
            indptr, indices = build_graph_rows(cov, index, m, inputs, cfg.image)
            g = SymbolicImage._from_device(cov, indptr, indices)
            keep, sweeps = non_leaving_dev(g)
            edges = g.edge_count
        new = cov.retain(keep)
        return edges, len(new), sweeps

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        device_step()
    D.enable_timing(True)
    D.phase_times()
    D.integrations()  # reset K1's work counters
    barrier()
    launches0 = D.launch_count()
    stream = torch.cuda.current_stream()
    step_ms = []
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between steps (outside the events)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            edges, kept, sweeps = device_step()
            b.record(stream)
            b.synchronize()
            step_ms.append(a.elapsed_time(b))
        barrier()
        t_wall = time.perf_counter() - t_wall
    launches = D.launch_count() - launches0
    phases = D.phase_times()
    # K1 work of this rank's timed steps: images = (cell, input, sample)
    # triples produced, ints = one-step integrations run (a grid vertex
    # shared by several cells' corner samples is integrated once)
    images_t, ints_t = D.integrations()
    ints_step = ints_t / args.steps
    ints_all = torch.tensor([float(ints_t)], dtype=torch.float64, device="cuda")
    if world > 1:
        all_reduce_(ints_all, op=dist.ReduceOp.SUM)
    ints_all_step = float(ints_all.item()) / args.steps
    D.enable_timing(False)
    ms = sum(step_ms) / len(step_ms)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        all_reduce_(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())

    # e2e through the reference-facing API with host buffers
    dep_h = cov.depths.copy()
    bits_h = cov.bits.copy()
    lo_h, hi_h = cov.lo.copy(), cov.hi.copy()
    pin = [torch.from_numpy(x).pin_memory() for x in (dep_h, bits_h, lo_h, hi_h)]
    h2d = sum(int(t.numel() * t.element_size()) for t in pin)
    e2e_ms = []
    d2h = 0
    e2e_clocks = None
    # each step ends with the device->host read of the keep mask, which
    # synchronises the stream: no device-wide barrier inside the loop
    barrier()
    with ClockSampler(local) as clk_e2e:
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            c2 = Covering(m.X, pin[0], pin[1], pin[2], pin[3], _sorted=True)
            if world > 1:  # the engine's multi-GPU call sequence (engine.run)
                keep, _, _ = build_and_prune_sharded(c2, c2.build_index(), m, inputs, cfg.image)
                mask = keep.cpu().numpy().astype(bool)
            else:
                g = build_graph_serial(c2, c2.build_index(), m, inputs, cfg.image)
                mask = non_leaving_mask(g)
            t1 = time.perf_counter()
            d2h = mask.nbytes
            if it >= args.warmup:
                e2e_ms.append((t1 - t0) * 1e3)
    e2e_clocks = clk_e2e.summary()
    e2e_mean = sum(e2e_ms) / len(e2e_ms)
    if world > 1:  # whole-job time: the slowest rank
        t = torch.tensor([e2e_mean], dtype=torch.float64, device="cuda")
        all_reduce_(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
    e2e_v = I / (e2e_mean / 1e3)

    # The same call sequence with the caller also reading the graph as numpy
    # (SymbolicImage.indptr / .indices, int64 as the reference returns them):
    # what a reference caller that inspects the CSR pays on top (the graph
    # otherwise stays on the device).  One GPU.
    host_graph = None
    if world == 1:
        hg_ms, hg_d2h = [], 0
        for it in range(2 + 3):
            t0 = time.perf_counter()
            c2 = Covering(m.X, pin[0], pin[1], pin[2], pin[3], _sorted=True)
            g = build_graph_serial(c2, c2.build_index(), m, inputs, cfg.image)
            mask = non_leaving_mask(g)
            ip_h, ix_h = g.indptr, g.indices
            t1 = time.perf_counter()
            hg_d2h = mask.nbytes + ip_h.nbytes + ix_h.nbytes
            if it >= 2:
                hg_ms.append((t1 - t0) * 1e3)
        hg = sum(hg_ms) / len(hg_ms)
        host_graph = {"value": I / (hg / 1e3), "unit": UNIT, "ms_per_step": hg,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": hg_d2h,
                      "path": "as e2e, plus the caller reading SymbolicImage.indptr / .indices "
                              "(int64 numpy, as the reference returns them)"}
        del g, ip_h, ix_h

    # GIS wall time to the converged invariant set (run()): config 2 (the
    # metric's config) and config 5 (the 4-D cart-pole config BASELINE's
    # scaling target is stated on); at N > 1 the engine shards each
    # iteration's build / prune / selection over the ranks; slowest rank
    from paper_2202_06111_b200 import run

    def gis_wall_s(cid, reps):
        rc = config(cid)
        walls = []
        for _ in range(reps):  # first run warms the allocator pool and index sizes
            barrier()
            t0 = time.perf_counter()
            res = run(rc)
            torch.cuda.synchronize()
            w = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            if world > 1:
                all_reduce_(w, op=dist.ReduceOp.MAX)
            walls.append(float(w.item()))
        return {"cold_s": walls[0], "warm_median_s": statistics.median(walls[1:]),
                "runs": len(walls), "final_cells": len(res.covering), "n_gpus": world}

    gis_wall = gis_wall_s(CONFIG_ID, 4)
    gis_wall5 = gis_wall_s(5, 3)

    probe = D.fp64_peak_tflops()  # measured DFMA-only throughput (8 chains per thread)
    # primary denominator: the datasheet fp64 peak, SMs x 64 DFMA
    # per clock x 2 flops x the max SM clock (NVML); the probe is reported beside
    clk_max = ClockSampler.max_clock(local)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak = sms * 128 * clk_max / 1e6 if clk_max else probe
    k1_ms, k1_n = phases["enclose"]
    flops_per_int = ARITH_FLOPS + SIN_CALLS * SIN_FLOPS
    # enclose phase time per step (one launch per step, or one per row chunk)
    # executed integrations (not images) per unit of K1 time: the fp64 work
    # the kernels actually did
    achieved = (ints_step * flops_per_int / (k1_ms / args.steps * 1e-3) / 1e12
                if k1_n else None)
    traffic, ncu_k1 = None, {}
    prof = ROOT / "profiles" / NCU_SUMMARY
    if prof.exists():
        try:
            ks = json.loads(prof.read_text())["kernels"]
            ncu_k1 = next(v for k, v in ks.items() if k.startswith("enclose_kernel"))
            traffic = ncu_k1.get("dram_bytes")
        except (ValueError, KeyError, StopIteration):
            traffic = None
    # K2 / K3 against HBM with SURVEY 8(d)'s algorithmic bytes (they are
    # latency-bound; the fraction says so)
    hbm = None
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            hbm = float(json.loads(mp.read_text())["hbm_gbs"])
        except (ValueError, KeyError):
            hbm = None
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if hbm else "B200_PROFILING.md fallback 7700 GB/s"
    hbm = hbm or 7700.0
    n, Vl, E = m.n, V / max(world, 1), edges / max(world, 1)
    k2_bytes = 2 * n * 8 * Vl * len(inputs) + 8 * (Vl + 1) + 4 * E
    k3_bytes = 4 * E + 8 * (Vl + 1) + 4 * Vl + sweeps * (Vl / 8)
    def ncu_bytes(summary, prefix):
        try:
            ks = json.loads((ROOT / "profiles" / summary).read_text())["kernels"]
            return next(v for k, v in ks.items() if k.startswith(prefix)).get("dram_bytes")
        except (OSError, ValueError, KeyError, StopIteration):
            return None

    secondary = []
    for name, key, nbytes, summ, prefix in (
            ("rows (K2)", "csr_rows", k2_bytes, NCU_SUMMARY, "rows_kernel<"),
            ("peel (K3)", "prune", k3_bytes, NCU_PEEL_SUMMARY, "peel_coop_kernel")):
        t = phases[key][0] / args.steps
        if t > 0:
            gbs = nbytes / (t * 1e-3) / 1e9
            secondary.append({"kernel": name, "bound": "hbm", "achieved": gbs, "peak": hbm,
                              "unit": "GB/s", "frac": gbs / hbm, "algorithmic_bytes": nbytes,
                              "traffic": ncu_bytes(summ, prefix), "ms": t,
                              "peak_source": hbm_src})
    exchange = None
    if world > 1:
        from paper_2202_06111_b200.distributed import exchange_mode

        exchange = ("fused peer-memory gis_peel_p2p" if exchange_mode() == "p2p"
                    else "rounds of local sweeps (gis_peel_local) + in-place all-gather of "
                         f"the bitmap per round ({dist.get_backend()})")
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    if cpu_line and cpu_line.get("value"):
        # the full config-2 pass at the sample's throughput, labelled as the
        # linear extrapolation BASELINE.md section 3 allows
        cpu_line["extrapolated_full_pass_s"] = I / cpu_line["value"]
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": I / (ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config 2 definition)",
        "config": {"workload": "pendulum-rk4-1024x1024 (BASELINE config 2): index + build + "
                               "prune + retain", "cells": V, "inputs": len(inputs),
                   "samples": S, "integrations_per_step": I,
                   "k1_integrations_run_per_step": ints_all_step,
                   "k1_sharing": "cell-corner samples that coincide bit for bit with the "
                                 "lower corner of the cell above are integrated once "
                                 "(DESIGN.md section 4); value counts every (cell, control, "
                                 "sample) image, the roofline counts integrations run",
                   "edges": edges, "kept": kept,
                   "sweeps": sweeps, "parallelism": f"rows sharded x{world}",
                   "dist_backend": backend if world > 1 else None,
                   "prune_exchange": exchange,
                   "l2": "flushed between steps (512 MiB write, outside the timed events)"},
        "roofline": {"bound": "fp64", "kernel": "enclose (K1)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": ("datasheet fp64: %d SMs x 64 DFMA/clk x 2 flops x %d MHz "
                                     "max SM clock (NVML); MEASURED_PEAKS.json and "
                                     "B200_PROFILING.md give no fp64 figure" % (sms, clk_max)
                                     if clk_max else "measured DFMA probe (NVML unavailable)"),
                     "peak_probe": probe,
                     "frac_of_probe": (achieved / probe) if achieved else None,
                     "probe_source": "gis_fp64_peak: DFMA-only kernel, 8 independent chains "
                                     "per thread, on this GPU",
                     "flops_per_integration": flops_per_int,
                     "flop_rule": "SURVEY 8(d): 426 arithmetic + 40 sin x 16 (the kernel's "
                                  "polynomial sin, executed flops)",
                     "frac_if_sin_priced_at_libm": (achieved * (ARITH_FLOPS + SIN_CALLS *
                                                    LIBM_SIN_FLOPS) / flops_per_int / peak
                                                    if achieved else None),
                     "flop_units": "integrations run by K1 per step (this rank)",
                     "fp64_issue_frac": (ints_step * DP_INSTR_PER_INT /
                                         (k1_ms / args.steps * 1e-3) / (peak * 1e12 / 2)
                                         if k1_n else None),
                     "secondary": secondary,
                     "ncu": {"summary": f"profiles/{NCU_SUMMARY}",
                             "executed_dp_tflops": ncu_k1.get("executed_dp_tflops"),
                             "executed_dp_frac": (ncu_k1["executed_dp_tflops"] / peak
                                                  if ncu_k1.get("executed_dp_tflops") else None),
                             "fp64_pipe_active_pct": ncu_k1.get("fp64_pipe_active_pct"),
                             # sm__sass_thread_inst_executed_op_{dfma,dmul,
                             # dadd}_pred_on of the capture, per integration
                             "dp_inst_per_integration": (
                                 {op: v / ints_step for op, v in  # one config-2 step
                                  ncu_k1["executed_dp_thread_inst"].items()}
                                 if ncu_k1.get("executed_dp_thread_inst") else None)}},
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items()},
        "cpu_baseline": cpu_line,
        "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_mean,
                "ms_min": min(e2e_ms) if e2e_ms else None,
                "ms_max": max(e2e_ms) if e2e_ms else None, "clocks": e2e_clocks,
                "path": ("Covering(host arrays) -> build_graph_serial -> non_leaving_mask -> numpy"
                         if world == 1 else "Covering(host arrays) -> build_and_prune_sharded "
                         f"(owned rows, prune exchange: {exchange}) -> numpy")},
        "e2e_host_graph": host_graph,
        "gis_wall_s_config2": gis_wall,
        "gis_wall_s_config5": gis_wall5,
        "gpu_launches": launches,
        "clocks": clocks,
        "wall_s_timed_region": t_wall,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int:
    """``--gpus N`` (N > 1) started as a plain process: re-exec this script
    under torch.distributed.run with one rank per GPU (rank r on GPU r via
    LOCAL_RANK), rendezvous on 127.0.0.1.  Refuses N > visible GPUs instead of
    measuring fewer.  NCCL's INIT logging stays on (the communicator ranks
    are then visible in the output); rank 0 alone prints the JSON line."""
    if not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if args.gpus > have and os.environ.get("GIS_DIST_BACKEND", "nccl") == "nccl":
            print(json.dumps({"error": f"--gpus {args.gpus} but {have} GPU(s) visible"}),
                  file=sys.stderr, flush=True)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def dry_run_arm(args) -> int:
    """The launcher and the max-over-ranks reduction without a GPU (gloo):
    what tests/test_bench_launcher.py drives at world 2 on CPU.  Each step is
    a fixed numpy workload; the printed line has the bench's schema."""
    import torch
    import torch.distributed as dist

    rank, world = _env_rank()
    if world > 1:
        dist.init_process_group("gloo")
    a = np.random.default_rng(rank).random(1 << 16)
    for _ in range(args.warmup):
        np.sort(a)
    times = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        np.sort(a)
        times.append(time.perf_counter() - t0)
    ms = torch.tensor([1e3 * sum(times) / len(times)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        units = world * a.size
        print(json.dumps({"metric": "dry-run sorted elements/s", "value": units / (ms.item() / 1e3),
                          "unit": "elements/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms.item(),
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic", "dry_run": True,
                          "config": {"workload": "launcher dry run (no GPU)",
                                     "local_rank_env": os.environ.get("LOCAL_RANK")}}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-pass", action="store_true",
                    help="reference arm: skip the one full config-2 reference pass")
    ap.add_argument("--cpu-baseline-only", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be at least 1")
    if args.cpu_baseline_only:
        print(json.dumps(cpu_baseline()), flush=True)
        return 0
    if args.impl == "reference":  # CPU work: rank 0 only, never spawns ranks
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    if args.dry_run:
        return dry_run_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
