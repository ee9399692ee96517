#!/usr/bin/env python3
"""SFSeg power-iteration benchmark (BASELINE.json metric: voxel-iterations/s,
achieved HBM GB/s vs roofline).

Workload (default): BASELINE.json configs[1] — T=80, H=480, W=854, C=1,
kernel 5x11x11 (radii 2,5,5; sigmas 0.5,1.5,1.5), 30 power iterations,
alpha=1, p=0.1, binarisation off (pure power iteration). One bench "step" is
one full solve: 30 iterations over the whole volume.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0). ``value`` is device-resident throughput (inputs
already in HBM, CUDA events on the library's launch stream, max over ranks);
``e2e`` is the same metric through the public C ABI call sfseg_run with pinned
host buffers (H2D of S and F, solve, D2H of the soft iterate and mask inside
the timed region; where the config's feature is S itself, f = x0 = S, the
caller passes one buffer and it crosses PCIe once). ``--impl reference`` times the reference's own CPU
implementation (oracle/_ref/libsfseg_ref.so, compiled from the reference
sources) on the host cores with a bounded sample of the same workload.

Arithmetic: the headline (--arith fast, default) is fp32 with fused
multiply-adds, inside the north star's parity gates (tests/test_gpu_parity.py);
--arith exact reproduces the reference's separately rounded products and
sums bit for bit (the step is bit-identical). On one GPU the line also carries
the other mode's numbers under "other_arith".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "voxel-iterations/s of SFSeg power iteration"
UNIT = "voxel-iter/s"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    Polls NVML in-process every `period` s (a spawned nvidia-smi needs
    ~100 ms to start, longer than a short timed region, and its exit can
    overlap the following measurements)."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int, period: float = 0.005):
        self.device, self.period = device, period
        self.samples, self.reasons, self.max_mhz, self.err = [], set(), None, None
        self._stop = threading.Event()
        self.nv = self.h = None
        try:
            import pynvml as nv
            import torch

            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(device)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nv = nv
        except Exception as e:  # no NVML: reported as unsampled
            self.err = f"{type(e).__name__}: {e}"

    def _poll_once(self):
        nv = self.nv
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for name, attr in self.NAMES:
            if r & getattr(nv, attr, 0):
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._poll_once()
            except Exception as e:
                self.err = str(e)
                return
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._stop.clear()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()
            try:
                self._poll_once()  # at least one sample at the end of the region
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": ["unsampled"], "note": self.err}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "nvml"}


def reference_cpu(problem, iterations, frames, threads, reps=1):
    """Reference CPU run() on a T-cropped sample of the workload."""
    from tests.oracle_lib import Reference

    ref = Reference()
    T, H, W = problem.shape
    from paper_1907_02731_b200 import synth

    sample = synth.config(int(problem.name[1]), frames=frames)[0]
    fs, _ = sample.generate()
    cfg = sample.cfg
    cfg.iterations = iterations
    cfg.binarize_start = iterations + 1
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.run(fs.unary, fs.pairwise, cfg, threads=threads)
        times.append(time.perf_counter() - t0)
    vox = frames * H * W * iterations
    return vox, times


def run_reference_arm(args):
    from paper_1907_02731_b200 import synth

    prob = synth.config(args.config)[0]
    threads = os.cpu_count() or 1
    frames = args.ref_frames
    iters = prob.cfg.iterations
    vox = None
    times = []
    for i in range(args.warmup + args.steps):
        vox, t = reference_cpu(prob, iters, frames, threads)
        if i >= args.warmup:
            times.extend(t)
    total = sum(times)
    value = vox * len(times) / total
    T, H, W = prob.shape
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"BASELINE configs[{args.config}] ({prob.name}) T-cropped to "
                               f"{frames} frames for the CPU", "shape": [frames, H, W],
                   "channels": prob.channels, "radii": list(prob.cfg.kernel.radii),
                   "sigmas": list(prob.cfg.kernel.sigmas), "iterations": iters},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"sfseg_ref::run on {frames}x{H}x{W}, C={prob.channels}, "
                                   f"{iters} iterations per step, cfg.threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--arith", default=os.environ.get("SFSEG_ARITH", "fast"),
                    choices=["exact", "fast"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-frames", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the time-sharded driver even on one GPU (testing)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        if rank == 0:
            run_reference_arm(args)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1907_02731_b200 import _native as N
    from paper_1907_02731_b200 import engine as E
    from paper_1907_02731_b200 import synth

    prob = synth.config(args.config)[0]
    cfg = prob.cfg
    cfg.arith = args.arith
    T, H, W = prob.shape
    Cn = prob.channels
    nvox = T * H * W
    iters = cfg.iterations
    same = prob.spec.feature_mode == synth.FEAT_SAME  # f = x0 = S (c0, c1, c3)

    # pinned host inputs, generated once. A time-sharded rank generates only
    # its buffer frames (own frames + halos): the generator is per frame, so
    # the slab equals those frames of the whole volume, and c4's 34 GB never
    # sits in one host process.
    sharded_run = world > 1 or args.sharded
    if sharded_run:
        from paper_1907_02731_b200.sharding import buffer_range, shard_range
        g0, g1 = buffer_range(T, *shard_range(T, world, rank), cfg.kernel.radii[0])
    else:
        g0, g1 = 0, T
    S = torch.empty((g1 - g0, H, W), dtype=torch.float32, pin_memory=True)
    F = [torch.empty((g1 - g0, H, W), dtype=torch.float32, pin_memory=True) for _ in range(Cn)]
    prob.generate(out=(S.numpy(), [f.numpy() for f in F]), frame_range=(g0, g1))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    clocks = ClockSampler(local)
    other = None  # the other arithmetic mode, measured the same way (1 GPU)
    if world == 1 and not args.sharded:
        ctx = E.Context(local)
        lib = ctx._lib
        # device-resident load (H2D once, outside the timed region)
        fptrs = (C.c_void_p * Cn)(*[f.data_ptr() for f in F])
        N.check(lib.sfseg_load(ctx.handle, T, H, W, Cn, C.c_void_p(S.data_ptr()),
                               C.cast(fptrs, C.c_void_p), None, N.SFSEG_MEM_HOST))

        def timed_solves(arith, sampler=None):
            """K solves timed on the library stream (CUDA events at the solve
            boundaries, no per-launch events: those would sit between the
            kernels of the programmatic-dependent-launch chain); then two
            solves with per-launch events for the fused kernel's average."""
            c2 = E.SfsegConfig(**{**cfg.__dict__, "arith": arith})
            p = c2.to_params()
            for _ in range(args.warmup):
                N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, iters, None))
            ctx.synchronize()
            barrier()
            solve_ms = []
            import contextlib
            with (sampler or contextlib.nullcontext()):
                for _ in range(args.steps):
                    N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, iters, None))
                    solve_ms.append(ctx.timing().solve_ms)
            ctx.synchronize()
            barrier()
            ctx.set_timing(True)
            kern_ms, launches = 0.0, 0
            for _ in range(2):
                N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, iters, None))
                tm = ctx.timing()
                kern_ms += tm.step_kernel_ms
                launches += tm.step_launches
            ctx.synchronize()
            ctx.set_timing(False)
            return sum(solve_ms), kern_ms / max(1, launches)

        total_ms, avg_launch_ms = timed_solves(args.arith, clocks)
        oth = "exact" if args.arith == "fast" else "fast"
        o_ms, o_launch = timed_solves(oth)
        other = {"arith": oth, "value": nvox * iters * args.steps / (o_ms * 1e-3),
                 "ms_per_step": o_ms / args.steps, "avg_launch_ms": o_launch}
        p = cfg.to_params()
    else:
        # time-sharded: rank r owns frames [t0, t1) plus rt halo frames
        from paper_1907_02731_b200.sharding import (CudaBackend, ShardedSolver, buffer_range,
                                                    shard_range)

        halo = cfg.kernel.radii[0]
        be = CudaBackend(local)
        solver = ShardedSolver(be, rank, world)
        t0, t1 = shard_range(T, world, rank)
        b0, b1 = buffer_range(T, t0, t1, halo)
        dS = S[b0 - g0:b1 - g0].cuda()
        dF = [f[b0 - g0:b1 - g0].cuda() for f in F]
        solver.load(T, H, W, dS, dF, None, halo)
        for _ in range(args.warmup):
            solver.solve_only(cfg)
        barrier()
        be.ctx.set_timing(True)  # per-launch events of this rank's fused kernel
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            ev0.record()
            be.after_exchange()  # the library stream starts after ev0
            for _ in range(args.steps):
                solver.solve_only(cfg)
            be.before_exchange()  # current stream waits for the library stream
            ev1.record()
            torch.cuda.synchronize()
        total_ms = ev0.elapsed_time(ev1)
        kms, kn = C.c_double(), C.c_int32()
        N.check(be.lib.sfseg_ctx_kernel_time(be.ctx.handle, C.byref(kms), C.byref(kn)))
        be.ctx.set_timing(False)
        barrier()
        avg_launch_ms = kms.value / max(1, kn.value)
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = nvox * iters * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernel (fused stencil): algorithmic bytes per
    # launch = 4 B x (x, S^p, F_c reads + one write) per voxel, one launch per
    # channel group
    sharded = world > 1 or args.sharded
    # (time-sharded: rank 0's launch over its own output frames; recomputed
    # halo frames are not algorithmic bytes)
    unit_vox = nvox if not sharded else (t1 - t0) * H * W
    # FAST with C > 1: one fused_step_mc HEAD + ceil(C/2) TAIL launches per
    # iteration; otherwise one launch per channel. The roofline is taken per
    # iteration: 4 (C + 3) B per voxel over the iteration's launches.
    mc = args.arith == "fast" and Cn > 1
    launches_per_iter = (1 + (Cn + 1) // 2) if mc else Cn
    bytes_per_launch = 4.0 * (Cn + 3) * unit_vox / launches_per_iter
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_c{args.config}_{args.arith}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")

    # end to end through the public C ABI from pinned host memory, per step
    e2e_t = []
    if not sharded:
        soft = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
        mask = torch.empty((T, H, W), dtype=torch.uint8, pin_memory=True)
        # configs whose feature IS the unary volume (f = x0 = S: c0, c1, c3)
        # pass one host buffer for both, as a caller with f = S does; the
        # library uploads it once (sfseg_load: a channel pointer equal to unary)
        e2e_fptrs = (C.c_void_p * Cn)(*[S.data_ptr() if same else f.data_ptr() for f in F])
        for i in range(args.e2e_steps + 1):
            barrier()
            t_0 = time.perf_counter()
            N.check(lib.sfseg_run(ctx.handle, T, H, W, Cn, C.c_void_p(S.data_ptr()),
                                  C.cast(e2e_fptrs, C.c_void_p), None, C.byref(p),
                                  C.c_void_p(soft.data_ptr()), C.c_void_p(mask.data_ptr()), None,
                                  N.SFSEG_MEM_HOST))
            if i > 0:  # first call warms the path
                e2e_t.append(time.perf_counter() - t_0)
        h2d = (1 + (0 if same else Cn)) * nvox * 4
        d2h = nvox * 4 + nvox
    else:
        soft = torch.empty((t1 - t0, H, W), dtype=torch.float32, pin_memory=True)
        mask = torch.empty((t1 - t0, H, W), dtype=torch.uint8, pin_memory=True)
        for i in range(args.e2e_steps + 1):
            barrier()
            t_0 = time.perf_counter()
            dS = S[b0 - g0:b1 - g0].to("cuda", non_blocking=True)
            dF = [f[b0 - g0:b1 - g0].to("cuda", non_blocking=True) for f in F]
            solver.load(T, H, W, dS, dF, None, halo)
            solver.run(cfg, out=(soft.numpy(), mask.numpy()))
            if i > 0:
                e2e_t.append(time.perf_counter() - t_0)
        h2d = (1 + Cn) * (b1 - b0) * H * W * 4 * world
        d2h = (t1 - t0) * H * W * 5 * world
    e2e_s = sum(e2e_t) / len(e2e_t)
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = nvox * iters / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            vox, times = reference_cpu(prob, iters, args.ref_frames, threads)
            cpu = {"value": vox / times[0], "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"sfseg_ref::run (reference compiled from its sources) on "
                             f"{args.ref_frames}x{H}x{W}, C={Cn}, {iters} iterations, "
                             f"cfg.threads={threads}; {times[0]:.1f} s"}
        except Exception as e:  # the reference build may be absent
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[{args.config}] ({prob.name})",
                       "shape": [T, H, W], "channels": Cn, "radii": list(cfg.kernel.radii),
                       "sigmas": list(cfg.kernel.sigmas), "iterations": iters,
                       "alpha": cfg.alpha, "p": cfg.p, "binarization": "off",
                       "arith": args.arith,
                       "l2": f"inputs larger than L2 ({(Cn + 2) * nvox * 4 / 1e6:.0f} MB read per iteration)",
                       "parallelism": f"time-sharded x{world} (rt-frame halos, NCCL)"
                       if world > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "kernel": (f"fused_step_mc<RT={cfg.kernel.radii[0]},R={max(cfg.kernel.radii[1:])}> "
                                    f"HEAD + {(Cn + 1) // 2} TAIL launches per iteration (FAST)" if mc else
                                    f"fused_step_rs<RT={cfg.kernel.radii[0]},R={max(cfg.kernel.radii[1:])}> (FAST)"
                                    if args.arith == "fast" else
                                    f"fused_step_ws<RT={cfg.kernel.radii[0]},R={max(cfg.kernel.radii[1:])},EXACT>"),
                         "avg_launch_ms": avg_launch_ms, "bytes_per_launch": bytes_per_launch},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "inputs": ("S, passed once as unary and feature (f = S)" if same and not sharded
                               else "S and every feature channel")},
            "clocks": clocks.summary(),
            # per iteration: the fused launches + one k_finalize
            "gpu_launches": args.steps * iters * (launches_per_iter + 1),
        }
        if other:
            # EXACT runs one launch per channel (the generic multi-pass path at
            # radii beyond the fused instantiations: no fused launch to time)
            o_lpi = Cn if other["arith"] == "exact" else (1 + (Cn + 1) // 2 if Cn > 1 else 1)
            other["roofline_frac"] = (4.0 * (Cn + 3) * unit_vox / o_lpi / (other["avg_launch_ms"] * 1e-3)
                                      / 1e9 / peak if other["avg_launch_ms"] > 0 else None)
            line["other_arith"] = other
        print(json.dumps(line), flush=True)
    if not sharded:
        ctx.close()
    else:
        be.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
