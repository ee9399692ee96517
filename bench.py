#!/usr/bin/env python3
"""SFSeg power-iteration benchmark (BASELINE.json metric: voxel-iterations/s,
achieved HBM GB/s vs roofline).

Workload (default, N=1): BASELINE.json configs[4] (c4) — T=1024, H=1080,
W=1920, C=3 feature channels, kernel 9x21x21 (radii 4,10,10; sigmas
0.5,1.5,1.5), 20 power iterations, alpha=1, p=0.1, binarisation off (pure
power iteration). It is the largest config and fits one B200 (76 GB
resident). One bench "step" is one full solve: 20 iterations over the whole
volume. --config selects another config; --config 3 times the whole batch of
14 independent clips (clip-sharded across ranks under torchrun).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0):
  value     device-resident throughput (inputs in HBM, CUDA events on the
            library stream, max over ranks);
  e2e       the same metric through the one-call C ABI entry sfseg_run with
            pinned host buffers (H2D of S and F, solve, D2H of the soft
            iterate and the mask inside the timed region);
  roofline  of the fused step (all its launches per iteration), against BOTH
            ceilings: HBM (4 (C+3) B per voxel-iteration over the measured
            copy bandwidth) and FP32 (2 flops per tap per convolved field
            per voxel over the FFMA2 peak measured in this run);
            "bound" names the ceiling with the larger floor time (c4/c2:
            fp32, c1/c3: hbm);
  cpu_baseline  the reference compiled from its own sources
            (oracle/_ref/libsfseg_ref.so) on the host cores: its global-step
            loop x = normalize_l2(sfseg_step(x)) (bench.cpp:154-155,
            bit-identical to run(), test_engine.cpp:276-297) and run()
            itself (engine.cpp:247-348), each on a bounded T-crop;
  configs   c0, c1, c2 and the c3 batch measured the same way (N=1).

--impl reference times the reference's global-step loop (the faster of its
two bit-identical forms, so the ratio against it is the conservative one) on
all host threads, each step a bounded T-crop of the same workload; its inputs
are made with numpy (same shapes and value distributions; no library of this
repo is loaded in that process).

Arithmetic: the headline (--arith fast, default) is fp32 with fused
multiply-adds, inside the north star's parity gates (tests/test_gpu_c4.py,
test_gpu_parity.py, test_gpu_fullsize.py); --arith exact reproduces the
reference's separately rounded products and sums (the step is bit-identical).
On one GPU the line also carries the other mode under "other_arith".
"""
from __future__ import annotations

import argparse
import contextlib
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


def _hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML,
    in-process, every `period` s)."""

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
                self._poll_once()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": ["unsampled"], "note": self.err}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "nvml"}


# ---------------------------------------------------------------------------
# workload arithmetic (DESIGN.md §5 / §7)

def fields_of(channels: int) -> int:
    """Convolved fields of the implemented formulation: u, f u, f^2 u for one
    channel (engine.cpp:92-100); the (C + 2)-field form for C > 1
    (fused_mc.cuh: u, Q u, f_c u)."""
    return 3 if channels == 1 else channels + 2


def flops_per_voxel(cfg, channels: int) -> int:
    """Algorithmic FP32 work of one step per voxel: every tap of every axis
    pass of every convolved field is one FMA (2 flops)."""
    rt, ry, rx = cfg.kernel.radii
    return 2 * fields_of(channels) * ((2 * rt + 1) + (2 * ry + 1) + (2 * rx + 1))


def bytes_per_voxel(channels: int) -> int:
    """Compulsory HBM bytes per voxel-iteration: read x, S^p and C channels,
    write y."""
    return 4 * (channels + 3)


def kernel_name(cfg, channels: int, arith: str) -> str:
    rt, r = cfg.kernel.radii[0], max(cfg.kernel.radii[1:])
    if arith == "fast" and channels > 1:
        head = "HEAD(u, Q u, f_1 u)" if channels % 2 else "HEAD(u, Q u)"
        return (f"fused_step_mc<RT={rt},R={r}> {head} + {channels // 2} TAIL "
                f"launch(es) per iteration (FAST, (C+2)-field form)")
    if arith == "fast":
        return f"fused_step_rs<RT={rt},R={r}> (FAST)"
    if channels > 1 or r > 5:
        return f"fused_step_mc<RT={rt},R={r},EXACT> one launch per channel"
    return f"fused_step_ws<RT={rt},R={r},EXACT>"


def roofline(cfg, channels, nvox, fused_ms_per_iter, hbm_peak, hbm_src, fp32_peak, traffic_bpv):
    """Roofline of the fused step per iteration against both ceilings."""
    sec = fused_ms_per_iter * 1e-3
    b = bytes_per_voxel(channels) * nvox
    f = flops_per_voxel(cfg, channels) * nvox
    hbm = {"achieved": b / sec / 1e9, "peak": hbm_peak, "unit": "GB/s",
           "frac": b / sec / 1e9 / hbm_peak, "peak_source": hbm_src,
           "bytes_per_iteration": b,
           "traffic": traffic_bpv * nvox if traffic_bpv else None}
    fp = {"achieved": f / sec / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
          "frac": (f / sec / 1e12 / fp32_peak) if fp32_peak else None,
          "peak_source": "sfseg_probe_fp32_peak: FFMA2 stream kernel, measured in this run",
          "flops_per_iteration": f}
    hbm_floor = b / (hbm_peak * 1e9)
    fp_floor = f / (fp32_peak * 1e12) if fp32_peak else 0.0
    bound = "fp32" if fp_floor > hbm_floor else "hbm"
    top = dict(fp if bound == "fp32" else hbm)
    top.update({"bound": bound,
                "unit_of_work": "one fused step (all its launches) over the volume, per iteration",
                "fused_ms_per_iteration": fused_ms_per_iter,
                "hbm": hbm, "fp32": fp})
    if bound == "fp32":
        top["traffic"] = hbm["traffic"]
    return top


def _traffic(idx, arith):
    """DRAM bytes per voxel-iteration of the fused step, from an ncu --set
    full capture (profiles/traffic_c<idx>_<arith>.json)."""
    f = ROOT / "profiles" / f"traffic_c{idx}_{arith}.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d.get("dram_bytes_per_voxel_iteration")
    return None


# ---------------------------------------------------------------------------
# reference (CPU) side

def numpy_inputs(idx, frames, seed=1234):
    """Inputs of BASELINE configs[idx] T-cropped to `frames`, made with numpy
    (moving soft ellipses + noise, same shapes and value ranges as
    synth.cpp's); used where no library of this repo may be loaded (the
    reference arm). Returns (S, [F_c], cfg, C)."""
    from paper_1907_02731_b200 import synth  # config() only: no library load

    prob = synth.config(idx, frames=frames)[0]
    T, H, W = prob.shape
    Cn = prob.channels
    rng = np.random.default_rng(seed + idx)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float32)
    nobj = 3 if idx == 4 else 1
    frac = {0: None, 1: 0.25, 2: 0.25, 3: 0.15, 4: 0.08}[idx]
    x0 = np.full((T, H, W), 0.1, np.float32)
    for k in range(nobj):
        if frac:
            a = np.sqrt(frac * H * W / np.pi) * rng.uniform(0.8, 1.2)
            b = frac * H * W / (np.pi * a)
        else:
            a, b = rng.uniform(10, 20, 2)
        cy, cx = rng.uniform(0.3, 0.7) * H, rng.uniform(0.3, 0.7) * W
        vy, vx = rng.uniform(1, 2, 2) * rng.choice([-1, 1], 2)
        inside = (0.9, 0.7, 0.5)[k]
        for t in range(T):
            m = ((yy - cy - vy * t) / b) ** 2 + ((xx - cx - vx * t) / a) ** 2 <= 1.0
            x0[t][m] = np.maximum(x0[t][m], inside)
    if idx == 0:
        x0 = np.clip(x0 + rng.uniform(-0.1, 0.1, x0.shape).astype(np.float32), 0, 1)
    elif idx in (1, 3):
        x0 = np.clip(x0 + rng.normal(0, 0.1, x0.shape).astype(np.float32), 0, 1)
    if idx == 2:
        F = [np.clip(x0 + rng.normal(0, 0.15, x0.shape).astype(np.float32), 0, 1) for _ in range(Cn)]
        S = np.mean(F, axis=0).astype(np.float32)
    elif idx == 4:
        S = x0
        F = [np.clip(x0 + rng.normal(0, 0.1, x0.shape).astype(np.float32), 0, 1) for _ in range(Cn)]
    else:
        S = x0
        F = [x0]
    return np.ascontiguousarray(S, np.float32), [np.ascontiguousarray(f, np.float32) for f in F], \
        prob.cfg, Cn


# T-crops of the CPU samples (frames, global-loop iterations, run() iterations):
# frames >= 2 rt + 1 so the t-pass is representative; ~5-15 s each on 16 threads
CPU_SAMPLE = {0: (8, 20, 20), 1: (12, 10, 3), 2: (12, 3, 1), 3: (24, 10, 3), 4: (12, 2, 1)}


def reference_cpu(idx, S, F, cfg, threads, iters, loop="global"):
    """Times the reference (compiled from its sources) on (S, F): the global
    step loop or run(); returns (voxel-iterations, seconds)."""
    from tests.oracle_lib import Reference

    ref = Reference()
    c = type(cfg)(**{**cfg.__dict__, "iterations": iters, "binarize_start": iters + 1})
    t0 = time.perf_counter()
    if loop == "global":
        ref.global_loop(S, F, c, iters, threads=threads)
    else:
        ref.run(S, F, c, threads=threads)
    return S.size * iters, time.perf_counter() - t0


def cpu_baseline(idx, threads):
    frames, gi, ri = CPU_SAMPLE[idx]
    S, F, cfg, Cn = numpy_inputs(idx, frames)
    T, H, W = S.shape
    vg, tg = reference_cpu(idx, S, F, cfg, threads, gi, "global")
    vr, tr = reference_cpu(idx, S, F, cfg, threads, ri, "run")
    return {"value": vg / tg, "unit": UNIT, "cores": threads, "kind": "reference",
            "loop": "global step x = normalize_l2(sfseg_step(x)) (bench.cpp:154-155)",
            "sample": f"sfseg_ref (compiled from the reference sources) global-step loop on "
                      f"{T}x{H}x{W}, C={Cn}, {gi} iterations, cfg.threads={threads}: {tg:.1f} s",
            "run_value": vr / tr,
            "run_sample": f"sfseg_ref::run (windowed Algorithm 1, engine.cpp:247-348) on the "
                          f"same crop, {ri} iteration(s): {tr:.1f} s"}


def run_reference_arm(args):
    threads = os.cpu_count() or 1
    frames, gi, _ = CPU_SAMPLE[args.config]
    S, F, cfg, Cn = numpy_inputs(args.config, frames)
    T, H, W = S.shape
    times, vox = [], 0
    for i in range(args.warmup + args.steps):
        vox, t = reference_cpu(args.config, S, F, cfg, threads, gi, "global")
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = vox * len(times) / total
    from paper_1907_02731_b200 import synth

    name = synth.config(args.config)[0].name
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak" if args.config == 3 else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy moving ellipses, same shapes and value ranges)",
        "config": {"workload": f"BASELINE configs[{args.config}] ({name}) T-cropped to "
                               f"{frames} frames for the CPU", "shape": [T, H, W],
                   "channels": Cn, "radii": list(cfg.kernel.radii),
                   "sigmas": list(cfg.kernel.sigmas), "iterations_per_step": gi},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "loop": "global step x = normalize_l2(sfseg_step(x)) (bench.cpp:154-155), "
                                 "bit-identical to run() and 3-7x faster",
                         "sample": f"sfseg_ref global-step loop on {T}x{H}x{W}, C={Cn}, {gi} "
                                   f"iterations per step, cfg.threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side

class Gpu:
    """One library context on one device: load, timed solves."""

    def __init__(self, device):
        from paper_1907_02731_b200 import _native as N
        from paper_1907_02731_b200 import engine as E

        self.N, self.E = N, E
        self.ctx = E.Context(device)
        self.lib = self.ctx._lib

    def load(self, S, F):
        N = self.N
        T, H, W = S.shape
        mem = N.SFSEG_MEM_DEVICE if hasattr(S, "is_cuda") and S.is_cuda else N.SFSEG_MEM_HOST
        ptr = (lambda a: a.data_ptr()) if mem == N.SFSEG_MEM_DEVICE else (lambda a: a.ctypes.data)
        fp = (C.c_void_p * len(F))(*[ptr(f) for f in F])
        N.check(self.lib.sfseg_load(self.ctx.handle, T, H, W, len(F), C.c_void_p(ptr(S)),
                                    C.cast(fp, C.c_void_p), None, mem))

    def timed_solves(self, cfg, steps, warmup, sampler=None):
        """K solves timed on the library stream (events at the solve
        boundaries only: per-launch events would sit inside the programmatic
        dependent-launch chain); then 2 solves with per-launch events for the
        fused step's time per iteration and its launch count."""
        N, lib, h = self.N, self.lib, self.ctx.handle
        p = cfg.to_params()
        for _ in range(warmup):
            N.check(lib.sfseg_solve(h, C.byref(p), 1, cfg.iterations, None))
        self.ctx.synchronize()
        solve_ms = []
        with (sampler or contextlib.nullcontext()):
            for _ in range(steps):
                N.check(lib.sfseg_solve(h, C.byref(p), 1, cfg.iterations, None))
                solve_ms.append(self.ctx.timing().solve_ms)
        self.ctx.synchronize()
        self.ctx.set_timing(True)
        kern_ms, launches = 0.0, 0
        for _ in range(2):
            N.check(lib.sfseg_solve(h, C.byref(p), 1, cfg.iterations, None))
            tm = self.ctx.timing()
            kern_ms += tm.step_kernel_ms
            launches += tm.step_launches
        self.ctx.synchronize()
        self.ctx.set_timing(False)
        iters = 2 * cfg.iterations
        return sum(solve_ms), kern_ms / iters, launches / iters

    def run_once(self, S, F, cfg, soft, mask):
        N = self.N
        T, H, W = S.shape
        fp = (C.c_void_p * len(F))(*[f.data_ptr() for f in F])
        p = cfg.to_params()
        N.check(self.lib.sfseg_run(self.ctx.handle, T, H, W, len(F), C.c_void_p(S.data_ptr()),
                                   C.cast(fp, C.c_void_p), None, C.byref(p),
                                   C.c_void_p(soft.data_ptr()), C.c_void_p(mask.data_ptr()), None,
                                   N.SFSEG_MEM_HOST))

    def close(self):
        self.ctx.close()


def launches_per_solve(cfg, channels, arith, lpi):
    """Kernels this library launches per solve: the fused step's launches
    and one k_finalize per iteration, plus one k_make_u (u = S^p x of
    iteration 1) on the multi-channel FAST path."""
    n = cfg.iterations * (int(round(lpi)) + 1)
    return n + (1 if arith == "fast" and channels > 1 else 0)


def measure_config(gpu, idx, arith, steps, warmup, hbm, hbm_src, fp32_peak, clocks=None):
    """Generates BASELINE configs[idx] on the host, loads it and times solves.
    c3 is the batch of 14 clips: each clip is loaded and solved in turn, and
    the batch's value is its total voxel-iterations over the summed solve
    times."""
    from paper_1907_02731_b200 import synth

    import torch

    probs = synth.config(idx)
    tot_vox_it, tot_ms, fused_ms, nv, launches = 0.0, 0.0, 0.0, 0, 0
    pinned = []  # c3: the batch's inputs in pinned host memory, for the batch e2e below
    for prob in probs:
        fs, _ = prob.generate()
        cfg = prob.cfg
        cfg.arith = arith
        F = [fs.unary] if prob.spec.feature_mode == synth.FEAT_SAME else fs.pairwise
        if idx == 3:
            hs = torch.empty(prob.shape, dtype=torch.float32, pin_memory=True)
            hs.numpy()[...] = fs.unary
            pinned.append(hs)
        gpu.load(fs.unary, F)
        ms, fk, lpi = gpu.timed_solves(cfg, steps, warmup, clocks)
        n = prob.voxels()
        tot_vox_it += n * cfg.iterations * steps
        tot_ms += ms
        fused_ms += fk * cfg.iterations  # per solve
        nv += n * cfg.iterations
        launches += launches_per_solve(cfg, prob.channels, arith, lpi)
    prob = probs[0]
    cfg = prob.cfg
    fms_iter = fused_ms / cfg.iterations  # every clip of a batch has the same iteration count
    nvox = sum(p.voxels() for p in probs)
    out = {"workload": f"BASELINE configs[{idx}] ({prob.name if idx != 3 else 'c3: 14 clips'})",
           "value": tot_vox_it / (tot_ms * 1e-3), "ms_per_step": tot_ms / steps,
           "ms_per_iteration": tot_ms / steps / cfg.iterations if idx != 3 else None,
           "kernel": kernel_name(cfg, prob.channels, arith),
           "roofline": roofline(cfg, prob.channels, nvox, fms_iter, hbm, hbm_src, fp32_peak,
                                _traffic(idx, arith)),
           "gpu_launches_per_step": launches,
           "shape": list(prob.shape) if idx != 3 else [list(p.shape) for p in probs],
           "channels": prob.channels, "radii": list(cfg.kernel.radii),
           "sigmas": list(cfg.kernel.sigmas), "iterations": cfg.iterations}
    if idx == 3:
        out["e2e"] = batch_e2e(gpu, pinned, cfg, nvox)
    return out


def batch_e2e(gpu, pinned, cfg, nvox):
    """The c3 batch end to end through sfseg_run_batch (include/sfseg_cuda.h):
    pinned host inputs -> soft + mask in pinned host memory, for 1, 2 and 3
    contexts on the device (with more than one, a clip's transfers run under
    another clip's solve). Wall clock around the one C-ABI call."""
    import torch

    E = gpu.E
    clips = [E.FeatureSet(h.numpy(), [h.numpy()]) for h in pinned]  # f = S: one upload per clip
    outs = [(torch.empty(h.shape, dtype=torch.float32, pin_memory=True).numpy(),
             torch.empty(h.shape, dtype=torch.uint8, pin_memory=True).numpy()) for h in pinned]
    by = {}
    extra = []
    try:
        for nctx in (1, 2, 3):
            while len(extra) < nctx - 1:
                extra.append(E.Context(gpu.ctx.device))
            ctxs = [gpu.ctx] + extra[:nctx - 1]
            E.run_batch(clips, cfg, ctxs=ctxs, outputs=outs)  # warms buffers and pools
            ts = []
            for _ in range(2):
                t0 = time.perf_counter()
                E.run_batch(clips, cfg, ctxs=ctxs, outputs=outs)
                ts.append(time.perf_counter() - t0)
            by[nctx] = nvox * cfg.iterations / (sum(ts) / len(ts))
    finally:
        for c in extra:
            c.close()
    best = max(by, key=by.get)
    return {"value": by[best], "unit": UNIT, "contexts": best,
            "by_contexts": {str(k): v for k, v in by.items()},
            "h2d_bytes_per_step": nvox * 4, "d2h_bytes_per_step": nvox * 5,
            "inputs": "S per clip, passed once as unary and feature (f = S)",
            "call": "sfseg_run_batch (include/sfseg_cuda.h): LPT queue over the contexts, "
                    "load + solve + download per clip"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--arith", default=os.environ.get("SFSEG_ARITH", "fast"),
                    choices=["exact", "fast"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the other configs (c1, c2, c3 batch) and the other arithmetic")
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
    from paper_1907_02731_b200 import synth

    hbm, hbm_src = _hbm_peak()
    fp32 = C.c_double(0.0)
    N.check(N.load_library().sfseg_probe_fp32_peak(local, C.byref(fp32)))
    fp32_peak = fp32.value

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    probs = synth.config(args.config)
    prob = probs[0]
    cfg = prob.cfg
    cfg.arith = args.arith
    Cn = prob.channels
    iters = cfg.iterations
    sharded = (world > 1 or args.sharded) and args.config != 3
    line_extra = {}

    if args.config == 3:
        # ---- c3: batch of independent clips, LPT clip sharding (no exchange)
        from paper_1907_02731_b200.sharding import assign_clips

        mine = assign_clips([p.voxels() for p in probs], world)[rank]
        gpu = Gpu(local)
        tot_ms, my_vox, fused_ms, launches = 0.0, 0, 0.0, 0
        pinned = []
        for i in mine:
            p = probs[i]
            fs, _ = p.generate()
            c = p.cfg
            c.arith = args.arith
            S = torch.from_numpy(fs.unary).pin_memory()
            pinned.append(S)
            gpu.load(fs.unary, [fs.unary])
            ms, fk, lpi = gpu.timed_solves(c, args.steps, args.warmup, clocks)
            tot_ms += ms
            fused_ms += fk * c.iterations
            my_vox += p.voxels()
            launches += args.steps * launches_per_solve(c, 1, args.arith, lpi)
        # end to end: this rank's clips through sfseg_run_batch (pinned host in and out)
        be = batch_e2e(gpu, pinned, cfg, my_vox)
        barrier()
        total_ms = max_over_ranks(tot_ms)
        e2e_s = max_over_ranks(my_vox * iters / be["value"])
        all_vox = sum(p.voxels() for p in probs)
        value = all_vox * iters * args.steps / (total_ms * 1e-3)
        fms_iter = fused_ms / iters  # this rank's clips (rank 0 prints)
        e2e = dict(be, value=all_vox * iters / e2e_s, h2d_bytes_per_step=all_vox * 4,
                   d2h_bytes_per_step=all_vox * 5)
        rl = roofline(cfg, 1, my_vox, fms_iter, hbm, hbm_src, fp32_peak, _traffic(3, args.arith))
        rl["kernel"] = kernel_name(cfg, 1, args.arith)
        gpu_launches = launches
        parallelism = f"clip-sharded x{world} (LPT by voxel count, no exchange)" if world > 1 \
            else "single GPU, 14 clips in turn"
        shape = [list(p.shape) for p in probs]
        scaling = "weak"
        other = None
    elif not sharded:
        # ---- one context, the whole volume resident in HBM
        gpu = Gpu(local)
        T, H, W = prob.shape
        same = prob.spec.feature_mode == synth.FEAT_SAME  # f = x0 = S (c0, c1)
        S = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
        F = [torch.empty((T, H, W), dtype=torch.float32, pin_memory=True) for _ in range(Cn)]
        prob.generate(out=(S.numpy(), [f.numpy() for f in F]))
        Fin = [S] if same else F
        gpu.load(S.numpy(), [f.numpy() for f in Fin])
        total_ms, fms_iter, lpi = gpu.timed_solves(cfg, args.steps, args.warmup, clocks)
        value = prob.voxels() * iters * args.steps / (total_ms * 1e-3)
        gpu_launches = args.steps * launches_per_solve(cfg, Cn, args.arith, lpi)
        rl = roofline(cfg, Cn, prob.voxels(), fms_iter, hbm, hbm_src, fp32_peak,
                      _traffic(args.config, args.arith))
        rl["kernel"] = kernel_name(cfg, Cn, args.arith)
        rl["launches_per_iteration"] = lpi
        other = None
        if not args.no_extras:
            oth = "exact" if args.arith == "fast" else "fast"
            c2 = type(cfg)(**{**cfg.__dict__, "arith": oth})
            o_ms, o_f, o_lpi = gpu.timed_solves(c2, 2, 1)
            o_rl = roofline(c2, Cn, prob.voxels(), o_f, hbm, hbm_src, fp32_peak, None)
            other = {"arith": oth, "value": prob.voxels() * iters * 2 / (o_ms * 1e-3),
                     "ms_per_step": o_ms / 2, "kernel": kernel_name(c2, Cn, oth),
                     "hbm_frac": o_rl["hbm"]["frac"], "fp32_frac": o_rl["fp32"]["frac"]}
        # opt-in FAST tap trimming (sfseg_ctx_set_tap_trim): an extra key, never
        # the headline; reported only where it changes the kernel's support
        if not args.no_extras and args.arith == "fast":
            eff = list(gpu.E.effective_radii(cfg))
            if eff != [int(r) for r in cfg.kernel.radii]:
                gpu.ctx.set_tap_trim(True)
                t_ms, t_f, t_lpi = gpu.timed_solves(cfg, 2, 1)
                gpu.ctx.set_tap_trim(False)
                line_extra["tap_trim"] = {
                    "note": "opt-in (sfseg_ctx_set_tap_trim / SFSEG_FAST_TRIM=1), off in every other "
                            "number of this line: taps at most 2^-24 of their axis's largest tap dropped",
                    "effective_radii": eff, "value": prob.voxels() * iters * 2 / (t_ms * 1e-3),
                    "ms_per_step": t_ms / 2, "fused_ms_per_iteration": t_f,
                    "launches_per_iteration": t_lpi}
        # end to end through sfseg_run from pinned host memory
        soft = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
        mask = torch.empty((T, H, W), dtype=torch.uint8, pin_memory=True)
        gpu.run_once(S, Fin, cfg, soft, mask)  # warms the path
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            gpu.run_once(S, Fin, cfg, soft, mask)
            ts.append(time.perf_counter() - t0)
        e2e_s = sum(ts) / len(ts)
        e2e = {"value": prob.voxels() * iters / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": len(set(id(f) for f in [S] + Fin)) * prob.voxels() * 4,
               "d2h_bytes_per_step": prob.voxels() * 5,
               "inputs": ("S, passed once as unary and feature (f = S)" if same
                          else "S and every feature channel"),
               "call": "sfseg_run (include/sfseg_cuda.h): load + solve + download in one call"}
        del S, F, Fin, soft, mask
        parallelism = "single GPU"
        shape = list(prob.shape)
        scaling = "strong"
        if not args.no_extras:
            cfgs = {}
            for idx in (0, 1, 2, 3):
                if idx == args.config:
                    continue
                # c0 (32768 voxels, ~0.3 ms per solve) is latency-bound: more solves per sample
                r = measure_config(gpu, idx, args.arith, 50 if idx == 0 else 3, 3, hbm, hbm_src,
                                   fp32_peak)
                cfgs[f"c{idx}"] = r
            line_extra["configs"] = cfgs
        gpu.close()
    else:
        # ---- time-sharded: rank r owns frames [t0, t1) plus rt halo frames
        from paper_1907_02731_b200.sharding import (CudaBackend, ShardedSolver, buffer_range,
                                                    shard_range)

        T, H, W = prob.shape
        halo = cfg.kernel.radii[0]
        t0, t1 = shard_range(T, world, rank)
        b0, b1 = buffer_range(T, t0, t1, halo)
        S = torch.empty((b1 - b0, H, W), dtype=torch.float32, pin_memory=True)
        F = [torch.empty((b1 - b0, H, W), dtype=torch.float32, pin_memory=True) for _ in range(Cn)]
        prob.generate(out=(S.numpy(), [f.numpy() for f in F]), frame_range=(b0, b1))
        be = CudaBackend(local)
        solver = ShardedSolver(be, rank, world)
        solver.load(T, H, W, S.cuda(), [f.cuda() for f in F], None, halo)
        # the second solve captures the loop into a CUDA graph; later ones replay it
        for _ in range(max(2, args.warmup)):
            solver.solve_only(cfg)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            ev0.record()
            be.after_exchange()
            for _ in range(args.steps):
                solver.solve_only(cfg)
            be.before_exchange()
            ev1.record()
            torch.cuda.synchronize()
        total_ms = max_over_ranks(ev0.elapsed_time(ev1))
        # the fused kernel's own time: one more solve, launched eagerly with
        # per-launch events (events cannot be read out of a graph replay)
        os.environ["SFSEG_SHARD_GRAPH"] = "0"
        be.ctx.set_timing(True)
        solver.solve_only(cfg)
        torch.cuda.synchronize()
        kms, kn = C.c_double(), C.c_int32()
        N.check(be.lib.sfseg_ctx_kernel_time(be.ctx.handle, C.byref(kms), C.byref(kn)))
        be.ctx.set_timing(False)
        os.environ.pop("SFSEG_SHARD_GRAPH", None)
        barrier()
        value = prob.voxels() * iters * args.steps / (total_ms * 1e-3)
        lpi = kn.value / max(1, iters)
        fms_iter = kms.value / max(1, iters)
        gpu_launches = args.steps * launches_per_solve(cfg, Cn, args.arith, lpi)
        rl = roofline(cfg, Cn, (t1 - t0) * H * W, fms_iter, hbm, hbm_src, fp32_peak,
                      _traffic(args.config, args.arith))
        rl["kernel"] = kernel_name(cfg, Cn, args.arith) + " (rank 0's shard)"
        soft = torch.empty((t1 - t0, H, W), dtype=torch.float32, pin_memory=True)
        mask = torch.empty((t1 - t0, H, W), dtype=torch.uint8, pin_memory=True)
        ts = []
        for i in range(args.e2e_steps + 1):
            barrier()
            t_0 = time.perf_counter()
            dS = S.to("cuda", non_blocking=True)
            dF = [f.to("cuda", non_blocking=True) for f in F]
            solver.load(T, H, W, dS, dF, None, halo)
            solver.run(cfg, out=(soft.numpy(), mask.numpy()))
            if i > 0:
                ts.append(time.perf_counter() - t_0)
        e2e_s = max_over_ranks(sum(ts) / len(ts))
        e2e = {"value": prob.voxels() * iters / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": (1 + Cn) * (b1 - b0) * H * W * 4 * world,
               "d2h_bytes_per_step": (t1 - t0) * H * W * 5 * world,
               "inputs": "S and every feature channel (each rank its frames + halos)"}
        be.close()
        parallelism = f"time-sharded x{world} (rt-frame halos by peer memory, NCCL all-gather)"
        shape = list(prob.shape)
        scaling = "strong"
        other = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, os.cpu_count() or 1)
        except Exception as e:  # the reference build may be absent
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[{args.config}] ({prob.name if args.config != 3 else 'c3: 14 clips'})",
                       "shape": shape, "channels": Cn, "radii": list(cfg.kernel.radii),
                       "sigmas": list(cfg.kernel.sigmas), "iterations": iters,
                       "alpha": cfg.alpha, "p": cfg.p, "binarization": "off",
                       "arith": args.arith,
                       "l2": "inputs larger than L2 (126 MB)" if args.config != 0 else "inputs fit L2",
                       "parallelism": parallelism},
            "roofline": rl,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": gpu_launches,
        }
        if other:
            line["other_arith"] = other
        line.update(line_extra)
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
