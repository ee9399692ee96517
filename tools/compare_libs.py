"""Bit-for-bit comparison and kernel timing of library builds (development aid):
python tools/compare_libs.py --lib build/exp/base/libsfseg_cuda.so build/exp/new/libsfseg_cuda.so \
    --config 1 --frames 24 --arith fast
Every library solves the same seeded problem; the soft vector, the mask and the
per-iteration norms of the later libraries must equal the first one's bits.
With --time it also prints the average fused-step launch time (CUDA events)."""
import argparse
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--lib", nargs="+", required=True)
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--clip", type=int, default=0)
ap.add_argument("--frames", type=int, default=None)
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--arith", default="fast")
ap.add_argument("--binarize", type=int, default=None, help="binarize_start override")
ap.add_argument("--time", action="store_true")
a = ap.parse_args()

prob = synth.config(a.config, frames=a.frames)[a.clip]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = a.arith
if a.iters:
    cfg.iterations = a.iters
if a.binarize is not None:
    cfg.binarize_start = a.binarize
T, H, W = prob.shape
n = cfg.iterations
ref = None
bad = 0
for path in a.lib:
    lib = N.load_library(path)
    h = C.c_void_p()
    N.check(lib.sfseg_ctx_create(0, C.byref(h)))
    q = cfg.to_params()
    fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
    N.check(lib.sfseg_load(h, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                           C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
    rec = (N.IterRecord * n)()
    if a.time:
        lib.sfseg_ctx_set_timing(h, 1)
    N.check(lib.sfseg_solve(h, C.byref(q), 1, n, rec))
    soft = np.empty((T, H, W), np.float32)
    mask = np.empty((T, H, W), np.uint8)
    N.check(lib.sfseg_download(h, cfg.final_threshold, C.c_void_p(soft.ctypes.data),
                               C.c_void_p(mask.ctypes.data), N.SFSEG_MEM_HOST))
    norms = np.array([r.l2_norm_pre_normalize for r in rec])
    msg = f"{path}: {prob.name} {T}x{H}x{W} C={prob.channels} {a.arith} {n} iterations"
    if a.time:
        best = None
        for _ in range(3):
            N.check(lib.sfseg_solve(h, C.byref(q), 1, n, None))
            lib.sfseg_ctx_synchronize(h)
            tm = N.Timing()
            lib.sfseg_ctx_get_timing(h, C.byref(tm))
            us = 1e3 * tm.step_kernel_ms / max(1, tm.step_launches)
            best = us if best is None else min(best, us)
        msg += f" launch_us={best:.1f}"
    if ref is None:
        ref = (soft, mask, norms)
        msg += " (baseline)"
    else:
        same = (np.array_equal(soft.view(np.uint32), ref[0].view(np.uint32)), np.array_equal(mask, ref[1]),
                np.array_equal(norms, ref[2]))
        msg += f" soft/mask/norms identical: {same}"
        if not all(same):
            bad += 1
            d = np.abs(soft.astype(np.float64) - ref[0])
            msg += f" max|diff|={d.max():.3e} at {np.unravel_index(d.argmax(), d.shape)}"
    print(msg, flush=True)
    lib.sfseg_ctx_destroy(h)
sys.exit(1 if bad else 0)
