"""Launch time of a FAST solve with and without tap trimming (development aid):
python tools/time_trim.py --config 4 --frames 64 --iters 4"""
import argparse
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--frames", type=int, default=64)
ap.add_argument("--iters", type=int, default=4)
a = ap.parse_args()
prob = synth.config(a.config, frames=a.frames)[0]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = "fast"
cfg.iterations = a.iters
cfg.binarize_start = a.iters + 1
T, H, W = prob.shape
lib = N.load_library()
soft = {}
for trim in (0, 1):
    h = C.c_void_p()
    N.check(lib.sfseg_ctx_create(0, C.byref(h)))
    N.check(lib.sfseg_ctx_set_tap_trim(h, trim))
    q = cfg.to_params()
    fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
    N.check(lib.sfseg_load(h, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                           C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
    lib.sfseg_ctx_set_timing(h, 1)
    best = None
    for _ in range(3):
        N.check(lib.sfseg_solve(h, C.byref(q), 1, a.iters, None))
        lib.sfseg_ctx_synchronize(h)
        tm = N.Timing()
        lib.sfseg_ctx_get_timing(h, C.byref(tm))
        ms = tm.step_kernel_ms / a.iters
        best = ms if best is None else min(best, ms)
    x = np.empty((T, H, W), np.float32)
    N.check(lib.sfseg_download(h, cfg.final_threshold, C.c_void_p(x.ctypes.data), None, N.SFSEG_MEM_HOST))
    soft[trim] = x
    print(f"{prob.name} {T}x{H}x{W} trim={trim}: fused kernels {best:.3f} ms per iteration", flush=True)
    lib.sfseg_ctx_destroy(h)
d = np.abs(soft[0].astype(np.float64) - soft[1])
print(f"max|trimmed - full| = {d.max():.3e} ({d.max() / soft[0].max():.3e} of max|x|)")
