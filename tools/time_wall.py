"""Wall time per iteration of untimed solves (no per-launch events, so the
programmatic-dependent-launch chain is intact) for library builds (development aid):
python tools/time_wall.py --lib a.so b.so --config 1"""
import argparse
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--lib", nargs="+", required=True)
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--frames", type=int, default=None)
ap.add_argument("--solves", type=int, default=10)
a = ap.parse_args()
prob = synth.config(a.config, frames=a.frames)[0]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = "fast"
cfg.binarize_start = cfg.iterations + 1
T, H, W = prob.shape
for rep in range(2):
    for path in a.lib:
        lib = N.load_library(path)
        h = C.c_void_p()
        N.check(lib.sfseg_ctx_create(0, C.byref(h)))
        q = cfg.to_params()
        fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
        N.check(lib.sfseg_load(h, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                               C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
        for _ in range(3):
            N.check(lib.sfseg_solve(h, C.byref(q), 1, cfg.iterations, None))
        lib.sfseg_ctx_synchronize(h)
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(a.solves):
                N.check(lib.sfseg_solve(h, C.byref(q), 1, cfg.iterations, None))
            lib.sfseg_ctx_synchronize(h)
            dt = (time.perf_counter() - t0) / (a.solves * cfg.iterations)
            best = dt if best is None else min(best, dt)
        print(f"{path}: {prob.name} wall {1e6 * best:.2f} us per iteration", flush=True)
        lib.sfseg_ctx_destroy(h)
