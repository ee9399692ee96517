"""Profiling driver: load a BASELINE config and run a few iterations (used
under ncu; never a bench number)."""
import argparse
import ctypes as C
import sys
sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--frames", type=int, default=None)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--arith", default="exact")
a = ap.parse_args()
prob = synth.config(a.config, frames=a.frames)[0]
fs, _ = prob.generate()
ctx = E.Context(0)
cfg = prob.cfg
cfg.arith = a.arith
cfg.iterations = a.iters
cfg.binarize_start = a.iters + 1
p = cfg.to_params()
T, H, W = prob.shape
fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
N.check(ctx._lib.sfseg_load(ctx.handle, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                            C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
N.check(ctx._lib.sfseg_solve(ctx.handle, C.byref(p), 1, a.iters, None))
ctx.synchronize()
print("ok", prob.name, prob.shape)
