"""Kernel timing of one library build (development aid for ablations):
python tools/time_solve.py [--lib path.so ...] --arith fast
Prints the average fused-step launch time (CUDA events) per library."""
import argparse
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--lib", nargs="*", default=[str(N.CUDA_LIB)])
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--arith", default="fast")
ap.add_argument("--frames", type=int, default=None)
a = ap.parse_args()
prob = synth.config(a.config, frames=a.frames)[0]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = a.arith
cfg.iterations = a.iters
cfg.binarize_start = a.iters + 1
T, H, W = prob.shape
for path in a.lib:
    lib = N.load_library(path)
    h = C.c_void_p()
    if lib.sfseg_ctx_create(0, C.byref(h)) != 0:
        print(path, "ctx_create:", lib.sfseg_last_error().decode())
        continue
    p = N.Params()
    lib.sfseg_params_default(C.byref(p))
    q = cfg.to_params()
    fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
    assert lib.sfseg_load(h, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                          C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST) == 0
    lib.sfseg_solve(h, C.byref(q), 1, a.iters, None)
    lib.sfseg_ctx_set_timing(h, 1)
    res = []
    import time
    walls = []
    for _ in range(3):
        lib.sfseg_ctx_synchronize(h)
        t0 = time.perf_counter()
        rc = lib.sfseg_solve(h, C.byref(q), 1, a.iters, None)
        lib.sfseg_ctx_synchronize(h)
        walls.append((time.perf_counter() - t0) / a.iters)
        tm = N.Timing()
        lib.sfseg_ctx_get_timing(h, C.byref(tm))
        res.append(tm.step_kernel_ms / max(1, tm.step_launches))
    err = lib.sfseg_last_error().decode() if rc else ""
    print(f"{path}: rc={rc} {err} launch_us={1e3 * min(res):.1f} (runs {[round(1e3 * r, 1) for r in res]}) "
          f"wall_ms_per_iteration={1e3 * min(walls):.3f}", flush=True)
    lib.sfseg_ctx_destroy(h)
