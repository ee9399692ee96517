"""BASELINE configs[3] (14 independent clips) on one GPU: every clip loaded
into one context and solved (25 iterations); device time from the library's
solve events. Prints the aggregate voxel-iterations/s (development aid; the
clip-sharded multi-GPU driver is sharding.run_clips)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth

arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
clips = synth.config(3)
ctx = E.Context(0)
lib = ctx._lib
tot_vox_it, tot_ms = 0, 0.0
for prob in clips:
    fs, _ = prob.generate()
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith})
    T, H, W = prob.shape
    fp = (C.c_void_p * prob.channels)(*[f.ctypes.data for f in fs.pairwise])
    N.check(lib.sfseg_load(ctx.handle, T, H, W, prob.channels, C.c_void_p(fs.unary.ctypes.data),
                           C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
    p = cfg.to_params()
    N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, None))  # warm
    best = 1e30
    for _ in range(3):
        N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, None))
        best = min(best, ctx.timing().solve_ms)
    vi = T * H * W * cfg.iterations
    tot_vox_it += vi
    tot_ms += best
    print(f"{prob.name}: {T}x{H}x{W} {best:.3f} ms per solve, {vi / best / 1e-3:.3e} vox-it/s", flush=True)
print(f"c3 ({len(clips)} clips, {arith}): {tot_vox_it / (tot_ms * 1e-3):.4e} voxel-iter/s, "
      f"{tot_ms:.2f} ms for the batch on one GPU")
