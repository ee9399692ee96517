import ctypes as C, sys, time, torch
sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N, engine as E, synth
prob = synth.config(1)[0]; T, H, W = prob.shape
S = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
F = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
prob.generate(out=(S.numpy(), [F.numpy()]))
cfg = prob.cfg; cfg.arith = "fast"; p = cfg.to_params()
ctx = E.Context(0); lib = ctx._lib
fp = (C.c_void_p * 1)(F.data_ptr())
def tm(f):
    ctx.synchronize(); t0 = time.perf_counter(); f(); ctx.synchronize(); return 1e3 * (time.perf_counter() - t0)
load = lambda: N.check(lib.sfseg_load(ctx.handle, T, H, W, 1, C.c_void_p(S.data_ptr()), C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
solve = lambda: N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, None))
for rep in range(3):
    a = tm(load); b = tm(solve); c = tm(solve); time.sleep(0.005); d = tm(solve)
    print(f"load {a:.2f} solve-after-load {b:.2f} solve-again {c:.2f} solve-after-5ms-idle {d:.2f}")
