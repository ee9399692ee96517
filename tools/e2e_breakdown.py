"""Where the end-to-end sfseg_run time goes (development aid): times load,
solve and download separately on the c1 workload from pinned host buffers."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth

prob = synth.config(1)[0]
T, H, W = prob.shape
S = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
F = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
prob.generate(out=(S.numpy(), [F.numpy()]))
soft = torch.empty((T, H, W), dtype=torch.float32, pin_memory=True)
mask = torch.empty((T, H, W), dtype=torch.uint8, pin_memory=True)
cfg = prob.cfg
cfg.arith = "fast"
p = cfg.to_params()
ctx = E.Context(0)
lib = ctx._lib
fp = (C.c_void_p * 1)(F.data_ptr())
for rep in range(4):
    ctx.synchronize()
    t0 = time.perf_counter()
    N.check(lib.sfseg_load(ctx.handle, T, H, W, 1, C.c_void_p(S.data_ptr()), C.cast(fp, C.c_void_p), None,
                           N.SFSEG_MEM_HOST))
    ctx.synchronize()
    t1 = time.perf_counter()
    N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, None))
    ctx.synchronize()
    t2 = time.perf_counter()
    N.check(lib.sfseg_download(ctx.handle, cfg.final_threshold, C.c_void_p(soft.data_ptr()),
                               C.c_void_p(mask.data_ptr()), N.SFSEG_MEM_HOST))
    ctx.synchronize()
    t3 = time.perf_counter()
    N.check(lib.sfseg_run(ctx.handle, T, H, W, 1, C.c_void_p(S.data_ptr()), C.cast(fp, C.c_void_p), None,
                          C.byref(p), C.c_void_p(soft.data_ptr()), C.c_void_p(mask.data_ptr()), None,
                          N.SFSEG_MEM_HOST))
    t4 = time.perf_counter()
    print(f"load {1e3 * (t1 - t0):.2f} ms  solve {1e3 * (t2 - t1):.2f} ms  download {1e3 * (t3 - t2):.2f} ms"
          f"  | sfseg_run {1e3 * (t4 - t3):.2f} ms")
