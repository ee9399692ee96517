"""Per-plane pipeline timeline of the fused kernel (debug build with
-DSFK_TRACE; tools/ablate.sh-style lib in lib/ablate/libsfseg_cuda_trace.so).
Runs a few c1 iterations and prints the average duration of every stage in
SM cycles (CTA 0..3, planes 8..100 of the last launch)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

path = sys.argv[1] if len(sys.argv) > 1 else "paper_1907_02731_b200/lib/ablate/libsfseg_cuda_trace.so"
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
lib = N.load_library(path)
lib.sfseg_debug_trace.argtypes = [C.c_void_p]
prob = synth.config(1)[0]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = arith
cfg.iterations = 3
cfg.binarize_start = 4
T, H, W = prob.shape
h = C.c_void_p()
assert lib.sfseg_ctx_create(0, C.byref(h)) == 0
q = cfg.to_params()
fp = (C.c_void_p * 1)(fs.pairwise[0].ctypes.data)
assert lib.sfseg_load(h, T, H, W, 1, C.c_void_p(fs.unary.ctypes.data), C.cast(fp, C.c_void_p), None,
                      N.SFSEG_MEM_HOST) == 0
lib.sfseg_solve(h, C.byref(q), 1, 3, None)
tr = np.zeros((4, 128, 16), np.uint64)
assert lib.sfseg_debug_trace(tr.ctypes.data) == 0
tr = tr.astype(np.int64)
lo, hi = 8, 100
names = {
    "A raw wait (1-0)": (0, 1, 0), "A products+bar (2-1)": (1, 2, 0), "A xb_empty wait (3-2)": (2, 3, 0),
    "A x-pass (4-3)": (3, 4, 0), "A end bar (5-4)": (4, 5, 0), "A loop tail->next raw wait (0'-5)": (5, 0, 1),
    "A per plane (0'-0)": (0, 0, 1),
    "B xb_full wait (7-6)": (6, 7, 0), "B y-pass (8-7)": (7, 8, 0), "B per plane (6'-6)": (6, 6, 1),
    "B slab wait (10-9)": (9, 10, 0), "B epi after slab (11-10)": (10, 11, 0),
    "B warp7 epi end - warp0 (12-11)": (11, 12, 0),
}
for c in range(4):
    print(f"CTA {c}:")
    for n, (a, b, nxt) in names.items():
        d = tr[c, lo + nxt:hi + nxt, b] - tr[c, lo:hi, a]
        d = d[(tr[c, lo:hi, a] > 0) & (tr[c, lo + nxt:hi + nxt, b] > 0)]
        if len(d):
            print(f"  {n:36s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  min {d.min():8d}  max {d.max():8d}")
    # when does B's xb_full wait end relative to A's x-pass end (same plane)?
    d = tr[c, lo:hi, 7] - tr[c, lo:hi, 4]
    print(f"  {'B sees xb_full - A x-pass end (7-4)':36s} mean {d.mean():8.0f}")
    d = tr[c, lo:hi, 3] - tr[c, lo - 2:hi - 2, 8]
    print(f"  {'A xb_empty ok - B y-pass(p-2) end':36s} mean {d.mean():8.0f}")
