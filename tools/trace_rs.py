"""Per-plane timeline of fused_step_rs (debug build with -DSFK_TRACE):
python tools/trace_rs.py build/lib_trace.so  -> mean stage durations in SM cycles."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth

lib = N.load_library(sys.argv[1])
lib.sfseg_debug_trace.argtypes = [C.c_void_p]
prob = synth.config(1)[0]
fs, _ = prob.generate()
cfg = prob.cfg
cfg.arith = "fast"
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
lo, hi = 8, 60
def span(c, x, y, off):
    """mean of ev_y[i + off] - ev_x[i]"""
    a = tr[c, lo:hi, x]
    b = tr[c, lo + off:hi + off, y]
    ok = (a > 0) & (b > 0)
    d = (b - a)[ok]
    return d.mean() if len(d) else float("nan")

for c in range(2):
    print(f"CTA {c}:")
    print("  A0: raw wait %.0f | xb_empty wait %.0f | x-pass %.0f | bar %.0f | issue+loop -> next %.0f | per plane %.0f" % (
        span(c, 0, 1, 0), span(c, 1, 2, 0), span(c, 2, 3, 0), span(c, 3, 4, 0), span(c, 4, 0, 1), span(c, 0, 0, 1)))
    print("  A2: wait+x-pass %.0f" % span(c, 13, 14, 0))
    # B: cnt-indexed 6,7,8 ; ecnt-indexed 9,10,11 with ecnt e <-> cnt e+2
    print("  B0: xb_full wait %.0f | y-pass %.0f | arrive+t-pass %.0f | slab wait %.0f | recomb+store %.0f | red+loop -> next y %.0f | per plane %.0f" % (
        span(c, 6, 7, 0), span(c, 7, 8, 0), np.nanmean([tr[c, i, 9] - tr[c, i + 2, 8] for i in range(lo, hi)]),
        span(c, 9, 10, 0), span(c, 10, 11, 0), np.nanmean([tr[c, i + 3, 6] - tr[c, i, 11] for i in range(lo, hi)]), span(c, 6, 6, 1)))
    print("  B xb_full seen - A0 x-pass end %.0f" % span(c, 3, 7, 0))
