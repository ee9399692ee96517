"""Out-of-bounds stores and uninitialised reads, checked without a sanitizer.

compute-sanitizer is refused on this GPU pool (tests/test_gpu_sanitizer.py
skips there), so the library carries its own check, SFSEG_DEBUG_GUARD=1:
every volume buffer is allocated with a 64 KiB guard band on either side, and
bands, buffer interiors and pitch padding are filled with a NaN pattern
instead of zeros. The workload of tests/sanitizer_workload.py (every fused
kernel family, the peer push, the stateless step) then has to

* leave every band word untouched (no kernel, TMA store or peer store writes
  outside its buffer), and
* produce finite results that are bit-identical to a normal run (nothing reads
  memory that no kernel wrote: halo frames, pitch padding, ring slots).

The reference's CPU loops index std::vector with no checks either
(CMakeLists.txt:26 has no sanitizer step); this is the sm_100a path's own.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run(out, guard):
    env = dict(os.environ)
    env.pop("SFSEG_DEBUG_GUARD", None)
    if guard:
        env["SFSEG_DEBUG_GUARD"] = "1"
        env["SFSEG_DEBUG_SYNC"] = "1"  # attribute an asynchronous fault to its kernel
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "sanitizer_workload.py"), "--out", str(out)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    return np.load(out)


def test_guard_bands_intact_and_poison_never_read(tmp_path):
    plain = _run(tmp_path / "plain.npz", guard=False)
    guarded = _run(tmp_path / "guard.npz", guard=True)
    assert sorted(plain.files) == sorted(guarded.files) and len(plain.files) >= 10
    for k in plain.files:
        assert np.isfinite(guarded[k]).all(), k
        assert np.array_equal(plain[k], guarded[k]), k


def test_guard_check_detects_a_stray_store():
    # the checker itself: a deliberate out-of-bounds write must be counted
    code = r"""
import ctypes as C, sys
sys.path.insert(0, %r)
import numpy as np
from paper_1907_02731_b200 import _native as N, engine as E
lib = N.load_library()
lib.sfseg_debug_check_guards.argtypes = [C.POINTER(C.c_ulonglong), C.POINTER(C.c_int32)]
S = np.random.default_rng(0).random((4, 40, 40), dtype=np.float32)
cfg = E.SfsegConfig(iterations=2, binarize_start=3, arith="fast")
E.run(E.FeatureSet(S, [S]), cfg)
bad, n = C.c_ulonglong(), C.c_int32()
N.check(lib.sfseg_debug_check_guards(C.byref(bad), C.byref(n)))
assert bad.value == 0 and n.value > 0, (bad.value, n.value)
N.check(lib.sfseg_debug_poke_guard(3))
N.check(lib.sfseg_debug_check_guards(C.byref(bad), C.byref(n)))
assert bad.value == 3, bad.value
print("detected")
""" % str(ROOT)
    env = dict(os.environ, SFSEG_DEBUG_GUARD="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and "detected" in r.stdout, (r.stdout + r.stderr)[-2000:]
