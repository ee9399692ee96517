"""sfseg_load_files / engine.run_files: SFSV containers streamed into device
memory (the load path of volume.cpp:142-184 feeding the
resident solve context). Results must equal the in-memory path bit for bit,
and every malformed file must fail with load_volume's status."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from tests import sfsv_util as U
from tests.oracle_lib import Reference, random_volume, reference_available

pytestmark = pytest.mark.gpu


def _write(path, v):
    # the reference's own writer where it is built (pins the format), else ours
    if reference_available():
        Reference().save_volume(path, v)
    else:
        U.write(path, v)


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_run_files_equals_in_memory_run(tmp_path, arith):
    prob = synth.config(2, frames=6)[0]  # C = 8 channels, radii (3, 7, 7)
    fs, _ = prob.generate()
    sl = (slice(None), slice(0, 70), slice(0, 100))
    S = np.ascontiguousarray(fs.unary[sl])
    F = [np.ascontiguousarray(f[sl]) for f in fs.pairwise]
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 6})
    _write(tmp_path / "S.sfsv", S)
    for i, f in enumerate(F):
        _write(tmp_path / f"F{i}.sfsv", f)
    got = E.run_files(tmp_path / "S.sfsv", [tmp_path / f"F{i}.sfsv" for i in range(len(F))], cfg)
    want = E.run(E.FeatureSet(S, F), cfg)
    assert np.array_equal(got.soft, want.soft)
    assert np.array_equal(got.mask, want.mask)
    assert [r.l2_norm_pre_normalize for r in got.trace.iterations] == \
        [r.l2_norm_pre_normalize for r in want.trace.iterations]


@pytest.mark.parametrize("shape", [(5, 480, 854), (3, 256, 1024), (1, 1, 1)])
def test_streamed_payload_is_exact(tmp_path, shape):
    # chunking (32 MB pinned buffers; 5x480x854 is 8.2 MB per field, so use
    # a taller file too), the re-pitch path (W % 32 != 0) and the direct path
    T, H, W = shape
    if T * H * W * 4 < (40 << 20) and shape != (1, 1, 1):
        T = (40 << 20) // (H * W * 4) + 1
    S = random_volume((T, H, W), 3)
    U.write(tmp_path / "S.sfsv", S)
    U.write(tmp_path / "x0.sfsv", S[::-1].copy())
    ctx = E.Context(0)
    lib = ctx._lib
    paths = (C.c_char_p * 1)(str(tmp_path / "S.sfsv").encode())
    N.check(lib.sfseg_load_files(ctx.handle, str(tmp_path / "S.sfsv").encode(),
                                 C.cast(paths, C.c_void_p), 1, str(tmp_path / "x0.sfsv").encode()))
    out = np.empty((T, H, W), np.float32)
    # before any iteration the visible iterate is x0 as stored (engine.cpp:267-270)
    N.check(lib.sfseg_download(ctx.handle, 0.5, out.ctypes.data_as(C.c_void_p), None,
                               N.SFSEG_MEM_HOST))
    assert np.array_equal(out, S[::-1])
    ctx.close()


def test_malformed_files_fail_like_load_volume(tmp_path):
    v = random_volume((2, 40, 70), 6)
    U.write(tmp_path / "ok.sfsv", v)
    ctx = E.Context(0)
    lib = ctx._lib
    for name, path, code in U.malformed_cases(tmp_path, v):
        if reference_available():
            assert Reference().load_volume_rc(path)[0] == code, name
        # as the unary volume, and as a pairwise channel next to a good unary
        for unary, chan in ((path, tmp_path / "ok.sfsv"), (tmp_path / "ok.sfsv", path)):
            paths = (C.c_char_p * 1)(str(chan).encode())
            rc = lib.sfseg_load_files(ctx.handle, str(unary).encode(), C.cast(paths, C.c_void_p), 1,
                                      None)
            assert rc == code, f"{name}: status {rc} ({lib.sfseg_last_error().decode()}), want {code}"
    # channel shape differs from the unary shape (volume.cpp:90-91)
    U.write(tmp_path / "small.sfsv", v[:, :20])
    paths = (C.c_char_p * 1)(str(tmp_path / "small.sfsv").encode())
    assert lib.sfseg_load_files(ctx.handle, str(tmp_path / "ok.sfsv").encode(),
                                C.cast(paths, C.c_void_p), 1, None) == N.SFSEG_ERR_SHAPE
    # a negative unary value (FeatureSet::validate roles, volume.cpp:76-81)
    U.write(tmp_path / "neg.sfsv", v - 0.5)
    paths = (C.c_char_p * 1)(str(tmp_path / "ok.sfsv").encode())
    assert lib.sfseg_load_files(ctx.handle, str(tmp_path / "neg.sfsv").encode(),
                                C.cast(paths, C.c_void_p), 1, None) == N.SFSEG_ERR_VALIDATION
    with pytest.raises(E.IoError):
        E.run_files(tmp_path / "nope.sfsv", [tmp_path / "ok.sfsv"], E.SfsegConfig())
    ctx.close()
