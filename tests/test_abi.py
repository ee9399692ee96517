"""C-ABI boundary tests that need no GPU: the libraries load, export every
entry point include/*.h declares, host-side configuration logic matches the
reference, and compute calls fail loudly (no CPU fallback) without a device."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import synth
from paper_1907_02731_b200.engine import (Context, KernelConfig, ParameterError, SfsegConfig,
                                          make_gaussian_kernel)
from tests.oracle_lib import Reference, reference_available

ROOT = Path(__file__).resolve().parents[1]


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfseg_[a-z0-9_]+)\s*\(", text)))


def test_cuda_library_exports_every_declared_symbol():
    lib = C.CDLL(str(N.CUDA_LIB))
    names = declared("sfseg_cuda.h")
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(N.EXPORTED_SYMBOLS) <= set(names)


def test_synth_library_exports_every_declared_symbol():
    lib = C.CDLL(str(N.SYNTH_LIB))
    for n in declared("sfseg_synth.h"):
        assert hasattr(lib, n), n


def test_dropin_library_exports_the_engine_and_conv3d_symbols():
    so = N.LIB_DIR / "libsfseg_engine_cuda.so"
    if not so.exists():
        pytest.skip("drop-in not built (needs the reference headers)")
    import subprocess

    syms = subprocess.run(["nm", "-DC", str(so)], capture_output=True, text=True).stdout
    for want in ["sfseg::SfsegConfig::validate() const", "sfseg::sfseg_step_channel(",
                 "sfseg::sfseg_step(", "sfseg::normalize_l2(", "sfseg::project_binary(",
                 "sfseg::threshold_final(", "sfseg::run(", "sfseg::make_gaussian_kernel(",
                 "sfseg::convolve_separable(", "sfseg::convolve_direct(",
                 "sfseg::separable_convolution_count()"]:
        assert any(want in ln and " T " in ln for ln in syms.splitlines()), want


def test_config_validation_mirrors_engine_cpp():
    SfsegConfig().validate()
    bad = [dict(alpha=0.0), dict(p=-0.1), dict(iterations=0), dict(binarize_start=0),
           dict(sigmoid_slope0=0.0), dict(slope_growth=0.5), dict(threshold_frac=0.0),
           dict(final_threshold=1.0), dict(kernel=KernelConfig((1, 3, 3), (0.5, 0.0, 1.5))),
           dict(kernel=KernelConfig((1, 3, -1), (0.5, 1.5, 1.5))), dict(temporal_window=0),
           dict(alpha=1.5)]
    for b in bad:
        with pytest.raises(ParameterError):
            SfsegConfig(**b).validate()
    SfsegConfig(alpha=1.5, allow_negative_affinity=True).validate()
    assert SfsegConfig(temporal_window=3).resolved_temporal_window() == 3
    assert SfsegConfig().resolved_temporal_window() == 1
    if reference_available():
        ref = Reference()
        for b in bad + [dict()]:
            ours = 0
            try:
                SfsegConfig(**b).validate()
            except ParameterError:
                ours = 1
            assert ours == (ref.validate(SfsegConfig(**b)) != 0)


def test_host_taps_match_reference_bit_for_bit():
    if not reference_available():
        pytest.skip("reference library not built")
    ref = Reference()
    for radii, sigmas in [((1, 3, 3), (0.5, 1.5, 1.5)), ((4, 10, 10), (0.5, 1.5, 1.5)),
                          ((3, 7, 7), (1e30, 5.0, 5.0)), ((0, 2, 5), (0.3, 2.2, 9.0))]:
        k = make_gaussian_kernel(sigmas, radii)
        rt, ry, rx = ref.make_kernel(radii, sigmas)
        assert np.array_equal(k.taps_t, rt) and np.array_equal(k.taps_y, ry)
        assert np.array_equal(k.taps_x, rx)
    tt, _, _ = ref.make_kernel((3, 7, 7), (1e30, 5.0, 5.0))
    assert np.all(tt == tt[0])  # sigma = 1e30 is a box


def test_no_cpu_fallback_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(N.CudaError):
        Context(0)


def test_synth_is_seeded_and_thread_count_invariant():
    prob = synth.config(0)[0]
    a, ma = prob.generate(threads=1, mask=True)
    b, mb = prob.generate(threads=7, mask=True)
    assert np.array_equal(a.unary, b.unary) and np.array_equal(ma, mb)
    assert a.unary.min() >= 0.0 and a.unary.max() <= 1.0
    assert 0.02 < ma.mean() < 0.5
    c2 = synth.config(2, frames=3)[0]
    fs, _ = c2.generate()
    assert len(fs.pairwise) == 8
    mean = sum(fs.pairwise[1:], fs.pairwise[0].copy())  # S = mean of channels (float32)
    assert np.allclose(fs.unary, mean / np.float32(8), atol=1e-6)
    clips = synth.config(3)
    assert len(clips) == 14 and all(21 <= p.shape[0] <= 279 for p in clips)
    assert {p.shape[1:] for p in clips} <= {(240, 320), (360, 640)}


def test_synth_rng_is_the_reference_stream():
    if not reference_available():
        pytest.skip("reference library not built")
    ref = Reference()
    assert np.array_equal(synth.xoshiro_u64(42, 100), ref.xoshiro_u64(42, 100))
    assert np.array_equal(synth.xoshiro_gaussian(42, 100), ref.xoshiro_gaussian(42, 100))


def test_convergence_criterion_is_validated_on_the_host():
    """run_until_converged rejects an unknown stopping rule before any device
    work (the C ABI returns SFSEG_ERR_PARAMETER for it as well)."""
    from paper_1907_02731_b200 import engine as E

    fs = E.FeatureSet(np.zeros((2, 4, 4), np.float32), [np.zeros((2, 4, 4), np.float32)])
    with pytest.raises(E.ParameterError):
        E.run_until_converged(fs, E.SfsegConfig(), 1e-6, criterion="residual")


@pytest.mark.parametrize("idx,frames,rng", [(1, 10, (3, 7)), (2, 6, (0, 2)), (4, 5, (2, 5))])
def test_synth_frame_range_is_the_slab_of_the_whole_volume(idx, frames, rng):
    # a time shard generates only its buffer frames (sfseg_synth_generate_frames)
    prob = synth.config(idx, frames=frames)[0]
    whole, m = prob.generate(mask=True)
    part, pm = prob.generate(mask=True, frame_range=rng)
    t0, t1 = rng
    assert np.array_equal(part.unary, whole.unary[t0:t1])
    assert all(np.array_equal(a, b[t0:t1]) for a, b in zip(part.pairwise, whole.pairwise))
    assert np.array_equal(pm, m[t0:t1])


def test_headers_are_plain_c99(tmp_path):
    # the drop-in boundary is a C ABI: both headers must compile as C (no C++
    # constructs, no torch / CUDA types in the signatures)
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        pytest.skip("no C compiler")
    src = tmp_path / "hdr.c"
    src.write_text('#include "sfseg_cuda.h"\n#include "sfseg_synth.h"\n'
                   "int main(void) { sfseg_clip c; sfseg_params p; sfseg_iter_record r;\n"
                   "  (void)c; (void)p; (void)r; return 0; }\n")
    inc = N.CUDA_LIB.parents[2] / "include"
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only",
                        f"-I{inc}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
