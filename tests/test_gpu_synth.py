"""Device-side synthetic generation against the host
generator (libsfseg_synth.so), on every BASELINE config (T-cropped).

sfseg_synth_generate_device jumps each (stream, frame) xoshiro256** generator
to a thread's run of pixels with GF(2) jump matrices and repeats the host's
draws with separately rounded double arithmetic, so:
  * the clean object mask, uniform-noise and noiseless fields are
    bit-identical to the host generator (c0 uniform noise, c2's geometry);
  * gaussian fields differ only where the device log/cos lands one ulp away
    from glibc and that survives the cast to float: at most one float ulp,
    in a tiny fraction of voxels (bounded below);
  * the generation is deterministic, and a run of pixels that straddles a row
    or starts mid-frame draws the same values as the sequential stream.
"""
import numpy as np
import pytest

from paper_1907_02731_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ULP1 = 2.0 ** -24  # one float ulp just below 1.0 (all values lie in [0, 1])

CASES = [(0, None, 0), (1, 3, 0), (2, 2, 0), (3, 3, 0), (3, 3, 5), (4, 2, 0)]


def _problem(cfg, frames, clip):
    return synth.config(cfg, frames=frames)[clip]


def _cmp(host, dev, gaussian, what):
    d = dev.cpu().numpy()
    if not gaussian:
        assert np.array_equal(host, d), f"{what}: {int(np.sum(host != d))} values differ"
        return
    diff = np.abs(host.astype(np.float64) - d.astype(np.float64))
    nd = int(np.count_nonzero(diff))
    assert float(diff.max()) <= 2 * ULP1, (what, float(diff.max()))
    assert nd <= max(2, 1e-4 * host.size), (what, nd, host.size)


@pytest.mark.parametrize("cfg,frames,clip", CASES)
def test_device_synth_matches_host_generator(cfg, frames, clip):
    prob = _problem(cfg, frames, clip)
    fs, mask = prob.generate(mask=True)
    S, F, m = prob.generate_device(mask=True)
    torch.cuda.synchronize()
    assert np.array_equal(mask, m.cpu().numpy())
    sp = prob.spec
    s_gauss = sp.noise == synth.NOISE_GAUSSIAN or sp.feature_mode == synth.FEAT_MEAN_OF_F
    _cmp(fs.unary, S, s_gauss, f"c{cfg} S")
    f_gauss = sp.feature_mode != synth.FEAT_SAME or s_gauss
    for c in range(prob.channels):
        _cmp(fs.pairwise[c], F[c], f_gauss, f"c{cfg} F{c}")


def test_device_synth_uniform_noise_bit_exact_multichunk():
    # c0's layout (uniform noise, one draw per pixel) on a plane that is not a
    # multiple of the 1024-pixel run and spans several runs per row
    prob = synth.config(0)[0]
    sp = prob.spec
    sp.height, sp.width, sp.frames = 37, 1500, 3
    prob.shape = (3, 37, 1500)
    fs, mask = prob.generate(mask=True)
    S, F, m = prob.generate_device(mask=True)
    assert np.array_equal(fs.unary, S.cpu().numpy())
    assert np.array_equal(fs.pairwise[0], F[0].cpu().numpy())
    assert np.array_equal(mask, m.cpu().numpy())


def test_device_synth_is_deterministic():
    prob = synth.config(1, frames=2)[0]
    a = prob.generate_device()
    b = prob.generate_device()
    assert torch.equal(a[0], b[0]) and all(torch.equal(x, y) for x, y in zip(a[1], b[1]))


def test_device_synth_rejects_bad_specs():
    prob = synth.config(0)[0]
    prob.spec.objects = 0
    with pytest.raises(ValueError):
        prob.generate_device()
