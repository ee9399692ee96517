"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/
libsfseg_ref.so, compiled unchanged from /root/reference/proj/src). Run in the
build container: python tests/golden/make_golden.py

The reference ships no golden vectors; these fixtures pin
the oracle and the GPU path on machines without the reference sources.
Inputs are stored with the outputs, so a fixture does not depend on the
generators that produced it."""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from paper_1907_02731_b200.engine import KernelConfig, SfsegConfig  # noqa: E402
from paper_1907_02731_b200 import synth  # noqa: E402
from tests.oracle_lib import Reference, random_volume  # noqa: E402


def params_dict(cfg):
    return dict(alpha=cfg.alpha, p=cfg.p, radii=np.array(cfg.kernel.radii),
                sigmas=np.array(cfg.kernel.sigmas), iterations=cfg.iterations,
                binarize_start=cfg.binarize_start, slope0=cfg.sigmoid_slope0,
                growth=cfg.slope_growth, threshold_frac=cfg.threshold_frac,
                final_threshold=cfg.final_threshold,
                allow_negative=int(cfg.allow_negative_affinity))


def main():
    ref = Reference()
    # 1. single-channel steps: the four cases of test_engine.cpp:161-191
    cases = [((4, 8, 8), 1.0, 0.1, (1, 3, 3), (0.5, 1.5, 1.5)),
             ((4, 8, 8), 0.7, 0.5, (1, 1, 1), (0.9, 0.9, 0.9)),
             ((3, 6, 6), 1.0, 0.0, (0, 2, 2), (1.0, 2.0, 2.0)),
             ((2, 5, 7), 0.5, 1.0, (1, 2, 2), (0.7, 1.2, 1.2))]
    out = {}
    for i, (shape, alpha, p, radii, sigmas) in enumerate(cases):
        cfg = SfsegConfig(alpha=alpha, p=p, kernel=KernelConfig(radii, sigmas))
        S, f, x = (random_volume(shape, 10 * i + k) for k in (1, 2, 3))
        out[f"step{i}_S"], out[f"step{i}_F"], out[f"step{i}_x"] = S, f, x
        out[f"step{i}_out"] = ref.step(x, S, [f], cfg)
        for k, v in params_dict(cfg).items():
            out[f"step{i}_cfg_{k}"] = v
    # 2. a 3-channel step (test_engine.cpp:193-215)
    cfg = SfsegConfig(p=0.3, kernel=KernelConfig((1, 2, 2), (0.6, 1.1, 1.1)))
    S = random_volume((3, 7, 7), 101)
    F = [random_volume((3, 7, 7), 102 + c) for c in range(3)]
    x = random_volume((3, 7, 7), 110)
    out.update(mc_S=S, mc_F=np.stack(F), mc_x=x, mc_out=ref.step(x, S, F, cfg))
    # 3. BASELINE configs[0] full run, binarisation off and on, checkpoints
    prob = synth.config(0)[0]
    fs, _ = prob.generate()
    out.update(c0_S=fs.unary, c0_F=fs.pairwise[0])
    for tag, start in (("pi", prob.cfg.iterations + 1), ("bin", 3)):
        cfg = SfsegConfig(**{**prob.cfg.__dict__, "binarize_start": start})
        soft, mask, norms, ck = ref.run(fs.unary, fs.pairwise, cfg, checkpoints=[1, 5, 10, 20])
        out[f"c0_{tag}_soft"], out[f"c0_{tag}_mask"] = soft, mask
        out[f"c0_{tag}_norms"], out[f"c0_{tag}_ck"] = norms, ck
        for k, v in params_dict(cfg).items():
            out[f"c0_{tag}_cfg_{k}"] = v
    # 4. separable convolution and kernel taps
    v = random_volume((5, 17, 23), 55)
    out.update(conv_v=v, conv_out=ref.convolve_separable(v, (2, 3, 4), (0.8, 1.3, 2.1)))
    tt, ty, tx = ref.make_kernel((2, 5, 5), (0.5, 1.5, 1.5))
    out.update(taps_t=tt, taps_y=ty, taps_x=tx)
    # 5. RNG streams (rng.hpp)
    out.update(rng_u64=ref.xoshiro_u64(20190708, 64), rng_gauss=ref.xoshiro_gaussian(7, 64))
    np.savez_compressed(HERE / "reference_vectors.npz", **out)
    print("wrote", HERE / "reference_vectors.npz")


if __name__ == "__main__":
    main()
