"""TEST INFRASTRUCTURE ONLY: a CPU backend for paper_1907_02731_b200.sharding
that computes each shard's step with the oracle (oracle/sfseg_oracle.c), so the
NCCL/gloo driver logic (halo exchange, frame-ordered reduction, projection)
can be tested on CPU processes. It mirrors the device semantics of the CUDA
shard API: iterate stored raw, normalise/sigmoid applied on load, per-frame
sums reduced in frame order by the same fixed tree as k_finalize_total.
"""
import math

import numpy as np
import torch

from paper_1907_02731_b200.sharding import StepIO
from tests.oracle_lib import Oracle


def finalize_order_sum(fs: np.ndarray) -> float:
    """k_finalize_total's order: 256 strided sequential sums, then a halving tree."""
    acc = [0.0] * 256
    for i, v in enumerate(fs.tolist()):
        acc[i % 256] += v
    k = 128
    while k > 0:
        for i in range(k):
            acc[i] += acc[i + k]
        k //= 2
    return acc[0]


class OracleBackend:
    def __init__(self):
        self.o = Oracle()

    def load(self, T, H, W, S, F, x0, t0, t1, halo):
        self.T, self.H, self.W, self.t0, self.t1, self.halo = T, H, W, t0, t1, halo
        self.b0 = max(0, t0 - halo)
        self.b1 = min(T, t1 + halo)
        to_np = lambda a: a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        self.S = np.ascontiguousarray(to_np(S), np.float32)
        self.F = [np.ascontiguousarray(to_np(f), np.float32) for f in F]
        self.x = np.ascontiguousarray(to_np(x0 if x0 is not None else S), np.float32).copy()
        self.y = [np.zeros_like(self.S), np.zeros_like(self.S)]
        self.cur = -1
        self.state = dict(mode=0, inv=1.0, theta=0.0, lam=0.0, max_unit=0.0)

    def _transform(self, y):
        st = self.state
        if st["mode"] == 0:
            return y
        xu = (y.astype(np.float64) * st["inv"]).astype(np.float32)
        if st["mode"] == 1:
            return xu
        z = st["lam"] * (xu.astype(np.float64) - st["theta"])
        return (1.0 / (1.0 + np.exp(-z))).astype(np.float32)

    def step(self, params, it):
        cfg = self.cfg
        src = self.x if self.cur < 0 else self.y[self.cur]
        dst = 0 if self.cur < 0 else 1 - self.cur
        xt = self._transform(src)
        full = self.o.step(xt, self.S, self.F, cfg)  # zero padding at the slab edges
        a, b = self.t0 - self.b0, self.t1 - self.b0
        out = self.y[dst]
        out[a:b] = full[a:b]
        self.cur = dst
        ys = out[a:b].astype(np.float64)
        self.frame_sum = np.array([np.sum(ys[t] ** 2) for t in range(b - a)], np.float64)
        self.frame_max = np.array([max(0.0, float(out[a + t].max())) for t in range(b - a)],
                                  np.float32)
        h = min(self.halo, b - a)
        v = lambda lo, hi: torch.from_numpy(out[lo:hi].reshape(-1))
        return StepIO(v(a, a + h) if self.t0 > 0 else None,
                      v(b - h, b) if self.t1 < self.T else None,
                      v(0, a) if self.t0 > 0 else None,
                      v(b, self.b1 - self.b0) if self.t1 < self.T else None,
                      torch.from_numpy(self.frame_sum), torch.from_numpy(self.frame_max))

    def before_exchange(self):
        pass

    def after_exchange(self):
        pass

    def norms(self, count):
        return self._norms[:count]

    def finalize(self, params, it, frame_sum, frame_max):
        cfg = self.cfg
        norm = math.sqrt(finalize_order_sum(frame_sum.numpy()))
        if norm == 0.0:
            raise RuntimeError("degenerate")
        inv = 1.0 / norm
        mx = float(np.float32(max(0.0, float(frame_max.numpy().max()))))
        max_unit = float(np.float32(np.float64(mx) * inv))
        mode = 2 if it >= cfg.binarize_start else 1
        lam = cfg.sigmoid_slope0 * cfg.slope_growth ** (it - cfg.binarize_start)
        self.state = dict(mode=mode, inv=inv, theta=cfg.threshold_frac * max_unit, lam=lam,
                          max_unit=max_unit)
        if it == 1:
            self._norms = []
        self._norms.append(norm)

    def download(self, frac, t0, t1):
        a, b = self.t0 - self.b0, self.t1 - self.b0
        x = self._transform(self.y[self.cur])[a:b]
        st = self.state
        m = np.float32(st["max_unit"])
        if st["mode"] == 2:
            m = np.float32(1.0 / (1.0 + math.exp(-st["lam"] * (float(m) - st["theta"]))))
        cut = np.float32(frac * float(m))
        return x, (x > cut).astype(np.uint8)

