"""Multi-rank (time-sharded) driver on CPU: gloo, world_size 2 and 3, with the
oracle as the per-shard compute. The CUDA path runs the same driver with
CudaBackend over NCCL (bench.py --gpus N); here the exchange and reduction
logic is checked: results must be bit-identical for any number of ranks and
match the single-process reference run within the north-star tolerance."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02731_b200.engine import KernelConfig, SfsegConfig
from paper_1907_02731_b200.sharding import ShardedSolver, buffer_range, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(T=9, H=20, W=36, C=1, seed=3):
    from tests.oracle_lib import random_volume

    S = random_volume((T, H, W), seed)
    F = [random_volume((T, H, W), seed + 1 + c) for c in range(C)]
    return S, F


def _cfg(binarize):
    return SfsegConfig(kernel=KernelConfig((2, 3, 3), (0.7, 1.2, 1.2)), iterations=4,
                       binarize_start=3 if binarize else 5, p=0.2)


def _worker(rank, world, port, binarize, C, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.shard_oracle_backend import OracleBackend

        S, F = _problem(C=C)
        T, H, W = S.shape
        cfg = _cfg(binarize)
        halo = cfg.kernel.radii[0]
        t0, t1 = shard_range(T, world, rank)
        b0, b1 = buffer_range(T, t0, t1, halo)
        solver = ShardedSolver(OracleBackend(), rank, world)
        solver.load(T, H, W, torch.from_numpy(S[b0:b1].copy()),
                    [torch.from_numpy(f[b0:b1].copy()) for f in F], None, halo)
        soft, mask, norms = solver.run(cfg)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), soft=soft, mask=mask, norms=norms,
                 t0=t0, t1=t1)
    finally:
        dist.destroy_process_group()


def _run(world, binarize, C, tmp_path):
    out = tmp_path / f"w{world}"
    out.mkdir()
    mp.spawn(_worker, args=(world, _free_port(), binarize, C, str(out)), nprocs=world, join=True)
    parts = [np.load(out / f"r{r}.npz") for r in range(world)]
    soft = np.concatenate([p["soft"] for p in parts])
    mask = np.concatenate([p["mask"] for p in parts])
    norms = parts[0]["norms"]
    for p in parts[1:]:
        assert np.array_equal(p["norms"], norms)  # every rank derived the same scalars
    return soft, mask, norms


@pytest.mark.parametrize("binarize,C", [(False, 1), (True, 2)])
def test_sharded_equals_single_and_reference(tmp_path, binarize, C):
    from tests.oracle_lib import Oracle

    s1, m1, n1 = _run(1, binarize, C, tmp_path)
    s2, m2, n2 = _run(2, binarize, C, tmp_path)
    s3, m3, n3 = _run(3, binarize, C, tmp_path)
    # GPU-count invariance: bit-identical for 1, 2, 3 ranks
    assert np.array_equal(s1, s2) and np.array_equal(s1, s3)
    assert np.array_equal(m1, m2) and np.array_equal(m1, m3)
    assert np.array_equal(n1, n2) and np.array_equal(n1, n3)
    # and the reference algorithm (serial fp64 norm) within tolerance
    S, F = _problem(C=C)
    soft, mask, norms, _ = Oracle().run(S, F, _cfg(binarize))
    assert np.max(np.abs(s1.astype(np.float64) - soft)) <= 1e-6
    assert np.allclose(n1, norms, rtol=1e-12)


def test_shard_ranges_cover_and_balance():
    for T in (1, 7, 80, 1024):
        for world in (1, 2, 3, 8):
            if world > T:
                continue
            rs = [shard_range(T, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == T
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
            for a, b in rs:
                lo, hi = buffer_range(T, a, b, 4)
                assert lo == max(0, a - 4) and hi == min(T, b + 4)


def _guard_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.shard_oracle_backend import OracleBackend

        S, F = _problem(C=2)
        F = [(2.0 * f - 0.5).astype(np.float32) for f in F]  # leaves [0, 1]: the guard rescales
        T, H, W = S.shape
        cfg = _cfg(False)
        t0, t1 = shard_range(T, world, rank)
        b0, b1 = buffer_range(T, t0, t1, cfg.kernel.radii[0])
        mine = [np.ascontiguousarray(f[b0:b1]) for f in F]
        before = [m.copy() for m in mine]
        solver = ShardedSolver(OracleBackend(), rank, world)
        solver.load(T, H, W, torch.from_numpy(S[b0:b1].copy()), mine, None, cfg.kernel.radii[0])
        unchanged = all(np.array_equal(a, b) for a, b in zip(mine, before))
        bad_cfg = False
        try:
            solver.run(SfsegConfig(**{**cfg.__dict__, "allow_negative_affinity": True,
                                      "alpha": 1.0}))
        except Exception:
            bad_cfg = True
        soft, mask, norms = solver.run(cfg)
        np.savez(os.path.join(out_dir, f"g{rank}.npz"), soft=soft, unchanged=unchanged,
                 bad_cfg=bad_cfg)
    finally:
        dist.destroy_process_group()


def test_sharded_unit_range_guard_uses_global_range_on_copies(tmp_path):
    """engine.cpp:254-259: channels outside [0, 1] are rescaled with the
    channel's GLOBAL min/max (an all-reduce across ranks), on copies (the
    caller's arrays keep their bits), and a solve whose config disagrees with
    the guard decision taken at load is refused."""
    from tests.oracle_lib import Oracle

    world = 2
    mp.spawn(_guard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"g{r}.npz") for r in range(world)]
    assert all(bool(p["unchanged"]) for p in parts)
    assert all(bool(p["bad_cfg"]) for p in parts)
    soft = np.concatenate([p["soft"] for p in parts])
    S, F = _problem(C=2)
    F = [(2.0 * f - 0.5).astype(np.float32) for f in F]
    want, _, _, _ = Oracle().run(S, F, _cfg(False))
    assert np.max(np.abs(soft.astype(np.float64) - want)) <= 1e-6
