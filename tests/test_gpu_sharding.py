"""CUDA shard API (sfseg_shard_*) on one GPU: two shard contexts stand in for
two ranks; the host copies the halos and concatenates the per-frame sums the
way NCCL send/recv + all-gather do in sharding.py. No kernel waits on
another (the exchange is host-driven), so this is a faithful single-GPU test
of the multi-GPU data path. The sharded result must equal the single-context
solve bit for bit."""
import numpy as np
import pytest
import torch

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from paper_1907_02731_b200.sharding import CudaBackend, buffer_range, shard_range

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,arith,binarize,idx", [
    (2, "exact", False, 1), (3, "fast", True, 1),
    (2, "fast", False, 2),  # C = 8: the (C + 2)-field launches (fused_mc.cuh) per shard
    (3, "fast", True, 4),   # C = 3, radii (4, 10, 10)
])
def test_shards_match_single_context(world, arith, binarize, idx):
    prob = synth.config(idx, frames=12)[0]
    fs, _ = prob.generate()
    if idx != 1:  # crop H, W so the test stays small
        fs = E.FeatureSet(np.ascontiguousarray(fs.unary[:, :100, :150]),
                          [np.ascontiguousarray(f[:, :100, :150]) for f in fs.pairwise])
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 6,
                           "binarize_start": 3 if binarize else 7})
    T, H, W = fs.unary.shape
    halo = cfg.kernel.radii[0]
    ranks = []
    for r in range(world):
        t0, t1 = shard_range(T, world, r)
        b0, b1 = buffer_range(T, t0, t1, halo)
        be = CudaBackend(0)
        be.load(T, H, W, np.ascontiguousarray(fs.unary[b0:b1]),
                [np.ascontiguousarray(f[b0:b1]) for f in fs.pairwise], None, t0, t1, halo)
        be.cfg = cfg
        ranks.append((be, t0, t1))
    params = cfg.to_params()
    norms = []
    for it in range(1, cfg.iterations + 1):
        ios = [be.step(params, it) for be, _, _ in ranks]
        for be, _, _ in ranks:
            be.before_exchange()
        for r in range(world - 1):  # halo exchange between neighbours
            ios[r + 1].recv_lo.copy_(ios[r].send_hi)
            ios[r].recv_hi.copy_(ios[r + 1].send_lo)
        fsum = torch.cat([io.frame_sum for io in ios]).contiguous()
        fmax = torch.cat([io.frame_max for io in ios]).contiguous()
        for be, _, _ in ranks:
            be.after_exchange()
            be.finalize(params, it, fsum, fmax)
    per_rank = [be.norms(cfg.iterations) for be, _, _ in ranks]
    assert all(p == per_rank[0] for p in per_rank)
    norms = per_rank[0]
    soft = np.concatenate([be.download(cfg.final_threshold, a, b)[0] for be, a, b in ranks])
    mask = np.concatenate([be.download(cfg.final_threshold, a, b)[1] for be, a, b in ranks])
    ref = E.run(fs, cfg)
    assert np.array_equal(soft, ref.soft)
    assert np.array_equal(mask, ref.mask)
    assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in ref.trace.iterations])
    for be, _, _ in ranks:
        be.close()


@pytest.mark.parametrize("world,arith,idx", [(2, "fast", 1), (3, "exact", 1), (3, "fast", 2)])
def test_peer_memory_halo_push_matches_single_context(world, arith, idx):
    # sfseg_shard_set_peers: the step pushes its edge frames into the
    # neighbours' halo frames itself (k_halo_push); the driver only gathers
    # the per-frame sums. Contexts of one process stand in for the ranks
    # (raw device pointers instead of IPC handles); the streams are ordered
    # through the host-side gather exactly as the NCCL all-gather orders them.
    prob = synth.config(idx, frames=12)[0]
    fs, _ = prob.generate()
    if idx != 1:
        fs = E.FeatureSet(np.ascontiguousarray(fs.unary[:, :100, :150]),
                          [np.ascontiguousarray(f[:, :100, :150]) for f in fs.pairwise])
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 5,
                           "binarize_start": 3})
    T, H, W = fs.unary.shape
    halo = cfg.kernel.radii[0]
    ranks = []
    for r in range(world):
        t0, t1 = shard_range(T, world, r)
        b0, b1 = buffer_range(T, t0, t1, halo)
        be = CudaBackend(0)
        be.load(T, H, W, np.ascontiguousarray(fs.unary[b0:b1]),
                [np.ascontiguousarray(f[b0:b1]) for f in fs.pairwise], None, t0, t1, halo)
        be.cfg = cfg
        ranks.append((be, t0, t1))
    blobs = [be.export(True) for be, _, _ in ranks]
    for r, (be, _, _) in enumerate(ranks):
        be.set_peers(blobs[r - 1] if r > 0 else None, blobs[r + 1] if r + 1 < world else None)
    params = cfg.to_params()
    for it in range(1, cfg.iterations + 1):
        ios = [be.step(params, it) for be, _, _ in ranks]
        for be, _, _ in ranks:
            be.before_exchange()
        fsum = torch.cat([io.frame_sum for io in ios]).contiguous()
        fmax = torch.cat([io.frame_max for io in ios]).contiguous()
        for be, _, _ in ranks:
            be.after_exchange()
            be.finalize(params, it, fsum, fmax)
    soft = np.concatenate([be.download(cfg.final_threshold, a, b)[0] for be, a, b in ranks])
    ref = E.run(fs, cfg)
    assert np.array_equal(soft, ref.soft)
    norms = ranks[0][0].norms(cfg.iterations)
    assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in ref.trace.iterations])
    # dropping the peers puts the halos back on the driver's send/recv
    for be, _, _ in ranks:
        be.set_peers(None, None)
        be.close()


@pytest.mark.parametrize("arith,idx,binarize", [("fast", 1, False), ("exact", 1, True), ("fast", 2, False)])
def test_sharded_driver_graph_replay_matches_eager(arith, idx, binarize):
    # ShardedSolver captures its iteration loop into a CUDA graph on the
    # second solve and replays it afterwards (no per-iteration host work):
    # eager, capture + replay and replay must give the single-context bits,
    # and a second configuration gets its own graph
    from paper_1907_02731_b200.sharding import ShardedSolver

    prob = synth.config(idx, frames=10)[0]
    fs, _ = prob.generate()
    if idx != 1:
        fs = E.FeatureSet(np.ascontiguousarray(fs.unary[:, :100, :150]),
                          [np.ascontiguousarray(f[:, :100, :150]) for f in fs.pairwise])
    T, H, W = fs.unary.shape
    base = {**prob.cfg.__dict__, "arith": arith, "binarize_start": 3 if binarize else 99}
    cfgs = [E.SfsegConfig(**{**base, "iterations": 5}), E.SfsegConfig(**{**base, "iterations": 4})]
    be = CudaBackend(0)
    solver = ShardedSolver(be, 0, 1)
    try:
        solver.load(T, H, W, fs.unary, fs.pairwise, None, cfgs[0].kernel.radii[0])
        for cfg in cfgs:
            ref = E.run(fs, cfg)
            for call in range(4):  # eager, capture + replay, replay, replay
                soft, mask, norms = solver.run(cfg)
                assert np.array_equal(soft, ref.soft), (cfg.iterations, call)
                assert np.array_equal(mask, ref.mask)
                assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in ref.trace.iterations])
        kinds = [type(v).__name__ for v in solver._graphs.values()]
        assert kinds == ["tuple", "tuple"], kinds  # both loops were captured
        # a reload drops the graphs (they point at the old buffers)
        solver.load(T, H, W, fs.unary, fs.pairwise, None, cfgs[0].kernel.radii[0])
        assert solver._graphs == {}
        soft, _, _ = solver.run(cfgs[0])
        assert np.array_equal(soft, E.run(fs, cfgs[0]).soft)
    finally:
        be.close()
