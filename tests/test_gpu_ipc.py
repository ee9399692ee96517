"""The multi-process time-sharded driver with the peer-memory halo exchange
(sharding.ShardedSolver + CudaBackend + sfseg_shard_export / set_peers over
CUDA IPC), two processes over gloo sharing the one GPU of the test box. No
kernel waits on another: each rank's next step is ordered behind the other's
halo push by the host-side all-gather, as the NCCL all-gather orders it
across GPUs. The sharded result must equal the single-context solve bit for
bit."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, outdir, arith):
    import torch.distributed as dist

    from paper_1907_02731_b200 import engine as E
    from paper_1907_02731_b200 import synth
    from paper_1907_02731_b200.sharding import CudaBackend, ShardedSolver, buffer_range, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = synth.config(1, frames=12)[0]
    fs, _ = prob.generate()
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 5, "binarize_start": 3})
    T, H, W = prob.shape
    halo = cfg.kernel.radii[0]
    t0, t1 = shard_range(T, world, rank)
    b0, b1 = buffer_range(T, t0, t1, halo)
    solver = ShardedSolver(CudaBackend(0), rank, world)
    solver.load(T, H, W, np.ascontiguousarray(fs.unary[b0:b1]),
                [np.ascontiguousarray(f[b0:b1]) for f in fs.pairwise], None, halo)
    soft, mask, norms = solver.run(cfg)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), soft=soft, mask=mask, norms=np.array(norms),
             p2p=np.array(solver.p2p))
    dist.barrier()
    solver.b.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("arith", ["fast", "exact"])
def test_ipc_peer_halo_two_processes(arith):
    import torch.multiprocessing as mp

    from paper_1907_02731_b200 import engine as E
    from paper_1907_02731_b200 import synth

    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(world, _free_port(), d, arith), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
        assert all(bool(p["p2p"]) for p in parts), "peer-memory exchange was not enabled"
        soft = np.concatenate([p["soft"] for p in parts])
        mask = np.concatenate([p["mask"] for p in parts])
        norms = parts[0]["norms"]
    prob = synth.config(1, frames=12)[0]
    fs, _ = prob.generate()
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 5, "binarize_start": 3})
    ref = E.run(fs, cfg)
    assert np.array_equal(soft, ref.soft)
    assert np.array_equal(mask, ref.mask)
    assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in ref.trace.iterations])
