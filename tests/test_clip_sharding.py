"""Clip sharding (BASELINE configs[3]: a batch of independent clips, no halo
exchange): LPT assignment properties on the real c3 batch, and a gloo
world-2 run where each rank solves its clips with the CPU oracle and rank 0
checks that the union covers the batch once with the single-rank results."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02731_b200 import synth
from paper_1907_02731_b200.sharding import assign_clips


def test_assignment_covers_each_clip_once_and_balances():
    vox = [p.voxels() for p in synth.config(3)]
    for world in (1, 2, 4, 8):
        parts = assign_clips(vox, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(vox)))
        loads = [sum(vox[i] for i in p) for p in parts]
        # LPT bound: max load <= mean + largest clip
        assert max(loads) <= sum(vox) / world + max(vox)
        assert parts == assign_clips(vox, world)  # deterministic
    assert assign_clips(vox, 1) == [sorted(range(len(vox)), key=lambda i: (-vox[i], i))]


def test_assignment_edge_cases():
    assert assign_clips([], 3) == [[], [], []]
    assert assign_clips([5], 2) == [[0], []]
    assert assign_clips([3, 3, 3, 3], 2) == [[0, 2], [1, 3]]
    with pytest.raises(ValueError):
        assign_clips([1], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _clips():
    from tests.oracle_lib import random_volume
    from paper_1907_02731_b200.engine import KernelConfig, SfsegConfig

    shapes = [(5, 12, 20), (3, 16, 16), (6, 10, 14), (4, 8, 24), (2, 20, 20)]
    cfg = SfsegConfig(kernel=KernelConfig((1, 2, 2), (0.7, 1.2, 1.2)), iterations=3,
                      binarize_start=4)
    return [(random_volume(s, 40 + i), [random_volume(s, 60 + i)], cfg) for i, s in enumerate(shapes)]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.oracle_lib import Oracle

        clips = _clips()
        mine = assign_clips([c[0].size for c in clips], world)[rank]
        res = {}
        for i in mine:
            S, F, cfg = clips[i]
            soft, mask, norms, _ = Oracle().run(S, F, cfg)
            res[str(i)] = soft
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
        dist.barrier()  # no data-path collective: only the end-of-batch join
    finally:
        dist.destroy_process_group()


def test_clip_batch_over_two_ranks(tmp_path):
    from tests.oracle_lib import Oracle, oracle_available

    if not oracle_available():
        pytest.skip("oracle not built")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    got = {}
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        for k in d.files:
            assert k not in got
            got[int(k)] = d[k]
    clips = _clips()
    assert sorted(got) == list(range(len(clips)))
    for i, (S, F, cfg) in enumerate(clips):
        soft, _, _, _ = Oracle().run(S, F, cfg)
        assert np.array_equal(got[i], soft)
