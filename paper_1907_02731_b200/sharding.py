"""Time-sharded SFSeg solve across GPUs (one process per GPU, NCCL).

The reference has no distributed backend (parallel.hpp is its
only parallelism); its per-frame Jacobi sweep (engine.cpp:287-325) is what
makes the time axis shardable: every frame of iterate k+1 depends only on
frames t-rt..t+rt of iterate k. Rank r owns a contiguous range of output
frames and keeps `halo` = rt frames of each neighbour:

  per iteration
    1. fused stencil on the rank's frames            (sfseg_shard_step)
    2. exchange the rt edge frames of the new iterate (NCCL send/recv)
    3. all-gather the per-frame canonical sums / max  (NCCL all-gather)
    4. every rank reduces the frames in frame order   (sfseg_shard_finalize)

Step 4 makes the norm, the projection scalars and therefore every iterate
bit-identical for any number of ranks. The unit-range guard of run()
(engine.cpp:254-259) needs the global min/max of each channel, so it is
applied here with an all-reduce before the channels are loaded.

A backend supplies steps 1, 4 and the device buffers; CudaBackend is the
product (libsfseg_cuda.so). tests/ drive the same driver with a CPU oracle
backend over gloo.

Batches of independent clips (BASELINE configs[3]) need no exchange at all:
assign_clips() packs them onto ranks by voxel count (longest processing time
first) and every rank runs its own clips with its own context.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N


def shard_range(T: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous frames [t0, t1) of rank `rank`."""
    base, rem = divmod(T, world)
    t0 = rank * base + min(rank, rem)
    return t0, t0 + base + (1 if rank < rem else 0)


def assign_clips(voxels: Sequence[int], world: int) -> List[List[int]]:
    """LPT bin-packing of independent clips onto `world` ranks by voxel count:
    clips in decreasing size (ties by index) each go to the least-loaded rank
    (ties by rank). Deterministic; returns the clip indices of every rank in
    the order they were assigned."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(voxels)), key=lambda i: (-int(voxels[i]), i))
    load = [0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(voxels[i])
    return out


def run_clips(clips, cfg, rank: int = 0, world: int = 1, ctxs=None, x0s=None):
    """Clip sharding: this rank's LPT share of a caller's
    batch of independent videos, run through sfseg_run_batch on ``ctxs`` (one
    or more contexts of this rank's GPU; two pipeline transfers under
    solves). No data-path collective. ``clips``: FeatureSets (all of the
    batch, so every rank computes the same assignment from the voxel counts).
    Returns {clip index: RunResult}."""
    from . import engine as E

    vox = [int(np.prod(np.shape(c.unary))) for c in clips]
    mine = assign_clips(vox, world)[rank]
    res = E.run_batch([clips[i] for i in mine], cfg,
                      x0s=None if x0s is None else [x0s[i] for i in mine], ctxs=ctxs)
    return dict(zip(mine, res))


def run_problems(problems, rank: int, world: int, ctxs=None, arith: Optional[str] = None):
    """run_clips for synthetic problems (synth.config(3)): only this rank's
    clips are generated. All clips of a config share one SfsegConfig."""
    from . import engine as E

    mine = assign_clips([p.voxels() for p in problems], world)[rank]
    if not mine:
        return {}
    cfg0 = problems[mine[0]].cfg
    cfg = cfg0 if arith is None else E.SfsegConfig(**{**cfg0.__dict__, "arith": arith})
    clips = [problems[i].generate()[0] for i in mine]
    return dict(zip(mine, E.run_batch(clips, cfg, ctxs=ctxs)))


def buffer_range(T: int, t0: int, t1: int, halo: int) -> Tuple[int, int]:
    return max(0, t0 - halo), min(T, t1 + halo)


class _DeviceView:
    """Zero-copy torch view of device memory owned by libsfseg_cuda."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


def device_tensor(ptr, count: int, dtype="float32"):
    import torch

    if not ptr or count == 0:
        return None
    typestr = {"float32": "<f4", "float64": "<f8", "uint8": "|u1"}[dtype]
    return torch.as_tensor(_DeviceView(int(ptr), int(count), typestr), device="cuda")


@dataclass
class StepIO:
    send_lo: object
    send_hi: object
    recv_lo: object
    recv_hi: object
    frame_sum: object
    frame_max: object


class CudaBackend:
    """Shard of the resident problem on one GPU (libsfseg_cuda shard API)."""

    def __init__(self, device: int = 0):
        import torch

        from .engine import Context

        self.ctx = Context(device)
        self.lib = self.ctx._lib
        # the library's stream, so NCCL (on torch's stream) can be ordered
        # against the kernels without host synchronisation
        self.stream = torch.cuda.ExternalStream(self.lib.sfseg_ctx_stream(self.ctx.handle),
                                                device=torch.device("cuda", device))
        self._keep_gathered = []

    def load(self, T, H, W, S_local, F_local, x0_local, t0, t1, halo):
        import torch

        self.T, self.H, self.W = T, H, W
        self._keep = [S_local] + list(F_local) + ([x0_local] if x0_local is not None else [])
        mem = N.SFSEG_MEM_DEVICE if isinstance(S_local, torch.Tensor) and S_local.is_cuda \
            else N.SFSEG_MEM_HOST
        ptr = lambda a: a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data
        fp = (C.c_void_p * len(F_local))(*[ptr(f) for f in F_local])
        N.check(self.lib.sfseg_shard_load(
            self.ctx.handle, T, H, W, len(F_local), t0, t1, halo, C.c_void_p(ptr(S_local)),
            C.cast(fp, C.c_void_p), C.c_void_p(ptr(x0_local)) if x0_local is not None else None,
            mem))

    def step(self, params, it) -> StepIO:
        io = N.ShardIO()
        N.check(self.lib.sfseg_shard_step(self.ctx.handle, C.byref(params), it, C.byref(io)))
        f = lambda p, b: device_tensor(p, b // 4, "float32")
        return StepIO(f(io.send_lo, io.send_lo_bytes), f(io.send_hi, io.send_hi_bytes),
                      f(io.recv_lo, io.recv_lo_bytes), f(io.recv_hi, io.recv_hi_bytes),
                      device_tensor(io.frame_sum, io.out_frames, "float64"),
                      device_tensor(io.frame_max, io.out_frames, "float32"))

    def export(self, same_process: bool) -> bytes:
        """Where this shard's iterate buffers live (CUDA IPC handles, or raw
        pointers for contexts of the same process): sfseg_shard_export."""
        blob = C.create_string_buffer(N.SFSEG_SHARD_EXPORT_BYTES)
        N.check(self.lib.sfseg_shard_export(self.ctx.handle, int(same_process), blob))
        return blob.raw

    def set_peers(self, lo: Optional[bytes], hi: Optional[bytes]) -> None:
        """From now on sfseg_shard_step pushes the edge frames into the
        neighbours' halos itself (peer-memory stores): no send/recv."""
        bl = C.create_string_buffer(lo, len(lo)) if lo else None
        bh = C.create_string_buffer(hi, len(hi)) if hi else None
        N.check(self.lib.sfseg_shard_set_peers(self.ctx.handle, bl, bh))

    def before_exchange(self):
        import torch

        torch.cuda.current_stream().wait_stream(self.stream)

    def after_exchange(self):
        import torch

        self.stream.wait_stream(torch.cuda.current_stream())

    def finalize(self, params, it, frame_sum, frame_max) -> None:
        self._keep_gathered.append((frame_sum, frame_max))  # alive until the stream passes
        N.check(self.lib.sfseg_shard_finalize(
            self.ctx.handle, C.byref(params), it, C.c_void_p(frame_sum.data_ptr()),
            C.c_void_p(frame_max.data_ptr()), None, N.SFSEG_MEM_DEVICE))

    def norms(self, count):
        out = (C.c_double * count)()
        N.check(self.lib.sfseg_shard_norms(self.ctx.handle, count, out))
        self._keep_gathered.clear()
        return list(out)

    def download(self, frac, t0, t1, out=None):
        if out is not None:  # caller-provided (e.g. pinned) host arrays
            soft, mask = out
        else:
            soft = np.empty((t1 - t0, self.H, self.W), np.float32)
            mask = np.empty((t1 - t0, self.H, self.W), np.uint8)
        N.check(self.lib.sfseg_shard_download(self.ctx.handle, float(frac),
                                              C.c_void_p(soft.ctypes.data),
                                              C.c_void_p(mask.ctypes.data), N.SFSEG_MEM_HOST))
        return soft, mask

    def close(self):
        self.ctx.close()


def global_unit_range_guard(F_local: Sequence, group=None) -> list:
    """scale_channel_into_unit_range (engine.cpp:228-243) with the channel's
    global min/max (all-reduce). Returns the rank's channels: the caller's
    own arrays where the guard leaves the bits alone, rescaled COPIES where
    it applies (the reference rescales a copy too, engine.cpp:254-259; a
    channel that aliases the unary volume must not change it)."""
    import torch
    import torch.distributed as dist

    out = []
    for f in F_local:
        t = f if isinstance(f, torch.Tensor) else torch.from_numpy(np.asarray(f))
        lo = t.min().reshape(1).clone()
        hi = t.max().reshape(1).clone()
        if dist.is_initialized():
            dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
        lo_v, hi_v = float(lo.item()), float(hi.item())
        if lo_v >= 0.0 and hi_v <= 1.0:
            out.append(f)  # leave the bits alone
            continue
        t = t.clone()
        if hi_v > lo_v:
            span = torch.tensor(hi_v, dtype=torch.float32) - torch.tensor(lo_v, dtype=torch.float32)
            t.sub_(torch.tensor(lo_v, dtype=torch.float32, device=t.device)).div_(span.to(t.device))
        else:
            t.fill_(min(max(lo_v, 0.0), 1.0))
        out.append(t if isinstance(f, torch.Tensor) else t.numpy())
    return out


class ShardedSolver:
    """Runs Algorithm 1 over `world` ranks of a process group."""

    def __init__(self, backend, rank: int, world: int, group=None):
        self.b = backend
        self.rank, self.world, self.group = rank, world, group
        self._graphs = {}  # params -> "seen" | "eager" | (CUDAGraph, kept tensors)

    def load(self, T, H, W, S_local, F_local, x0_local, halo, allow_negative_affinity=False):
        """allow_negative_affinity must match the SfsegConfig the solve runs
        with (run() checks): off, the channels get the unit-range guard."""
        self.T, self.H, self.W, self.halo = T, H, W, halo
        self._graphs = {}  # captured loops point at the previous problem's buffers
        self.t0, self.t1 = shard_range(T, self.world, self.rank)
        self.allow_negative = bool(allow_negative_affinity)
        if not self.allow_negative:
            F_local = global_unit_range_guard(F_local, self.group)
        self.b.load(T, H, W, S_local, F_local, x0_local, self.t0, self.t1, halo)
        self.tmax = max(shard_range(T, self.world, r)[1] - shard_range(T, self.world, r)[0]
                        for r in range(self.world))
        self.p2p = False
        if self.world > 1 and hasattr(self.b, "export") and os.environ.get("SFSEG_P2P", "1") != "0":
            self._enable_p2p()

    def _enable_p2p(self):
        """Peer-memory halo exchange: every rank opens its neighbours' iterate
        buffers (CUDA IPC) and the step kernel stream pushes the edge frames
        into them. All-or-nothing across the group: if any rank cannot open
        its peers, every rank keeps the NCCL send/recv."""
        import torch
        import torch.distributed as dist

        blobs = [None] * self.world
        dist.all_gather_object(blobs, self.b.export(False), group=self.group)
        ok = 1
        try:
            self.b.set_peers(blobs[self.rank - 1] if self.rank > 0 else None,
                             blobs[self.rank + 1] if self.rank + 1 < self.world else None)
        except N.Error:
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32,
                            device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        self.p2p = bool(flag.item())
        if not self.p2p and ok:
            self.b.set_peers(None, None)  # some rank failed: everyone stays on NCCL

    def _exchange(self, io: StepIO):
        import torch.distributed as dist

        if self.world == 1 or self.p2p:  # p2p: the step already pushed the halos
            return
        ops = []
        if io.send_lo is not None:  # my first frames -> rank-1's upper halo
            ops.append(dist.P2POp(dist.isend, io.send_lo, self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, io.recv_lo, self.rank - 1, self.group))
        if io.send_hi is not None:
            ops.append(dist.P2POp(dist.isend, io.send_hi, self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, io.recv_hi, self.rank + 1, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def _gather(self, local, dtype):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return local
        pad = torch.zeros(self.tmax, dtype=dtype, device=local.device)
        pad[: local.numel()] = local
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad, group=self.group)
        parts = []
        for r in range(self.world):
            a, b = shard_range(self.T, self.world, r)
            parts.append(bufs[r][: b - a])
        return torch.cat(parts).contiguous()  # frame order

    def _gather_sums(self, frame_sum, frame_max):
        """Both per-frame vectors in ONE all-gather (frame max widened to fp64,
        exactly): one collective per iteration instead of two. Returns
        (sums fp64, max fp32) in frame order."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return frame_sum, frame_max
        n, tm = frame_sum.numel(), self.tmax
        dev = frame_sum.device
        packed = torch.zeros(2 * tm, dtype=torch.float64, device=dev)
        packed[:n] = frame_sum
        packed[tm:tm + n] = frame_max.to(torch.float64)
        if packed.is_cuda and dist.get_backend(self.group) != "nccl":
            packed = packed.cpu()  # gloo gathers host tensors (tests: ranks sharing one GPU)
        try:
            allp = torch.empty(self.world * 2 * tm, dtype=torch.float64, device=packed.device)
            dist.all_gather_into_tensor(allp, packed, group=self.group)
            bufs = list(allp.view(self.world, 2 * tm))
        except (RuntimeError, AttributeError, NotImplementedError):  # backends without it
            bufs = [torch.empty_like(packed) for _ in range(self.world)]
            dist.all_gather(bufs, packed, group=self.group)
        sums, maxs = [], []
        for r in range(self.world):
            a, b = shard_range(self.T, self.world, r)
            sums.append(bufs[r][: b - a])
            maxs.append(bufs[r][tm: tm + b - a])
        return (torch.cat(sums).to(dev).contiguous(),
                torch.cat(maxs).to(torch.float32).to(dev).contiguous())

    def _check_cfg(self, cfg):
        if bool(cfg.allow_negative_affinity) != self.allow_negative:
            from .engine import ParameterError

            raise ParameterError("allow_negative_affinity differs from the one the channels were "
                                 "loaded with (the unit-range guard is applied at load)")

    def _iterate(self, cfg, params) -> None:
        """Enqueues iterations 1..cfg.iterations: step (halos pushed to the
        peers by the kernel), one all-gather of the per-frame partials,
        finalize. No host synchronisation."""
        for it in range(1, cfg.iterations + 1):
            io = self.b.step(params, it)
            self.b.before_exchange()
            self._exchange(io)
            fs, fm = self._gather_sums(io.frame_sum, io.frame_max)
            self.b.after_exchange()
            self.b.finalize(params, it, fs, fm)

    def _graphable(self) -> bool:
        """The whole loop can be captured into one CUDA graph when nothing in
        it touches the host: a real CudaBackend, halos by peer memory (or one
        rank) and an NCCL (or no) all-gather. One rank: on by default
        (SFSEG_SHARD_GRAPH=0 turns it off). Several ranks: the capture then
        includes the NCCL all-gather, which could only be exercised on
        single-GPU boxes so far, so it is opt-in (SFSEG_SHARD_GRAPH=1)."""
        import torch.distributed as dist

        env = os.environ.get("SFSEG_SHARD_GRAPH", "")
        if env == "0" or not hasattr(self.b, "stream"):
            return False
        if self.world == 1:
            return True
        return (env == "1" and self.p2p and dist.is_initialized()
                and dist.get_backend(self.group) == "nccl")

    def _solve(self, cfg) -> None:
        """One solve. The first solve of a loaded problem with a configuration
        runs the loop eagerly (it also builds every lazily allocated buffer).
        The second captures the same loop — kernels, peer pushes, the NCCL
        all-gather — into a CUDA graph on the library's stream and replays it,
        as does every later one: no per-iteration host work at all. A load
        followed by a single solve (the end-to-end call) never pays a capture."""
        import torch

        self._check_cfg(cfg)
        params = cfg.to_params()
        self.b.cfg = cfg
        key = bytes(params)
        state = self._graphs.get(key) if self._graphable() else "eager"
        if state is None:
            self._graphs[key] = "seen"
            state = "eager"
        if state == "eager":
            self._iterate(cfg, params)
            return
        if state == "seen":
            self.b.ctx.synchronize()
            kept = len(self.b._keep_gathered)
            try:
                g = torch.cuda.CUDAGraph()
                # thread_local: another thread's CUDA calls (the NCCL watchdog's event
                # queries) must not invalidate the capture
                with torch.cuda.graph(g, stream=self.b.stream, capture_error_mode="thread_local"):
                    self._iterate(cfg, params)  # recorded, not run
            except Exception:
                # capture refused (a backend or library call that cannot be
                # captured): stay eager for good
                torch.cuda.synchronize()
                del self.b._keep_gathered[kept:]
                self._graphs[key] = "eager"
                self._iterate(cfg, params)
                return
            # the gathered tensors live in the graph's pool: keep them with it
            state = (g, self.b._keep_gathered[kept:])
            del self.b._keep_gathered[kept:]
            self._graphs[key] = state
        with torch.cuda.stream(self.b.stream):
            state[0].replay()

    def run(self, cfg, out=None) -> Tuple[np.ndarray, np.ndarray, List[float]]:
        """out: optional preallocated host (soft, mask) arrays for this rank's
        frames (the download lands there)."""
        self._solve(cfg)
        norms = self.b.norms(cfg.iterations)
        if out is not None:
            soft, mask = self.b.download(cfg.final_threshold, self.t0, self.t1, out=out)
        else:
            soft, mask = self.b.download(cfg.final_threshold, self.t0, self.t1)
        return soft, mask, norms

    def solve_only(self, cfg) -> None:
        """The iteration loop without the download (benchmark timing)."""
        self._solve(cfg)
