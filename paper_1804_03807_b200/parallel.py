"""Multi-GPU plumbing: one process per GPU, paths sharded into equal
contiguous ranges of the path index space, finite endpoints gathered to
rank 0 for classification.

The reference's only parallelism is the single-host work crew
(parallel.py:69-137); paths are independent, so the data path has no
collective.  The single exchange per stage is the endpoint gather (NCCL on
GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Equal contiguous shards; the first total % world ranks get one more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_strided(total: int, rank: int, world: int) -> tuple[int, int, int]:
    """Strided shard (first, stride, count): rank r owns path indices r, r + world,
    r + 2 world, ... -- a uniform sample of the index space, so ranks get equal
    work even where path cost varies along the index order (contiguous C5
    shards differ by 5 % in work, tools/probe_shards.py)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank, world, (int(total) - rank + world - 1) // world


@dataclass
class DistContext:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    initialized_here: bool = False

    @classmethod
    def from_env(cls, expect_world: int | None = None, backend: str | None = None) -> "DistContext":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        if expect_world is not None and world not in (1, expect_world):
            raise ValueError(f"WORLD_SIZE={world} but --gpus {expect_world}")
        ctx = cls(rank, world, local)
        if world > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                if backend is None:
                    import torch

                    backend = "nccl" if torch.cuda.is_available() else "gloo"
                if backend == "nccl":
                    import torch

                    torch.cuda.set_device(local)
                dist.init_process_group(backend=backend)
                ctx.initialized_here = True
        return ctx

    def shard(self, total: int) -> tuple[int, int]:
        return shard_range(total, self.rank, self.world)

    def shard_strided(self, total: int) -> tuple[int, int, int]:
        return shard_strided(total, self.rank, self.world)

    def _device(self):
        import torch
        import torch.distributed as dist

        if dist.get_backend() == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return float(v)
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(v)], dtype=torch.float64, device=self._device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v) -> int:
        if self.world == 1:
            return int(v)
        import torch
        import torch.distributed as dist

        t = torch.tensor([int(v)], dtype=torch.int64, device=self._device())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item())

    def close(self):
        if self.initialized_here:
            import torch.distributed as dist

            dist.destroy_process_group()


def compact_finite(x_end, status):
    """The succeeded endpoints of a shard in path order: on a CUDA tensor the
    library's own compaction kernels (nid_compact_finite, the K7 pre-pass of
    SURVEY §2.2), on a CPU tensor (gloo tests) a boolean mask."""
    import torch

    if not x_end.is_cuda:
        return x_end[(status == 0) | (status == 2)]
    import ctypes as C

    from . import _lib

    P = int(status.shape[0])
    if P == 0:
        return x_end[:0]
    L = _lib.lib()
    n = int(x_end.shape[1])
    x_end = x_end.contiguous()
    out = torch.empty_like(x_end)
    cnt = C.c_longlong(0)
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(L.nid_compact_finite(n, P, C.c_void_p(x_end.data_ptr()), C.c_void_p(status.data_ptr()), 0, 1,
                                    C.c_void_p(out.data_ptr()), None, P, C.byref(cnt), C.c_void_p(stream or None)), L)
    return out[: cnt.value]


def gather_finite(ctx: DistContext, x_end, status):
    """Compact this rank's succeeded endpoints (status converged/singular)
    and gather them to rank 0: all_gather of counts, then an all_gather of
    the padded blocks (NCCL has no variable-size gather).  Returns the
    concatenated [F, n, 2] tensor on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    pts = compact_finite(x_end, status)
    if ctx.world == 1:
        return pts
    cnt = torch.tensor([pts.shape[0]], dtype=torch.int64, device=pts.device)
    counts = [torch.zeros_like(cnt) for _ in range(ctx.world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(pts.shape[1:]), dtype=pts.dtype, device=pts.device)
    pad[: pts.shape[0]] = pts
    blocks = [torch.empty_like(pad) for _ in range(ctx.world)]
    dist.all_gather(blocks, pad)
    if ctx.rank != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(blocks, counts)], dim=0)


# ---------------------------------------------------------------- stage drivers
#
# The stage drivers (solve_top, cascade_step / run_cascade, membership_batch,
# refine_batch) shard through one active context: every rank runs the same
# host logic on the same inputs, tracks only its strided share of the stage's
# paths (the reference's fan-outs cascade.py:229-230, :311-312,
# filtering.py:114-115 split across processes), and one all_gather per stage
# hands every rank the whole stage's records in job order -- which is also the
# re-sharding for the next cascade level.  Classification that
# needs a global view (dedup / multiplicity, filtering.py:140-150) runs on
# rank 0 and its decision is broadcast (`on_root`).

_ACTIVE: DistContext | None = None


def activate(ctx: DistContext | None) -> None:
    """Make ctx the context the stage drivers shard through (None: single rank)."""
    global _ACTIVE
    _ACTIVE = ctx


def active() -> DistContext | None:
    return _ACTIVE if _ACTIVE is not None and _ACTIVE.world > 1 else None


def group_shard(ngroups: int, rank: int, world: int) -> np.ndarray:
    """Strided share of `ngroups` job groups: r, r + world, ..."""
    return np.arange(rank, int(ngroups), world, dtype=np.int64)


def allgather_rows(ctx: DistContext, local: np.ndarray, ngroups: int) -> np.ndarray:
    """Every rank holds the float64 rows of its strided share of `ngroups`
    groups (local: [own groups, F]); returns all rows [ngroups, F] in group
    order on every rank.  One padded all_gather (NCCL has no variable-count
    gather); rows travel as raw bits, so NaN payloads survive."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, dtype=np.float64)
    F = local.shape[1]
    per = (int(ngroups) + ctx.world - 1) // ctx.world  # the largest share
    dev = ctx._device()
    pad = torch.zeros((per, F), dtype=torch.float64, device=dev)
    if local.shape[0]:
        pad[: local.shape[0]] = torch.from_numpy(local).to(dev)
    blocks = [torch.empty_like(pad) for _ in range(ctx.world)]
    dist.all_gather(blocks, pad)
    out = np.empty((int(ngroups), F), np.float64)
    for r, b in enumerate(blocks):
        cnt = len(group_shard(ngroups, r, ctx.world))
        out[r::ctx.world] = b[:cnt].cpu().numpy()
    return out


def allreduce_sum(ctx: DistContext, values) -> list:
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=ctx._device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]


def on_root(fn, *args):
    """Run fn(*args) on rank 0 only and broadcast its (picklable) result, so a
    decision taken from a global view is the same on every rank.  Without an
    active multi-rank context this is just fn(*args)."""
    ctx = active()
    if ctx is None:
        return fn(*args)
    import torch.distributed as dist

    box = [fn(*args) if ctx.rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def merge_shards(parts: list[np.ndarray]) -> np.ndarray:
    return np.concatenate(parts, axis=0) if parts else np.zeros((0,))
