"""Multi-GPU drivers (one process per GPU, torch.distributed over NCCL).

Two ways the DPM path shards:

* z-slab sharding of ONE volume (config 5): rank r owns planes
  [z0_r, z1_r).  It projects its slab and takes the exact 2D moments of the
  slab images in GLOBAL coordinates (the z0 offset is folded into the image
  origins), so the per-rank 2D-moment limb accumulators simply add: one
  all-reduce SUM of B * P * n2d * 4 int64 limbs (2.7 KiB at order 6) -- the
  only exchange step -- then every rank runs the device epilogue.  Integer
  limb sums are exact and order-independent, so results are bit-identical for
  any world size.
* batch sharding of independent volumes (config 4): rank r owns a contiguous
  range of volumes; no data-path collective (an optional all-gather assembles
  the per-volume results).

Everything host-side here is backend-agnostic (gloo on CPU in the tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def slab_bounds(n_planes: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced z-range [z0, z1) of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_planes, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def batch_bounds(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced range of volume indices for ``rank``."""
    return slab_bounds(count, world, rank)


def allreduce_limbs(acc: torch.Tensor, group=None) -> torch.Tensor:
    """Sum 2D-moment limb accumulators across ranks in place (exact: int64
    two's-complement addition of uint64 limb sums, no overflow for < 2^31 ranks)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def moments_zslab(slab: torch.Tensor, order: int, z0: int, n_global: int, offset: int = 0, group=None,
                  stream=None):
    """Exact 3D moments of a volume z-slab-sharded across the group.

    ``slab`` is this rank's [N_r, M, L] voxels (global planes z0 .. z0+N_r-1)
    on its CUDA device.  Returns the engine.DeviceMoments of the WHOLE volume
    (identical on every rank)."""
    from . import engine

    engine.check_order(order)
    d = engine.make_desc(slab, offset, z0)
    engine.check_envelope(d.L, d.M, n_global, d.dtype, order)
    acc = engine.moments2d_partial(slab, order, offset=offset, z0=z0, stream=stream, n_global=n_global)
    allreduce_limbs(acc, group)
    return engine.derive(acc, order, stream=stream, kind=engine.acc_kind(slab, order, offset, z0))


def moments_batch_sharded(volumes: torch.Tensor, order: int, offset: int = 0, gather: bool = False, group=None):
    """Moments of this rank's shard of a batch ([B_r, N, M, L]); with ``gather``
    the fp64 results of all ranks are all-gathered (config 4, optional C2)."""
    from . import engine

    res = engine.moments(volumes, order, offset=offset)
    if gather and dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        world = dist.get_world_size(group)
        sizes = torch.tensor([res.f64.shape[0]], device=res.f64.device)
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        mx = int(max(s.item() for s in all_sizes))
        pad = torch.zeros((mx, res.f64.shape[1]), dtype=res.f64.dtype, device=res.f64.device)
        pad[: res.f64.shape[0]] = res.f64
        parts = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        return res, torch.cat([p[: int(s.item())] for p, s in zip(parts, all_sizes)])
    return res, None
