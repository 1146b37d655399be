"""Multi-GPU plumbing for the two sharding modes of SURVEY.md §8(e).

* Batches of pairs (C2-C4): pairs are independent, so each rank takes a
  contiguous shard and there is no data-path collective (weak scaling).
* One large pair (C5): the disparity axis is split into slabs; every rank
  aggregates its slab over the (identical, deterministically rebuilt) MST and
  produces one u64 key per pixel, (order-preserving f32 cost << 32 | d).  The
  lexicographic minimum of the keys is the reference's first argmin over the
  full range (aggregation.py:320-326: strict '<' fold keeps the smaller d on
  ties), so one all-reduce(MIN) over the keys finishes the job.  NCCL reduces
  signed int64, so keys travel with their top bit flipped (a monotone map
  from u64 to i64 order).
"""

from __future__ import annotations

import numpy as np

SIGN = np.int64(-(2**63))


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous near-equal shard of range(n_items) for `rank`."""
    base, rem = divmod(n_items, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def slab(d_max: int, rank: int, world: int) -> tuple[int, int]:
    """Disparity slab [x0, x0 + nx) of rank over 0..d_max."""
    r = shard(d_max + 1, rank, world)
    return r.start, len(r)


def keys_to_signed(keys):
    """u64 keys stored in an int64 tensor/array -> order-equivalent int64."""
    return keys ^ SIGN if isinstance(keys, np.ndarray) else keys ^ int(SIGN)


def keys_from_signed(keys):
    return keys_to_signed(keys)


def pack_keys_host(cost: np.ndarray, disp: np.ndarray) -> np.ndarray:
    """Host restatement of the device key packing (aggregate.cu pack_key) for
    tests: u64 = ord(f32 cost) << 32 | d, returned as int64 bit patterns."""
    b = np.asarray(cost, np.float32).view(np.uint32).astype(np.uint64)
    neg = (b & np.uint64(0x80000000)) != 0
    o = np.where(neg, (~b) & np.uint64(0xFFFFFFFF), b | np.uint64(0x80000000))
    k = (o << np.uint64(32)) | np.asarray(disp, np.uint64)
    return k.view(np.int64)


def allreduce_min_keys(keys, group=None):
    """In-place MIN all-reduce of u64 keys held in an int64 torch tensor."""
    import torch.distributed as dist

    s = keys_to_signed(keys)
    dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
    keys.copy_(keys_from_signed(s))
    return keys


def run_slab_baseline(left_u8, right_u8, d_max: int, rank: int, world: int, group=None,
                      gamma: float = 0.1, cost=None):
    """Dense MST pipeline on one pair for this rank's disparity slab (the
    one-call pipeline, every rank rebuilding the same deterministic MST), then
    one all-reduce(MIN) over the packed keys in int64 order.  Returns
    (disparity int32, min_cost f32) device tensors of the full range."""
    from . import engine as E

    x0, nx = slab(d_max, rank, world)
    out = E.run_baseline_fused(left_u8, right_u8, d_max, gamma, cost or E.CostConsts(), x0=x0, nx=nx)
    if world == 1:
        return out.disparity, out.min_cost
    import torch.distributed as dist

    keys = E.keys_pack(out.disparity, out.min_cost, signed_order=True)
    dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    disp, mc = E.keys_unpack(keys, signed_order=True)
    return disp.view(out.disparity.shape), mc.view(out.min_cost.shape)
