"""Multi-rank host logic on CPU (gloo, world_size 2): pair sharding covers
the batch exactly once, and the disparity-slab split reduced with an
all-reduce(MIN) over packed (cost, d) keys reproduces the full-range first
argmin (the C5 plan).  Per-slab aggregated costs come from the
CPU oracle here; on the GPU the same keys come from hdp_aggregate_wta."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1509_08197_b200.distributed import (allreduce_min_keys, pack_keys_host, shard,
                                                       slab)
        from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

        spec = SceneSpec(8, 30, 48, 15, 5, 0.3, 8.0, 5)
        # (1) pair sharding: each rank processes its shard; gather the ids
        own = list(shard(spec.batch, rank, world))
        mine = torch.tensor(own + [-1] * (spec.batch - len(own)))
        allids = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allids, mine)
        ids = sorted(int(x) for t in allids for x in t.tolist() if x >= 0)
        # (2) disparity slabs of one pair
        sc = make_scene(spec, 0)
        d, best, _, vol, off = O._layer_wta(sc.pair.left.data.astype(np.float64),
                                            sc.pair.right.data.astype(np.float64), spec.d_max,
                                            O.build_forest_mst(sc.pair.left.data.astype(np.float64),
                                                               spec.d_max), 0.1, want_volume=True)
        full = vol.reshape(-1, spec.d_max + 1).astype(np.float32)
        x0, nx = slab(spec.d_max, rank, world)
        part = full[:, x0:x0 + nx]
        j = np.argmin(part, axis=1)
        keys = pack_keys_host(part[np.arange(part.shape[0]), j], x0 + j)
        kt = torch.from_numpy(keys.copy())
        allreduce_min_keys(kt)
        got_d = (kt.numpy().view(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        result_q.put((rank, ids, got_d, np.argmin(full, axis=1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_and_slab_min_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, got, want in res:
        assert ids == list(range(5))
        np.testing.assert_array_equal(got, want)
