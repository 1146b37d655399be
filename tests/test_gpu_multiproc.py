"""Two ranks (processes) reduce GPU-produced disparity-slab keys: the C5 split
of SURVEY.md §8(e) end to end on the device path.  Each rank runs the one-call
dense pipeline on its slab (hdp_dense_pipeline -> hdp_keys_pack, int64 order),
the keys meet in one all-reduce(MIN), and the unpacked maps must equal the
single-process full-range run.  Only one GPU is available to the tests, so both
ranks share cuda:0 and the reduction runs over gloo on host copies of the keys
(the ranks' kernels never wait on each other); bench.py runs the same step over
NCCL with one GPU per rank."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    return make_scene(SceneSpec(14, 150, 260, 96, 20, 0.4, 8.0, 1), 0)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08197_b200 import engine as E
        from paper_1509_08197_b200.distributed import slab

        torch.cuda.set_device(0)
        sc = _scene()
        L = torch.from_numpy(sc.pair.left.data[None]).cuda()
        R = torch.from_numpy(sc.pair.right.data[None]).cuda()
        x0, nx = slab(96, rank, world)
        out = E.run_baseline_fused(L, R, 96, x0=x0, nx=nx)
        keys = E.keys_pack(out.disparity, out.min_cost, signed_order=True).cpu()
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
        disp, mc = E.keys_unpack(keys.cuda(), signed_order=True)
        q.put((rank, disp.cpu().numpy(), mc.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_reduce_gpu_slab_keys():
    import torch
    import torch.multiprocessing as mp

    from paper_1509_08197_b200 import engine as E

    sc = _scene()
    full = E.run_baseline_batch(torch.from_numpy(sc.pair.left.data[None]).cuda(),
                                torch.from_numpy(sc.pair.right.data[None]).cuda(), 96)
    want_d = full.disparity.cpu().numpy().ravel()
    want_c = full.min_cost.cpu().numpy().ravel()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=500) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, d, c in res:
        np.testing.assert_array_equal(d, want_d)
        np.testing.assert_array_equal(c, want_c)
