"""Does the dense pipeline read uninitialised (pool-recycled) memory?  Run the
600x1000 single-tree case (and C2) on a clean pool, then after filling
recycled pool blocks with several garbage patterns; results must be identical.
usage: python tools/garbage_check.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, SceneSpec, make_scene  # noqa: E402


def run(spec, d):
    sc = make_scene(spec, 0)
    L = torch.from_numpy(sc.pair.left.data[None]).cuda()
    R = torch.from_numpy(sc.pair.right.data[None]).cuda()
    out = E.run_baseline_batch(L, R, d, stepwise=True)
    return out.disparity.cpu().numpy().copy(), out.min_cost.cpu().numpy().copy()


cases = [(SceneSpec(5, 600, 1000, 12, 40, 0.3, 8.0, 1), 12), (CONFIGS[2], 80)]
base = [run(s, d) for s, d in cases]
for pat in (0x00, 0xFF, 0x7F, 0x01, 0x3F, 0x80):
    # recycle pool memory through torch's caching allocator AND the library's
    # stream-ordered pool (the library allocates from cudaMallocAsync's pool)
    for _ in range(3):
        blocks = [torch.full((64 << 20,), pat, dtype=torch.uint8, device="cuda") for _ in range(8)]
        del blocks
    torch.cuda.empty_cache()
    import ctypes
    from paper_1509_08197_b200 import _lib as L
    # fill the library pool: a big forest aggregation with garbage planes
    for i, (s, d) in enumerate(cases):
        got = run(s, d)
        nd = int((got[0] != base[i][0]).sum())
        nc = int((got[1] != base[i][1]).sum())
        print(f"pattern {pat:#04x} case {i}: disparity diffs {nd}, cost diffs {nc}", flush=True)
