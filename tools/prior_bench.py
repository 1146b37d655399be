"""Device time of the sampled-prior kernel per pyramid level (CUDA events),
C2 (8 pairs, 3 levels) and C4 (8 pairs, 5 levels).
usage: python tools/prior_bench.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, make_batch  # noqa: E402

for cid, levels in ((2, 3), (4, 5)):
    spec = CONFIGS[cid]
    sc = make_batch(cid, 8)
    L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
    R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
    lv = E.build_levels(L, R, spec.d_max, levels, 2, True)
    for lev in lv[:-1]:
        ms = []
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c, k = E.prior_counts(lev)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        print(f"C{cid} L{lev.level} {lev.h}x{lev.w} d{lev.d_max}: prior {min(ms[1:]):.3f} ms "
              f"kept {k.cpu().numpy()[:2].tolist()}", flush=True)
