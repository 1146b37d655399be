"""One sampled-prior launch (C4 level 1, 8 pairs) for ncu.
usage: python tools/prior_one.py [level]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, make_batch  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = CONFIGS[4]
sc = make_batch(4, 8)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
lv = E.build_levels(L, R, spec.d_max, 5, 2, True)
for rep in range(2):
    c, k = E.prior_counts(lv[level])
torch.cuda.synchronize()
print("ok", k.cpu().numpy()[:2])
