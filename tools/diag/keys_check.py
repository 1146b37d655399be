"""Every node must receive an argmin key from the aggregation kernels: with
HDP_KEYS_POISON=1 the keys buffer starts all-ones, so a node no kernel writes
comes out as disparity -1.  Counts such nodes for several shapes.
usage: HDP_KEYS_POISON=1 python tools/keys_check.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, SceneSpec, make_scene  # noqa: E402

for spec, d in [(SceneSpec(5, 600, 1000, 12, 40, 0.3, 8.0, 1), 12), (CONFIGS[2], 80), (CONFIGS[1], 16),
                (SceneSpec(7, 61, 83, 20, 10, 0.3, 8.0, 3), 20), (SceneSpec(5, 120, 720, 512, 24, 0.4, 8.0, 1), 512)]:
    sc = make_scene(spec, 0)
    L = torch.from_numpy(sc.pair.left.data[None]).cuda()
    R = torch.from_numpy(sc.pair.right.data[None]).cuda()
    for stepwise in (True, False):
        out = E.run_baseline_batch(L, R, d, stepwise=stepwise)
        dd = out.disparity.cpu().numpy()
        bad = np.argwhere(dd < 0)
        print(f"{spec.height}x{spec.width} d{d} stepwise={stepwise}: unwritten {len(bad)} {bad[:5].tolist()}",
              flush=True)
