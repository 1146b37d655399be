"""Per-rep device time and memory of an HDP leg (variance diagnosis).
usage: python tools/c4_reps.py [leg] [reps]"""
import os
import subprocess
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS  # noqa: E402
from paper_1509_08197_b200.hdp_model import GmmModel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_hdp"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = bench.WORKLOADS[name]
spec, scenes = bench.scenes_for(name, 0)
L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
model = GmmModel.parse(bench.load_model_text())
pre = SIZE_CLASS_PRESETS[wl["size_class"]]
for r in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    E.run_hdp_batch(L, R, spec.d_max, model, levels=wl["levels"], delta0=pre["delta0"], beta=pre["beta"],
                    tree_kind=wl.get("tree", "mst"))
    e1.record()
    torch.cuda.synchronize()
    used = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()
    print(f"rep {r}: {e0.elapsed_time(e1):8.1f} ms  torch reserved {torch.cuda.memory_reserved() / 2**30:6.1f} GiB "
          f"max alloc {torch.cuda.max_memory_allocated() / 2**30:6.1f} GiB  nvidia-smi used {used}", flush=True)
