"""Run a pipeline R times on one config (for ncu launch lists / profiles)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.hdp_model import GmmModel
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--mode", default="dense")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--levels", type=int, default=3)
a = ap.parse_args()
spec = CONFIGS[a.config]
sc = make_batch(a.config, a.batch)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
model = GmmModel.parse(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "default.gmm")).read())
for _ in range(a.reps):
    if a.mode == "dense":
        E.run_baseline_batch(L, R, spec.d_max)
    else:
        E.run_hdp_batch(L, R, spec.d_max, model, levels=a.levels)
torch.cuda.synchronize()
print("done")
