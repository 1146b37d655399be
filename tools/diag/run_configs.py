"""Run every BASELINE.json configuration once on the GPU (timing + basic
sanity vs ground truth).  Diagnostics for DESIGN.md, not the bench.

usage: python tools/run_configs.py [--configs 1,2,3,4,5] [--c4-batch 8] [--c3-batch 32]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.hdp_model import GmmModel  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, make_scene  # noqa: E402

# (pipeline, levels, size class) per config (ST absent -> mst)
PLAN = {1: ("hdp", 2, "half"), 2: ("both", 3, "half"), 3: ("hdp", 4, "half"),
        4: ("hdp", 5, "full"), 5: ("dense", 0, None)}


def err_rate(disp, gt, occ):
    ok = ~occ
    return 100.0 * float((np.abs(disp - gt)[ok] >= 2).mean())


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--c4-batch", type=int, default=8)
    ap.add_argument("--c3-batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    model = GmmModel.parse(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                             "default.gmm")).read())
    for cid in [int(x) for x in a.configs.split(",")]:
        spec = CONFIGS[cid]
        batch = {3: a.c3_batch, 4: a.c4_batch}.get(cid, spec.batch)
        t = time.time()
        scenes = [make_scene(spec, i) for i in range(batch)]
        gen = time.time() - t
        L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
        R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
        gt = np.stack([s.gt_left.values for s in scenes])
        occ = np.stack([s.occlusion for s in scenes])
        kind, levels, size = PLAN[cid]
        n = batch * spec.height * spec.width
        print(f"C{cid}: {batch} x {spec.height}x{spec.width} d{spec.d_max} (gen {gen:.1f}s)", flush=True)
        if kind in ("dense", "both"):
            for r in range(a.reps):
                out, dt = timed(lambda: E.run_baseline_batch(L, R, spec.d_max))
            hyps = n * (spec.d_max + 1)
            e = err_rate(out.disparity.cpu().numpy(), gt, occ)
            print(f"   dense MST: {dt*1e3:9.2f} ms  {hyps/dt/1e9:7.2f} Gpd/s  {batch/dt:8.1f} pairs/s"
                  f"  err>=2 {e:5.2f}%", flush=True)
        if kind in ("hdp", "both"):
            d0, beta = (0.064, 0.6) if size == "half" else (0.004, 0.95)
            for r in range(a.reps):
                outs, dt = timed(lambda: E.run_hdp_batch(L, R, spec.d_max, model, levels=levels,
                                                         delta0=d0, beta=beta))
            hyps = sum(int(o.stored_entries.sum()) for o in outs)
            e = err_rate(outs[-1].disparity.cpu().numpy(), gt, occ)
            ratios = [round(float(np.mean(o.search_ratio)), 4) for o in outs]
            rounds = [o.extra.get("dr_rounds") for o in outs]
            print(f"   HDP L{levels} ({size}): {dt*1e3:9.2f} ms  {batch/dt:8.1f} pairs/s  "
                  f"{hyps/dt/1e9:6.3f} Gpd/s  err>=2 {e:5.2f}%  R_l {ratios}  rounds {rounds}",
                  flush=True)
        del L, R
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
