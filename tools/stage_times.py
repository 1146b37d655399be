"""Per-stage wall times of the batched pipelines (synchronised; diagnostics,
not a bench number)."""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.hdp_model import GmmModel  # noqa: E402
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--size-class", default="half")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--skip-hdp", action="store_true")
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--tree", default="mst")
    a = ap.parse_args()
    spec = CONFIGS[a.config]
    t = time.time()
    scenes = make_batch(a.config, a.batch)
    print(f"generated {len(scenes)} pairs in {time.time() - t:.1f}s", flush=True)
    Lh = np.stack([s.pair.left.data for s in scenes])
    Rh = np.stack([s.pair.right.data for s in scenes])
    L = torch.from_numpy(Lh).cuda()
    R = torch.from_numpy(Rh).cuda()
    model = GmmModel.parse(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                             "default.gmm")).read())
    d0, beta = (0.064, 0.6) if a.size_class == "half" else (0.004, 0.95)
    for rep in range(a.reps):
        if not a.skip_dense:
            torch.cuda.synchronize()
            t = time.perf_counter()
            out = E.run_baseline_batch(L, R, spec.d_max, timing=True)
            torch.cuda.synchronize()
            tot = time.perf_counter() - t
            print(f"dense rep{rep}: total {tot*1e3:.2f} ms  stages "
                  + " ".join(f"{k}={v*1e3:.2f}" for k, v in out.timings.items()), flush=True)
        if not a.skip_hdp:
            torch.cuda.synchronize()
            t = time.perf_counter()
            outs = E.run_hdp_batch(L, R, spec.d_max, model, levels=a.levels, delta0=d0, beta=beta,
                                   timing=True, tree_kind=a.tree)
            torch.cuda.synchronize()
            tot = time.perf_counter() - t
            print(f"hdp rep{rep}: total {tot*1e3:.2f} ms", flush=True)
            for o in outs:
                print(f"   L{o.level} {o.h}x{o.w} d{o.d_max}: trees {o.n_trees.tolist()[:3]} "
                      f"ratio {np.round(o.search_ratio[:3], 4).tolist()} rounds "
                      f"{o.extra.get('dr_rounds')} "
                      + " ".join(f"{k}={v*1e3:.2f}" for k, v in o.timings.items()), flush=True)


if __name__ == "__main__":
    main()
