"""A/B check of Boruvka with and without edge contraction on random graphs."""
import os, sys, subprocess, json
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1509_08197_b200 import engine as E
rng = np.random.default_rng(0)
out = []
for t in range(200):
    n = int(rng.integers(2, 80)); m = int(rng.integers(1, 3 * n))
    u = rng.integers(0, n, m); v = rng.integers(0, n, m)
    keep = u != v; u, v = u[keep], v[keep]
    key = (rng.permutation(len(u)).astype(np.int64) << 32) | np.arange(len(u), dtype=np.int64)
    eu = torch.tensor(u, dtype=torch.int32, device="cuda"); ev = torch.tensor(v, dtype=torch.int32, device="cuda")
    k = torch.tensor(key, dtype=torch.int64, device="cuda")
    it, comp, r = E.mst(n, eu, ev, k)
    out.append([int(it.sum()), r, comp.cpu().tolist()])
print(__import__("json").dumps(out))
'''
a = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, "HDP_MST_FULL": "0"})
b = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env={**os.environ, "HDP_MST_FULL": "1"})
A, B = json.loads(a.stdout), json.loads(b.stdout)
bad = [i for i in range(len(A)) if A[i][0] != B[i][0] or A[i][2] != B[i][2]]
print("mismatches", len(bad), "of", len(A), [(i, A[i][0], B[i][0], A[i][1], B[i][1]) for i in bad[:5]])
