"""Per-CTA / per-warp timelines of the aggregation kernels (diagnostics build).

Build:  make -C paper_1509_08197_b200/csrc BUILD=/root/repo/.ab/bprof \
            OUT=/root/repo/.ab/libprof.so EXTRA=-DHDP_AGG_PROFILE
Run:    HDP_LIB=/root/repo/.ab/libprof.so python tools/agg_prof.py [cid]

Kinds: 1 up chunk (t1 desc, t2 staged, t3 computed), 2 down chunk (t1 desc,
t2 staged, t3 recurrence, t4 argmin), 3 seg up (t1 staged, t2 light gather,
t3 local pass + publish, t4 look-back), 4 seg down (t1 staged, t2 local pass,
t3 look-back).  Times in microseconds."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_08197_b200 import _lib, engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, make_batch  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = CONFIGS[cid]
sc = make_batch(cid, 1) if cid == 5 else make_batch(cid)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
lib = _lib.load()
fn = lib.hdp_debug_prof
fn.restype = C.c_longlong
fn.argtypes = [C.c_void_p, C.c_longlong]
for _ in range(2):
    E.run_baseline_batch(L, R, spec.d_max)
torch.cuda.synchronize()
fn(None, 0)
E.run_baseline_batch(L, R, spec.d_max)
torch.cuda.synchronize()
n = fn(None, 0)
E.run_baseline_batch(L, R, spec.d_max)
torch.cuda.synchronize()
buf = np.zeros((n, 8), dtype=np.uint64)
n = fn(buf.ctypes.data, n)
rec = buf[:n]
kind = (rec[:, 0] >> np.uint64(56)).astype(np.int64)
sm = ((rec[:, 0] >> np.uint64(40)) & np.uint64(0xffff)).astype(np.int64)
aux = (rec[:, 0] & np.uint64(0xffffffff)).astype(np.int64)
t = rec[:, 1:7].astype(np.float64)
t0 = t[:, 0].min()
tt = (t - t0) / 1e3
names = {1: ("up chunk", ["desc", "stage", "compute", "-", "tail"]),
         2: ("down chunk", ["desc", "stage", "recur", "argmin", "tail"]),
         3: ("seg up", ["stage", "light", "local", "lookback", "final"]),
         4: ("seg down", ["stage", "local", "lookback", "-", "final"])}
print(f"records {n}, span {tt[:, 5].max():.1f} us")
for k, (nm, st) in names.items():
    sel = kind == k
    if not sel.any():
        continue
    x = tt[sel]
    dur = x[:, 5] - x[:, 0]
    print(f"\n{nm}: {sel.sum()} items, total busy {dur.sum():.0f} item-us, mean {dur.mean():.2f} us, "
          f"p50 {np.median(dur):.2f}, p99 {np.percentile(dur, 99):.2f}")
    prev = x[:, 0]
    for j, s in enumerate(st):
        cur = x[:, j + 1]
        ok = cur > 0
        if s == "-" or not ok.any():
            continue
        d = cur[ok] - prev[ok] if j < 4 else x[ok, 5] - prev[ok]
        print(f"   {s:>9}: mean {d.mean():6.2f}  p50 {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f} us")
        prev = np.where(ok, cur, prev)
    if k in (3, 4):
        cnt = aux[sel] & 0xff
        segi = (aux[sel] >> 8) & 0x3fffff
        nxt = (aux[sel] >> 30) & 1
        solo = (segi == 0) & (nxt == 0)
        print(f"   nodes/seg mean {cnt.mean():.1f}; single-segment paths {solo.mean()*100:.0f}%")
# concurrency over time (5 us bins): chunk CTAs and segment warps resident
edges = np.arange(0, tt[:, 5].max() + 5, 5.0)
print("\n   t(us)  upC  dnC  upS  dnS   (mean resident items per SM)")
for lo in edges:
    hi = lo + 5
    row = []
    for k in (1, 2, 3, 4):
        x = tt[kind == k]
        ov = np.clip(np.minimum(x[:, 5], hi) - np.maximum(x[:, 0], lo), 0, None).sum() / 5.0 / 148
        row.append(ov)
    if sum(row) > 0:
        print(f"  {lo:6.0f} " + " ".join(f"{v:4.1f}" for v in row))
