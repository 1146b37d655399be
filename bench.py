"""Benchmark of the HDP stereo hot path on B200 (contract: DESIGN.md §6).

Workload (BASELINE.json configs[1] = C2): a batch of 8 synthetic pairs
463x370 RGB, d_max 80, per GPU.  One step = the dense full-range MST pipeline
(run_baseline_pipeline: edges -> MST -> rooting/layout -> fused cost +
two-pass aggregation + WTA) over the batch; `value` is aggregated
pixel-disparity hypotheses per second (Gpd/s) over all GPUs.  The 3-level
HDP pipeline on the same batch is timed the same way and reported under
"hdp".  Multi-GPU (torchrun): every rank owns its own 8 pairs (weak scaling,
no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_ID = 2
LEVELS = 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-hdp", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-pairs", type=int, default=8)
    return ap.parse_args()


def load_model():
    from paper_1509_08197_b200.hdp_model import GmmModel

    with open(os.path.join(REPO, "tests", "golden", "default.gmm")) as fh:
        return GmmModel.parse(fh.read())


def batch_for_rank(rank: int):
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    spec = CONFIGS[CONFIG_ID]
    scenes = [make_scene(spec, rank * spec.batch + i) for i in range(spec.batch)]
    L = np.stack([s.pair.left.data for s in scenes])
    R = np.stack([s.pair.right.data for s in scenes])
    return spec, L, R


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def agg_traffic():
    """DRAM bytes per aggregation call from the committed ncu --set full capture
    (profiles/r01_aggregate_traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_aggregate_traffic.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["bytes_per_call"])
    except (OSError, ValueError, KeyError):
        return None


def hbm_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def cpu_baseline_dense(L, R, d_max, pairs, hdp=False, model=None):
    """The reference algorithm on host cores: the CPU oracle (C restatement
    of treestereo, oracle/), one pair per thread (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    O.lib()
    n = min(pairs, L.shape[0])
    cores = min(n, os.cpu_count() or 1)

    def one(i):
        if hdp:
            return O.run_hdp(L[i], R[i], d_max, model, levels=LEVELS)
        return O.run_baseline(L[i], R[i], d_max)

    t = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(one, range(n)))
    return time.perf_counter() - t, n, cores


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O

    spec, L, R = batch_for_rank(0)
    hyps = L.shape[0] * spec.height * spec.width * (spec.d_max + 1)
    times = []
    for s in range(args.warmup + args.steps):
        dt, n, cores = cpu_baseline_dense(L, R, spec.d_max, L.shape[0])
        if s >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = hyps / t / 1e9
    model_layers = O.parse_gmm(open(os.path.join(REPO, "tests", "golden", "default.gmm")).read())
    hdp_t, hn, _ = cpu_baseline_dense(L, R, spec.d_max, L.shape[0], hdp=True, model=model_layers)
    line = {
        "impl": "reference", "metric": "aggregated pixel-disparity hypotheses/s (dense MST, C2)",
        "value": value, "unit": "Gpd/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: 8 pairs 463x370 RGB d_max 80, dense MST full range",
                   "batch": int(L.shape[0])},
        "cpu_baseline": {"value": value, "unit": "Gpd/s", "cores": cores, "kind": "port",
                         "sample": f"{L.shape[0]} C2 pairs per step, one pair per thread"},
        "e2e": {"value": value, "unit": "Gpd/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "hdp": {"pairs_per_s": hn / hdp_t, "ms_per_step": hdp_t * 1e3},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1509_08197_b200 import _lib
    from paper_1509_08197_b200 import engine as E

    lib = _lib.load()
    spec, Lh, Rh = batch_for_rank(rank)
    B, H, W = Lh.shape[:3]
    d_max = spec.d_max
    N = B * H * W
    hyps = N * (d_max + 1)
    Ld = torch.from_numpy(Lh).cuda()
    Rd = torch.from_numpy(Rh).cuda()
    Lp = torch.from_numpy(Lh).pin_memory()
    Rp = torch.from_numpy(Rh).pin_memory()
    model = load_model()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def timed(fn, steps, warmup):
        ms = []
        for s in range(warmup + steps):
            flush.fill_(float(s))  # evict L2 (126 MB) between steps, untimed
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(s >= warmup)
            e1.record()
            torch.cuda.synchronize()
            if s >= warmup:
                ms.append(e0.elapsed_time(e1))
        return ms


    agg_ms: list = []

    def dense(timed_step):
        # one library call per step (hdp_dense_pipeline: sub-batches on their own
        # streams); each sub-batch's aggregation call is timed with device events
        E.run_baseline_fused(Ld, Rd, d_max, agg_ms=agg_ms if timed_step else None)

    # warm-up + timed dense steps with clocks sampled during the timed region
    with ClockSampler(local) as clk:
        l0 = lib.hdp_launch_count()
        dense_ms = timed(dense, args.steps, args.warmup)
        launches = (lib.hdp_launch_count() - l0) // (args.steps + args.warmup)
    n_sub = max(1, min(E.DENSE_SUB_BATCHES, B))
    entries, nodes = hyps / n_sub, N / n_sub  # per aggregation call (one sub-batch)

    # results land in pinned host buffers (allocated once, like the inputs)
    Od = torch.empty((B, H, W), dtype=torch.int32).pin_memory()
    Oc = torch.empty((B, H, W), dtype=torch.float32).pin_memory()

    def e2e(timed_step):
        E.run_baseline_host(Lp, Rp, d_max, out=(Od, Oc))

    e2e_ms = timed(e2e, args.steps, 1)

    hdp = None
    if not args.no_hdp:
        hdp_info = {}

        def hdp_step(timed_step):
            outs = E.run_hdp_batch(Ld, Rd, d_max, model, levels=LEVELS)
            hdp_info["hyps"] = int(sum(int(o.stored_entries.sum()) for o in outs))
            hdp_info["ratios"] = [float(np.mean(o.search_ratio)) for o in outs]
            hdp_info["rounds"] = [o.extra.get("dr_rounds") for o in outs]

        hdp_ms = timed(hdp_step, args.steps, max(1, args.warmup))
        hdp = {"ms_per_step": statistics.mean(hdp_ms), "hyps_per_step": hdp_info["hyps"],
               "levels": LEVELS, "search_ratios_top_to_0": hdp_info["ratios"],
               "hdpf_rounds_top_to_0": hdp_info["rounds"]}

    def reduce_max(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_dense = reduce_max(sum(dense_ms) / 1e3)  # seconds for K steps, max over ranks
    t_e2e = reduce_max(sum(e2e_ms) / 1e3)
    if hdp:
        t_hdp = reduce_max(sum(hdp_ms) / 1e3)
        hdp["pairs_per_s"] = world * B * args.steps / t_hdp
        hdp["gpd_per_s"] = world * hdp["hyps_per_step"] * args.steps / t_hdp / 1e9
        hdp["ms_per_step"] = t_hdp / args.steps * 1e3
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    value = world * hyps * args.steps / t_dense / 1e9
    peak, peak_kind = hbm_peak()
    t_agg = statistics.mean(agg_ms) / 1e3
    algo_bytes = 8 * entries + 30 * nodes  # 8 B/hypothesis + 30 B/pixel
    achieved = algo_bytes / t_agg / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": agg_traffic(), "peak_kind": peak_kind,
            "kernel": ("hdp_aggregate_wta (fused cost + up/down passes + WTA), one call per step"
                       if n_sub == 1 else
                       f"hdp_aggregate_wta (fused cost + up/down passes + WTA), one call per sub-batch of "
                       f"{B // n_sub} pairs, timed while the other sub-batches run beside it"),
            "kernel_ms": t_agg * 1e3, "algorithmic_bytes": algo_bytes}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        dt, n, cores = cpu_baseline_dense(Lh, Rh, d_max, args.cpu_pairs)
        cpu = {"value": n * H * W * (d_max + 1) / dt / 1e9, "unit": "Gpd/s", "cores": cores,
               "kind": "port", "sample": f"{n} C2 pairs (dense MST), one pair per thread"}
    line = {
        "metric": "aggregated pixel-disparity hypotheses/s (dense MST, C2)",
        "value": value, "unit": "Gpd/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_dense / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Voronoi scenes, SURVEY §8d)",
        "config": {"workload": "C2: 8 pairs/GPU 463x370 RGB d_max 80, dense MST full range",
                   "batch_per_gpu": B, "pairs_per_s": world * B * args.steps / t_dense,
                   "l2": "256 MiB buffer written between timed steps",
                   "parallelism": f"pairs sharded, {world} rank(s)"},
        "e2e": {"value": world * hyps * args.steps / t_e2e / 1e9, "unit": "Gpd/s",
                "h2d_bytes_per_step": int(Lh.nbytes + Rh.nbytes),
                "d2h_bytes_per_step": int(N * 4 * 2)},
        "roofline": roof,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "hdp": hdp,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
