"""Benchmark of the HDP stereo hot path on B200 (contract: DESIGN.md §6).

Headline (default --config c5): BASELINE.json configs[4], the largest
configuration and the one north_star quotes the aggregation roofline on: one
synthetic 2880x1988 RGB pair, d_max 512, dense full-range MST pipeline
(run_baseline_pipeline: edges -> MST -> rooting/layout -> fused cost +
two-pass aggregation + WTA).  `value` = aggregated pixel-disparity hypotheses
per second (Gpd/s, 2.94 G hypotheses per pair).  Under torchrun (N > 1) the
pair is split into N disparity slabs, one per rank, whose packed (cost, d)
keys meet in one NCCL all-reduce(MIN) inside the timed step (strong scaling).

Legs in the same JSON line (`legs`), each with value / e2e / roofline /
cpu_baseline: C2 dense (8 pairs 463x370 d80), C2 HDP (3 levels, half preset),
C3 segment tree + HDP (32 pairs 695x555 d120, 4 levels), C4 segment tree + HDP
(64 pairs 1390x1110 d240, 5 levels, full preset).  Under torchrun every
rank runs its own pairs of the batched legs (weak scaling, no collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c5|c2|c2_hdp|c3_hdp|c4_hdp] [--legs c2,c2_hdp,c3_hdp,c4_hdp|none]
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

# workload definitions: BASELINE.json configs, SURVEY.md §8d presets
WORKLOADS = {
    "c5": dict(cid=5, kind="dense", batch=1,
               desc="C5: 1 pair 2880x1988 RGB d_max 512, dense MST full range"),
    "c2": dict(cid=2, kind="dense", batch=8,
               desc="C2: 8 pairs/GPU 463x370 RGB d_max 80, dense MST full range"),
    "c2_hdp": dict(cid=2, kind="hdp", batch=8, levels=3, size_class="half",
                   desc="C2: 8 pairs/GPU 463x370 RGB d_max 80, HDP 3 levels (half preset), MST"),
    "c3_hdp": dict(cid=3, kind="hdp", batch=32, levels=4, size_class="half", tree="st",
                   desc="C3: 32 pairs/GPU 695x555 RGB d_max 120, segment tree + HDP 4 levels (half preset)"),
    "c4_hdp": dict(cid=4, kind="hdp", batch=64, levels=5, size_class="full", tree="st",
                   desc="C4: 64 pairs/GPU 1390x1110 RGB d_max 240, segment tree + HDP 5 levels (full preset)"),
}
METRIC = "aggregated pixel-disparity hypotheses/s (Gpd/s) and stereo pairs/s, vs HBM roofline"
L2_NOTE = "256 MiB buffer written between timed steps (L2 is 126 MB)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--legs", default="c2,c2_hdp,c3_hdp,c4_hdp")
    ap.add_argument("--leg-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"os_cpu_count": os.cpu_count(), "lscpu_model": model}


def load_model_text():
    with open(os.path.join(REPO, "tests", "golden", "default.gmm")) as fh:
        return fh.read()


def scenes_for(name: str, rank: int, batch: int | None = None):
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    wl = WORKLOADS[name]
    spec = CONFIGS[wl["cid"]]
    b = wl["batch"] if batch is None else batch
    # C5 is one pair shared by all ranks (slabs); batched legs: own pairs per rank
    start = 0 if wl["cid"] == 5 else rank * b
    return spec, [make_scene(spec, start + i) for i in range(b)]


def config_dict(name: str, world: int, batch: int):
    wl = WORKLOADS[name]
    d = {"workload": wl["desc"], "config_id": wl["cid"], "pairs_per_gpu": batch,
         "pipeline": "dense" if wl["kind"] == "dense" else f"hdp levels={wl['levels']} {wl['size_class']}",
         "tree": wl.get("tree", "mst"),
         "l2": L2_NOTE}
    if wl["cid"] == 5:
        d["parallelism"] = f"disparity slabs x{world}, NCCL all-reduce(MIN) of packed keys"
    else:
        d["parallelism"] = f"pairs sharded, {world} rank(s)"
    return d


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


def committed_traffic(name: str):
    """DRAM bytes (read + write) of one launch of the leg's dominant kernel
    call from this round's committed ncu --set full capture
    (profiles/r02_traffic_<leg>.json, tools/ncu_traffic.py), or None."""
    path = os.path.join(REPO, "profiles", f"r02_traffic_{name}.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["bytes_per_call"])
    except (OSError, ValueError, KeyError):
        return None


def hbm_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------ CPU reference
def cpu_threads():
    return max(1, os.cpu_count() or 1)


def cpu_dense_pairs(L, R, d_max, n_pairs):
    """The reference algorithm (oracle C port of treestereo, float64) on the
    host cores: one pair per thread (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    O.lib()
    n = min(n_pairs, len(L))
    threads = min(n, cpu_threads())
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: O.run_baseline(L[i], R[i], d_max), range(n)))
    return time.perf_counter() - t, n, threads


def cpu_hdp_pairs(L, R, d_max, levels, size_class, n_pairs, tree="mst"):
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    O.lib()
    model = O.parse_gmm(load_model_text())
    n = min(n_pairs, len(L))
    threads = min(n, cpu_threads())
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda i: O.run_hdp(L[i], R[i], d_max, model, levels=levels,
                                                size_class=size_class, tree_kind=tree), range(n)))
    hyps = sum(sum(o.stored_entries for o in oo) for oo in outs)
    return time.perf_counter() - t, n, threads, hyps


def cpu_c5_sample(L, R, d_max):
    """Bounded sample of the C5 pair on the host: the full tree build
    (single-threaded, as in the reference) plus ONE round of the streamed
    aggregation -- every thread one disparity chunk of the size a full run
    uses (oracle.chunk_plan); the full pair's time is the tree plus that round
    times the rounds a full run needs.  Returns (t_pair, info)."""
    from oracle import oracle as O

    O.lib()
    threads = min(cpu_threads(), 64)
    I = np.asarray(L, np.float64)
    h, w = I.shape[:2]
    t0 = time.perf_counter()
    u, v, wt = O.build_edge_list(I)
    forest = O.build_hdpf(u, v, wt, h * w, O.full_masks(h * w, 0), 0, 0.0, O.mst_edge_order(wt))
    t1 = time.perf_counter()
    chunk = O.chunk_plan(h * w, d_max, threads)
    n_chunks = -(-(d_max + 1) // chunk)
    starts = [i * chunk for i in range(min(threads, n_chunks))]
    O.run_baseline_chunked(L, R, d_max, chunk=chunk, threads=threads, forest=forest, starts=starts)
    t2 = time.perf_counter()
    rounds = -(-n_chunks // threads)
    t_pair = (t1 - t0) + (t2 - t1) * rounds
    return t_pair, {"threads": threads, "lanes": len(starts) * chunk, "chunk": chunk, "rounds": rounds,
                    "tree_s": t1 - t0, "round_s": t2 - t1}


def cpu_leg(name, Lh, Rh, spec):
    """cpu_baseline object for a leg (rank 0, N=1)."""
    wl = WORKLOADS[name]
    npx = spec.height * spec.width
    if wl["cid"] == 5:
        t, info = cpu_c5_sample(Lh[0], Rh[0], spec.d_max)
        return {"value": npx * (spec.d_max + 1) / t / 1e9, "unit": "Gpd/s", "cores": info["threads"],
                "kind": "port", "pairs_per_s": 1.0 / t,
                "sample": (f"C5 pair: full tree build ({info['tree_s']:.1f} s, 1 thread) + one round of "
                           f"{info['threads']} disparity chunks of {info['chunk']} lanes "
                           f"({info['round_s']:.1f} s); a full pair needs {info['rounds']} rounds: "
                           f"{t:.1f} s per pair"), **host_info()}
    if wl["kind"] == "dense":
        dt, n, thr = cpu_dense_pairs(Lh, Rh, spec.d_max, len(Lh))
        return {"value": n * npx * (spec.d_max + 1) / dt / 1e9, "unit": "Gpd/s", "cores": thr,
                "kind": "port", "pairs_per_s": n / dt,
                "sample": f"{n} pairs of the leg's batch, one pair per thread", **host_info()}
    n_pairs = min(len(Lh), 16 if wl["cid"] == 4 else 8, cpu_threads())
    dt, n, thr, hyps = cpu_hdp_pairs(Lh, Rh, spec.d_max, wl["levels"], wl["size_class"], n_pairs,
                                     wl.get("tree", "mst"))
    return {"value": hyps / dt / 1e9, "unit": "Gpd/s", "cores": thr, "kind": "port",
            "pairs_per_s": n / dt,
            "sample": f"{n} of the leg's {len(Lh)} pairs, one pair per thread (HDP stored entries "
                      f"over all levels per second)", **host_info()}


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle C port; the
    Python reference cannot travel to the GPU box) on all host cores, rank 0."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    wl = WORKLOADS[name]
    spec, scenes = scenes_for(name, 0)
    Lh = np.stack([s.pair.left.data for s in scenes])
    Rh = np.stack([s.pair.right.data for s in scenes])
    npx = spec.height * spec.width
    times, sample = [], None
    for s in range(args.warmup + args.steps):
        if wl["cid"] == 5:
            t, info = cpu_c5_sample(Lh[0], Rh[0], spec.d_max)
            hyps, cores = npx * (spec.d_max + 1), info["threads"]
            sample = (f"per step: the C5 tree build + one round of {cores} chunks of {info['chunk']} lanes; "
                      f"a full pair = tree + {info['rounds']} rounds (extrapolated)")
        elif wl["kind"] == "dense":
            t, n, cores = cpu_dense_pairs(Lh, Rh, spec.d_max, len(Lh))
            hyps = n * npx * (spec.d_max + 1)
            sample = f"per step: {n} pairs, one per thread"
        else:
            n_pairs = min(len(Lh), cpu_threads())
            t, n, cores, hyps = cpu_hdp_pairs(Lh, Rh, spec.d_max, wl["levels"], wl["size_class"], n_pairs,
                                              wl.get("tree", "mst"))
            sample = f"per step: {n} pairs, one per thread"
        if s >= args.warmup:
            times.append((t, hyps))
    t = sum(x[0] for x in times) / len(times)
    value = statistics.mean(x[1] / x[0] for x in times) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpd/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if wl["cid"] == 5 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Voronoi scenes, SURVEY §8d)",
        "config": config_dict(name, args.gpus, len(Lh)),
        "cpu_baseline": {"value": value, "unit": "Gpd/s", "cores": cores, "kind": "port",
                         "sample": sample, **host_info()},
        "e2e": {"value": value, "unit": "Gpd/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def accuracy(scenes, disp_dev):
    """err >= 1 / >= 2 px of the final maps against the scenes' ground truth
    (non-occluded pixels), scored on the device (evaluation.error_rates_device)."""
    import torch

    from paper_1509_08197_b200.evaluation import error_rates_device

    gt = torch.from_numpy(np.stack([s.gt_left.values for s in scenes]).astype(np.int32)).cuda()
    occ = torch.from_numpy(np.stack([s.occlusion for s in scenes]).astype(np.uint8)).cuda()
    r = error_rates_device(disp_dev.contiguous(), gt, occ, (1, 2))
    return {"err_ge_1_pct": float(r[:, 0].mean()), "err_ge_2_pct": float(r[:, 1].mean()),
            "pixels": "non-occluded", "scored": "on the device (hdp_error_counts)"}


# ------------------------------------------------------------------ GPU arm
class Runner:
    def __init__(self, args):
        import torch

        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        from paper_1509_08197_b200 import _lib

        self.lib = _lib.load()
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        self.args = args
        self.cpu_todo = []

    def timed(self, fn, steps, warmup):
        """Device-timed steps (CUDA events on the current stream), L2 flushed
        and a barrier before each; returns per-step ms."""
        torch = self.torch
        ms = []
        for s in range(warmup + steps):
            self.flush.fill_(float(s))
            torch.cuda.synchronize()
            if self.dist:
                self.dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(s >= warmup)
            e1.record()
            torch.cuda.synchronize()
            if s >= warmup:
                ms.append(e0.elapsed_time(e1))
        return ms

    def reduce_max(self, x):
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    # ---- dense legs (C5 headline, C2)
    def dense(self, name, steps, warmup, with_cpu):
        torch = self.torch
        from paper_1509_08197_b200 import aggregation as A
        from paper_1509_08197_b200 import engine as E
        from paper_1509_08197_b200.distributed import run_slab_baseline, slab

        spec, scenes = scenes_for(name, self.rank)
        wl = WORKLOADS[name]
        Lh = np.stack([s.pair.left.data for s in scenes])
        Rh = np.stack([s.pair.right.data for s in scenes])
        B, H, W = Lh.shape[:3]
        d_max = spec.d_max
        slabs = wl["cid"] == 5 and self.world > 1
        x0, nx = slab(d_max, self.rank, self.world) if slabs else (0, d_max + 1)
        Ld = torch.from_numpy(Lh).cuda()
        Rd = torch.from_numpy(Rh).cuda()
        agg_ms: list = []

        def step(timed_step):
            if slabs:
                run_slab_baseline(Ld, Rd, d_max, self.rank, self.world)
            else:
                E.run_baseline_fused(Ld, Rd, d_max, agg_ms=agg_ms if timed_step else None)

        l0 = self.lib.hdp_launch_count()
        dev_ms = self.timed(step, steps, warmup)
        launches = (self.lib.hdp_launch_count() - l0) // (steps + warmup)
        # per-rank slab aggregation time (the roofline kernel) from a probe run
        if slabs:
            E.run_baseline_fused(Ld, Rd, d_max, x0=x0, nx=nx, agg_ms=agg_ms)

        pairs = [s.pair for s in scenes]

        def e2e(timed_step):
            # the reference-signature API: StereoPair in (host numpy), PipelineResult out
            if slabs:
                ld, rd, ready = E.stage_pairs([p.left.data for p in pairs], [p.right.data for p in pairs])
                torch.cuda.current_stream().wait_event(ready)
                dd, cc = run_slab_baseline(ld, rd, d_max, self.rank, self.world)
                dd.cpu().numpy(), cc.cpu().numpy()
            else:
                A.run_baseline_pipeline_batch(pairs)

        e2e_ms = self.timed(e2e, steps, 1)
        acc = None
        if not slabs:
            acc = accuracy(scenes, E.run_baseline_fused(Ld, Rd, d_max).disparity)
        hyps = B * H * W * (d_max + 1)
        n_lanes = nx
        t_dev = self.reduce_max(sum(dev_ms) / 1e3)
        t_e2e = self.reduce_max(sum(e2e_ms) / 1e3)
        units = hyps if slabs else self.world * hyps  # slabs: one pair shared by all ranks
        pairs_done = B if slabs else self.world * B
        out = {
            "value": units * steps / t_dev / 1e9, "unit": "Gpd/s",
            "ms_per_step": t_dev / steps * 1e3, "ms_steps": [round(x, 3) for x in dev_ms],
            "pairs_per_s": pairs_done * steps / t_dev,
            "scaling": "strong" if slabs else "weak",
            "config": config_dict(name, self.world, B),
            "e2e": {"value": units * steps / t_e2e / 1e9, "unit": "Gpd/s",
                    "h2d_bytes_per_step": int(Lh.nbytes + Rh.nbytes),
                    "d2h_bytes_per_step": int(B * H * W * (4 + 8)),  # int32 disparity + float64 min cost
                    "path": "aggregation.run_baseline_pipeline_batch (StereoPair list in, "
                            "PipelineResult list out)" if not slabs else
                            "pinned staging + distributed.run_slab_baseline + D2H"},
            "gpu_launches": int(launches),
            "accuracy": acc,
        }
        t_agg = statistics.mean(agg_ms) / 1e3
        entries = B * H * W * n_lanes
        algo = 8 * entries + 30 * B * H * W  # 8 B/hypothesis + 30 B/pixel
        peak, peak_kind = hbm_peak()
        out["roofline"] = {
            "bound": "hbm", "achieved": algo / t_agg / 1e9, "peak": peak, "unit": "GB/s",
            "frac": algo / t_agg / 1e9 / peak, "traffic": committed_traffic(name), "peak_kind": peak_kind,
            "kernel": "hdp_aggregate_wta (fused cost + up/down passes + WTA), one call per step"
                      + (" (this rank's slab)" if slabs else ""),
            "kernel_ms": t_agg * 1e3, "algorithmic_bytes": algo,
            "algorithmic_bytes_rule": "8 B per hypothesis (A-up written + read) + 30 B per pixel",
            "share_of_step": t_agg * 1e3 / (t_dev / steps * 1e3)}
        if with_cpu:
            self.cpu_todo.append((out, name, Lh, Rh, spec))
        return out

    # ---- HDP legs
    def hdp(self, name, steps, warmup, with_cpu):
        torch = self.torch
        from paper_1509_08197_b200 import aggregation as A
        from paper_1509_08197_b200 import engine as E
        from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS, AggregationParams
        from paper_1509_08197_b200.hdp_model import GmmModel

        wl = WORKLOADS[name]
        spec, scenes = scenes_for(name, self.rank)
        Lh = np.stack([s.pair.left.data for s in scenes])
        Rh = np.stack([s.pair.right.data for s in scenes])
        B = Lh.shape[0]
        model = GmmModel.parse(load_model_text())
        pre = SIZE_CLASS_PRESETS[wl["size_class"]]
        Ld = torch.from_numpy(Lh).cuda()
        Rd = torch.from_numpy(Rh).cuda()
        info = {}

        def step(timed_step):
            outs = E.run_hdp_batch(Ld, Rd, spec.d_max, model, levels=wl["levels"], delta0=pre["delta0"],
                                   beta=pre["beta"], tree_kind=wl.get("tree", "mst"))
            if "hyps" not in info:
                info["final"] = outs[-1].disparity
                info["hyps"] = int(sum(int(o.stored_entries.sum()) for o in outs))
                info["nodes"] = int(sum(B * o.h * o.w for o in outs))
                info["ratios"] = [float(np.mean(o.search_ratio)) for o in outs]
                info["rounds"] = [o.extra.get("dr_rounds") for o in outs]

        l0 = self.lib.hdp_launch_count()
        dev_ms = self.timed(step, steps, warmup)
        launches = (self.lib.hdp_launch_count() - l0) // (steps + warmup)
        pairs = [s.pair for s in scenes]
        params = AggregationParams(levels=wl["levels"], size_class=wl["size_class"])
        stage = {}

        def e2e(timed_step):
            res = A.run_hdp_pipeline_batch(pairs, model, params, tree_kind=wl.get("tree", "mst"))
            stage.update(res[0].metrics["seconds"])

        e2e_ms = self.timed(e2e, steps, 1)
        t_dev = self.reduce_max(sum(dev_ms) / 1e3)
        t_e2e = self.reduce_max(sum(e2e_ms) / 1e3)
        hyps = info["hyps"]
        algo = 8 * hyps + 30 * info["nodes"]
        peak, peak_kind = hbm_peak()
        npx = spec.height * spec.width
        out = {
            "value": self.world * hyps * steps / t_dev / 1e9, "unit": "Gpd/s",
            "ms_per_step": t_dev / steps * 1e3, "ms_steps": [round(x, 3) for x in dev_ms],
            "e2e_ms_steps": [round(x, 3) for x in e2e_ms],
            "pairs_per_s": self.world * B * steps / t_dev,
            "dense_equivalent_gpd_s": self.world * B * npx * (spec.d_max + 1) * steps / t_dev / 1e9,
            "scaling": "weak", "config": config_dict(name, self.world, B),
            "hyps_per_step": hyps, "levels": wl["levels"],
            "search_ratios_top_to_0": info["ratios"], "hdpf_rounds_top_to_0": info["rounds"],
            "e2e": {"value": self.world * hyps * steps / t_e2e / 1e9, "unit": "Gpd/s",
                    "pairs_per_s": self.world * B * steps / t_e2e,
                    "h2d_bytes_per_step": int(Lh.nbytes + Rh.nbytes),
                    "d2h_bytes_per_step": int(8 * info["nodes"]),  # int32 d + f32 cost, every level
                    "path": "aggregation.run_hdp_pipeline_batch (StereoPair list in, PipelineResult "
                            "list out, every level's maps)",
                    "stage_seconds_pair0": stage},
            "roofline": {"bound": "hbm", "achieved": algo / (t_dev / steps) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": algo / (t_dev / steps) / 1e9 / peak,
                         "traffic": None, "peak_kind": peak_kind,
                         "kernel": "whole HDP step (every level: prior, HDPF, tree build, aggregation); "
                                   "latency-bound, not bandwidth-bound",
                         "algorithmic_bytes": algo,
                         "algorithmic_bytes_rule": "sum over levels of 8 B x stored entries + 30 B x pixels"},
            "gpu_launches": int(launches),
            "accuracy": accuracy(scenes, info["final"]),
        }
        if with_cpu:
            self.cpu_todo.append((out, name, Lh, Rh, spec))
        return out

    def run_cpu_legs(self):
        """The CPU baselines run after every GPU leg has been timed, so that no
        host thread pool is busy (or winding down) beside a timed GPU step."""
        for out, name, Lh, Rh, spec in self.cpu_todo:
            out["cpu_baseline"] = cpu_leg(name, Lh, Rh, spec)
        self.cpu_todo = []

    def leg(self, name, steps, warmup, with_cpu):
        if WORKLOADS[name]["kind"] == "dense":
            return self.dense(name, steps, warmup, with_cpu)
        return self.hdp(name, steps, warmup, with_cpu)


def run_ours(args):
    r = Runner(args)
    with_cpu = r.world == 1 and not args.no_cpu_baseline
    with ClockSampler(r.local) as clk:
        head = r.leg(args.config, args.steps, args.warmup, with_cpu and r.rank == 0)
    clocks = clk.summary()
    legs = {}
    names = [x for x in args.legs.split(",") if x and x != "none" and x != args.config]
    for name in names:
        legs[name] = r.leg(name, args.leg_steps, max(3, min(args.warmup, 3)), with_cpu and r.rank == 0)
    if r.rank != 0:
        if r.dist:
            r.dist.destroy_process_group()
        return
    r.run_cpu_legs()
    line = {
        "metric": METRIC, "value": head["value"], "unit": "Gpd/s", "n_gpus": r.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Voronoi scenes of BASELINE.json's configs, SURVEY §8d)",
        "config": head["config"], "pairs_per_s": head["pairs_per_s"],
        "e2e": head["e2e"], "roofline": head["roofline"], "cpu_baseline": head.get("cpu_baseline"),
        "gpu_launches": head["gpu_launches"], "accuracy": head.get("accuracy"), "clocks": clocks, "legs": legs,
    }
    print(json.dumps(line), flush=True)
    if r.dist:
        r.dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
