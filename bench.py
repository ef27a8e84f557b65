#!/usr/bin/env python3
"""Benchmark: kNN-graph build points/sec on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 -- workload C2 (BASELINE configs[1]): 1M x 128-d Gaussian-mixture fp32
         (reference generator gen_random_dataset(1e6, 128, clustered, 42,
         clusters=1000)), k = 32; one step = one full lock-free NN-Descent
         local build (nn_descent, nndescent.cpp:225-259) with the dataset
         resident in HBM.
N > 1 -- C5-regime weak scaling: N x 1M x 128-d clustered(16), k = 32, M = 2,
         search beam 128 / 96 entry points (acceptance.cpp:76-88); one step =
         one build_distributed (refine.cpp:504-586) over N GPUs: partition ->
         local builds -> binary-tree refine -> grouped merge -> flat refine ->
         external ids, pulls over NVLink.  Launched under torchrun, rank 0
         drives the N GPUs (one host thread per GPU-rank); the other ranks
         join the timing barrier.

value  = points / device time (CUDA events on the library's stream), inputs
         resident in HBM (the dataset, 512 MB per GPU, is larger than L2, so
         no L2 flush is needed between steps).
e2e    = the same through the public API with pinned HOST buffers: H2D of the
         dataset and D2H of the N x k graph inside every timed step.
roofline: the dominant kernel (the join, k_join) -- algorithmic bytes per
         launch (feature rows staged once per point + id lists + slot
         atomics, counted on device) / its average CUDA-event duration, vs
         the measured HBM copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline: the reference's own CPU nn_descent (oracle/_ref, compiled from
         the unmodified sources) on a bounded 100K-point sample of the same
         workload, all host threads (rank 0, N = 1 only).
"""
import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kNN-graph build points/sec at recall@10 ≥ ref (1/2/4/8 B200); HBM GB/s"
PER_GPU = 1_000_000
DIMS = 128
K = 32


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("KNNG_BENCH_NO_SMI"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", ",".join(str(g) for g in range(self.gpus))],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout):
        t = time.time()
        while self.proc and not self.lines and time.time() - t < timeout:
            time.sleep(0.05)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    return ws, rank


def init_pg(ws):
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
        return dist
    return None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sample_rows(n, count=10000, seed=12345):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(count, n), replace=False)).astype(np.uint64)


def recall10(knng, x_dev, ids, rows):
    gt, _ = knng.brute_force_knng(x_dev, 10, rows=rows)
    gt = gt.cpu().numpy() if hasattr(gt, "cpu") else gt
    ids = ids.cpu().numpy() if hasattr(ids, "cpu") else ids
    sub = ids[rows.astype(np.int64), :10]
    hits = sum(len(np.intersect1d(sub[i], gt[i])) for i in range(len(rows)))
    return hits / (len(rows) * 10.0)


def reference_recall(name):
    p = os.path.join(ROOT, "tests", "golden", "reference_recall.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(name)
        if d:
            what = "nn_descent" if d["ranks"] == 1 else f"build_distributed P={d['ranks']}"
            return d["recall_at_10"], (f"reference {what} on the same data and seeds, "
                                       f"{d['sample_rows']} sampled rows ({name})")
    if name.startswith("c2"):
        return 0.981, "SURVEY.md §6 (reference nn_descent at 1M, 500 sampled rows)"
    return None, f"reference not yet measured for {name} (tests/golden/make_reference_recall.py)"


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref) -- cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------


def cpu_reference_step(x_sample, k, ranks=1):
    from oracle.bindings import Ref
    R = Ref()
    threads = R.hardware_concurrency()
    t = time.perf_counter()
    if ranks == 1:
        R.nn_descent(x_sample, k, seed=1, workers=0)
    else:
        cfg = R.refine_config(ranks, 2, k, nn_seed=1, search_seed=1, seed=1, beam_width=128,
                              num_entry_points=96)
        R.build_distributed(x_sample, cfg)
    secs = time.perf_counter() - t
    return secs, (threads if ranks == 1 else ranks)


def run_reference_arm(args, ws, rank):
    dist = init_pg(ws)
    if rank != 0:
        barrier(dist)
        return
    import paper_2605_27691_b200 as knng
    if args.gpus == 1:
        n_sample = 100_000
        x = knng.gen_random_dataset(PER_GPU, DIMS, "clustered", 42, 1000)[:n_sample].copy()
        ranks, workload = 1, "C2 sample: first 100K rows of the 1M x 128 clustered(1000) dataset"
    else:
        # the reference runs P single-threaded ranks (refine.cpp:156, 384):
        # ~40 s per 50K-point step at P=2, so the sample stays at 50K
        n_sample = 50_000
        x = knng.gen_random_dataset(n_sample, DIMS, "clustered", 42, 16)
        ranks, workload = args.gpus, (f"C4-regime sample: 50K x 128 clustered(16), "
                                      f"build_distributed P={args.gpus} M=2, beam 128 / 96")
    times = []
    cores = 1
    warm = min(args.warmup, 1)  # CPU path: warm-up only pages code/data in
    for i in range(warm + args.steps):
        secs, cores = cpu_reference_step(x, K, ranks)
        if i >= warm:
            times.append(secs)
    ms = 1000.0 * statistics.mean(times)
    value = n_sample / (ms / 1000.0)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": warm, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generator, seed 42)",
            "config": {"workload": workload, "n": n_sample, "dims": DIMS, "k": K},
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores,
                             "kind": "reference", "sample": workload},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    barrier(dist)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ramp", action="store_true", help="skip the clock ramp (profiling runs)")
    ap.add_argument("--per-gpu", type=int, default=PER_GPU)
    args = ap.parse_args()
    # a full collection of the interpreter's (torch-sized) heap between two
    # builds leaves the GPU idle inside the timed region: collect now, then
    # keep the collector off for the run
    gc.collect()
    gc.disable()
    ws, rank = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, ws, rank)
    dist = init_pg(ws)
    if ws > 1:
        return run_multi(args, ws, rank, dist)
    import torch

    import paper_2605_27691_b200 as knng
    knng.lib()
    ctx = knng.context()
    ngpu = args.gpus
    assert ctx.device_count >= ngpu, f"{ngpu} GPUs requested, {ctx.device_count} visible"
    stream = torch.cuda.ExternalStream(ctx.stream(0), device="cuda:0")
    per = args.per_gpu
    n = per * ngpu
    t0 = time.time()
    if ngpu == 1:
        x_host = knng.gen_random_dataset(n, DIMS, "clustered", 42, 1000)
        workload = "C2: 1M x 128-d clustered(1000) fp32, k=32, nn_descent local build"
        ref_name = "c2_1m_clustered1000_k32"
    else:
        # C4 regime (clustered(16), beam 128 / 96 entries) at the
        # C5 width, 1M points per GPU (weak scaling).  clustered(1000) would
        # leave the per-cluster kNN graphs disconnected, so random entry points
        # could not reach a query's cluster in the remote graphs.
        x_host = knng.gen_random_dataset(n, DIMS, "clustered", 42, 16)
        workload = (f"C4-regime weak scaling: {ngpu} x 1M x 128-d clustered(16) fp32, k=32, "
                    f"build_distributed P={ngpu} M=2 (partition, local NN-descent, tree "
                    f"refine, grouped merge, flat refine; beam 128 / 96 entries)")
        ref_name = f"dist_p{ngpu}_{ngpu}m_clustered16_k32"
    gen_s = time.time() - t0
    pinned = torch.empty(x_host.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = x_host
    x_np_pinned = pinned.numpy()
    x_dev = pinned.to("cuda:0")
    torch.cuda.synchronize()

    params = knng.NnDescentParams(k=K, seed=1)
    cfg = knng.RefineConfig(ranks=ngpu, groups=2, k=K, seed=1, nn=knng.NnDescentParams(k=K, seed=1),
                            search=knng.SearchParams(k_s=K, beam_width=128, num_entry_points=96,
                                                     seed=1))

    def step(x, stats=None):
        if ngpu == 1:
            return knng.nn_descent(x, params, stats=stats)
        return knng.build_distributed(x, cfg)

    stats_list = []
    # untimed clock ramp: the first builds on a fresh box run at low SM clocks
    # (measured 2199 / 919 / 842 / 307 ms before settling at ~270 ms), so keep
    # stepping until two consecutive steps agree within 5% (cap 12 steps / 60 s)
    ramp = []
    t_ramp = time.time()
    # (and the first builds of a process also vary while the driver and pool
    # settle): step until three consecutive steps agree within 2%
    while not args.no_ramp and len(ramp) < 20 and time.time() - t_ramp < 60:
        torch.cuda.synchronize()
        t = time.perf_counter()
        step(x_dev)
        torch.cuda.synchronize()
        ramp.append(time.perf_counter() - t)
        # at least 8 builds: a process's builds 4-7 were still seen to vary
        if len(ramp) >= 8 and max(ramp[-3:]) <= 1.02 * min(ramp[-3:]):
            break
    for _ in range(args.warmup):
        step(x_dev)
    barrier(dist)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    res = None
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(ngpu) as clocks:
        # nvidia-smi's NVML start-up can stall the GPU briefly: let the sampler
        # deliver its first sample (and one untimed step) before timing starts
        clocks.wait_first(10.0)
        step(x_dev)
        torch.cuda.synchronize()
        launches0 = knng.kernel_launches()
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            step_ev[0].record(stream)
        for i in range(args.steps):
            # per-stage statistics (CUDA events per stage) on the last step only
            st = knng.NnDescentStats() if i == args.steps - 1 else None
            res = step(x_dev, st if ngpu == 1 else None)
            if st is not None:
                stats_list.append(st)
            with torch.cuda.stream(stream):
                step_ev[i + 1].record(stream)
        with torch.cuda.stream(stream):
            ev[1].record(stream)
        torch.cuda.synchronize()
        launches = knng.kernel_launches() - launches0
    dev_ms = ev[0].elapsed_time(ev[1]) / args.steps
    step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps)]
    ms = max_over_ranks(dist, dev_ms)
    value = n / (ms / 1000.0)

    # e2e through the public API with pinned host buffers
    e2e_times = []
    for i in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = step(x_np_pinned)
        e2e_times.append(time.perf_counter() - t)
    e2e_ms = max_over_ranks(dist, 1000.0 * statistics.mean(e2e_times))
    graph = out.graph if ngpu > 1 else out
    h2d = n * DIMS * 4
    d2h = n * K * 8 + (n * K if ngpu == 1 else 0)  # ids + dists (+ u8 flags)

    # quality: recall@10 on 10K sampled rows vs exact brute force (GPU)
    g_ids = res.graph.ids if ngpu > 1 else res.ids
    rows = sample_rows(n)
    rec = recall10(knng, x_dev, g_ids, rows)
    ref_rec, ref_src = reference_recall(ref_name)

    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": ngpu,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generator gen_random_dataset, seed 42)",
            "config": {"workload": workload, "n": n, "dims": DIMS, "k": K,
                       "l2_flush": "inputs larger than L2 (dataset %.0f MB)" % (h2d / 1e6),
                       "parallelism": f"partition x{ngpu}" if ngpu > 1 else "single GPU"},
            "recall_at_10": rec, "reference_recall_at_10": ref_rec,
            "reference_recall_source": ref_src, "recall_rows": len(rows),
            "e2e": {"value": n / (e2e_ms / 1000.0), "unit": "points/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "clocks": clocks.summary(), "setup_gen_s": gen_s,
            "clock_ramp_ms": [round(1000 * t, 1) for t in ramp],
            "step_ms": [round(t, 2) for t in step_ms]}

    if ngpu == 1:
        st = stats_list[-1]
        peak, peak_src = load_peaks()
        # algorithmic bytes of the join: feature rows staged
        # once per point + the id lists read + 8 B slot atomics (RMW = 16 B)
        join_bytes = st.staged_rows * DIMS * 4 + st.staged_rows * 4 + st.offers * 16
        per_launch = join_bytes / max(1, st.join_launches)
        avg_ms = st.join_ms / max(1, st.join_launches)
        achieved = per_launch / (avg_ms / 1000.0) / 1e9
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "r01_join_traffic.json")
        if os.path.exists(tp):
            tj = json.load(open(tp))
            traffic, traffic_src = tj["traffic_bytes"], tj["capture"]
        # the join is bound by exact-order fp32 arithmetic (sub, mul, add per
        # dim, no FMA -- parity forbids reassociation/contraction), not HBM:
        # report that roofline too (non-FMA fp32 peak = SMs x 128 x clock)
        join_ops = st.pairs * DIMS * 3
        fp32_peak = 148 * 128 * (clocks.summary().get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
        line["roofline"] = {"kernel": "k_join (nndescent.cu)", "bound": "hbm",
                            "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": traffic,
                            "traffic_source": traffic_src, "peak_source": peak_src,
                            "compute": {"bound": "fp32 non-FMA (exact-order distances)",
                                        "achieved_tops": join_ops / (st.join_ms / 1000.0) / 1e12,
                                        "peak_tops": fp32_peak,
                                        "frac": join_ops / (st.join_ms / 1000.0) / 1e12 / fp32_peak},
                            "algorithmic_bytes_per_launch": per_launch,
                            "avg_launch_ms": avg_ms, "join_share_of_step": st.join_ms / ms,
                            "offer_kernel_ms_per_step": st.offer_ms,
                            "offers_per_point": st.offers / n,
                            "stage_ms_per_step": st.stage_ms, "build_device_ms": st.total_ms,
                            "offers_per_iter": st.offers_per_iter,
                            "pairs_per_iter": st.pairs_per_iter,
                            "sigma_per_point": st.pairs / n,
                            "staged_rows_per_point": st.staged_rows / n,
                            "iterations": st.iterations}
        line["gpu_launches"] = int(launches)
        if not args.no_cpu_baseline:
            try:
                xs = x_host[:100_000].copy()
                secs, cores = cpu_reference_step(xs, K, 1)
                line["cpu_baseline"] = {
                    "value": 100_000 / secs, "unit": "points/s", "cores": cores,
                    "kind": "reference",
                    "sample": "reference nn_descent(workers=all) on the first 100K rows of "
                              "the C2 dataset (k=32, same seeds)"}
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
    else:
        line["phases_s"] = {"partition": res.partition_s, "local": res.local_s,
                            "tree": res.tree_s, "merge": res.merge_s, "flat": res.flat_s,
                            "etc": res.etc_s}
        line["comm"] = {"gets": len(res.comm_log), "wire_bytes": sum(c.bytes for c in res.comm_log)}
        line["gpu_launches"] = int(launches)
        # local-build phase efficiency (north_star: >= 85% 1->N on this phase):
        # the same rank-0 share built alone on one GPU, in this run
        part = knng.partition_dataset(x_dev, ngpu, cfg.seed, gather=False)
        lo, hi = int(part.offsets[0]), int(part.offsets[1])
        idx = torch.from_numpy(part.to_external[lo:hi].astype(np.int64)).to("cuda:0")
        xs = x_dev.index_select(0, idx).contiguous()
        p0 = knng.NnDescentParams(k=K, seed=1)
        knng.nn_descent(xs, p0)
        t1 = []
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            knng.nn_descent(xs, p0)
            torch.cuda.synchronize()
            t1.append(time.perf_counter() - t)
        one = min(t1)
        line["local_phase"] = {"ms": 1000 * res.local_s, "single_gpu_same_share_ms": 1000 * one,
                               "efficiency": one / res.local_s if res.local_s else None,
                               "note": "rank-0 partition built alone on one GPU in the same run"}
    print(json.dumps(line), flush=True)
    barrier(dist)


def allreduce(dist, vals, op="max"):
    import torch
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def run_multi(args, ws, rank, dist):
    """N > 1 under torchrun: one process per GPU.  Every rank builds and
    refines its own share on its own GPU (knng_build_distributed_rank; CUDA
    IPC handles over the gloo group, one-sided NVLink pulls); each rank times
    its steps with CUDA events on its own stream, the max over ranks is the
    step time."""
    import torch

    import paper_2605_27691_b200 as knng
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    knng.lib()
    ctx = knng.context()
    assert ctx.device_count >= ws, f"{ws} ranks need {ws} visible GPUs"
    stream = torch.cuda.ExternalStream(ctx.stream(local), device=f"cuda:{local}")
    n = args.per_gpu * ws
    t0 = time.time()
    x_host = knng.gen_random_dataset(n, DIMS, "clustered", 42, 16)
    gen_s = time.time() - t0
    workload = (f"C4-regime weak scaling: {ws} x 1M x 128-d clustered(16) fp32, k=32, "
                f"build_distributed P={ws} M=2 (partition, local NN-descent, tree refine, "
                f"grouped merge, flat refine; beam 128 / 96 entries), one process per GPU")
    ref_name = f"dist_p{ws}_{ws}m_clustered16_k32"
    pinned = torch.empty(x_host.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = x_host
    x_np_pinned = pinned.numpy()
    x_dev = pinned.to(f"cuda:{local}")
    torch.cuda.synchronize()
    cfg = knng.RefineConfig(ranks=ws, groups=2, k=K, seed=1, nn=knng.NnDescentParams(k=K, seed=1),
                            search=knng.SearchParams(k_s=K, beam_width=128, num_entry_points=96,
                                                     seed=1))
    ag = knng.torch_allgather()

    def step(x):
        return knng.build_distributed_rank(x, cfg, rank, ws, ag, device=local)

    ramp = []
    t_ramp = time.time()
    while not args.no_ramp and len(ramp) < 20:
        torch.cuda.synchronize()
        t = time.perf_counter()
        step(x_dev)
        torch.cuda.synchronize()
        el, = allreduce(dist, [time.perf_counter() - t])
        ramp.append(el)
        stop = (len(ramp) >= 8 and max(ramp[-3:]) <= 1.02 * min(ramp[-3:])) or \
            time.time() - t_ramp > 60
        stop, = allreduce(dist, [1.0 if stop else 0.0])
        if stop:
            break
    for _ in range(args.warmup):
        step(x_dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    sampler = ClockSampler(ws) if rank == 0 else None
    if sampler:
        sampler.__enter__()
        sampler.wait_first(10.0)
    step(x_dev)
    barrier(dist)
    torch.cuda.synchronize()
    launches0 = knng.kernel_launches()
    with torch.cuda.stream(stream):
        ev[0].record(stream)
    res = None
    for i in range(args.steps):
        res = step(x_dev)
        with torch.cuda.stream(stream):
            ev[i + 1].record(stream)
    torch.cuda.synchronize()
    launches = knng.kernel_launches() - launches0
    barrier(dist)
    if sampler:
        sampler.__exit__()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    dev_ms = ev[0].elapsed_time(ev[args.steps]) / args.steps
    ms, = allreduce(dist, [dev_ms])
    step_ms_max = allreduce(dist, step_ms)
    launches_all, = allreduce(dist, [launches], op="sum")
    phases = allreduce(dist, [res.partition_s, res.local_s, res.tree_s, res.merge_s, res.flat_s,
                              res.etc_s])

    # e2e through the public API: pinned host dataset in, this rank's rows out
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        barrier(dist)
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = step(x_np_pinned)
        e2e.append(time.perf_counter() - t)
    e2e_ms, = allreduce(dist, [1000.0 * statistics.mean(e2e)])
    h2d = n * DIMS * 4             # each rank reads its block from pinned memory (zero-copy)
    d2h = n * K * 8 + n * 4        # all ranks' rows: ids + dists + external row ids
    del out

    # recall@10 on ~10K sampled rows (each rank samples its own rows)
    rows_ext = res.rows.cpu().numpy().astype(np.uint64)
    rng = np.random.default_rng(12345 + rank)
    pick = np.sort(rng.choice(len(rows_ext), size=min(len(rows_ext), 10000 // ws), replace=False))
    gt, _ = knng.brute_force_knng(x_dev, 10, rows=rows_ext[pick], device=local)
    gt = gt.cpu().numpy() if hasattr(gt, "cpu") else gt
    mine = res.graph.ids.cpu().numpy()[pick, :10]
    hits = sum(len(np.intersect1d(mine[i], gt[i])) for i in range(len(pick)))
    hits_all, cnt_all = allreduce(dist, [hits, len(pick)], op="sum")
    rec = hits_all / (cnt_all * 10.0)
    ref_rec, ref_src = reference_recall(ref_name)

    # local-build phase efficiency: rank 0's share built alone, ranks idle
    local_phase = None
    barrier(dist)
    if rank == 0:
        part = knng.partition_dataset(x_dev, ws, cfg.seed, gather=False, device=local)
        lo, hi = int(part.offsets[0]), int(part.offsets[1])
        idx = torch.from_numpy(part.to_external[lo:hi].astype(np.int64)).to(f"cuda:{local}")
        xs = x_dev.index_select(0, idx).contiguous()
        p0 = knng.NnDescentParams(k=K, seed=1)
        knng.nn_descent(xs, p0)
        t1 = []
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            knng.nn_descent(xs, p0)
            torch.cuda.synchronize()
            t1.append(time.perf_counter() - t)
        one = min(t1)
        local_phase = {"ms": 1000 * phases[1], "single_gpu_same_share_ms": 1000 * one,
                       "efficiency": one / phases[1] if phases[1] else None,
                       "note": "rank-0 share built alone on one GPU in the same run; local phase "
                               "= max over ranks"}
    barrier(dist)
    if rank == 0:
        line = {"metric": METRIC, "value": n / (ms / 1000.0), "unit": "points/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (reference generator gen_random_dataset, seed 42)",
                "config": {"workload": workload, "n": n, "dims": DIMS, "k": K,
                           "l2_flush": "inputs larger than L2 (dataset %.0f MB)" % (n * DIMS * 4 / 1e6),
                           "parallelism": f"partition x{ws}, one process per GPU"},
                "recall_at_10": rec, "reference_recall_at_10": ref_rec,
                "reference_recall_source": ref_src, "recall_rows": int(cnt_all),
                "e2e": {"value": n / (e2e_ms / 1000.0), "unit": "points/s", "ms_per_step": e2e_ms,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "clocks": sampler.summary() if sampler else None, "setup_gen_s": gen_s,
                "clock_ramp_ms": [round(1000 * t, 1) for t in ramp],
                "step_ms": [round(t, 2) for t in step_ms_max],
                "phases_s": dict(zip(("partition", "local", "tree", "merge", "flat", "etc"),
                                     phases)),
                "comm": {"gets": len(res.comm_log),
                         "wire_bytes": sum(c.bytes for c in res.comm_log)},
                "gpu_launches": int(launches_all), "local_phase": local_phase}
        print(json.dumps(line), flush=True)
    barrier(dist)


if __name__ == "__main__":
    main()
