"""Single-GPU nn_descent at the north_star shapes that the bench does not run.

  python tools/run_shapes.py c3|c4_1gpu|c5_rank [--steps S]

c3       1M x 960 clustered(1000), k=32         (BASELINE configs[2])
c4_1gpu  10M x 96 clustered(16), k=32            (C4's whole dataset on one GPU: the
                                                  1-GPU side of the local-build efficiency)
c5_rank  12.5M x 128 clustered(16), k=32         (C5's per-rank share at P=8)

Prints one JSON line: device time per build (CUDA events on the library stream),
peak device memory in use during the build (NVML, sampled every 20 ms), recall@10
on 2,000 sampled rows vs the GPU brute force, per-stage times.
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_27691_b200 as knng  # noqa: E402

SHAPES = {
    "c3": (1_000_000, 960, 1000),
    "c4_1gpu": (10_000_000, 96, 16),
    "c5_rank": (12_500_000, 128, 16),
}


class MemPeak:
    def __init__(self, dev=0):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        self.peak = 0
        self.run = True

    def used(self):
        return self.nv.nvmlDeviceGetMemoryInfo(self.h).used

    def loop(self):
        while self.run:
            self.peak = max(self.peak, self.used())
            time.sleep(0.02)

    def __enter__(self):
        self.base = self.used()
        self.t = threading.Thread(target=self.loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.run = False
        self.t.join()


def main():
    name = sys.argv[1]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--steps" else 2
    n, d, cl = SHAPES[name]
    t0 = time.time()
    xh = knng.gen_random_dataset(n, d, "clustered", 42, cl)
    gen_s = time.time() - t0
    x = torch.from_numpy(xh).cuda()
    del xh
    ctx = knng.context()
    stream = torch.cuda.ExternalStream(ctx.stream(0), device="cuda:0")
    p = knng.NnDescentParams(k=32, seed=1)
    with MemPeak() as mp:
        base = mp.base
        knng.nn_descent(x, p)  # warm-up (workspace sizing)
        torch.cuda.synchronize()
        times = []
        st = None
        for _ in range(steps):
            st = knng.NnDescentStats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            g = knng.nn_descent(x, p, stats=st)
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    rows = np.sort(np.random.default_rng(12345).choice(n, 2000, replace=False)).astype(np.uint64)
    gt, _ = knng.brute_force_knng(x, 10, rows=rows)
    gt = gt.cpu().numpy()
    ids = g.ids.cpu().numpy()[rows.astype(np.int64), :10] if hasattr(g.ids, "cpu") else \
        g.ids[rows.astype(np.int64), :10]
    rec = sum(len(np.intersect1d(ids[i], gt[i])) for i in range(len(rows))) / (len(rows) * 10.0)
    ms = min(times)
    print(json.dumps(dict(
        shape=name, n=n, dims=d, clusters=cl, k=32, build_ms=[round(t, 1) for t in times],
        points_per_s=n / (ms / 1000.0), recall_at_10=rec, recall_rows=len(rows),
        iterations=st.iterations, peak_mem_gb=round(mp.peak / 1e9, 2),
        peak_over_baseline_gb=round((mp.peak - base) / 1e9, 2),
        dataset_gb=round(n * d * 4 / 1e9, 2), gen_s=round(gen_s, 1),
        stage_ms={k: round(v, 1) for k, v in st.stage_ms.items()},
        gpu=torch.cuda.get_device_name(0))), flush=True)


if __name__ == "__main__":
    main()
