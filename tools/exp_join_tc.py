"""A/B of the join kernels on one dataset: KNNG_JOIN=exact (exact-order CUDA-core
join, the default) vs KNNG_JOIN=tc (the tensor-core join).  Separate processes (the env var is read
at build time).  Prints build time, stages, recall@10 on 10K rows, and checks
stored distances against the exact recomputation.

  python tools/exp_join_tc.py [c2|c3|c1] [--one tc|exact]
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"c2": (1_000_000, 128, "clustered", 1000, 32), "c3": (1_000_000, 960, "clustered", 1000, 32),
          "c1": (100_000, 128, "uniform", 0, 10), "c4s": (2_000_000, 96, "clustered", 16, 32),
          "small": (20_000, 32, "clustered", 20, 16)}


def one(shape):
    import numpy as np
    import torch

    import paper_2605_27691_b200 as knng
    n, d, dist, cl, k = SHAPES[shape]
    x = torch.from_numpy(knng.gen_random_dataset(n, d, dist, 42, cl)).cuda()
    p = knng.NnDescentParams(k=k, seed=1)
    knng.nn_descent(x, p)
    times, st = [], None
    for _ in range(3):
        st = knng.NnDescentStats()
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = knng.nn_descent(x, p, stats=st)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    rows = np.sort(np.random.default_rng(12345).choice(n, min(n, 10000), replace=False)).astype(np.uint64)
    gt, _ = knng.brute_force_knng(x, 10, rows=rows)
    gt = gt.cpu().numpy()
    ids = g.ids.cpu().numpy()
    dd = g.dists.cpu().numpy()
    sub = ids[rows.astype(np.int64), :10]
    rec = sum(len(np.intersect1d(sub[i], gt[i])) for i in range(len(rows))) / (len(rows) * 10.0)
    # stored distances == exact recomputation (bit-exact), sampled
    rr = rows[:2000].astype(np.int64)
    ii = np.repeat(rr, k)
    jj = ids[rr].reshape(-1)
    ex = knng.row_distances(x, ii.astype(np.uint64), jj.astype(np.uint64))
    ex = ex.cpu().numpy() if hasattr(ex, "cpu") else ex
    bad = int(np.sum(ex.view(np.uint32) != dd[rr].reshape(-1).view(np.uint32)))
    srt = bool(np.all(np.diff(dd, axis=1) >= 0))
    selfref = int(np.sum(ids == np.arange(n)[:, None]))
    dup = int(sum(len(set(r)) != k for r in ids[rr]))
    print(json.dumps(dict(shape=shape, join=os.environ.get("KNNG_JOIN", "exact"), ms=[round(1000 * t, 1) for t in times],
                          recall10=rec, iterations=st.iterations, stage_ms={a: round(b, 1) for a, b in st.stage_ms.items()},
                          pairs=st.pairs, offers=st.offers, staged_rows=st.staged_rows,
                          bad_dists=bad, sorted=srt, self_refs=selfref, dup_rows=dup,
                          accepted=st.accepted_per_iter)), flush=True)


if __name__ == "__main__":
    shape = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if "--one" in sys.argv:
        one(shape)
    else:
        for mode in ("exact", "tc"):
            env = dict(os.environ, KNNG_JOIN=mode)
            subprocess.run([sys.executable, __file__, shape, "--one", mode], env=env, check=False)
