"""C2-shaped cosine build (1M x 128 clustered(1000), k=32, metric=cosine):
device ms per build and recall@10 on 2000 sampled rows against the GPU brute
force (measurement only)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_27691_b200 as knng
xh = knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)
x = torch.from_numpy(xh).cuda()
p = knng.NnDescentParams(k=32, seed=1)
out = {}
for metric in ("l2", "cosine"):
    ms = []
    for _ in range(4):
        st = knng.NnDescentStats()
        g = knng.nn_descent(x, p, stats=st, metric=metric)
        ms.append(round(st.total_ms, 1))
    rows = np.random.default_rng(0).choice(len(xh), 2000, replace=False).astype(np.uint64)
    gi, _ = knng.brute_force_knng(xh, 10, rows=rows, metric=metric)
    ids = g.ids if isinstance(g.ids, np.ndarray) else g.ids.cpu().numpy()
    out[metric] = {"build_ms": ms, "iterations": st.iterations,
                   "recall_at_10": knng.recall_at_k(ids[rows.astype(np.int64)], gi, 10)}
print(json.dumps(out))
