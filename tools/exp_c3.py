"""C3: 1M x 960-d fp32, k=32, single-GPU nn_descent (+ recall@10 on 2000 rows)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_27691_b200 as knng
n, d = int(os.environ.get("N", "1000000")), 960
x = torch.from_numpy(knng.gen_random_dataset(n, d, os.environ.get("DIST", "clustered"), 42,
                                             int(os.environ.get("CL", "1000")))).cuda()
p = knng.NnDescentParams(k=32, seed=1)
knng.nn_descent(x, p)
st = knng.NnDescentStats()
torch.cuda.synchronize(); t = time.perf_counter()
g = knng.nn_descent(x, p, stats=st)
torch.cuda.synchronize(); dt = time.perf_counter() - t
rows = np.sort(np.random.default_rng(12345).choice(n, 2000, replace=False)).astype(np.uint64)
gt, _ = knng.brute_force_knng(x, 10, rows=rows)
gt = gt.cpu().numpy(); ids = g.ids.cpu().numpy()[rows.astype(np.int64), :10]
rec = sum(len(np.intersect1d(ids[i], gt[i])) for i in range(len(rows))) / (len(rows) * 10.0)
print(json.dumps(dict(n=n, d=d, secs=dt, points_per_s=n / dt, recall10=rec, iterations=st.iterations,
                      stage_ms={k: round(v, 1) for k, v in st.stage_ms.items()})))
