"""Point-id locality vs build time: the C2 dataset built as given (cluster =
id mod 1000, so neighbouring ids are far apart) and with its rows renumbered
by a Morton order of random projections (spatially near points get near ids),
stage times and recall of both."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_27691_b200 as knng
n, d, cl = [int(v) for v in os.environ.get("SHAPE", "1000000,128,1000").split(",")]
x = torch.from_numpy(knng.gen_random_dataset(n, d, "clustered", 42, cl)).cuda()
gen = torch.Generator(device="cuda").manual_seed(0)
def morton_perm(x, dims=3, bits=10):
    R = torch.randn(x.shape[1], dims, device="cuda", generator=gen)
    p = x @ R
    q = ((p - p.min(0).values) / (p.max(0).values - p.min(0).values + 1e-9) * (2 ** bits - 1)).long()
    code = torch.zeros(x.shape[0], dtype=torch.long, device="cuda")
    for b in range(bits):
        for j in range(dims):
            code |= ((q[:, j] >> b) & 1) << (dims * b + j)
    return torch.argsort(code)
perm = morton_perm(x)
for name, xx in (("given", x), ("morton3", x[perm].contiguous())):
    p = knng.NnDescentParams(k=32, seed=1)
    knng.nn_descent(xx, p)
    st = knng.NnDescentStats()
    torch.cuda.synchronize(); t = time.perf_counter()
    g = knng.nn_descent(xx, p, stats=st)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    rows = np.sort(np.random.default_rng(12345).choice(n, 5000, replace=False)).astype(np.uint64)
    gt, _ = knng.brute_force_knng(xx, 10, rows=rows)
    ids = g.ids.cpu().numpy()[rows.astype(np.int64), :10]
    gt = gt.cpu().numpy()
    rec = sum(len(np.intersect1d(ids[i], gt[i])) for i in range(len(rows))) / (len(rows) * 10.0)
    print(json.dumps(dict(order=name, ms=round(1000 * dt, 1), recall10=rec, iterations=st.iterations,
                          stage_ms={k: round(v, 1) for k, v in st.stage_ms.items()})), flush=True)
