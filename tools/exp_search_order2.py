"""Query order vs search throughput: the same queries searched in their given
(random) order and sorted by a 1-D / 2-D random projection, so that
concurrently running warps walk nearby parts of the graph (L2 reuse)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "2000000"))
d = int(os.environ.get("D", "96"))
x = torch.from_numpy(knng.gen_random_dataset(2 * n, d, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
sg = knng.optimize_graph(g, base, 32)
sp = knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1)
gen = torch.Generator(device="cuda").manual_seed(0)
R = torch.randn(d, 2, device="cuda", generator=gen)
proj = qry @ R
def morton(p):
    q = ((p - p.min(0).values) / (p.max(0).values - p.min(0).values + 1e-9) * 65535).long()
    code = torch.zeros(q.shape[0], dtype=torch.long, device="cuda")
    for b in range(16):
        code |= ((q[:, 0] >> b) & 1) << (2 * b) | ((q[:, 1] >> b) & 1) << (2 * b + 1)
    return code
orders = {"given": None, "proj1d": torch.argsort(proj[:, 0]), "morton2d": torch.argsort(morton(proj))}
for name, perm in orders.items():
    qq = qry if perm is None else qry[perm].contiguous()
    knng.ann_search(qq, sg, base, sp)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        knng.ann_search(qq, sg, base, sp)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print(json.dumps(dict(order=name, n=n, d=d, secs=[round(t, 3) for t in ts], qps=n / min(ts))), flush=True)
