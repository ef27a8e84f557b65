"""Does processing queries in a locality order (grouped by nearest random
pivot) speed up k_search?  Results per query are order-independent."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = 1_000_000
x = torch.from_numpy(knng.gen_random_dataset(2 * n, 128, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
sg = knng.optimize_graph(g, base, 32)
sp = knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1)

def timed(q):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = knng.ann_search(q, sg, base, sp)
    torch.cuda.synchronize(); return time.perf_counter() - t, r

timed(qry)
t0, r0 = timed(qry)
for npiv in (256, 4096, 65536):
    torch.cuda.synchronize(); t = time.perf_counter()
    piv = qry[torch.randperm(n, device="cuda")[:npiv]]
    # nearest pivot via ||q||^2 - 2 q.p + ||p||^2 (ordering only: tf32 is fine)
    qn = (qry * qry).sum(1, keepdim=True)
    pn = (piv * piv).sum(1)
    best = torch.empty(n, dtype=torch.int64, device="cuda")
    for s in range(0, n, 262144):
        d = qn[s:s + 262144] - 2 * qry[s:s + 262144] @ piv.T + pn
        best[s:s + 262144] = d.argmin(1)
    perm = torch.argsort(best)
    qp = qry[perm].contiguous()
    torch.cuda.synchronize(); t_order = time.perf_counter() - t
    t1, r1 = timed(qp)
    same = bool(torch.equal(r1.ids, r0.ids[perm])) and bool(torch.equal(r1.dists, r0.dists[perm]))
    print(json.dumps(dict(pivots=npiv, base_s=round(t0, 4), ordered_s=round(t1, 4),
                          order_cost_s=round(t_order, 4), identical=same)), flush=True)
