"""Search in the Morton processing order (default for >= 65536 queries) vs the
given order (KNNG_SEARCH_ORDER=0): timings and bit-identity.  C4 regime:
clustered(16), N points, D dims (env), k_s 32, beam 128, 96 entries."""
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
res = {}
for order in ("0", "1", "0", "1"):
    os.environ["KNNG_SEARCH_ORDER"] = order
    ts = []
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = knng.ann_search(qry, sg, base, sp, diagnostics=True)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    if order in res:
        a = res[order]
    res[order] = r
    print(json.dumps(dict(order=order, n=n, d=d, secs=[round(t, 3) for t in ts],
                          qps=n / min(ts))), flush=True)
a, b = res["0"], res["1"]
same = all(bool(torch.equal(u, v)) for u, v in ((a.ids, b.ids), (a.dists.view(torch.int32), b.dists.view(torch.int32)),
                                                  (a.hops, b.hops), (a.scored, b.scored)))
print(json.dumps(dict(bit_identical=same)))
