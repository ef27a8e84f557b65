"""Sweep search smem shapes (KNNG_SEARCH_DCH / KNNG_SEARCH_VIS / KNNG_SEARCH_PIPE)
in one process over a C4/C5-regime graph (clustered(16), beam 128 / 96 entries);
checks bit-identity against exact mode.  N points, D dims (env)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "1000000"))
d = int(os.environ.get("D", "128"))
x = torch.from_numpy(knng.gen_random_dataset(2 * n, d, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
sg = knng.optimize_graph(g, base, 32)
sp = knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1)
ref = knng.ann_search(qry, sg, base, sp, diagnostics=True)
CFGS = [(32, 512, 0), (32, 256, 0), (16, 512, 0), (16, 256, 0), (32, 512, 1), (32, 256, 1),
        (16, 256, 1), (64, 512, 1)]
if os.environ.get("CFGS"):
    CFGS = [tuple(int(v) for v in c.split(",")) for c in os.environ["CFGS"].split(";")]
for cfg in CFGS:
    os.environ["KNNG_SEARCH_DCH"], os.environ["KNNG_SEARCH_VIS"] = str(cfg[0]), str(cfg[1])
    os.environ["KNNG_SEARCH_PIPE"] = str(cfg[2])
    ts = []
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = knng.ann_search(qry, sg, base, sp)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    ok = bool(torch.equal(r.ids, ref.ids)) and bool(torch.equal(r.dists.view(torch.int32), ref.dists.view(torch.int32)))
    sc = ref.scored.double().sum().item()
    gbs = (sc * d * 4 + ref.hops.double().sum().item() * 32 * 4) / min(ts) / 1e9
    print(json.dumps(dict(n=n, d=d, dch=cfg[0], vis=cfg[1], pipe=cfg[2],
                          secs=[round(t, 3) for t in ts], qps=n / min(ts), exact_equal=ok,
                          exact_scored_per_query=sc / n, algorithmic_gbs=gbs)), flush=True)
