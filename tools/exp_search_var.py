"""Run-to-run variance of the remote-refine search at the C4 P=2 shape: 5M
queries against a 5M x 96 clustered(16) graph, the searched set copied into a
fresh allocation before every repetition (as the flat phase pulls it).
KNNG_SEARCH_DYN=0/1: static query slots vs a fetch counter.  Env N, D, REPS."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "5000000"))
d = int(os.environ.get("D", "96"))
reps = int(os.environ.get("REPS", "6"))
x = torch.from_numpy(knng.gen_random_dataset(2 * n, d, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
sg = knng.optimize_graph(g, base, 32)
sp = knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1)
ref = None
for dyn in ("0", "1", "0", "1"):
    os.environ["KNNG_SEARCH_DYN"] = dyn
    ts = []
    for rep in range(reps):
        keep = []
        b2 = base.clone(); s2 = sg.clone()
        keep.append(torch.empty(int(1e8) * (rep % 3 + 1), dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize(); t = time.perf_counter()
        r = knng.ann_search(qry, s2, b2, sp)
        torch.cuda.synchronize(); ts.append(round(time.perf_counter() - t, 3))
        del b2, s2, keep
    same = True
    if ref is None:
        ref = r
    else:
        same = bool(torch.equal(r.ids, ref.ids)) and bool(torch.equal(r.dists.view(torch.int32), ref.dists.view(torch.int32)))
    print(json.dumps(dict(dyn=dyn, n=n, d=d, secs=ts, min=min(ts), max=max(ts), same=same)), flush=True)
