"""Search-kernel experiment: C5-regime data, 1M-point graph, beam 128 / 96 entries."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "1000000"))
x = torch.from_numpy(knng.gen_random_dataset(2 * n, 128, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
torch.cuda.synchronize()
t = time.perf_counter(); sg = knng.optimize_graph(g, base, 32); torch.cuda.synchronize()
print("optimize_graph s", time.perf_counter() - t, flush=True)
for beam, ent in ((128, 96), (64, 16)):
    sp = knng.SearchParams(k_s=32, beam_width=beam, num_entry_points=ent, seed=1)
    ref = None
    for diag in (True, False, False):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = knng.ann_search(qry, sg, base, sp, diagnostics=diag)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        out = dict(beam=beam, entries=ent, exact=diag, secs=dt, qps=n / dt)
        if diag:
            ref = r
            h = r.hops.float(); s = r.scored.float()
            out.update(hops_mean=h.mean().item(), scored_mean=s.mean().item(),
                       gather_gbs=s.sum().item() * 512 / dt / 1e9)
        else:
            out["ids_equal"] = bool(torch.equal(r.ids, ref.ids))
            out["dists_equal"] = bool(torch.equal(r.dists.view(torch.int32), ref.dists.view(torch.int32)))
        print(json.dumps(out), flush=True)
