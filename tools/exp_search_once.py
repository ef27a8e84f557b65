"""C4-shape remote-refine searches (cache mode, the refine path): N base
points and N queries (clustered(16), D dims), k_s 32, beam 128, 96 entries;
REPS timed repetitions (0: one untimed search, for profilers).  Env N, D, REPS."""
import os, sys, time, json, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "2000000"))
d = int(os.environ.get("D", "96"))
reps = int(os.environ.get("REPS", "3"))
x = torch.from_numpy(knng.gen_random_dataset(2 * n, d, "clustered", 42, 16)).cuda()
base, qry = x[:n].contiguous(), x[n:].contiguous()
g = knng.nn_descent(base, knng.NnDescentParams(k=32, seed=1))
sg = knng.optimize_graph(g, base, 32)
sp = knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1)
ts = []
for rep in range(max(reps, 1)):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = knng.ann_search(qry, sg, base, sp)
    torch.cuda.synchronize(); ts.append(round(time.perf_counter() - t, 4))
h = hashlib.sha1(r.ids.cpu().numpy().tobytes() + r.dists.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps(dict(n=n, d=d, secs=ts if reps else None, qps=n / min(ts), result_sha1=h)))
