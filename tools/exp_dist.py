"""Repeated build_distributed on G GPUs (C5-regime, G x 1M x 128 clustered(16))
with per-phase times, to find the source of step-time variance."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
G = int(os.environ.get("G", "2"))
per = int(os.environ.get("PER", "1000000"))
x = torch.from_numpy(knng.gen_random_dataset(G * per, 128, "clustered", 42, 16)).cuda()
cfg = knng.RefineConfig(ranks=G, groups=2, k=32, seed=1, nn=knng.NnDescentParams(k=32, seed=1),
                        search=knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1))
for i in range(int(os.environ.get("REPS", "6"))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = knng.build_distributed(x, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps(dict(i=i, wall_s=round(dt, 3), **{k: round(v, 3) for k, v in r.phases.items()},
                          partition_s=round(r.partition_s, 3), hops=r.search_hops,
                          scored=r.search_scored, nnd_iters=r.nnd_iterations)), flush=True)
