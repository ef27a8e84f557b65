"""nn_descent stage breakdown on a named dataset (after warm builds)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n = int(os.environ.get("N", "1000000"))
cl = int(os.environ.get("CL", "16"))
d = int(os.environ.get("D", "128"))
x = torch.from_numpy(knng.gen_random_dataset(n, d, "clustered", 42, cl)).cuda()
p = knng.NnDescentParams(k=32, seed=1)
for _ in range(int(os.environ.get("WARM", "3"))):
    knng.nn_descent(x, p)
st = knng.NnDescentStats()
knng.nn_descent(x, p, stats=st)
print(json.dumps(dict(n=n, clusters=cl, d=d, total_ms=st.total_ms, iterations=st.iterations,
                      stage_ms={k: round(v, 2) for k, v in st.stage_ms.items()},
                      pairs_per_iter=st.pairs_per_iter, offers_per_iter=st.offers_per_iter)))
