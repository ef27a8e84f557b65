"""C2 build (1M x 128 clustered(1000), k=32): per-stage device ms for the
join slice width given by KNNG_JOIN_DC (tuning experiment)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2605_27691_b200 as knng
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
p = knng.NnDescentParams(k=32, seed=1)
rows = []
for _ in range(4):
    st = knng.NnDescentStats()
    g = knng.nn_descent(x, p, stats=st)
    rows.append((st.total_ms, st.join_ms))
torch.cuda.synchronize()
ids = g.ids if isinstance(g.ids, np.ndarray) else g.ids.cpu().numpy()
print(json.dumps({"dc": os.environ.get("KNNG_JOIN_DC", "32"), "total_ms": [round(a, 1) for a, _ in rows],
                  "join_ms": [round(b, 1) for _, b in rows], "pairs": st.pairs,
                  "ids_sum": int(ids.astype(np.uint64).sum())}))
