"""Per-stage device times of consecutive C2 builds (which stage carries the
occasional slow build?)."""
import os, sys, json, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
gc.disable()
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
p = knng.NnDescentParams(k=32, seed=1)
for _ in range(3):
    knng.nn_descent(x, p)
for i in range(16):
    st = knng.NnDescentStats()
    knng.nn_descent(x, p, stats=st)
    print(round(st.total_ms, 1), {k: round(v, 1) for k, v in st.stage_ms.items() if v > 1}, flush=True)
