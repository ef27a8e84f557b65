"""Phase trace of the N=1 e2e call (pinned host dataset in, host graph out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KNNG_TRACE"] = "1"
import numpy as np, torch, paper_2605_27691_b200 as knng
x = knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)
pinned = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = x
xp = pinned.numpy()
p = knng.NnDescentParams(k=32, seed=1)
for i in range(4):
    t = time.perf_counter()
    g = knng.nn_descent(xp, p)
    print("e2e call", i, round(1000 * (time.perf_counter() - t), 1), "ms", flush=True)
