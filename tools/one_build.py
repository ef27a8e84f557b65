import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_2605_27691_b200 as knng
n, d, cl = [int(v) for v in sys.argv[1:4]]
x = torch.from_numpy(knng.gen_random_dataset(n, d, "clustered", 42, cl)).cuda()
st = knng.NnDescentStats()
g = knng.nn_descent(x, knng.NnDescentParams(k=32, seed=1), stats=st)
print(st.iterations, st.stage_ms)
