"""One C2 build (1M x 128 clustered(1000), k=32) after two warm builds -- ncu driver."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
p = knng.NnDescentParams(k=32, seed=1)
for _ in range(int(os.environ.get("BUILDS", "3"))):
    g = knng.nn_descent(x, p)
torch.cuda.synchronize()
print("ok")
