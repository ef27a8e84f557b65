import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KNNG_TRACE"] = "1"
import torch, paper_2605_27691_b200 as knng
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
st = knng.NnDescentStats()
knng.nn_descent(x, knng.NnDescentParams(k=32, seed=1), stats=st)
print(st.stage_ms)
