import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
def free():
    f, t = torch.cuda.mem_get_info(0)
    return round(f / 2**30, 2)
x = knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 16)
xd = torch.from_numpy(x).cuda()
print("start free GB", free(), flush=True)
for i in range(3):
    knng.nn_descent(xd, knng.NnDescentParams(k=32, seed=1))
    print("after nn_descent", i, free(), flush=True)
cfg = knng.RefineConfig(ranks=2, groups=2, k=32, seed=1, nn=knng.NnDescentParams(k=32, seed=1),
                        search=knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1))
for i in range(3):
    r = knng.build_distributed(xd, cfg)
    print("after build_distributed(dev)", i, free(), r.phases, flush=True)
for i in range(2):
    r = knng.build_distributed(x, cfg)
    print("after build_distributed(host)", i, free(), flush=True)
