import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
def free():
    return [round(torch.cuda.mem_get_info(d)[0] / 2**30, 2) for d in range(torch.cuda.device_count())]
x = knng.gen_random_dataset(2_000_000, 128, "clustered", 42, 16)
xd = torch.from_numpy(x).cuda()
print("devices", knng.context().device_count, "start free GB", free(), flush=True)
cfg = knng.RefineConfig(ranks=2, groups=2, k=32, seed=1, nn=knng.NnDescentParams(k=32, seed=1),
                        search=knng.SearchParams(k_s=32, beam_width=128, num_entry_points=96, seed=1))
for i in range(3):
    try:
        r = knng.build_distributed(xd, cfg)
        print("dev", i, free(), {k: round(v, 3) for k, v in r.phases.items()}, r.partition_s, flush=True)
    except Exception as e:
        print("ERR", i, e, free(), flush=True)
for i in range(2):
    try:
        r = knng.build_distributed(x, cfg)
        print("host", i, free(), flush=True)
    except Exception as e:
        print("ERR host", i, e, free(), flush=True)
