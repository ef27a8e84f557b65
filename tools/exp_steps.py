"""Per-build event times for consecutive nn_descent builds, with and without
per-stage statistics, to localise the occasional slow step."""
import os, sys, json, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
gc.disable()
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
ctx = knng.context()
stream = torch.cuda.ExternalStream(ctx.stream(0), device="cuda:0")
p = knng.NnDescentParams(k=32, seed=1)
for _ in range(4):
    knng.nn_descent(x, p)
for mode in ("stats", "nostats", "stats", "nostats"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        ev[0].record(stream)
    for i in range(8):
        st = knng.NnDescentStats() if mode == "stats" else None
        knng.nn_descent(x, p, stats=st)
        with torch.cuda.stream(stream):
            ev[i + 1].record(stream)
    torch.cuda.synchronize()
    print(mode, [round(ev[i].elapsed_time(ev[i + 1]), 1) for i in range(8)], flush=True)
