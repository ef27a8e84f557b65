"""Reproduce bench.py's N=1 timed loop with host traces (KNNG_TRACE)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KNNG_TRACE"] = "1"
import torch, paper_2605_27691_b200 as knng
x_host = knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)
pinned = torch.empty(x_host.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = x_host
x = pinned.to("cuda:0"); torch.cuda.synchronize()
ctx = knng.context()
stream = torch.cuda.ExternalStream(ctx.stream(0), device="cuda:0")
params = knng.NnDescentParams(k=32, seed=1)
for i in range(3):
    knng.nn_descent(x, params)
res = None
for i in range(4):
    st = knng.NnDescentStats()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e[0].record(stream)
    res = knng.nn_descent(x, params, stats=st)
    t1 = time.perf_counter()
    e[1].record(stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps(dict(i=i, call_ms=(t1 - t0) * 1e3, wall_ms=(t2 - t0) * 1e3,
                          event_ms=e[0].elapsed_time(e[1]), build_ms=st.total_ms)), flush=True)
