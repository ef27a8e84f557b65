"""Experiment: host vs device time of nn_descent with/without nvidia-smi polling."""
import os, sys, time, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_27691_b200 as knng
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 1000)).cuda()
ctx = knng.context()
stream = torch.cuda.ExternalStream(ctx.stream(0), device="cuda:0")
def run(tag):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    st = knng.NnDescentStats()
    torch.cuda.synchronize()
    t = time.perf_counter()
    ev[0].record(stream)
    knng.nn_descent(x, knng.NnDescentParams(k=32, seed=1), stats=st)
    ev[1].record(stream)
    torch.cuda.synchronize()
    host = (time.perf_counter() - t) * 1e3
    print(json.dumps(dict(tag=tag, host_ms=host, event_ms=ev[0].elapsed_time(ev[1]),
                          build_device_ms=st.total_ms, stages=st.stage_ms)), flush=True)
for i in range(3): run("plain")
os.environ["KNNG_TRACE"] = "1"
for i in range(4): run("traced")
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "200"],
                     stdout=subprocess.DEVNULL)
for i in range(3): run("smi200")
p.terminate()
for i in range(2): run("plain-after")
