"""One nn_descent build (k = 32) of N x D clustered(CL), printed with its
stage times; REPS builds (default 2: the first warms up).
    python tools/one_build.py N D CL [REPS]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
n, d, cl = [int(v) for v in sys.argv[1:4]]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
x = torch.from_numpy(knng.gen_random_dataset(n, d, "clustered", 42, cl)).cuda()
for _ in range(reps):
    st = knng.NnDescentStats()
    torch.cuda.synchronize(); t = time.perf_counter()
    g = knng.nn_descent(x, knng.NnDescentParams(k=32, seed=1),
                        stats=None if os.environ.get("NOSTATS") else st)
    torch.cuda.synchronize()
    print(dict(env={k: v for k, v in os.environ.items() if k.startswith("KNNG_")}, n=n, d=d,
               secs=round(time.perf_counter() - t, 3), iters=st.iterations,
               stage_ms={k: round(v, 1) for k, v in st.stage_ms.items()}), flush=True)
