import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2605_27691_b200 as knng
for cl in (1000, 16):
    x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, cl)).cuda()
    for rep in range(2):
        st = knng.NnDescentStats()
        knng.nn_descent(x, knng.NnDescentParams(k=32, seed=1), stats=st)
        print(json.dumps(dict(clusters=cl, iters=st.iterations, total=st.total_ms,
                              stages={k: round(v, 1) for k, v in st.stage_ms.items()},
                              offers=st.offers_per_iter, pairs=st.pairs_per_iter)), flush=True)
