#!/bin/bash
# four independent processes (one per GPU) running consecutive C4-regime local builds
for g in 0 1 2 3; do
  CUDA_VISIBLE_DEVICES=$g python - > gpurun_out/stagevar_mp_$g.log 2>&1 <<'PY' &
import os, sys, gc
sys.path.insert(0, os.getcwd())
import torch, paper_2605_27691_b200 as knng
gc.disable()
x = torch.from_numpy(knng.gen_random_dataset(1_000_000, 128, "clustered", 42, 16)).cuda()
p = knng.NnDescentParams(k=32, seed=1)
for _ in range(3):
    knng.nn_descent(x, p)
for i in range(12):
    st = knng.NnDescentStats()
    knng.nn_descent(x, p, stats=st)
    print(round(st.total_ms, 1), {k: round(v, 1) for k, v in st.stage_ms.items() if v > 5}, flush=True)
PY
done
wait
