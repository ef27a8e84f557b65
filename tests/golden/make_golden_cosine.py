"""Mint the cosine-metric golden fixture (tests/golden/cosine.npz) from the
UNMODIFIED reference (oracle/_ref/libknng_ref.so, every shim dataset built
with MetricKind::cosine via kr_set_metric), workers = 1.  Pins the C
restatement's cosine_t (core.hpp:41-55) in tests/test_oracle.py and every
cosine kernel of the CUDA path in tests/test_cosine_gpu.py.  Needs
/root/reference, so it runs here; the fixture is committed.

    python tests/golden/make_golden_cosine.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import Ref  # noqa: E402


def main():
    R = Ref()
    R.set_metric(1)
    # d = 36: two 32-dim join chunks plus a 4-dim tail; zero rows exercise the
    # zero-vector rule (distance 1.0, core.hpp:51)
    x = R.gen_random_dataset(2000, 36, "clustered", 3, 10)
    x[[5, 77, 1500]] = 0.0
    rng = np.random.default_rng(2)
    pi = rng.integers(0, len(x), 4000).astype(np.uint32)
    pj = rng.integers(0, len(x), 4000).astype(np.uint32)
    pi[:3], pj[:3] = 5, [6, 77, 5]
    pd = np.array([R.cosine(x[a], x[b]) for a, b in zip(pi, pj)], np.float32)
    # odd dims: the scalar (non-float4) paths
    x7 = R.gen_random_dataset(300, 7, "gaussian", 8)
    p7 = np.array([R.cosine(x7[a], x7[299 - a]) for a in range(300)], np.float32)

    ii, idd, iff = R.init_random_graph(x, 12, 5)
    nn_i, nn_d, nn_f, acc, _ = R.nn_descent(x, 16, seed=3, workers=1)
    sg = R.optimize_graph(nn_i, nn_d, x, 16)
    sg8 = R.optimize_graph(nn_i, nn_d, x, 8)
    q = R.gen_random_dataset(500, 36, "clustered", 4, 10)
    si, sd, sh, ss = R.ann_search(q, sg, x, 16, 64, 16, 0, 9)
    gi, gd = R.brute_force(x, 10, workers=0)
    g7i, g7d = R.brute_force(x7, 8, workers=0)
    out = dict(x=x, pair_i=pi, pair_j=pj, pair_d=pd, x7=x7, pair7_d=p7,
               init_ids=ii, init_d=idd, nn_ids=nn_i, nn_d=nn_d, sg=sg, sg8=sg8, q=q,
               s_ids=si, s_d=sd, s_hops=sh, s_scored=ss, bf_ids=gi, bf_d=gd, bf7_ids=g7i,
               bf7_d=g7d)
    for P in (2, 4):
        cfg = R.refine_config(P, 2, 16, nn_seed=2, search_seed=2, seed=2, beam_width=64)
        di, dd, _, _, _ = R.build_distributed(x, cfg)
        out[f"p{P}_ids"], out[f"p{P}_d"] = di, dd
    R.set_metric(0)
    np.savez_compressed(os.path.join(HERE, "cosine.npz"), **out)
    print("cosine fixture written to", HERE)


if __name__ == "__main__":
    main()
