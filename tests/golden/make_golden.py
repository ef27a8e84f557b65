"""Mint the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs oracle/_ref/libknng_ref.so (the reference sources compiled in place by
oracle/Makefile) with workers = 1 (the deterministic schedule) and stores
inputs + outputs as small .npz files.  These pin both the C restatement
(tests/test_oracle.py) and the CUDA path (tests/test_parity_gpu.py).  Needs
/root/reference, so it runs here, not on the GPU box; the fixtures are
committed.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import Ref  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def main():
    R = Ref()
    # --- generator: pins gen_random_dataset (evalio.cpp:242-272) -----------
    gen = {}
    for dist, cl in [("uniform", 0), ("gaussian", 0), ("clustered", 7)]:
        gen[dist] = R.gen_random_dataset(257, 9, dist, 42, cl)
    save("gen", **gen)

    # --- core: merge_rows random streams (test_core.cpp:183-210 shape) ------
    rng = np.random.default_rng(31)
    rows = 200
    a_ids = np.zeros((rows, 20), np.uint32)
    a_d = np.zeros((rows, 20), np.float32)
    b_ids = np.zeros((rows, 20), np.uint32)
    b_d = np.zeros((rows, 20), np.float32)
    m_ids = np.zeros((rows, 10), np.uint32)
    m_d = np.zeros((rows, 10), np.float32)
    m_n = np.zeros(rows, np.uint32)
    for r in range(rows):
        ids = rng.choice(40, size=40, replace=False).astype(np.uint32)
        dist = (rng.integers(0, 32, size=40) * 0.25).astype(np.float32)
        # one distance per id (a single metric computes them)
        ai, bi = ids[:20].copy(), np.concatenate([ids[10:20], ids[20:30]])
        ad, bd = dist[:20].copy(), np.concatenate([dist[10:20], dist[20:30]])
        oa = np.lexsort((ai, ad))
        ob = np.lexsort((bi, bd))
        a_ids[r], a_d[r] = ai[oa], ad[oa]
        b_ids[r], b_d[r] = bi[ob], bd[ob]
        oi, od = R.merge_rows(a_ids[r], a_d[r], b_ids[r], b_d[r], 10)
        m_n[r] = len(oi)
        m_ids[r, :len(oi)], m_d[r, :len(oi)] = oi, od
    save("merge_rows", a_ids=a_ids, a_d=a_d, b_ids=b_ids, b_d=b_d, out_ids=m_ids, out_d=m_d,
         out_n=m_n)

    # --- nndescent stages ---------------------------------------------------
    x = R.gen_random_dataset(2000, 16, "clustered", 3, 10)
    ii, idd, iff = R.init_random_graph(x, 12, 5)
    s = R.sample_neighbors(ii, idd, iff, 0.5, 7, 3)
    # a graph with some flags already consumed: second sampling round
    s2 = R.sample_neighbors(ii, idd, s["flags"], 0.5, 7, 4)
    nn_i, nn_d, nn_f, acc, _ = R.nn_descent(x, 16, seed=3, workers=1)
    save("nndescent", x=x, init_ids=ii, init_d=idd, init_f=iff,
         s_bound=np.array([s["bound"]]), s_flags=s["flags"],
         s_new_fwd=s["new_fwd"][0], s_new_fwd_n=s["new_fwd"][1],
         s_old_fwd=s["old_fwd"][0], s_old_fwd_n=s["old_fwd"][1],
         s_new_rev=s["new_rev"][0], s_new_rev_n=s["new_rev"][1],
         s_old_rev=s["old_rev"][0], s_old_rev_n=s["old_rev"][1],
         s2_flags=s2["flags"], s2_new_fwd=s2["new_fwd"][0], s2_new_fwd_n=s2["new_fwd"][1],
         s2_old_fwd=s2["old_fwd"][0], s2_old_fwd_n=s2["old_fwd"][1],
         s2_new_rev=s2["new_rev"][0], s2_new_rev_n=s2["new_rev"][1],
         s2_old_rev=s2["old_rev"][0], s2_old_rev_n=s2["old_rev"][1],
         nn_ids=nn_i, nn_d=nn_d, nn_f=nn_f, nn_accepted=acc)

    # --- graphopt + annsearch on the reference's own graph -----------------
    sg = R.optimize_graph(nn_i, nn_d, x, 16)
    sg8 = R.optimize_graph(nn_i, nn_d, x, 8)
    q = R.gen_random_dataset(500, 16, "clustered", 4, 10)
    si, sd, sh, ss = R.ann_search(q, sg, x, 16, 64, 16, 0, 9)
    si2, sd2, sh2, ss2 = R.ann_search(q, sg, x, 32, 128, 96, 0, 11)
    # self-search (test_annsearch.cpp:46-58 shape)
    selfi, selfd, _, _ = R.ann_search(x[:300].copy(), sg, x, 10, 64, 16, 0, 5)
    save("search", x=x, nn_ids=nn_i, nn_d=nn_d, sg=sg, sg8=sg8, q=q, ids=si, d=sd, hops=sh,
         scored=ss, ids2=si2, d2=sd2, hops2=sh2, scored2=ss2, self_ids=selfi, self_d=selfd)

    # --- partition ------------------------------------------------------------
    xp = R.gen_random_dataset(10001, 2, "uniform", 2)
    te, off = R.partition(xp, 4, 9)
    x8 = R.gen_random_dataset(8, 4, "uniform", 1)
    te8, off8 = R.partition(x8, 4, 5)
    xbig = np.zeros((1000003, 1), np.float32)
    tebig, offbig = R.partition(xbig, 8, 1)
    # the 1M permutation is kept as its head + a position-weighted checksum
    w = np.arange(1, len(tebig) + 1, dtype=np.uint64)
    big_sum = np.array([int((tebig.astype(np.uint64) * w).sum(dtype=np.uint64))], np.uint64)
    save("partition", te=te, off=off, te8=te8, off8=off8, tebig_head=tebig[:4096],
         tebig_sum=big_sum, offbig=offbig)

    # --- brute force ----------------------------------------------------------
    gi, gd = R.brute_force(x, 10, workers=0)
    save("bruteforce", x=x, ids=gi, d=gd)

    # --- distributed pipeline ----------------------------------------------------
    dist = {"x": x}
    for P in (1, 2, 4, 8):
        cfg = R.refine_config(P, 2, 16, nn_seed=2, search_seed=2, seed=2, beam_width=64)
        di, dd, ph, gets, by = R.build_distributed(x, cfg)
        dist[f"p{P}_ids"], dist[f"p{P}_d"] = di, dd
        dist[f"p{P}_gets"] = np.array([gets, by], np.uint64)
    cfg = R.refine_config(4, 2, 16, nn_seed=2, search_seed=2, seed=2)
    lg_i, lg_d = R.build_local_graphs(x, cfg)
    te4, off4, loc4 = R.partition(x, 4, 2, gather=True)
    r0_i, r0_d = R.refine_from_local(x, cfg, lg_i, lg_d, 0)
    r1_i, r1_d = R.refine_from_local(x, cfg, lg_i, lg_d, 1)
    cfg8 = R.refine_config(8, 2, 16, nn_seed=2, search_seed=2, seed=2, beam_width=128,
                           num_entry_points=96)
    lg8_i, lg8_d = R.build_local_graphs(x, cfg8)
    te8b, off8b, loc8 = R.partition(x, 8, 2, gather=True)
    r8_i, r8_d = R.refine_from_local(x, cfg8, lg8_i, lg8_d, 0)
    dist.update(local4_ids=lg_i, local4_d=lg_d, te4=te4, off4=off4, x_perm4=loc4,
                refine4_ids=r0_i, refine4_d=r0_d, a2a4_ids=r1_i, a2a4_d=r1_d,
                local8_ids=lg8_i, local8_d=lg8_d, off8=off8b, x_perm8=loc8, refine8_ids=r8_i,
                refine8_d=r8_d)
    save("distributed", **dist)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
