"""The C restatement (oracle/knng_oracle.c) against the golden fixtures minted
from the unmodified reference (tests/golden/make_golden.py).  CPU only.

Every comparison is bit-exact: ids, and float32 distances compared as bits.
"""
import numpy as np
import pytest

from oracle.bindings import KoSearchParams  # noqa: F401


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_generator(golden, oracle):
    g = golden("gen")
    for dist, cl in [("uniform", 0), ("gaussian", 0), ("clustered", 7)]:
        assert np.array_equal(bits(oracle.gen_random_dataset(257, 9, dist, 42, cl)), bits(g[dist]))


def test_l2_golden_values(oracle):
    # test_core.cpp:47-53
    assert oracle.l2([0.0, 0.0], [3.0, 4.0]) == 5.0
    assert oracle.l2([1.0, 2.0], [1.0, 2.0]) == 0.0


def test_merge_rows(golden, oracle):
    g = golden("merge_rows")
    for r in range(g["a_ids"].shape[0]):
        oi, od = oracle.merge_rows(g["a_ids"][r], g["a_d"][r], g["b_ids"][r], g["b_d"][r], 10)
        n = int(g["out_n"][r])
        assert len(oi) == n
        assert np.array_equal(oi, g["out_ids"][r, :n])
        assert np.array_equal(bits(od), bits(g["out_d"][r, :n]))


def test_init_random_graph(golden, oracle):
    g = golden("nndescent")
    ids, d, f = oracle.init_random_graph(g["x"], 12, 5)
    assert np.array_equal(ids, g["init_ids"])
    assert np.array_equal(bits(d), bits(g["init_d"]))
    assert np.array_equal(f, g["init_f"])


def _cmp_lists(a_mat, a_n, b_mat, b_n):
    assert np.array_equal(a_n, b_n)
    for p in range(len(a_n)):
        assert np.array_equal(a_mat[p, :a_n[p]], b_mat[p, :b_n[p]]), p


def test_sample_neighbors_two_rounds(golden, oracle):
    g = golden("nndescent")
    s = oracle.sample_neighbors(g["init_ids"], g["init_f"], 0.5, 7, 3)
    assert s["bound"] == int(g["s_bound"][0])
    assert np.array_equal(s["flags"], g["s_flags"])
    for key in ("new_fwd", "old_fwd", "new_rev", "old_rev"):
        _cmp_lists(*s[key], g["s_" + key], g["s_" + key + "_n"])
    s2 = oracle.sample_neighbors(g["init_ids"], g["s_flags"], 0.5, 7, 4)
    assert np.array_equal(s2["flags"], g["s2_flags"])
    for key in ("new_fwd", "old_fwd", "new_rev", "old_rev"):
        _cmp_lists(*s2[key], g["s2_" + key], g["s2_" + key + "_n"])


def test_nn_descent_workers1(golden, oracle):
    g = golden("nndescent")
    ids, d, f, acc = oracle.nn_descent(g["x"], 16, seed=3)
    assert np.array_equal(ids, g["nn_ids"])
    assert np.array_equal(bits(d), bits(g["nn_d"]))
    assert np.array_equal(f, g["nn_f"])
    assert np.array_equal(acc, g["nn_accepted"])
    assert oracle.check_invariants(ids, d) == 0


def test_optimize_graph(golden, oracle):
    g = golden("search")
    assert np.array_equal(oracle.optimize_graph(g["nn_ids"], g["nn_d"], g["x"], 16), g["sg"])
    assert np.array_equal(oracle.optimize_graph(g["nn_ids"], g["nn_d"], g["x"], 8), g["sg8"])


def test_ann_search(golden, oracle):
    g = golden("search")
    i, d, h, s = oracle.ann_search(g["q"], g["sg"], g["x"], 16, 64, 16, 0, 9)
    assert np.array_equal(i, g["ids"]) and np.array_equal(bits(d), bits(g["d"]))
    assert np.array_equal(h, g["hops"]) and np.array_equal(s, g["scored"])
    i, d, h, s = oracle.ann_search(g["q"], g["sg"], g["x"], 32, 128, 96, 0, 11)
    assert np.array_equal(i, g["ids2"]) and np.array_equal(bits(d), bits(g["d2"]))
    assert np.array_equal(h, g["hops2"]) and np.array_equal(s, g["scored2"])


def test_partition(golden, oracle):
    g = golden("partition")
    te, off = oracle.partition(10001, 4, 9)
    assert np.array_equal(te, g["te"]) and np.array_equal(off, g["off"])
    assert list(off) == [0, 2501, 5001, 7501, 10001]  # test_refine.cpp:59-64
    te8, off8 = oracle.partition(8, 4, 5)
    assert np.array_equal(te8, g["te8"]) and list(off8) == [0, 2, 4, 6, 8]
    teb, offb = oracle.partition(1000003, 8, 1)
    w = np.arange(1, len(teb) + 1, dtype=np.uint64)
    assert np.array_equal(teb[:4096], g["tebig_head"])
    assert int((teb.astype(np.uint64) * w).sum(dtype=np.uint64)) == int(g["tebig_sum"][0])
    with pytest.raises(ValueError):
        oracle.partition(8, 9, 0)


def test_brute_force(golden, oracle):
    g = golden("bruteforce")
    rows = np.arange(0, 2000, 3, dtype=np.uint64)
    i, d = oracle.brute_force_rows(g["x"], rows, 10)
    assert np.array_equal(i, g["ids"][rows]) and np.array_equal(bits(d), bits(g["d"][rows]))


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_build_distributed(golden, oracle, P):
    g = golden("distributed")
    cfg = oracle.refine_config(P, 2, 16, nn_seed=2, search_seed=2, seed=2, beam_width=64)
    i, d = oracle.build_distributed(g["x"], cfg)
    assert np.array_equal(i, g[f"p{P}_ids"]) and np.array_equal(bits(d), bits(g[f"p{P}_d"]))


def test_refine_from_local(golden, oracle):
    g = golden("distributed")
    cfg = oracle.refine_config(4, 2, 16, nn_seed=2, search_seed=2, seed=2)
    te, off = oracle.partition(2000, 4, 2)
    for mode, key in [(0, "refine4"), (1, "a2a4")]:
        i, d = oracle.refine_from_local(g["x"], cfg, te, off, g["local4_ids"], g["local4_d"], mode)
        assert np.array_equal(i, g[key + "_ids"]) and np.array_equal(bits(d), bits(g[key + "_d"]))
    cfg8 = oracle.refine_config(8, 2, 16, nn_seed=2, search_seed=2, seed=2, beam_width=128,
                                num_entry_points=96)
    te8, off8 = oracle.partition(2000, 8, 2)
    i, d = oracle.refine_from_local(g["x"], cfg8, te8, off8, g["local8_ids"], g["local8_d"], 0)
    assert np.array_equal(i, g["refine8_ids"]) and np.array_equal(bits(d), bits(g["refine8_d"]))


def test_tree_schedule_worked_example(oracle):
    # test_refine.cpp:69-76
    import ctypes as C
    L = oracle.L
    L.ko_tree_schedule.restype = C.c_long
    L.ko_tree_schedule.argtypes = [C.c_size_t] * 4 + [C.POINTER(C.c_size_t),
                                                      C.POINTER(C.c_size_t)]
    hi = C.c_size_t(0)
    partners = (C.c_size_t * 8)()
    assert L.ko_tree_schedule(8, 2, 0, 0, C.byref(hi), partners) == 0 and partners[0] == 1
    assert L.ko_tree_schedule(8, 2, 0, 1, C.byref(hi), partners) == 0
    assert list(partners[:2]) == [2, 3] and hi.value == 2
    assert L.ko_tree_levels(8, 2) == 2 and L.ko_tree_levels(4, 4) == 0


# ---------------------------------------------------------------------------
# cosine metric (core.hpp:41-55), pinned by tests/golden/cosine.npz (minted
# from the reference with MetricKind::cosine datasets)
# ---------------------------------------------------------------------------


def test_cosine_golden_values(oracle):
    # test_core.cpp:55-70: parallel -> 0, orthogonal -> 1, zero vector -> 1
    assert oracle.cosine([1.0, 2.0], [2.0, 4.0]) == 0.0
    assert oracle.cosine([1.0, 0.0], [0.0, 3.0]) == 1.0
    assert oracle.cosine([0.0, 0.0], [1.0, 1.0]) == 1.0


def test_cosine_pairs(golden, oracle):
    g = golden("cosine")
    x = g["x"]
    d = np.array([oracle.cosine(x[a], x[b]) for a, b in zip(g["pair_i"], g["pair_j"])],
                 np.float32)
    assert np.array_equal(bits(d), bits(g["pair_d"]))
    x7 = g["x7"]
    d7 = np.array([oracle.cosine(x7[a], x7[299 - a]) for a in range(300)], np.float32)
    assert np.array_equal(bits(d7), bits(g["pair7_d"]))


def test_cosine_stages(golden, oracle):
    g = golden("cosine")
    x = g["x"]
    ii, idd, _ = oracle.init_random_graph(x, 12, 5, metric=1)
    assert np.array_equal(ii, g["init_ids"]) and np.array_equal(bits(idd), bits(g["init_d"]))
    ni, nd, _, _ = oracle.nn_descent(x, 16, seed=3, metric=1)
    assert np.array_equal(ni, g["nn_ids"]) and np.array_equal(bits(nd), bits(g["nn_d"]))
    assert np.array_equal(oracle.optimize_graph(g["nn_ids"], g["nn_d"], x, 16, metric=1), g["sg"])
    assert np.array_equal(oracle.optimize_graph(g["nn_ids"], g["nn_d"], x, 8, metric=1), g["sg8"])
    i, d, h, s = oracle.ann_search(g["q"], g["sg"], x, 16, 64, 16, 0, 9, metric=1)
    assert np.array_equal(i, g["s_ids"]) and np.array_equal(bits(d), bits(g["s_d"]))
    assert np.array_equal(h, g["s_hops"]) and np.array_equal(s, g["s_scored"])
    bi, bd = oracle.brute_force_rows(x, np.arange(len(x)), 10, metric=1)
    assert np.array_equal(bi, g["bf_ids"]) and np.array_equal(bits(bd), bits(g["bf_d"]))


MEMORY_CASES = {  # tests/golden/make_golden_memory.py (double_buffer is timing-only)
    "p4_skip": (4, 2, True, 0, 64, 16), "p4_concat1": (4, 2, False, 1, 64, 16),
    "p4_concat1g": (4, 2, False, 1 << 30, 64, 16), "p8_skip": (8, 2, True, 0, 128, 96),
    "p8_concat1": (8, 2, False, 1, 128, 96), "p8_m4": (8, 4, False, 0, 64, 16),
    "p8_m4_db": (8, 4, False, 0, 64, 16)}


@pytest.mark.parametrize("name", sorted(MEMORY_CASES))
def test_memory_pressure_paths_vs_reference(golden, oracle, name):
    """skip_tree_phase / max_concat_bytes (refine.cpp:160-183) and M = 4 with
    double_buffer (refine.cpp:343-350): the C restatement equals the unmodified
    reference on the same local graphs."""
    g, m = golden("distributed"), golden("memory_paths")
    P, M, skip, mcb, beam, ent = MEMORY_CASES[name]
    cfg = oracle.refine_config(P, M, 16, nn_seed=2, search_seed=2, seed=2, beam_width=beam,
                               num_entry_points=ent, skip_tree=skip, max_concat_bytes=mcb)
    te, off = oracle.partition(2000, P, 2)
    i, d = oracle.refine_from_local(g["x"], cfg, te, off, g[f"local{P}_ids"],
                                    g[f"local{P}_d"], 0)
    assert np.array_equal(i, m[name + "_ids"]) and np.array_equal(bits(d), bits(m[name + "_d"]))
    if name in ("p4_skip", "p4_concat1", "p8_skip", "p8_concat1"):
        # the skip really changed the schedule (else the case would not test it)
        base = g["refine4_ids"] if P == 4 else g["refine8_ids"]
        assert not np.array_equal(i, base)
    if name == "p4_concat1g":
        assert np.array_equal(i, g["refine4_ids"])
