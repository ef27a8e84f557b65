"""Cosine metric (MetricKind::cosine, cosine_t core.hpp:41-55) on the CUDA path.

Each row's norm chain (sum x*x in index order, no FMA) does not depend on its
partner, so the kernels compute it once per row and run only the dot chain
per pair, finishing with the reference's 1 - dot / (sqrt(na) * sqrt(nb)),
clamped at 0, zero vector -> 1.  Held to the same bar as l2: bit-exact ids and
float bits against tests/golden/cosine.npz (minted from the unmodified
reference with cosine datasets) for every deterministic stage; NN-Descent and
the distributed build by invariants, exact stored distances and recall.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(np.asarray(a), np.float32).view(np.uint32)


def recall(ids, gt, k_eval=10):
    hits = 0
    for r in range(gt.shape[0]):
        hits += len(np.intersect1d(ids[r, :k_eval], gt[r, :k_eval]))
    return hits / (gt.shape[0] * k_eval)


def test_cosine_golden_values(knng):
    # test_core.cpp:55-70
    x = np.array([[1.0, 2.0], [2.0, 4.0], [0.0, 3.0], [0.0, 0.0]], np.float32)
    d = knng.row_distances(x, [0, 2, 3, 1], [1, 3, 0, 2], metric="cosine")
    assert d[0] == 0.0 and d[1] == 1.0 and d[2] == 1.0
    assert 0.0 < d[3] < 1.0
    with pytest.raises(ValueError):
        knng.row_distances(x, [0], [1], metric="dot")


def test_cosine_row_distances_bitexact(knng, golden):
    g = golden("cosine")
    d = knng.row_distances(g["x"], g["pair_i"], g["pair_j"], metric="cosine")
    assert np.array_equal(bits(d), bits(g["pair_d"]))
    d7 = knng.row_distances(g["x7"], np.arange(300), np.arange(300)[::-1], metric="cosine")
    assert np.array_equal(bits(d7), bits(g["pair7_d"]))


def test_cosine_init_random_graph_bitexact(knng, golden):
    g = golden("cosine")
    out = knng.init_random_graph(g["x"], 12, 5, metric="cosine")
    assert np.array_equal(out.ids, g["init_ids"])
    assert np.array_equal(bits(out.dists), bits(g["init_d"]))


def test_cosine_nn_descent(knng, oracle, golden):
    g = golden("cosine")
    x = g["x"]
    out = knng.nn_descent(x, k=16, seed=3, metric="cosine")
    assert oracle.check_invariants(out.ids, out.dists) == 0
    rows = np.repeat(np.arange(len(x)), 16)
    flat = out.ids.reshape(-1)
    sel = np.random.default_rng(0).integers(0, len(flat), 4000)
    ref = np.array([oracle.cosine(x[rows[s]], x[flat[s]]) for s in sel], np.float32)
    assert np.array_equal(bits(out.dists.reshape(-1)[sel]), bits(ref))
    again = knng.nn_descent(x, k=16, seed=3, metric="cosine")
    assert np.array_equal(out.ids, again.ids)
    ref_recall = recall(g["nn_ids"], g["bf_ids"])
    mine = recall(out.ids, g["bf_ids"])
    assert mine >= ref_recall - 0.005, (mine, ref_recall)


def test_cosine_optimize_graph_bitexact(knng, golden):
    g = golden("cosine")
    graph = knng.KnnGraph(g["nn_ids"], g["nn_d"])
    assert np.array_equal(knng.optimize_graph(graph, g["x"], 16, metric="cosine"), g["sg"])
    assert np.array_equal(knng.optimize_graph(graph, g["x"], 8, metric="cosine"), g["sg8"])


def test_cosine_ann_search_bitexact(knng, golden):
    g = golden("cosine")
    r = knng.ann_search(g["q"], g["sg"], g["x"], knng.SearchParams(16, 64, 16, 0, 9),
                        diagnostics=True, metric="cosine")
    assert np.array_equal(r.ids, g["s_ids"]) and np.array_equal(bits(r.dists), bits(g["s_d"]))
    assert np.array_equal(r.hops, g["s_hops"]) and np.array_equal(r.scored, g["s_scored"])


def test_cosine_brute_force_bitexact(knng, golden):
    g = golden("cosine")
    i, d = knng.brute_force_knng(g["x"], 10, metric="cosine")
    assert np.array_equal(i, g["bf_ids"]) and np.array_equal(bits(d), bits(g["bf_d"]))
    i, d = knng.brute_force_knng(g["x7"], 8, metric="cosine")
    assert np.array_equal(i, g["bf7_ids"]) and np.array_equal(bits(d), bits(g["bf7_d"]))


def test_cosine_u8_matches_oracle(knng, oracle):
    # cosine_t<uint8_t>: bytes promoted to float; products of bytes are exact
    x = np.random.default_rng(4).integers(0, 256, (1500, 20)).astype(np.uint8)
    x[3] = 0
    i, d = knng.brute_force_knng(x, 10, metric="cosine")
    oi, od = oracle.brute_force_rows(x, np.arange(len(x)), 10, metric=1)
    assert np.array_equal(i, oi) and np.array_equal(bits(d), bits(od))


@pytest.mark.parametrize("P", [2, 4])
def test_cosine_build_distributed(knng, golden, oracle, P):
    g = golden("cosine")
    cfg = knng.RefineConfig(ranks=P, groups=2, k=16, seed=2,
                            nn=knng.NnDescentParams(k=16, seed=2),
                            search=knng.SearchParams(k_s=16, beam_width=64, num_entry_points=16,
                                                     seed=2))
    r = knng.build_distributed(g["x"], cfg, metric="cosine")
    assert oracle.check_invariants(r.graph.ids, r.graph.dists, local=False) == 0
    x = g["x"]
    rows = np.repeat(np.arange(len(x)), 16)
    flat = r.graph.ids.reshape(-1)
    sel = np.random.default_rng(1).integers(0, len(flat), 2000)
    ref = np.array([oracle.cosine(x[rows[s]], x[flat[s]]) for s in sel], np.float32)
    assert np.array_equal(bits(r.graph.dists.reshape(-1)[sel]), bits(ref))
    ref_recall = recall(g[f"p{P}_ids"], g["bf_ids"])
    assert recall(r.graph.ids, g["bf_ids"]) >= ref_recall - 0.02
