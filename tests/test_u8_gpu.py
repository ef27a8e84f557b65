"""u8 elements (ElemKind::u8, l2_u8 core.hpp:32-39): the reference promotes
every byte to float before the sequential sum, so the B200 path expands u8
rows to f32 once on the device.  Bit-exact against the C oracle's l2_u8 for
brute force, optimize_graph and ann_search; NN-Descent and build_distributed
on u8 equal the same GPU build on the f32 copy; the comm log charges the
reference's 1-byte dataset elements (wire.cpp region sizes)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _u8(n, d, seed):
    rng = np.random.default_rng(seed)
    centers = rng.integers(0, 256, size=(12, d))
    lab = rng.integers(0, 12, size=n)
    return np.clip(centers[lab] + rng.normal(0, 18, size=(n, d)), 0, 255).astype(np.uint8)


def test_u8_brute_force_and_graph_stages_match_oracle(knng, oracle):
    x = _u8(3000, 24, 1)
    rows = np.arange(0, 3000, 7, dtype=np.uint64)
    gi, gd = knng.brute_force_knng(x, 10, rows=rows)
    oi, od = oracle.brute_force_rows(x, rows, 10)
    assert np.array_equal(np.asarray(gi), oi)
    assert np.array_equal(np.asarray(gd).view(np.uint32), od.view(np.uint32))
    g = knng.nn_descent(x, knng.NnDescentParams(k=16, seed=2))
    sg = knng.optimize_graph(g, x, 16)
    osg = oracle.optimize_graph(g.ids, g.dists, x, 16)
    assert np.array_equal(np.asarray(sg), osg)
    q = _u8(500, 24, 9)
    sp = knng.SearchParams(k_s=10, beam_width=32, num_entry_points=16, seed=4)
    r = knng.ann_search(q, sg, x, sp, diagnostics=True)
    oi, od, oh, osc = oracle.ann_search(q, osg, x, k_s=10, beam_width=32, num_entry_points=16,
                                        seed=4)
    assert np.array_equal(np.asarray(r.ids), oi)
    assert np.array_equal(np.asarray(r.dists).view(np.uint32), od.view(np.uint32))
    assert np.array_equal(np.asarray(r.hops), oh) and np.array_equal(np.asarray(r.scored), osc)


def test_u8_builds_equal_f32_copy(knng):
    x = _u8(4000, 16, 3)
    p = knng.NnDescentParams(k=16, seed=5)
    a, b = knng.nn_descent(x, p), knng.nn_descent(x.astype(np.float32), p)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists.view(np.uint32),
                                                           b.dists.view(np.uint32))
    cfg = knng.RefineConfig(ranks=2, groups=2, k=16, seed=7, nn=knng.NnDescentParams(k=16, seed=3),
                            search=knng.SearchParams(k_s=16, beam_width=32, num_entry_points=16,
                                                     seed=5))
    ra, rb = knng.build_distributed(x, cfg), knng.build_distributed(x.astype(np.float32), cfg)
    assert np.array_equal(ra.graph.ids, rb.graph.ids)
    assert np.array_equal(ra.graph.dists.view(np.uint32), rb.graph.dists.view(np.uint32))
    # dataset regions are charged at 1 byte per element (22-byte wire header)
    ds_a = [g.bytes for g in ra.comm_log if g.region == "dataset"]
    ds_b = [g.bytes for g in rb.comm_log if g.region == "dataset"]
    assert ds_a and all(ba - 22 == (bb - 22) // 4 for ba, bb in zip(ds_a, ds_b))
