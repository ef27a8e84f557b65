"""search_throughput_probe (annsearch.cpp:131-155): one row per case in input
order, num_queries = |queries|, positive QPS; an empty query set and
non-ascending sizes are usage errors (std::invalid_argument)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_search_throughput_probe(knng):
    sp = knng.SearchParams(k_s=10, beam_width=32, num_entry_points=16, seed=1)
    cases = []
    for n in (2000, 6000):
        x = knng.gen_random_dataset(n, 16, "clustered", 11, 8)
        g = knng.nn_descent(x, knng.NnDescentParams(k=16, seed=1))
        cases.append((n, knng.optimize_graph(g, x, 16), x))
    q = knng.gen_random_dataset(500, 16, "clustered", 12, 8)
    rows = knng.search_throughput_probe(cases, q, sp)
    assert [r.source_count for r in rows] == [2000, 6000]
    assert all(r.num_queries == 500 and r.seconds > 0 and r.qps > 0 for r in rows)
    with pytest.raises(knng.InvalidArgument):
        knng.search_throughput_probe(cases[::-1], q, sp)
    with pytest.raises(knng.InvalidArgument):
        knng.search_throughput_probe(cases, np.zeros((0, 16), np.float32), sp)


def test_read_vecs_to_device(knng, tmp_path):
    rng = np.random.default_rng(5)
    x = rng.normal(size=(400001, 24)).astype(np.float32)  # 38 MB: more than one staging buffer
    p = str(tmp_path / "x.fvecs")
    knng.write_vecs(p, x)
    y = knng.read_vecs(p, "f32", device=0)
    assert y.is_cuda and np.array_equal(y.cpu().numpy().view(np.uint32), x.view(np.uint32))
    b = rng.integers(0, 256, size=(5000, 96)).astype(np.uint8)
    knng.write_vecs(str(tmp_path / "b.bvecs"), b)
    z = knng.read_vecs(str(tmp_path / "b.bvecs"), "u8", device=0)
    assert np.array_equal(z.cpu().numpy(), b)
