"""The C-ABI boundary without a GPU: the library loads, exports every entry
point include/knng_c.h declares, its host-side functions (generator, wire
output, tree schedule, validation) match the reference, and compute calls fail
loudly -- never a silent CPU fallback -- when no GPU is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knng_c.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(knng_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(knng):
    L = knng.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), f"{s} declared in knng_c.h but not exported"
    # the Python mirror binds every declared symbol
    assert sorted(knng.exported_symbols()) == syms


def test_abi_version(knng):
    assert knng.abi_version() == 1


def test_generator_matches_reference(knng, golden):
    g = golden("gen")
    for dist, cl in [("uniform", 0), ("gaussian", 0), ("clustered", 7)]:
        x = knng.gen_random_dataset(257, 9, dist, 42, cl)
        assert np.array_equal(x.view(np.uint32), g[dist].view(np.uint32))
    with pytest.raises(knng.InvalidArgument):
        knng.gen_random_dataset(10, 3, "clustered", 1, 0)


def test_wire_roundtrip(knng, tmp_path):
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 1 << 31, size=(37, 5)).astype(np.uint32)
    d = rng.random((37, 5)).astype(np.float32)
    p = str(tmp_path / "g.knng")
    knng.save_graph(knng.KnnGraph(ids, d), p)
    raw = open(p, "rb").read()
    # wire.hpp:14-19: magic KNNG, kind 1 (knng), rows, cols, elem 0, ids, dists
    assert len(raw) == 22 + 37 * 5 * 8
    assert raw[:4] == (0x474E4E4B).to_bytes(4, "little") and raw[4] == 1
    assert int.from_bytes(raw[5:13], "little") == 37 and int.from_bytes(raw[13:21], "little") == 5
    assert raw[21] == 0
    assert raw[22:22 + ids.nbytes] == ids.tobytes()
    g = knng.load_graph(p)
    assert np.array_equal(g.ids, ids) and np.array_equal(g.dists.view(np.uint32), d.view(np.uint32))
    open(p, "wb").write(raw[:-1])
    with pytest.raises(knng.FormatError):
        knng.load_graph(p)


def test_tree_schedule(knng):
    # test_refine.cpp:69-110
    assert knng.tree_schedule(8, 2, 0, 0)[2] == [1]
    assert knng.tree_schedule(8, 2, 0, 1)[2] == [2, 3]
    assert knng.tree_schedule(8, 2, 0, 0)[:2] == (0, 1)
    assert knng.tree_schedule(8, 2, 0, 1)[1] == 2
    assert knng.tree_levels(8, 2) == 2
    assert knng.tree_levels(4, 4) == 0
    with pytest.raises(knng.InvalidArgument):
        knng.tree_schedule(4, 4, 0, 0)
    p = 2
    while p <= 64:
        m = 2
        while m <= p:
            for rank in range(p):
                for level in range(knng.tree_levels(p, m)):
                    lo, hi, partners = knng.tree_schedule(p, m, rank, level)
                    size = 1 << level
                    assert hi - lo == size and len(partners) == size and lo <= rank < hi
                    plo = partners[0]
                    assert partners[-1] == plo + size - 1
                    assert plo == hi or plo + size == lo
                    assert min(lo, plo) % (2 * size) == 0
            m *= 2
        p *= 2


def test_compute_without_gpu_fails_loudly(knng):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    x = np.zeros((10, 4), np.float32)
    with pytest.raises(knng.KnngError):
        knng.nn_descent(x, k=3)


def test_nn_descent_out_validation(knng):
    # nn_descent(out=...) checks the caller's buffers before any device work
    x = np.zeros((10, 4), np.float32)
    bad = [knng.KnnGraph(np.zeros((10, 2), np.uint32), np.zeros((10, 3), np.float32), None),
           knng.KnnGraph(np.zeros((10, 3), np.uint64), np.zeros((10, 3), np.float32), None),
           knng.KnnGraph(np.zeros((10, 3), np.uint32), np.zeros((3, 10), np.float32).T, None),
           knng.KnnGraph(np.zeros((10, 3), np.uint32), np.zeros((10, 3), np.float32),
                         np.zeros((10, 3), np.uint32))]
    for g in bad:
        with pytest.raises(knng.InvalidArgument):
            knng.nn_descent(x, k=3, out=g)


def test_build_distributed_rank_out_validation(knng):
    # build_distributed_rank(out=...) checks the caller's buffers first
    x = np.zeros((10, 4), np.float32)
    cfg = knng.RefineConfig(ranks=2, groups=2, k=3)
    bad = (np.zeros((5, 2), np.uint32), np.zeros((5, 3), np.float32), np.zeros(5, np.uint32))
    with pytest.raises(knng.InvalidArgument):
        knng.build_distributed_rank(x, cfg, 0, 2, allgather=lambda b, n: b, out=bad)


def test_cpp_dropin_compiles(knng):
    """include/knng_b200.hpp (the reference's C++ API over the C-ABI) builds
    and links against libknng_b200.so; tests/cpp/dropin_test.cpp restates
    reference test cases through it (run on the GPU by test_parity_gpu)."""
    import subprocess
    res = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert os.path.exists(os.path.join(ROOT, "build", "dropin_test"))
