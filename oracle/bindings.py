"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/liboracle.so``       -- the plain-C restatement (knng_oracle.c);
* ``oracle/_ref/libknng_ref.so`` -- the unmodified reference
  (/root/reference/proj/src) behind the ``ref_capi.cpp`` shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2605_27691_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libknng_ref.so")

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
sz = C.c_size_t

DIST = {"uniform": 0, "gaussian": 1, "clustered": 2}


def build():
    """Run oracle/Makefile (C restatement always; reference when present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class KoDataset(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", sz), ("dims", sz), ("elem", C.c_int),
                ("metric", C.c_int)]


class KoNndParams(C.Structure):
    _fields_ = [("k", sz), ("delta", C.c_double), ("rho", C.c_double), ("max_iters", sz),
                ("candidate_capacity", sz), ("seed", C.c_uint64)]


class KoSearchParams(C.Structure):
    _fields_ = [("k_s", sz), ("beam_width", sz), ("num_entry_points", sz), ("max_hops", sz),
                ("seed", C.c_uint64)]


class KoRefineConfig(C.Structure):
    _fields_ = [("ranks", sz), ("groups", sz), ("k", sz), ("k_s", sz), ("out_degree", sz),
                ("nn", KoNndParams), ("search", KoSearchParams), ("skip_tree_phase", C.c_int),
                ("max_concat_bytes", sz), ("seed", C.c_uint64)]


def _ds(x: np.ndarray, metric: int = 0) -> KoDataset:
    assert x.flags.c_contiguous
    elem = 0 if x.dtype == np.float32 else 1
    return KoDataset(x.ctypes.data, x.shape[0], x.shape[1], elem, metric)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.ko_mix_seed.restype = C.c_uint64
        L.ko_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ko_l2_f32.restype = C.c_float
        L.ko_l2_f32.argtypes = [f32p, f32p, sz]
        L.ko_cosine_f32.restype = C.c_float
        L.ko_cosine_f32.argtypes = [f32p, f32p, sz]
        L.ko_gen_random_dataset.argtypes = [sz, sz, C.c_int, C.c_uint64, sz, f32p]
        L.ko_init_random_graph.argtypes = [C.POINTER(KoDataset), sz, C.c_uint64, u32p, f32p, u8p]
        L.ko_sample_neighbors.restype = sz
        L.ko_sample_neighbors.argtypes = [u32p, u8p, sz, sz, C.c_double, C.c_uint64, sz,
                                          u32p, u32p, u32p, u32p, u32p, u32p, u32p, u32p]
        L.ko_nn_descent.restype = C.c_long
        L.ko_nn_descent.argtypes = [C.POINTER(KoDataset), C.POINTER(KoNndParams), u32p, f32p,
                                    u8p, u64p]
        L.ko_optimize_graph.argtypes = [u32p, f32p, sz, sz, C.POINTER(KoDataset), sz, u32p]
        L.ko_ann_search.argtypes = [C.POINTER(KoDataset), u32p, sz, sz, C.POINTER(KoDataset),
                                    C.POINTER(KoSearchParams), u32p, f32p, u32p, u32p]
        L.ko_partition.argtypes = [sz, sz, C.c_uint64, u32p, u64p]
        L.ko_tree_levels.restype = C.c_long
        L.ko_tree_levels.argtypes = [sz, sz]
        L.ko_merge_rows_flat.restype = sz
        L.ko_merge_rows_flat.argtypes = [u32p, f32p, sz, u32p, f32p, sz, sz, u32p, f32p]
        L.ko_check_graph_invariants.argtypes = [u32p, f32p, sz, sz, C.c_int]
        L.ko_build_distributed.argtypes = [C.POINTER(KoDataset), C.POINTER(KoRefineConfig),
                                           u32p, f32p]
        L.ko_refine_from_local.argtypes = [C.POINTER(KoDataset), C.POINTER(KoRefineConfig),
                                           u32p, u64p, u32p, f32p, C.c_int]
        L.ko_translate_to_external.argtypes = [u32p, sz, sz, u32p, f32p, u32p, f32p]
        L.ko_brute_force_rows.argtypes = [C.POINTER(KoDataset), u64p, sz, sz, u32p, f32p]
        L.ko_recall_rows.restype = C.c_double
        L.ko_recall_rows.argtypes = [u32p, sz, u32p, sz, sz, sz]

    # -- wrappers -----------------------------------------------------------
    def mix_seed(self, a, b):
        return self.L.ko_mix_seed(a, b)

    def l2(self, a, b):
        return self.L.ko_l2_f32(np.ascontiguousarray(a, np.float32),
                                np.ascontiguousarray(b, np.float32), len(a))

    def cosine(self, a, b):
        return self.L.ko_cosine_f32(np.ascontiguousarray(a, np.float32),
                                    np.ascontiguousarray(b, np.float32), len(a))

    def gen_random_dataset(self, n, dims, dist, seed, clusters=0):
        out = np.empty((n, dims), np.float32)
        rc = self.L.ko_gen_random_dataset(n, dims, DIST[dist], seed, clusters, out)
        if rc:
            raise ValueError("gen_random_dataset: invalid arguments")
        return out

    def init_random_graph(self, x, k, seed, metric=0):
        n = x.shape[0]
        ids = np.empty((n, k), np.uint32)
        d = np.empty((n, k), np.float32)
        f = np.empty((n, k), np.uint8)
        ds = _ds(x, metric)
        if self.L.ko_init_random_graph(C.byref(ds), k, seed, ids, d, f):
            raise ValueError("init_random_graph: need 1 <= k < N")
        return ids, d, f

    def sample_neighbors(self, ids, flags, rho, seed, it):
        n, k = ids.shape
        import math
        b = int(math.ceil(rho * k))
        ids = np.ascontiguousarray(ids, np.uint32)
        flags = np.array(flags, np.uint8, copy=True)
        nf = np.zeros((n, max(b, 1)), np.uint32)
        of = np.zeros((n, k), np.uint32)
        nr = np.zeros((n, max(b, 1)), np.uint32)
        orv = np.zeros((n, max(b, 1)), np.uint32)
        cnt = [np.zeros(n, np.uint32) for _ in range(4)]
        self.L.ko_sample_neighbors(ids, flags, n, k, rho, seed, it, nf, cnt[0], of, cnt[1],
                                   nr, cnt[2], orv, cnt[3])
        return dict(bound=b, flags=flags, new_fwd=(nf, cnt[0]), old_fwd=(of, cnt[1]),
                    new_rev=(nr, cnt[2]), old_rev=(orv, cnt[3]))

    def nn_descent(self, x, k, delta=1e-4, rho=0.5, max_iters=100, cap=0, seed=0, metric=0):
        n = x.shape[0]
        ids = np.empty((n, k), np.uint32)
        d = np.empty((n, k), np.float32)
        f = np.empty((n, k), np.uint8)
        acc = np.zeros(max(max_iters, 1), np.uint64)
        p = KoNndParams(k, delta, rho, max_iters, cap, seed)
        ds = _ds(x, metric)
        it = self.L.ko_nn_descent(C.byref(ds), C.byref(p), ids, d, f, acc)
        if it < 0:
            raise ValueError("nn_descent: invalid arguments")
        return ids, d, f, acc[:it].copy()

    def optimize_graph(self, ids, dists, x, out_degree, metric=0):
        n, k = ids.shape
        od = out_degree or k
        sg = np.empty((n, od), np.uint32)
        ds = _ds(x, metric)
        if self.L.ko_optimize_graph(np.ascontiguousarray(ids, np.uint32),
                                    np.ascontiguousarray(dists, np.float32), n, k,
                                    C.byref(ds), out_degree, sg):
            raise ValueError("optimize_graph: invalid arguments")
        return sg

    def ann_search(self, q, sg, v, k_s=10, beam_width=64, num_entry_points=16, max_hops=0,
                   seed=0, metric=0):
        nq = q.shape[0]
        sg = np.ascontiguousarray(sg, np.uint32)
        n, deg = sg.shape if sg.ndim == 2 else (v.shape[0], 0)
        ids = np.empty((nq, k_s), np.uint32)
        d = np.empty((nq, k_s), np.float32)
        hops = np.empty(nq, np.uint32)
        scored = np.empty(nq, np.uint32)
        p = KoSearchParams(k_s, beam_width, num_entry_points, max_hops, seed)
        qd, vd = _ds(q, metric), _ds(v, metric)
        sgf = sg.reshape(-1) if sg.size else np.zeros(1, np.uint32)
        if self.L.ko_ann_search(C.byref(qd), sgf, v.shape[0], deg, C.byref(vd), C.byref(p),
                                ids, d, hops, scored):
            raise ValueError("ann_search: invalid arguments")
        return ids, d, hops, scored

    def partition(self, n, ranks, seed):
        te = np.empty(n, np.uint32)
        off = np.empty(ranks + 1, np.uint64)
        if self.L.ko_partition(n, ranks, seed, te, off):
            raise ValueError("partition_dataset: need 1 <= P <= N")
        return te, off

    def merge_rows(self, a_ids, a_d, b_ids, b_d, k):
        oi = np.empty(k, np.uint32)
        od = np.empty(k, np.float32)
        c = self.L.ko_merge_rows_flat(np.ascontiguousarray(a_ids, np.uint32),
                                      np.ascontiguousarray(a_d, np.float32), len(a_ids),
                                      np.ascontiguousarray(b_ids, np.uint32),
                                      np.ascontiguousarray(b_d, np.float32), len(b_ids), k,
                                      oi, od)
        return oi[:c], od[:c]

    def check_invariants(self, ids, d, local=True):
        n, k = ids.shape
        return self.L.ko_check_graph_invariants(np.ascontiguousarray(ids, np.uint32),
                                                np.ascontiguousarray(d, np.float32), n, k,
                                                1 if local else 0)

    @staticmethod
    def refine_config(ranks, groups=2, k=32, k_s=0, out_degree=0, delta=1e-4, rho=0.5,
                      max_iters=100, cap=0, nn_seed=0, beam_width=64, num_entry_points=16,
                      max_hops=0, search_seed=0, skip_tree=False, max_concat_bytes=0, seed=0):
        return KoRefineConfig(ranks, groups, k, k_s, out_degree,
                              KoNndParams(k, delta, rho, max_iters, cap, nn_seed),
                              KoSearchParams(k_s or k, beam_width, num_entry_points, max_hops,
                                             search_seed),
                              1 if skip_tree else 0, max_concat_bytes, seed)

    def build_distributed(self, x, cfg):
        n = x.shape[0]
        ids = np.empty((n, cfg.k), np.uint32)
        d = np.empty((n, cfg.k), np.float32)
        ds = _ds(x)
        if self.L.ko_build_distributed(C.byref(ds), C.byref(cfg), ids, d):
            raise ValueError("build_distributed: invalid configuration")
        return ids, d

    def refine_from_local(self, x, cfg, to_external, offsets, ids, d, mode=0):
        ids = np.array(ids, np.uint32, copy=True)
        d = np.array(d, np.float32, copy=True)
        ds = _ds(x)
        if self.L.ko_refine_from_local(C.byref(ds), C.byref(cfg),
                                       np.ascontiguousarray(to_external, np.uint32),
                                       np.ascontiguousarray(offsets, np.uint64), ids, d, mode):
            raise ValueError("refine: invalid configuration")
        return ids, d

    def translate_to_external(self, to_external, ids, d):
        n, k = ids.shape
        oi = np.empty_like(ids)
        od = np.empty_like(d)
        self.L.ko_translate_to_external(np.ascontiguousarray(to_external, np.uint32), n, k,
                                        np.ascontiguousarray(ids), np.ascontiguousarray(d),
                                        oi, od)
        return oi, od

    def brute_force_rows(self, x, rows, k, metric=0):
        rows = np.ascontiguousarray(rows, np.uint64)
        ids = np.empty((len(rows), k), np.uint32)
        d = np.empty((len(rows), k), np.float32)
        ds = _ds(x, metric)
        if self.L.ko_brute_force_rows(C.byref(ds), rows, len(rows), k, ids, d):
            raise ValueError("brute_force_knng: k must be < N")
        return ids, d

    def recall(self, test_ids, truth_ids, k_eval):
        t = np.ascontiguousarray(test_ids, np.uint32)
        g = np.ascontiguousarray(truth_ids, np.uint32)
        return self.L.ko_recall_rows(t, t.shape[1], g, g.shape[1], t.shape[0], k_eval)


# --------------------------------------------------------------------------
# The reference itself
# --------------------------------------------------------------------------
class CRefineCfg(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("ranks", "groups", "k", "k_s", "out_degree")] + [
        ("delta", C.c_double), ("rho", C.c_double)] + [
        (n, C.c_uint64) for n in ("max_iters", "cap", "nn_seed", "beam_width",
                                  "num_entry_points", "max_hops", "search_seed", "skip_tree",
                                  "double_buffer", "max_concat_bytes", "seed")]


class RefError(RuntimeError):
    pass


class Ref:
    """The unmodified reference (oracle/_ref/libknng_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.kr_last_error.restype = C.c_char_p
        L.kr_hardware_concurrency.restype = C.c_uint
        L.kr_gen_random_dataset.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                            C.c_uint64, f32p]
        L.kr_l2.restype = C.c_float
        L.kr_l2.argtypes = [f32p, f32p, C.c_uint64]
        L.kr_cosine.restype = C.c_float
        L.kr_cosine.argtypes = [f32p, f32p, C.c_uint64]
        L.kr_set_metric.argtypes = [C.c_int]
        L.kr_init_random_graph.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_uint64, u32p, f32p, u8p]
        L.kr_sample_neighbors.argtypes = [u32p, f32p, u8p, C.c_uint64, C.c_uint64, C.c_double,
                                          C.c_uint64, C.c_uint64] + [u32p] * 8
        L.kr_nn_descent.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                    C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                    u32p, f32p, u8p, u64p, C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_double)]
        L.kr_optimize_graph.argtypes = [u32p, f32p, C.c_uint64, C.c_uint64, f32p, C.c_uint64,
                                        C.c_uint64, u32p, C.c_uint64]
        L.kr_ann_search.argtypes = [f32p, C.c_uint64, u32p, C.c_uint64, C.c_uint64, f32p,
                                    C.c_uint64] + [C.c_uint64] * 6 + [u32p, f32p, u32p, u32p]
        L.kr_partition.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                                   u64p, C.c_void_p]
        L.kr_merge_rows.restype = C.c_uint64
        L.kr_merge_rows.argtypes = [u32p, f32p, C.c_uint64, u32p, f32p, C.c_uint64, C.c_uint64,
                                    u32p, f32p]
        L.kr_brute_force.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                     u32p, f32p]
        L.kr_build_distributed.argtypes = [f32p, C.c_uint64, C.c_uint64, C.POINTER(CRefineCfg),
                                           u32p, f32p, f64p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64)]
        L.kr_build_local_graphs.argtypes = [f32p, C.c_uint64, C.c_uint64,
                                            C.POINTER(CRefineCfg), u32p, f32p]
        L.kr_refine_from_local.argtypes = [f32p, C.c_uint64, C.c_uint64, C.POINTER(CRefineCfg),
                                           u32p, f32p, C.c_int, C.c_void_p]
        L.kr_build_distributed_staged.argtypes = [f32p, C.c_uint64, C.c_uint64,
                                                  C.POINTER(CRefineCfg), u32p, f32p, f64p,
                                                  C.c_double]

    def _chk(self, rc):
        if rc == 1:
            raise ValueError(self.L.kr_last_error().decode())
        if rc:
            raise RefError(self.L.kr_last_error().decode())

    def hardware_concurrency(self):
        return int(self.L.kr_hardware_concurrency())

    def gen_random_dataset(self, n, dims, dist, seed, clusters=0):
        out = np.empty((n, dims), np.float32)
        self._chk(self.L.kr_gen_random_dataset(n, dims, DIST[dist], seed, clusters, out))
        return out

    def init_random_graph(self, x, k, seed):
        n, d = x.shape
        ids = np.empty((n, k), np.uint32)
        ds = np.empty((n, k), np.float32)
        f = np.empty((n, k), np.uint8)
        self._chk(self.L.kr_init_random_graph(x, n, d, k, seed, ids, ds, f))
        return ids, ds, f

    def sample_neighbors(self, ids, dists, flags, rho, seed, it):
        import math
        n, k = ids.shape
        b = int(math.ceil(rho * k))
        flags = np.array(flags, np.uint8, copy=True)
        nf = np.zeros((n, max(b, 1)), np.uint32)
        of = np.zeros((n, k), np.uint32)
        nr = np.zeros((n, max(b, 1)), np.uint32)
        orv = np.zeros((n, max(b, 1)), np.uint32)
        cnt = [np.zeros(n, np.uint32) for _ in range(4)]
        self._chk(self.L.kr_sample_neighbors(np.ascontiguousarray(ids, np.uint32),
                                             np.ascontiguousarray(dists, np.float32), flags,
                                             n, k, rho, seed, it, nf, cnt[0], of, cnt[1], nr,
                                             cnt[2], orv, cnt[3]))
        return dict(bound=b, flags=flags, new_fwd=(nf, cnt[0]), old_fwd=(of, cnt[1]),
                    new_rev=(nr, cnt[2]), old_rev=(orv, cnt[3]))

    def nn_descent(self, x, k, delta=1e-4, rho=0.5, max_iters=100, cap=0, seed=0, workers=1):
        n, dm = x.shape
        ids = np.empty((n, k), np.uint32)
        d = np.empty((n, k), np.float32)
        f = np.empty((n, k), np.uint8)
        acc = np.zeros(max(max_iters, 1), np.uint64)
        it = C.c_uint64(0)
        secs = C.c_double(0)
        self._chk(self.L.kr_nn_descent(x, n, dm, k, delta, rho, max_iters, cap, seed, workers,
                                       ids, d, f, acc, C.byref(it), C.byref(secs)))
        return ids, d, f, acc[:it.value].copy(), secs.value

    def optimize_graph(self, ids, dists, x, out_degree, workers=1):
        n, k = ids.shape
        od = out_degree or k
        sg = np.empty((n, od), np.uint32)
        self._chk(self.L.kr_optimize_graph(np.ascontiguousarray(ids, np.uint32),
                                           np.ascontiguousarray(dists, np.float32), n, k, x,
                                           x.shape[1], out_degree, sg, workers))
        return sg

    def ann_search(self, q, sg, v, k_s=10, beam_width=64, num_entry_points=16, max_hops=0,
                   seed=0, workers=1):
        nq, dm = q.shape
        sg = np.ascontiguousarray(sg, np.uint32)
        deg = sg.shape[1] if sg.ndim == 2 else 0
        ids = np.empty((nq, k_s), np.uint32)
        d = np.empty((nq, k_s), np.float32)
        hops = np.empty(nq, np.uint32)
        scored = np.empty(nq, np.uint32)
        sgf = sg.reshape(-1) if sg.size else np.zeros(1, np.uint32)
        self._chk(self.L.kr_ann_search(q, nq, sgf, v.shape[0], deg, v, dm, k_s, beam_width,
                                       num_entry_points, max_hops, seed, workers, ids, d, hops,
                                       scored))
        return ids, d, hops, scored

    def partition(self, x, ranks, seed, gather=False):
        n, dm = x.shape
        te = np.empty(n, np.uint32)
        off = np.empty(ranks + 1, np.uint64)
        loc = np.empty((n, dm), np.float32) if gather else None
        self._chk(self.L.kr_partition(x, n, dm, ranks, seed, te, off,
                                      loc.ctypes.data if gather else None))
        return (te, off, loc) if gather else (te, off)

    def set_metric(self, metric):
        """Metric of every dataset the shims build afterwards (0 l2, 1 cosine)."""
        self.L.kr_set_metric(metric)

    def cosine(self, a, b):
        return self.L.kr_cosine(np.ascontiguousarray(a, np.float32),
                                np.ascontiguousarray(b, np.float32), len(a))

    def merge_rows(self, a_ids, a_d, b_ids, b_d, k):
        oi = np.empty(k, np.uint32)
        od = np.empty(k, np.float32)
        c = self.L.kr_merge_rows(np.ascontiguousarray(a_ids, np.uint32),
                                 np.ascontiguousarray(a_d, np.float32), len(a_ids),
                                 np.ascontiguousarray(b_ids, np.uint32),
                                 np.ascontiguousarray(b_d, np.float32), len(b_ids), k, oi, od)
        return oi[:c], od[:c]

    def brute_force(self, x, k, workers=0):
        n, dm = x.shape
        ids = np.empty((n, k), np.uint32)
        d = np.empty((n, k), np.float32)
        self._chk(self.L.kr_brute_force(x, n, dm, k, workers, ids, d))
        return ids, d

    @staticmethod
    def refine_config(ranks, groups=2, k=32, k_s=0, out_degree=0, delta=1e-4, rho=0.5,
                      max_iters=100, cap=0, nn_seed=0, beam_width=64, num_entry_points=16,
                      max_hops=0, search_seed=0, skip_tree=False, double_buffer=False,
                      max_concat_bytes=0, seed=0):
        return CRefineCfg(ranks, groups, k, k_s, out_degree, delta, rho, max_iters, cap,
                          nn_seed, beam_width, num_entry_points, max_hops, search_seed,
                          1 if skip_tree else 0, 1 if double_buffer else 0, max_concat_bytes,
                          seed)

    def build_distributed(self, x, cfg):
        n, dm = x.shape
        ids = np.empty((n, cfg.k), np.uint32)
        d = np.empty((n, cfg.k), np.float32)
        ph = np.zeros(5, np.float64)
        gets = C.c_uint64(0)
        by = C.c_uint64(0)
        self._chk(self.L.kr_build_distributed(x, n, dm, C.byref(cfg), ids, d, ph,
                                              C.byref(gets), C.byref(by)))
        return ids, d, ph, gets.value, by.value

    def build_distributed_staged(self, x, cfg, watchdog_s=6 * 3600.0):
        """build_distributed with concurrent local builds and a long barrier
        watchdog (ref_capi.cpp kr_build_distributed_staged): the large-N
        reference runs.  Returns external-id graph + (local, tree, merge, flat) s."""
        n, dm = x.shape
        ids = np.empty((n, cfg.k), np.uint32)
        d = np.empty((n, cfg.k), np.float32)
        ph = np.zeros(4, np.float64)
        self._chk(self.L.kr_build_distributed_staged(x, n, dm, C.byref(cfg), ids, d, ph,
                                                     watchdog_s))
        return ids, d, ph

    def build_local_graphs(self, x, cfg):
        n, dm = x.shape
        ids = np.empty((n, cfg.k), np.uint32)
        d = np.empty((n, cfg.k), np.float32)
        self._chk(self.L.kr_build_local_graphs(x, n, dm, C.byref(cfg), ids, d))
        return ids, d

    def refine_from_local(self, x, cfg, ids, d, mode=0):
        n, dm = x.shape
        ids = np.array(ids, np.uint32, copy=True)
        d = np.array(d, np.float32, copy=True)
        self._chk(self.L.kr_refine_from_local(x, n, dm, C.byref(cfg), ids, d, mode, None))
        return ids, d
