"""Python mirror of the reference's public API over the B200 C-ABI.

Same names, argument meanings and error behaviour as the reference's C++
headers (/root/reference/proj/include/knng/*.hpp); every call goes through
``libknng_b200.so`` (include/knng_c.h).  There is no CPU fallback: importing
this module on a machine without the built library raises, and every compute
call raises ``CudaError`` without a GPU.

Arrays: numpy arrays are host buffers (copied to the GPU inside the call);
torch CUDA tensors are device buffers (used in place, outputs stay on the
device).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNNG_LIB") or os.path.join(_PKG, "libknng_b200.so")

# ---------------------------------------------------------------------------
# errors (status codes map 1:1 onto the reference's exceptions)
# ---------------------------------------------------------------------------


class KnngError(RuntimeError):
    pass


class InvalidArgument(KnngError, ValueError):
    """std::invalid_argument"""


class WorldError(KnngError):
    """WorldError distsim.hpp:19-21"""


class WorldAborted(WorldError):
    """WorldAborted distsim.hpp:24-26"""


class FormatError(KnngError):
    """FormatError evalio.hpp:14-16 / wire corruption"""


class LogicError(KnngError):
    """std::logic_error"""


class CudaError(KnngError):
    pass


_STATUS = {1: InvalidArgument, 2: WorldError, 3: WorldAborted, 4: FormatError, 5: LogicError,
           6: CudaError, 7: MemoryError, 8: KnngError}

MEM_HOST, MEM_DEVICE = 0, 1

# ---------------------------------------------------------------------------
# ABI structs (include/knng_c.h)
# ---------------------------------------------------------------------------


class _Dataset(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", C.c_uint64), ("dims", C.c_uint64),
                ("elem_kind", C.c_uint8), ("metric", C.c_uint8), ("mem", C.c_uint8),
                ("reserved", C.c_uint8)]


class _Graph(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("dists", C.c_void_p), ("flags", C.c_void_p),
                ("n", C.c_uint64), ("k", C.c_uint64), ("mem", C.c_uint8),
                ("reserved", C.c_uint8 * 7)]


class _NndParams(C.Structure):
    _fields_ = [("k", C.c_uint64), ("delta", C.c_double), ("rho", C.c_double),
                ("max_iters", C.c_uint64), ("candidate_capacity", C.c_uint64),
                ("seed", C.c_uint64), ("workers", C.c_uint64)]


class _NndStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("accepted_per_iter", C.c_void_p),
                ("accepted_cap", C.c_uint64), ("pairs", C.c_uint64),
                ("staged_rows", C.c_uint64), ("offers", C.c_uint64), ("join_ms", C.c_double),
                ("total_ms", C.c_double), ("join_launches", C.c_uint64),
                ("launches", C.c_uint64), ("offer_ms", C.c_double),
                ("stage_ms", C.c_double * 8), ("offers_per_iter", C.c_void_p),
                ("pairs_per_iter", C.c_void_p)]


class _SearchParams(C.Structure):
    _fields_ = [("k_s", C.c_uint64), ("beam_width", C.c_uint64),
                ("num_entry_points", C.c_uint64), ("max_hops", C.c_uint64),
                ("seed", C.c_uint64), ("workers", C.c_uint64)]


class _RefineConfig(C.Structure):
    _fields_ = [("ranks", C.c_uint64), ("groups", C.c_uint64), ("k", C.c_uint64),
                ("k_s", C.c_uint64), ("out_degree", C.c_uint64), ("nn", _NndParams),
                ("search", _SearchParams), ("skip_tree_phase", C.c_uint8),
                ("double_buffer", C.c_uint8), ("capture_snapshots", C.c_uint8),
                ("reserved", C.c_uint8 * 5), ("max_concat_bytes", C.c_uint64),
                ("seed", C.c_uint64)]


class _DistResult(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("local_s", "tree_s", "merge_s", "flat_s", "etc_s",
                                          "partition_s")] + [
        (n, C.c_uint64) for n in ("levels", "merge_epoch", "flat_epoch", "comm_gets",
                                  "comm_bytes", "search_hops", "search_scored", "nnd_pairs",
                                  "nnd_iterations", "num_snapshots")]


class _GetRecord(C.Structure):
    _fields_ = [("src", C.c_uint64), ("target", C.c_uint64), ("region", C.c_char * 16),
                ("bytes", C.c_uint64), ("epoch", C.c_uint64)]


_vp = C.c_void_p
_u64 = C.c_uint64
_SIGS = {
    "knng_abi_version": (C.c_int, []),
    "knng_ctx_create_on": (C.c_int, [_vp, C.c_int, _vp]),
    "knng_kernel_launches": (C.c_uint64, []),
    "knng_last_error": (C.c_char_p, []),
    "knng_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "knng_ctx_destroy": (None, [_vp]),
    "knng_ctx_device_count": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "knng_ctx_stream": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "knng_row_distances": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _vp, _vp, _u64, _vp]),
    "knng_merge_rows": (C.c_int, [_vp, C.c_int, _u64, _vp, _vp, _u64, _vp, _vp, _u64, _u64, _vp,
                                  _vp, _vp]),
    "knng_init_random_graph": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _u64, _u64,
                                         C.POINTER(_Graph)]),
    "knng_sample_neighbors": (C.c_int, [_vp, C.c_int, C.POINTER(_Graph), C.c_double, _u64, _u64]
                              + [_vp] * 8 + [C.POINTER(_u64)]),
    "knng_nn_descent": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), C.POINTER(_NndParams),
                                  C.POINTER(_Graph), C.POINTER(_NndStats)]),
    "knng_optimize_graph": (C.c_int, [_vp, C.c_int, C.POINTER(_Graph), C.POINTER(_Dataset), _u64,
                                      _vp]),
    "knng_ann_search": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _vp, _u64, _u64,
                                  C.POINTER(_Dataset), C.POINTER(_SearchParams), C.c_uint8, _vp,
                                  _vp, _vp, _vp]),
    "knng_ann_search_scored_ids": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _vp, _u64, _u64,
                                             C.POINTER(_Dataset), C.POINTER(_SearchParams),
                                             C.c_uint8, _vp, _vp, _vp, _vp, _vp, _u64]),
    "knng_partition": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _u64, _u64, C.c_uint8, _vp,
                                 _vp, _vp]),
    "knng_tree_levels": (C.c_int, [_u64, _u64, C.POINTER(_u64)]),
    "knng_tree_schedule": (C.c_int, [_u64, _u64, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64),
                                     _vp]),
    "knng_merge_results": (C.c_int, [_vp, C.c_int, C.POINTER(_Graph), _vp, _vp, _u64, _u64]),
    "knng_translate_to_external": (C.c_int, [_vp, C.c_int, _vp, _u64, _u64, _vp, _vp, _vp, _vp]),
    "knng_build_distributed": (C.c_int, [_vp, C.POINTER(_Dataset), C.POINTER(_RefineConfig),
                                         C.POINTER(_Graph), C.POINTER(_DistResult), _vp, _vp,
                                         _u64]),
    "knng_build_distributed_rank": (C.c_int, [_vp, C.c_int, _u64, _u64, _vp, _vp,
                                              C.POINTER(_Dataset), C.POINTER(_RefineConfig), _vp,
                                              _vp, _vp, C.c_int, C.POINTER(_u64),
                                              C.POINTER(_DistResult)]),
    "knng_vecs_shape": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_u64), C.POINTER(_u64)]),
    "knng_read_vecs": (C.c_int, [_vp, C.c_int, C.c_char_p, C.c_int, _vp, _u64, _u64, C.c_uint8]),
    "knng_write_vecs": (C.c_int, [C.c_char_p, C.c_int, _vp, _u64, _u64]),
    "knng_search_throughput_probe": (C.c_int, [_vp, C.c_int, _vp, _u64, C.POINTER(_Dataset),
                                               C.POINTER(_SearchParams), _vp]),
    "knng_refine": (C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(_RefineConfig), _vp, _vp, _vp,
                              C.c_int, C.POINTER(_DistResult)]),
    "knng_refine_phase": (C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(_RefineConfig), _vp, C.c_int,
                                    C.POINTER(_u64), _vp, _vp, _vp, _vp,
                                    C.POINTER(_DistResult)]),
    "knng_effective_groups": (C.c_int, [C.POINTER(_RefineConfig), _vp, _u64, C.POINTER(_u64)]),
    "knng_last_comm_log": (C.c_int, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "knng_brute_force": (C.c_int, [_vp, C.c_int, C.POINTER(_Dataset), _vp, _u64, _u64, C.c_uint8,
                                   _vp, _vp]),
    "knng_gen_random_dataset": (C.c_int, [_u64, _u64, C.c_int, _u64, _u64, _vp]),
    "knng_save_graph": (C.c_int, [C.POINTER(_Graph), C.c_char_p]),
    "knng_load_graph_header": (C.c_int, [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64)]),
    "knng_load_graph": (C.c_int, [C.c_char_p, C.POINTER(_Graph)]),
}

_LIB = None


def lib() -> C.CDLL:
    """The loaded C-ABI library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2605_27691_b200.build)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def exported_symbols() -> List[str]:
    return list(_SIGS)


def _check(rc: int):
    if rc != 0:
        msg = lib().knng_last_error().decode(errors="replace")
        raise _STATUS.get(rc, KnngError)(msg)


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


class Context:
    def __init__(self, num_devices: int = 0, devices: Optional[Sequence[int]] = None):
        h = C.c_void_p()
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            _check(lib().knng_ctx_create_on(arr, len(devices), C.byref(h)))
        else:
            _check(lib().knng_ctx_create(num_devices, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().knng_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def device_count(self) -> int:
        n = C.c_int(0)
        _check(lib().knng_ctx_device_count(self.h, C.byref(n)))
        return n.value

    def stream(self, device: int = 0) -> int:
        s = C.c_void_p()
        _check(lib().knng_ctx_stream(self.h, device, C.byref(s)))
        return s.value or 0


_CTX: Optional[Context] = None


def context(devices: Optional[Sequence[int]] = None) -> Context:
    """The process-wide context (created on first use: every visible GPU, or
    `devices` -- e.g. a torchrun rank's own GPU)."""
    global _CTX
    if _CTX is None:
        _CTX = Context(0, devices)
    return _CTX


# ---------------------------------------------------------------------------
# buffers
# ---------------------------------------------------------------------------


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _ptr(x) -> int:
    if x is None:
        return 0
    if _is_torch_cuda(x):
        assert x.is_contiguous()
        return x.data_ptr()
    assert isinstance(x, np.ndarray) and x.flags.c_contiguous, "C-contiguous array expected"
    return x.ctypes.data


def _mem(x) -> int:
    return MEM_DEVICE if _is_torch_cuda(x) else MEM_HOST


def _as_rows(x):
    """2-d f32 rows, or u8 rows kept as u8 (ElemKind::u8, core.hpp:14)."""
    if _is_torch_cuda(x):
        import torch
        assert x.dtype in (torch.float32, torch.uint8) and x.dim() == 2
        return x.contiguous()
    if isinstance(x, np.ndarray) and x.dtype == np.uint8:
        x = np.ascontiguousarray(x)
    else:
        x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise InvalidArgument("dataset must be a 2-D array (N x dims)")
    return x


def _is_u8(x) -> bool:
    if _is_torch_cuda(x):
        import torch
        return x.dtype == torch.uint8
    return getattr(x, "dtype", None) == np.uint8


def _metric_code(metric) -> int:
    """metric_from_string core.cpp:13-16 ("l2" | "cosine"; MetricKind core.hpp:15)."""
    if metric in (0, "l2"):
        return 0
    if metric in (1, "cosine"):
        return 1
    raise ValueError(f"unknown metric: {metric}")


def _dataset(x, metric: int = 0) -> _Dataset:
    return _Dataset(_ptr(x), x.shape[0], x.shape[1], 1 if _is_u8(x) else 0, metric, _mem(x), 0)


def _empty_like_mem(x, shape, dtype):
    if _is_torch_cuda(x):
        import torch
        tdt = {np.uint32: torch.int32, np.float32: torch.float32, np.uint8: torch.uint8,
               np.uint64: torch.int64}[dtype]
        return torch.empty(shape, dtype=tdt, device=x.device)
    return np.empty(shape, dtype=dtype)


def _itemsize(a) -> int:
    return a.element_size() if hasattr(a, "element_size") else a.itemsize


def _is_contiguous(a) -> bool:
    return a.is_contiguous() if hasattr(a, "is_contiguous") else a.flags["C_CONTIGUOUS"]


def _device_of(x) -> int:
    return x.device.index if _is_torch_cuda(x) else 0


# ---------------------------------------------------------------------------
# reference-shaped data classes
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class NnDescentParams:
    """nndescent.hpp:12-20"""
    k: int = 32
    delta: float = 0.0001
    rho: float = 0.5
    max_iters: int = 100
    candidate_capacity: int = 0
    seed: int = 0
    workers: int = 0

    def _c(self) -> _NndParams:
        return _NndParams(self.k, self.delta, self.rho, self.max_iters, self.candidate_capacity,
                          self.seed, self.workers)


@dataclasses.dataclass
class NnDescentStats:
    """nndescent.hpp:113-116 + device counters"""
    accepted_per_iter: List[int] = dataclasses.field(default_factory=list)
    iterations: int = 0
    pairs: int = 0
    staged_rows: int = 0
    offers: int = 0
    join_ms: float = 0.0
    offer_ms: float = 0.0
    total_ms: float = 0.0
    stage_ms: dict = dataclasses.field(default_factory=dict)
    offers_per_iter: List[int] = dataclasses.field(default_factory=list)
    pairs_per_iter: List[int] = dataclasses.field(default_factory=list)
    join_launches: int = 0
    launches: int = 0


@dataclasses.dataclass
class SearchParams:
    """annsearch.hpp:12-19"""
    k_s: int = 10
    beam_width: int = 64
    num_entry_points: int = 16
    max_hops: int = 0
    seed: int = 0
    workers: int = 0

    def _c(self) -> _SearchParams:
        return _SearchParams(self.k_s, self.beam_width, self.num_entry_points, self.max_hops,
                             self.seed, self.workers)


@dataclasses.dataclass
class RefineConfig:
    """refine.hpp:37-52"""
    ranks: int = 1
    groups: int = 2
    k: int = 32
    k_s: int = 0
    out_degree: int = 0
    nn: NnDescentParams = dataclasses.field(default_factory=NnDescentParams)
    search: SearchParams = dataclasses.field(default_factory=SearchParams)
    skip_tree_phase: bool = False
    double_buffer: bool = False
    max_concat_bytes: int = 0
    seed: int = 0
    capture_snapshots: bool = False

    def _c(self) -> _RefineConfig:
        c = _RefineConfig()
        c.ranks, c.groups, c.k, c.k_s, c.out_degree = (self.ranks, self.groups, self.k, self.k_s,
                                                       self.out_degree)
        c.nn = self.nn._c()
        c.nn.k = self.k
        c.search = self.search._c()
        c.skip_tree_phase = 1 if self.skip_tree_phase else 0
        c.double_buffer = 1 if self.double_buffer else 0
        c.capture_snapshots = 1 if self.capture_snapshots else 0
        c.max_concat_bytes = self.max_concat_bytes
        c.seed = self.seed
        return c


@dataclasses.dataclass
class KnnGraph:
    """core.hpp:156-179: N x k ids / dists (+ transient flags)."""
    ids: object
    dists: object
    flags: object = None

    @property
    def num_sources(self):
        return self.ids.shape[0]

    @property
    def k(self):
        return self.ids.shape[1]


@dataclasses.dataclass
class SearchResult:
    """annsearch.hpp:22-34 (+ SearchDiagnostics hops / scored counts)."""
    ids: object
    dists: object
    hops: object = None
    scored: object = None


@dataclasses.dataclass
class Partition:
    """refine.hpp:57-67 (locals concatenated in internal order)."""
    to_external: np.ndarray
    offsets: np.ndarray
    locals_concat: Optional[np.ndarray] = None

    def num_ranks(self):
        return len(self.offsets) - 1

    def size_of(self, r):
        return int(self.offsets[r + 1] - self.offsets[r])

    def local(self, r):
        return self.locals_concat[int(self.offsets[r]):int(self.offsets[r + 1])]


@dataclasses.dataclass
class GetRecord:
    """distsim.hpp:28-34"""
    src: int
    target: int
    region: str
    bytes: int
    epoch: int


@dataclasses.dataclass
class DistBuildResult:
    """refine.hpp:91-107"""
    graph: KnnGraph
    local_s: float = 0.0
    tree_s: float = 0.0
    merge_s: float = 0.0
    flat_s: float = 0.0
    etc_s: float = 0.0
    partition_s: float = 0.0
    levels: int = 0
    merge_epoch: int = 0
    flat_epoch: int = 0
    comm_log: List[GetRecord] = dataclasses.field(default_factory=list)
    search_hops: int = 0
    search_scored: int = 0
    nnd_pairs: int = 0
    nnd_iterations: int = 0
    snapshots: list = dataclasses.field(default_factory=list)  # (label, KnnGraph)

    @property
    def phases(self):
        return dict(local=self.local_s, tree=self.tree_s, merge=self.merge_s, flat=self.flat_s,
                    etc=self.etc_s)


# ---------------------------------------------------------------------------
# API (names follow the reference)
# ---------------------------------------------------------------------------


def abi_version() -> int:
    return lib().knng_abi_version()


def kernel_launches() -> int:
    """CUDA kernels launched by the library in this process so far."""
    return int(lib().knng_kernel_launches())


def gen_random_dataset(n: int, dims: int, dist: str = "uniform", seed: int = 0,
                       clusters: int = 0) -> np.ndarray:
    """evalio.cpp:242-272 (reference generator, bit-exact)."""
    code = {"uniform": 0, "gaussian": 1, "clustered": 2}[dist]
    out = np.empty((n, dims), np.float32) if n > 0 and dims > 0 else np.empty((1, 1), np.float32)
    _check(lib().knng_gen_random_dataset(n, dims, code, seed, clusters, out.ctypes.data))
    return out


def row_distances(x, i: Sequence[int], j: Sequence[int], device: int = 0,
                  metric: str = "l2") -> np.ndarray:
    """Dataset::row_distance core.hpp:84-95, batched, exact order."""
    x = _as_rows(x)
    i = np.ascontiguousarray(i, np.uint32)
    j = np.ascontiguousarray(j, np.uint32)
    out = np.empty(len(i), np.float32)
    ds = _dataset(x, _metric_code(metric))
    _check(lib().knng_row_distances(context().h, device, C.byref(ds), _ptr(i), _ptr(j), len(i),
                                    _ptr(out)))
    return out


def merge_rows_batch(a_ids, a_d, b_ids, b_d, k: int, device: int = 0):
    """merge_rows core.cpp:114-134 for every row of (rows x na) and (rows x nb)."""
    a_ids = np.ascontiguousarray(a_ids, np.uint32)
    a_d = np.ascontiguousarray(a_d, np.float32)
    b_ids = np.ascontiguousarray(b_ids, np.uint32)
    b_d = np.ascontiguousarray(b_d, np.float32)
    if a_ids.ndim == 1:
        a_ids, a_d, b_ids, b_d = a_ids[None], a_d[None], b_ids[None], b_d[None]
    rows, na = a_ids.shape
    nb = b_ids.shape[1]
    oi = np.empty((rows, k), np.uint32)
    od = np.empty((rows, k), np.float32)
    oc = np.empty(rows, np.uint32)
    _check(lib().knng_merge_rows(context().h, device, rows, _ptr(a_ids), _ptr(a_d), na,
                                 _ptr(b_ids), _ptr(b_d), nb, k, _ptr(oi), _ptr(od), _ptr(oc)))
    return oi, od, oc


def merge_rows(a_ids, a_d, b_ids, b_d, k: int):
    """Single-row merge_rows: returns (ids, dists) of the <= k merged entries."""
    oi, od, oc = merge_rows_batch(a_ids, a_d, b_ids, b_d, k)
    return oi[0, :oc[0]], od[0, :oc[0]]


def init_random_graph(x, k: int, seed: int, device: Optional[int] = None,
                      metric: str = "l2") -> KnnGraph:
    """nndescent.cpp:29-62"""
    x = _as_rows(x)
    dev = _device_of(x) if device is None else device
    n = x.shape[0]
    g = KnnGraph(_empty_like_mem(x, (n, k), np.uint32), _empty_like_mem(x, (n, k), np.float32),
                 _empty_like_mem(x, (n, k), np.uint8))
    cg = _Graph(_ptr(g.ids), _ptr(g.dists), _ptr(g.flags), n, k, _mem(x))
    ds = _dataset(x, _metric_code(metric))
    _check(lib().knng_init_random_graph(context().h, dev, C.byref(ds), k, seed, C.byref(cg)))
    return g


def sample_neighbors(graph: KnnGraph, rho: float, seed: int, iteration: int, device: int = 0):
    """nndescent.cpp:64-129 on a host graph; graph.flags consumed in place.
    Returns dict(bound, new_fwd, old_fwd, new_rev, old_rev) of per-point lists."""
    ids = np.ascontiguousarray(graph.ids, np.uint32)
    dists = np.ascontiguousarray(graph.dists, np.float32)
    assert isinstance(graph.flags, np.ndarray) and graph.flags.flags.c_contiguous
    n, k = ids.shape
    import math
    b = max(int(math.ceil(rho * k)), 1) if 0.0 < rho <= 1.0 else 1
    arrs = [np.zeros((n, b), np.uint32), np.zeros(n, np.uint32), np.zeros((n, k), np.uint32),
            np.zeros(n, np.uint32), np.zeros((n, b), np.uint32), np.zeros(n, np.uint32),
            np.zeros((n, b), np.uint32), np.zeros(n, np.uint32)]
    cg = _Graph(_ptr(ids), _ptr(dists), _ptr(graph.flags), n, k, MEM_HOST)
    bound = C.c_uint64(0)
    _check(lib().knng_sample_neighbors(context().h, device, C.byref(cg), rho, seed, iteration,
                                       *[_ptr(a) for a in arrs], C.byref(bound)))

    def lists(mat, cnt):
        return [mat[p, :cnt[p]].copy() for p in range(n)]

    return dict(bound=bound.value, new_fwd=lists(arrs[0], arrs[1]),
                old_fwd=lists(arrs[2], arrs[3]), new_rev=lists(arrs[4], arrs[5]),
                old_rev=lists(arrs[6], arrs[7]),
                raw=dict(new_fwd=(arrs[0], arrs[1]), old_fwd=(arrs[2], arrs[3]),
                         new_rev=(arrs[4], arrs[5]), old_rev=(arrs[6], arrs[7])))


def nn_descent(x, params: Optional[NnDescentParams] = None, stats: Optional[NnDescentStats] = None,
               device: Optional[int] = None, metric: str = "l2", out: Optional[KnnGraph] = None,
               **kw) -> KnnGraph:
    """nn_descent nndescent.cpp:225-259 (lock-free NN-Descent on the B200).

    `out`: a KnnGraph to write into (n x k ids u32 / dists f32 / flags u8, or
    flags None), on the same side as `x` -- e.g. pinned host tensors reused
    across calls, so the graph comes back by a direct DMA."""
    p = params or NnDescentParams(**kw)
    x = _as_rows(x)
    dev = _device_of(x) if device is None else device
    n = x.shape[0]
    k = p.k
    if k <= 0 or n <= k:
        raise InvalidArgument("init_random_graph: need 1 <= k < N")
    if out is None:
        g = KnnGraph(_empty_like_mem(x, (n, k), np.uint32),
                     _empty_like_mem(x, (n, k), np.float32),
                     _empty_like_mem(x, (n, k), np.uint8))
    else:
        g = out
        for a, isz in ((g.ids, 4), (g.dists, 4), (g.flags, 1)):
            if a is None and isz == 1:
                continue
            if tuple(a.shape) != (n, k) or _mem(a) != _mem(x) or _itemsize(a) != isz or \
                    not _is_contiguous(a):
                raise InvalidArgument("nn_descent: out must be contiguous n x k on x's side")
    cg = _Graph(_ptr(g.ids), _ptr(g.dists), _ptr(g.flags), n, k, _mem(x))
    ds = _dataset(x, _metric_code(metric))
    cp = p._c()
    acc = np.zeros(max(p.max_iters, 1), np.uint64)
    st = _NndStats()
    st.accepted_per_iter = acc.ctypes.data
    st.accepted_cap = len(acc)
    off_it = np.zeros(max(p.max_iters, 1), np.uint64)
    pair_it = np.zeros(max(p.max_iters, 1), np.uint64)
    st.offers_per_iter = off_it.ctypes.data
    st.pairs_per_iter = pair_it.ctypes.data
    _check(lib().knng_nn_descent(context().h, dev, C.byref(ds), C.byref(cp), C.byref(cg),
                                 C.byref(st) if stats is not None else None))
    if stats is not None:
        stats.iterations = st.iterations
        stats.accepted_per_iter = [int(v) for v in acc[:st.iterations]]
        stats.pairs, stats.staged_rows, stats.offers = st.pairs, st.staged_rows, st.offers
        stats.join_ms, stats.total_ms, stats.offer_ms = st.join_ms, st.total_ms, st.offer_ms
        stats.offers_per_iter = [int(v) for v in off_it[:st.iterations]]
        stats.pairs_per_iter = [int(v) for v in pair_it[:st.iterations]]
        stats.stage_ms = dict(zip(("init", "sample", "lists", "join", "offer", "apply",
                                   "readback"), list(st.stage_ms)[:7]))
        stats.join_launches, stats.launches = st.join_launches, st.launches
    return g


def optimize_graph(graph: KnnGraph, x, out_degree: int = 0, workers: int = 0,
                   device: Optional[int] = None, metric: str = "l2"):
    """graphopt.cpp:24-105 -> n x out_degree search-graph ids."""
    x = _as_rows(x)
    dev = _device_of(x) if device is None else device
    n, k = graph.ids.shape
    od = out_degree or k
    mem = _mem(graph.ids)
    if mem == MEM_HOST:
        ids = np.ascontiguousarray(graph.ids, np.uint32)
        dists = np.ascontiguousarray(graph.dists, np.float32)
    else:
        ids, dists = graph.ids.contiguous(), graph.dists.contiguous()
    if od > k:
        raise InvalidArgument("optimize_graph: out_degree must be <= k")
    sg = _empty_like_mem(graph.ids, (n, od), np.uint32)
    cg = _Graph(_ptr(ids), _ptr(dists), None, n, k, mem)
    ds = _dataset(x, _metric_code(metric))
    _check(lib().knng_optimize_graph(context().h, dev, C.byref(cg), C.byref(ds), out_degree,
                                     _ptr(sg)))
    return sg


def ann_search(queries, sgraph, vectors, params: Optional[SearchParams] = None,
               diagnostics: bool = False, device: Optional[int] = None, metric: str = "l2",
               **kw) -> SearchResult:
    """annsearch.cpp:50-129 (bit-identical to the reference's greedy search)."""
    p = params or SearchParams(**kw)
    q = _as_rows(queries)
    v = _as_rows(vectors)
    dev = _device_of(q) if device is None else device
    mem = _mem(q)
    if mem == MEM_HOST:
        sg = np.ascontiguousarray(sgraph, np.uint32)
    else:
        sg = sgraph.contiguous()
    n_sg = sg.shape[0] if sg.ndim == 2 else 0
    deg = sg.shape[1] if sg.ndim == 2 else 0
    nq = q.shape[0]
    out_i = _empty_like_mem(q, (nq, p.k_s), np.uint32)
    out_d = _empty_like_mem(q, (nq, p.k_s), np.float32)
    hops = _empty_like_mem(q, (nq,), np.uint32) if diagnostics else None
    scored = _empty_like_mem(q, (nq,), np.uint32) if diagnostics else None
    qd, vd = _dataset(q, _metric_code(metric)), _dataset(v, _metric_code(metric))
    if sg.size == 0 and mem == MEM_HOST:
        sg = np.zeros(1, np.uint32)
    _check(lib().knng_ann_search(context().h, dev, C.byref(qd), _ptr(sg), n_sg, deg, C.byref(vd),
                                 C.byref(p._c()), mem, _ptr(out_i), _ptr(out_d), _ptr(hops),
                                 _ptr(scored)))
    return SearchResult(out_i, out_d, hops, scored)


_VECS = {"f32": (0, np.float32), "u8": (1, np.uint8), "i32": (2, np.int32)}


def vecs_shape(path, kind: str = "f32"):
    """(rows, dims) of a .fvecs/.bvecs/.ivecs file, every row validated
    (evalio.cpp:31-66 checks; FormatError on malformed input)."""
    code, _ = _VECS[kind]
    r, d = _u64(0), _u64(0)
    _check(lib().knng_vecs_shape(os.fsencode(path), code, C.byref(r), C.byref(d)))
    return r.value, d.value


def read_vecs(path, kind: str = "f32", device: Optional[int] = None):
    """read_vecs / read_ivecs evalio.cpp:31-100 -> numpy (rows x dims), or a
    CUDA tensor on `device` (streamed through pinned buffers)."""
    code, dt = _VECS[kind]
    rows, dims = vecs_shape(path, kind)
    if device is None:
        out = np.empty((rows, dims), dt)
        mem = MEM_HOST
    else:
        import torch
        tdt = {np.float32: torch.float32, np.uint8: torch.uint8, np.int32: torch.int32}[dt]
        out = torch.empty((rows, dims), dtype=tdt, device=f"cuda:{device}")
        mem = MEM_DEVICE
    _check(lib().knng_read_vecs(context().h if device is not None else None,
                                device or 0, os.fsencode(path), code, _ptr(out), rows, dims, mem))
    return out


def write_vecs(path, x, kind: Optional[str] = None):
    """write_vecs / write_ivecs evalio.cpp:68-123 (bit-exact round trip)."""
    x = np.ascontiguousarray(x)
    kind = kind or {np.dtype(np.float32): "f32", np.dtype(np.uint8): "u8",
                    np.dtype(np.int32): "i32"}[x.dtype]
    code, dt = _VECS[kind]
    x = np.ascontiguousarray(x, dt)
    _check(lib().knng_write_vecs(os.fsencode(path), code, _ptr(x), x.shape[0], x.shape[1]))


class _ThroughputCase(C.Structure):
    _fields_ = [("source_count", C.c_uint64), ("sg_ids", C.c_void_p), ("sg_n", C.c_uint64),
                ("degree", C.c_uint64), ("vectors", C.POINTER(_Dataset)), ("sg_mem", C.c_uint8)]


class _ThroughputRow(C.Structure):
    _fields_ = [("source_count", C.c_uint64), ("num_queries", C.c_uint64),
                ("seconds", C.c_double), ("qps", C.c_double)]


@dataclasses.dataclass
class ThroughputRow:
    """annsearch.hpp:59-64"""
    source_count: int
    num_queries: int
    seconds: float
    qps: float


def search_throughput_probe(cases, queries, params: "SearchParams",
                            device: Optional[int] = None,
                            metric: str = "l2") -> List[ThroughputRow]:
    """annsearch.cpp:131-155: `cases` = [(source_count, sgraph, vectors), ...]
    in ascending source_count; seconds are device time of each search."""
    q = _as_rows(queries)
    dev = _device_of(q) if device is None else device
    keep = []
    arr = (_ThroughputCase * max(1, len(cases)))()
    for i, (count, sg, vec) in enumerate(cases):
        v = _as_rows(vec)
        sgm = sg if _is_torch_cuda(sg) else np.ascontiguousarray(sg, np.uint32)
        ds = _dataset(v, _metric_code(metric))
        keep += [v, sgm, ds]
        arr[i] = _ThroughputCase(count, _ptr(sgm), sgm.shape[0], sgm.shape[1], C.pointer(ds),
                                 _mem(sgm))
    rows = (_ThroughputRow * max(1, len(cases)))()
    qd = _dataset(q, _metric_code(metric))
    _check(lib().knng_search_throughput_probe(context().h, dev, arr, len(cases), C.byref(qd),
                                              C.byref(params._c()), rows))
    return [ThroughputRow(rows[i].source_count, rows[i].num_queries, rows[i].seconds,
                          rows[i].qps) for i in range(len(cases))]


def partition_dataset(x, ranks: int, seed: int, gather: bool = True, device: int = 0) -> Partition:
    """refine.cpp:86-126 (bit-exact permutation computed on the GPU)."""
    x = _as_rows(x)
    n = x.shape[0]
    te = np.empty(max(n, 1), np.uint32)
    off = np.empty(ranks + 1, np.uint64)
    host_gather = gather and isinstance(x, np.ndarray)
    u8 = _is_u8(x)
    # f32 rows are gathered by the library; u8 rows are gathered here (an
    # exact byte copy keeps ElemKind::u8, refine.cpp:116-124)
    loc = np.empty_like(x) if (host_gather and not u8) else None
    ds = _dataset(x)
    _check(lib().knng_partition(context().h, device, C.byref(ds), ranks, seed, MEM_HOST,
                                _ptr(te), _ptr(off), _ptr(loc)))
    if host_gather and u8:
        loc = x[te[:n].astype(np.int64)]
    return Partition(te[:n], off, loc)


def tree_levels(ranks: int, groups: int) -> int:
    out = C.c_uint64(0)
    _check(lib().knng_tree_levels(ranks, groups, C.byref(out)))
    return out.value


def tree_schedule(ranks: int, groups: int, rank: int, level: int):
    """refine.cpp:134-149 -> (group_lo, group_hi, partners)"""
    lo, hi = C.c_uint64(0), C.c_uint64(0)
    partners = np.zeros(max(ranks, 1), np.uint64)
    _check(lib().knng_tree_schedule(ranks, groups, rank, level, C.byref(lo), C.byref(hi),
                                    _ptr(partners)))
    return lo.value, hi.value, [int(v) for v in partners[:1 << level]]


def merge_results_into(graph: KnnGraph, res_ids, res_dists, id_base: int, device: int = 0):
    """refine.cpp:49-60 (in place on a host graph)."""
    ids = np.ascontiguousarray(graph.ids, np.uint32)
    d = np.ascontiguousarray(graph.dists, np.float32)
    ri = np.ascontiguousarray(res_ids, np.uint32)
    rd = np.ascontiguousarray(res_dists, np.float32)
    n, k = ids.shape
    cg = _Graph(_ptr(ids), _ptr(d), None, n, k, MEM_HOST)
    _check(lib().knng_merge_results(context().h, device, C.byref(cg), _ptr(ri), _ptr(rd),
                                    ri.shape[1], id_base))
    graph.ids, graph.dists = ids, d
    return graph


def translate_to_external(to_external, ids, dists, device: int = 0):
    """refine.cpp:395-416"""
    te = np.ascontiguousarray(to_external, np.uint32)
    ids = np.ascontiguousarray(ids, np.uint32)
    dists = np.ascontiguousarray(dists, np.float32)
    n, k = ids.shape
    oi, od = np.empty_like(ids), np.empty_like(dists)
    _check(lib().knng_translate_to_external(context().h, device, _ptr(te), n, k, _ptr(ids),
                                            _ptr(dists), _ptr(oi), _ptr(od)))
    return oi, od


def _comm_log() -> List[GetRecord]:
    cnt = C.c_uint64(0)
    _check(lib().knng_last_comm_log(context().h, None, 0, C.byref(cnt)))
    recs = (_GetRecord * max(cnt.value, 1))()
    _check(lib().knng_last_comm_log(context().h, recs, cnt.value, C.byref(cnt)))
    return [GetRecord(r.src, r.target, r.region.decode(), r.bytes, r.epoch)
            for r in recs[:cnt.value]]


def _dist_result(graph, r: _DistResult) -> DistBuildResult:
    return DistBuildResult(graph=graph, local_s=r.local_s, tree_s=r.tree_s, merge_s=r.merge_s,
                           flat_s=r.flat_s, etc_s=r.etc_s, partition_s=r.partition_s,
                           levels=r.levels, merge_epoch=r.merge_epoch, flat_epoch=r.flat_epoch,
                           comm_log=_comm_log(), search_hops=r.search_hops,
                           search_scored=r.search_scored, nnd_pairs=r.nnd_pairs,
                           nnd_iterations=r.nnd_iterations)


def build_distributed(x, cfg: RefineConfig, metric: str = "l2") -> DistBuildResult:
    """refine.cpp:504-586: partition -> local NN-Descent -> tree refine ->
    grouped merge -> flat refine -> external ids, on the context's GPUs
    (rank r on GPU r mod #GPUs)."""
    x = _as_rows(x)
    n = x.shape[0]
    k = cfg.k
    out = KnnGraph(_empty_like_mem(x, (n, k), np.uint32), _empty_like_mem(x, (n, k), np.float32))
    cg = _Graph(_ptr(out.ids), _ptr(out.dists), None, n, k, _mem(x))
    ds = _dataset(x, _metric_code(metric))
    res = _DistResult()
    cc = cfg._c()
    nsnap = 0
    snap_i = snap_d = None
    if cfg.capture_snapshots:
        nsnap = 2 + 8  # local + up to 8 tree levels + flat
        snap_i = np.zeros((nsnap, n, k), np.uint32)
        snap_d = np.zeros((nsnap, n, k), np.float32)
    _check(lib().knng_build_distributed(context().h, C.byref(ds), C.byref(cc), C.byref(cg),
                                        C.byref(res), _ptr(snap_i), _ptr(snap_d), nsnap))
    out_r = _dist_result(out, res)
    if cfg.capture_snapshots:
        levels = res.levels
        labels = ["local"] + [f"tree_level_{i}" for i in range(levels)] + (
            ["flat"] if cfg.ranks > 1 else [])
        out_r.snapshots = [(lab, KnnGraph(snap_i[s], snap_d[s]))
                           for s, lab in enumerate(labels[:res.num_snapshots])]
    return out_r


# knng_allgather_fn: int (*)(void* user, const void* in, uint64_t bytes, void* out)
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


def torch_allgather(group=None):
    """Host transport for build_distributed_rank over torch.distributed: an
    all-gather of CPU byte tensors (use a gloo group; the default group if it
    is gloo)."""
    import torch
    import torch.distributed as dist

    def fn(inp, nbytes):
        buf = torch.frombuffer(bytearray(C.string_at(inp, nbytes)), dtype=torch.uint8)
        outs = [torch.empty(nbytes, dtype=torch.uint8)
                for _ in range(dist.get_world_size(group))]
        dist.all_gather(outs, buf, group=group)
        return torch.cat(outs).numpy().tobytes()
    return fn


@dataclasses.dataclass
class RankBuildResult(DistBuildResult):
    """This rank's part of build_distributed: graph rows + their external ids."""
    rows: Optional[object] = None


def build_distributed_rank(x, cfg: RefineConfig, rank: int, world_size: int,
                           allgather=None, device: Optional[int] = None,
                           metric: str = "l2", out=None) -> RankBuildResult:
    """One rank of build_distributed (refine.cpp:504-586) in this process, for
    one process per GPU.  Collective over `allgather(bytes_in, nbytes) ->
    bytes_out` (default: torch_allgather() on the default group).  Every rank
    passes the same full dataset; returns the rank's rows (external ids) and
    their external row ids (graph.ids[i] is the neighbor list of row rows[i]).
    `out`: (ids u32 [cap, k], dists f32 [cap, k], rows u32 [cap]) on x's side,
    cap = ceil(n / world_size) -- e.g. pinned host buffers reused across calls."""
    x = _as_rows(x)
    n = x.shape[0]
    k = cfg.k
    cap = -(-n // world_size)
    if out is None:
        out_i = _empty_like_mem(x, (cap, k), np.uint32)
        out_d = _empty_like_mem(x, (cap, k), np.float32)
        out_r = _empty_like_mem(x, (cap,), np.uint32)
    else:
        out_i, out_d, out_r = out
        for a, shape, isz in ((out_i, (cap, k), 4), (out_d, (cap, k), 4), (out_r, (cap,), 4)):
            if tuple(a.shape) != shape or _mem(a) != _mem(x) or _itemsize(a) != isz or \
                    not _is_contiguous(a):
                raise InvalidArgument("build_distributed_rank: out must be contiguous "
                                      "[cap, k] / [cap, k] / [cap] on x's side")
    ag = allgather or torch_allgather()
    err = []

    def thunk(user, inp, nbytes, out):
        try:
            data = ag(inp, nbytes)
            C.memmove(out, data, len(data))
            return 0
        except Exception as e:  # reported as KNNG_EWORLD by the library
            err.append(e)
            return 1
    cb = _ALLGATHER_FN(thunk)
    ds = _dataset(x, _metric_code(metric))
    res = _DistResult()
    cc = cfg._c()
    rows = _u64(0)
    dev = device if device is not None else _device_of(x)
    rc = lib().knng_build_distributed_rank(context().h, dev, rank, world_size, cb, None,
                                           C.byref(ds), C.byref(cc), _ptr(out_i), _ptr(out_d),
                                           _ptr(out_r), _mem(x), C.byref(rows), C.byref(res))
    if rc != 0 and err:
        raise WorldError(f"host transport failed: {err[0]!r}")
    _check(rc)
    m = rows.value
    r = _dist_result(KnnGraph(out_i[:m], out_d[:m]), res)
    return RankBuildResult(**{f.name: getattr(r, f.name) for f in dataclasses.fields(r)},
                           rows=out_r[:m])


def refine(x_perm, cfg: RefineConfig, offsets, ids, dists, mode: int = 0) -> DistBuildResult:
    """World-level drivers from local graphs: mode 0 = binary_tree_refine ->
    grouped_merge -> flat_refine, mode 1 = all_to_all_refine (refine.hpp:117-136)."""
    x = np.ascontiguousarray(x_perm, np.float32)
    ids = np.array(ids, np.uint32, copy=True)
    dists = np.array(dists, np.float32, copy=True)
    off = np.ascontiguousarray(offsets, np.uint64)
    res = _DistResult()
    cc = cfg._c()
    _check(lib().knng_refine(context().h, _ptr(x), x.shape[0], x.shape[1], C.byref(cc),
                             _ptr(off), _ptr(ids), _ptr(dists), mode, C.byref(res)))
    return _dist_result(KnnGraph(ids, dists), res)


def effective_groups(cfg: RefineConfig, offsets, dims: int) -> int:
    """refine.cpp:160-183: M, or P when the tree phase is skipped."""
    off = np.ascontiguousarray(offsets, np.uint64)
    cc = cfg._c()
    cc.ranks = len(off) - 1
    out = _u64(0)
    _check(lib().knng_effective_groups(C.byref(cc), _ptr(off), dims, C.byref(out)))
    return out.value


REFINE_PHASES = {"all_to_all_refine": 1, "binary_tree_refine": 2, "grouped_merge": 3,
                 "flat_refine": 4}


def refine_phase(x_perm, cfg: RefineConfig, offsets, ids, dists, phase: str, epoch: int = 0,
                 group_graphs=None):
    """One world-level phase driver (refine.hpp:117-136) on a world at `epoch`.
    Returns (graph, group search graphs (grouped_merge) or None, epoch after,
    DistBuildResult with the phase's gets).  group_graphs (flat_refine): the
    per-rank blocks grouped_merge returned."""
    x = np.ascontiguousarray(x_perm, np.float32)
    ids = np.array(ids, np.uint32, copy=True)
    dists = np.array(dists, np.float32, copy=True)
    off = np.ascontiguousarray(offsets, np.uint64)
    cc = cfg._c()
    cc.ranks = len(off) - 1
    ph = REFINE_PHASES[phase]
    od = cfg.out_degree or cfg.k
    g = effective_groups(cfg, off, x.shape[1])
    gsz = (len(off) - 1) // g
    blocks = [int(off[(r // gsz) * gsz + gsz] - off[(r // gsz) * gsz]) * od
              for r in range(len(off) - 1)]
    sg_out = np.zeros(sum(blocks), np.uint32) if ph == 3 else None
    sg_in = (np.ascontiguousarray(np.concatenate([np.asarray(b, np.uint32).ravel()
                                                  for b in group_graphs]))
             if ph == 4 else None)
    ep = _u64(epoch)
    res = _DistResult()
    _check(lib().knng_refine_phase(context().h, _ptr(x), x.shape[0], x.shape[1], C.byref(cc),
                                   _ptr(off), ph, C.byref(ep), _ptr(ids), _ptr(dists),
                                   _ptr(sg_in) if sg_in is not None else None,
                                   _ptr(sg_out) if sg_out is not None else None, C.byref(res)))
    sgs = None
    if sg_out is not None:
        at = np.cumsum([0] + blocks)
        sgs = [sg_out[at[r]:at[r + 1]].reshape(-1, od) for r in range(len(blocks))]
    return KnnGraph(ids, dists), sgs, ep.value, _dist_result(KnnGraph(ids, dists), res)


def brute_force_knng(x, k: int, rows=None, device: Optional[int] = None, metric: str = "l2"):
    """evalio.cpp:125-147 for `rows` (default all) -> (ids, dists) q x k."""
    x = _as_rows(x)
    dev = _device_of(x) if device is None else device
    n = x.shape[0]
    if rows is None:
        rows = np.arange(n, dtype=np.uint64)
    rows = np.ascontiguousarray(rows, np.uint64)
    q = len(rows)
    oi = _empty_like_mem(x, (q, k), np.uint32)
    od = _empty_like_mem(x, (q, k), np.float32)
    ds = _dataset(x, _metric_code(metric))
    _check(lib().knng_brute_force(context().h, dev, C.byref(ds), _ptr(rows), q, k, _mem(x),
                                  _ptr(oi), _ptr(od)))
    return oi, od


def recall_at_k(test_ids, truth_ids, k_eval: int) -> float:
    """evalio.cpp:170-192 (host, measurement only)."""
    t = np.asarray(test_ids)[:, :k_eval]
    g = np.asarray(truth_ids)[:, :k_eval]
    hits = 0
    for r in range(t.shape[0]):
        hits += len(np.intersect1d(t[r], g[r], assume_unique=False))
    return hits / float(t.shape[0] * k_eval)


def distance_threshold_recall(test_dists, ref_dists, k_eval: int) -> float:
    """evalio.cpp:199-215 (host, measurement only): per row, the share of the
    first k_eval test distances <= the reference row's k_eval-th distance,
    averaged over rows in row order."""
    t = np.asarray(test_dists, np.float32)
    g = np.asarray(ref_dists, np.float32)
    if k_eval == 0 or k_eval > t.shape[1] or k_eval > g.shape[1]:
        raise InvalidArgument("distance_threshold_recall: k_eval out of range")
    if t.shape[0] != g.shape[0]:
        raise InvalidArgument("distance_threshold_recall: graphs not comparable")
    thr = g[:, k_eval - 1:k_eval]
    # rows are sorted, so the leading run <= thr is the count of entries <= thr
    # only if the run is contiguous; count the run exactly as the reference does
    run = np.cumprod(t <= thr, axis=1).sum(axis=1)
    total = 0.0
    for c in np.minimum(run, k_eval):
        total += float(c) / float(k_eval)
    return total / float(t.shape[0])


def save_graph(graph: KnnGraph, path: str):
    """evalio.cpp:274-276 (wire region, wire.cpp:76-82)."""
    ids = np.ascontiguousarray(graph.ids, np.uint32)
    d = np.ascontiguousarray(graph.dists, np.float32)
    cg = _Graph(_ptr(ids), _ptr(d), None, ids.shape[0], ids.shape[1], MEM_HOST)
    _check(lib().knng_save_graph(C.byref(cg), os.fsencode(path)))


def load_graph(path: str) -> KnnGraph:
    n, k = C.c_uint64(0), C.c_uint64(0)
    _check(lib().knng_load_graph_header(os.fsencode(path), C.byref(n), C.byref(k)))
    ids = np.empty((n.value, k.value), np.uint32)
    d = np.empty((n.value, k.value), np.float32)
    cg = _Graph(_ptr(ids), _ptr(d), None, n.value, k.value, MEM_HOST)
    _check(lib().knng_load_graph(os.fsencode(path), C.byref(cg)))
    return KnnGraph(ids, d)
