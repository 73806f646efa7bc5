"""Thin ctypes binding over libvdmc.so (include/vdmc.h).  Argument marshalling only:
every step of the counting path runs in the library's CUDA kernels.  PyTorch supplies
device memory, streams and process groups.  There is no CPU fallback: if the library or a
CUDA device is missing, these functions raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libvdmc.so")   # VDMC_LIB (read at first load) selects an A/B build

VDMC_OK = 0
STATUS = {1: "VDMC_EINVAL", 2: "VDMC_ERANGE", 3: "VDMC_ESELFLOOP", 4: "VDMC_EASYM",
          5: "VDMC_EORDER", 6: "VDMC_EK", 7: "VDMC_ENOMEM", 8: "VDMC_ECUDA", 9: "VDMC_ENODEV",
          10: "VDMC_ENCCL"}

# Every symbol include/vdmc.h declares (tests check the .so exports exactly these)
EXPORTS = ["vdmc_build_graph_edges", "vdmc_build_graph", "vdmc_symmetrize", "vdmc_free_host", "vdmc_count",
           "vdmc_count_kind", "vdmc_count_ex", "vdmc_count_edges", "vdmc_get_edges", "vdmc_plan", "vdmc_split_costs", "vdmc_root_range",
           "vdmc_num_classes", "vdmc_class_ids", "vdmc_num_classes_kind", "vdmc_class_ids_kind", "vdmc_class_ids32",
           "vdmc_get_info", "vdmc_get_order", "vdmc_kernel_launches", "vdmc_comm_unique_id",
           "vdmc_comm_init", "vdmc_comm_free", "vdmc_count_distributed", "vdmc_free_graph", "vdmc_trim",
           "vdmc_last_error"]


class VdmcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Range(ctypes.Structure):
    _fields_ = [("task_lo", ctypes.c_int64), ("task_hi", ctypes.c_int64)]


class Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("arcs", ctypes.c_int64),
                ("ntasks", ctypes.c_int64), ("max_degree", ctypes.c_int64), ("device", ctypes.c_int32),
                ("build_ms", ctypes.c_float)]


class CountOptions(ctypes.Structure):
    """vdmc_count_options (include/vdmc.h); every path option is result-preserving."""
    _fields_ = [("kind", ctypes.c_int32), ("star_block", ctypes.c_int32), ("cross_block", ctypes.c_int32),
                ("heavy_global", ctypes.c_int32), ("force_big", ctypes.c_int32), ("layered", ctypes.c_int32),
                ("acc64", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("ca_capacity", ctypes.c_int64), ("timings_ms", ctypes.POINTER(ctypes.c_float))]


OPTION_KEYS = ("star_block", "cross_block", "heavy_global", "force_big", "ca_capacity", "layered", "acc64")


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def lib():
    """Load libvdmc.so (built by __graft_entry__.build()); raise if it is missing."""
    global _lib, LIB_PATH
    if _lib is None:
        LIB_PATH = os.environ.get("VDMC_LIB") or LIB_PATH
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libvdmc.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "vdmc_build_graph_edges": (_i32, [_i64, _i64, _vp, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp,
                                              ctypes.POINTER(_vp)]),
            "vdmc_build_graph": (_i32, [_i64, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp)]),
            "vdmc_symmetrize": (_i32, [_i64, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                       ctypes.POINTER(_vp)]),
            "vdmc_free_host": (None, [_vp]),
            "vdmc_count": (_i32, [_vp, ctypes.c_int, _vp, ctypes.POINTER(Range), _vp]),
            "vdmc_count_kind": (_i32, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(Range), _vp]),
            "vdmc_count_ex": (_i32, [_vp, ctypes.c_int, _vp, ctypes.POINTER(Range), ctypes.POINTER(CountOptions),
                                     _vp]),
            "vdmc_root_range": (_i32, [_vp, _i64, _i64, ctypes.POINTER(Range)]),
            "vdmc_count_edges": (_i32, [_vp, ctypes.c_int, _vp, ctypes.POINTER(Range),
                                        ctypes.POINTER(CountOptions), _vp]),
            "vdmc_get_edges": (_i32, [_vp, _vp, _vp]),
            "vdmc_comm_unique_id": (_i32, [_vp]),
            "vdmc_comm_init": (_i32, [ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, ctypes.POINTER(_vp)]),
            "vdmc_comm_free": (None, [_vp]),
            "vdmc_count_distributed": (_i32, [_vp, ctypes.c_int, ctypes.POINTER(CountOptions), _vp, ctypes.c_int,
                                              _vp, _vp]),
            "vdmc_num_classes_kind": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
            "vdmc_class_ids_kind": (_i32, [ctypes.c_int, ctypes.c_int, _vp]),
            "vdmc_class_ids32": (_i32, [ctypes.c_int, ctypes.c_int, _vp]),
            "vdmc_plan": (_i32, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Range)]),
            "vdmc_split_costs": (_i32, [_vp, _i64, ctypes.c_int, ctypes.POINTER(Range)]),
            "vdmc_num_classes": (ctypes.c_int, [ctypes.c_int]),
            "vdmc_class_ids": (_i32, [ctypes.c_int, _vp]),
            "vdmc_get_info": (_i32, [_vp, ctypes.POINTER(Info)]),
            "vdmc_get_order": (_i32, [_vp, _vp]),
            "vdmc_kernel_launches": (_i64, []),
            "vdmc_free_graph": (None, [_vp]),
            "vdmc_trim": (_i32, [ctypes.c_int]),
            "vdmc_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st != VDMC_OK:
        raise VdmcError(st, lib().vdmc_last_error().decode())


DIRECTED, UNDIRECTED = 0, 1
_KINDS = {"directed": DIRECTED, "undirected": UNDIRECTED, DIRECTED: DIRECTED, UNDIRECTED: UNDIRECTED}


def _kind(kind) -> int:
    if kind not in _KINDS:
        raise ValueError(f"motif kind {kind!r} not in ('directed', 'undirected')")
    return _KINDS[kind]


def num_classes(k: int, kind="directed") -> int:
    return lib().vdmc_num_classes_kind(k, _kind(kind))


def class_ids(k: int, kind="directed") -> np.ndarray:
    """Column ids (canonical paper index, ascending); uint32 (k = 5 indices have 20 bits)."""
    kd = _kind(kind)
    C = num_classes(k, kd)
    if C < 0:
        _check(lib().vdmc_class_ids32(k, kd, None))
    out = np.zeros(C, np.uint32)
    _check(lib().vdmc_class_ids32(k, kd, out.ctypes.data))
    return out


def split_costs(prefix: np.ndarray, nparts: int):
    prefix = np.ascontiguousarray(prefix, dtype=np.int64)
    parts = (Range * nparts)()
    _check(lib().vdmc_split_costs(prefix.ctypes.data if prefix.size else None, prefix.size, nparts, parts))
    return [(p.task_lo, p.task_hi) for p in parts]


def symmetrize(n: int, indptr, nbr, device: int = 0):
    """The paper's directed CSR (Indices, Neighbors) -> the G_U CSR with direction
    codes (indptr int64 [n+1], nbr int32 [nnz], dir uint8 [nnz]), via vdmc_symmetrize."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    nb = np.ascontiguousarray(nbr, dtype=np.int32)
    a, b, c = _vp(), _vp(), _vp()
    _check(lib().vdmc_symmetrize(n, ip.ctypes.data, nb.ctypes.data if nb.size else None, device,
                                 ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    try:
        ind = np.ctypeslib.as_array(ctypes.cast(a, ctypes.POINTER(ctypes.c_int64)), (n + 1,)).copy()
        nnz = int(ind[n])
        if nnz:
            nbo = np.ctypeslib.as_array(ctypes.cast(b, ctypes.POINTER(ctypes.c_int32)), (nnz,)).copy()
            dr = np.ctypeslib.as_array(ctypes.cast(c, ctypes.POINTER(ctypes.c_uint8)), (nnz,)).copy()
        else:
            nbo, dr = np.zeros(0, np.int32), np.zeros(0, np.uint8)
    finally:
        for p in (a, b, c):
            lib().vdmc_free_host(p)
    return ind, nbo, dr


def _options(kind, options, timings):
    o = CountOptions()
    o.kind = _kind(kind)
    for key, val in (options or {}).items():
        if key not in OPTION_KEYS:
            raise ValueError(f"unknown count option {key!r}; known: {OPTION_KEYS}")
        setattr(o, key, int(val))
    buf = None
    if timings is not None:
        buf = (ctypes.c_float * 4)()
        o.timings_ms = ctypes.cast(buf, ctypes.POINTER(ctypes.c_float))
    return o, buf


def trim(device: int = 0) -> None:
    """Release the library's idle cached device blocks on `device` (vdmc_trim)."""
    _check(lib().vdmc_trim(device))


def kernel_launches() -> int:
    return int(lib().vdmc_kernel_launches())


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Graph:
    """A graph resident on one GPU (vdmc_graph).  Build from a directed edge list."""

    def __init__(self, n: int, src, dst, rank=None, device: int = 0, stream=None):
        import torch
        self._h = _vp()
        rk = None
        if rank is not None:
            rk = np.ascontiguousarray(rank, dtype=np.int32)
        if isinstance(src, torch.Tensor) and src.is_cuda:
            if not (isinstance(dst, torch.Tensor) and dst.is_cuda and dst.device == src.device):
                raise ValueError("src and dst must be CUDA tensors on the same device")
            if src.dtype != torch.int32 or dst.dtype != torch.int32 or src.numel() != dst.numel():
                raise ValueError("src and dst must be int32 tensors of equal length")
            src, dst = src.contiguous(), dst.contiguous()
            device = src.device.index
            with torch.cuda.device(device):
                st = lib().vdmc_build_graph_edges(n, src.numel(), src.data_ptr(), dst.data_ptr(), 1,
                                                  rk.ctypes.data if rk is not None else None, device,
                                                  _stream_ptr(stream), ctypes.byref(self._h))
        else:
            s = np.ascontiguousarray(src, dtype=np.int32)
            d = np.ascontiguousarray(dst, dtype=np.int32)
            with torch.cuda.device(device):
                st = lib().vdmc_build_graph_edges(n, s.size, s.ctypes.data if s.size else None,
                                                  d.ctypes.data if d.size else None, 0,
                                                  rk.ctypes.data if rk is not None else None, device,
                                                  _stream_ptr(stream), ctypes.byref(self._h))
        _check(st)
        self.device = device
        self.info = self._info()

    @classmethod
    def from_sym_csr(cls, n: int, indptr, nbr, dirc, rank=None, device: int = 0) -> "Graph":
        """Build from the symmetric G_U CSR + direction codes (vdmc_build_graph)."""
        self = cls.__new__(cls)
        self._h = _vp()
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        nb = np.ascontiguousarray(nbr, dtype=np.int32)
        dc = np.ascontiguousarray(dirc, dtype=np.uint8)
        rk = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
        _check(lib().vdmc_build_graph(n, ip.ctypes.data, nb.ctypes.data if nb.size else None,
                                      dc.ctypes.data if dc.size else None,
                                      rk.ctypes.data if rk is not None else None, device, ctypes.byref(self._h)))
        self.device = device
        self.info = self._info()
        return self

    def _info(self) -> dict:
        inf = Info()
        _check(lib().vdmc_get_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in Info._fields_}

    @property
    def n(self) -> int:
        return self.info["n"]

    @property
    def ntasks(self) -> int:
        return self.info["ntasks"]

    def order(self) -> np.ndarray:
        out = np.zeros(max(self.n, 1), np.int32)
        _check(lib().vdmc_get_order(self._h, out.ctypes.data))
        return out[: self.n]

    def count(self, k: int, out=None, work=None, stream=None, kind="directed", options=None, timings=None):
        """uint64 counts [n][C] as an int64 torch tensor on the graph's device (same bits).
        kind: "directed" (13 / 199 classes) or "undirected" (2 / 6 classes of G_U).
        options: dict of result-preserving path options (OPTION_KEYS, vdmc_count_options).
        timings: a dict to receive device times in ms (the call then synchronises the stream)."""
        import torch
        kd = _kind(kind)
        C = num_classes(k, kd)
        o, buf = _options(kd, options, timings)
        if C < 0:
            _check(lib().vdmc_count_ex(self._h, k, None, None, ctypes.byref(o), None))
        if out is None:
            out = torch.empty((self.n, C), dtype=torch.int64, device=f"cuda:{self.device}")
        if not (out.is_cuda and out.device.index == self.device and out.dtype == torch.int64
                and out.is_contiguous() and tuple(out.shape) == (self.n, C)):
            raise ValueError(f"out must be a contiguous int64 [{self.n}, {C}] tensor on cuda:{self.device}")
        rng = None
        if work is not None:
            rng = Range(int(work[0]), int(work[1]))
        with torch.cuda.device(self.device):
            _check(lib().vdmc_count_ex(self._h, k, out.data_ptr() if out.numel() else None,
                                       ctypes.byref(rng) if rng is not None else None, ctypes.byref(o),
                                       _stream_ptr(stream)))
        if timings is not None:
            timings.update(zip(["schedule", "enum", "finalize", "count"], list(buf)))
        return out

    def count_edges(self, k: int, out=None, work=None, stream=None, kind="directed", timings=None):
        """Edge-level counts: uint64 [edges][C] as an int64 tensor on
        the graph's device; rows in the order of edges() (u < v original ids, lexicographic)."""
        import torch
        kd = _kind(kind)
        C = num_classes(k, kd)
        o, buf = _options(kd, None, timings)
        if C < 0:
            _check(lib().vdmc_count_edges(self._h, k, None, None, ctypes.byref(o), None))
        E = self.ntasks
        if out is None:
            out = torch.empty((E, C), dtype=torch.int64, device=f"cuda:{self.device}")
        if not (out.is_cuda and out.device.index == self.device and out.dtype == torch.int64
                and out.is_contiguous() and tuple(out.shape) == (E, C)):
            raise ValueError(f"out must be a contiguous int64 [{E}, {C}] tensor on cuda:{self.device}")
        rng = None if work is None else Range(int(work[0]), int(work[1]))
        with torch.cuda.device(self.device):
            _check(lib().vdmc_count_edges(self._h, k, out.data_ptr() if out.numel() else None,
                                          ctypes.byref(rng) if rng is not None else None, ctypes.byref(o),
                                          _stream_ptr(stream)))
        if timings is not None:
            timings.update(zip(["schedule", "enum", "finalize", "count"], list(buf)))
        return out

    def edges(self):
        """(u, v) original ids of each edge row of count_edges (u < v, lexicographic)."""
        E = self.ntasks
        u = np.zeros(max(E, 1), np.int32)
        v = np.zeros(max(E, 1), np.int32)
        with_dev = __import__("torch").cuda.device(self.device)
        with with_dev:
            _check(lib().vdmc_get_edges(self._h, u.ctypes.data, v.ctypes.data))
        return u[:E], v[:E]

    def plan(self, k: int, nparts: int):
        parts = (Range * nparts)()
        _check(lib().vdmc_plan(self._h, k, nparts, parts))
        return [(p.task_lo, p.task_hi) for p in parts]

    def root_range(self, pos_lo: int, pos_hi: int):
        """Task slice of the roots at order positions [pos_lo, pos_hi) (vdmc_root_range)."""
        r = Range()
        _check(lib().vdmc_root_range(self._h, pos_lo, pos_hi, ctypes.byref(r)))
        return (r.task_lo, r.task_hi)

    def close(self):
        if getattr(self, "_h", None):
            lib().vdmc_free_graph(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def count(n: int, src, dst, k: int, device: int = 0, rank=None, kind="directed"):
    """One-shot: build the graph on `device`, count k-motifs, return a host uint64 [n][C]."""
    g = Graph(n, src, dst, rank=rank, device=device)
    try:
        out = g.count(k, kind=kind)
        return out.cpu().numpy().view(np.uint64)
    finally:
        g.close()


class Comm:
    """An NCCL communicator owned by libvdmc (vdmc_comm).  torch.distributed only moves the
    128-byte unique id from rank 0 to the others (any backend, gloo included)."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist
        world = dist.get_world_size(group)
        me = dist.get_rank(group)
        uid = (ctypes.c_uint8 * 128)()
        if me == 0:
            _check(lib().vdmc_comm_unique_id(uid))
        obj = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        self._h = _vp()
        self.rank, self.world, self.device = me, world, device
        _check(lib().vdmc_comm_init(world, me, uid, device, ctypes.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().vdmc_comm_free(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def count_distributed(g: Graph, k: int, comm: Comm, root: int = 0, kind="directed", stream=None, options=None):
    """Multi-GPU count through the C ABI (vdmc_count_distributed): the graph is
    replicated on every rank; rank p counts the p-th cost-balanced task slice into a private
    partial; one ncclReduce (uint64 sum) gives `root` (a rank of comm) the full matrix.
    Returns the [n][C] tensor on root, None elsewhere."""
    import torch
    kd = _kind(kind)
    C = num_classes(k, kd)
    o, _ = _options(kd, options, None)
    out = None
    if comm.rank == root:
        out = torch.empty((g.n, C), dtype=torch.int64, device=f"cuda:{g.device}")
    with torch.cuda.device(g.device):
        _check(lib().vdmc_count_distributed(g._h, k, ctypes.byref(o), comm._h, root,
                                            out.data_ptr() if out is not None and out.numel() else None,
                                            _stream_ptr(stream)))
    return out


def count_slices_reduce(g, k: int, group=None, dst_rank: int = 0, kind="directed"):
    """The same decomposition with torch.distributed as the reduce (any backend): rank p counts
    slice p of g.plan(k, world) and dist.reduce sums the partials on dst_rank (a rank of
    `group`).  Host-logic twin of count_distributed, testable with gloo."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    parts = g.plan(k, world)
    out = g.count(k, work=parts[me], kind=kind)
    dst = dist.get_global_rank(group, dst_rank) if group is not None else dst_rank
    dist.reduce(out, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return out
