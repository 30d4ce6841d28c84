"""Python mirror of the reference `blocktet` API for the hot path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/blocktet/*.hpp) so parity tests read like the
reference's own tests. Storage is device-resident: ``FEFunction.values[l]``
is a CUDA float64 tensor holding FEFunction::values[l][cell][entry]
flattened (cells outer, slots inner). Everything goes through the C ABI in
include/blocktet_b200.h; torch provides device memory and the stream.

Reference exception types map to:
  std::invalid_argument -> InvalidArgument (ValueError)
  std::out_of_range     -> OutOfRange (IndexError)
  std::domain_error     -> DomainError (ArithmeticError)
  std::logic_error      -> LogicError (RuntimeError)
  std::runtime_error    -> SolverError (RuntimeError)
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import traceback
import weakref
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import bt_field, bt_fmg_row, bt_form, bt_multigrid_config, bt_smoother_config

# bt_allreduce_fn: int (*)(double* buf, int64_t n, void* stream, void* user)
_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
_SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)


class _DeviceArray:
    """__cuda_array_interface__ view of n fp64 values at a device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}

_L = _lib.lib


class InvalidArgument(ValueError):
    pass


class OutOfRange(IndexError):
    pass


class DomainError(ArithmeticError):
    pass


class LogicError(RuntimeError):
    pass


class SolverError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERR = {1: InvalidArgument, 2: OutOfRange, 3: DomainError, 4: LogicError, 5: SolverError, 6: CudaError,
        7: CudaError}


def _check(status: int):
    if status:
        raise _ERR.get(status, RuntimeError)(_L.bt_last_error().decode())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor):
    if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise InvalidArgument("expected a contiguous CUDA float64 tensor")
    return C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------
# micro_index.hpp
# ---------------------------------------------------------------------------
class Subgroup(enum.IntEnum):
    V = 0
    EdgeX = 1
    EdgeY = 2
    EdgeZ = 3
    EdgeXY = 4
    EdgeXZ = 5
    EdgeYZ = 6
    EdgeXYZ = 7
    CellIUp = 20
    CellIDown = 21
    CellIIUp = 22
    CellIIDown = 23
    CellIIIUp = 24
    CellIIIDown = 25


def n_tri(w):
    return _L.bt_n_tri(w)


def n_tet(w):
    return _L.bt_n_tet(w)


def width_formula(g, level):
    return _L.bt_width_formula(int(g), level)


def width(g, level):
    out = C.c_int()
    _check(_L.bt_width(int(g), level, C.byref(out)))
    return out.value


def linearize(w, p):
    return _L.bt_linearize(w, p[0], p[1], p[2])


def linearize_checked(w, p):
    """linearize_checked (micro_index.hpp:150-154): OutOfRange outside I_tet(w)."""
    out = C.c_int64()
    _check(_L.bt_linearize_checked(w, int(p[0]), int(p[1]), int(p[2]), C.byref(out)))
    return out.value


def linearize_aos(w, m, p, d):
    """m * linearize(w, p) + d (micro_index.hpp:167-170)."""
    out = C.c_int64()
    _check(_L.bt_linearize_aos(w, m, int(p[0]), int(p[1]), int(p[2]), d, C.byref(out)))
    return out.value


def linearize_soa(w, m, p, d):
    """d * n_tet(w) + linearize(w, p) (micro_index.hpp:172-175)."""
    out = C.c_int64()
    _check(_L.bt_linearize_soa(w, m, int(p[0]), int(p[1]), int(p[2]), d, C.byref(out)))
    return out.value


@dataclass
class CoarseMesh:
    """parse_mesh's result (coarse_mesh.hpp:37-47): vertex coordinates and
    cell vertex ids after the orientation repair; `text` re-serialises it."""
    vertex_coords: np.ndarray
    cells: np.ndarray
    n_warnings: int = 0

    def n_vertices(self):
        return len(self.vertex_coords)

    def n_cells(self):
        return len(self.cells)

    @property
    def text(self):
        lines = [f"vertices {self.n_vertices()}"]
        lines += [" ".join(repr(float(c)) for c in v) for v in self.vertex_coords]
        lines.append(f"cells {self.n_cells()}")
        lines += [" ".join(str(int(q)) for q in c) for c in self.cells]
        return "\n".join(lines) + "\n"


def parse_mesh(text: str) -> CoarseMesh:
    """parse_mesh (coarse_mesh.hpp:225-308), with the reference's error messages."""
    nv, nc, nw = C.c_int(), C.c_int(), C.c_int()
    _check(_L.bt_mesh_parse(text.encode(), C.byref(nv), C.byref(nc), None, None, C.byref(nw)))
    xyz = np.zeros((nv.value, 3))
    cells = np.zeros((nc.value, 4), np.int32)
    _check(_L.bt_mesh_parse(text.encode(), C.byref(nv), C.byref(nc), xyz.ctypes.data_as(C.c_void_p),
                            cells.ctypes.data_as(C.c_void_p), C.byref(nw)))
    return CoarseMesh(xyz, cells, nw.value)


def delinearize(w, t):
    out = (C.c_int * 3)()
    _check(_L.bt_delinearize(w, t, out))
    return (out[0], out[1], out[2])


def subgroup_offsets(g):
    out = (C.c_int * 12)()
    n = _L.bt_subgroup_offsets(int(g), out)
    return [tuple(out[3 * i: 3 * i + 3]) for i in range(n)]


def index_set(w):
    return [(i, j, k) for k in range(w) for j in range(w - k) for i in range(w - k - j)]


# ---------------------------------------------------------------------------
# spaces / grid / functions (fe_function.hpp)
# ---------------------------------------------------------------------------
class LayoutKind(enum.IntEnum):
    AoS = 0
    SoA = 1


@dataclass(frozen=True)
class SpaceDescriptor:
    name: str
    space: int  # bt_space
    layout: LayoutKind = LayoutKind.AoS


def p1_space(layout=LayoutKind.AoS):
    return SpaceDescriptor("p1", 0, layout)


def edge_space(layout=LayoutKind.AoS):
    """The seven edge subgroups (N1E1 storage)."""
    return SpaceDescriptor("edges", 2, layout)


class Grid:
    """Grid (fe_function.hpp:92): mesh + per-level interface identification,
    held as implicit macro face/edge/vertex tables on the device."""

    def __init__(self, mesh_text, min_level: int, max_level: int, device: Optional[int] = None):
        """Grid(CoarseMesh, min, max) as the reference (fe_function.hpp:105),
        or the mesh text directly."""
        if isinstance(mesh_text, CoarseMesh):
            mesh_text = mesh_text.text
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        torch.cuda.init()
        h = C.c_void_p()
        _check(_L.bt_grid_create(mesh_text.encode(), min_level, max_level, device, C.byref(h)))
        self._h = h
        self.mesh_text = mesh_text

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.bt_grid_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def n_cells(self):
        return _L.bt_num_cells(self._h)

    def min_level(self):
        return _L.bt_grid_min_level(self._h)

    def max_level(self):
        return _L.bt_grid_max_level(self._h)

    def has_level(self, l):
        return self.min_level() <= l <= self.max_level()

    def space_size(self, space: int, level: int) -> int:
        return _L.bt_space_size(self._h, space, level)

    # ---- multi-GPU cell partition ---------------------------
    def set_partition(self, rank: int, nranks: int, allreduce=None, comm="auto"):
        """Restrict this handle's compute to the cell block of `rank` out of
        `nranks` (bt_grid_set_partition). `allreduce(tensor)` sums a device
        tensor over the ranks in place, stream-ordered on the current stream
        (or blocking); default torch.distributed.all_reduce.
        Call before allocating vectors and before compute_stencil: vectors of
        a partitioned grid hold the rank's cells only (space_size is local).
        The library calls `allreduce` itself (bt_grid_set_allreduce) inside
        syncs, dots, applies and solvers, which become collectives: every
        rank calls them in the same order. `comm` ("auto", None or a Comm):
        the native NCCL data plane, which replaces the hook (see set_comm);
        "auto" creates it when torch.distributed runs over NCCL."""
        _check(_L.bt_grid_set_partition(self._h, rank, nranks))
        self._allreduce = allreduce
        self._xbufs = {}
        ref = weakref.ref(self)
        dev = self.device

        def hook(ptr, n, stream, user):
            try:
                g = ref()
                t = torch.as_tensor(_DeviceArray(ptr, n), device=f"cuda:{dev}")
                # stream-ordered: the collective is queued on the library's stream
                s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.default_stream(dev)
                with torch.cuda.stream(s):
                    g.allreduce(t)
                return 0
            except Exception:  # reported as BT_RUNTIME_ERROR by the library
                traceback.print_exc()
                return 1

        self._hook = _ALLREDUCE_FN(hook)
        _check(_L.bt_grid_set_allreduce(self._h, C.cast(self._hook, C.c_void_p), None))
        # the native data plane (neighbour-only NCCL send/recv inside the
        # library) whenever the ranks run torch.distributed over NCCL and no
        # custom allreduce was given; BT_XCHG=hook keeps the Python hook
        self._comm = None
        self._sr_hook = None
        mode = os.environ.get("BT_XCHG", "auto")  # auto | nccl | sendrecv | allreduce (A/B knob)
        if comm == "auto":
            comm = None
            if allreduce is None and nranks > 1 and mode != "allreduce":
                import torch.distributed as dist
                if dist.is_available() and dist.is_initialized():
                    if dist.get_backend() == "nccl" and mode != "sendrecv":
                        comm = nccl_comm(rank, nranks, dev)
                    else:
                        self._set_sendrecv_torch()
        if comm is not None:
            self.set_comm(comm)

    def _set_sendrecv_torch(self):
        """The library's neighbour exchange over torch.distributed point-to-
        point messages (bt_grid_set_sendrecv), staged through the host: the
        transport for process groups without NCCL (gloo, CPU tests)."""
        dev = self.device

        def sr(npeers, peers, soff, roff, sbuf, rbuf, stream, user):
            try:
                import torch.distributed as dist
                s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.default_stream(dev)
                s.synchronize()
                ns, nr = soff[npeers], roff[npeers]
                send = torch.as_tensor(_DeviceArray(sbuf, ns), device=f"cuda:{dev}").cpu() if ns else None
                recv = torch.empty(nr, dtype=torch.float64)
                reqs = []
                for i in range(npeers):
                    if soff[i + 1] > soff[i]:
                        reqs.append(dist.isend(send[soff[i]:soff[i + 1]].clone(), peers[i]))
                    if roff[i + 1] > roff[i]:
                        reqs.append(dist.irecv(recv[roff[i]:roff[i + 1]], peers[i]))
                for r in reqs:
                    r.wait()
                if nr:
                    torch.as_tensor(_DeviceArray(rbuf, nr), device=f"cuda:{dev}").copy_(recv)
                    torch.cuda.synchronize(dev)
                return 0
            except Exception:  # reported as BT_RUNTIME_ERROR by the library
                traceback.print_exc()
                return 1

        self._sr_hook = _SENDRECV_FN(sr)
        _check(_L.bt_grid_set_sendrecv(self._h, C.cast(self._sr_hook, C.c_void_p), None))

    def set_comm(self, comm: Optional["Comm"]):
        """Attach the ranks' NCCL communicator (bt_grid_set_comm): the
        library then exchanges interface values neighbour-only over NCCL and
        sums dot partials with ncclAllReduce, with no Python on the path."""
        _check(_L.bt_grid_set_comm(self._h, comm._h if comm is not None else None))
        self._comm = comm

    def data_plane(self) -> str:
        """'nccl' (native neighbour exchange), 'sendrecv' (the neighbour
        exchange over torch.distributed messages), 'allreduce' (the hook) or
        'none'."""
        if getattr(self, "_comm", None) is not None:
            return "nccl"
        if getattr(self, "_sr_hook", None) is not None:
            return "sendrecv"
        return "allreduce" if getattr(self, "_hook", None) is not None else "none"

    def partition(self):
        """(rank, nranks, cell_begin, cell_end)"""
        r, n, b, e = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_L.bt_grid_partition(self._h, C.byref(r), C.byref(n), C.byref(b), C.byref(e)))
        return r.value, n.value, b.value, e.value

    def partitioned(self) -> bool:
        return self.partition()[1] > 1

    def allreduce(self, t: torch.Tensor):
        fn = getattr(self, "_allreduce", None)
        if fn is not None:
            fn(t)
        else:
            import torch.distributed as dist
            dist.all_reduce(t)

    def xchg_buffer(self, l) -> Optional[torch.Tensor]:
        n = _L.bt_xchg_size(self._h, l)
        if n < 0:
            _check(4)  # BT_LOGIC_ERROR, message from bt_last_error
        if n == 0:
            return None
        bufs = getattr(self, "_xbufs", None)
        if bufs is None:
            bufs = self._xbufs = {}
        b = bufs.get(l)
        if b is None or b.numel() != n:
            b = bufs[l] = torch.zeros(n, dtype=torch.float64, device=f"cuda:{self.device}")
        return b

    def masks(self, level, cell, g):
        n = n_tet(width_formula(g, level))
        o = np.zeros(n, np.uint8)
        d = np.zeros(n, np.uint8)
        _check(_L.bt_grid_masks(self._h, level, cell, int(g), o.ctypes.data_as(_lib.PU8),
                                d.ctypes.data_as(_lib.PU8)))
        return o, d

    def groups(self, level, space=0):
        ng, nm = C.c_int64(), C.c_int64()
        _check(_L.bt_grid_groups(self._h, level, space, C.byref(ng), C.byref(nm), None, None, None, None))
        off = np.zeros(ng.value + 1, np.int64)
        cell = np.zeros(nm.value, np.int32)
        g = np.zeros(nm.value, np.int32)
        t = np.zeros(nm.value, np.int64)
        _check(_L.bt_grid_groups(self._h, level, space, C.byref(ng), C.byref(nm),
                                 off.ctypes.data_as(_lib.PI64), cell.ctypes.data_as(_lib.PI32),
                                 g.ctypes.data_as(_lib.PI32), t.ctypes.data_as(_lib.PI64)))
        return off, cell, g, t


def cubes_mesh_text(n: int, perturb: float = 0.1, seed: int = 0) -> str:
    need = _L.bt_cubes_mesh_text(n, perturb, seed, None, 0)
    buf = C.create_string_buffer(need + 1)
    _L.bt_cubes_mesh_text(n, perturb, seed, buf, need + 1)
    return buf.value.decode()


def box_mesh_text(nx: int, ny: int, nz: int, perturb: float = 0.0, seed: int = 0) -> str:
    """nx x ny x nz unit cubes x 6 Kuhn tets (bt_box_mesh_text)."""
    need = _L.bt_box_mesh_text(nx, ny, nz, perturb, seed, None, 0)
    if need < 0:
        raise InvalidArgument("box_mesh_text: dimensions must be >= 1")
    buf = C.create_string_buffer(need + 1)
    _L.bt_box_mesh_text(nx, ny, nz, perturb, seed, buf, need + 1)
    return buf.value.decode()


def blocked_mesh_text(nx: int, ny: int, nz: int, block=(2, 2, 2), h: float = 1.0, perturb: float = 0.1,
                      seed: int = 0) -> str:
    """nx x ny x nz cubes of side h x 6 Kuhn tets, cubes numbered block-major
    (bt_blocked_mesh_text): contiguous cell ranges are compact blocks."""
    bx, by, bz = block
    need = _L.bt_blocked_mesh_text(nx, ny, nz, bx, by, bz, h, perturb, seed, None, 0)
    if need < 0:
        raise InvalidArgument("blocked_mesh_text: dimensions, blocks and h must be positive")
    buf = C.create_string_buffer(need + 1)
    _L.bt_blocked_mesh_text(nx, ny, nz, bx, by, bz, h, perturb, seed, buf, need + 1)
    return buf.value.decode()


def ref_tet_text():
    return "# reference tetrahedron\nvertices 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ncells 1\n0 1 2 3\n"


def cube_kuhn_text():
    """coarse_mesh.hpp:344-368: unit cube, six tets around the (0,0,0)-(1,1,1) diagonal."""
    lines = ["# unit cube, six tetrahedra around the main diagonal", "vertices 8"]
    corner = []
    for vid in range(8):
        c = (vid & 1, (vid >> 1) & 1, (vid >> 2) & 1)
        corner.append(c)
        lines.append(f"{c[0]} {c[1]} {c[2]}")
    lines.append("cells 6")
    for axes in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
        c = [0, 0, 0, 7]
        c[1] = 1 << axes[0]
        c[2] = c[1] | (1 << axes[1])
        v0 = np.array(corner[c[0]], float)
        u, w, z = (np.array(corner[c[k]], float) - v0 for k in (1, 2, 3))
        if np.dot(u, np.cross(w, z)) < 0:
            c[2], c[3] = c[3], c[2]
        lines.append(" ".join(map(str, c)))
    return "\n".join(lines) + "\n"


@dataclass
class FEFunction:
    grid: Grid
    descriptor: SpaceDescriptor
    min_level: int
    max_level: int
    values: Dict[int, torch.Tensor] = field(default_factory=dict)

    def check_level(self, l):
        if l < self.min_level or l > self.max_level:
            raise OutOfRange("level not allocated")
        return l - self.min_level

    def level(self, l) -> torch.Tensor:
        self.check_level(l)
        return self.values[l]

    def entries(self):
        """Subgroups of the space's entries, in storage order (SpaceDescriptor::entries)."""
        return [0] if self.descriptor.space == 0 else ([0] if self.descriptor.space == 1 else []) + list(range(1, 8))

    def slots_of(self, l, entry=None):
        """Slots of one entry (FEFunction::slots_of, fe_function.hpp:245-248),
        or of a whole cell when entry is None."""
        ents = self.entries()
        if entry is None:
            return sum(n_tet(width_formula(g, l)) for g in ents)
        if not 0 <= entry < len(ents):
            raise OutOfRange("entry out of range")
        return n_tet(width_formula(ents[entry], l))

    def offset(self, l, entry, t, d=0):
        """Layout-aware slot offset of (t, d) (FEFunction::offset,
        fe_function.hpp:257-261): m t + d (AoS) or d slots + t (SoA); every
        space here has m = 1 per entry, where the two coincide."""
        m = 1
        if not 0 <= d < m:
            raise OutOfRange("linearize: bad DoF index")
        return m * int(t) + d if self.descriptor.layout == LayoutKind.AoS else d * self.slots_of(l, entry) + int(t)

    def array(self, l, cell, entry=None):
        """This rank's values of `cell` (and one entry of it): a view into
        values[l]. Cells outside the rank's block raise OutOfRange."""
        self.check_level(l)
        _, _, b, e = self.grid.partition()
        if not b <= cell < e:
            raise OutOfRange("cell not held by this rank")
        n = self.slots_of(l)
        base = (cell - b) * n
        if entry is None:
            return self.values[l][base:base + n]
        ents = self.entries()
        first = sum(n_tet(width_formula(g, l)) for g in ents[:entry]) if 0 <= entry < len(ents) else 0
        return self.values[l][base + first:base + first + self.slots_of(l, entry)]

    def host(self, l) -> np.ndarray:
        return self.values[l].cpu().numpy()

    def at(self, l, cell, entry, t, d=0):
        a = self.array(l, cell, entry)
        o = self.offset(l, entry, t, d)
        if not 0 <= o < a.numel():
            raise OutOfRange("slot out of range")
        return float(a[o].item())


def allocate(descriptor: SpaceDescriptor, grid: Grid, min_level: int = -1, max_level: int = -1) -> FEFunction:
    if grid is None:
        raise InvalidArgument("allocate: grid required")
    if min_level < 0:
        min_level = grid.min_level()
    if max_level < 0:
        max_level = grid.max_level()
    if not grid.has_level(min_level) or not grid.has_level(max_level) or min_level > max_level:
        raise OutOfRange("allocate: levels outside grid range")
    dev = torch.device("cuda", grid.device)
    vals = {l: torch.zeros(grid.space_size(descriptor.space, l), dtype=torch.float64, device=dev)
            for l in range(min_level, max_level + 1)}
    return FEFunction(grid, descriptor, min_level, max_level, vals)


def _compatible(a: FEFunction, b: FEFunction, l):
    if a.grid is not b.grid:
        raise InvalidArgument("functions live on different grids")
    if a.descriptor.space != b.descriptor.space:
        raise InvalidArgument("descriptor mismatch")
    a.check_level(l)
    b.check_level(l)


def assign(fn: FEFunction, l, value):
    fn.check_level(l)
    _check(_L.bt_assign(fn.grid.handle, fn.descriptor.space, l, _ptr(fn.values[l]), float(value), _stream()))


def scale(fn: FEFunction, l, s):
    fn.check_level(l)
    _check(_L.bt_scale(fn.grid.handle, fn.descriptor.space, l, _ptr(fn.values[l]), float(s), _stream()))


def copy(src: FEFunction, dst: FEFunction, l):
    _compatible(src, dst, l)
    _check(_L.bt_copy(src.grid.handle, src.descriptor.space, l, _ptr(src.values[l]), _ptr(dst.values[l]),
                      _stream()))


def axpy(y: FEFunction, a, x: FEFunction, l):
    _compatible(x, y, l)
    _check(_L.bt_axpy(y.grid.handle, y.descriptor.space, l, _ptr(y.values[l]), float(a), _ptr(x.values[l]),
                      _stream()))


def xchg_plan_host(mesh_text: str, level: int, rank: int, nranks: int) -> dict:
    """The exchange plan of one rank, built on the host without CUDA
    (bt_xchg_plan_host): entry arrays slot / buf / base / count / dir and the
    buffer size. For tests of the partition logic on CPU."""
    bs = C.c_int64()
    n = _L.bt_xchg_plan_host(mesh_text.encode(), level, rank, nranks, C.byref(bs), None, None, None, None, None)
    if n < 0:
        raise InvalidArgument(_L.bt_last_error().decode())
    slot = np.zeros(n, np.int64)
    buf = np.zeros(n, np.int32)
    base = np.zeros(n, np.int32)
    count = np.zeros(n, np.int32)
    d = np.zeros(n, np.uint8)
    _L.bt_xchg_plan_host(mesh_text.encode(), level, rank, nranks, C.byref(bs), slot.ctypes.data_as(_lib.PI64),
                         buf.ctypes.data_as(_lib.PI32), base.ctypes.data_as(_lib.PI32),
                         count.ctypes.data_as(_lib.PI32), d.ctypes.data_as(_lib.PU8))
    return {"buf_size": bs.value, "slot": slot, "buf": buf, "base": base, "count": count, "dir": d}


def xchg_peers_host(mesh_text: str, level: int, rank: int, nranks: int) -> dict:
    """The neighbour plan of one rank's P1 exchange, built on the host
    (bt_xchg_peers_host): {"sends": (peer, pos), "recvs": (peer, pos)} int32
    arrays in message order. For tests of the data plane on CPU."""
    out = {}
    for which, key in ((0, "sends"), (1, "recvs")):
        n = _L.bt_xchg_peers_host(mesh_text.encode(), level, rank, nranks, which, None, None)
        if n < 0:
            raise InvalidArgument(_L.bt_last_error().decode())
        peer = np.zeros(n, np.int32)
        pos = np.zeros(n, np.int32)
        _L.bt_xchg_peers_host(mesh_text.encode(), level, rank, nranks, which, peer.ctypes.data_as(_lib.PI32),
                              pos.ctypes.data_as(_lib.PI32))
        out[key] = (peer, pos)
    return out


class Comm:
    """The ranks' NCCL communicator (bt_comm): the library's native
    multi-GPU data plane. Every rank constructs it with the same 128-byte
    unique id (Comm.unique_id() on one rank, shared out of band)."""

    def __init__(self, unique_id: bytes, rank: int, nranks: int, device: int):
        if len(unique_id) != 128:
            raise InvalidArgument("Comm: the unique id is 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _check(_L.bt_comm_create(C.cast(buf, _lib.PU8), rank, nranks, device, C.byref(h)))
        self._h = h
        self.rank, self.nranks, self.device = rank, nranks, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(_L.bt_comm_unique_id(C.cast(buf, _lib.PU8)))
        return bytes(buf)

    def close(self):
        if getattr(self, "_h", None):
            _L.bt_comm_destroy(self._h)
            self._h = None


_COMMS: Dict[tuple, Comm] = {}


def nccl_comm(rank: int, nranks: int, device: int) -> Comm:
    """The process's Comm over the torch.distributed world (rank 0 draws
    the id, broadcast over the default group), created once per
    (rank, nranks, device) and kept for the life of the process."""
    key = (rank, nranks, device)
    if key not in _COMMS:
        import torch.distributed as dist
        obj = [Comm.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        _COMMS[key] = Comm(obj[0], rank, nranks, device)
    return _COMMS[key]


def partition_range(n_cells: int, rank: int, nranks: int):
    """Cells [begin, end) of `rank` (bt_grid_set_partition's block partition)."""
    return n_cells * rank // nranks, n_cells * (rank + 1) // nranks


def xchg_pack(fn: FEFunction, l, buf: Optional[torch.Tensor]):
    """Multi-GPU protocol step 1: this rank's replica values of rank-spanning
    interface groups into buf (zeros elsewhere)."""
    fn.check_level(l)
    if buf is not None:
        _check(_L.bt_xchg_pack(fn.grid.handle, l, _ptr(fn.values[l]), _ptr(buf), _stream()))


def xchg_finish(fn: FEFunction, l, mode: int, buf: Optional[torch.Tensor], src: Optional[FEFunction] = None):
    """Multi-GPU protocol step 3 (after the caller's allreduce of buf): local
    groups plus member-order reduction of the rank-spanning ones. mode: 0
    sync_additive, 1 sync with Dirichlet identity rows from src, 2
    sync_broadcast, 3 impose_dirichlet (src), 4 zero_dirichlet."""
    fn.check_level(l)
    _check(_L.bt_xchg_finish(fn.grid.handle, l, int(mode), _ptr(fn.values[l]),
                             _ptr(src.values[l]) if src is not None else None,
                             _ptr(buf) if buf is not None else None, _stream()))


def _exchange(fn: FEFunction, l, mode: int, src: Optional[FEFunction] = None):
    """pack -> the grid's allreduce -> finish (bt_exchange)"""
    fn.check_level(l)
    _check(_L.bt_exchange(fn.grid.handle, l, int(mode), _ptr(fn.values[l]),
                          _ptr(src.values[l]) if src is not None else None, _stream()))


def dot_cells(x: FEFunction, y: FEFunction, l) -> np.ndarray:
    """Owned-DoF dot partial of every cell (0 for other ranks' cells)."""
    _compatible(x, y, l)
    out = np.zeros(x.grid.n_cells())
    _check(_L.bt_dot_cells(x.grid.handle, x.descriptor.space, l, _ptr(x.values[l]), _ptr(y.values[l]),
                           out.ctypes.data_as(_lib.PD), _stream()))
    return out


def dot(x: FEFunction, y: FEFunction, l) -> float:
    _compatible(x, y, l)
    out = C.c_double()
    _check(_L.bt_dot(x.grid.handle, x.descriptor.space, l, _ptr(x.values[l]), _ptr(y.values[l]), C.byref(out),
                     _stream()))
    return out.value


def norm2(x: FEFunction, l) -> float:
    return math.sqrt(dot(x, x, l))


def sync_additive(fn: FEFunction, l):
    fn.check_level(l)
    if fn.descriptor.space == 2:
        _check(_L.bt_n1e1_sync(fn.grid.handle, l, _ptr(fn.values[l]), _stream()))
        return
    _check(_L.bt_sync_additive(fn.grid.handle, fn.descriptor.space, l, _ptr(fn.values[l]), _stream()))


def sync_broadcast(fn: FEFunction, l):
    fn.check_level(l)
    _check(_L.bt_sync_broadcast(fn.grid.handle, fn.descriptor.space, l, _ptr(fn.values[l]), _stream()))


def random_fill(fn: FEFunction, l, seed):
    """On a partitioned grid each rank fills its own cells with their part of
    the single-GPU stream, then the exchange broadcasts rank-spanning groups
    (collective: every rank must call it)."""
    fn.check_level(l)
    _check(_L.bt_random_fill(fn.grid.handle, fn.descriptor.space, l, int(seed), _ptr(fn.values[l]), _stream()))
    if fn.grid.partitioned() and fn.descriptor.space == 0:
        _exchange(fn, l, 2)


def zero_dirichlet(fn: FEFunction, l):
    """detail::zero_dirichlet (solvers.hpp:66)."""
    fn.check_level(l)
    _check(_L.bt_zero_dirichlet(fn.grid.handle, l, _ptr(fn.values[l]), _stream()))


def impose_dirichlet(src: FEFunction, dst: FEFunction, l):
    """detail::impose_dirichlet (operators.hpp:98)."""
    _compatible(src, dst, l)
    _check(_L.bt_impose_dirichlet(dst.grid.handle, l, _ptr(src.values[l]), _ptr(dst.values[l]), _stream()))


def hadamard(fn: FEFunction, diag: FEFunction, l, divide: bool):
    """detail::hadamard (solvers.hpp:53-64)."""
    _compatible(fn, diag, l)
    _check(_L.bt_hadamard(fn.grid.handle, l, _ptr(fn.values[l]), _ptr(diag.values[l]), int(divide), _stream()))


def owned_dof_count(fn: FEFunction, l):
    fn.check_level(l)
    return _L.bt_owned_dof_count(fn.grid.handle, fn.descriptor.space, l)


# ---------------------------------------------------------------------------
# forms / operators (forms.hpp, operators.hpp)
# ---------------------------------------------------------------------------
class FormKind(enum.IntEnum):
    Diffusion = 0
    Mass = 1
    DivKGrad = 2


@dataclass(frozen=True)
class Coefficient:
    """Device-evaluable replacement of FormId's std::function coefficient
    (forms.hpp:31): kind 0 constant, 1 sin product, 2 affine."""
    kind: int
    c: tuple

    @staticmethod
    def constant(c0):
        return Coefficient(0, (float(c0), 0.0, 0.0, 0.0))

    @staticmethod
    def sin_product(c0=1.0, c1=0.5, freq=2.0 * math.pi):
        return Coefficient(1, (float(c0), float(c1), float(freq), 0.0))

    @staticmethod
    def affine(c0, cx, cy, cz):
        return Coefficient(2, (float(c0), float(cx), float(cy), float(cz)))


@dataclass(frozen=True)
class FormId:
    kind: FormKind = FormKind.Diffusion
    k: Optional[Coefficient] = None

    @staticmethod
    def diffusion():
        return FormId(FormKind.Diffusion)

    @staticmethod
    def mass():
        return FormId(FormKind.Mass)

    @staticmethod
    def div_k_grad(coeff: Coefficient):
        if coeff is None:
            raise InvalidArgument("div_k_grad needs a coefficient")
        return FormId(FormKind.DivKGrad, coeff)

    def constant_coefficient(self):
        return self.kind != FormKind.DivKGrad

    def c_struct(self):
        f = bt_form()
        f.kind = int(self.kind)
        f.coeff_kind = self.k.kind if self.k else 0
        for i, v in enumerate(self.k.c if self.k else (0.0, 0.0, 0.0, 0.0)):
            f.c[i] = v
        return f


class ApplyMode(enum.IntEnum):
    Replace = 0
    Add = 1


class BC(enum.IntEnum):
    None_ = 0
    DirichletIdentity = 1


class SweepDirection(enum.IntEnum):
    Forward = 0
    Backward = 1


def _require_pair(src: FEFunction, dst: FEFunction, l):
    if src.descriptor.space != 0 or dst.descriptor.space != 0:
        raise InvalidArgument("operator kernels require a P1 function")
    _compatible(src, dst, l)
    if src is dst:
        raise InvalidArgument("source and destination must be distinct")


class StencilTable:
    """StencilTable (operators.hpp:174): per-cell merged rows, typed
    lattice-boundary rows and the assembled diagonal, device-resident."""

    def __init__(self, form: FormId, grid: Grid, level: int):
        self.grid = grid
        self.form = form.kind
        self.level = level
        h = C.c_void_p()
        f = form.c_struct()
        _check(_L.bt_stencil_create(grid.handle, C.byref(f), level, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.bt_stencil_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def rows(self) -> np.ndarray:
        out = np.zeros(15 * self.grid.n_cells())
        _check(_L.bt_stencil_rows(self._h, out.ctypes.data_as(_lib.PD)))
        return out.reshape(-1, 15)

    def diagonal(self) -> torch.Tensor:
        d = torch.zeros(self.grid.space_size(0, self.level), dtype=torch.float64,
                        device=torch.device("cuda", self.grid.device))
        _check(_L.bt_stencil_diagonal(self._h, _ptr(d), _stream()))
        return d


def compute_stencil(form: FormId, grid: Grid, l: int) -> StencilTable:
    if not form.constant_coefficient():
        raise InvalidArgument("compute_stencil: variable-coefficient forms are unsupported")
    if grid is None:
        raise InvalidArgument("compute_stencil: grid required")
    return StencilTable(form, grid, l)


def apply_stencil(table: StencilTable, src: FEFunction, dst: FEFunction, l, bc=BC.None_, threads=1):
    _require_pair(src, dst, l)
    if table.level != l or table.grid is not src.grid:
        raise InvalidArgument("apply_stencil: table/grid mismatch")
    _check(_L.bt_apply_stencil(table.handle, _ptr(src.values[l]), _ptr(dst.values[l]), int(bc), _stream()))


def apply_elementwise(form: FormId, src: FEFunction, dst: FEFunction, l, mode=ApplyMode.Replace, bc=BC.None_,
                      threads=1):
    _require_pair(src, dst, l)
    f = form.c_struct()
    _check(_L.bt_apply_elementwise(src.grid.handle, C.byref(f), l, _ptr(src.values[l]), _ptr(dst.values[l]),
                                   int(mode), int(bc), None, _stream()))


def extract_diagonal(form_or_table, diag: FEFunction, l, threads=1):
    if isinstance(form_or_table, StencilTable):
        t = form_or_table
        if t.level != l or t.grid is not diag.grid:
            raise InvalidArgument("extract_diagonal: table/grid mismatch")
        _check(_L.bt_stencil_diagonal(t.handle, _ptr(diag.values[l]), _stream()))
        return
    f = form_or_table.c_struct()
    _check(_L.bt_extract_diagonal(diag.grid.handle, C.byref(f), l, _ptr(diag.values[l]), _stream()))


# ---------------------------------------------------------------------------
# transfers and multigrid (solvers.hpp)
# ---------------------------------------------------------------------------
def _check_transfer(coarse: FEFunction, fine: FEFunction, fine_l):
    if coarse.grid is not fine.grid:
        raise InvalidArgument("transfer: functions live on different grids")
    fine.check_level(fine_l)
    coarse.check_level(fine_l - 1)


def prolongate_p1(coarse: FEFunction, fine: FEFunction, fine_l, add=False):
    _check_transfer(coarse, fine, fine_l)
    _check(_L.bt_prolongate(fine.grid.handle, fine_l, _ptr(coarse.values[fine_l - 1]), _ptr(fine.values[fine_l]),
                            int(add), _stream()))


def restrict_p1(fine: FEFunction, coarse: FEFunction, fine_l):
    _check_transfer(coarse, fine, fine_l)
    _check(_L.bt_restrict(fine.grid.handle, fine_l, _ptr(fine.values[fine_l]), _ptr(coarse.values[fine_l - 1]),
                          _stream()))


class KernelKind(enum.IntEnum):
    Elementwise = 0
    Stencil = 1


class SmootherKind(enum.IntEnum):
    Jacobi = 0
    GaussSeidel = 1
    Chebyshev = 2


@dataclass
class SmootherConfig:
    kind: SmootherKind = SmootherKind.GaussSeidel
    omega: float = 0.8
    order: int = 2
    lo: float = 0.25
    hi: float = 1.1
    nu1: int = 1
    nu2: int = 1

    @staticmethod
    def gauss_seidel():
        return SmootherConfig()

    @staticmethod
    def jacobi(omega=0.8):
        return SmootherConfig(kind=SmootherKind.Jacobi, omega=omega)

    @staticmethod
    def chebyshev(order=2):
        return SmootherConfig(kind=SmootherKind.Chebyshev, order=order)

    def c_struct(self):
        return bt_smoother_config(int(self.kind), self.omega, self.order, self.lo, self.hi, self.nu1, self.nu2)

    def as_array(self):
        return [int(self.kind), self.omega, self.order, self.lo, self.hi, self.nu1, self.nu2]


@dataclass
class MultigridConfig:
    coarse_level: int = 2
    cycles: int = 5
    coarse_tol: float = 1e-12
    coarse_maxit: int = 4000

    def c_struct(self):
        return bt_multigrid_config(self.coarse_level, self.cycles, self.coarse_tol, self.coarse_maxit)


class GridHierarchy:
    """GridHierarchy (solvers.hpp:308) on the device: per-level operator
    tables, assembled diagonals, lazy spectral estimates, work vectors."""

    def __init__(self, grid: Grid, form: FormId, kernel=KernelKind.Stencil, threads=1):
        self.grid = grid
        self.form = form
        self.kernel = kernel
        h = C.c_void_p()
        f = form.c_struct()
        _check(_L.bt_hierarchy_create(grid.handle, C.byref(f), int(kernel), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.bt_hierarchy_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def diagonal(self, l) -> torch.Tensor:
        p = C.c_void_p()
        _check(_L.bt_hierarchy_diagonal(self._h, l, C.byref(p)))
        tmp = allocate(p1_space(), self.grid, l, l)
        _check(_L.bt_copy(self.grid.handle, 0, l, p, _ptr(tmp.values[l]), _stream()))
        return tmp.values[l]


def make_hierarchy(grid: Grid, form: FormId, kernel=KernelKind.Stencil, threads=1) -> GridHierarchy:
    if grid is None:
        raise InvalidArgument("make_hierarchy: grid required")
    if kernel == KernelKind.Stencil and not form.constant_coefficient():
        raise InvalidArgument("stencil kernel requires a constant-coefficient form")
    return GridHierarchy(grid, form, kernel, threads)


def hierarchy_apply(h: GridHierarchy, x: FEFunction, y: FEFunction, l, bc=BC.DirichletIdentity):
    _require_pair(x, y, l)
    _check(_L.bt_hierarchy_apply(h.handle, l, _ptr(x.values[l]), _ptr(y.values[l]), int(bc), _stream()))


def spectral_estimate(h: GridHierarchy, l) -> float:
    out = C.c_double()
    _check(_L.bt_estimate_lambda_max(h.handle, l, C.byref(out), _stream()))
    return out.value


def smooth(h: GridHierarchy, cfg: SmootherConfig, rhs: FEFunction, x: FEFunction, l, sweeps,
           direction=SweepDirection.Forward):
    _require_pair(rhs, x, l)
    c = cfg.c_struct()
    _check(_L.bt_smooth(h.handle, C.byref(c), _ptr(rhs.values[l]), _ptr(x.values[l]), l, sweeps, int(direction),
                        _stream()))


@dataclass
class IterationRow:
    """IterationRow (solvers.hpp:21); `seconds` is not reported."""
    level: int
    cycle: int
    residual: float
    error: float


@dataclass
class IterationReport:
    residuals: List[float]
    iterations: int
    residual: float
    converged: bool
    rows: List[IterationRow] = field(default_factory=list)


def cg(h: GridHierarchy, rhs: FEFunction, x: FEFunction, l, tol, maxit) -> IterationReport:
    """cg (solvers.hpp:84) with hierarchy_apply(.., DirichletIdentity) as the
    operator (the reference's std::function operator argument cannot cross
    the C ABI; every reference caller passes this operator)."""
    _require_pair(rhs, x, l)
    hist = np.zeros(max(maxit, 1))
    it = C.c_int()
    _check(_L.bt_cg(h.handle, l, tol, maxit, _ptr(rhs.values[l]), _ptr(x.values[l]),
                    hist.ctypes.data_as(_lib.PD), C.byref(it), _stream()))
    res = list(hist[: it.value])
    r = res[-1] if res else 0.0
    return IterationReport(res, it.value, r, bool(res) and r <= tol)


def gauss_seidel_sweep(table: StencilTable, rhs: FEFunction, x: FEFunction, l, direction=None, threads=1):
    """gauss_seidel_sweep (operators.hpp:327-387): lexicographic Gauss-Seidel on
    each cell's interior (hyperplane wavefronts, bitwise the sequential
    order), then Jacobi on the other vertices with the assembled diagonal."""
    _require_pair(rhs, x, l)
    if table.level != l or table.grid is not x.grid:
        raise InvalidArgument("gauss_seidel_sweep: table/grid mismatch")
    backward = direction is not None and int(direction) == int(SweepDirection.Backward)
    _check(_L.bt_gauss_seidel_sweep(table.handle, _ptr(rhs.values[l]), _ptr(x.values[l]), int(backward), None,
                                    _stream()))


def _field(f: Coefficient):
    s = bt_field()
    s.kind = int(f.kind)
    for i, v in enumerate(f.c):
        s.c[i] = v
    return s


def interpolate(fn: FEFunction, l, f: Coefficient):
    """interpolate (fe_function.hpp:454-477) for P1 functions; the function
    is a device-evaluable field (Coefficient kinds) instead of a callable."""
    fn.check_level(l)
    if fn.descriptor.space != 0:
        raise InvalidArgument("interpolate: P1 functions only")
    s = _field(f)
    _check(_L.bt_interpolate(fn.grid.handle, l, C.byref(s), _ptr(fn.values[l]), _stream()))


def l2_error(fn: FEFunction, l, exact: Coefficient) -> float:
    """l2_error (solvers.hpp:613-648)."""
    fn.check_level(l)
    if fn.descriptor.space != 0:
        raise InvalidArgument("l2_error: P1 functions only")
    s = _field(exact)
    out = C.c_double()
    _check(_L.bt_l2_error(fn.grid.handle, l, _ptr(fn.values[l]), C.byref(s), C.byref(out), _stream()))
    return out.value


def fmg(h: GridHierarchy, finest, rhs_levels: List[FEFunction], x: FEFunction, sm: SmootherConfig,
        mg: MultigridConfig, exact: Optional[Coefficient] = None) -> IterationReport:
    """fmg (solvers.hpp:547-604). rhs_levels[i] belongs to level
    mg.coarse_level + i; `exact` (a field) replaces the error callback with
    l2_error against it."""
    if finest < mg.coarse_level:
        raise InvalidArgument("fmg: finest below coarse level")
    if len(rhs_levels) != finest - mg.coarse_level + 1:
        raise InvalidArgument("fmg: one rhs per level expected")
    x.check_level(finest)
    ptrs = (C.c_void_p * len(rhs_levels))()
    for i, r in enumerate(rhs_levels):
        r.check_level(mg.coarse_level + i)
        ptrs[i] = _ptr(r.values[mg.coarse_level + i])
    nmax = 1 + mg.cycles * (finest - mg.coarse_level)
    rows = (bt_fmg_row * nmax)()
    n = C.c_int()
    s, m = sm.c_struct(), mg.c_struct()
    ex = _field(exact) if exact is not None else None
    _check(_L.bt_fmg(h.handle, finest, ptrs, _ptr(x.values[finest]), C.byref(s), C.byref(m),
                     C.byref(ex) if ex is not None else None, rows, nmax, C.byref(n), _stream()))
    out = [IterationRow(rows[i].level, rows[i].cycle, rows[i].residual, rows[i].error) for i in range(n.value)]
    return IterationReport([r.residual for r in out], mg.cycles * (finest - mg.coarse_level),
                           out[-1].residual if out else 0.0, True, out)


def v_cycle(h: GridHierarchy, l, rhs: FEFunction, x: FEFunction, sm: SmootherConfig, mg: MultigridConfig):
    if mg.coarse_level < h.grid.min_level() or l < mg.coarse_level:  # solvers.hpp:512-513
        raise InvalidArgument("v_cycle: level range invalid")
    _require_pair(rhs, x, l)
    s = sm.c_struct()
    m = mg.c_struct()
    _check(_L.bt_v_cycle(h.handle, l, _ptr(rhs.values[l]), _ptr(x.values[l]), C.byref(s), C.byref(m), _stream()))


# ---------------------------------------------------------------------------
# Nedelec N1E1 curl-curl + mass (no reference implementation)
# ---------------------------------------------------------------------------
class N1E1Operator:
    """alpha curl curl + beta identity on the lowest-order edge space of one
    level (7 edge subgroups per macro-cell), device-resident."""

    def __init__(self, grid: Grid, level: int, alpha: float = 1.0, beta: float = 1.0):
        self.grid = grid
        self.level = level
        h = C.c_void_p()
        _check(_L.bt_n1e1_create(grid.handle, level, float(alpha), float(beta), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.bt_n1e1_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h


def apply_n1e1(op: N1E1Operator, src: FEFunction, dst: FEFunction, l=None, bc=BC.DirichletIdentity):
    l = op.level if l is None else l
    if src.descriptor.space != 2 or dst.descriptor.space != 2:
        raise InvalidArgument("N1E1 operator requires edge-space functions")
    _compatible(src, dst, l)
    if src is dst:
        raise InvalidArgument("source and destination must be distinct")
    _check(_L.bt_apply_n1e1(op.handle, _ptr(src.values[l]), _ptr(dst.values[l]), int(bc), _stream()))
