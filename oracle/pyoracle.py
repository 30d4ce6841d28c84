"""TEST INFRASTRUCTURE — ctypes access to the two CPU checkers.

* ``Oracle``    wraps ``oracle/liboracle.so``: the C restatement of the
  reference algorithms (oracle/bt_oracle.c). Travels to the GPU box.
* ``Reference`` wraps ``oracle/_ref/libbtref.so``: the unmodified reference
  headers compiled by oracle/Makefile (only buildable where /root/reference is
  mounted; the built .so travels with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module. The product (paper_2308_01792_b200) never does.
Both classes expose the same method names so tests can run one suite against
either.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbtref.so")

_P = C.POINTER(C.c_double)
_PU8 = C.POINTER(C.c_uint8)
_PI64 = C.POINTER(C.c_int64)
_PI32 = C.POINTER(C.c_int32)


def _dp(a):
    return a.ctypes.data_as(_P)


def kparams(kind=1, c0=1.0, c1=0.5, c2=2.0 * np.pi, c3=0.0):
    """Coefficient descriptor shared by oracle, reference shim and product.

    kind 0: k = c0; kind 1: k = c0 + c1 sin(c2 x) sin(c2 y) sin(c2 z);
    kind 2: k = c0 + c1 x + c2 y + c3 z.  (BASELINE config 3 is kind 1 with
    c0 = 1, c1 = 0.5, c2 = 2*pi.)
    """
    return np.array([kind, c0, c1, c2, c3], dtype=np.float64)


def width_formula(g, level):
    n = 1 << level
    if g == 0:
        return n + 1
    if g in (7, 9, 11, 13, 15, 16, 17, 18, 19, 22, 23, 24, 25):
        return n - 1
    if g == 21:
        return n - 2
    return n


def n_tet(w):
    return w * (w + 1) * (w + 2) // 6 if w > 0 else 0


def load_oracle():
    if not os.path.exists(ORACLE_SO):
        raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
    lib = C.CDLL(ORACLE_SO)
    lib.bo_grid_new.restype = C.c_void_p
    lib.bo_grid_new.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]
    lib.bo_grid_free.argtypes = [C.c_void_p]
    lib.bo_space_size.restype = C.c_int64
    lib.bo_space_size.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.bo_random_fill.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, _P]
    lib.bo_sync.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P]
    lib.bo_dot.restype = C.c_double
    lib.bo_dot.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.bo_owned_count.restype = C.c_int64
    lib.bo_owned_count.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.bo_group_count.restype = C.c_int64
    lib.bo_group_count.argtypes = [C.c_void_p, C.c_int, _PI64]
    lib.bo_groups.argtypes = [C.c_void_p, C.c_int, _PI64, _PI32, _PI32, _PI64]
    lib.bo_masks.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _PU8, _PU8]
    lib.bo_grid_ncells.argtypes = [C.c_void_p]
    lib.bo_mesh_cells.argtypes = [C.c_void_p, _PI32, _P, C.c_char_p]
    lib.bo_compute_stencil.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.bo_class_matrices.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P]
    lib.bo_local_matrix.argtypes = [C.c_int, _P, _P, _P]
    lib.bo_apply_stencil.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P, _P]
    lib.bo_apply_elementwise.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_int, C.c_int, _P, _P]
    lib.bo_extract_diagonal.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, _P]
    lib.bo_prolongate.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.bo_restrict.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.bo_zero_dirichlet.argtypes = [C.c_void_p, C.c_int, _P]
    lib.bo_impose_dirichlet.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.bo_hier_new.restype = C.c_void_p
    lib.bo_hier_new.argtypes = [C.c_void_p, C.c_int, _P, C.c_int]
    lib.bo_hier_free.argtypes = [C.c_void_p]
    lib.bo_hier_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.bo_hier_diag.restype = _P
    lib.bo_hier_diag.argtypes = [C.c_void_p, C.c_int]
    lib.bo_hier_lambda.restype = C.c_double
    lib.bo_hier_lambda.argtypes = [C.c_void_p, C.c_int]
    lib.bo_smooth.argtypes = [C.c_void_p, _P, C.c_int, C.c_int, C.c_int, _P, _P]
    lib.bo_cg.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, _P, _P, _P, C.POINTER(C.c_int)]
    lib.bo_vcycles.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_double, C.c_int, C.c_int, _P, _P, _P]
    lib.bo_cubes_mesh_text.restype = C.c_int64
    lib.bo_cubes_mesh_text.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_char_p, C.c_int64]
    lib.bo_last_error.restype = C.c_char_p
    lib.bo_linearize.restype = C.c_int64
    lib.bo_linearize.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    lib.bo_delinearize.argtypes = [C.c_int, C.c_int64, _PI32]
    lib.bo_width_formula.argtypes = [C.c_int, C.c_int]
    lib.bo_subgroup_offsets.argtypes = [C.c_int, _PI32]
    lib.bo_n1e1_apply.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, _P, _P]
    lib.bo_n1e1_local.argtypes = [_P, C.c_double, C.c_double, _P]
    lib.bo_n1e1_sync.argtypes = [C.c_void_p, C.c_int, _P]
    lib.bo_n1e1_signs.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int8)]
    lib.bo_n1e1_random_fill.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _P]
    lib.bo_n1e1_gradient.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.bo_n1e1_constant_field.argtypes = [C.c_void_p, C.c_int, _P, _P]
    return lib


def load_reference():
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} missing (reference not built)")
    lib = C.CDLL(REF_SO)
    lib.ref_new.restype = C.c_void_p
    lib.ref_new.argtypes = [C.c_char_p, C.c_int, C.c_int]
    lib.ref_free.argtypes = [C.c_void_p]
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_ncells.argtypes = [C.c_void_p]
    lib.ref_space_size.restype = C.c_int64
    lib.ref_space_size.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.ref_masks.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _PU8, _PU8]
    lib.ref_group_count.restype = C.c_int64
    lib.ref_group_count.argtypes = [C.c_void_p, C.c_int, _PI64]
    lib.ref_groups.argtypes = [C.c_void_p, C.c_int, _PI64, _PI32, _PI32, _PI64]
    lib.ref_owned_dof_count.restype = C.c_int64
    lib.ref_owned_dof_count.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.ref_random_fill.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, _P]
    lib.ref_sync.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P]
    lib.ref_dot.restype = C.c_double
    lib.ref_dot.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.ref_stencil_rows.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.ref_class_matrices.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P]
    lib.ref_apply_stencil.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int]
    lib.ref_apply_elementwise.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int]
    lib.ref_extract_diagonal.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, _P]
    lib.ref_prolongate.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.ref_restrict.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.ref_hierarchy.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_int]
    lib.ref_hierarchy_diag.argtypes = [C.c_void_p, C.c_int, _P]
    lib.ref_hierarchy_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, _P]
    lib.ref_lambda_max.restype = C.c_double
    lib.ref_lambda_max.argtypes = [C.c_void_p, C.c_int]
    lib.ref_smooth.argtypes = [C.c_void_p, _P, C.c_int, C.c_int, C.c_int, _P, _P]
    lib.ref_cg.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, _P, _P, _P, C.POINTER(C.c_int)]
    lib.ref_vcycles.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_double, C.c_int, C.c_int, _P, _P, _P, _P]
    lib.ref_zero_dirichlet.argtypes = [C.c_void_p, C.c_int, _P]
    lib.ref_interpolate.argtypes = [C.c_void_p, C.c_int, _P, _P]
    lib.ref_l2_error.argtypes = [C.c_void_p, C.c_int, _P, _P, _P]
    lib.ref_fmg.argtypes = [C.c_void_p, C.c_int, _P, C.c_int, C.c_double, C.c_int, C.c_int, _P, _P, _P, _P,
                            C.POINTER(C.c_int)]
    lib.ref_time_apply.restype = C.c_double
    lib.ref_time_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P]
    lib.ref_subgroup_offsets.argtypes = [C.c_int, _PI32]
    lib.ref_width_formula.argtypes = [C.c_int, C.c_int]
    lib.ref_linearize.restype = C.c_int64
    lib.ref_linearize.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    lib.ref_mesh_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4 + [_PI32, _P, C.c_char_p]
    return lib


def _sm(sm):
    return np.asarray(sm, dtype=np.float64)


class _Base:
    """Common numpy-facing API. Vectors are flat float64 arrays of one level."""

    lo: int
    hi: int

    def size(self, space, level):
        raise NotImplementedError

    def zeros(self, level, space=0):
        return np.zeros(self.size(space, level))


class Oracle(_Base):
    """The C restatement. with_edges=False builds only vertex masks/groups."""

    def __init__(self, mesh_text, lo, hi, with_edges=True):
        self.lib = load_oracle()
        err = C.create_string_buffer(512)
        self.h = self.lib.bo_grid_new(mesh_text.encode(), lo, hi, int(with_edges), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.lo, self.hi, self.with_edges = lo, hi, with_edges
        self.ncells = self.lib.bo_grid_ncells(self.h)
        self._hier = None

    def __del__(self):
        try:
            if getattr(self, "_hier", None):
                self.lib.bo_hier_free(self._hier)
            if getattr(self, "h", None):
                self.lib.bo_grid_free(self.h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            raise RuntimeError(self.lib.bo_last_error().decode())

    def size(self, space, level):
        return self.lib.bo_space_size(self.h, space, level)

    def random_fill(self, level, seed, space=0):
        x = self.zeros(level, space)
        self.lib.bo_random_fill(self.h, space, level, seed, _dp(x))
        return x

    def sync(self, level, v, broadcast=False, space=0):
        v = np.ascontiguousarray(v, dtype=np.float64).copy()
        self.lib.bo_sync(self.h, space, level, int(broadcast), _dp(v))
        return v

    def dot(self, level, x, y, space=0):
        return self.lib.bo_dot(self.h, space, level, _dp(np.ascontiguousarray(x)), _dp(np.ascontiguousarray(y)))

    def owned_count(self, level, space=0):
        return self.lib.bo_owned_count(self.h, space, level)

    def masks(self, level, cell, g):
        n = n_tet(width_formula(g, level))
        o = np.zeros(n, np.uint8)
        d = np.zeros(n, np.uint8)
        self._chk(self.lib.bo_masks(self.h, level, cell, g, o.ctypes.data_as(_PU8), d.ctypes.data_as(_PU8)))
        return o, d

    def groups(self, level):
        m = C.c_int64()
        ng = self.lib.bo_group_count(self.h, level, C.byref(m))
        off = np.zeros(ng + 1, np.int64)
        cell = np.zeros(m.value, np.int32)
        g = np.zeros(m.value, np.int32)
        t = np.zeros(m.value, np.int64)
        self.lib.bo_groups(self.h, level, off.ctypes.data_as(_PI64), cell.ctypes.data_as(_PI32),
                           g.ctypes.data_as(_PI32), t.ctypes.data_as(_PI64))
        return off, cell, g, t

    def mesh_cells(self):
        cells = np.zeros(4 * self.ncells, np.int32)
        maps = np.zeros(12 * self.ncells)
        self.lib.bo_mesh_cells(self.h, cells.ctypes.data_as(_PI32), _dp(maps), None)
        return cells.reshape(-1, 4), maps.reshape(-1, 12)

    def stencil_rows(self, form, level):
        rows = np.zeros(15 * self.ncells)
        diag = self.zeros(level)
        self._chk(self.lib.bo_compute_stencil(self.h, form, level, _dp(rows), _dp(diag)))
        return rows.reshape(-1, 15), diag

    def class_matrices(self, form, level, cell):
        out = np.zeros(96)
        self._chk(self.lib.bo_class_matrices(self.h, form, level, cell, _dp(out)))
        return out.reshape(6, 4, 4)

    def apply_stencil(self, level, x, bc=0, form=0):
        y = self.zeros(level)
        self._chk(self.lib.bo_apply_stencil(self.h, form, level, bc, _dp(np.ascontiguousarray(x)), _dp(y)))
        return y

    def apply_elementwise(self, level, x, form=2, kp=None, bc=0, y=None, add=False):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        y = self.zeros(level) if y is None else np.array(y, dtype=np.float64)
        self._chk(self.lib.bo_apply_elementwise(self.h, form, _dp(kp), level, int(add), bc,
                                                _dp(np.ascontiguousarray(x)), _dp(y)))
        return y

    def extract_diagonal(self, level, form=2, kp=None):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        d = self.zeros(level)
        self._chk(self.lib.bo_extract_diagonal(self.h, form, _dp(kp), level, _dp(d)))
        return d

    def prolongate(self, fine_level, coarse):
        f = self.zeros(fine_level)
        self.lib.bo_prolongate(self.h, fine_level, _dp(np.ascontiguousarray(coarse)), _dp(f))
        return f

    def restrict(self, fine_level, fine):
        c = self.zeros(fine_level - 1)
        self.lib.bo_restrict(self.h, fine_level, _dp(np.ascontiguousarray(fine)), _dp(c))
        return c

    def zero_dirichlet(self, level, x):
        x = np.array(x, dtype=np.float64)
        self.lib.bo_zero_dirichlet(self.h, level, _dp(x))
        return x

    # --- hierarchy / solvers
    def make_hierarchy(self, form=2, kp=None, kernel=0):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        if self._hier:
            self.lib.bo_hier_free(self._hier)
        self._hier = self.lib.bo_hier_new(self.h, form, _dp(kp), kernel)
        if not self._hier:
            raise ValueError(self.lib.bo_last_error().decode())

    def hier_apply(self, level, x, bc=1):
        y = self.zeros(level)
        self._chk(self.lib.bo_hier_apply(self._hier, level, bc, _dp(np.ascontiguousarray(x)), _dp(y)))
        return y

    def hier_diag(self, level):
        p = self.lib.bo_hier_diag(self._hier, level)
        return np.ctypeslib.as_array(p, shape=(self.size(0, level),)).copy()

    def lambda_max(self, level):
        return self.lib.bo_hier_lambda(self._hier, level)

    def smooth(self, level, sm, rhs, x, sweeps=1, backward=False):
        x = np.array(x, dtype=np.float64)
        self._chk(self.lib.bo_smooth(self._hier, _dp(_sm(sm)), level, sweeps, int(backward),
                                     _dp(np.ascontiguousarray(rhs)), _dp(x)))
        return x

    def cg(self, level, rhs, x, tol, maxit):
        x = np.array(x, dtype=np.float64)
        hist = np.zeros(max(maxit, 1))
        it = C.c_int()
        self._chk(self.lib.bo_cg(self._hier, level, tol, maxit, _dp(np.ascontiguousarray(rhs)), _dp(x),
                                 _dp(hist), C.byref(it)))
        return x, hist[: it.value]

    def vcycles(self, level, sm, rhs, x, cycles, coarse_level=2, coarse_tol=1e-12, coarse_maxit=4000):
        x = np.array(x, dtype=np.float64)
        hist = np.zeros(cycles + 1)
        self._chk(self.lib.bo_vcycles(self._hier, level, _dp(_sm(sm)), coarse_level, coarse_tol, coarse_maxit,
                                      cycles, _dp(np.ascontiguousarray(rhs)), _dp(x), _dp(hist)))
        return x, hist

    # --- N1E1 (restatement only; no reference)
    def n1e1_apply(self, level, x, alpha=1.0, beta=1.0, bc=1):
        y = self.zeros(level, space=2)
        self._chk(self.lib.bo_n1e1_apply(self.h, level, alpha, beta, bc, _dp(np.ascontiguousarray(x)), _dp(y)))
        return y

    def n1e1_sync(self, level, v):
        v = np.array(v, dtype=np.float64)
        self.lib.bo_n1e1_sync(self.h, level, _dp(v))
        return v

    def n1e1_random_fill(self, level, seed):
        v = self.zeros(level, space=2)
        self.lib.bo_n1e1_random_fill(self.h, level, seed, _dp(v))
        return v

    def n1e1_gradient(self, level, phi):
        u = self.zeros(level, space=2)
        self.lib.bo_n1e1_gradient(self.h, level, _dp(np.ascontiguousarray(phi)), _dp(u))
        return u

    def n1e1_constant_field(self, level, c3):
        u = self.zeros(level, space=2)
        self.lib.bo_n1e1_constant_field(self.h, level, _dp(np.asarray(c3, np.float64)), _dp(u))
        return u

    def n1e1_signs(self, level):
        off, cell, g, t = self.groups(level)
        s = np.zeros(len(cell), np.int8)
        self.lib.bo_n1e1_signs(self.h, level, s.ctypes.data_as(C.POINTER(C.c_int8)))
        return s

    def n1e1_local(self, corners, alpha=1.0, beta=1.0):
        out = np.zeros(36)
        self._chk(self.lib.bo_n1e1_local(_dp(np.asarray(corners, np.float64).ravel().copy()), alpha, beta, _dp(out)))
        return out.reshape(6, 6)


class Reference(_Base):
    """The compiled reference (oracle/_ref/libbtref.so)."""

    def __init__(self, mesh_text, lo, hi):
        self.lib = load_reference()
        self.h = self.lib.ref_new(mesh_text.encode(), lo, hi)
        if not self.h:
            raise ValueError(self.lib.ref_last_error().decode())
        self.lo, self.hi = lo, hi
        self.ncells = self.lib.ref_ncells(self.h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.ref_free(self.h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def size(self, space, level):
        return self.lib.ref_space_size(self.h, space, level)

    def random_fill(self, level, seed, space=0):
        x = self.zeros(level, space)
        self._chk(self.lib.ref_random_fill(self.h, space, level, seed, _dp(x)))
        return x

    def sync(self, level, v, broadcast=False, space=0):
        v = np.ascontiguousarray(v, dtype=np.float64).copy()
        self._chk(self.lib.ref_sync(self.h, space, level, int(broadcast), _dp(v)))
        return v

    def dot(self, level, x, y, space=0):
        return self.lib.ref_dot(self.h, space, level, _dp(np.ascontiguousarray(x)), _dp(np.ascontiguousarray(y)))

    def owned_count(self, level, space=0):
        return self.lib.ref_owned_dof_count(self.h, space, level)

    def masks(self, level, cell, g):
        n = n_tet(width_formula(g, level))
        o = np.zeros(n, np.uint8)
        d = np.zeros(n, np.uint8)
        self._chk(self.lib.ref_masks(self.h, level, cell, g, o.ctypes.data_as(_PU8), d.ctypes.data_as(_PU8)))
        return o, d

    def groups(self, level):
        m = C.c_int64()
        ng = self.lib.ref_group_count(self.h, level, C.byref(m))
        off = np.zeros(ng + 1, np.int64)
        cell = np.zeros(m.value, np.int32)
        g = np.zeros(m.value, np.int32)
        t = np.zeros(m.value, np.int64)
        self.lib.ref_groups(self.h, level, off.ctypes.data_as(_PI64), cell.ctypes.data_as(_PI32),
                            g.ctypes.data_as(_PI32), t.ctypes.data_as(_PI64))
        return off, cell, g, t

    def mesh_cells(self):
        nv, nc, nf, ne = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self.lib.ref_mesh_info(self.h, C.byref(nv), C.byref(nc), C.byref(nf), C.byref(ne), None, None, None)
        cells = np.zeros(4 * nc.value, np.int32)
        self.lib.ref_mesh_info(self.h, C.byref(nv), C.byref(nc), C.byref(nf), C.byref(ne),
                               cells.ctypes.data_as(_PI32), None, None)
        return cells.reshape(-1, 4)

    def stencil_rows(self, form, level):
        rows = np.zeros(15 * self.ncells)
        diag = self.zeros(level)
        self._chk(self.lib.ref_stencil_rows(self.h, form, level, _dp(rows), _dp(diag)))
        return rows.reshape(-1, 15), diag

    def class_matrices(self, form, level, cell):
        out = np.zeros(96)
        self._chk(self.lib.ref_class_matrices(self.h, form, level, cell, _dp(out)))
        return out.reshape(6, 4, 4)

    def apply_stencil(self, level, x, bc=0, form=0, threads=1):
        y = self.zeros(level)
        self._chk(self.lib.ref_apply_stencil(self.h, form, level, bc, _dp(np.ascontiguousarray(x)), _dp(y), threads))
        return y

    def apply_elementwise(self, level, x, form=2, kp=None, bc=0, y=None, add=False, threads=1):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        y = self.zeros(level) if y is None else np.array(y, dtype=np.float64)
        self._chk(self.lib.ref_apply_elementwise(self.h, form, _dp(kp), level, int(add), bc,
                                                 _dp(np.ascontiguousarray(x)), _dp(y), threads))
        return y

    def extract_diagonal(self, level, form=2, kp=None):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        d = self.zeros(level)
        self._chk(self.lib.ref_extract_diagonal(self.h, form, _dp(kp), level, _dp(d)))
        return d

    def prolongate(self, fine_level, coarse):
        f = self.zeros(fine_level)
        self._chk(self.lib.ref_prolongate(self.h, fine_level, _dp(np.ascontiguousarray(coarse)), _dp(f)))
        return f

    def restrict(self, fine_level, fine):
        c = self.zeros(fine_level - 1)
        self._chk(self.lib.ref_restrict(self.h, fine_level, _dp(np.ascontiguousarray(fine)), _dp(c)))
        return c

    def zero_dirichlet(self, level, x):
        x = np.array(x, dtype=np.float64)
        self._chk(self.lib.ref_zero_dirichlet(self.h, level, _dp(x)))
        return x

    def make_hierarchy(self, form=2, kp=None, kernel=0, threads=1):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        self._chk(self.lib.ref_hierarchy(self.h, form, _dp(kp), kernel, threads))

    def hier_apply(self, level, x, bc=1):
        y = self.zeros(level)
        self._chk(self.lib.ref_hierarchy_apply(self.h, level, bc, _dp(np.ascontiguousarray(x)), _dp(y)))
        return y

    def hier_diag(self, level):
        d = self.zeros(level)
        self._chk(self.lib.ref_hierarchy_diag(self.h, level, _dp(d)))
        return d

    def lambda_max(self, level):
        return self.lib.ref_lambda_max(self.h, level)

    def smooth(self, level, sm, rhs, x, sweeps=1, backward=False):
        x = np.array(x, dtype=np.float64)
        self._chk(self.lib.ref_smooth(self.h, _dp(_sm(sm)), level, sweeps, int(backward),
                                      _dp(np.ascontiguousarray(rhs)), _dp(x)))
        return x

    def cg(self, level, rhs, x, tol, maxit):
        x = np.array(x, dtype=np.float64)
        hist = np.zeros(max(maxit, 1))
        it = C.c_int()
        self._chk(self.lib.ref_cg(self.h, level, tol, maxit, _dp(np.ascontiguousarray(rhs)), _dp(x),
                                  _dp(hist), C.byref(it)))
        return x, hist[: it.value]

    def vcycles(self, level, sm, rhs, x, cycles, coarse_level=2, coarse_tol=1e-12, coarse_maxit=4000,
                seconds=None):
        x = np.array(x, dtype=np.float64)
        hist = np.zeros(cycles + 1)
        secs = np.zeros(cycles)
        self._chk(self.lib.ref_vcycles(self.h, level, _dp(_sm(sm)), coarse_level, coarse_tol, coarse_maxit,
                                       cycles, _dp(np.ascontiguousarray(rhs)), _dp(x), _dp(hist), _dp(secs)))
        if seconds is not None:
            seconds[:] = secs
        return x, hist

    def interpolate(self, level, fp):
        """fp = (kind, c0, c1, c2, c3) as kparams"""
        out = self.zeros(level)
        self._chk(self.lib.ref_interpolate(self.h, level, _dp(np.asarray(fp, np.float64)), _dp(out)))
        return out

    def l2_error(self, level, x, fp):
        out = np.zeros(1)
        self._chk(self.lib.ref_l2_error(self.h, level, _dp(np.ascontiguousarray(x)),
                                        _dp(np.asarray(fp, np.float64)), _dp(out)))
        return float(out[0])

    def fmg(self, finest, sm, rhs_levels, coarse_level, cycles, coarse_tol=1e-12, coarse_maxit=4000, fp=None):
        """rows (level, cycle, residual, error) and the finest solution"""
        rhs = np.ascontiguousarray(np.concatenate(rhs_levels))
        x = self.zeros(finest)
        rows = np.zeros(4 * (1 + cycles * (finest - coarse_level)))
        n = C.c_int()
        fpa = _dp(np.asarray(fp, np.float64)) if fp is not None else None
        self._chk(self.lib.ref_fmg(self.h, finest, _dp(_sm(sm)), coarse_level, coarse_tol, coarse_maxit, cycles,
                                   _dp(rhs), _dp(x), fpa, _dp(rows), C.byref(n)))
        return rows[: 4 * n.value].reshape(-1, 4), x

    def time_apply(self, level, x, kind=0, form=0, kp=None, bc=0, reps=3, threads=1):
        kp = kparams() if kp is None else np.asarray(kp, np.float64)
        return self.lib.ref_time_apply(self.h, kind, form, _dp(kp), level, bc, reps, threads,
                                       _dp(np.ascontiguousarray(x)))


# ---- builtin meshes (coarse_mesh.hpp:335-368, restated as text) ----------

def ref_tet_text():
    return "# reference tetrahedron\nvertices 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ncells 1\n0 1 2 3\n"


def cube_kuhn_text():
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


def cubes_mesh_text(n, perturb=0.1, seed=0):
    """Oracle's n^3-cube Kuhn mesh generator (builder decision)."""
    lib = load_oracle()
    need = lib.bo_cubes_mesh_text(n, perturb, seed, None, 0)
    buf = C.create_string_buffer(need + 1)
    lib.bo_cubes_mesh_text(n, perturb, seed, buf, need + 1)
    return buf.value.decode()


TWO_TETS = "vertices 5\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n1 1 1\ncells 2\n0 1 2 3\n1 2 3 4\n"
