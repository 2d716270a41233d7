"""ctypes wrapper of oracle/fed_oracle.c (plain fp64, single thread).

TEST INFRASTRUCTURE ONLY -- see the header of fed_oracle.c.  The C file is
compiled with plain `gcc -O2` (no fast-math, no OpenMP) into
oracle/libfed_oracle.so on first use.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fed_oracle.c")
_LIB = os.path.join(_HERE, "libfed_oracle.so")
_lock = threading.Lock()
_lib = None

ORA_OK, ORA_ERR_UNSTABLE = 0, 6


def build_oracle(force: bool = False) -> str:
    """Compile fed_oracle.c -> libfed_oracle.so (idempotent)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


class _Problem(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64), ("n_elems", C.c_int64), ("n_faces", C.c_int64),
        ("xyz", C.c_void_p), ("conn", C.c_void_p), ("faces", C.c_void_p), ("face_bc", C.c_void_p),
        ("n_face_bcs", C.c_int32),
        ("bc_kind", C.c_void_p), ("bc_q", C.c_void_p), ("bc_h", C.c_void_p),
        ("bc_Tinf", C.c_void_p), ("bc_eps", C.c_void_p),
        ("n_dir", C.c_int64), ("dir_nodes", C.c_void_p), ("dir_T", C.c_void_p),
        ("q_vol", C.c_void_p), ("T0", C.c_void_p),
        ("rho", C.c_double), ("c0", C.c_double), ("beta_c", C.c_double),
        ("D_ref", C.c_double * 6), ("beta_k", C.c_double),
        ("nodes_per_elem", C.c_int32), ("nodes_per_face", C.c_int32),
        ("n_k", C.c_int32), ("k_T", C.c_void_p), ("k_v", C.c_void_p),
        ("n_c", C.c_int32), ("c_T", C.c_void_p), ("c_v", C.c_void_p),
        ("bc_area_mode", C.c_void_p),
    ]


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build_oracle())
        P = C.c_void_p
        lib.ora_hex_kernel.argtypes = [P, P, P, P]
        lib.ora_hex_kernel.restype = C.c_int
        lib.ora_build_G.argtypes = [P, C.c_double, P]
        lib.ora_element_load.argtypes = [P, P, P, P, P]
        lib.ora_quad_area.argtypes = [P, P]
        lib.ora_quad_area.restype = C.c_double
        lib.ora_sym_max_eig.argtypes = [P, C.c_int]
        lib.ora_sym_max_eig.restype = C.c_double
        lib.ora_element_lambda8.argtypes = [P, P, C.c_double]
        lib.ora_element_lambda8.restype = C.c_double
        lib.ora_tet_lambda.argtypes = [P, P, C.c_double]
        lib.ora_tet_lambda.restype = C.c_double
        lib.ora_tet_kernel.argtypes = [P, P, P]
        lib.ora_tet_kernel.restype = C.c_int
        lib.ora_build_G_n.argtypes = [P, C.c_double, P, C.c_int]
        lib.ora_element_load_n.argtypes = [P, P, P, P, P, C.c_int]
        lib.ora_table_eval.argtypes = [P, P, C.c_int, C.c_double]
        lib.ora_table_eval.restype = C.c_double
        lib.ora_tri_area.argtypes = [P, P]
        lib.ora_tri_area.restype = C.c_double
        lib.ora_dt_crit.argtypes = [P, C.c_double, C.c_double]
        lib.ora_dt_crit.restype = C.c_double
        lib.ora_create.argtypes = [P, C.c_double, C.POINTER(C.c_int)]
        lib.ora_create.restype = C.c_void_p
        lib.ora_destroy.argtypes = [P]
        lib.ora_step.argtypes = [P, C.c_int64]
        lib.ora_step.restype = C.c_int
        for nm in ("ora_get_T", "ora_set_T", "ora_get_mass", "ora_get_F", "ora_get_Q"):
            getattr(lib, nm).argtypes = [P, P]
        lib.ora_get_step.argtypes = [P]
        lib.ora_get_step.restype = C.c_int64
        lib.ora_compute_loads.argtypes = [P, P, P, P]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class _Packed:
    """Keeps the numpy buffers alive while C reads them."""

    def __init__(self, prob, T0=None):
        self.xyz = _c(prob.xyz, np.float64)
        self.conn = _c(prob.conn, np.int32)
        npf = 3 if getattr(prob, "nodes_per_face", 4) == 3 else 4
        self.faces = _c(prob.faces.reshape(-1, npf) if prob.faces.size else np.zeros((0, npf)), np.int32)
        self.face_bc = _c(prob.face_bc if prob.face_bc.size else np.zeros(0), np.int32)
        bcs = prob.face_bcs
        self.kind = _c([b.kind for b in bcs] or [0], np.int32)
        self.q = _c([b.q for b in bcs] or [0], np.float64)
        self.h = _c([b.h for b in bcs] or [0], np.float64)
        self.Ti = _c([b.T_inf for b in bcs] or [0], np.float64)
        self.eps = _c([b.eps for b in bcs] or [0], np.float64)
        self.amode = _c([getattr(b, "area_mode", 0) for b in bcs] or [0], np.int32)
        self.dn = _c(prob.dir_nodes if prob.dir_nodes.size else np.zeros(0), np.int32)
        self.dT = _c(prob.dir_T if prob.dir_T.size else np.zeros(0), np.float64)
        self.qv = None if prob.q_vol is None else _c(prob.q_vol, np.float64)
        self.T0 = _c(prob.T0 if T0 is None else T0, np.float64)
        m = prob.material
        s = _Problem()
        s.n_nodes, s.n_elems, s.n_faces = self.xyz.shape[0], self.conn.shape[0], self.faces.shape[0]
        s.xyz, s.conn, s.faces, s.face_bc = _ptr(self.xyz), _ptr(self.conn), _ptr(self.faces), _ptr(self.face_bc)
        s.n_face_bcs = len(bcs)
        s.bc_kind, s.bc_q, s.bc_h = _ptr(self.kind), _ptr(self.q), _ptr(self.h)
        s.bc_Tinf, s.bc_eps = _ptr(self.Ti), _ptr(self.eps)
        s.bc_area_mode = _ptr(self.amode)
        s.n_dir = self.dn.shape[0]
        s.dir_nodes, s.dir_T = _ptr(self.dn), _ptr(self.dT)
        s.q_vol = _ptr(self.qv)
        s.T0 = _ptr(self.T0)
        s.rho, s.c0, s.beta_c, s.beta_k = m.rho, m.c0, m.beta_c, m.beta_k
        for i in range(6):
            s.D_ref[i] = m.D_ref[i]
        s.nodes_per_elem = int(self.conn.shape[1])
        s.nodes_per_face = npf
        kt = getattr(m, "k_table", None)
        ct = getattr(m, "c_table", None)
        self.kT = None if kt is None else _c(kt[0], np.float64)
        self.kv = None if kt is None else _c(kt[1], np.float64)
        self.cT = None if ct is None else _c(ct[0], np.float64)
        self.cv = None if ct is None else _c(ct[1], np.float64)
        s.n_k = 0 if kt is None else int(self.kT.size)
        s.k_T, s.k_v = _ptr(self.kT), _ptr(self.kv)
        s.n_c = 0 if ct is None else int(self.cT.size)
        s.c_T, s.c_v = _ptr(self.cT), _ptr(self.cv)
        self.s = s


def dt_crit(prob, T_lo=None, T_hi=None) -> float:
    """Element-bound critical step over [T_lo, T_hi] (reading 8c-13)."""
    lib = _load()
    pk = _Packed(prob)
    lo = prob.T_lo if T_lo is None else T_lo
    hi = prob.T_hi if T_hi is None else T_hi
    return float(lib.ora_dt_crit(C.byref(pk.s), lo, hi))


class Oracle:
    """Stateful oracle run: create (stages i, ii), step (stage iii), read T."""

    def __init__(self, prob, dt: float, T0=None):
        lib = _load()
        self._pk = _Packed(prob, T0)
        err = C.c_int(0)
        self._h = lib.ora_create(C.byref(self._pk.s), float(dt), C.byref(err))
        if not self._h:
            raise ValueError(f"oracle create failed: status {err.value}")
        self.N = prob.n_nodes
        self.dt = float(dt)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _load().ora_destroy(h)
            self._h = None

    def step(self, n: int = 1) -> int:
        return int(_load().ora_step(self._h, int(n)))

    def _get(self, fn):
        out = np.empty(self.N, dtype=np.float64)
        getattr(_load(), fn)(self._h, out.ctypes.data)
        return out

    def T(self):
        return self._get("ora_get_T")

    def mass(self):
        return self._get("ora_get_mass")

    def set_T(self, T):
        a = _c(T, np.float64)
        _load().ora_set_T(self._h, a.ctypes.data)

    def loads(self, T):
        """(F_int, Q) at the field T, without stepping."""
        a = _c(T, np.float64)
        F = np.empty(self.N)
        Q = np.empty(self.N)
        _load().ora_compute_loads(self._h, a.ctypes.data, F.ctypes.data, Q.ctypes.data)
        return F, Q

    @property
    def step_index(self) -> int:
        return int(_load().ora_get_step(self._h))


def hex_kernel(x8):
    """(B 3x8, scale = 8 det J, det J) of one hex (Eq. 17)."""
    lib = _load()
    x = _c(x8, np.float64).reshape(8, 3)
    B = np.empty((3, 8))
    sc = C.c_double(0)
    det = C.c_double(0)
    st = lib.ora_hex_kernel(x.ctypes.data, B.ctypes.data, C.addressof(sc), C.addressof(det))
    if st != 0:
        raise ValueError("degenerate hex")
    return B, sc.value, det.value


def build_G(B, scale):
    lib = _load()
    Bc = _c(B, np.float64)
    G = np.empty((8, 3))
    lib.ora_build_G(Bc.ctypes.data, float(scale), G.ctypes.data)
    return G


def element_load(B, G, D3x3, Te):
    lib = _load()
    Bc, Gc, Dc, Tc = _c(B, np.float64), _c(G, np.float64), _c(D3x3, np.float64), _c(Te, np.float64)
    F = np.empty(8)
    lib.ora_element_load(Bc.ctypes.data, Gc.ctypes.data, Dc.ctypes.data, Tc.ctypes.data, F.ctypes.data)
    return F


def quad_area(xyz, f4):
    lib = _load()
    x = _c(xyz, np.float64)
    f = _c(f4, np.int32)
    return float(lib.ora_quad_area(x.ctypes.data, f.ctypes.data))


def sym_max_eig(A):
    lib = _load()
    a = _c(A, np.float64)
    return float(lib.ora_sym_max_eig(a.ctypes.data, a.shape[0]))


def element_lambda8(x8, D6, rhoc):
    lib = _load()
    x = _c(x8, np.float64)
    d = _c(D6, np.float64)
    return float(lib.ora_element_lambda8(x.ctypes.data, d.ctypes.data, float(rhoc)))


def tet_kernel(x4):
    """(B 3x4, V) of one linear tetrahedron (Eq. 18)."""
    lib = _load()
    x = _c(x4, np.float64).reshape(4, 3)
    B = np.empty((3, 4))
    V = C.c_double(0)
    if lib.ora_tet_kernel(x.ctypes.data, B.ctypes.data, C.addressof(V)) != 0:
        raise ValueError("degenerate or inverted tet")
    return B, V.value


def element_load_n(B, G, D3x3, Te):
    lib = _load()
    npe = int(np.asarray(Te).size)
    Bc, Gc, Dc, Tc = _c(B, np.float64), _c(G, np.float64), _c(D3x3, np.float64), _c(Te, np.float64)
    F = np.empty(npe)
    lib.ora_element_load_n(Bc.ctypes.data, Gc.ctypes.data, Dc.ctypes.data, Tc.ctypes.data, F.ctypes.data, npe)
    return F


def build_G_n(B, scale):
    lib = _load()
    Bc = _c(B, np.float64)
    npe = Bc.shape[1]
    G = np.empty((npe, 3))
    lib.ora_build_G_n(Bc.ctypes.data, float(scale), G.ctypes.data, npe)
    return G


def tet_lambda(x4, D6, rhoc):
    lib = _load()
    x = _c(x4, np.float64)
    d = _c(D6, np.float64)
    return float(lib.ora_tet_lambda(x.ctypes.data, d.ctypes.data, float(rhoc)))


def tri_area(xyz, f3):
    lib = _load()
    x = _c(xyz, np.float64)
    f = _c(f3, np.int32)
    return float(lib.ora_tri_area(x.ctypes.data, f.ctypes.data))


def table_eval(Tt, vt, T):
    """Piecewise-linear, end-clamped property table."""
    lib = _load()
    a, b = _c(Tt, np.float64), _c(vt, np.float64)
    return float(lib.ora_table_eval(a.ctypes.data, b.ctypes.data, int(a.size), float(T)))
