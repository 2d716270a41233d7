"""Thin ctypes binding of libfed.so (include/fed.h) -- argument marshalling only.

Every step of the FED-FEM path runs in the library's sm_100a kernels; this
module only converts numpy arrays / problem descriptions into the C structs
and raises on non-zero status.  There is no CPU fallback: if libfed.so is
missing or a CUDA device is unavailable the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FED_LIB selects another build of the same ABI (e.g. libfed_checked.so, the build
# with device-side bounds / colour-race checks)
LIB_PATH = os.environ.get("FED_LIB") or os.path.join(_HERE, "libfed.so")

FED_OK, FED_ERR_INVALID, FED_ERR_MESH, FED_ERR_NOMEM = 0, 1, 2, 3
FED_ERR_CUDA, FED_ERR_NCCL, FED_ERR_UNSTABLE, FED_ERR_STATE = 4, 5, 6, 7
FED_BC_FLUX, FED_BC_CONV, FED_BC_RAD = 1, 2, 3
FED_SCATTER_AUTO, FED_SCATTER_ATOMIC, FED_SCATTER_CHUNK, FED_SCATTER_CHUNK_CAS = 0, 1, 2, 3
FED_SCATTER_CHUNK_REG, FED_SCATTER_CHUNK_REGC = 4, 5
FED_SCATTER_ATOMIC_WARP, FED_SCATTER_COLOR_PASSES, FED_SCATTER_GATHER = 6, 7, 8
FED_TRANSPORT_NCCL, FED_TRANSPORT_PEER = 0, 1

EXPORTED = ("fed_options_default", "fed_create", "fed_step", "fed_run_until_steady", "fed_get_temperature", "fed_set_temperature",
            "fed_get_info", "fed_set_timing", "fed_get_timing", "fed_get_rank_timing", "fed_nccl_unique_id", "fed_debug_plan",
            "fed_debug_chunks", "fed_debug_nodal", "fed_debug_dataflow", "fed_debug_gather", "fed_debug_time_rank",
            "fed_last_error", "fed_destroy")


class FedError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"fed status {status}: {msg}")
        self.status = status


class fed_mesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_elems", C.c_int64), ("n_faces", C.c_int64),
                ("xyz", C.c_void_p), ("conn", C.c_void_p), ("faces", C.c_void_p), ("face_bc", C.c_void_p),
                ("nodes_per_elem", C.c_int32), ("nodes_per_face", C.c_int32)]


class fed_material(C.Structure):
    _fields_ = [("rho", C.c_double), ("c0", C.c_double), ("beta_c", C.c_double),
                ("D_ref", C.c_double * 6), ("beta_k", C.c_double),
                ("n_k_table", C.c_int32), ("k_table_T", C.c_void_p), ("k_table_val", C.c_void_p),
                ("n_c_table", C.c_int32), ("c_table_T", C.c_void_p), ("c_table_val", C.c_void_p)]


class fed_face_bc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("q", C.c_double), ("h", C.c_double), ("T_inf", C.c_double),
                ("eps", C.c_double), ("area_mode", C.c_int32)]


class fed_bcs(C.Structure):
    _fields_ = [("n_face_bcs", C.c_int32), ("face_bcs", C.c_void_p), ("n_dirichlet", C.c_int64),
                ("dir_nodes", C.c_void_p), ("dir_T", C.c_void_p), ("q_vol", C.c_void_p), ("T0", C.c_void_p)]


# device-memory hook of fed_options (fed.h): void *alloc(size_t, int32 device, void *ctx),
# void free(void *ptr, size_t, int32 device, void *ctx)
DEV_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
DEV_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)


class fed_options(C.Structure):
    _fields_ = [("precision", C.c_int32), ("dt", C.c_double), ("dt_factor", C.c_double),
                ("T_lo", C.c_double), ("T_hi", C.c_double), ("T_abort", C.c_double),
                ("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_id", C.c_void_p), ("scatter", C.c_int32), ("chunk_elems", C.c_int32),
                ("graph_steps", C.c_int32), ("transport", C.c_int32), ("local_ranks", C.c_int32),
                ("resident", C.c_int32), ("dev_alloc", DEV_ALLOC), ("dev_free", DEV_FREE),
                ("alloc_ctx", C.c_void_p), ("wait_timeout_s", C.c_double),
                ("chunk_order", C.c_int32)]


class fed_info(C.Structure):
    _fields_ = [("dt", C.c_double), ("dt_crit", C.c_double), ("step", C.c_int64), ("t", C.c_double),
                ("fail_step", C.c_int64), ("precision", C.c_int32), ("scatter", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("temperature_dependent", C.c_int32),
                ("n_nodes_global", C.c_int64), ("n_elems_global", C.c_int64),
                ("n_nodes_local", C.c_int64), ("n_elems_local", C.c_int64),
                ("n_interior", C.c_int64), ("n_special", C.c_int64), ("n_interface", C.c_int64),
                ("n_chunks", C.c_int64), ("n_chunks_interface", C.c_int64), ("n_bc_entries", C.c_int64),
                ("max_colors", C.c_int32), ("chunk_elems", C.c_int32),
                ("kernel_launches_per_step", C.c_int64), ("kernel_launches_total", C.c_int64),
                ("device_bytes", C.c_int64), ("nodes_per_elem", C.c_int32), ("colored", C.c_int32),
                ("resident", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class fed_timing(C.Structure):
    _fields_ = [("element_ms", C.c_double), ("node_ms", C.c_double), ("exchange_ms", C.c_double),
                ("element_launches", C.c_int64), ("node_launches", C.c_int64), ("exchange_count", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load(path: str = LIB_PATH):
    """Load libfed.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built; run `python -m paper_1909_03355_b200.build`")
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.fed_options_default.argtypes = [P]
    lib.fed_options_default.restype = None
    lib.fed_create.argtypes = [P, P, P, P, C.POINTER(C.c_void_p)]
    lib.fed_step.argtypes = [P, C.c_int64]
    lib.fed_run_until_steady.argtypes = [P, C.c_double, C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_double)]
    lib.fed_run_until_steady.restype = C.c_int
    lib.fed_get_temperature.argtypes = [P, P, C.c_int64]
    lib.fed_set_temperature.argtypes = [P, P, C.c_int64]
    lib.fed_get_info.argtypes = [P, P]
    lib.fed_set_timing.argtypes = [P, C.c_int32]
    lib.fed_get_timing.argtypes = [P, P]
    lib.fed_get_rank_timing.argtypes = [P, C.c_int32, P]
    lib.fed_nccl_unique_id.argtypes = [P]
    lib.fed_debug_plan.argtypes = [P, P, P, P, P, P]
    lib.fed_debug_nodal.argtypes = [P, P, P, C.c_int64]
    lib.fed_debug_dataflow.argtypes = [P, P, P, P, P, P, P, P]
    lib.fed_debug_chunks.argtypes = [P, P, P, P, P]
    lib.fed_debug_gather.argtypes = [P, P, P, P, P]
    lib.fed_debug_time_rank.argtypes = [P, C.c_int32, C.c_int64, C.POINTER(C.c_double)]
    lib.fed_last_error.argtypes = []
    lib.fed_last_error.restype = C.c_char_p
    lib.fed_destroy.argtypes = [P]
    lib.fed_destroy.restype = None
    for nm in ("fed_create", "fed_step", "fed_get_temperature", "fed_set_temperature", "fed_get_info",
               "fed_set_timing", "fed_get_timing", "fed_get_rank_timing", "fed_nccl_unique_id", "fed_debug_plan", "fed_debug_nodal",
               "fed_debug_dataflow", "fed_debug_gather", "fed_debug_time_rank",
               "fed_debug_chunks"):
        getattr(lib, nm).restype = C.c_int
    _lib = lib
    return lib


def _check(st):
    if st != FED_OK:
        raise FedError(st, load().fed_last_error().decode())


def fed_last_error() -> str:
    return load().fed_last_error().decode()


def fed_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().fed_nccl_unique_id(buf))
    return buf.raw


def torch_allocator():
    """(dev_alloc, dev_free) hooks backed by PyTorch's CUDA caching allocator, so a
    torch-hosted caller pools the context's device memory with its own tensors
    (fed.h fed_options.dev_alloc).  Marshalling only: the allocations are made by
    torch.cuda.caching_allocator_alloc / caching_allocator_delete."""
    import torch

    def _alloc(nbytes, device, _ctx):
        try:
            with torch.cuda.device(int(device)):
                return int(torch.cuda.caching_allocator_alloc(int(nbytes), int(device)))
        except Exception:
            return None

    def _free(ptr, _nbytes, _device, _ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    return DEV_ALLOC(_alloc), DEV_FREE(_free)


def options(**kw) -> fed_options:
    """fed_options with fed_options_default(), then the given fields.  Extra keys:
    nccl_id (bytes), torch_alloc=True (device memory from torch's allocator)."""
    o = fed_options()
    load().fed_options_default(C.byref(o))
    for k, v in kw.items():
        if k == "nccl_id" and v is not None and not isinstance(v, int):
            o._nccl_buf = C.create_string_buffer(bytes(v), 128)   # keep alive with o
            v = C.addressof(o._nccl_buf)
        if k == "torch_alloc":
            if v:
                o._hooks = torch_allocator()                      # keep the callbacks alive with o
                o.dev_alloc, o.dev_free = o._hooks
            continue
        setattr(o, k, v)
    return o


class Fed:
    """Owner of one fed_ctx.  Arguments are numpy arrays in the layout of fed.h."""

    def __init__(self, xyz, conn, faces=None, face_bc=None, face_bcs=(), dir_nodes=None, dir_T=None,
                 q_vol=None, T0=None, material=None, opts: Optional[fed_options] = None, nodes_per_face=None,
                 **opt_kw):
        lib = load()
        self._keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a

        xyz = arr(xyz, np.float64)
        conn = arr(conn, np.int32)
        npe = int(conn.shape[1])
        npf = int(nodes_per_face) if nodes_per_face else (4 if npe == 8 else 3)
        nf = 0 if faces is None else int(np.asarray(faces).reshape(-1, npf).shape[0])
        faces = arr(np.asarray(faces).reshape(-1, npf), np.int32) if nf else None
        face_bc = arr(face_bc, np.int32) if nf else None
        m = fed_mesh(int(xyz.shape[0]), int(conn.shape[0]), nf, xyz.ctypes.data, conn.ctypes.data,
                     faces.ctypes.data if nf else None, face_bc.ctypes.data if nf else None, npe, npf)
        mat = fed_material()
        mat.rho, mat.c0, mat.beta_c, mat.beta_k = material.rho, material.c0, material.beta_c, material.beta_k
        for i in range(6):
            mat.D_ref[i] = material.D_ref[i]
        kt = getattr(material, "k_table", None)
        ct = getattr(material, "c_table", None)
        if kt is not None:
            kT, kv = arr(kt[0], np.float64), arr(kt[1], np.float64)
            mat.n_k_table, mat.k_table_T, mat.k_table_val = int(kT.size), kT.ctypes.data, kv.ctypes.data
        if ct is not None:
            cT, cv = arr(ct[0], np.float64), arr(ct[1], np.float64)
            mat.n_c_table, mat.c_table_T, mat.c_table_val = int(cT.size), cT.ctypes.data, cv.ctypes.data
        nb = len(face_bcs)
        bc_arr = (fed_face_bc * max(nb, 1))()
        for i, b in enumerate(face_bcs):
            bc_arr[i] = fed_face_bc(int(b.kind), float(b.q), float(b.h), float(b.T_inf), float(b.eps),
                                    int(getattr(b, "area_mode", 0)))
        self._keep.append(bc_arr)
        dn = arr(dir_nodes, np.int32) if dir_nodes is not None and len(dir_nodes) else None
        dT = arr(dir_T, np.float64) if dn is not None else None
        qv = arr(q_vol, np.float64)
        t0 = arr(T0, np.float64)
        b = fed_bcs(nb, C.addressof(bc_arr), 0 if dn is None else int(dn.shape[0]),
                    None if dn is None else dn.ctypes.data, None if dT is None else dT.ctypes.data,
                    None if qv is None else qv.ctypes.data, None if t0 is None else t0.ctypes.data)
        o = opts if opts is not None else options(**opt_kw)
        self.opts = o
        h = C.c_void_p()
        _check(lib.fed_create(C.byref(m), C.byref(mat), C.byref(b), C.byref(o), C.byref(h)))
        self._h = h
        self.n_nodes = int(xyz.shape[0])
        self._keep = []

    @classmethod
    def from_problem(cls, prob, **opt_kw):
        """Marshal a fed_inputs.Problem (problem statement only)."""
        kw = dict(T_lo=prob.T_lo, T_hi=prob.T_hi, dt_factor=prob.dt_factor)
        kw.update(opt_kw)
        return cls(prob.xyz, prob.conn, prob.faces, prob.face_bc, prob.face_bcs, prob.dir_nodes, prob.dir_T,
                   prob.q_vol, prob.T0, prob.material, nodes_per_face=getattr(prob, "nodes_per_face", None), **kw)

    def close(self):
        if getattr(self, "_h", None):
            load().fed_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def step(self, n: int = 1):
        _check(load().fed_step(self._h, int(n)))

    def run_until_steady(self, tol: float = 1e-3, max_steps: int = 1_000_000, check_every: int = 100):
        """Steady-state mode: returns (steps_taken, last max |dT|)."""
        n = C.c_int64(0)
        d = C.c_double(0)
        _check(load().fed_run_until_steady(self._h, float(tol), int(max_steps), int(check_every), C.byref(n),
                                           C.byref(d)))
        return n.value, d.value

    def temperature(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.n_nodes, dtype=np.float64)
        _check(load().fed_get_temperature(self._h, out.ctypes.data, self.n_nodes))
        return out

    def set_temperature(self, T):
        a = np.ascontiguousarray(T, dtype=np.float64)
        _check(load().fed_set_temperature(self._h, a.ctypes.data, self.n_nodes))

    def info(self) -> dict:
        i = fed_info()
        _check(load().fed_get_info(self._h, C.byref(i)))
        return i.as_dict()

    def set_timing(self, on: bool):
        _check(load().fed_set_timing(self._h, 1 if on else 0))

    def timing(self) -> dict:
        t = fed_timing()
        _check(load().fed_get_timing(self._h, C.byref(t)))
        return t.as_dict()

    def rank_timing(self, rank: int) -> dict:
        """Kernel times of one slab of a local_ranks group (rank 0 of a single context)."""
        t = fed_timing()
        _check(load().fed_get_rank_timing(self._h, int(rank), C.byref(t)))
        return t.as_dict()

    def debug_plan(self):
        lib = load()
        ns = C.c_int64(0)
        _check(lib.fed_debug_plan(self._h, None, C.byref(ns), None, None, None))
        node_map = np.empty(self.n_nodes, np.int32)
        ch = np.empty(ns.value, np.int32)
        co = np.empty(ns.value, np.int32)
        el = np.empty(ns.value, np.int32)
        _check(lib.fed_debug_plan(self._h, node_map.ctypes.data, C.byref(ns), ch.ctypes.data, co.ctypes.data,
                                  el.ctypes.data))
        return {"node_map": node_map, "slot_chunk": ch, "slot_color": co, "slot_elem": el}

    def debug_chunks(self):
        lib = load()
        nc = C.c_int64(0)
        ns = C.c_int64(0)
        _check(lib.fed_debug_chunks(self._h, C.byref(nc), None, None, None))
        _check(lib.fed_debug_plan(self._h, None, C.byref(ns), None, None, None))
        hdr = np.empty((nc.value, 8), np.int32)
        col = np.empty((nc.value, 33), np.int32)
        c16 = np.empty((ns.value, self.info()["nodes_per_elem"]), np.uint16)
        _check(lib.fed_debug_chunks(self._h, C.byref(nc), hdr.ctypes.data, col.ctypes.data, c16.ctypes.data))
        return hdr, col, c16

    def debug_dataflow(self):
        """Resident/flow dataflow tables: (adj_ptr, adj, sp_list, sp_own) or None."""
        lib = load()
        nc, na, ns = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        _check(lib.fed_debug_dataflow(self._h, C.byref(nc), C.byref(na), C.byref(ns), None, None, None, None))
        if nc.value == 0:
            return None
        ptr = np.empty(nc.value + 1, np.int32)
        adj = np.empty(max(1, na.value), np.int32)
        spl = np.empty(max(1, ns.value), np.int32)
        own = np.empty(max(1, ns.value), np.uint8)
        _check(lib.fed_debug_dataflow(self._h, None, None, None, ptr.ctypes.data, adj.ctypes.data, spl.ctypes.data,
                                      own.ctypes.data))
        return ptr, adj[:na.value], spl[:ns.value], own[:ns.value]

    def debug_nodal(self):
        V = np.empty(self.n_nodes)
        c = np.empty(self.n_nodes)
        _check(load().fed_debug_nodal(self._h, V.ctypes.data, c.ctypes.data, self.n_nodes))
        return V, c

    def debug_gather(self):
        """Multi-rank readout layout: (slice offsets, caller ids by owner rank, this
        rank's pack list of internal ids); None for a single-rank context."""
        lib = load()
        P = C.c_int32(0)
        _check(lib.fed_debug_gather(self._h, C.byref(P), None, None, None))
        if P.value == 0:
            return None
        off = np.empty(P.value + 1, np.int64)
        _check(lib.fed_debug_gather(self._h, C.byref(P), off.ctypes.data, None, None))
        ids = np.empty(int(off[-1]), np.int32)
        r = self.info()["rank"]
        pack = np.empty(int(off[r + 1] - off[r]), np.int32)
        _check(lib.fed_debug_gather(self._h, C.byref(P), off.ctypes.data, ids.ctypes.data, pack.ctypes.data))
        return off, ids, pack

    def debug_time_rank(self, rank: int, n_steps: int) -> float:
        """ms per step of slab `rank` of a local rank group stepped alone (timing only;
        the field is undefined afterwards)."""
        ms = C.c_double(0)
        _check(load().fed_debug_time_rank(self._h, int(rank), int(n_steps), C.byref(ms)))
        return ms.value
