"""Seeded synthetic problem generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the FED-FEM method (no Jacobians, no
element operators, no lumping, no time step, no boundary loads).  It only
writes down the *problem statement* of each BASELINE.json config -- mesh
coordinates and connectivity, boundary-face lists, material parameters,
boundary records, initial field and source density -- as plain numpy arrays.
Both `oracle/` and `paper_1909_03355_b200/` consume these arrays through
their own, independent code.

Conventions:
  * hex8 corner order: bottom face counter-clockwise seen from +zeta, then
    the top face above it.  Natural signs of corner a:
    (---),(+--),(++-),(-+-),(--+),(+-+),(+++),(-++).
  * natural numbering is x-fastest: node id = i + (nx+1)*(j + (ny+1)*k),
    element id = i + nx*(j + ny*k)
  * boundary-condition kinds: FLUX=1 (W/m^2 into the body), CONV=2 (h, T_inf),
    RAD=3 (eps, T_inf) -- PAPER.md Eqs. 4, 5, 7, signs per 8c-11.
  * "edge 0.1 m": cfg1 element edge 0.1 m (1 m cube); cfg2-5 cube edge 0.1 m
    (SURVEY.md 8c-15).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

BC_FLUX, BC_CONV, BC_RAD = 1, 2, 3

SIDES = ("x0", "x1", "y0", "y1", "z0", "z1")


@dataclass
class FaceBC:
    kind: int
    q: float = 0.0       # W/m^2 (FLUX)
    h: float = 0.0       # W/(m^2 K) (CONV)
    T_inf: float = 0.0   # degC (CONV, RAD)
    eps: float = 0.0     # emissivity (RAD)
    area_mode: int = 0   # 0: corners get A_f/n; 1: uniform nodal area per record (NEXT-3)


@dataclass
class Material:
    rho: float
    c0: float
    beta_c: float          # c(T) = c0*(1+beta_c*T)
    D_ref: tuple           # (xx, yy, zz, xy, yz, xz) W/(m K)
    beta_k: float          # D(T) = D_ref*(1+beta_k*T)
    # NEXT-2: piecewise-linear tables ((T...), (value...)), clamped at the ends;
    # k_table multiplies D_ref (replaces 1+beta_k T), c_table replaces c0(1+beta_c T)
    k_table: Optional[tuple] = None
    c_table: Optional[tuple] = None


@dataclass
class Problem:
    name: str
    xyz: np.ndarray                 # (N,3) float64, metres
    conn: np.ndarray                # (E,8) int32
    faces: np.ndarray               # (F,4) int32 boundary quads
    face_bc: np.ndarray             # (F,)  int32 index into face_bcs, -1 adiabatic
    face_bcs: List[FaceBC]
    dir_nodes: np.ndarray           # (D,) int32
    dir_T: np.ndarray               # (D,) float64
    q_vol: Optional[np.ndarray]     # (N,) float64 W/m^3 at nodes, or None
    T0: np.ndarray                  # (N,) float64 degC
    material: Material
    steps: int
    precisions: tuple               # e.g. (64,) or (32, 64)
    T_lo: float                     # temperature range for the TD critical step
    T_hi: float
    dt_factor: float = 0.9
    grid: tuple = ()                # (nx, ny, nz) for structured meshes
    meta: dict = field(default_factory=dict)
    nodes_per_face: int = 4         # 4 (quads, hex meshes) or 3 (triangles, tet meshes)

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_elems(self) -> int:
        return int(self.conn.shape[0])


# ----------------------------------------------------------------------------
# structured meshes
# ----------------------------------------------------------------------------

def grid_nodes(nx, ny, nz, Lx, Ly, Lz):
    """(N,3) coordinates of an (nx+1)(ny+1)(nz+1) lattice, x-fastest."""
    xs = np.linspace(0.0, Lx, nx + 1)
    ys = np.linspace(0.0, Ly, ny + 1)
    zs = np.linspace(0.0, Lz, nz + 1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)


def grid_conn(nx, ny, nz):
    """(E,8) int32 hex8 connectivity in S:93 order, element id x-fastest."""
    sx, sy = 1, nx + 1
    sz = (nx + 1) * (ny + 1)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = (i * sx + j * sy + k * sz).ravel().astype(np.int64)
    off = np.array([0, sx, sx + sy, sy, sz, sz + sx, sz + sx + sy, sz + sy], dtype=np.int64)
    return (base[:, None] + off[None, :]).astype(np.int32)


def grid_faces(nx, ny, nz):
    """Boundary quads of the box, per side, as (F,4) int32 node ids."""
    sx, sy = 1, nx + 1
    sz = (nx + 1) * (ny + 1)

    def quads(a_n, b_n, fixed_off, da, db):
        b, a = np.meshgrid(np.arange(b_n), np.arange(a_n), indexing="ij")
        base = (fixed_off + a * da + b * db).ravel().astype(np.int64)
        return np.stack([base, base + da, base + da + db, base + db], axis=1).astype(np.int32)

    return {
        "z0": quads(nx, ny, 0, sx, sy),
        "z1": quads(nx, ny, nz * sz, sx, sy),
        "y0": quads(nx, nz, 0, sx, sz),
        "y1": quads(nx, nz, ny * sy, sx, sz),
        "x0": quads(ny, nz, 0, sy, sz),
        "x1": quads(ny, nz, nx * sx, sy, sz),
    }


def side_nodes(nx, ny, nz, side):
    """Node ids lying on one side of the box (structured numbering)."""
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    sel = {"x0": i == 0, "x1": i == nx, "y0": j == 0, "y1": j == ny, "z0": k == 0, "z1": k == nz}[side]
    ids = (i + (nx + 1) * (j + (ny + 1) * k))[sel]
    return np.sort(ids.ravel()).astype(np.int32)


def boundary_node_mask(nx, ny, nz):
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    m = (i == 0) | (i == nx) | (j == 0) | (j == ny) | (k == 0) | (k == nz)
    return m.ravel()


def assemble_faces(nx, ny, nz, side_bc: dict):
    """Concatenate the faces of the sides listed in side_bc {side: bc_index}."""
    per = grid_faces(nx, ny, nz)
    fl, bl = [], []
    for s in SIDES:
        if s in side_bc:
            f = per[s]
            fl.append(f)
            bl.append(np.full(f.shape[0], side_bc[s], dtype=np.int32))
    if not fl:
        return np.zeros((0, 4), np.int32), np.zeros((0,), np.int32)
    return np.concatenate(fl), np.concatenate(bl)


# ----------------------------------------------------------------------------
# BASELINE.json configs (readings 8c-13..18)
# ----------------------------------------------------------------------------

CFG_N = {1: 10, 2: 64, 3: 128, 4: 256, 5: 384}
CFG_STEPS = {1: 2000, 2: 10000, 3: 5000, 4: 1000, 5: 500}

K_T = Material(rho=7800.0, c0=460.0, beta_c=0.001, D_ref=(50.0, 50.0, 50.0, 0.0, 0.0, 0.0), beta_k=0.002)


def cfg3_tensor():
    """BJ.cfg3 conductivity: D = Q D0 Q^T, Q from QR of default_rng(3) normals
    with diag(R) > 0 and det Q = +1.  Returns the 6 numbers
    (xx, yy, zz, xy, yz, xz).  Pure problem-statement data."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(R))[None, :]
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    D0 = np.array([[10.0, 5.0, 5.0], [5.0, 30.0, 5.0], [5.0, 5.0, 50.0]])
    D = Q @ D0 @ Q.T
    return (D[0, 0], D[1, 1], D[2, 2], D[0, 1], D[1, 2], D[0, 2])


def make_config(cfg: int, n: Optional[int] = None, steps: Optional[int] = None,
                renumber: bool = True) -> Problem:
    """Build BASELINE.json config `cfg` (1..5).  `n` overrides the grid size
    (scaled-down CI variants keep every other parameter), `steps` the step
    count."""
    nn = CFG_N[cfg] if n is None else int(n)
    st = CFG_STEPS[cfg] if steps is None else int(steps)
    nx = ny = nz = nn
    if cfg == 1:
        L = 0.1 * nn
        xyz = grid_nodes(nx, ny, nz, L, L, L)
        conn = grid_conn(nx, ny, nz)
        faces, face_bc = assemble_faces(nx, ny, nz, {})
        dn = side_nodes(nx, ny, nz, "x0")
        mat = Material(7800.0, 460.0, 0.0, (50.0, 50.0, 50.0, 0.0, 0.0, 0.0), 0.0)
        return Problem("cfg1", xyz, conn, faces, face_bc, [], dn, np.full(dn.size, 100.0),
                       None, np.zeros(xyz.shape[0]), mat, st, (64,), 0.0, 0.0, 0.9, (nx, ny, nz),
                       {"L": L, "h": 0.1})
    L = 0.1
    h = L / nn
    if cfg == 2:
        xyz = grid_nodes(nx, ny, nz, L, L, L)
        conn = grid_conn(nx, ny, nz)
        bcs = [FaceBC(BC_FLUX, q=1e5), FaceBC(BC_CONV, h=25.0, T_inf=20.0)]
        faces, face_bc = assemble_faces(nx, ny, nz, {"z0": 0, "z1": 1, "x0": 1, "x1": 1, "y0": 1, "y1": 1})
        return Problem("cfg2", xyz, conn, faces, face_bc, bcs, np.zeros(0, np.int32), np.zeros(0),
                       None, np.full(xyz.shape[0], 20.0), K_T, st, (32, 64), 20.0, 500.0, 0.9,
                       (nx, ny, nz), {"L": L, "h": h})
    if cfg == 3:
        xyz = grid_nodes(nx, ny, nz, L, L, L)
        conn = grid_conn(nx, ny, nz)
        bcs = [FaceBC(BC_RAD, eps=0.8, T_inf=20.0)]
        faces, face_bc = assemble_faces(nx, ny, nz, {"z1": 0})
        dn = side_nodes(nx, ny, nz, "z0")
        mat = Material(1.0, 3.6e6, 0.0, cfg3_tensor(), 0.0)
        return Problem("cfg3", xyz, conn, faces, face_bc, bcs, dn, np.full(dn.size, 500.0),
                       None, np.full(xyz.shape[0], 20.0), mat, st, (32,), 20.0, 20.0, 0.9,
                       (nx, ny, nz), {"L": L, "h": h})
    if cfg == 4:
        xyz = grid_nodes(nx, ny, nz, L, L, L)
        interior = ~boundary_node_mask(nx, ny, nz)
        rng = np.random.default_rng(7)
        xyz[interior] += rng.uniform(-0.2 * h, 0.2 * h, size=(int(interior.sum()), 3))
        conn = grid_conn(nx, ny, nz)
        bcs = [FaceBC(BC_CONV, h=50.0, T_inf=20.0)]
        faces, face_bc = assemble_faces(nx, ny, nz, {s: 0 for s in SIDES})
        x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
        T0 = 20.0 + 80.0 * np.sin(np.pi * x / L) * np.sin(np.pi * y / L) * np.sin(np.pi * z / L)
        meta = {"L": L, "h": h}
        if renumber:
            rng = np.random.default_rng(11)
            node_perm = rng.permutation(xyz.shape[0])
            elem_perm = rng.permutation(conn.shape[0])
            inv = np.empty_like(node_perm)
            inv[node_perm] = np.arange(node_perm.size)
            xyz = xyz[node_perm]
            T0 = T0[node_perm]
            conn = inv[conn[elem_perm]].astype(np.int32)
            faces = inv[faces].astype(np.int32)
            meta["node_perm"] = node_perm   # new id j <- natural id node_perm[j]
            meta["elem_perm"] = elem_perm
        return Problem("cfg4", xyz, conn, faces, face_bc, bcs, np.zeros(0, np.int32), np.zeros(0),
                       None, T0, K_T, st, (32,), 20.0, 100.0, 0.9, (nx, ny, nz), meta)
    if cfg == 5:
        xyz = grid_nodes(nx, ny, nz, L, L, L)
        conn = grid_conn(nx, ny, nz)
        bcs = [FaceBC(BC_CONV, h=25.0, T_inf=20.0)]
        faces, face_bc = assemble_faces(nx, ny, nz, {"z1": 0, "x0": 0, "x1": 0, "y0": 0, "y1": 0})
        c = np.array([0.05, 0.05, 0.05])
        sig = 0.01
        r2 = ((xyz - c[None, :]) ** 2).sum(axis=1)
        q_vol = 1e8 * np.exp(-r2 / (2.0 * sig * sig))
        return Problem("cfg5", xyz, conn, faces, face_bc, bcs, np.zeros(0, np.int32), np.zeros(0),
                       q_vol, np.full(xyz.shape[0], 20.0), K_T, st, (32,), 20.0, 100.0, 0.9,
                       (nx, ny, nz), {"L": L, "h": h})
    raise ValueError(f"unknown config {cfg}")


# ----------------------------------------------------------------------------
# small parity-only inputs (SURVEY.md 8d "Extra parity-only inputs")
# ----------------------------------------------------------------------------

def box_problem(nx, ny, nz, L=(1.0, 1.0, 1.0), material: Optional[Material] = None,
                side_bc: Optional[dict] = None, face_bcs: Optional[list] = None,
                dirichlet: Optional[dict] = None, T0=0.0, q_vol=None, steps=10,
                jitter=0.0, seed=0, affine: Optional[np.ndarray] = None,
                shuffle_seed: Optional[int] = None, name="box") -> Problem:
    """General structured box problem for tests.

    side_bc: {side: bc_index}; dirichlet: {side: T}; jitter: fraction of the
    spacing for interior-node perturbation; affine: 3x3 matrix applied to the
    coordinates (x -> A x); shuffle_seed: random renumbering of nodes and
    elements (corner order preserved)."""
    material = material or Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0.0, 0.0, 0.0), 0.0)
    xyz = grid_nodes(nx, ny, nz, *L)
    if jitter > 0:
        hmin = min(L[0] / nx, L[1] / ny, L[2] / nz)
        interior = ~boundary_node_mask(nx, ny, nz)
        rng = np.random.default_rng(seed)
        xyz[interior] += rng.uniform(-jitter * hmin, jitter * hmin, size=(int(interior.sum()), 3))
    if affine is not None:
        xyz = xyz @ np.asarray(affine, dtype=np.float64).T
    conn = grid_conn(nx, ny, nz)
    faces, face_bc = assemble_faces(nx, ny, nz, side_bc or {})
    dn_list, dT_list = [], []
    seen = set()
    for s, T in (dirichlet or {}).items():
        for nid in side_nodes(nx, ny, nz, s):
            if int(nid) not in seen:
                seen.add(int(nid))
                dn_list.append(int(nid))
                dT_list.append(float(np.asarray(T(xyz[nid][None, :])).ravel()[0]) if callable(T) else float(T))
    dn = np.array(dn_list, dtype=np.int32)
    dT = np.array(dT_list, dtype=np.float64)
    N = xyz.shape[0]
    T0a = np.asarray(T0(xyz) if callable(T0) else np.full(N, float(T0)), dtype=np.float64)
    qv = None if q_vol is None else np.asarray(q_vol(xyz) if callable(q_vol) else q_vol, dtype=np.float64)
    meta = {}
    if shuffle_seed is not None:
        rng = np.random.default_rng(shuffle_seed)
        node_perm = rng.permutation(N)
        elem_perm = rng.permutation(conn.shape[0])
        inv = np.empty_like(node_perm)
        inv[node_perm] = np.arange(N)
        xyz = xyz[node_perm]
        T0a = T0a[node_perm]
        if qv is not None:
            qv = qv[node_perm]
        conn = inv[conn[elem_perm]].astype(np.int32)
        faces = inv[faces].astype(np.int32)
        dn = inv[dn].astype(np.int32)
        meta["node_perm"] = node_perm
    return Problem(name, xyz, conn, faces, face_bc, list(face_bcs or []), dn, dT, qv, T0a,
                   material, steps, (32, 64), 0.0, 0.0, 0.9, (nx, ny, nz), meta)


def random_hexes(n_elem: int, seed: int = 0, distort: float = 0.25):
    """`n_elem` disconnected, randomly distorted, positively oriented hexes.
    Returns (xyz (8n,3), conn (n,8)).  Each hex is a unit cube corner set
    perturbed by U(-distort, distort), then randomly rotated/scaled/shifted."""
    rng = np.random.default_rng(seed)
    nat = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                    [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64) * 0.5
    xs = []
    for _ in range(n_elem):
        p = nat + rng.uniform(-distort, distort, size=(8, 3)) * 0.5
        Q, _r = np.linalg.qr(rng.standard_normal((3, 3)))
        if np.linalg.det(Q) < 0:
            Q[:, 0] = -Q[:, 0]
        s = rng.uniform(0.5, 2.0, size=3)
        p = (p * s[None, :]) @ Q.T + rng.uniform(-5, 5, size=3)[None, :]
        xs.append(p)
    xyz = np.concatenate(xs)
    conn = np.arange(8 * n_elem, dtype=np.int32).reshape(n_elem, 8)
    return xyz, conn


def random_field(n: int, seed: int = 0, lo: float = 0.0, hi: float = 100.0):
    """U[lo,hi] nodal temperature field from default_rng(seed)."""
    return np.random.default_rng(seed).uniform(lo, hi, size=n)


def random_spd_tensor(seed: int = 0, lo: float = 5.0, hi: float = 300.0):
    """A random symmetric positive definite conductivity (xx,yy,zz,xy,yz,xz)."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    lam = rng.uniform(lo, hi, size=3)
    D = Q @ np.diag(lam) @ Q.T
    return (D[0, 0], D[1, 1], D[2, 2], D[0, 1], D[1, 2], D[0, 2])


# ----------------------------------------------------------------------------
# tet4 meshes (NEXT-1): Kuhn split of every hex into 6 tets along the (0, 6)
# diagonal -- the same split in every cell, hence conforming
# ----------------------------------------------------------------------------

KUHN = np.array([[0, 1, 2, 6], [0, 2, 3, 6], [0, 3, 7, 6], [0, 7, 4, 6], [0, 4, 5, 6], [0, 5, 1, 6]])


def tet_conn_from_hex(hconn):
    """(6E, 4) int32 tets from (E, 8) hexes in S:93 order (all positively oriented)."""
    return hconn[:, KUHN].reshape(-1, 4).astype(np.int32)


def boundary_triangles(tconn):
    """Faces of the tets that belong to exactly one tet, as (F, 3) node ids."""
    f = np.concatenate([tconn[:, [0, 1, 2]], tconn[:, [0, 1, 3]], tconn[:, [0, 2, 3]], tconn[:, [1, 2, 3]]])
    key = np.sort(f, axis=1)
    _, idx, cnt = np.unique(key, axis=0, return_index=True, return_counts=True)
    return f[idx[cnt == 1]].astype(np.int32)


def tet_box_problem(nx, ny, nz, L=(1.0, 1.0, 1.0), material: Optional[Material] = None,
                    side_bc: Optional[dict] = None, face_bcs: Optional[list] = None,
                    dirichlet: Optional[dict] = None, T0=0.0, q_vol=None, steps=10,
                    jitter=0.0, seed=0, affine: Optional[np.ndarray] = None, shuffle_seed: Optional[int] = None,
                    name="tetbox") -> Problem:
    """Box of Kuhn-split tets; arguments as box_problem.  Boundary triangles
    get the BC of the box side they lie on."""
    hb = box_problem(nx, ny, nz, L=L, material=material, dirichlet=dirichlet, T0=T0, q_vol=q_vol,
                     steps=steps, jitter=jitter, seed=seed, affine=affine, name=name)
    tconn = tet_conn_from_hex(hb.conn)
    tri = boundary_triangles(tconn)
    # side of each boundary triangle from the structured node index of its nodes
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    ii, jj, kk = i.ravel()[tri], j.ravel()[tri], k.ravel()[tri]
    tests = {"x0": (ii == 0).all(1), "x1": (ii == nx).all(1), "y0": (jj == 0).all(1), "y1": (jj == ny).all(1),
             "z0": (kk == 0).all(1), "z1": (kk == nz).all(1)}
    fl, bl = [], []
    for sname in SIDES:
        if side_bc and sname in side_bc:
            sel = tests[sname]
            fl.append(tri[sel])
            bl.append(np.full(int(sel.sum()), side_bc[sname], dtype=np.int32))
    faces = np.concatenate(fl) if fl else np.zeros((0, 3), np.int32)
    face_bc = np.concatenate(bl) if bl else np.zeros(0, np.int32)
    xyz, T0a, qv, dn = hb.xyz, hb.T0, hb.q_vol, hb.dir_nodes
    meta = dict(hb.meta)
    if shuffle_seed is not None:
        rng = np.random.default_rng(shuffle_seed)
        node_perm = rng.permutation(xyz.shape[0])
        elem_perm = rng.permutation(tconn.shape[0])
        inv = np.empty_like(node_perm)
        inv[node_perm] = np.arange(node_perm.size)
        xyz = xyz[node_perm]
        T0a = T0a[node_perm]
        qv = None if qv is None else qv[node_perm]
        tconn = inv[tconn[elem_perm]].astype(np.int32)
        faces = inv[faces].astype(np.int32)
        dn = inv[dn].astype(np.int32)
        meta["node_perm"] = node_perm
    return Problem(name, xyz, tconn, faces, face_bc, list(face_bcs or []), dn, hb.dir_T, qv, T0a, hb.material,
                   steps, (32, 64), 0.0, 0.0, 0.9, (nx, ny, nz), meta, nodes_per_face=3)


def paper_tet_problem(n=19, td=False, steps=2000):
    """Shape of the paper's Sec. 4.6 timing workload: a 0.1 m cube
    of ~40 000 linear tets (here the Kuhn split of an n^3 grid: n = 19 gives
    41 154 tets / 8 000 nodes vs the paper's 40 021 / 7 872), isotropic
    k = 200, rho = 1000, c = 2000, T0 = 37 degC held on z = 0, a flux
    into z = L.  TD variant uses the cfg2-type linear laws (tables: NEXT-2)."""
    mat = Material(1000.0, 2000.0, 0.001 if td else 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.002 if td else 0.0)
    p = tet_box_problem(n, n, n, L=(0.1, 0.1, 0.1), material=mat, side_bc={"z1": 0},
                        face_bcs=[FaceBC(BC_FLUX, q=2e4)], dirichlet={"z0": 37.0}, T0=37.0, steps=steps,
                        name="paper_tet" + ("_td" if td else ""))
    p.T_lo, p.T_hi = 37.0, 137.0
    return p


def paper_td_material():
    """Sec. 4.2.2 temperature-dependent properties:
    k = 200 W/(m degC) at 37 degC rising 6 per degC to 2000 at 337 degC, c = 2000
    J/(kg degC) at 37 degC to 8000 at 337 degC, rho = 1000, linear in between,
    clamped outside."""
    return Material(1000.0, 2000.0, 0.0, (1.0, 1.0, 1.0, 0.0, 0.0, 0.0), 0.0,
                    k_table=((37.0, 337.0), (200.0, 2000.0)), c_table=((37.0, 337.0), (2000.0, 8000.0)))
