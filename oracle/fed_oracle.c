/*
 * fed_oracle.c -- plain, slow, single-threaded fp64 CPU oracle of the FED-FEM
 * per-time-step path (Zhang & Chauhan, arXiv 1909.03355, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path in
 * paper_1909_03355_b200/ (and never includes include/fed.h).
 *
 * It follows the paper's three stages (Sec. 3.5) literally:
 *   (i)  pre-computation: per element det(J), B (3x8), G = 8 det(J) B^T
 *        (Eqs. 17, 19); lumped nodal mass (equal split,
 *        SPEC S:274); coefficient A = dt / M  (Eq. 14).
 *   (ii) initialisation: T = T0, Dirichlet nodes set to T_r.
 *   (iii) time stepping: element loop F_e = G D(T) B T_e (Eq. 20),
 *        F = sum_e F_e (Eq. 11); net nodal heat flows Q from the face
 *        loop (Eqs. 4, 5, 7) and volumetric source; explicit nodal
 *        update T += A / c(T) * (Q - F) (Eq. 16, sign reading 8c-1);
 *        Dirichlet re-applied.
 *
 * Readings of the paper (all listed in DESIGN.md "Readings"):
 *   R1 sign: K PSD, F_int = +K T, update uses (Q - F_int)
 *   R2 A = dt / (rho V_n): "rho" of Eq. 14 is the lumped mass (8c-2)
 *   R3 lumped volume: equal split 8 det J / 8 per node         (8c-3)
 *   R4 one Gauss point at xi = 0, weight 8, no hourglass       (8c-4)
 *   R6 TD conductivity: evaluate at element nodes, average
 *   R7 c(T) at the node's own current temperature
 *   R9 face loads: each face corner receives A_f/n * q(T_corner) (8c-9);
 *      quad A_f by the two-triangle split (1,2,3)+(1,3,4)
 *   tet4 (NEXT-1): Eq. 18, G = V B^T (Eq. 19), lumping V/4 per node
 *   R10 radiation in Kelvin via T_z = -273.15, sigma = 5.67e-8
 *   R11 q>0 heats; convection/radiation remove heat when T>T_inf (8c-11)
 *   R12 Dirichlet overwrites (wins over face loads)
 *   R13 critical step: element eigenvalue bound over [T_lo,T_hi] (8c-13)
 *
 * Parity pins: tests/test_oracle_pins.py, test_oracle_source_pins.py (the
 * volumetric source Q_vol,n = q_vol(x_n) V_n), test_oracle_tet_pins.py,
 * test_oracle_table_pins.py, test_oracle_bc_pins.py -- every function here is
 * pinned by a closed form, a worked example or an invariant (DESIGN.md sec. 4
 * lists function -> pin); none is "unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_ERR_INVALID 1
#define ORA_ERR_MESH 2
#define ORA_ERR_NOMEM 3
#define ORA_ERR_UNSTABLE 6

#define ORA_BC_FLUX 1
#define ORA_BC_CONV 2
#define ORA_BC_RAD 3

static const double SIGMA_SB = 5.67e-8;
static const double T_ZERO = -273.15;     /* P:69 (T_z) */

/* natural coordinates (xi, eta, zeta) of the 8 corners, SPEC S:93 order */
static const double NATC[8][3] = {
    {-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
    {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};

typedef struct {
  int64_t n_nodes, n_elems, n_faces;
  const double *xyz;       /* [n_nodes][3] */
  const int32_t *conn;     /* [n_elems][8] */
  const int32_t *faces;    /* [n_faces][4] */
  const int32_t *face_bc;  /* [n_faces]    */
  int32_t n_face_bcs;
  const int32_t *bc_kind;
  const double *bc_q, *bc_h, *bc_Tinf, *bc_eps;
  int64_t n_dir;
  const int32_t *dir_nodes;
  const double *dir_T;
  const double *q_vol;     /* [n_nodes] W/m^3 at nodes, or NULL */
  const double *T0;        /* [n_nodes] */
  double rho, c0, beta_c;
  double D_ref[6];         /* xx yy zz xy yz xz */
  double beta_k;
  int32_t nodes_per_elem;  /* 8 (hex8, Eq. 17) or 4 (tet4, Eq. 18); 0 = 8 */
  int32_t nodes_per_face;  /* 4 (quads) or 3 (triangles); 0 = 4 */
  /* NEXT-2: piecewise-linear property tables, clamped at
   * the ends.  n_k > 0: k(T) = D_ref * k_tab(T) (replaces 1 + beta_k T);
   * n_c > 0: c(T) = c_tab(T) (replaces c0 (1 + beta_c T)). */
  int32_t n_k;
  const double *k_T, *k_v;
  int32_t n_c;
  const double *c_T, *c_v;
  /* NEXT-3: per face-BC record, 0 = each face corner
   * gets A_f / n_corners, 1 = "concentrated" loads: every unique node of the
   * record's faces gets the same area (sum of face areas) / (#unique nodes).
   * NULL = all 0. */
  const int32_t *bc_area_mode;
} ora_problem;

typedef struct {
  int64_t N, E, F;
  int npe, npf;     /* nodes per element / per boundary face */
  int32_t *conn;
  double *B;        /* [E][3][8]  temperature gradient matrix at xi = 0 */
  double *G;        /* [E][8][3]  G = 8 det(J) B^T   (Eq. 19)           */
  double *M;        /* [N] lumped mass rho * V_n                          */
  double *A;        /* [N] coefficient dt / M  (Eq. 14)                   */
  double *Qvol;     /* [N] s(x_n) V_n  (W)                                */
  int32_t *faces;   /* [F][4] */
  int32_t *face_bc; /* [F] */
  double *face_area;/* [F] */
  int32_t nbc;
  int32_t *bc_kind;
  double *bc_q, *bc_h, *bc_Tinf, *bc_eps;
  uint8_t *is_dir;
  double *dir_val;  /* [N] prescribed T_r where is_dir */
  double D[3][3];   /* reference conductivity tensor */
  double rho, c0, beta_c, beta_k, dt;
  int n_k, n_c;
  double k_T[64], k_v[64], c_T[64], c_v[64];
  int32_t *bc_mode;     /* [nbc] */
  double *bc_uarea;     /* [nbc] uniform nodal area (mode 1) */
  int64_t *uniq_ptr;    /* [nbc + 1] */
  int32_t *uniq_nodes;  /* unique nodes of the mode-1 records' faces */
  double *T, *Fint, *Q;
  int64_t step;
} ora_state;

/* ---------------------------------------------------------------------- */
/* element geometry: Eq. 17 at the single Gauss point xi = 0              */
/* ---------------------------------------------------------------------- */

/* J_ij = d x_j / d xi_i at the centre = sum_a dN_a/dxi_i * x_aj,
 * dN_a/dxi_i(0) = NATC[a][i] / 8 (trilinear shape functions).
 * B = J^-1 dN/dxi  (3x8),  scale = 8 det J.  Returns 0 or ORA_ERR_MESH. */
int ora_hex_kernel(const double *x8, double *B, double *scale, double *detJ_out) {
  double J[3][3], Ji[3][3], dN[3][8];
  for (int i = 0; i < 3; ++i)
    for (int a = 0; a < 8; ++a) dN[i][a] = NATC[a][i] / 8.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int a = 0; a < 8; ++a) s += dN[i][a] * x8[3 * a + j];
      J[i][j] = s;
    }
  double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
             - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
             + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  if (detJ_out) *detJ_out = det;
  if (!(det > 0.0)) return ORA_ERR_MESH;
  /* inverse by the adjugate */
  Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  for (int i = 0; i < 3; ++i)
    for (int a = 0; a < 8; ++a) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += Ji[i][k] * dN[k][a];
      B[8 * i + a] = s;
    }
  *scale = 8.0 * det;
  return ORA_OK;
}

/* Eq. 19: G = 8 det(J) B^T  (8x3) */
void ora_build_G(const double *B, double scale, double *G) {
  for (int a = 0; a < 8; ++a)
    for (int i = 0; i < 3; ++i) G[3 * a + i] = scale * B[8 * i + a];
}

/* Eq. 20: F_e = G D B T_e, evaluated as three dense products. */
void ora_element_load(const double *B, const double *G, const double *D9, const double *Te, double *Fe) {
  double g[3], Dg[3];
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int a = 0; a < 8; ++a) s += B[8 * i + a] * Te[a];
    g[i] = s;
  }
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int j = 0; j < 3; ++j) s += D9[3 * i + j] * g[j];
    Dg[i] = s;
  }
  for (int a = 0; a < 8; ++a) {
    double s = 0.0;
    for (int i = 0; i < 3; ++i) s += G[3 * a + i] * Dg[i];
    Fe[a] = s;
  }
}

/* Eq. 18: linear tetrahedron.  Shape functions N_a = c_0a + c_1a x +
 * c_2a y + c_3a z with N_a(x_b) = delta_ab, i.e. the columns of the inverse of
 * the 4x4 matrix with rows [1 x_b y_b z_b]; B[i][a] = c_{i+1,a} (3x4, constant);
 * V = det / 6.  Inverse by Gauss-Jordan elimination with partial pivoting. */
int ora_tet_kernel(const double *x4, double *B, double *V) {
  double m[4][8];
  for (int b = 0; b < 4; ++b) {
    m[b][0] = 1.0;
    for (int j = 0; j < 3; ++j) m[b][1 + j] = x4[3 * b + j];
    for (int j = 0; j < 4; ++j) m[b][4 + j] = (b == j) ? 1.0 : 0.0;
  }
  double det = 1.0;
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    for (int r = col + 1; r < 4; ++r)
      if (fabs(m[r][col]) > fabs(m[piv][col])) piv = r;
    if (m[piv][col] == 0.0) return ORA_ERR_MESH;
    if (piv != col) {
      for (int j = 0; j < 8; ++j) { double t = m[col][j]; m[col][j] = m[piv][j]; m[piv][j] = t; }
      det = -det;
    }
    det *= m[col][col];
    double d = m[col][col];
    for (int j = 0; j < 8; ++j) m[col][j] /= d;
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      double f = m[r][col];
      for (int j = 0; j < 8; ++j) m[r][j] -= f * m[col][j];
    }
  }
  /* m[:,4:8] = inverse of the row matrix; column a holds (c_0a .. c_3a) */
  for (int i = 0; i < 3; ++i)
    for (int a = 0; a < 4; ++a) B[4 * i + a] = m[1 + i][4 + a];
  *V = det / 6.0;
  return (*V > 0.0) ? ORA_OK : ORA_ERR_MESH;
}

/* Eq. 19/20 for an element with npe nodes: G (npe x 3), B (3 x npe) */
void ora_element_load_n(const double *B, const double *G, const double *D9, const double *Te, double *Fe,
                        int npe) {
  double g[3], Dg[3];
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int a = 0; a < npe; ++a) s += B[npe * i + a] * Te[a];
    g[i] = s;
  }
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int j = 0; j < 3; ++j) s += D9[3 * i + j] * g[j];
    Dg[i] = s;
  }
  for (int a = 0; a < npe; ++a) {
    double s = 0.0;
    for (int i = 0; i < 3; ++i) s += G[3 * a + i] * Dg[i];
    Fe[a] = s;
  }
}

void ora_build_G_n(const double *B, double scale, double *G, int npe) {
  for (int a = 0; a < npe; ++a)
    for (int i = 0; i < 3; ++i) G[3 * a + i] = scale * B[npe * i + a];
}

/* single row -> constant; below / above the table -> end row (clamped);
 * otherwise linear interpolation between the bracketing rows. */
double ora_table_eval(const double *Tt, const double *vt, int n, double T) {
  if (n == 1 || T <= Tt[0]) return vt[0];
  if (T >= Tt[n - 1]) return vt[n - 1];
  for (int i = 0; i + 1 < n; ++i)
    if (T <= Tt[i + 1]) return vt[i] + (vt[i + 1] - vt[i]) * (T - Tt[i]) / (Tt[i + 1] - Tt[i]);
  return vt[n - 1];
}

static void full_tensor(const double *d6, double D[3][3]) {
  D[0][0] = d6[0]; D[1][1] = d6[1]; D[2][2] = d6[2];
  D[0][1] = D[1][0] = d6[3];
  D[1][2] = D[2][1] = d6[4];
  D[0][2] = D[2][0] = d6[5];
}

/* quad area = triangle (1,2,3) + triangle (1,3,4) */
static double tri_area(const double *p, const double *q, const double *r) {
  double u[3], v[3], c[3];
  for (int i = 0; i < 3; ++i) { u[i] = q[i] - p[i]; v[i] = r[i] - p[i]; }
  c[0] = u[1] * v[2] - u[2] * v[1];
  c[1] = u[2] * v[0] - u[0] * v[2];
  c[2] = u[0] * v[1] - u[1] * v[0];
  return 0.5 * sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
}

double ora_tri_area(const double *xyz, const int32_t *f3) {
  return tri_area(xyz + 3 * (int64_t)f3[0], xyz + 3 * (int64_t)f3[1], xyz + 3 * (int64_t)f3[2]);
}

double ora_quad_area(const double *xyz, const int32_t *f4) {
  const double *p0 = xyz + 3 * (int64_t)f4[0], *p1 = xyz + 3 * (int64_t)f4[1];
  const double *p2 = xyz + 3 * (int64_t)f4[2], *p3 = xyz + 3 * (int64_t)f4[3];
  return tri_area(p0, p1, p2) + tri_area(p0, p2, p3);
}

/* ---------------------------------------------------------------------- */
/* symmetric eigenvalues by cyclic Jacobi rotations (textbook)            */
/* ---------------------------------------------------------------------- */
static double jacobi_max_eig(double *a, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < n; ++p) {
      diag += a[p * n + p] * a[p * n + p];
      for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
    }
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = a[p * n + q];
        if (apq == 0.0) continue;
        double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {      /* columns p, q */
          double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {      /* rows p, q */
          double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  double m = a[0];
  for (int p = 1; p < n; ++p) if (a[p * n + p] > m) m = a[p * n + p];
  return m;
}

double ora_sym_max_eig(const double *A, int n) {
  double a[64];
  if (n > 8) return NAN;
  memcpy(a, A, sizeof(double) * n * n);
  return jacobi_max_eig(a, n);
}

/* largest eigenvalue of M_e^-1 K_e for one element, K_e = G D B (8x8, Eq. 22
 * form) and M_e = rho c * 8 det J / 8 per node (equal-split lumping). */
double ora_element_lambda8(const double *x8, const double *D6, double rhoc) {
  double B[24], G[24], scale, det, D[3][3], K[64];
  if (ora_hex_kernel(x8, B, &scale, &det) != ORA_OK) return NAN;
  ora_build_G(B, scale, G);
  full_tensor(D6, D);
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) s += G[3 * a + i] * D[i][j] * B[8 * j + b];
      K[8 * a + b] = s / (rhoc * scale / 8.0);
    }
  return jacobi_max_eig(K, 8);
}

/* largest eigenvalue of M_e^-1 K_e for one tet4, K_e = V B^T D B (4x4, Eq. 22
 * tet branch) and M_e = rho c V / 4 per node (equal-split lumping). */
double ora_tet_lambda(const double *x4, const double *D6, double rhoc) {
  double B[12], V, D[3][3], K[16];
  if (ora_tet_kernel(x4, B, &V) != ORA_OK) return NAN;
  full_tensor(D6, D);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) s += V * B[4 * i + a] * D[i][j] * B[4 * j + b];
      K[4 * a + b] = s / (rhoc * V / 4.0);
    }
  return jacobi_max_eig(K, 4);
}

/* Critical step (Eq. 29; reading 8c-13): dt_crit = min_e 2 / lambda_e,
 * lambda_e = max_{T in {T_lo, T_hi}} lambda_max(J^-T D(T) J^-1) / (rho c(T)).
 * lambda_max(J^-T D J^-1) is obtained from the 3x3 matrix J^-T D J^-1 by Jacobi
 * rotations; J^-1 here is recovered from B = J^-1 dN/dxi via the identity
 * dN/dxi (dN/dxi)^T = I/8, i.e. J^-1 = 8 B (dN/dxi)^T. */
static double k_of(const ora_problem *p, double T) {
  return p->n_k ? ora_table_eval(p->k_T, p->k_v, p->n_k, T) : 1.0 + p->beta_k * T;
}
static double c_of(const ora_problem *p, double T) {
  return p->n_c ? ora_table_eval(p->c_T, p->c_v, p->n_c, T) : p->c0 * (1.0 + p->beta_c * T);
}
/* max over T in [T_lo, T_hi] of k(T) / (rho c(T)): both are linear between
 * consecutive breakpoints, so the ratio is monotone there and the maximum is
 * attained at T_lo, T_hi or a breakpoint inside the range. */
static double worst_k_over_rhoc(const ora_problem *p, double T_lo, double T_hi) {
  double best = -INFINITY;
  double cand[130];
  int nc = 0;
  cand[nc++] = T_lo;
  cand[nc++] = T_hi;
  for (int i = 0; i < p->n_k; ++i) if (p->k_T[i] > T_lo && p->k_T[i] < T_hi) cand[nc++] = p->k_T[i];
  for (int i = 0; i < p->n_c; ++i) if (p->c_T[i] > T_lo && p->c_T[i] < T_hi) cand[nc++] = p->c_T[i];
  for (int i = 0; i < nc; ++i) {
    double r = k_of(p, cand[i]) / (p->rho * c_of(p, cand[i]));
    if (r > best) best = r;
  }
  return best;
}

double ora_dt_crit(const ora_problem *p, double T_lo, double T_hi) {
  double D[3][3];
  full_tensor(p->D_ref, D);
  double best = INFINITY;
  const double kc = worst_k_over_rhoc(p, T_lo, T_hi);
  if (p->nodes_per_elem == 4) {   /* tet4: literal 4x4 element eigenvalue, scaled by k(T)/c(T) */
    for (int64_t e = 0; e < p->n_elems; ++e) {
      double x4[12];
      for (int a = 0; a < 4; ++a)
        for (int j = 0; j < 3; ++j) x4[3 * a + j] = p->xyz[3 * (int64_t)p->conn[4 * e + a] + j];
      double lam0 = ora_tet_lambda(x4, p->D_ref, 1.0);
      if (!(lam0 > 0)) return NAN;
      if (2.0 / (lam0 * kc) < best) best = 2.0 / (lam0 * kc);
    }
    return best;
  }
  for (int64_t e = 0; e < p->n_elems; ++e) {
    double x8[24], B[24], scale, det, Ji[3][3], Kx[9];
    for (int a = 0; a < 8; ++a)
      for (int j = 0; j < 3; ++j) x8[3 * a + j] = p->xyz[3 * (int64_t)p->conn[8 * e + a] + j];
    if (ora_hex_kernel(x8, B, &scale, &det) != ORA_OK) return NAN;
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) {
        double s = 0.0;
        for (int a = 0; a < 8; ++a) s += B[8 * i + a] * NATC[a][k] / 8.0;
        Ji[i][k] = 8.0 * s;
      }
    /* X = Ji^T D Ji */
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) s += Ji[k][i] * D[k][l] * Ji[l][j];
        Kx[3 * i + j] = s;
      }
    double lam0 = ora_sym_max_eig(Kx, 3);
    if (2.0 / (lam0 * kc) < best) best = 2.0 / (lam0 * kc);
  }
  return best;
}

/* ---------------------------------------------------------------------- */
/* stage (i) + (ii): create                                                */
/* ---------------------------------------------------------------------- */
void ora_destroy(ora_state *s);

ora_state *ora_create(const ora_problem *p, double dt, int *err) {
  *err = ORA_OK;
  if (!p || p->n_nodes <= 0 || p->n_elems <= 0 || !(dt > 0) || !(p->rho > 0) || !(p->c0 > 0)) {
    *err = ORA_ERR_INVALID;
    return NULL;
  }
  ora_state *s = (ora_state *)calloc(1, sizeof(ora_state));
  if (!s) { *err = ORA_ERR_NOMEM; return NULL; }
  int64_t N = p->n_nodes, E = p->n_elems, F = p->n_faces;
  s->N = N; s->E = E; s->F = F;
  s->npe = p->nodes_per_elem == 4 ? 4 : 8;
  s->npf = p->nodes_per_face == 3 ? 3 : 4;
  if ((p->nodes_per_elem != 0 && p->nodes_per_elem != 4 && p->nodes_per_elem != 8) ||
      (p->nodes_per_face != 0 && p->nodes_per_face != 3 && p->nodes_per_face != 4)) {
    free(s);
    *err = ORA_ERR_INVALID;
    return NULL;
  }
  const int npe = s->npe, npf = s->npf;
  s->conn = (int32_t *)malloc(sizeof(int32_t) * 8 * E);
  s->B = (double *)malloc(sizeof(double) * 24 * E);
  s->G = (double *)malloc(sizeof(double) * 24 * E);
  s->M = (double *)calloc(N, sizeof(double));
  s->A = (double *)calloc(N, sizeof(double));
  s->Qvol = (double *)calloc(N, sizeof(double));
  s->faces = (int32_t *)malloc(sizeof(int32_t) * 4 * (F > 0 ? F : 1));
  s->face_bc = (int32_t *)malloc(sizeof(int32_t) * (F > 0 ? F : 1));
  s->face_area = (double *)malloc(sizeof(double) * (F > 0 ? F : 1));
  s->nbc = p->n_face_bcs;
  int nb = p->n_face_bcs > 0 ? p->n_face_bcs : 1;
  s->bc_kind = (int32_t *)calloc(nb, sizeof(int32_t));
  s->bc_q = (double *)calloc(nb, sizeof(double));
  s->bc_h = (double *)calloc(nb, sizeof(double));
  s->bc_Tinf = (double *)calloc(nb, sizeof(double));
  s->bc_eps = (double *)calloc(nb, sizeof(double));
  s->is_dir = (uint8_t *)calloc(N, 1);
  s->dir_val = (double *)calloc(N, sizeof(double));
  s->T = (double *)calloc(N, sizeof(double));
  s->Fint = (double *)calloc(N, sizeof(double));
  s->Q = (double *)calloc(N, sizeof(double));
  if (!s->conn || !s->B || !s->G || !s->M || !s->A || !s->Qvol || !s->faces || !s->face_bc ||
      !s->face_area || !s->bc_kind || !s->bc_q || !s->bc_h || !s->bc_Tinf || !s->bc_eps ||
      !s->is_dir || !s->dir_val || !s->T || !s->Fint || !s->Q) {
    ora_destroy(s);
    *err = ORA_ERR_NOMEM;
    return NULL;
  }
  memcpy(s->conn, p->conn, sizeof(int32_t) * npe * E);
  if (p->n_k < 0 || p->n_k > 64 || p->n_c < 0 || p->n_c > 64) { ora_destroy(s); *err = ORA_ERR_INVALID; return NULL; }
  s->n_k = p->n_k;
  s->n_c = p->n_c;
  for (int i = 0; i < p->n_k; ++i) { s->k_T[i] = p->k_T[i]; s->k_v[i] = p->k_v[i]; }
  for (int i = 0; i < p->n_c; ++i) { s->c_T[i] = p->c_T[i]; s->c_v[i] = p->c_v[i]; }
  full_tensor(p->D_ref, s->D);
  s->rho = p->rho; s->c0 = p->c0; s->beta_c = p->beta_c; s->beta_k = p->beta_k; s->dt = dt;

  /* (i)-2: per element det J, B, G (Eqs. 17, 19) */
  double *V = (double *)calloc(N, sizeof(double));
  if (!V) { ora_destroy(s); *err = ORA_ERR_NOMEM; return NULL; }
  for (int64_t e = 0; e < E; ++e) {
    double xe[24], scale, det;
    for (int a = 0; a < npe; ++a) {
      int32_t n = p->conn[npe * e + a];
      if (n < 0 || n >= N) { free(V); ora_destroy(s); *err = ORA_ERR_MESH; return NULL; }
      for (int j = 0; j < 3; ++j) xe[3 * a + j] = p->xyz[3 * (int64_t)n + j];
    }
    int st = npe == 8 ? ora_hex_kernel(xe, s->B + 24 * e, &scale, &det)    /* Eq. 17: scale = 8 det J */
                      : ora_tet_kernel(xe, s->B + 24 * e, &scale);        /* Eq. 18: scale = V       */
    if (st != ORA_OK) { free(V); ora_destroy(s); *err = ORA_ERR_MESH; return NULL; }
    ora_build_G_n(s->B + 24 * e, scale, s->G + 24 * e, npe);               /* Eq. 19 */
    /* (i)-3: lumped mass, equal split of the element volume */
    for (int a = 0; a < npe; ++a) V[p->conn[npe * e + a]] += scale / npe;
  }
  for (int64_t n = 0; n < N; ++n) {
    if (!(V[n] > 0.0)) { free(V); ora_destroy(s); *err = ORA_ERR_MESH; return NULL; }
    s->M[n] = p->rho * V[n];
    s->A[n] = dt / s->M[n];                                   /* Eq. 14 */
    s->Qvol[n] = p->q_vol ? p->q_vol[n] * V[n] : 0.0;         /* nodal quadrature */
  }
  free(V);
  /* boundary faces */
  for (int64_t f = 0; f < F; ++f) {
    for (int k = 0; k < npf; ++k) {
      int32_t n = p->faces[npf * f + k];
      if (n < 0 || n >= N) { ora_destroy(s); *err = ORA_ERR_MESH; return NULL; }
      s->faces[4 * f + k] = n;
    }
    s->face_bc[f] = p->face_bc ? p->face_bc[f] : -1;
    if (s->face_bc[f] >= p->n_face_bcs) { ora_destroy(s); *err = ORA_ERR_INVALID; return NULL; }
    s->face_area[f] = npf == 4 ? ora_quad_area(p->xyz, p->faces + 4 * f) : ora_tri_area(p->xyz, p->faces + 3 * f);
  }
  for (int b = 0; b < p->n_face_bcs; ++b) {
    s->bc_kind[b] = p->bc_kind[b];
    s->bc_q[b] = p->bc_q[b]; s->bc_h[b] = p->bc_h[b];
    s->bc_Tinf[b] = p->bc_Tinf[b]; s->bc_eps[b] = p->bc_eps[b];
  }
  /* NEXT-3: uniform nodal area per record = sum of face areas / #unique nodes */
  s->bc_mode = (int32_t *)calloc(nb, sizeof(int32_t));
  s->bc_uarea = (double *)calloc(nb, sizeof(double));
  s->uniq_ptr = (int64_t *)calloc(nb + 1, sizeof(int64_t));
  s->uniq_nodes = (int32_t *)malloc(sizeof(int32_t) * (4 * (F > 0 ? F : 1)));
  uint8_t *mark = (uint8_t *)calloc(N, 1);
  if (!s->bc_mode || !s->bc_uarea || !s->uniq_ptr || !s->uniq_nodes || !mark) {
    free(mark); ora_destroy(s); *err = ORA_ERR_NOMEM; return NULL;
  }
  int64_t nu = 0;
  for (int b = 0; b < p->n_face_bcs; ++b) {
    s->bc_mode[b] = p->bc_area_mode ? p->bc_area_mode[b] : 0;
    s->uniq_ptr[b] = nu;
    if (s->bc_mode[b] != 1) continue;
    double total = 0.0;
    int64_t start = nu;
    for (int64_t f = 0; f < F; ++f) {
      if (s->face_bc[f] != b) continue;
      total += s->face_area[f];
      for (int k = 0; k < npf; ++k) {
        int32_t n = s->faces[4 * f + k];
        if (!mark[n]) { mark[n] = 1; s->uniq_nodes[nu++] = n; }
      }
    }
    for (int64_t i = start; i < nu; ++i) mark[s->uniq_nodes[i]] = 0;
    s->bc_uarea[b] = nu > start ? total / (double)(nu - start) : 0.0;
  }
  s->uniq_ptr[p->n_face_bcs] = nu;
  free(mark);
  /* (ii): initial field and Dirichlet values */
  for (int64_t n = 0; n < N; ++n) s->T[n] = p->T0 ? p->T0[n] : 0.0;
  for (int64_t d = 0; d < p->n_dir; ++d) {
    int32_t n = p->dir_nodes[d];
    if (n < 0 || n >= N) { ora_destroy(s); *err = ORA_ERR_MESH; return NULL; }
    s->is_dir[n] = 1;
    s->dir_val[n] = p->dir_T[d];
    s->T[n] = p->dir_T[d];
  }
  s->step = 0;
  return s;
}

void ora_destroy(ora_state *s) {
  if (!s) return;
  free(s->conn); free(s->B); free(s->G); free(s->M); free(s->A); free(s->Qvol);
  free(s->faces); free(s->face_bc); free(s->face_area);
  free(s->bc_kind); free(s->bc_q); free(s->bc_h); free(s->bc_Tinf); free(s->bc_eps);
  free(s->is_dir); free(s->dir_val); free(s->T); free(s->Fint); free(s->Q);
  free(s->bc_mode); free(s->bc_uarea); free(s->uniq_ptr); free(s->uniq_nodes);
  free(s);
}

/* ---------------------------------------------------------------------- */
/* stage (iii) pieces                                                      */
/* ---------------------------------------------------------------------- */

/* (iii)-1 + 2.1: F = sum_e F_e, F_e = G D(T) B T_e (Eqs. 11, 20).  D(T) of an
 * element: k evaluated at each element node, then averaged. */
void ora_internal_load(const ora_state *s, const double *T, double *F) {
  for (int64_t n = 0; n < s->N; ++n) F[n] = 0.0;
  const int npe = s->npe;
  for (int64_t e = 0; e < s->E; ++e) {
    const int32_t *c = s->conn + npe * e;
    double Te[8], Fe[8], D9[9];
    for (int a = 0; a < npe; ++a) Te[a] = T[c[a]];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int a = 0; a < npe; ++a)
          acc += s->D[i][j] * (s->n_k ? ora_table_eval(s->k_T, s->k_v, s->n_k, Te[a]) : 1.0 + s->beta_k * Te[a]);
        D9[3 * i + j] = acc / npe;
      }
    ora_element_load_n(s->B + 24 * e, s->G + 24 * e, D9, Te, Fe, npe);
    for (int a = 0; a < npe; ++a) F[c[a]] += Fe[a];
  }
}

/* heat flux into the body through a face of record b at nodal temperature Tn */
static double bc_flux(const ora_state *s, int b, double Tn) {
  if (s->bc_kind[b] == ORA_BC_FLUX) return s->bc_q[b];                      /* Eq. 5 */
  if (s->bc_kind[b] == ORA_BC_CONV) return -s->bc_h[b] * (Tn - s->bc_Tinf[b]); /* Eq. 4 */
  if (s->bc_kind[b] == ORA_BC_RAD) {                                        /* Eq. 7 */
    double Ta = Tn - T_ZERO, Tb = s->bc_Tinf[b] - T_ZERO;
    return -SIGMA_SB * s->bc_eps[b] * (Ta * Ta * Ta * Ta - Tb * Tb * Tb * Tb);
  }
  return 0.0;
}

/* net nodal heat flows Q (Eq. 2): volumetric source + boundary-face loop. */
void ora_external_load(const ora_state *s, const double *T, double *Q) {
  for (int64_t n = 0; n < s->N; ++n) Q[n] = s->Qvol[n];
  for (int64_t f = 0; f < s->F; ++f) {
    int b = s->face_bc[f];
    if (b < 0) continue;                                      /* Eq. 6 adiabatic */
    if (s->bc_mode[b] == 1) continue;                         /* concentrated: below */
    double a4 = s->face_area[f] / s->npf;    /* each corner gets A_f / (#corners) */
    for (int k = 0; k < s->npf; ++k) {
      int32_t n = s->faces[4 * f + k];
      Q[n] += a4 * bc_flux(s, b, T[n]);
    }
  }
  for (int b = 0; b < s->nbc; ++b)
    for (int64_t i = s->uniq_ptr[b]; i < s->uniq_ptr[b + 1]; ++i) {
      int32_t n = s->uniq_nodes[i];
      Q[n] += s->bc_uarea[b] * bc_flux(s, b, T[n]);
    }
}

/* one explicit step (Eq. 16) in the order of P:212-216 / S:381 */
int ora_step(ora_state *s, int64_t nsteps) {
  int unstable = 0;
  for (int64_t k = 0; k < nsteps; ++k) {
    ora_internal_load(s, s->T, s->Fint);
    ora_external_load(s, s->T, s->Q);
    for (int64_t n = 0; n < s->N; ++n) {
      if (s->is_dir[n]) { s->T[n] = s->dir_val[n]; continue; }
      double c = s->n_c ? ora_table_eval(s->c_T, s->c_v, s->n_c, s->T[n]) : s->c0 * (1.0 + s->beta_c * s->T[n]);
      s->T[n] = s->A[n] / c * (s->Q[n] - s->Fint[n]) + s->T[n];
      if (!isfinite(s->T[n])) unstable = 1;
    }
    s->step += 1;
  }
  return unstable ? ORA_ERR_UNSTABLE : ORA_OK;
}

void ora_get_T(const ora_state *s, double *out) { memcpy(out, s->T, sizeof(double) * s->N); }
void ora_set_T(ora_state *s, const double *in) { memcpy(s->T, in, sizeof(double) * s->N); }
void ora_get_mass(const ora_state *s, double *out) { memcpy(out, s->M, sizeof(double) * s->N); }
void ora_get_F(const ora_state *s, double *out) { memcpy(out, s->Fint, sizeof(double) * s->N); }
void ora_get_Q(const ora_state *s, double *out) { memcpy(out, s->Q, sizeof(double) * s->N); }
int64_t ora_get_step(const ora_state *s) { return s->step; }
void ora_compute_loads(ora_state *s, const double *T, double *F, double *Q) {
  ora_internal_load(s, T, F);
  ora_external_load(s, T, Q);
}
