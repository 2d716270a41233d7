// fed_plan.cpp -- host planning + fp64 pre-computation for the B200 FED-FEM path.
//
// Stage (i) of PAPER.md Sec. 3.5, re-designed for the device:
//  * per element the compact operator P_e = (det J / 8) J^-T D_ref J^-1
//    (6 words).  With the natural-sign matrix S (8x3) and B = J^-1 S^T / 8,
//    Eq. 17/20 F_e = 8 det J B^T D B T_e = S P_e S^T T_e exactly, so the
//    kernel reads 6 numbers per element instead of B (24) + scale (Eq. 19).
//  * lumped volume V_n = sum_{e ∋ n} 8 det J_e / 8 (equal split, R3) and the
//    coefficient dt / (rho c0 V_n) (Eq. 14 for TD, Eq. 21 for TI, R2).
//  * per boundary node and face-BC record the tributary area sum A_f / 4
//    (R9); the face loop of Eqs. 4/5/7 then runs node-wise on the device.
//  * critical step dt_crit = min_e 2 / lambda_e (Eq. 29, R13) with
//    lambda_e = max_{T in {T_lo,T_hi}} lambda_max(J^-T D(T) J^-1) / (rho c(T)),
//    lambda_max by the closed trigonometric formula for symmetric 3x3.
// plus the device layout: z-slab partition, Morton locality order, element
// chunks with colours, node classification (chunk-interior vs special).
#include "fed_plan.h"

#include <algorithm>
#include <limits>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#include <parallel/algorithm>
#endif

namespace fed {

static const int NAT[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                              {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};

double sym3_max_eig(const double a[3][3]) {
  double p1 = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
  double q = (a[0][0] + a[1][1] + a[2][2]) / 3.0;
  double d0 = a[0][0] - q, d1 = a[1][1] - q, d2 = a[2][2] - q;
  double p2 = d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * p1;
  if (p2 <= 0.0) return q;
  double p = std::sqrt(p2 / 6.0);
  double b[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) b[i][j] = (a[i][j] - (i == j ? q : 0.0)) / p;
  double detb = b[0][0] * (b[1][1] * b[2][2] - b[1][2] * b[2][1]) -
                b[0][1] * (b[1][0] * b[2][2] - b[1][2] * b[2][0]) +
                b[0][2] * (b[1][0] * b[2][1] - b[1][1] * b[2][0]);
  double r = detb / 2.0;
  r = r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r);
  double phi = std::acos(r) / 3.0;
  return q + 2.0 * p * std::cos(phi);
}

namespace {

struct Geo {
  double det;
  double Ji[3][3];
};

// Centre Jacobian J_ij = d x_j / d xi_i = (1/8) sum_a s_ai x_aj (Eq. 17 at xi = 0)
inline bool element_geometry(const double *xyz, const int32_t *c, Geo &g, double *max_edge) {
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double x[8][3];
  for (int a = 0; a < 8; ++a)
    for (int j = 0; j < 3; ++j) x[a][j] = xyz[3 * (int64_t)c[a] + j];
  for (int a = 0; a < 8; ++a)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) J[i][j] += NAT[a][i] * x[a][j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[i][j] *= 0.125;
  double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  g.det = det;
  if (max_edge) {
    static const int E12[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    double m = 0.0;
    for (int k = 0; k < 12; ++k) {
      double d = 0.0;
      for (int j = 0; j < 3; ++j) {
        double t = x[E12[k][1]][j] - x[E12[k][0]][j];
        d += t * t;
      }
      m = d > m ? d : m;
    }
    *max_edge = std::sqrt(m);
  }
  if (!(det > 0.0)) return false;
  double id = 1.0 / det;
  g.Ji[0][0] = c00 * id;
  g.Ji[1][0] = c01 * id;
  g.Ji[2][0] = c02 * id;
  g.Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  g.Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  g.Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  g.Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  g.Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  g.Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  return true;
}

// tet4: J_ij = (x_{i+1} - x_0)_j, i.e. dx/dxi for the barycentric coordinates
// xi_1..3; grad N_a = column a of J^-1 (a = 1..3), grad N_0 = -sum; V = det J / 6
inline bool tet_geometry(const double *xyz, const int32_t *c, Geo &g, double *max_edge) {
  double x[4][3], J[3][3];
  for (int a = 0; a < 4; ++a)
    for (int j = 0; j < 3; ++j) x[a][j] = xyz[3 * (int64_t)c[a] + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[i][j] = x[i + 1][j] - x[0][j];
  double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  g.det = det;
  if (max_edge) {
    double m = 0.0;
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        double d = 0.0;
        for (int j = 0; j < 3; ++j) d += (x[b][j] - x[a][j]) * (x[b][j] - x[a][j]);
        m = d > m ? d : m;
      }
    // same relative degeneracy threshold as the hex (det ~ h^3 there, ~h^3 here)
    *max_edge = std::sqrt(m);
  }
  if (!(det > 0.0)) return false;
  double id = 1.0 / det;
  g.Ji[0][0] = c00 * id;
  g.Ji[1][0] = c01 * id;
  g.Ji[2][0] = c02 * id;
  g.Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  g.Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  g.Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  g.Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  g.Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  g.Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  return true;
}

// tet4 element eigenvalue factor: lambda_max(M_e^-1 K_e) = 4 lambda_max(L^T X L) / (rho c)
// with K_e = S^T (V X) S, S S^T = I + 1 1^T = L L^T (constant Cholesky factor)
inline double tet_lambda_factor(const double X[3][3]) {
  static const double L[3][3] = {{1.4142135623730951, 0, 0},
                                 {0.7071067811865475, 1.2247448713915889, 0},
                                 {0.7071067811865475, 0.4082482904638631, 1.1547005383792515}};
  double T[3][3], Y[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[i][j] = X[i][0] * L[0][j] + X[i][1] * L[1][j] + X[i][2] * L[2][j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Y[i][j] = L[0][i] * T[0][j] + L[1][i] * T[1][j] + L[2][i] * T[2][j];
  return 4.0 * sym3_max_eig(Y);
}

// X = J^-T D J^-1
inline void xform(const Geo &g, const double D[3][3], double X[3][3]) {
  double T[3][3];
  for (int k = 0; k < 3; ++k)
    for (int j = 0; j < 3; ++j) T[k][j] = D[k][0] * g.Ji[0][j] + D[k][1] * g.Ji[1][j] + D[k][2] * g.Ji[2][j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) X[i][j] = g.Ji[0][i] * T[0][j] + g.Ji[1][i] * T[1][j] + g.Ji[2][i] * T[2][j];
}

inline uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

template <class It, class Cmp>
void psort(It b, It e, Cmp cmp) {
#ifdef _OPENMP
  __gnu_parallel::sort(b, e, cmp);
#else
  std::sort(b, e, cmp);
#endif
}

}  // namespace

// Shared-memory bank layout of one chunk (element kernel).
// In a colour phase the lanes of a warp gather T_e and read-modify-write F_e of 32
// elements, corner by corner: one shared-memory instruction per corner touches 32
// chunk-local nodes.  With nb banks of the word size (32 for fp32; 16 for fp64,
// whose 64-bit accesses are served per half-warp), an instruction is conflict-free
// when its nodes sit in distinct banks.  Greedy colouring of the nodes with the nb
// banks (most-constrained node first, fewest conflicts, then the least-filled bank)
// gives every node a bank; its position is then nb * (rank within its bank) + bank,
// separately for the interior region (streamed by 1-D TMA, so its holes become
// padding nodes in HBM) and the shared-node region (gathered by index, holes cost
// only shared memory).  Result: pos[i] for local node i (interior nodes first, in
// the order given), and the two region sizes (multiples of nb).
struct BankLayout {
  std::vector<int32_t> pos;
  int32_t r_int = 0, r_sp = 0;
};

void bank_layout(const std::vector<std::vector<int32_t>> &insts, int n_int, int n_sp, int nb, BankLayout &out) {
  const int nl = n_int + n_sp;
  std::vector<int32_t> deg(nl, 0), ptr(nl + 1, 0);
  for (const auto &in : insts)
    for (int32_t v : in) deg[v]++;
  for (int v = 0; v < nl; ++v) ptr[v + 1] = ptr[v] + deg[v];
  std::vector<int32_t> adj(ptr[nl]), fill(ptr.begin(), ptr.end() - 1);
  for (int32_t j = 0; j < (int32_t)insts.size(); ++j)
    for (int32_t v : insts[j]) adj[fill[v]++] = j;
  std::vector<int32_t> order(nl);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return deg[a] > deg[b]; });
  std::vector<uint16_t> icnt(insts.size() * (size_t)nb, 0);
  std::vector<int32_t> bank(nl, 0), cnt_int(nb, 0), cnt_sp(nb, 0), cost(nb);
  for (int32_t v : order) {
    std::fill(cost.begin(), cost.end(), 0);
    for (int32_t k = ptr[v]; k < ptr[v + 1]; ++k) {
      const uint16_t *c = &icnt[(size_t)adj[k] * nb];
      for (int b = 0; b < nb; ++b) cost[b] += c[b];
    }
    std::vector<int32_t> &cnt = v < n_int ? cnt_int : cnt_sp;
    int best = 0;
    for (int b = 1; b < nb; ++b)
      if (cost[b] < cost[best] || (cost[b] == cost[best] && cnt[b] < cnt[best])) best = b;
    bank[v] = best;
    cnt[best]++;
    for (int32_t k = ptr[v]; k < ptr[v + 1]; ++k) icnt[(size_t)adj[k] * nb + best]++;
  }
  int mi = 0, ms = 0;
  for (int b = 0; b < nb; ++b) {
    mi = std::max(mi, cnt_int[b]);
    ms = std::max(ms, cnt_sp[b]);
  }
  out.r_int = mi * nb;
  out.r_sp = ms * nb;
  out.pos.assign(nl, 0);
  std::fill(cnt_int.begin(), cnt_int.end(), 0);
  std::fill(cnt_sp.begin(), cnt_sp.end(), 0);
  for (int v = 0; v < nl; ++v) {
    std::vector<int32_t> &cnt = v < n_int ? cnt_int : cnt_sp;
    out.pos[v] = nb * cnt[bank[v]]++ + bank[v];
  }
}

fed_status build_plan(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs,
                      const fed_options *opts, Plan &pl, std::string &err) {
  // ------------------------------------------------------------------ validation
  if (!mesh || !mat || !bcs || !opts) { err = "null argument"; return FED_ERR_INVALID; }
  const int64_t N = mesh->n_nodes, E = mesh->n_elems, F = mesh->n_faces;
  const int npe = mesh->nodes_per_elem == 0 ? 8 : mesh->nodes_per_elem;  // hex8 (Eq. 17) or tet4 (Eq. 18)
  const int npf = mesh->nodes_per_face == 0 ? (npe == 8 ? 4 : 3) : mesh->nodes_per_face;
  if (npe != 8 && npe != 4) { err = "nodes_per_elem must be 8 (hex8) or 4 (tet4)"; return FED_ERR_INVALID; }
  if (npf != 4 && npf != 3) { err = "nodes_per_face must be 4 (quads) or 3 (triangles)"; return FED_ERR_INVALID; }
  if (N <= 0 || E <= 0 || F < 0) { err = "n_nodes and n_elems must be > 0, n_faces >= 0"; return FED_ERR_INVALID; }
  if (N >= INT32_MAX || E >= INT32_MAX) { err = "mesh too large for int32 indices"; return FED_ERR_INVALID; }
  if (!mesh->xyz || !mesh->conn) { err = "mesh.xyz and mesh.conn are required"; return FED_ERR_INVALID; }
  if (F > 0 && (!mesh->faces || !mesh->face_bc)) { err = "mesh.faces / face_bc required when n_faces > 0"; return FED_ERR_INVALID; }
  if (opts->precision != 32 && opts->precision != 64) { err = "precision must be 32 or 64"; return FED_ERR_INVALID; }
  if (opts->nranks < 1 || opts->rank < 0 || opts->rank >= opts->nranks) { err = "bad rank / nranks"; return FED_ERR_INVALID; }
  if (!(mat->rho > 0) || !(mat->c0 > 0) || !std::isfinite(mat->beta_c) || !std::isfinite(mat->beta_k)) {
    err = "material: rho and c0 must be > 0, betas finite";
    return FED_ERR_INVALID;
  }
  double D[3][3] = {{mat->D_ref[0], mat->D_ref[3], mat->D_ref[5]},
                    {mat->D_ref[3], mat->D_ref[1], mat->D_ref[4]},
                    {mat->D_ref[5], mat->D_ref[4], mat->D_ref[2]}};
  {
    double m1 = D[0][0], m2 = D[0][0] * D[1][1] - D[0][1] * D[1][0];
    double m3 = D[0][0] * (D[1][1] * D[2][2] - D[1][2] * D[2][1]) - D[0][1] * (D[1][0] * D[2][2] - D[1][2] * D[2][0]) +
                D[0][2] * (D[1][0] * D[2][1] - D[1][1] * D[2][0]);
    if (!(m1 > 0) || !(m2 > 0) || !(m3 > 0)) { err = "material: D_ref must be symmetric positive definite"; return FED_ERR_INVALID; }
  }
  const int nb = bcs->n_face_bcs;
  if (nb < 0 || (nb > 0 && !bcs->face_bcs)) { err = "bcs.face_bcs"; return FED_ERR_INVALID; }
  for (int b = 0; b < nb; ++b) {
    const fed_face_bc &r = bcs->face_bcs[b];
    if (r.kind != FED_BC_FLUX && r.kind != FED_BC_CONV && r.kind != FED_BC_RAD) { err = "bad face-bc kind"; return FED_ERR_INVALID; }
    if (!std::isfinite(r.q) || !std::isfinite(r.h) || !std::isfinite(r.T_inf) || !std::isfinite(r.eps) || r.h < 0 ||
        r.eps < 0 || r.eps > 1 || (r.kind == FED_BC_RAD && !(r.T_inf > -273.15)) ||
        (r.area_mode != 0 && r.area_mode != 1)) {
      err = "bad face-bc parameters";
      return FED_ERR_INVALID;
    }
  }
  if (bcs->n_dirichlet < 0 || (bcs->n_dirichlet > 0 && (!bcs->dir_nodes || !bcs->dir_T))) { err = "bcs dirichlet arrays"; return FED_ERR_INVALID; }
  for (int64_t d = 0; d < bcs->n_dirichlet; ++d)
    if (bcs->dir_nodes[d] < 0 || bcs->dir_nodes[d] >= N || !std::isfinite(bcs->dir_T[d])) {
      err = "Dirichlet node index out of range or non-finite value";
      return FED_ERR_MESH;
    }
  for (int64_t f = 0; f < F; ++f) {
    if (mesh->face_bc[f] < -1 || mesh->face_bc[f] >= nb) { err = "face_bc index out of range"; return FED_ERR_INVALID; }
    for (int k = 0; k < npf; ++k)
      if (mesh->faces[npf * f + k] < 0 || mesh->faces[npf * f + k] >= N) { err = "face node index out of range"; return FED_ERR_MESH; }
  }
  {
    int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int64_t i = 0; i < npe * E; ++i) bad |= (mesh->conn[i] < 0 || mesh->conn[i] >= N);
    if (bad) { err = "element connectivity index out of range"; return FED_ERR_MESH; }
  }

  pl.precision = opts->precision;
  pl.npe = npe;
  pl.npf = npf;
  pl.rank = opts->rank;
  pl.nranks = opts->nranks;
  pl.scatter = (atomic_family(opts->scatter) || opts->scatter == FED_SCATTER_CHUNK_CAS ||
                opts->scatter == FED_SCATTER_CHUNK_REG || opts->scatter == FED_SCATTER_CHUNK) ? opts->scatter
                                                                                      : FED_SCATTER_CHUNK_REGC;
  if (pl.scatter != FED_SCATTER_ATOMIC && atomic_family(pl.scatter) && opts->nranks > 1) {
    err = "the ATOMIC_WARP / COLOR_PASSES / GATHER baselines are single-rank";
    return FED_ERR_INVALID;
  }
  if (pl.scatter == FED_SCATTER_ATOMIC_WARP && npe != 8) { err = "ATOMIC_WARP pairs hex8 corners"; return FED_ERR_INVALID; }
  pl.rho = mat->rho;
  pl.c0 = mat->c0;
  pl.beta_c = mat->beta_c;
  pl.beta_k = mat->beta_k;
  for (int i = 0; i < 6; ++i) pl.D_ref[i] = mat->D_ref[i];
  // NEXT-2 tables: validate (strictly increasing T, positive values, <= 32 points)
  auto take_table = [&](int n, const double *Tt, const double *vt, std::vector<double> &oT, std::vector<double> &ov,
                        const char *what) -> bool {
    if (n == 0) return true;
    if (n < 0 || n > 32 || !Tt || !vt) { err = std::string(what) + " table: 1..32 points required"; return false; }
    for (int i = 0; i < n; ++i) {
      if (!std::isfinite(Tt[i]) || !(vt[i] > 0) || (i > 0 && !(Tt[i] > Tt[i - 1]))) {
        err = std::string(what) + " table: temperatures strictly increasing, values > 0";
        return false;
      }
      oT.push_back(Tt[i]);
      ov.push_back(vt[i]);
    }
    return true;
  };
  if (!take_table(mat->n_k_table, mat->k_table_T, mat->k_table_val, pl.k_tab_T, pl.k_tab_v, "k")) return FED_ERR_INVALID;
  if (!take_table(mat->n_c_table, mat->c_table_T, mat->c_table_val, pl.c_tab_T, pl.c_tab_v, "c")) return FED_ERR_INVALID;
  pl.td = (!pl.k_tab_T.empty() || !pl.c_tab_T.empty()) ? 2 : ((mat->beta_c != 0.0 || mat->beta_k != 0.0) ? 1 : 0);
  if (pl.td == 2 && pl.k_tab_T.size() <= 2 && pl.c_tab_T.size() <= 2) {
    // tables of one or two points are clamped linear functions ("linear interpolation
    // between points", clamped outside): the kernels evaluate them like the linear
    // laws (td 3), with the per-node clamp; a property without a table keeps its law
    const double inf = std::numeric_limits<double>::infinity();
    auto clamped = [&](const std::vector<double> &Tt, const std::vector<double> &vt, double law_v0, double law_s,
                       double *o) {
      if (Tt.empty()) {  // the linear law: v0 + s T, unclamped
        o[0] = -inf; o[1] = inf; o[2] = law_v0; o[3] = law_s; o[4] = 0.0;
      } else if (Tt.size() == 1) {  // constant
        o[0] = Tt[0]; o[1] = Tt[0]; o[2] = vt[0]; o[3] = 0.0; o[4] = Tt[0];
      } else {
        o[0] = Tt[0]; o[1] = Tt[1]; o[2] = vt[0]; o[3] = (vt[1] - vt[0]) / (Tt[1] - Tt[0]); o[4] = Tt[0];
      }
    };
    clamped(pl.k_tab_T, pl.k_tab_v, 1.0, mat->beta_k, pl.kl);
    clamped(pl.c_tab_T, pl.c_tab_v, mat->c0, mat->c0 * mat->beta_c, pl.cl);
    pl.td = 3;
  }
  pl.T_abort = opts->T_abort > 0 ? opts->T_abort : 1e6;
  pl.N_glob = N;
  pl.E_glob = E;

  // ------------------------------------------------------------------ per-element pass
  const double *xyz = mesh->xyz;
  const int32_t *conn = mesh->conn;
  std::vector<double> det(E);
  double bmin[3] = {INFINITY, INFINITY, INFINITY}, bmax[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t n = 0; n < N; ++n)
    for (int j = 0; j < 3; ++j) {
      double v = xyz[3 * n + j];
      if (!std::isfinite(v)) { err = "non-finite node coordinate"; return FED_ERR_MESH; }
      bmin[j] = v < bmin[j] ? v : bmin[j];
      bmax[j] = v > bmax[j] ? v : bmax[j];
    }
  // max over T in [T_lo, T_hi] of k(T)/k_ref / (rho c(T)): k and c are linear between
  // consecutive breakpoints, so the ratio's maximum sits at an end or a breakpoint
  auto tab = [](const std::vector<double> &Tt, const std::vector<double> &vt, double T) {
    if (T <= Tt[0]) return vt[0];
    for (size_t i = 0; i + 1 < Tt.size(); ++i)
      if (T <= Tt[i + 1]) return vt[i] + (vt[i + 1] - vt[i]) * (T - Tt[i]) / (Tt[i + 1] - Tt[i]);
    return vt.back();
  };
  std::vector<double> cand = {opts->T_lo, opts->T_hi};
  for (double t : pl.k_tab_T) if (t > opts->T_lo && t < opts->T_hi) cand.push_back(t);
  for (double t : pl.c_tab_T) if (t > opts->T_lo && t < opts->T_hi) cand.push_back(t);
  double lam_fac = 0.0;
  for (double T : cand) {
    double num = pl.k_tab_T.empty() ? 1.0 + mat->beta_k * T : tab(pl.k_tab_T, pl.k_tab_v, T);
    double cc = pl.c_tab_T.empty() ? mat->c0 * (1.0 + mat->beta_c * T) : tab(pl.c_tab_T, pl.c_tab_v, T);
    double den = mat->rho * cc;
    if (!(den > 0) || !(num > 0)) { err = "k(T) or c(T) not positive on [T_lo, T_hi]"; return FED_ERR_INVALID; }
    lam_fac = std::max(lam_fac, num / den);
  }
  int64_t bad_elem = -1;
  double lam_max = 0.0;
#pragma omp parallel
  {
    int64_t my_bad = -1;
    double my_lam = 0.0;
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
      Geo g;
      double he = 0;
      bool ok = npe == 8 ? element_geometry(xyz, conn + npe * e, g, &he) : tet_geometry(xyz, conn + npe * e, g, &he);
      det[e] = g.det;
      if (!ok || !(g.det > 1e-12 * he * he * he)) {
        if (my_bad < 0) my_bad = e;
        continue;
      }
      double X[3][3];
      xform(g, D, X);
      double l = npe == 8 ? sym3_max_eig(X) : tet_lambda_factor(X);
      my_lam = l > my_lam ? l : my_lam;
    }
#pragma omp critical
    {
      if (my_bad >= 0 && (bad_elem < 0 || my_bad < bad_elem)) bad_elem = my_bad;
      lam_max = my_lam > lam_max ? my_lam : lam_max;
    }
  }
  if (bad_elem >= 0) {
    err = "element " + std::to_string(bad_elem) + " has det J <= 0 (or degenerate) at its centre";
    return FED_ERR_MESH;
  }
  pl.dt_crit = 2.0 / (lam_max * lam_fac);
  if (std::isnan(opts->dt) || std::isnan(opts->dt_factor)) { err = "dt / dt_factor is NaN"; return FED_ERR_INVALID; }
  pl.dt = opts->dt > 0 ? opts->dt : (opts->dt_factor > 0 ? opts->dt_factor : 0.9) * pl.dt_crit;
  if (!(pl.dt > 0) || !std::isfinite(pl.dt)) { err = "invalid time step"; return FED_ERR_INVALID; }

  // lumped volumes: sequential accumulation in caller element order (deterministic on every rank)
  std::vector<double> Vg(N, 0.0);
  for (int64_t e = 0; e < E; ++e)
    for (int a = 0; a < npe; ++a) Vg[conn[npe * e + a]] += npe == 8 ? det[e] : det[e] / 24.0;  // 8detJ/8 | (detJ/6)/4
  std::vector<double>().swap(det);

  // quantised element centroids: cell indices on a grid whose spacing per axis is
  // the median element extent along that axis (sampled), so structured meshes with
  // non-cubic cells still get one cell per element and 8 parity colours
  double hq[3];
  {
    const int64_t stride = std::max<int64_t>(1, E / 65536);
    std::vector<double> ext[3];
    for (int64_t e = 0; e < E; e += stride) {
      // extent along j: mean of the upper half of the node coordinates minus the mean
      // of the lower half (node jitter averages out, unlike max - min)
      for (int j = 0; j < 3; ++j) {
        double x[8];
        for (int a = 0; a < npe; ++a) x[a] = xyz[3 * (int64_t)conn[npe * e + a] + j];
        std::sort(x, x + npe);
        double lo = 0, hi = 0;
        for (int a = 0; a < npe / 2; ++a) {
          lo += x[a];
          hi += x[npe - 1 - a];
        }
        ext[j].push_back((hi - lo) / (npe / 2));
      }
    }
    const double vol_box = std::max(bmax[0] - bmin[0], 1e-300) * std::max(bmax[1] - bmin[1], 1e-300) *
                           std::max(bmax[2] - bmin[2], 1e-300);
    const double h_cube = std::cbrt(vol_box / (double)E);
    for (int j = 0; j < 3; ++j) {
      std::nth_element(ext[j].begin(), ext[j].begin() + ext[j].size() / 2, ext[j].end());
      const double m = ext[j][ext[j].size() / 2];
      hq[j] = (m > 1e-3 * h_cube && std::isfinite(m)) ? m : h_cube;
    }
  }
  std::vector<uint32_t> qx(E), qy(E), qz(E);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    double c[3] = {0, 0, 0};
    for (int a = 0; a < npe; ++a)
      for (int j = 0; j < 3; ++j) c[j] += xyz[3 * (int64_t)conn[npe * e + a] + j];
    uint32_t q[3];
    for (int j = 0; j < 3; ++j) {
      double v = std::floor((c[j] / npe - bmin[j]) / hq[j]);
      v = v < 0 ? 0 : (v > 2097151.0 ? 2097151.0 : v);
      q[j] = (uint32_t)v;
    }
    qx[e] = q[0];
    qy[e] = q[1];
    qz[e] = q[2];
  }

  // ------------------------------------------------------------------ z-slab partition
  const int P = pl.nranks, R = pl.rank;
  std::vector<int32_t> elem_rank;
  std::vector<int32_t> rmin(N, INT32_MAX), rmax(N, -1);
  if (P > 1) {
    uint32_t qzmax = 0;
    for (int64_t e = 0; e < E; ++e) qzmax = std::max(qzmax, qz[e]);
    std::vector<int64_t> hist((size_t)qzmax + 2, 0);
    for (int64_t e = 0; e < E; ++e) hist[qz[e]]++;
    std::vector<int32_t> layer_rank((size_t)qzmax + 1);
    int64_t cum = 0;
    for (uint32_t v = 0; v <= qzmax; ++v) {
      double mid = (double)cum + 0.5 * (double)hist[v];
      int r = (int)std::floor(mid * P / (double)E);
      layer_rank[v] = r < 0 ? 0 : (r >= P ? P - 1 : r);
      cum += hist[v];
    }
    elem_rank.resize(E);
    for (int64_t e = 0; e < E; ++e) elem_rank[e] = layer_rank[qz[e]];
    for (int64_t e = 0; e < E; ++e)
      for (int a = 0; a < npe; ++a) {
        int32_t n = conn[npe * e + a];
        rmin[n] = std::min(rmin[n], elem_rank[e]);
        rmax[n] = std::max(rmax[n], elem_rank[e]);
      }
  } else {
    for (int64_t i = 0; i < npe * E; ++i) {
      rmin[conn[i]] = 0;
      rmax[conn[i]] = 0;
    }
  }
  for (int64_t n = 0; n < N; ++n) {
    if (rmax[n] < 0) { err = "node " + std::to_string(n) + " is not used by any element"; return FED_ERR_MESH; }
    if (rmax[n] - rmin[n] > 1) { err = "slab partition too thin: a node is shared by non-adjacent ranks"; return FED_ERR_INVALID; }
  }

  // local elements in Morton order of their cell index
  std::vector<int32_t> loc;
  loc.reserve(P > 1 ? E / P + 1 : E);
  for (int64_t e = 0; e < E; ++e)
    if (P == 1 || elem_rank[e] == R) loc.push_back((int32_t)e);
  if (loc.empty()) { err = "rank has no elements (too many ranks for this mesh)"; return FED_ERR_INVALID; }
  std::vector<int32_t>().swap(elem_rank);
  {
    std::vector<uint64_t> key(E);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)loc.size(); ++i) {
      int32_t e = loc[i];
      key[e] = spread3(qx[e]) | (spread3(qy[e]) << 1) | (spread3(qz[e]) << 2);
    }
    psort(loc.begin(), loc.end(), [&](int32_t a, int32_t b) { return key[a] != key[b] ? key[a] < key[b] : a < b; });
  }
  pl.E_loc = (int64_t)loc.size();

  // node flags: special = touched by > 1 chunk, face BC, Dirichlet, interface
  std::vector<uint8_t> flag(N, 0);  // bit0 bc, bit1 dirichlet, bit2 interface
  for (int64_t f = 0; f < F; ++f)
    if (mesh->face_bc[f] >= 0)
      for (int k = 0; k < npf; ++k) flag[mesh->faces[npf * f + k]] |= 1;
  for (int64_t d = 0; d < bcs->n_dirichlet; ++d) flag[bcs->dir_nodes[d]] |= 2;
  for (int64_t n = 0; n < N; ++n)
    if (rmin[n] != rmax[n]) flag[n] |= 4;

  // ------------------------------------------------------------------ chunks
  int chunk = opts->chunk_elems > 0 ? opts->chunk_elems : 0;
  if (chunk == 0) {
    chunk = 1024;
    const int64_t cap = (int64_t)(opts->precision == 32 ? 4 : 2) * pl.sm_count;  // resident CTAs (fed_kernels.cuh)
    const bool resident_cand = opts->nranks == 1 && opts->resident >= 0 &&
                               (opts->scatter == FED_SCATTER_AUTO || opts->scatter == FED_SCATTER_CHUNK_REGC ||
                                (npe == 4 && opts->scatter == FED_SCATTER_CHUNK_REG));
    if (resident_cand && (pl.E_loc + chunk - 1) / chunk <= cap) {
      // resident mode: the smallest power-of-two chunk whose chunks all fit at once
      while (chunk > 128 && (pl.E_loc + chunk / 2 - 1) / (chunk / 2) <= cap) chunk /= 2;
    } else {
      // streaming: keep >= ~4 chunks per SM-resident slot on small meshes
      while (chunk > 128 && pl.E_loc / chunk < 4 * pl.sm_count) chunk /= 2;
    }
  }
  if (chunk < 32 || chunk > 4096 || (chunk & 31)) { err = "chunk_elems must be a multiple of 32 in [32, 4096]"; return FED_ERR_INVALID; }
  if (opts->chunk_order != 0 && opts->chunk_order != 1) { err = "chunk_order must be 0 or 1"; return FED_ERR_INVALID; }
  pl.chunk_elems = chunk;
  const int maxl = max_local_nodes(chunk);
  pl.max_local = maxl;

  std::vector<int64_t> cbeg;  // chunk boundaries in loc
  {
    std::vector<int32_t> stamp(N, -1);
    int64_t cur = 0;
    int nloc = 0, ne = 0;
    cbeg.push_back(0);
    for (int64_t i = 0; i < (int64_t)loc.size(); ++i) {
      const int32_t *c = conn + npe * (int64_t)loc[i];
      int nnew = 0;
      for (int a = 0; a < npe; ++a) {
        bool dup = false;
        for (int b = 0; b < a; ++b) dup |= (c[b] == c[a]);
        if (!dup && stamp[c[a]] != (int32_t)cur) ++nnew;
      }
      if (ne == chunk || nloc + nnew > maxl - 7) {
        cbeg.push_back(i);
        ++cur;
        nloc = 0;
        ne = 0;
        nnew = 0;
        for (int a = 0; a < npe; ++a) {
          bool dup = false;
          for (int b = 0; b < a; ++b) dup |= (c[b] == c[a]);
          if (!dup) ++nnew;
        }
      }
      for (int a = 0; a < npe; ++a) stamp[c[a]] = (int32_t)cur;
      nloc += nnew;
      ++ne;
    }
    cbeg.push_back((int64_t)loc.size());
  }
  const int64_t nch = (int64_t)cbeg.size() - 1;
  // Launch order of the chunks: layer-major.  The chunks are Morton bricks (e.g. 16 x 8 x 8
  // cells at 1024 elements); launched in Morton order, two chunks sharing a face can be
  // thousands of chunks apart (across a high Morton bit), so the shared nodes' T lines and
  // the F lines their partial loads are reduced into have left L2 before the second
  // toucher runs.  Ordered by (z layer, y row, x) of their mean cell, every neighbour is at
  // most about one layer of chunks away -- within what L2 holds of the streamed step.
  std::vector<int32_t> corder(nch);
  std::iota(corder.begin(), corder.end(), 0);
  if (opts->chunk_order == 0 && nch > 1) {
    std::vector<double> mz(nch), my(nch), mx(nch);
    std::vector<int32_t> ez(nch), ey(nch);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
      double sx = 0, sy = 0, sz = 0;
      uint32_t lo[3] = {UINT32_MAX, UINT32_MAX, UINT32_MAX}, hi[3] = {0, 0, 0};
      for (int64_t i = cbeg[c]; i < cbeg[c + 1]; ++i) {
        const int32_t e = loc[i];
        sx += qx[e]; sy += qy[e]; sz += qz[e];
        lo[1] = std::min(lo[1], qy[e]); hi[1] = std::max(hi[1], qy[e]);
        lo[2] = std::min(lo[2], qz[e]); hi[2] = std::max(hi[2], qz[e]);
      }
      const double n = (double)(cbeg[c + 1] - cbeg[c]);
      mx[c] = sx / n; my[c] = sy / n; mz[c] = sz / n;
      ey[c] = (int32_t)(hi[1] - lo[1] + 1);
      ez[c] = (int32_t)(hi[2] - lo[2] + 1);
    }
    // layer / row heights: the median chunk extent in z / y (cells)
    std::vector<int32_t> t(ez);
    std::nth_element(t.begin(), t.begin() + nch / 2, t.end());
    const double Lz = std::max(1, t[nch / 2]);
    t = ey;
    std::nth_element(t.begin(), t.begin() + nch / 2, t.end());
    const double Ly = std::max(1, t[nch / 2]);
    std::vector<int64_t> kz(nch), ky(nch);
    for (int64_t c = 0; c < nch; ++c) {
      kz[c] = (int64_t)std::floor(mz[c] / Lz);
      ky[c] = (int64_t)std::floor(my[c] / Ly);
    }
    std::stable_sort(corder.begin(), corder.end(), [&](int32_t a, int32_t b) {
      if (kz[a] != kz[b]) return kz[a] < kz[b];
      if (ky[a] != ky[b]) return ky[a] < ky[b];
      return mx[a] < mx[b];
    });
  }
  // interface chunks first (they are launched before the exchange)
  std::vector<uint8_t> ch_if(nch, 0);
  if (P > 1) {
    for (int64_t c = 0; c < nch; ++c)
      for (int64_t i = cbeg[c]; i < cbeg[c + 1] && !ch_if[c]; ++i)
        for (int a = 0; a < npe; ++a)
          if (flag[conn[npe * (int64_t)loc[i] + a]] & 4) ch_if[c] = 1;
    std::stable_partition(corder.begin(), corder.end(), [&](int32_t c) { return ch_if[c] != 0; });
  }
  pl.n_chunks = nch;
  pl.n_chunks_if = 0;
  for (int64_t c = 0; c < nch; ++c) pl.n_chunks_if += ch_if[c];

  // colours inside each chunk: preferred colour = parity of the cell index (8 colours on
  // structured grids); greedy fallback to the lowest free colour
  std::vector<int32_t> ecolor(loc.size());
  {
    std::vector<uint32_t> mask(N, 0);
    int maxc = 0;
    bool overflow = false;
    for (int64_t c = 0; c < nch && !overflow; ++c) {
      for (int64_t i = cbeg[c]; i < cbeg[c + 1]; ++i) {
        int32_t e = loc[i];
        const int32_t *cn = conn + npe * (int64_t)e;
        uint32_t used = 0;
        for (int a = 0; a < npe; ++a) used |= mask[cn[a]];
        int pref = (int)((qx[e] & 1) | ((qy[e] & 1) << 1) | ((qz[e] & 1) << 2));
        int col = pref;
        if (used & (1u << pref)) {
          col = -1;
          for (int k = 0; k < kMaxColors; ++k)
            if (!(used & (1u << k))) { col = k; break; }
          if (col < 0) { overflow = true; break; }
        }
        ecolor[i] = col;
        maxc = std::max(maxc, col + 1);
        for (int a = 0; a < npe; ++a) mask[cn[a]] |= 1u << col;
      }
      for (int64_t i = cbeg[c]; i < cbeg[c + 1]; ++i)
        for (int a = 0; a < npe; ++a) mask[conn[npe * (int64_t)loc[i] + a]] = 0;
    }
    if (overflow) {  // not colourable within 32 colours: only the compare-and-swap modes apply
      std::fill(ecolor.begin(), ecolor.end(), 0);
      maxc = 1;
      pl.colored = 0;
    }
    pl.max_colors_used = maxc;
  }
  // staged modes are hex8-only; colour-phase modes need valid colours
  if (npe == 4 && pl.scatter == FED_SCATTER_CHUNK) pl.scatter = FED_SCATTER_CHUNK_REGC;
  if (npe == 4 && pl.scatter == FED_SCATTER_CHUNK_CAS) pl.scatter = FED_SCATTER_CHUNK_REG;
  if (!pl.colored && pl.scatter == FED_SCATTER_CHUNK) pl.scatter = pl.npe == 8 ? FED_SCATTER_CHUNK_CAS : FED_SCATTER_CHUNK_REG;
  if (!pl.colored && pl.scatter == FED_SCATTER_CHUNK_REGC) pl.scatter = FED_SCATTER_CHUNK_REG;
  if (opts->scatter == FED_SCATTER_AUTO && pl.scatter == FED_SCATTER_CHUNK_REGC) {
    // colour phases pay off when every chunk has <= 8 colours of <= 128 elements (the
    // register fast path: structured-like chunks); with more, smaller colours most
    // threads idle in each phase, and one compare-and-swap phase is faster (measured
    // on Kuhn tets: 28 colours, 0.70 -> see DESIGN.md)
    bool fast = pl.max_colors_used <= 8;
    for (int64_t c = 0; fast && c < nch; ++c) {
      int cnt[kMaxColors] = {0};
      for (int64_t i = cbeg[c]; i < cbeg[c + 1]; ++i) cnt[ecolor[i]]++;
      for (int q = 0; q < kMaxColors; ++q) fast = fast && cnt[q] <= 128;
    }
    if (!fast) pl.scatter = FED_SCATTER_CHUNK_REG;
  }
  // the streaming hex colour-phase kernel reads 12-bit packed local positions
  // (fed_api.cu): chunks of more than 4096 local nodes take the compare-and-swap mode
  // under AUTO, and are an error when CHUNK_REGC is asked for explicitly
  if (npe == 8 && pl.scatter == FED_SCATTER_CHUNK_REGC && maxl > 4096) {
    if (opts->scatter != FED_SCATTER_AUTO) {
      err = "FED_SCATTER_CHUNK_REGC: chunk_elems too large for the 12-bit packed connectivity (<= 2624)";
      return FED_ERR_INVALID;
    }
    pl.scatter = FED_SCATTER_CHUNK_REG;
  }
  // slots: chunk-major (final chunk order), colour-sorted, padded to a multiple of 8;
  // inside a colour, elements in lexicographic (z, y, x) cell order so that the 32
  // lanes of a warp touch a compact 2-D block of same-parity nodes (bank spread)
  std::vector<int64_t> slot_off(nch + 1, 0);
  for (int64_t k = 0; k < nch; ++k) {
    int64_t c = corder[k];
    int64_t ne = cbeg[c + 1] - cbeg[c];
    slot_off[k + 1] = slot_off[k] + ((ne + 7) / 8) * 8;
  }
  pl.n_slots = slot_off[nch];
  pl.slot_elem.assign(pl.n_slots, -1);
  pl.slot_chunk.assign(pl.n_slots, -1);
  pl.slot_color.assign(pl.n_slots, -1);
  pl.color_off.assign(nch * (kMaxColors + 1), 0);
  for (int64_t k = 0; k < nch; ++k) {
    int64_t c = corder[k];
    int cnt[kMaxColors + 1] = {0};
    for (int64_t i = cbeg[c]; i < cbeg[c + 1]; ++i) cnt[ecolor[i] + 1]++;
    for (int q = 0; q < kMaxColors; ++q) cnt[q + 1] += cnt[q];
    for (int q = 0; q <= kMaxColors; ++q) pl.color_off[k * (kMaxColors + 1) + q] = cnt[q];
    std::vector<int64_t> ord(cbeg[c + 1] - cbeg[c]);
    std::iota(ord.begin(), ord.end(), cbeg[c]);
    if (pl.scatter != FED_SCATTER_ATOMIC_WARP)  // ATOMIC_WARP keeps the Morton order: x-pairs in lanes (2k, 2k+1)
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
      int32_t ex = loc[x], ey = loc[y];
      if (ecolor[x] != ecolor[y]) return ecolor[x] < ecolor[y];
      if (qz[ex] != qz[ey]) return qz[ex] < qz[ey];
      if (qy[ex] != qy[ey]) return qy[ex] < qy[ey];
      return qx[ex] < qx[ey];
    });
    for (size_t j = 0; j < ord.size(); ++j) {
      int64_t i = ord[j];
      int64_t s = slot_off[k] + (int64_t)j;
      pl.slot_elem[s] = loc[i];
      pl.slot_chunk[s] = (int32_t)k;
      pl.slot_color[s] = ecolor[i];
    }
  }
  if (pl.scatter == FED_SCATTER_COLOR_PASSES) {
    // the chunk colours must be a valid colouring of the whole mesh: no node may be
    // shared by two elements of one colour (holds for the parity colours of
    // structured meshes)
    if (!pl.colored) { err = "COLOR_PASSES: the mesh could not be coloured"; return FED_ERR_INVALID; }
    std::vector<uint32_t> seen(N, 0);
    for (int64_t s = 0; s < pl.n_slots; ++s) {
      const int32_t e = pl.slot_elem[s];
      if (e < 0) continue;
      const uint32_t bit = 1u << pl.slot_color[s];
      for (int a = 0; a < npe; ++a) {
        uint32_t &m = seen[conn[npe * (int64_t)e + a]];
        if (m & bit) { err = "COLOR_PASSES: chunk colours are not a valid global colouring of this mesh"; return FED_ERR_INVALID; }
        m |= bit;
      }
    }
    pl.cp_off.assign(kMaxColors + 1, 0);
    for (int64_t s = 0; s < pl.n_slots; ++s)
      if (pl.slot_elem[s] >= 0) pl.cp_off[pl.slot_color[s] + 1]++;
    for (int q = 0; q < kMaxColors; ++q) pl.cp_off[q + 1] += pl.cp_off[q];
    pl.cp_list.resize(pl.cp_off[kMaxColors]);
    std::vector<int32_t> fill(pl.cp_off.begin(), pl.cp_off.end() - 1);
    for (int64_t s = 0; s < pl.n_slots; ++s)
      if (pl.slot_elem[s] >= 0) pl.cp_list[fill[pl.slot_color[s]]++] = (int32_t)s;
  }
  std::vector<int32_t>().swap(ecolor);
  std::vector<uint32_t>().swap(qx);
  std::vector<uint32_t>().swap(qy);
  std::vector<uint32_t>().swap(qz);

  // quantised node positions (for the bank-conflict-aware chunk-local numbering)
  std::vector<int32_t> qn(3 * N);
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int j = 0; j < 3; ++j) {
      double v = std::floor((xyz[3 * n + j] - bmin[j]) / hq[j] + 0.5);
      qn[3 * n + j] = (int32_t)(v < 0 ? 0 : (v > 2e9 ? 2e9 : v));
    }
  // sort key of a node inside its chunk: parity class, then (z, y, x) of the half-grid
  auto node_key = [&](int32_t n, const int32_t *mn) -> uint64_t {
    uint64_t x = (uint64_t)(qn[3 * (int64_t)n] - mn[0]), y = (uint64_t)(qn[3 * (int64_t)n + 1] - mn[1]),
             z = (uint64_t)(qn[3 * (int64_t)n + 2] - mn[2]);
    uint64_t par = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2);
    x = std::min<uint64_t>(x >> 1, 0xfffff);
    y = std::min<uint64_t>(y >> 1, 0xfffff);
    z = std::min<uint64_t>(z >> 1, 0x7fff);
    return (par << 61) | (z << 40) | (y << 20) | x;
  };
  std::vector<int32_t> chunk_min(3 * nch, INT32_MAX);

  // ------------------------------------------------------------------ node classification
  std::vector<int32_t> first_chunk(N, -1);
  for (int64_t k = 0; k < nch; ++k)
    for (int64_t s = slot_off[k]; s < slot_off[k + 1]; ++s) {
      int32_t e = pl.slot_elem[s];
      if (e < 0) continue;
      for (int a = 0; a < npe; ++a) {
        int32_t n = conn[npe * (int64_t)e + a];
        if (first_chunk[n] < 0)
          first_chunk[n] = (int32_t)k;
        else if (first_chunk[n] != (int32_t)k)
          flag[n] |= 8;  // multi-chunk
      }
    }
  auto is_special = [&](int32_t n) { return (flag[n] & (1 | 2 | 4 | 8)) != 0; };

  pl.node_map.assign(N, -1);
  std::vector<int32_t> int_start(nch, 0), n_int(nch, 0);
  int64_t next = 0;
  // per chunk: interior nodes (touched by this chunk only) and shared nodes, each in
  // (parity class, half-grid z, y, x) order; then the bank layout of both (colour
  // modes with valid colours only; otherwise the compact order is kept)
  std::vector<std::vector<int32_t>> ch_int(nch), ch_sp(nch);
  std::vector<BankLayout> ch_lay(nch);
  const bool colour_groups = pl.colored && (pl.scatter == FED_SCATTER_CHUNK || pl.scatter == FED_SCATTER_CHUNK_REGC);
  const bool do_banks = !atomic_family(pl.scatter);
  const int nbank = pl.precision == 32 ? 32 : 16;  // banks of the word size; lanes per wavefront
  const int maxl_bank = 2 * chunk + 256;
  {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = 0; k < nch; ++k) {
      int32_t *mn = &chunk_min[3 * k];
      std::vector<int32_t> &ti = ch_int[k], &ts = ch_sp[k];
      for (int64_t s = slot_off[k]; s < slot_off[k + 1]; ++s) {
        int32_t e = pl.slot_elem[s];
        if (e < 0) continue;
        for (int a = 0; a < npe; ++a) {
          int32_t n = conn[npe * (int64_t)e + a];
          for (int j = 0; j < 3; ++j) mn[j] = std::min(mn[j], qn[3 * (int64_t)n + j]);
          (is_special(n) ? ts : ti).push_back(n);
        }
      }
      for (auto *t : {&ti, &ts}) {
        std::sort(t->begin(), t->end());
        t->erase(std::unique(t->begin(), t->end()), t->end());
        std::sort(t->begin(), t->end(), [&](int32_t x, int32_t y) {
          uint64_t kx = node_key(x, mn), ky = node_key(y, mn);
          return kx != ky ? kx < ky : x < y;
        });
      }
      BankLayout &L = ch_lay[k];
      const int ni = (int)ti.size(), ns = (int)ts.size();
      bool ok = false;
      if (do_banks) {
        // local ids: interior 0..ni-1, shared ni..ni+ns-1 (binary search in sorted copies)
        std::vector<std::pair<int32_t, int32_t>> lid;
        lid.reserve(ni + ns);
        for (int i = 0; i < ni; ++i) lid.push_back({ti[i], i});
        for (int i = 0; i < ns; ++i) lid.push_back({ts[i], ni + i});
        std::sort(lid.begin(), lid.end());
        auto local = [&](int32_t n) {
          return std::lower_bound(lid.begin(), lid.end(), std::make_pair(n, INT32_MIN))->second;
        };
        // warp (fp32) / half-warp (fp64) instructions: nb consecutive slots of a colour
        // (colour modes) or of the chunk (compare-and-swap modes), one per corner
        std::vector<std::vector<int32_t>> insts;
        const int32_t *co = &pl.color_off[k * (kMaxColors + 1)];
        auto add_groups = [&](int64_t a, int64_t b) {
          for (int64_t g = a; g < b; g += nbank)
            for (int q = 0; q < npe; ++q) {
              std::vector<int32_t> in;
              for (int64_t s = g; s < std::min<int64_t>(b, g + nbank); ++s) {
                int32_t e = pl.slot_elem[slot_off[k] + s];
                if (e >= 0) in.push_back(local(conn[npe * (int64_t)e + q]));
              }
              if (in.size() > 1) insts.push_back(std::move(in));
            }
        };
        if (colour_groups)
          for (int c = 0; c < kMaxColors; ++c) add_groups(co[c], co[c + 1]);
        else
          add_groups(0, slot_off[k + 1] - slot_off[k]);
        bank_layout(insts, ni, ns, nbank, L);
        ok = L.r_int + L.r_sp <= maxl_bank;
      }
      if (!ok) {  // compact layout
        L.pos.resize(ni + ns);
        const int nip = (ni + 7) & ~7;
        for (int i = 0; i < ni; ++i) L.pos[i] = i;
        for (int i = 0; i < ns; ++i) L.pos[ni + i] = i;
        L.r_int = nip;
        L.r_sp = ns;
      }
    }
  }
  for (int64_t k = 0; k < nch; ++k) {
    next = (next + 7) & ~(int64_t)7;  // 8-node aligned interior ranges (1-D TMA needs 16 B)
    int_start[k] = (int32_t)next;
    const std::vector<int32_t> &ti = ch_int[k];
    for (size_t i = 0; i < ti.size(); ++i) pl.node_map[ti[i]] = (int32_t)(next + ch_lay[k].pos[i]);
    next += ch_lay[k].r_int;   // holes of the bank layout are padding nodes
    n_int[k] = (int32_t)(next - int_start[k]);
    std::vector<int32_t>().swap(ch_int[k]);
  }
  pl.N_int = (next + 7) & ~(int64_t)7;
  // specials: interface with rank-1 (sorted by caller id), interface with rank+1, then the rest
  std::vector<int32_t> sp_nodes;
  if (P > 1) {
    for (int64_t n = 0; n < N; ++n)
      if ((flag[n] & 4) && first_chunk[n] >= 0 && rmin[n] == R - 1) sp_nodes.push_back((int32_t)n);
    pl.n_if_lo = (int64_t)sp_nodes.size();
    for (int64_t n = 0; n < N; ++n)
      if ((flag[n] & 4) && first_chunk[n] >= 0 && rmax[n] == R + 1) sp_nodes.push_back((int32_t)n);
    pl.n_if = (int64_t)sp_nodes.size();
  }
  for (int64_t i = 0; i < (int64_t)sp_nodes.size(); ++i) pl.node_map[sp_nodes[i]] = (int32_t)(pl.N_int + i);
  // then nodes with face BCs / Dirichlet, then shared nodes without boundary data
  // (uniform warps in the node kernel), each group in first-touch order.  The
  // boundary group comes first because its node-kernel blocks are the slow ones (the
  // face records are a second, per-node round trip): started in the first wave they
  // overlap the plain blocks instead of forming the kernel's tail (FED_BND_FIRST=0:
  // the round-1 order, plain group first, for A/B)
  const char *bf_env = std::getenv("FED_BND_FIRST");
  const bool bnd_first = !(bf_env && bf_env[0] == '0');
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t k = 0; k < nch; ++k)
      for (int64_t s = slot_off[k]; s < slot_off[k + 1]; ++s) {
        int32_t e = pl.slot_elem[s];
        if (e < 0) continue;
        for (int a = 0; a < npe; ++a) {
          int32_t n = conn[npe * (int64_t)e + a];
          bool bnd = (flag[n] & (1 | 2)) != 0;
          if (is_special(n) && pl.node_map[n] < 0 && bnd == ((pass == 0) == bnd_first)) {
            pl.node_map[n] = (int32_t)(pl.N_int + (int64_t)sp_nodes.size());
            sp_nodes.push_back(n);
          }
        }
      }
  pl.N_sp = (int64_t)sp_nodes.size();
  pl.N_loc = pl.N_int + pl.N_sp;
  pl.node_global.assign(pl.N_loc, -1);
  for (int64_t n = 0; n < N; ++n)
    if (pl.node_map[n] >= 0) pl.node_global[pl.node_map[n]] = (int32_t)n;
  pl.node_owned.assign(pl.N_loc, 1);
  for (int64_t i = 0; i < pl.N_loc; ++i)
    if (pl.node_global[i] < 0) pl.node_owned[i] = 0;                         // alignment padding
  for (int64_t s = 0; s < pl.n_if_lo; ++s) pl.node_owned[pl.N_int + s] = 0;  // owned by rank-1
  if (P > 1 && pl.want_gather) {
    // readout layout: owner = rmin (the lower rank of an interface), caller-id order
    pl.gather_off.assign(P + 1, 0);
    for (int64_t n = 0; n < N; ++n) pl.gather_off[rmin[n] + 1]++;
    for (int r = 0; r < P; ++r) pl.gather_off[r + 1] += pl.gather_off[r];
    pl.gather_ids.assign(N, -1);
    std::vector<int64_t> pos(pl.gather_off.begin(), pl.gather_off.end() - 1);
    for (int64_t n = 0; n < N; ++n) {
      pl.gather_ids[pos[rmin[n]]++] = (int32_t)n;
      if (rmin[n] == R) pl.own_pack.push_back(pl.node_map[n]);
    }
  }
  if (P > 1) {
    if (pl.n_if_lo > 0) {
      pl.nbr_rank.push_back(R - 1);
      pl.nbr_off.push_back(0);
      pl.nbr_cnt.push_back((int32_t)pl.n_if_lo);
    }
    if (pl.n_if > pl.n_if_lo) {
      pl.nbr_rank.push_back(R + 1);
      pl.nbr_off.push_back((int32_t)pl.n_if_lo);
      pl.nbr_cnt.push_back((int32_t)(pl.n_if - pl.n_if_lo));
    }
  }

  // ------------------------------------------------------------------ chunk tables + conn
  pl.chunk_hdr.assign(nch * kChunkHdr, 0);
  const int wbytes = pl.precision / 8;
  pl.conn16.assign(pl.n_slots * npe, 0);
  if (atomic_family(pl.scatter)) pl.conn32.assign(pl.n_slots * npe, -1);
  {
    std::vector<int32_t> sp_local(pl.N_sp, -1);
    std::vector<int32_t> tmp;   // the chunk's shared-node region: special index per slot, -1 = hole
    for (int64_t k = 0; k < nch; ++k) {
      int64_t ne = 0;
      for (int64_t s = slot_off[k]; s < slot_off[k + 1]; ++s) ne += pl.slot_elem[s] >= 0;
      const int32_t n_int_pad = (n_int[k] + 7) & ~7;
      const BankLayout &L = ch_lay[k];
      const std::vector<int32_t> &ts = ch_sp[k];
      const size_t ni = L.pos.size() - ts.size();
      tmp.assign((size_t)L.r_sp, -1);
      for (size_t j = 0; j < ts.size(); ++j) {
        const int32_t si = pl.node_map[ts[j]] - (int32_t)pl.N_int;
        const int32_t p = L.pos[ni + j];
        tmp[p] = si;
        sp_local[si] = n_int_pad + p;
      }
      int32_t *h = &pl.chunk_hdr[k * kChunkHdr];
      h[CH_ELEM_OFF] = (int32_t)slot_off[k];
      h[CH_N_ELEM] = (int32_t)ne;
      h[CH_N_PAD] = (int32_t)(slot_off[k + 1] - slot_off[k]);
      h[CH_INT_START] = int_start[k];
      h[CH_N_INT] = n_int[k];
      h[CH_SP_OFF] = (int32_t)pl.sp_list.size();
      h[CH_N_SP] = (int32_t)tmp.size();
      int nc = 0;
      for (int q = 0; q < kMaxColors; ++q)
        if (pl.color_off[k * (kMaxColors + 1) + q + 1] > pl.color_off[k * (kMaxColors + 1) + q]) nc = q + 1;
      h[CH_N_COLORS] = nc;
      for (int q = 1; q <= 8; ++q) h[CH_COLOR_OFF1 + q - 1] = pl.color_off[k * (kMaxColors + 1) + q];
      if (n_int_pad + (int64_t)tmp.size() > maxl_bank) { err = "internal: chunk exceeds local node capacity"; return FED_ERR_INVALID; }
      if ((n_int_pad + (int64_t)tmp.size()) * wbytes > 65535) { err = "chunk_elems too large for 16-bit shared-memory offsets at this precision"; return FED_ERR_INVALID; }
      pl.max_local_used = std::max<int>(pl.max_local_used, (int)((n_int_pad + (int64_t)tmp.size() + 7) & ~7));
      pl.max_int_used = std::max<int>(pl.max_int_used, (n_int_pad + 7) & ~7);
      pl.max_sp_used = std::max<int>(pl.max_sp_used, (int)((tmp.size() + 7) & ~(size_t)7));
      for (int32_t s : tmp) pl.sp_list.push_back(s);
      while (pl.sp_list.size() & 3) pl.sp_list.push_back(-1);  // 16-B aligned per chunk (1-D TMA)
      for (int64_t s = slot_off[k]; s < slot_off[k + 1]; ++s) {
        int32_t e = pl.slot_elem[s];
        if (e < 0) continue;
        for (int a = 0; a < npe; ++a) {
          int32_t i = pl.node_map[conn[npe * (int64_t)e + a]];
          int32_t l = i < pl.N_int ? i - int_start[k] : sp_local[i - pl.N_int];
          pl.conn16[npe * s + a] = (uint16_t)(l * wbytes);  // byte offset into the chunk's shared arrays
          if (!pl.conn32.empty()) pl.conn32[npe * s + a] = i;
        }
      }
      for (int32_t s : tmp)
        if (s >= 0) sp_local[s] = -1;
      std::vector<int32_t>().swap(ch_sp[k]);
    }
  }

  if (pl.scatter == FED_SCATTER_GATHER) {  // node -> incident (slot, corner)
    pl.g_ptr.assign(pl.N_loc + 1, 0);
    for (int64_t q = 0; q < pl.n_slots * npe; ++q)
      if (pl.conn32[q] >= 0) pl.g_ptr[pl.conn32[q] + 1]++;
    for (int64_t n = 0; n < pl.N_loc; ++n) pl.g_ptr[n + 1] += pl.g_ptr[n];
    pl.g_list.resize(pl.g_ptr[pl.N_loc]);
    std::vector<int32_t> fill(pl.g_ptr.begin(), pl.g_ptr.end() - 1);
    for (int64_t q = 0; q < pl.n_slots * npe; ++q)
      if (pl.conn32[q] >= 0) pl.g_list[fill[pl.conn32[q]]++] = (int32_t)(((q / npe) << 3) | (q % npe));
  }

  // ------------------------------------------------------------------ resident-mode tables
  // (only for meshes small enough that every chunk can own a CTA for a whole run)
  if (P == 1 && nch <= 2048 &&
      (pl.scatter == FED_SCATTER_CHUNK_REGC || (npe == 4 && pl.scatter == FED_SCATTER_CHUNK_REG))) {
    std::vector<int32_t> tptr(pl.N_sp + 1, 0), tl;
    for (int64_t k = 0; k < nch; ++k) {
      const int32_t *h = &pl.chunk_hdr[k * kChunkHdr];
      for (int32_t j = 0; j < h[CH_N_SP]; ++j)
        if (pl.sp_list[h[CH_SP_OFF] + j] >= 0) tptr[pl.sp_list[h[CH_SP_OFF] + j] + 1]++;
    }
    for (int64_t q = 0; q < pl.N_sp; ++q) tptr[q + 1] += tptr[q];
    tl.resize(tptr[pl.N_sp]);
    std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t k = 0; k < nch; ++k) {  // chunk order: the first toucher is the lowest chunk
      const int32_t *h = &pl.chunk_hdr[k * kChunkHdr];
      for (int32_t j = 0; j < h[CH_N_SP]; ++j) {
        const int32_t q = pl.sp_list[h[CH_SP_OFF] + j];
        if (q >= 0) tl[fill[q]++] = (int32_t)k;
      }
    }
    pl.sp_own.assign(pl.sp_list.size(), 0);
    pl.chunk_nbr_ptr.assign(nch + 1, 0);
    std::vector<int32_t> nb;
    for (int64_t k = 0; k < nch; ++k) {
      const int32_t *h = &pl.chunk_hdr[k * kChunkHdr];
      nb.clear();
      for (int32_t j = 0; j < h[CH_N_SP]; ++j) {
        const int32_t q = pl.sp_list[h[CH_SP_OFF] + j];
        if (q < 0) continue;
        pl.sp_own[h[CH_SP_OFF] + j] = tl[tptr[q]] == (int32_t)k;
        for (int32_t t = tptr[q]; t < tptr[q + 1]; ++t)
          if (tl[t] != (int32_t)k) nb.push_back(tl[t]);
      }
      std::sort(nb.begin(), nb.end());
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      for (int32_t x : nb) pl.chunk_nbr.push_back(x);
      pl.chunk_nbr_ptr[k + 1] = (int32_t)pl.chunk_nbr.size();
    }
  }

  // ------------------------------------------------------------------ per-slot operator P_e
  pl.P.assign(6 * pl.n_slots, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < pl.n_slots; ++s) {
    int32_t e = pl.slot_elem[s];
    if (e < 0) continue;
    Geo g;
    if (npe == 8)
      element_geometry(xyz, conn + npe * (int64_t)e, g, nullptr);
    else
      tet_geometry(xyz, conn + npe * (int64_t)e, g, nullptr);
    double X[3][3];
    xform(g, D, X);
    // hex: P = (det J / 8) J^-T D J^-1 (F_e = S P S^T T_e);  tet: P = V J^-T D J^-1, V = det J / 6
    double f = npe == 8 ? g.det * 0.125 : g.det / 6.0;
    pl.P[0 * pl.n_slots + s] = f * X[0][0];
    pl.P[1 * pl.n_slots + s] = f * X[1][1];
    pl.P[2 * pl.n_slots + s] = f * X[2][2];
    pl.P[3 * pl.n_slots + s] = f * 0.5 * (X[0][1] + X[1][0]);
    pl.P[4 * pl.n_slots + s] = f * 0.5 * (X[1][2] + X[2][1]);
    pl.P[5 * pl.n_slots + s] = f * 0.5 * (X[0][2] + X[2][0]);
  }

  // ------------------------------------------------------------------ nodal arrays
  pl.V.resize(pl.N_loc);
  pl.coef.resize(pl.N_loc);
  pl.T0.resize(pl.N_loc);
  if (bcs->q_vol) pl.Qvol.resize(pl.N_loc);
  for (int64_t i = 0; i < pl.N_loc; ++i) {
    int32_t g = pl.node_global[i];
    if (g < 0) {  // alignment padding node: never referenced by an element
      pl.V[i] = 0.0;
      pl.coef[i] = 0.0;
      pl.T0[i] = 0.0;
      if (bcs->q_vol) pl.Qvol[i] = 0.0;
      continue;
    }
    double v = Vg[g];
    pl.V[i] = v;
    pl.coef[i] = pl.td >= 2 ? pl.dt / (mat->rho * v) : pl.dt / (mat->rho * mat->c0 * v);
    pl.T0[i] = bcs->T0 ? bcs->T0[g] : 0.0;
    if (bcs->q_vol) pl.Qvol[i] = bcs->q_vol[g] * v;
  }
  if (bcs->T0)
    for (int64_t n = 0; n < N; ++n)
      if (!std::isfinite(bcs->T0[n])) { err = "non-finite T0"; return FED_ERR_INVALID; }
  if (bcs->q_vol)
    for (int64_t n = 0; n < N; ++n)
      if (!std::isfinite(bcs->q_vol[n])) { err = "non-finite q_vol"; return FED_ERR_INVALID; }

  // Dirichlet (held fixed, wins over face loads)
  pl.sp_dir.assign(pl.N_sp, 0);
  pl.sp_dirT.assign(pl.N_sp, 0.0);
  for (int64_t d = 0; d < bcs->n_dirichlet; ++d) {
    int32_t i = pl.node_map[bcs->dir_nodes[d]];
    if (i < 0) continue;  // other rank
    pl.sp_dir[i - pl.N_int] = 1;
    pl.sp_dirT[i - pl.N_int] = bcs->dir_T[d];
    pl.T0[i] = bcs->dir_T[d];
  }

  // face-BC entries: per special node and record, the tributary area sum_f A_f / 4
  {
    struct Ent {
      int32_t s, b;
      double a;
      int64_t ord;
    };
    std::vector<Ent> ent;
    std::vector<double> rec_area(nb, 0.0);       // NEXT-3: per-record total area
    auto face_area = [&](int64_t f) {
      const int32_t *q = mesh->faces + (int64_t)npf * f;
      const double *p0 = xyz + 3 * (int64_t)q[0], *p1 = xyz + 3 * (int64_t)q[1], *p2 = xyz + 3 * (int64_t)q[2];
      double d1[3], d2[3];
      if (npf == 4) {  // planar quad: half |diag x diag|
        const double *p3 = xyz + 3 * (int64_t)q[3];
        for (int j = 0; j < 3; ++j) { d1[j] = p2[j] - p0[j]; d2[j] = p3[j] - p1[j]; }
      } else {  // triangle: half |edge x edge|
        for (int j = 0; j < 3; ++j) { d1[j] = p1[j] - p0[j]; d2[j] = p2[j] - p0[j]; }
      }
      double cx = d1[1] * d2[2] - d1[2] * d2[1], cy = d1[2] * d2[0] - d1[0] * d2[2], cz = d1[0] * d2[1] - d1[1] * d2[0];
      return 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
    };
    for (int64_t f = 0; f < F; ++f) {
      int b = mesh->face_bc[f];
      if (b < 0) continue;
      if (bcs->face_bcs[b].area_mode == 1) {      // concentrated loads: collected below
        rec_area[b] += face_area(f);
        continue;
      }
      const int32_t *q = mesh->faces + (int64_t)npf * f;
      const double area = face_area(f);
      for (int k = 0; k < npf; ++k) {
        int32_t i = pl.node_map[q[k]];
        if (i < 0) continue;
        ent.push_back({(int32_t)(i - pl.N_int), b, area / npf, (int64_t)ent.size()});
      }
    }
    {
      // uniform nodal area per record = sum of face areas / #unique nodes (all ranks
      // use the global face list, so interface copies get identical entries)
      std::vector<int32_t> mark(N, -1);
      std::vector<std::vector<int32_t>> uniq(nb);
      for (int64_t f = 0; f < F; ++f) {
        int b = mesh->face_bc[f];
        if (b < 0 || bcs->face_bcs[b].area_mode != 1) continue;
        for (int k = 0; k < npf; ++k) {
          int32_t n = mesh->faces[(int64_t)npf * f + k];
          if (mark[n] != b) { mark[n] = b; uniq[b].push_back(n); }
        }
        // a node can belong to faces of several records; mark is per record pass
      }
      for (int b = 0; b < nb; ++b) {
        if (uniq[b].empty()) continue;
        // re-check uniqueness within the record (mark was overwritten by other records)
        std::sort(uniq[b].begin(), uniq[b].end());
        uniq[b].erase(std::unique(uniq[b].begin(), uniq[b].end()), uniq[b].end());
        const double ua = rec_area[b] / (double)uniq[b].size();
        for (int32_t n : uniq[b]) {
          int32_t i = pl.node_map[n];
          if (i < 0) continue;
          ent.push_back({(int32_t)(i - pl.N_int), b, ua, (int64_t)ent.size()});
        }
      }
    }
    std::sort(ent.begin(), ent.end(), [](const Ent &x, const Ent &y) {
      return x.s != y.s ? x.s < y.s : (x.b != y.b ? x.b < y.b : x.ord < y.ord);
    });
    pl.bc_ptr.assign(pl.N_sp + 1, 0);
    size_t j = 0;
    for (int64_t s = 0; s < pl.N_sp; ++s) {
      pl.bc_ptr[s] = (int32_t)pl.bc_idx.size();
      while (j < ent.size() && ent[j].s == s) {
        int b = ent[j].b;
        double a = 0.0;
        while (j < ent.size() && ent[j].s == s && ent[j].b == b) a += ent[j++].a;
        pl.bc_idx.push_back(b);
        pl.bc_area.push_back(a);
      }
    }
    pl.bc_ptr[pl.N_sp] = (int32_t)pl.bc_idx.size();
  }
  for (size_t j = 0; j < pl.bc_idx.size(); ++j) {
    const fed_face_bc &r = bcs->face_bcs[pl.bc_idx[j]];
    double a = pl.bc_area[j];
    pl.bc_ekind.push_back((int8_t)r.kind);
    pl.bc_tinf.push_back(r.T_inf);
    pl.bc_coef.push_back(r.kind == FED_BC_FLUX ? a * r.q : (r.kind == FED_BC_CONV ? a * r.h : a * (r.eps * 5.67e-8)));
  }
  pl.sp_kind.assign(pl.N_sp, 0);
  for (int64_t s = 0; s < pl.N_sp; ++s)
    pl.sp_kind[s] = pl.sp_dir[s] ? 2 : (pl.bc_ptr[s + 1] > pl.bc_ptr[s] ? 1 : 0);
  for (int b = 0; b < nb; ++b) {
    const fed_face_bc &r = bcs->face_bcs[b];
    pl.bc_kind.push_back(r.kind);
    pl.bc_q.push_back(r.q);
    pl.bc_h.push_back(r.h);
    pl.bc_Tinf.push_back(r.T_inf);
    pl.bc_eps.push_back(r.eps);
  }
  return FED_OK;
}

}  // namespace fed
