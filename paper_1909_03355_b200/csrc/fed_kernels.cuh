// fed_kernels.cuh -- sm_100a kernels of the FED-FEM time step (internal).
//
// Per step (Sec. 3.5 stage iii):
//   element_chunk_kernel : element thermal loads F_e = S P_e S^T T_e (== G D B T_e,
//                          Eqs. 17/19/20) accumulated per chunk in shared memory;
//                          fused explicit update (Eq. 16) of chunk-interior nodes;
//                          red.global.add of chunk partial loads of shared nodes.
//   element_atomic_kernel: baseline scatter, 8 red.global.add per element.
//   node_kernel          : face loads (Eqs. 4/5/7), interface combine, Dirichlet
//                          (Eq. 3), explicit update of the remaining nodes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fed {

constexpr int kThreads = 128;        // element-kernel CTA size
constexpr int kNodeThreads = 256;    // node-kernel CTA size
constexpr int kMaxColorsDev = 32;

template <typename R>
struct StepArgs {
  R *T;               // [N_loc] temperatures (in place)
  R *F;               // [N_loc] nodal internal loads; chunk mode uses [N_int, N_loc) only
  const R *coef;      // [N_loc] dt / (rho c0 V_n)
  const R *Qvol;      // [N_loc] volumetric nodal source (W) or nullptr
  // element data (slot order)
  const uint4 *conn16;      // [n_slots] 8 x uint16 chunk-local node ids
  const int4 *conn32;       // [n_slots][2] internal node ids (atomic mode)
  const R *P;               // [6][n_slots] compact operator planes xx yy zz xy yz xz
  int64_t n_slots;
  const int32_t *chunk_hdr; // [n_chunks][8]
  const int32_t *color_off; // [n_chunks][33]
  const int32_t *sp_list;
  // special nodes s = n - N_int
  const int32_t *bc_ptr;
  const int32_t *bc_idx;
  const R *bc_area;
  const uint8_t *sp_dir;
  const R *sp_dirT;
  const int32_t *bc_kind;
  const R *bc_q, *bc_h, *bc_Tinf, *bc_eps;
  const R *Frx;             // [n_if] received partial loads (nranks > 1)
  int64_t n_if, n_if_lo;
  int64_t N_int, N_loc, N_sp;
  R beta_k, beta_c, T_abort;
  int max_local, chunk_cap;
  // step bookkeeping
  const long long *step;        // device step counter
  unsigned long long *fail_step; // first unstable step (ULLONG_MAX = none)
  unsigned int *done;            // node-kernel block counter
  long long *step_rw;            // same counter, written by the last node block
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D TMA: global -> shared bulk copy completing on an mbarrier (SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void red_add(float *p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ float rabs(float x) { return fabsf(x); }
__device__ __forceinline__ double rabs(double x) { return fabs(x); }

template <typename R>
__device__ __forceinline__ void flag_unstable(const StepArgs<R> &a, R Tn) {
  if (!(rabs(Tn) <= a.T_abort)) atomicMin(a.fail_step, (unsigned long long)(*a.step));
}

// ---------------------------------------------------------------- element math
// u = S^T T_e, v = phi P u, f_a = s_a . v  (S rows = natural signs, S:93 order)
template <typename R, bool TD>
__device__ __forceinline__ void element_forces(const R t[8], R p0, R p1, R p2, R p3, R p4, R p5, R beta_k,
                                               R f[8]) {
  R u0 = (t[1] + t[2] + t[5] + t[6]) - (t[0] + t[3] + t[4] + t[7]);
  R u1 = (t[2] + t[3] + t[6] + t[7]) - (t[0] + t[1] + t[4] + t[5]);
  R u2 = (t[4] + t[5] + t[6] + t[7]) - (t[0] + t[1] + t[2] + t[3]);
  R v0 = p0 * u0 + p3 * u1 + p5 * u2;
  R v1 = p3 * u0 + p1 * u1 + p4 * u2;
  R v2 = p5 * u0 + p4 * u1 + p2 * u2;
  if (TD) {  // phi_e = mean_a (1 + beta_k T_a): nodal evaluation then average
    R s = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
    R phi = R(1) + beta_k * (s * R(0.125));
    v0 *= phi;
    v1 *= phi;
    v2 *= phi;
  }
  R A = v0 + v1, B = v0 - v1;
  f[6] = A + v2;
  f[2] = A - v2;
  f[5] = B + v2;
  f[1] = B - v2;
  f[0] = -f[6];
  f[4] = -f[2];
  f[3] = -f[5];
  f[7] = -f[1];
}

template <typename R, bool TD>
__device__ __forceinline__ R explicit_update(R T, R F, R Q, R coef, R beta_c) {
  // Eq. 16 with reading R1: T + dt / (M c(T)) (Q - F_int), c(T) = c0 (1 + beta_c T)
  R d = coef * (Q - F);
  if (TD) d = d / (R(1) + beta_c * T);
  return T + d;
}

// ---------------------------------------------------------------- chunk kernel
// Shared memory layout (bytes, 16-aligned):
//   [0,16)                 mbarrier
//   conn   chunk_cap * 16
//   P      6 * chunk_cap * sizeof(R)
//   sT     max_local * sizeof(R)
//   sF     max_local * sizeof(R)
//   sSp    max_local * 4
//   sCol   (kMaxColorsDev + 1) * 4
template <typename R>
__host__ __device__ inline size_t chunk_smem_bytes(int chunk_cap, int max_local) {
  size_t b = 16;
  b += (size_t)chunk_cap * 16;
  b += (size_t)6 * chunk_cap * sizeof(R);
  b += (size_t)max_local * sizeof(R) * 2;
  b += (size_t)max_local * 4;
  b += (kMaxColorsDev + 1) * 4;
  return (b + 15) & ~(size_t)15;
}

template <typename R, bool TD>
__global__ void __launch_bounds__(kThreads) element_chunk_kernel(StepArgs<R> a, int chunk_base) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  uint4 *sConn = reinterpret_cast<uint4 *>(smem + 16);
  R *sP = reinterpret_cast<R *>(smem + 16 + (size_t)a.chunk_cap * 16);
  R *sT = sP + 6 * a.chunk_cap;
  R *sF = sT + a.max_local;
  int *sSp = reinterpret_cast<int *>(sF + a.max_local);
  int *sCol = sSp + a.max_local;

  const int tid = threadIdx.x;
  const int c = chunk_base + blockIdx.x;
  const int *h = a.chunk_hdr + (size_t)c * 8;
  const int elem_off = h[0], n_pad = h[2], int_start = h[3], n_int = h[4], sp_off = h[5], n_sp = h[6],
            n_col = h[7];

  if (tid == 0) {
    // stage (1-D TMA) the chunk's element records: connectivity + 6 operator planes
    mbar_init(bar, 1);
    fence_mbar_init();
    fence_proxy_async();
    const uint32_t pbytes = (uint32_t)(n_pad * sizeof(R));
    mbar_expect_tx(bar, (uint32_t)n_pad * 16u + 6u * pbytes);
    bulk_g2s(sConn, a.conn16 + elem_off, (uint32_t)n_pad * 16u, bar);
#pragma unroll
    for (int q = 0; q < 6; ++q) bulk_g2s(sP + q * a.chunk_cap, a.P + (size_t)q * a.n_slots + elem_off, pbytes, bar);
  }
  // gather the chunk's nodal temperatures (interior: contiguous; shared: via list)
  for (int l = tid; l < n_int; l += kThreads) {
    sT[l] = a.T[int_start + l];
    sF[l] = R(0);
  }
  for (int l = tid; l < n_sp; l += kThreads) {
    int s = a.sp_list[sp_off + l];
    sSp[l] = s;
    sT[n_int + l] = a.T[a.N_int + s];
    sF[n_int + l] = R(0);
  }
  if (tid <= kMaxColorsDev) sCol[tid] = a.color_off[(size_t)c * (kMaxColorsDev + 1) + tid];
  __syncthreads();
  mbar_wait(bar, 0);

  // colour phases: elements of one colour share no node -> plain shared-memory RMW
  for (int k = 0; k < n_col; ++k) {
    const int e1 = sCol[k + 1];
    for (int e = sCol[k] + tid; e < e1; e += kThreads) {
      uint4 cc = sConn[e];
      int idx[8] = {(int)(cc.x & 0xffffu), (int)(cc.x >> 16), (int)(cc.y & 0xffffu), (int)(cc.y >> 16),
                    (int)(cc.z & 0xffffu), (int)(cc.z >> 16), (int)(cc.w & 0xffffu), (int)(cc.w >> 16)};
      R t[8], f[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) t[q] = sT[idx[q]];
      element_forces<R, TD>(t, sP[e], sP[a.chunk_cap + e], sP[2 * a.chunk_cap + e], sP[3 * a.chunk_cap + e],
                            sP[4 * a.chunk_cap + e], sP[5 * a.chunk_cap + e], a.beta_k, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) sF[idx[q]] += f[q];
    }
    __syncthreads();
  }

  // fused explicit update of chunk-interior nodes (Eq. 16); they have no face
  // load, no Dirichlet value and are touched by no other chunk
  for (int l = tid; l < n_int; l += kThreads) {
    const int n = int_start + l;
    const R Q = a.Qvol ? a.Qvol[n] : R(0);
    R Tn = explicit_update<R, TD>(sT[l], sF[l], Q, a.coef[n], a.beta_c);
    a.T[n] = Tn;
    flag_unstable(a, Tn);
  }
  // shared nodes: reduce the chunk's partial loads into F
  for (int l = tid; l < n_sp; l += kThreads) red_add(a.F + a.N_int + sSp[l], sF[n_int + l]);
}

// ---------------------------------------------------------------- atomic baseline
template <typename R, bool TD>
__global__ void __launch_bounds__(256) element_atomic_kernel(StepArgs<R> a) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n_slots) return;
  int4 c0 = __ldg(a.conn32 + 2 * s), c1 = __ldg(a.conn32 + 2 * s + 1);
  if (c0.x < 0) return;  // padding slot
  int idx[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  R t[8], f[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) t[q] = __ldg(a.T + idx[q]);
  element_forces<R, TD>(t, __ldg(a.P + s), __ldg(a.P + a.n_slots + s), __ldg(a.P + 2 * a.n_slots + s),
                        __ldg(a.P + 3 * a.n_slots + s), __ldg(a.P + 4 * a.n_slots + s),
                        __ldg(a.P + 5 * a.n_slots + s), a.beta_k, f);
#pragma unroll
  for (int q = 0; q < 8; ++q) red_add(a.F + idx[q], f[q]);
}

// ---------------------------------------------------------------- node kernel
template <typename R>
__device__ __forceinline__ R face_load(const StepArgs<R> &a, int s, R T) {
  // sum over the node's face-BC records of (sum_f A_f/4) q_b(T)   (Eqs. 4, 5, 7; R9-R11)
  R Q = R(0);
  const int j1 = a.bc_ptr[s + 1];
  for (int j = a.bc_ptr[s]; j < j1; ++j) {
    const int b = a.bc_idx[j];
    const int kind = a.bc_kind[b];
    R q;
    if (kind == 1) {
      q = a.bc_q[b];
    } else if (kind == 2) {
      q = -a.bc_h[b] * (T - a.bc_Tinf[b]);
    } else {
      // sigma eps [(T-Tz)^4 - (Tinf-Tz)^4] factored to avoid cancellation (Kelvin)
      const R Ta = T + R(273.15), Tb = a.bc_Tinf[b] + R(273.15);
      q = -R(5.67e-8) * a.bc_eps[b] * ((T - a.bc_Tinf[b]) * (Ta + Tb) * (Ta * Ta + Tb * Tb));
    }
    Q += a.bc_area[j] * q;
  }
  return Q;
}

template <typename R, bool TD>
__global__ void __launch_bounds__(kNodeThreads) node_kernel(StepArgs<R> a, int64_t start) {
  const int64_t n = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n < a.N_loc) {
    R F = a.F[n];
    a.F[n] = R(0);
    const R T = a.T[n];
    if (n < a.N_int) {
      const R Q = a.Qvol ? a.Qvol[n] : R(0);
      R Tn = explicit_update<R, TD>(T, F, Q, a.coef[n], a.beta_c);
      a.T[n] = Tn;
      flag_unstable(a, Tn);
    } else {
      const int s = (int)(n - a.N_int);
      if (s < a.n_if) F = (s < a.n_if_lo) ? (a.Frx[s] + F) : (F + a.Frx[s]);  // lower rank's part first
      if (a.sp_dir[s]) {
        a.T[n] = a.sp_dirT[s];  // Dirichlet held (Eq. 3)
      } else {
        R Q = a.Qvol ? a.Qvol[n] : R(0);
        Q += face_load(a, s, T);
        R Tn = explicit_update<R, TD>(T, F, Q, a.coef[n], a.beta_c);
        a.T[n] = Tn;
        flag_unstable(a, Tn);
      }
    }
  }
  // the last block to finish advances the device step counter
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      *a.step_rw += 1;
      *a.done = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- utilities
template <typename R>
__global__ void to_double_kernel(const R *src, double *dst, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (double)src[i];
}
template <typename R>
__global__ void from_double_kernel(const double *src, R *dst, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (R)src[i];
}
__global__ void scatter_owned_kernel(const double *Tloc, const int32_t *node_global, const uint8_t *owned,
                                     double *Tglob, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && owned[i]) Tglob[node_global[i]] = Tloc[i];
}

}  // namespace fed
