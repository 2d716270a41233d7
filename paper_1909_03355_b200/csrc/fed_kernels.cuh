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

#include <type_traits>

namespace fed {

constexpr int kThreads = 128;        // element-kernel CTA size
constexpr int kMaxColorsDev = 32;

// Checked build (-DFED_DEVICE_CHECKS, libfed_checked.so; compute-sanitizer is not
// available on this pool): every plan-driven index is bounds-checked on the device
// and colour phases are checked for write conflicts; a failed check sets bit `code`
// of *check_err (no trap, the kernel carries on) and fed_step reports it.
//   0 shared-memory offset of a corner   1 shared-node id    2 interior node range
//   3 two elements of one colour phase share a node          4 element slot range
//   5 face-record range    7 node-kernel range
#ifdef FED_DEVICE_CHECKS
#define FED_DCHECK(a, cond, code)                                    \
  do {                                                               \
    if (!(cond)) atomicOr((a).check_err, 1u << (code));              \
  } while (0)
constexpr bool kChecked = true;
#else
#define FED_DCHECK(a, cond, code) \
  do {                            \
  } while (0)
constexpr bool kChecked = false;
#endif

template <typename R>
struct StepArgs {
  R *T;               // [N_loc] temperatures (in place)
  R *F;               // [N_loc] nodal internal loads; chunk mode uses [N_int, N_loc) only
  const R *coef;      // [N_loc] dt / (rho c0 V_n)
  const R *Qvol;      // [N_loc] volumetric nodal source (W) or nullptr
  // element data (slot order)
  const uint4 *conn16;      // [n_slots] 8 x uint16 chunk-local node ids
  const uint4 *rec12;       // [n_slots] fp32 hex MODE 3: 8 x 12-bit packed chunk-local ids (x, y, z) + P_xx (w)
  const int4 *conn32;       // [n_slots][2] internal node ids (atomic mode)
  const R *P;               // [6][n_slots] compact operator planes xx yy zz xy yz xz
  int64_t n_slots;
  const int32_t *chunk_hdr; // [n_chunks][8]
  const int32_t *color_off; // [n_chunks][33]
  const int32_t *sp_list;
  // special nodes s = n - N_int
  const int32_t *bc_ptr;           // [N_sp + 1] CSR over packed boundary records
  const R *bc_coef;                // [n_ent] area x (q | h | eps sigma)
  const R *bc_tinf;                // [n_ent] ambient temperature (conv, rad)
  const int8_t *bc_ekind;          // [n_ent] FED_BC_*
  const uint8_t *sp_kind;          // [N_sp] 0 plain, 1 face-BC entries, 2 Dirichlet
  const R *sp_dirT;
  const R *Frx;             // [n_if] received partial loads (nranks > 1)
  int64_t n_if, n_if_lo;
  int64_t N_int, N_loc, N_sp;
  R beta_k, beta_c, T_abort;
  R c0;                          // used with TDK == 2 only (coef = dt / (rho V) there)
  // TDK 3 (tables of <= 2 points, clamped linear; coef = dt / (rho V)):
  //   phi(T) = kl_v0 + kl_s (clamp(T, kl_lo, kl_hi) - kl_T0),  c(T) = cl_v0 + cl_s (clamp(T, cl_lo, cl_hi) - cl_T0)
  R kl_lo, kl_hi, kl_v0, kl_s, kl_T0;
  R cl_lo, cl_hi, cl_v0, cl_s, cl_T0;
  const R *kt;                    // NEXT-2 conductivity multiplier table [T | v | slope] (n_kt points) or null
  const R *ct;                   // NEXT-2 specific-heat table [T | v | slope] (n_ct points) or null
  int n_kt, n_ct;
  int max_local, chunk_cap;
  int max_int, max_sp;           // streaming element kernel: coef / Q and shared-list capacities
  // step bookkeeping: the step index of a launch is *step_base + k_off;
  // step_base only advances in advance_step_kernel, after a batch of steps
  const long long *step_base;
  int k_off;
  unsigned long long *fail_step; // first unstable step (ULLONG_MAX = none)
  unsigned int *dTmax;           // monitored step: max |T_new - T_old| as float bits, or null
  // PEER transport (nranks > 1, fed.h FED_TRANSPORT_PEER): the interface partial loads
  // live in a step-parity double buffer that the neighbour ranks read straight from
  // this rank's memory (NVLink peer loads), instead of an NCCL send/recv into Frx
  R *Fif;                              // [2][n_if] own interface partial loads, or null
  const R *pF_lo, *pF_hi;              // my slice inside rank-1's / rank+1's Fif (or null)
  int64_t pstride_lo, pstride_hi;      // the neighbours' n_if (parity stride of their Fif)
  unsigned long long *psig_lo, *psig_hi;  // neighbour flags this rank writes (step + 1)
  unsigned long long *sig;             // [2] own flags: [0] from rank-1, [1] from rank+1
  unsigned int *if_done;               // CTA counter of the interface chunks, or null
  int n_sig_ctas;                      // the launch's first n_sig_ctas CTAs are the interface chunks
  unsigned int *peer_err;              // set when a neighbour flag did not arrive in time
  unsigned long long wait_ns;          // bound on a device-side wait (fed_options.wait_timeout_s)
  int free_run;                        // per-rank timing only (fed_debug_time_rank): skip PEER waits
  unsigned int *check_err;             // checked build: failed device checks (bit per check)
  float l2_stream;                     // fraction of the streamed-once loads (element records, interior
                                       // node ranges) issued with the L2 evict_first policy
};


// warp-aggregated max of non-negative float values into *dst (float bits are
// monotone for x >= 0); call with every active thread of the warp
__device__ __forceinline__ void warp_max_to(unsigned int *dst, float v) {
  const unsigned mask = __activemask();
  unsigned m = __reduce_max_sync(mask, __float_as_uint(v));
  if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicMax(dst, m);
}

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
// ... with an L2 cache policy (streamed-once node ranges)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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

// Programmatic dependent launch (PTX griddepcontrol, sm_90+): with the launch
// attribute set, the next kernel in the stream may start once every CTA of this one
// has called launch_dependents; its wait() returns when this grid has completed and
// its memory is visible.  Launched without the attribute both are no-ops.  The step
// kernels therefore do everything that reads only static data (chunk header, element
// records, coef / Q, shared-node list) before wait() and everything that touches T,
// F or the exchange buffers after it.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// system-scope release store / acquire load of a step flag (peer memory over NVLink)
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// streamed element records (read once per step): no L1 allocation, so the lines of
// the loads in flight do not compete with the rest of L1 (measured ~1 % on cfg5), and
// an L2 cache policy `pol` (createpolicy): evict_first for the streamed-once data keeps
// L2 for the lines that ARE re-read within a step -- the shared nodes' T and the F lines
// their partial loads are reduced into, touched by ~2.2 chunks each
__device__ __forceinline__ uint64_t l2_policy(float frac_evict_first) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol)
               : "f"(frac_evict_first));
  return pol;
}
// L2 evict_last policy for data re-read within or across steps (FED_L2_KEEP bits:
// 1 chunk headers (element kernel), 2 / 4 shared-node T / F in the node kernel,
// 8 / 16 the element kernel's shared-node T gather / F reductions); 0 = plain accesses.
// Default 1 + 16 (measured, cfg5 fp32, same box, 2 runs each: 0.5557 / 0.5521 ->
// 0.5434 / 0.5431 ms/step; the F lines the chunks reduce into stay in L2 for the node
// kernel, 0.073 -> 0.068 ms).  The node-kernel bits (2, 4) made it twice as slow.
#ifndef FED_L2_KEEP
#define FED_L2_KEEP 17
#endif
// Node kernel: the per-node operands outside the 16-byte planes (interface loads,
// face records, Dirichlet values) loaded for the G nodes of an access together
// (node_update_group); 0 = one node at a time (node_update), for A/B.
#ifndef FED_NODE_GROUP
#define FED_NODE_GROUP 1
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int4 ld_keep(const int4 *p, uint64_t pol) {
  int4 v;
  asm("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_keep(const float *p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_add_keep(float *p, float v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_keep(double *p, double v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// (node kernel: plain asm, so the loads batch like the unhinted vector loads)
__device__ __forceinline__ float4 ld_keep4(const float *p, uint64_t pol) {
  float4 v;
  asm("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep4(float *p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol));
}
__device__ __forceinline__ uint4 ld_rec(const uint4 *p, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ld_rec(const uint2 *p, uint64_t pol) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_rec(const uint32_t *p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_rec(const float *p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_rec(const double *p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ float rabs(float x) { return fabsf(x); }
__device__ __forceinline__ double rabs(double x) { return fabs(x); }

template <typename R>
__device__ __forceinline__ void flag_unstable(const StepArgs<R> &a, R Tn) {
  if (!(rabs(Tn) <= a.T_abort)) atomicMin(a.fail_step, (unsigned long long)(*a.step_base + a.k_off));
}

// ---------------------------------------------------------------- element math
// u = S^T T_e, v = phi P u, f_a = s_a . v  (S rows = natural signs, S:93 order).
// Pair sums are shared between the three gradient components and (TDK 1) the
// nodal mean of the linear conductivity law: 18 adds for u and the mean.
template <typename R, bool SCALE>
__device__ __forceinline__ void element_forces(const R t[8], R p0, R p1, R p2, R p3, R p4, R p5, R phi,
                                               R f[8]) {
  const R p01 = t[0] + t[1], p23 = t[2] + t[3], p45 = t[4] + t[5], p67 = t[6] + t[7];
  const R lo = p01 + p23, hi = p45 + p67;
  R u0 = ((t[1] - t[0]) + (t[2] - t[3])) + ((t[5] - t[4]) + (t[6] - t[7]));
  R u1 = (p23 - p01) + (p67 - p45);
  R u2 = hi - lo;
  if (SCALE) {  // phi_e = mean over the element's nodes of k(T_a)/k_ref
    u0 *= phi;
    u1 *= phi;
    u2 *= phi;
  }
  const R v0 = p0 * u0 + p3 * u1 + p5 * u2;
  const R v1 = p3 * u0 + p1 * u1 + p4 * u2;
  const R v2 = p5 * u0 + p4 * u1 + p2 * u2;
  const R A = v0 + v1, B = v0 - v1;
  f[6] = A + v2;
  f[2] = A - v2;
  f[5] = B + v2;
  f[1] = B - v2;
  f[0] = -f[6];
  f[4] = -f[2];
  f[3] = -f[5];
  f[7] = -f[1];
}

// tet4 (Eq. 18): d = (T1-T0, T2-T0, T3-T0), f_{1..3} = phi P d, f_0 = -sum;
// P = V J^-T D J^-1 (6 words, symmetric)
template <typename R, bool SCALE>
__device__ __forceinline__ void tet_forces(const R t[4], R p0, R p1, R p2, R p3, R p4, R p5, R phi, R f[4]) {
  R d0 = t[1] - t[0], d1 = t[2] - t[0], d2 = t[3] - t[0];
  R v0 = p0 * d0 + p3 * d1 + p5 * d2;
  R v1 = p3 * d0 + p1 * d1 + p4 * d2;
  R v2 = p5 * d0 + p4 * d1 + p2 * d2;
  if (SCALE) {
    v0 *= phi;
    v1 *= phi;
    v2 *= phi;
  }
  f[1] = v0;
  f[2] = v1;
  f[3] = v2;
  f[0] = -((v0 + v1) + v2);
}

// shared-memory element at a byte offset (chunk-local connectivity stores byte
// offsets = position * sizeof(R), so no scaling instruction per corner)
template <typename R>
__device__ __forceinline__ R &sm_at(R *base, int off) {
  return *reinterpret_cast<R *>(reinterpret_cast<char *>(base) + off);
}

// connectivity record of NPE uint16 chunk-local byte offsets
template <int NPE> struct ConnRec;
template <> struct ConnRec<8> {
  using T = uint4;
  __device__ __forceinline__ static void unpack(const uint4 &c, int *idx) {
    idx[0] = c.x & 0xffffu; idx[1] = c.x >> 16; idx[2] = c.y & 0xffffu; idx[3] = c.y >> 16;
    idx[4] = c.z & 0xffffu; idx[5] = c.z >> 16; idx[6] = c.w & 0xffffu; idx[7] = c.w >> 16;
  }
};
template <> struct ConnRec<4> {
  using T = uint2;
  __device__ __forceinline__ static void unpack(const uint2 &c, int *idx) {
    idx[0] = c.x & 0xffffu; idx[1] = c.x >> 16; idx[2] = c.y & 0xffffu; idx[3] = c.y >> 16;
  }
};

// hex8 connectivity packed to 12 bits per corner (streaming colour-phase kernel):
// 96 bits as (a.x, a.y, b), field q = chunk-local position at bits 12q..12q+11.
// unpack yields byte offsets (position * sizeof(R)): one shift (a funnel shift for
// the two fields that straddle a word) and one mask per corner.
struct Conn12 {
  uint2 a;
  uint32_t b;
};
template <typename R> struct ConnRec12 {
  using T = Conn12;
  __device__ __forceinline__ static void unpack(const Conn12 &c, int *idx) {
    constexpr int S = sizeof(R) == 4 ? 2 : 3;  // log2(sizeof(R))
    constexpr uint32_t M = 0xfffu << S;
    idx[0] = (int)((c.a.x << S) & M);
    idx[1] = (int)((c.a.x >> (12 - S)) & M);
    idx[2] = (int)(__funnelshift_r(c.a.x, c.a.y, 24 - S) & M);
    idx[3] = (int)((c.a.y >> (4 - S)) & M);
    idx[4] = (int)((c.a.y >> (16 - S)) & M);
    idx[5] = (int)(__funnelshift_r(c.a.y, c.b, 28 - S) & M);
    idx[6] = (int)((c.b >> (8 - S)) & M);
    idx[7] = (int)((c.b >> (20 - S)) & M);
  }
};

// piecewise-linear table, clamped at the ends (NEXT-2).  tab = [T_0..T_{n-1},
// v_0..v_{n-1}, s_0..s_{n-2}] with the segment slopes s_i = (v_{i+1} - v_i) /
// (T_{i+1} - T_i) precomputed in fp64 on the host, so an evaluation is a search over
// the breakpoints and one FMA, v_i + s_i (T - T_i) -- no division per lookup
// The segment is found by an unrolled binary search (<= 32 points) on the clamped T,
// branch-free apart from the uniform n > 2 test; tab may live in shared memory (the
// streaming element kernel stages both tables per CTA) or global memory.
constexpr int kTabMax = 32;                       // points per table (fed.h)
__device__ __forceinline__ float rclamp(float T, float lo, float hi) { return fminf(fmaxf(T, lo), hi); }
__device__ __forceinline__ double rclamp(double T, double lo, double hi) { return fmin(fmax(T, lo), hi); }
template <typename R>
__device__ __forceinline__ R table_eval(const R *tab, int n, R T) {
  const R Tc = rclamp(T, tab[0], tab[n - 1]);
  int i = 0;
  if (n > 2) {
#pragma unroll
    for (int step = kTabMax / 2; step >= 1; step >>= 1)
      if (i + step <= n - 2 && Tc > tab[i + step]) i += step;
  }
  return tab[n + i] + tab[2 * n + i] * (Tc - tab[i]);
}
// conductivity multiplier k(T)/k_ref at a node (TDK 1: linear law, TDK 2: table or law);
// kt: the table to use (a staged copy), else a.kt
template <typename R, int TDK>
__device__ __forceinline__ R phi_of(const StepArgs<R> &a, R T, const R *kt = nullptr) {
  if (TDK == 3) return a.kl_v0 + a.kl_s * (rclamp(T, a.kl_lo, a.kl_hi) - a.kl_T0);
  if (TDK == 2 && a.n_kt) return table_eval(kt ? kt : a.kt, a.n_kt, T);
  return R(1) + a.beta_k * T;
}
// per-node conductivity multipliers of a chunk's local nodes (TDK 2, tables): four
// independent table searches in flight per thread -- each search is a chain of
// dependent shared-memory reads, and this pass sits between the shared-node gather
// and the first colour phase of every CTA
template <typename R>
__device__ __forceinline__ void phi_pass(const StepArgs<R> &a, const R *sT, R *sPhi, int n, int tid, const R *kt) {
  constexpr int U = 4;
  for (int l0 = tid; l0 < n; l0 += U * kThreads) {
    R v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int l = l0 + j * kThreads;
      v[j] = phi_of<R, 2>(a, l < n ? sT[l] : sT[l0], kt);
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (l0 + j * kThreads < n) sPhi[l0 + j * kThreads] = v[j];
  }
}
// element factor phi_e = mean_a phi(T_a); TDK 2 reads per-node values from
// shared memory (SPHI: the chunk kernels, sPhi filled once per chunk) or looks them up
template <typename R, int TDK, int NPE, bool SPHI = true>
__device__ __forceinline__ R elem_phi(const StepArgs<R> &a, const R *t, const int *idx, const R *sPhi) {
  if (TDK == 0) return R(1);
  if (TDK == 1) {  // linear law: mean of (1 + beta T_a) == 1 + beta mean(T_a)
    R s;
    if constexpr (NPE == 8)  // same pair sums as element_forces (shared by the compiler)
      s = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
    else
      s = (t[0] + t[1]) + (t[2] + t[3]);
    return R(1) + a.beta_k * (s * (R(1) / R(NPE)));
  }
  if (TDK == 3) {  // clamped linear: mean_a phi(T_a) = v0 + s (mean_a clamp(T_a) - T0)
    R s = R(0);
#pragma unroll
    for (int q = 0; q < NPE; ++q) s += rclamp(t[q], a.kl_lo, a.kl_hi);
    return a.kl_v0 + a.kl_s * (s * (R(1) / R(NPE)) - a.kl_T0);
  }
  R s = R(0);
#pragma unroll
  for (int q = 0; q < NPE; ++q) {
    if constexpr (SPHI)
      s += sm_at(const_cast<R *>(sPhi), idx[q]);
    else
      s += phi_of<R, 2>(a, t[q]);
  }
  return s * (R(1) / R(NPE));
}

template <typename R, int TDK, int NPE, bool SPHI = true>
__device__ __forceinline__ void elem_forces(const StepArgs<R> &a, const R *t, const int *idx, const R *sPhi,
                                            const R *pp, R *f) {
  const R phi = elem_phi<R, TDK, NPE, SPHI>(a, t, idx, sPhi);
  if constexpr (NPE == 8)
    element_forces<R, TDK != 0>(t, pp[0], pp[1], pp[2], pp[3], pp[4], pp[5], phi, f);
  else
    tet_forces<R, TDK != 0>(t, pp[0], pp[1], pp[2], pp[3], pp[4], pp[5], phi, f);
}

// c(T) / c_scale at a node: TDK 0 -> 1 (coef holds dt/(rho c V)); TDK 1 -> 1 + beta_c T
// (coef = dt/(rho c0 V)); TDK 2 -> table or c0 (1 + beta_c T) (coef = dt/(rho V))
template <typename R, int TDK>
__device__ __forceinline__ R c_factor(const StepArgs<R> &a, R T, const R *ct = nullptr) {
  if (TDK == 0) return R(1);
  if (TDK == 1) return R(1) + a.beta_c * T;
  if (TDK == 3) return a.cl_v0 + a.cl_s * (rclamp(T, a.cl_lo, a.cl_hi) - a.cl_T0);
  if (a.n_ct) return table_eval(ct ? ct : a.ct, a.n_ct, T);
  return a.c0 * (R(1) + a.beta_c * T);
}

template <typename R, int TDK>
__device__ __forceinline__ R explicit_update(const StepArgs<R> &a, R T, R F, R Q, R coef, const R *ct = nullptr) {
  // Eq. 16 with reading R1: T + dt / (M c(T)) (Q - F_int)
  R d = coef * (Q - F);
  if (TDK != 0) {
    if constexpr (sizeof(R) == 4)
      d = __fdividef(d, c_factor<R, TDK>(a, T, ct));  // 2 ulp on the increment, << the fp32 tolerance
    else
      d = d / c_factor<R, TDK>(a, T, ct);
  }
  return T + d;
}

// 4 consecutive values with 16-byte accesses (global or shared memory)
template <typename R> struct Vec4;
template <> struct Vec4<float> {
  float v[4];
  __device__ __forceinline__ void load(const float *p) {
    float4 x = *reinterpret_cast<const float4 *>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  __device__ __forceinline__ void store(float *p) const {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec4<double> {
  double v[4];
  __device__ __forceinline__ void load(const double *p) {
    double2 x = reinterpret_cast<const double2 *>(p)[0], y = reinterpret_cast<const double2 *>(p)[1];
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
  }
  __device__ __forceinline__ void store(double *p) const {
    reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
  }
};

// One 16-byte access per thread: 4 floats or 2 doubles.  The element kernels'
// interior epilogue reads shared memory and writes HBM with these, so a warp's
// instruction covers 512 contiguous bytes in both precisions (two 16-byte halves
// of a 32-byte double Vec4 per thread would leave a 32-byte stride: 2-way bank
// conflicts and half-filled sectors per instruction).
template <typename R> struct Vec16;
template <> struct Vec16<float> : Vec4<float> { static constexpr int n = 4; };
template <> struct Vec16<double> {
  static constexpr int n = 2;
  double v[2];
  __device__ __forceinline__ void load(const double *p) {
    double2 x = *reinterpret_cast<const double2 *>(p);
    v[0] = x.x; v[1] = x.y;
  }
  __device__ __forceinline__ void store(double *p) const {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
  }
};

// ---------------------------------------------------------------- peer signalling
// PEER transport: the interface chunks are the first n_sig_ctas CTAs of the
// step's element launch (dispatched first, so they finish early).  Each fences its
// reductions and counts itself done; the last one publishes "step k's interface
// loads are complete" as the value k + 1 in the neighbours' flags (release, system
// scope) while the interior chunks are still running.  Flags only grow, so they
// never need resetting.  Call with all threads of the CTA.
template <typename R>
__device__ __forceinline__ void signal_peers(const StepArgs<R> &a) {
  if ((int)blockIdx.x >= a.n_sig_ctas) return;  // uniform per CTA
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(a.if_done, 1u);
    if (prev == (unsigned)a.n_sig_ctas - 1u) {
      __threadfence_system();
      *a.if_done = 0u;  // next launch is stream-ordered after this one
      const unsigned long long v = (unsigned long long)(*a.step_base + a.k_off) + 1ull;
      if (a.psig_lo) st_release_sys(a.psig_lo, v);
      if (a.psig_hi) st_release_sys(a.psig_hi, v);
    }
  }
}

// Node kernel side: thread 0 of a block that holds interface nodes waits until
// both neighbours have published this step (bounded by a.wait_ns, then peer_err is
// set and the block proceeds, so a lost peer never hangs the GPU; fed_step reports
// the failure and the state is undefined).
template <typename R>
__device__ __forceinline__ void wait_peers(const StepArgs<R> &a, unsigned long long target) {
  if (a.free_run) return;
  const unsigned long long t0 = globaltimer_ns();
  for (int d = 0; d < 2; ++d) {
    const bool need = d == 0 ? a.n_if_lo > 0 : a.n_if > a.n_if_lo;
    if (!need) continue;
    while (ld_acquire_sys(a.sig + d) < target) {
      if (globaltimer_ns() - t0 > a.wait_ns) {
        atomicOr(a.peer_err, 1u);
        break;
      }
      __nanosleep(100);
    }
  }
}

template <typename R>
__device__ __forceinline__ R face_load(const StepArgs<R> &a, int s, R T) {
  // sum over the node's face-BC records of (sum_f A_f/4) q_b(T)   (Eqs. 4, 5, 7; R9-R11)
  // packed record j: coef = (sum_f A_f/4) x (q | h | eps sigma), tinf, kind
  R Q = R(0);
  const int j1 = a.bc_ptr[s + 1];
  FED_DCHECK(a, a.bc_ptr[s] >= 0 && a.bc_ptr[s] <= j1, 5);
  for (int j = a.bc_ptr[s]; j < j1; ++j) {
    const int kind = a.bc_ekind[j];
    const R cf = a.bc_coef[j], Ti = a.bc_tinf[j];
    if (kind == 1) {
      Q += cf;                                           // Eq. 5: flux into the body
    } else if (kind == 2) {
      Q -= cf * (T - Ti);                                // Eq. 4: h (T - T_inf)
    } else {
      // Eq. 7: eps sigma [(T-Tz)^4 - (Tinf-Tz)^4], factored to avoid cancellation (Kelvin)
      const R Ta = T + R(273.15), Tb = Ti + R(273.15);
      Q -= cf * ((T - Ti) * (Ta + Tb) * (Ta * Ta + Tb * Tb));
    }
  }
  return Q;
}

// ---------------------------------------------------------------- chunk kernel
// Shared memory layout (bytes, 16-aligned):
//   [0,16)                 mbarrier
//   conn   chunk_cap * 16                 (1-D TMA)
//   P      6 * chunk_cap * sizeof(R)      (1-D TMA)
//   sT     max_local * sizeof(R)          interior part by 1-D TMA, shared part gathered
//   sF     max_local * sizeof(R)
//   sCoef  max_local * sizeof(R)          interior part by 1-D TMA
//   sQ     max_local * sizeof(R)          interior part by 1-D TMA (only with a source)
//   sSp    max_local * 4
//   sCol   (kMaxColorsDev + 1) * 4
// Chunk-local node ids: [0, n_int) interior (8-padded to n_int_pad), then the
// shared ("special") nodes at [n_int_pad, n_int_pad + n_sp).
// Streaming element kernel: sT, sF hold every local node (max_local), sCoef and sQ
// only the TMA-streamed interior range (max_int), sSp the shared-node list
// (max_sp).  The smaller the footprint, the more of the SM's unified L1 stays cache
// for the record loads (measured: 38 -> 32 KB per CTA, 0.677 -> 0.653 ms/step).
template <typename R>
__host__ __device__ inline size_t stream_smem_bytes(int chunk_cap, int max_local, int max_int, int max_sp,
                                                    bool staged, bool phi) {
  size_t b = 16;
  if (phi) b += (size_t)max_local * sizeof(R) + 16 + (size_t)2 * 3 * kTabMax * sizeof(R);  // sPhi + staged tables
  if (staged) {
    b += (size_t)chunk_cap * 16;
    b += (size_t)6 * chunk_cap * sizeof(R);
  }
  b += (size_t)max_local * sizeof(R) * 2 + (size_t)max_int * sizeof(R) * 2;
  b += (size_t)max_sp * 4;
  b += (kMaxColorsDev + 1) * 4;
  b = (b + 15) & ~(size_t)15;
  if (kChecked) b += (size_t)max_local * 4;  // per-node touch counters of a colour phase
  return (b + 15) & ~(size_t)15;
}

// LS > 0 (resident kernel): sT and sF are LS entries each, so sF sits at a
// compile-time distance from sT and one address register serves both (immediate
// offset); the other arrays keep max_local entries.
constexpr int kLS = 2304;  // >= the bank-layout capacity 2 * chunk + 256 of chunks <= 1024

template <typename R>
__host__ __device__ inline size_t chunk_smem_bytes(int chunk_cap, int max_local, bool staged, bool phi = false,
                                                   int ls = 0) {
  size_t b = 16;
  if (phi) b += (size_t)max_local * sizeof(R) + 16;
  if (staged) {
    b += (size_t)chunk_cap * 16;
    b += (size_t)6 * chunk_cap * sizeof(R);
  }
  b += (size_t)(ls > 0 ? ls : max_local) * sizeof(R) * 2 + (size_t)max_local * sizeof(R) * 2;
  b += (size_t)max_local * 4;
  b += (kMaxColorsDev + 1) * 4;
  return (b + 15) & ~(size_t)15;
}

template <typename R>
__device__ __forceinline__ void smem_add(R *p, R v) { atomicAdd(p, v); }  // CAS loop on sm_100a

// MODE 0: element records staged by 1-D TMA; colour phases (plain shared-memory
//         read-modify-write, one barrier per colour)
// MODE 1: element records staged by 1-D TMA; shared-memory compare-and-swap adds
// MODE 2: element records loaded straight into registers (coalesced 16 B / 4 B
//         loads issued before the barrier); compare-and-swap adds; no staging
//         buffers -> ~3x less shared memory per CTA, higher occupancy
// MODE 3: colour phases with element records loaded straight into registers;
//         the next colour's records are in flight while the current one runs
#ifndef FED_TDK2_CTAS
#define FED_TDK2_CTAS 6
#endif
template <typename R, int TDK, int MODE, int NPE, int LS = 0>
// MODE 3 residency: 7 CTAs/SM in fp32 (<= 72 registers, tabulated k/c included since
// the tables carry precomputed slopes: 80 -> 72 registers, 24 -> 16 B of spills), 4 in
// fp64 (<= 128) -- made possible by loading the later colours' records during the
// phases (fast path)
__global__ void __launch_bounds__(kThreads, MODE == 3 ? (sizeof(R) == 4 ? (TDK == 2 ? FED_TDK2_CTAS : 7) : 4) : 1)
element_chunk_kernel(StepArgs<R> a, int chunk_base) {
  static_assert(NPE == 8 || MODE >= 2, "staged modes are hex8-only");
  static_assert(LS == 0 || MODE == 3, "fixed sT/sF stride only in the colour-phase register mode");
  // MODE 3 fp32 hex reads one 16-byte record per element (12-bit packed connectivity
  // + P_xx) and five operator planes; the other kernels the 16-bit byte offsets (16 B)
  // and six planes
  constexpr bool C12 = MODE == 3 && NPE == 8 && sizeof(R) == 4;
  using CR = std::conditional_t<C12, ConnRec12<R>, ConnRec<NPE>>;
  using CT = typename CR::T;
  using CT16 = typename ConnRec<NPE>::T;
  const CT16 *gconn = reinterpret_cast<const CT16 *>(a.conn16);
  constexpr bool STAGED = MODE < 2;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  uint4 *sConn = reinterpret_cast<uint4 *>(smem + 16);
  R *sP = reinterpret_cast<R *>(smem + 16 + (STAGED ? (size_t)a.chunk_cap * 16 : 0));
  R *sT = sP + (STAGED ? 6 * a.chunk_cap : 0);
  R *sF = sT + (LS > 0 ? LS : a.max_local);
  R *sCoef = sF + (LS > 0 ? LS : a.max_local);
  R *sQ = sCoef + a.max_int;
  int *sSp = reinterpret_cast<int *>(sQ + a.max_int);
  int *sCol = sSp + a.max_sp;
  // TDK 2: per-node conductivity multipliers phi(T_l) (tables), after sCol, 16-aligned
  R *sPhi = TDK == 2 ? reinterpret_cast<R *>((reinterpret_cast<uintptr_t>(sCol + kMaxColorsDev + 1) + 15) &
                                             ~uintptr_t(15))
                     : nullptr;
  // TDK 2: the k and c tables staged per CTA after sPhi (3 kTabMax entries each)
  R *sKt = TDK == 2 ? sPhi + a.max_local : nullptr;
  R *sCt = TDK == 2 ? sKt + 3 * kTabMax : nullptr;
  // checked build: colour-phase touch counters after everything else (16-aligned)
  int *sChk = reinterpret_cast<int *>(
      (reinterpret_cast<uintptr_t>(TDK == 2 ? (void *)(sCt + 3 * kTabMax) : (void *)(sCol + kMaxColorsDev + 1)) + 15) &
      ~uintptr_t(15));

  const int tid = threadIdx.x;
  const int c = chunk_base + blockIdx.x;
  // 64-byte chunk header (fed_plan.h): one dependent load before everything else
  const int4 *h4 = reinterpret_cast<const int4 *>(a.chunk_hdr) + (size_t)c * 4;
#if FED_L2_KEEP & 1
  const uint64_t polk_h = l2_keep_policy();
  const int4 h0 = ld_keep(h4, polk_h), h1 = ld_keep(h4 + 1, polk_h);
#else
  const int4 h0 = __ldg(h4), h1 = __ldg(h4 + 1);
#endif
  const int elem_off = h0.x, n_elem = h0.y, n_pad = h0.z, int_start = h0.w, n_int = h1.x, sp_off = h1.y,
            n_sp = h1.z, n_col = h1.w;
  const int n_int_pad = (n_int + 7) & ~7;
  FED_DCHECK(a, int_start >= 0 && int_start + n_int_pad <= a.N_int + 8 && n_int_pad + n_sp <= a.max_local &&
                    n_int_pad <= a.max_int && n_sp <= a.max_sp, 2);
  FED_DCHECK(a, elem_off >= 0 && elem_off + n_pad <= a.n_slots && n_elem <= n_pad, 4);
  const int n_loc_bytes = (n_int_pad + n_sp) * (int)sizeof(R);
  if (kChecked)
    for (int l = tid; l < n_int_pad + n_sp; l += kThreads) sChk[l] = 0;
  if constexpr (TDK == 2) {  // static data: before the dependency wait; used after a barrier
    if (a.n_kt)
      for (int l = tid; l < 3 * a.n_kt - 1; l += kThreads) sKt[l] = __ldg(a.kt + l);
    if (a.n_ct)
      for (int l = tid; l < 3 * a.n_ct - 1; l += kThreads) sCt[l] = __ldg(a.ct + l);
  }
  // after the prologue barrier: wait for the 1-D TMA (interior node data + the chunk's
  // shared-node list), then gather the shared nodes' T (they are also read by other
  // chunks, so they are not in the streamed range); TDK 2: per-node phi for k(T)
  auto after_wait = [&]() {
    mbar_wait(bar, 0);
    constexpr int G = 8;  // independent loads in flight per thread
    for (int base = 0; base < n_sp; base += G * kThreads) {
      R tv[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int l = base + j * kThreads + tid;
        const int si = l < n_sp ? sSp[l] : -1;
        FED_DCHECK(a, si < a.N_sp, 1);
#if FED_L2_KEEP & 8
        tv[j] = si >= 0 && (!kChecked || si < a.N_sp) ? ld_keep(a.T + a.N_int + si, l2_keep_policy()) : R(0);
#else
        tv[j] = si >= 0 && (!kChecked || si < a.N_sp) ? a.T[a.N_int + si] : R(0);
#endif
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int l = base + j * kThreads + tid;
        if (l < n_sp) sT[n_int_pad + l] = tv[j];
      }
    }
    __syncthreads();
    if constexpr (TDK == 2) {
      phi_pass<R>(a, sT, sPhi, n_int_pad + n_sp, tid, sKt);
      __syncthreads();
    }
  };

  pdl_trigger();  // the next kernel's CTAs may be scheduled once every CTA got here
  const uint32_t nbytes = (uint32_t)(n_int_pad * sizeof(R));
  const uint64_t pol = l2_policy(a.l2_stream);  // streamed-once data: evict first from L2
  if (tid == 0) {
    // 1-D TMA (SASS UBLKCP) on one mbarrier: the contiguous interior-node ranges of
    // T, coef (and Q), the chunk's shared-node list, and in the staged modes the
    // element records (connectivity + 6 operator planes).  Static data first; the
    // interior T (written by the previous step) after the dependency wait below.
    mbar_init(bar, 1);
    fence_mbar_init();
    fence_proxy_async();
    const uint32_t pbytes = (uint32_t)(n_pad * sizeof(R));
    const uint32_t sbytes = (uint32_t)(((n_sp + 3) & ~3) * 4);
    const int nn = a.Qvol ? 3 : 2;
    mbar_expect_tx(bar, (STAGED ? (uint32_t)n_pad * 16u + 6u * pbytes : 0u) + (uint32_t)nn * nbytes + sbytes);
    if (STAGED) {
      bulk_g2s(sConn, a.conn16 + elem_off, (uint32_t)n_pad * 16u, bar);
#pragma unroll
      for (int q = 0; q < 6; ++q) bulk_g2s(sP + q * a.chunk_cap, a.P + (size_t)q * a.n_slots + elem_off, pbytes, bar);
    }
    if (nbytes) {
      bulk_g2s(sCoef, a.coef + int_start, nbytes, bar, pol);
      if (a.Qvol) bulk_g2s(sQ, a.Qvol + int_start, nbytes, bar, pol);
    }
    if (sbytes) bulk_g2s(sSp, a.sp_list + sp_off, sbytes, bar, pol);
    // T of this step's interior nodes: after the previous kernel (programmatic-launch
    // dependency wait, a no-op otherwise); the other threads wait before the gather
    pdl_wait();
    if (nbytes) bulk_g2s(sT, a.T + int_start, nbytes, bar, pol);
  }
  auto issue_T = [&]() { pdl_wait(); };
  for (int l = tid; l < n_int_pad + n_sp; l += kThreads) sF[l] = R(0);
  if (MODE == 0 && tid <= kMaxColorsDev) sCol[tid] = a.color_off[(size_t)c * (kMaxColorsDev + 1) + tid];
  if constexpr (MODE == 3) {
    auto load_el = [&](int e, CT &cc, R *pp) {
      if constexpr (C12) {
        const uint4 r = ld_rec(a.rec12 + elem_off + e, pol);
        cc.a = make_uint2(r.x, r.y);
        cc.b = r.z;
        pp[0] = __uint_as_float(r.w);
#pragma unroll
        for (int q = 1; q < 6; ++q) pp[q] = ld_rec(a.P + (size_t)q * a.n_slots + elem_off + e, pol);
      } else {
        cc = ld_rec(gconn + elem_off + e, pol);
#pragma unroll
        for (int q = 0; q < 6; ++q) pp[q] = ld_rec(a.P + (size_t)q * a.n_slots + elem_off + e, pol);
      }
    };
    auto do_el = [&](const CT &cc, const R *pp) {
      int idx[NPE];
      CR::unpack(cc, idx);
      R t[NPE], f[NPE];
      if (kChecked) {
#pragma unroll
        for (int q = 0; q < NPE; ++q) {
          FED_DCHECK(a, idx[q] < n_loc_bytes && idx[q] % (int)sizeof(R) == 0, 0);
          if (idx[q] >= n_loc_bytes) idx[q] = 0;
          atomicAdd(&sChk[idx[q] / (int)sizeof(R)], 1);
        }
      }
#pragma unroll
      for (int q = 0; q < NPE; ++q) t[q] = sm_at(sT, idx[q]);
      elem_forces<R, TDK, NPE>(a, t, idx, sPhi, pp, f);
#pragma unroll
      for (int q = 0; q < NPE; ++q) sm_at(sF, idx[q]) += f[q];
    };
    // checked build, after a colour phase's barrier: every node an element of the phase
    // touched was touched once (elements of one colour share no node); then reset
    auto check_phase = [&](bool had, const CT &cc) {
      if (!kChecked) return;
      int idx[NPE];
      CR::unpack(cc, idx);
      if (had && NPE == 8)
#pragma unroll
        for (int q = 0; q < NPE; ++q)
          if (idx[q] < n_loc_bytes) FED_DCHECK(a, sChk[idx[q] / (int)sizeof(R)] == 1, 3);
      __syncthreads();
      if (had)
#pragma unroll
        for (int q = 0; q < NPE; ++q)
          if (idx[q] < n_loc_bytes) sChk[idx[q] / (int)sizeof(R)] = 0;
      __syncthreads();
    };
    // fast path (structured-like chunks): <= 8 colours of <= kThreads elements ->
    // every element record of the thread is loaded up front, one round trip
#if FED_L2_KEEP & 1
    const int4 h2 = ld_keep(h4 + 2, polk_h), h3 = ld_keep(h4 + 3, polk_h);  // colour offsets 1..8 (header words 8..15)
#else
    const int4 h2 = __ldg(h4 + 2), h3 = __ldg(h4 + 3);  // colour offsets 1..8 (header words 8..15)
#endif
    const int cof[9] = {0, h2.x, h2.y, h2.z, h2.w, h3.x, h3.y, h3.z, h3.w};
    bool fast = n_col <= 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) fast = fast && (cof[k + 1] - cof[k] <= kThreads);
    if (fast) {
      CT cc[8];
      R pp[8][6];
      // fp32: records of colours 0..3 are loaded up front, colours 4-5 during phase 1
      // and 6-7 during phase 3, into the registers that finished colours free again
      // (each load still has three phases to arrive): at most 50 live record
      // registers instead of 80, so 7 CTAs share an SM (cfg5 element kernel 0.596 ->
      // 0.538 ms, same box; colours 6-7 at phase 2 with 6 CTAs/SM gave 0.548).
      // fp64 stays at 4 CTAs/SM either way, so it loads colours 0..5 up front and
      // 6-7 during phase 2 (the fp32 schedule costs it 924 -> 1138 us in ncu).
      constexpr bool kStag = sizeof(R) == 4;
      constexpr int KE = kStag ? 4 : 6;
#pragma unroll
      for (int k = 0; k < KE; ++k) {
        const int e = cof[k] + tid;
        if (e < cof[k + 1]) load_el(e, cc[k], pp[k]);
      }
      issue_T();
      __syncthreads();
      after_wait();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (kStag ? (k == 1 || k == 3) : k == 2) {
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            const int kk = (kStag && k == 1 ? 4 : 6) + k2;
            const int e = cof[kk] + tid;
            if (e < cof[kk + 1]) load_el(e, cc[kk], pp[kk]);
          }
        }
        if (k < n_col) {
          if (cof[k] + tid < cof[k + 1]) do_el(cc[k], pp[k]);
          __syncthreads();
          check_phase(cof[k] + tid < cof[k + 1], cc[k]);
        }
      }
    } else {
    if (tid <= kMaxColorsDev) sCol[tid] = a.color_off[(size_t)c * (kMaxColorsDev + 1) + tid];
    CT ccA = {};
    R pA[6];
    const int c0 = cof[0], c1 = cof[1];
    bool vA = n_col > 0 && c0 + tid < c1;
    if (vA) load_el(c0 + tid, ccA, pA);
    issue_T();
    __syncthreads();
    after_wait();
    for (int k = 0; k < n_col; ++k) {
      CT ccB = {};
      R pB[6];
      const int nb = sCol[k + 1], ne1 = (k + 1 < n_col) ? sCol[k + 2] : nb;
      const bool vB = nb + tid < ne1;
      if (vB) load_el(nb + tid, ccB, pB);
      if (vA) do_el(ccA, pA);
      for (int e = sCol[k] + tid + kThreads; e < nb; e += kThreads) {
        CT cc;
        R pp[6];
        load_el(e, cc, pp);
        do_el(cc, pp);
      }
      __syncthreads();
      ccA = ccB;
#pragma unroll
      for (int q = 0; q < 6; ++q) pA[q] = pB[q];
      vA = vB;
    }
    }
  } else if constexpr (MODE == 2) {
    // batches of up to 4 elements per thread; the first batch's loads overlap the prologue
    constexpr int EPT = 4;
    for (int base = 0; base < n_elem; base += EPT * kThreads) {
      CT cc[EPT];
      R pp[EPT][6];
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = base + j * kThreads + tid;
        if (e < n_elem) {
          cc[j] = __ldg(gconn + elem_off + e);
#pragma unroll
          for (int q = 0; q < 6; ++q) pp[j][q] = __ldg(a.P + (size_t)q * a.n_slots + elem_off + e);
        }
      }
      if (base == 0) {
        issue_T();
        __syncthreads();
        after_wait();
      }
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = base + j * kThreads + tid;
        if (e < n_elem) {
          int idx[NPE];
          CR::unpack(cc[j], idx);
          R t[NPE], f[NPE];
#pragma unroll
          for (int q = 0; q < NPE; ++q) t[q] = sm_at(sT, idx[q]);
          elem_forces<R, TDK, NPE>(a, t, idx, sPhi, pp[j], f);
#pragma unroll
          for (int q = 0; q < NPE; ++q) smem_add(&sm_at(sF, idx[q]), f[q]);
        }
      }
    }
    if (n_elem == 0) {
      issue_T();
      __syncthreads();
      after_wait();
    }
    __syncthreads();
  } else {
    issue_T();
    __syncthreads();
    after_wait();
  }

  if (MODE == 0) {
    // colour phases: elements of one colour share no node -> plain shared-memory RMW
    for (int k = 0; k < n_col; ++k) {
      const int e1 = sCol[k + 1];
      for (int e = sCol[k] + tid; e < e1; e += kThreads) {
        uint4 cc = sConn[e];
        int idx[8] = {(int)(cc.x & 0xffffu), (int)(cc.x >> 16), (int)(cc.y & 0xffffu), (int)(cc.y >> 16),
                      (int)(cc.z & 0xffffu), (int)(cc.z >> 16), (int)(cc.w & 0xffffu), (int)(cc.w >> 16)};
        R t[8], f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = sm_at(sT, idx[q]);
        const R pe[6] = {sP[e], sP[a.chunk_cap + e], sP[2 * a.chunk_cap + e], sP[3 * a.chunk_cap + e],
                         sP[4 * a.chunk_cap + e], sP[5 * a.chunk_cap + e]};
        elem_forces<R, TDK, 8>(a, t, idx, sPhi, pe, f);
#pragma unroll
        for (int q = 0; q < 8; ++q) sm_at(sF, idx[q]) += f[q];
      }
      __syncthreads();
    }
  } else if (MODE >= 2) {
    // element records were loaded into registers in the prologue branch above
  } else {
    for (int e = tid; e < n_elem; e += kThreads) {
      uint4 cc = sConn[e];
      int idx[8] = {(int)(cc.x & 0xffffu), (int)(cc.x >> 16), (int)(cc.y & 0xffffu), (int)(cc.y >> 16),
                    (int)(cc.z & 0xffffu), (int)(cc.z >> 16), (int)(cc.w & 0xffffu), (int)(cc.w >> 16)};
      R t[8], f[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) t[q] = sm_at(sT, idx[q]);
      const R pe[6] = {sP[e], sP[a.chunk_cap + e], sP[2 * a.chunk_cap + e], sP[3 * a.chunk_cap + e],
                       sP[4 * a.chunk_cap + e], sP[5 * a.chunk_cap + e]};
      elem_forces<R, TDK, 8>(a, t, idx, sPhi, pe, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) smem_add(&sm_at(sF, idx[q]), f[q]);
    }
    __syncthreads();
  }

  // fused explicit update of chunk-interior nodes (Eq. 16); they have no face
  // load, no Dirichlet value and are touched by no other chunk
  // (16-byte accesses, 4 fp32 / 2 fp64 nodes per thread: n_int is a multiple of
  // 8, the interior range starts 8-aligned)
  float dmax = 0.f;
  constexpr int G = Vec16<R>::n;
  for (int l = G * tid; l < n_int; l += G * kThreads) {
    Vec16<R> T4, F4, C4, Q4, N4;
    T4.load(sT + l);
    F4.load(sF + l);
    C4.load(sCoef + l);
    if (a.Qvol) Q4.load(sQ + l);
#pragma unroll
    for (int q = 0; q < G; ++q) {
      N4.v[q] = explicit_update<R, TDK>(a, T4.v[q], F4.v[q], a.Qvol ? Q4.v[q] : R(0), C4.v[q], sCt);
      flag_unstable(a, N4.v[q]);
      dmax = fmaxf(dmax, (float)rabs(N4.v[q] - T4.v[q]));
    }
    N4.store(a.T + int_start + l);
  }
  if (a.dTmax) warp_max_to(a.dTmax, dmax);
  // shared nodes: reduce the chunk's partial loads into F (PEER transport: interface
  // nodes into this step's parity buffer, which the neighbour reads)
  {
    // shared nodes into F (PEER transport: interface nodes into this step's parity
    // buffer Fif[g & 1], which the neighbour reads)
    R *Fl = a.F + a.N_int;
    R *Fi = a.Fif ? a.Fif + ((*a.step_base + a.k_off) & 1) * a.n_if : Fl;
    for (int l = tid; l < n_sp; l += kThreads) {
      const int s = sSp[l];  // -1: hole of the bank layout
      FED_DCHECK(a, s < a.N_sp, 1);
#if FED_L2_KEEP & 16
      if (s >= 0 && (!kChecked || s < a.N_sp)) red_add_keep(s < a.n_if ? Fi + s : Fl + s, sF[n_int_pad + l], l2_keep_policy());
#else
      if (s >= 0 && (!kChecked || s < a.N_sp)) red_add(s < a.n_if ? Fi + s : Fl + s, sF[n_int_pad + l]);
#endif
    }
  }
  if (a.if_done) signal_peers(a);
}

// ---------------------------------------------------------------- atomic baseline
template <typename R, int TDK, int NPE>
__global__ void __launch_bounds__(256) element_atomic_kernel(StepArgs<R> a) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n_slots) return;
  int idx[NPE];
  int4 c0 = __ldg(a.conn32 + (NPE / 4) * s);
  idx[0] = c0.x; idx[1] = c0.y; idx[2] = c0.z; idx[3] = c0.w;
  if constexpr (NPE == 8) {
    int4 c1 = __ldg(a.conn32 + 2 * s + 1);
    idx[4] = c1.x; idx[5] = c1.y; idx[6] = c1.z; idx[7] = c1.w;
  }
  if (idx[0] < 0) return;  // padding slot
  R t[NPE], f[NPE], pp[6];
#pragma unroll
  for (int q = 0; q < NPE; ++q) t[q] = __ldg(a.T + idx[q]);
#pragma unroll
  for (int q = 0; q < 6; ++q) pp[q] = __ldg(a.P + (size_t)q * a.n_slots + s);
  elem_forces<R, TDK, NPE, false>(a, t, idx, (const R *)nullptr, pp, f);
#pragma unroll
  for (int q = 0; q < NPE; ++q) red_add(a.F + idx[q], f[q]);
}

// ---------------------------------------------------------------- measured scatter baselines
// One thread per element slot over global node arrays (conn32: internal node ids).
// VAR 1 (FED_SCATTER_ATOMIC_WARP): slots in Morton order, so lanes (2k, 2k+1) are
//   usually x-neighbours; the even lane adds the odd lane's loads of the four
//   shared nodes (corners 0,3,4,7 of the odd lane = 1,2,6,5 of the even lane,
//   checked by node id) and the odd lane skips those red.global.add.
// VAR 2 (FED_SCATTER_COLOR_PASSES): slots list[begin, end) of one colour, plain
//   read-modify-write of F (no two elements of a colour share a node).
// VAR 3 (FED_SCATTER_GATHER): the element flux v_e = phi P S^T T_e to v[3][slots].
template <typename R, int TDK, int NPE, int VAR>
__global__ void __launch_bounds__(256) element_scatter_kernel(StepArgs<R> a, const int32_t *list, int64_t begin,
                                                              int64_t end, R *v) {
  const int64_t t = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < end;
  const int64_t s = VAR == 2 ? (live ? list[t] : 0) : t;
  int idx[NPE];
  bool valid = live;
  if (live) {
    int4 c0 = __ldg(a.conn32 + (NPE / 4) * s);
    idx[0] = c0.x; idx[1] = c0.y; idx[2] = c0.z; idx[3] = c0.w;
    if constexpr (NPE == 8) {
      int4 c1 = __ldg(a.conn32 + 2 * s + 1);
      idx[4] = c1.x; idx[5] = c1.y; idx[6] = c1.z; idx[7] = c1.w;
    }
    valid = idx[0] >= 0;  // padding slot
  }
  R t8[NPE], f[NPE], pp[6];
  if (valid) {
#pragma unroll
    for (int q = 0; q < NPE; ++q) t8[q] = __ldg(a.T + idx[q]);
#pragma unroll
    for (int q = 0; q < 6; ++q) pp[q] = __ldg(a.P + (size_t)q * a.n_slots + s);
  }
  if constexpr (VAR == 3) {
    if (!valid) return;
    // v = phi P u with u = S^T T_e (hex: natural signs; tet: edge differences)
    const R phi = elem_phi<R, TDK, NPE, false>(a, t8, idx, (const R *)nullptr);
    R u0, u1, u2;
    if constexpr (NPE == 8) {
      u0 = ((t8[1] - t8[0]) + (t8[2] - t8[3])) + ((t8[5] - t8[4]) + (t8[6] - t8[7]));
      u1 = ((t8[2] + t8[3]) - (t8[0] + t8[1])) + ((t8[6] + t8[7]) - (t8[4] + t8[5]));
      u2 = ((t8[4] + t8[5]) + (t8[6] + t8[7])) - ((t8[0] + t8[1]) + (t8[2] + t8[3]));
    } else {
      u0 = t8[1] - t8[0];
      u1 = t8[2] - t8[0];
      u2 = t8[3] - t8[0];
    }
    if (TDK != 0) {
      u0 *= phi;
      u1 *= phi;
      u2 *= phi;
    }
    v[s] = pp[0] * u0 + pp[3] * u1 + pp[5] * u2;
    v[a.n_slots + s] = pp[3] * u0 + pp[1] * u1 + pp[4] * u2;
    v[2 * a.n_slots + s] = pp[5] * u0 + pp[4] * u1 + pp[2] * u2;
    return;
  } else {
    if (valid) elem_forces<R, TDK, NPE, false>(a, t8, idx, (const R *)nullptr, pp, f);
    if constexpr (VAR == 2) {
      if (!valid) return;
#pragma unroll
      for (int q = 0; q < NPE; ++q) a.F[idx[q]] += f[q];  // one colour: no conflicts
    } else {
      // x-pair aggregation: even lane absorbs the odd lane's loads at shared nodes
      unsigned skip = 0;
      if constexpr (NPE == 8) {
        const int lane = threadIdx.x & 31;
        const int mine[4] = {1, 2, 6, 5}, theirs[4] = {0, 3, 7, 4};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int ni = __shfl_down_sync(0xffffffffu, valid ? idx[theirs[k]] : -1, 1);
          const R nf = __shfl_down_sync(0xffffffffu, valid ? f[theirs[k]] : R(0), 1);
          const bool take = valid && !(lane & 1) && lane < 31 && ni >= 0 && ni == idx[mine[k]];
          if (take) f[mine[k]] += nf;
          const int took = __shfl_up_sync(0xffffffffu, take ? 1 : 0, 1);
          if ((lane & 1) && took) skip |= 1u << theirs[k];
        }
      }
      if (!valid) return;
#pragma unroll
      for (int q = 0; q < NPE; ++q)
        if (!(skip & (1u << q))) red_add(a.F + idx[q], f[q]);
    }
  }
}

// FED_SCATTER_GATHER phase 2: F_n = sum over the node's (slot, corner) of s_corner . v_slot
template <typename R, int NPE>
__global__ void __launch_bounds__(256) gather_kernel(StepArgs<R> a, const int32_t *g_ptr, const int32_t *g_list,
                                                     const R *v) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.N_loc) return;
  R F = R(0);
  const int j1 = __ldg(g_ptr + n + 1);
  for (int j = __ldg(g_ptr + n); j < j1; ++j) {
    const int e = __ldg(g_list + j);
    const int64_t s = e >> 3;
    const int q = e & 7;
    const R v0 = __ldg(v + s), v1 = __ldg(v + a.n_slots + s), v2 = __ldg(v + 2 * a.n_slots + s);
    if constexpr (NPE == 8) {
      // natural signs of the S:93 corner order
      const R sx = (q == 1 || q == 2 || q == 5 || q == 6) ? R(1) : R(-1);
      const R sy = (q == 2 || q == 3 || q == 6 || q == 7) ? R(1) : R(-1);
      const R sz = q >= 4 ? R(1) : R(-1);
      F += sx * v0 + sy * v1 + sz * v2;
    } else {
      F += q == 0 ? -((v0 + v1) + v2) : (q == 1 ? v0 : (q == 2 ? v1 : v2));
    }
  }
  a.F[n] = F;
}

// ---------------------------------------------------------------- node kernel
template <typename R, int TDK>
__device__ __forceinline__ R node_update(const StepArgs<R> &a, int64_t n, R T, R F, R coef, R Q, int kind,
                                         long long step) {
  if (n >= a.N_int) {
    const int s = (int)(n - a.N_int);
    if (s < a.n_if) {
      if (a.Fif) {
        // PEER: own parity buffer + the neighbour's, loaded from its memory; then clear
        // the other parity (the neighbour finished reading it: its flag for this step
        // was raised after its previous node update)
        const int64_t p = step & 1;
        const R own = __ldcg(a.Fif + p * a.n_if + s);
        a.Fif[(p ^ 1) * a.n_if + s] = R(0);
        const R rx = s < a.n_if_lo ? __ldcv(a.pF_lo + p * a.pstride_lo + s)
                                   : __ldcv(a.pF_hi + p * a.pstride_hi + (s - a.n_if_lo));
        F = s < a.n_if_lo ? rx + own : own + rx;  // lower rank's part first
      } else {
        F = (s < a.n_if_lo) ? (a.Frx[s] + F) : (F + a.Frx[s]);  // lower rank's part first
      }
    }
    if (kind == 2) return a.sp_dirT[s];                                      // Dirichlet held (Eq. 3)
    if (kind == 1) Q += face_load(a, s, T);
  }
  R Tn = explicit_update<R, TDK>(a, T, F, Q, coef);
  flag_unstable(a, Tn);
  return Tn;
}

// One face-BC record's term, accumulated exactly as face_load's loop body does
template <typename R>
__device__ __forceinline__ void face_term_acc(R &Q, int kind, R cf, R Ti, R T) {
  if (kind == 1) {
    Q += cf;
  } else if (kind == 2) {
    Q -= cf * (T - Ti);
  } else {
    const R Ta = T + R(273.15), Tb = Ti + R(273.15);
    Q -= cf * ((T - Ti) * (Ta + Tb) * (Ta * Ta + Tb * Tb));
  }
}

// node_update of the G consecutive nodes n..n+G-1 of one 16-byte access, with the
// per-node operands that live outside the 16-byte planes -- interface loads (own and
// received / the neighbour's), face-record ranges, first face records, Dirichlet
// values -- loaded for all G nodes together: one round trip per kind of operand
// instead of one (interface, Dirichlet) or two (face records) per node.  Same
// arithmetic, in the same order, as node_update.
template <typename R, int TDK>
__device__ __forceinline__ void node_update_group_special(const StepArgs<R> &a, int64_t n, const Vec16<R> &T4,
                                                       const Vec16<R> &F4, const Vec16<R> &C4, const Vec16<R> &Q4,
                                                       bool hasQ, unsigned K, long long step, Vec16<R> &Tn) {
  constexpr int G = Vec16<R>::n;
  R F[G], Q[G];
#pragma unroll
  for (int q = 0; q < G; ++q) { F[q] = F4.v[q]; Q[q] = hasQ ? Q4.v[q] : R(0); }
  {
    const int s0 = (int)(n - a.N_int);
    if (s0 < a.n_if) {
      if (a.Fif) {
        // PEER: own parity buffer + the neighbour's (see node_update)
        const int64_t p = step & 1;
        R own[G], rx[G];
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int s = s0 + q;
          own[q] = R(0); rx[q] = R(0);
          if (s < a.n_if) {
            own[q] = __ldcg(a.Fif + p * a.n_if + s);
            rx[q] = s < a.n_if_lo ? __ldcv(a.pF_lo + p * a.pstride_lo + s)
                                  : __ldcv(a.pF_hi + p * a.pstride_hi + (s - a.n_if_lo));
          }
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int s = s0 + q;
          if (s < a.n_if) {
            a.Fif[(p ^ 1) * a.n_if + s] = R(0);
            F[q] = s < a.n_if_lo ? rx[q] + own[q] : own[q] + rx[q];  // lower rank's part first
          }
        }
      } else {
        R rx[G];
#pragma unroll
        for (int q = 0; q < G; ++q) rx[q] = s0 + q < a.n_if ? a.Frx[s0 + q] : R(0);
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int s = s0 + q;
          if (s < a.n_if) F[q] = s < a.n_if_lo ? (rx[q] + F[q]) : (F[q] + rx[q]);
        }
      }
    }
    bool any_face = false, any_dir = false;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      any_face |= ((K >> (8 * q)) & 0xffu) == 1u;
      any_dir |= ((K >> (8 * q)) & 0xffu) == 2u;
    }
    if (any_face) {
      int j[G + 1];
#pragma unroll
      for (int q = 0; q <= G; ++q) j[q] = a.bc_ptr[s0 + q];
      int ek[G];
      R cf[G], ti[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        ek[q] = 0; cf[q] = R(0); ti[q] = R(0);
        if (((K >> (8 * q)) & 0xffu) == 1u && j[q] < j[q + 1]) {
          ek[q] = a.bc_ekind[j[q]]; cf[q] = a.bc_coef[j[q]]; ti[q] = a.bc_tinf[j[q]];
        }
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (((K >> (8 * q)) & 0xffu) == 1u) {
          FED_DCHECK(a, j[q] >= 0 && j[q] <= j[q + 1], 5);
          R Qf = R(0);
          if (j[q] < j[q + 1]) face_term_acc(Qf, ek[q], cf[q], ti[q], T4.v[q]);
          for (int jj = j[q] + 1; jj < j[q + 1]; ++jj)
            face_term_acc(Qf, (int)a.bc_ekind[jj], a.bc_coef[jj], a.bc_tinf[jj], T4.v[q]);
          Q[q] += Qf;
        }
      }
    }
    R dT[G];
    if (any_dir) {
#pragma unroll
      for (int q = 0; q < G; ++q) dT[q] = ((K >> (8 * q)) & 0xffu) == 2u ? a.sp_dirT[s0 + q] : R(0);
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if (any_dir && ((K >> (8 * q)) & 0xffu) == 2u) {
        Tn.v[q] = dT[q];                                              // Dirichlet held (Eq. 3)
      } else {
        Tn.v[q] = explicit_update<R, TDK>(a, T4.v[q], F[q], Q[q], C4.v[q]);
        flag_unstable(a, Tn.v[q]);
      }
    }
  }
}

template <typename R, int TDK>
__device__ __forceinline__ void node_update_group_plain(const StepArgs<R> &a, const Vec16<R> &T4, const Vec16<R> &F4,
                                                        const Vec16<R> &C4, const Vec16<R> &Q4, bool hasQ, Vec16<R> &Tn) {
#pragma unroll
  for (int q = 0; q < Vec16<R>::n; ++q) {
    Tn.v[q] = explicit_update<R, TDK>(a, T4.v[q], F4.v[q], hasQ ? Q4.v[q] : R(0), C4.v[q]);
    flag_unstable(a, Tn.v[q]);
  }
}

// Nodal update of nodes [start, N_loc): NodeShape<R>::vec consecutive nodes per
// thread, every operand loaded up front with 16-byte vector loads (start is
// 8-aligned).  The kernel is latency-bound (one batch of loads per thread), so the
// shape is chosen for residency (same-box A/B on cfg5): fp32 8 nodes x 128 threads,
// <= 51 registers, 10 CTAs/SM (80.5 -> 77 us against 256 threads; 64 registers and
// 4 CTAs/SM had cost 164 vs 120 us cold); fp64 4 nodes x 256 threads, 5 CTAs/SM
// (176 -> 137 us against 8 nodes x 256 at 3 CTAs/SM).
template <typename R>
struct NodeShape {
  static constexpr int vec = sizeof(R) == 8 ? 4 : 8;
  static constexpr int threads = sizeof(R) == 8 ? 256 : 128;
  static constexpr int min_ctas = sizeof(R) == 8 ? 5 : 10;
  static constexpr int64_t per_block = (int64_t)vec * threads;
};

// The PEER transport (a.Fif set) is a run-time branch on purpose: a compile-time
// single-rank instantiation without it measured 3x slower on cfg5 (0.191 vs 0.069
// ms, same box, same loads and DRAM bytes; long-scoreboard stalls 47.6 vs 9.5 per
// issue) -- profiles/r2_node_kernel_regression.txt
template <typename R, int TDK>
__global__ void __launch_bounds__(NodeShape<R>::threads, NodeShape<R>::min_ctas) node_kernel(StepArgs<R> a, int64_t start) {
  constexpr int kThr = NodeShape<R>::threads, G = Vec16<R>::n, H = NodeShape<R>::vec / G;
  // the block owns [b0, b1); access h of thread t covers nodes b0 + h G kThr + G t ..+G-1,
  // so each warp instruction reads or writes 512 contiguous bytes
  const int64_t b0 = start + NodeShape<R>::per_block * blockIdx.x, b1 = b0 + NodeShape<R>::per_block;
  FED_DCHECK(a, start >= 0 && start <= a.N_loc && (start & 7) == 0, 7);
  pdl_trigger();
  long long step = 0;
  float dmax = 0.f;
  if (b1 <= a.N_loc) {
    Vec16<R> T4[H], F4[H], C4[H], Q4[H], Z;
    unsigned K[H];
    // every operand in one batch of loads, after the dependency wait of a
    // programmatic launch (splitting off the static operands before the wait made a
    // second round trip: 0.068 -> 0.288 ms on cfg5, same box)
    pdl_wait();
    if (a.Fif) {  // PEER: blocks holding interface nodes wait for the neighbours' loads
      step = *a.step_base + a.k_off;
      if (b0 < a.N_int + a.n_if && b1 > a.N_int) {
        if (threadIdx.x == 0) wait_peers(a, (unsigned long long)step + 1ull);
        __syncthreads();
      }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int64_t n = b0 + (int64_t)h * G * kThr + G * threadIdx.x;
      if constexpr (sizeof(R) == 4 && (FED_L2_KEEP & 6)) {
        const uint64_t pk = l2_keep_policy();
        float4 x;
        if (FED_L2_KEEP & 2) { x = ld_keep4((const float *)(a.T + n), pk); T4[h].v[0] = x.x; T4[h].v[1] = x.y; T4[h].v[2] = x.z; T4[h].v[3] = x.w; }
        else T4[h].load(a.T + n);
        if (FED_L2_KEEP & 4) { x = ld_keep4((const float *)(a.F + n), pk); F4[h].v[0] = x.x; F4[h].v[1] = x.y; F4[h].v[2] = x.z; F4[h].v[3] = x.w; }
        else F4[h].load(a.F + n);
      } else {
        T4[h].load(a.T + n);
        F4[h].load(a.F + n);
      }
      C4[h].load(a.coef + n);
      if (a.Qvol) Q4[h].load(a.Qvol + n);
      K[h] = 0u;
      if (n >= a.N_int) {  // groups of G never straddle N_int (8-aligned)
        const uint8_t *kp = a.sp_kind + (n - a.N_int);
        K[h] = G == 4 ? *reinterpret_cast<const unsigned *>(kp) : *reinterpret_cast<const uint16_t *>(kp);
      }
    }
#if FED_NODE_GROUP
    bool sp = false;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int64_t n = b0 + (int64_t)h * G * kThr + G * threadIdx.x;
      sp |= n >= a.N_int && (K[h] != 0u || n - a.N_int < a.n_if);
    }
    const bool special_warp = __any_sync(0xffffffffu, sp);
#endif
#pragma unroll
    for (int q = 0; q < G; ++q) Z.v[q] = R(0);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      if constexpr (sizeof(R) == 4 && (FED_L2_KEEP & 4))
        st_keep4((float *)(a.F + b0 + (int64_t)h * G * kThr + G * threadIdx.x), make_float4(0.f, 0.f, 0.f, 0.f), l2_keep_policy());
      else
        Z.store(a.F + b0 + (int64_t)h * G * kThr + G * threadIdx.x);
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int64_t n = b0 + (int64_t)h * G * kThr + G * threadIdx.x;
      Vec16<R> Tn;
#if FED_NODE_GROUP
      // warps holding a special node (interface, face BC, Dirichlet) take the grouped
      // special path; the others (most of the launch) the plain one, so the special
      // path's extra live values do not cost the plain warps registers or spills
      if (special_warp && n >= a.N_int && (K[h] != 0u || n - a.N_int < a.n_if))
        node_update_group_special<R, TDK>(a, n, T4[h], F4[h], C4[h], Q4[h], a.Qvol != nullptr, K[h], step, Tn);
      else
        node_update_group_plain<R, TDK>(a, T4[h], F4[h], C4[h], Q4[h], a.Qvol != nullptr, Tn);
#pragma unroll
      for (int q = 0; q < G; ++q) dmax = fmaxf(dmax, (float)rabs(Tn.v[q] - T4[h].v[q]));
#else
#pragma unroll
      for (int q = 0; q < G; ++q) {
        Tn.v[q] = node_update<R, TDK>(a, n + q, T4[h].v[q], F4[h].v[q], C4[h].v[q],
                                     a.Qvol ? Q4[h].v[q] : R(0), (int)((K[h] >> (8 * q)) & 0xffu), step);
        dmax = fmaxf(dmax, (float)rabs(Tn.v[q] - T4[h].v[q]));
      }
#endif
      if constexpr (sizeof(R) == 4 && (FED_L2_KEEP & 2))
        st_keep4((float *)(a.T + n), make_float4(Tn.v[0], Tn.v[1], Tn.v[2], Tn.v[3]), l2_keep_policy());
      else
        Tn.store(a.T + n);
    }
  } else {
    // the ragged last block: one node per thread and access
    pdl_wait();
    if (a.Fif) {
      step = *a.step_base + a.k_off;
      if (b0 < a.N_int + a.n_if) {
        if (threadIdx.x == 0) wait_peers(a, (unsigned long long)step + 1ull);
        __syncthreads();
      }
    }
    for (int64_t n = b0 + threadIdx.x; n < a.N_loc; n += kThr) {
      R F = a.F[n];
      a.F[n] = R(0);
      int kind = n >= a.N_int ? a.sp_kind[n - a.N_int] : 0;
      const R T0 = a.T[n];
      a.T[n] = node_update<R, TDK>(a, n, T0, F, a.coef[n], a.Qvol ? a.Qvol[n] : R(0), kind, step);
      dmax = fmaxf(dmax, (float)rabs(a.T[n] - T0));
    }
  }
  if (a.dTmax) warp_max_to(a.dTmax, dmax);
}

__global__ void advance_step_kernel(long long *step_base, long long n) { *step_base += n; }

// ---------------------------------------------------------------- resident mode
// Small meshes (every chunk can own a CTA): ONE cooperative launch runs all n steps
// of a fed_step call.  A CTA keeps its chunk's element records in registers and its
// nodes' T, coef, Q in shared memory for the whole run; interior nodes never touch
// HBM between the first load and the final write-back.  Steps are ordered by
// dataflow, not by kernel boundaries: chunk c starts step g once every chunk
// sharing a node with it has published done = g (it finished step g-1).  The
// shared nodes' update (Eq. 16, face loads, Dirichlet) is then recomputed by every
// chunk touching the node from the complete partial-load sum F^{g-1}; all touchers
// compute the same value, the owner (lowest touching chunk) also stores it.  Loads
// of step g go to F[g % 3]: the touchers of a node are pairwise neighbours, so they
// are at most one step apart; F[(g+1) % 3] (last read at step g-1, next written at
// step g+1) is cleared by the owner during step g.  A finalize pass (node_kernel)
// applies the last step's shared-node update after the launch.
template <typename R>
struct ResArgs {
  int n_steps;
  long long g0;                      // global index of the call's first step
  const int32_t *nbr_ptr, *nbr;      // chunk adjacency (CSR)
  const uint8_t *sp_own;             // parallel to sp_list: 1 = this chunk owns the node
  unsigned long long *done;          // [n_chunks] last completed global step + 1
  R *F3;                             // [3][f3_stride] partial-load buffers by step % 3
  int64_t f3_stride;                 // N_sp rounded up to 8 (16-byte aligned buffers)
  unsigned int *err;                 // dependency wait timed out (bit 0)
  unsigned int *abort;               // set on error: every waiter leaves
};

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int kResidentCtasPerSm32 = 4, kResidentCtasPerSm64 = 2;  // register budget of the loop state

// hex8: colour phases (<= 8 colours of <= kThreads elements, plain RMW); tet4: one
// phase of compare-and-swap adds over <= 8 elements per thread (chunks <= 1024)
template <typename R, int TDK, int LS, int NPE>
__global__ void __launch_bounds__(kThreads, sizeof(R) == 4 ? kResidentCtasPerSm32 : kResidentCtasPerSm64)
resident_kernel(StepArgs<R> a, ResArgs<R> r) {
  using CR = ConnRec<NPE>;
  using CT = typename CR::T;
  const CT *gconn = reinterpret_cast<const CT *>(a.conn16);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  R *sT = reinterpret_cast<R *>(smem + 16);
  R *sF = sT + (LS > 0 ? LS : a.max_local);
  R *sCoef = sF + (LS > 0 ? LS : a.max_local);
  R *sQ = sCoef + a.max_local;
  int *sSp = reinterpret_cast<int *>(sQ + a.max_local);
  int *sCol = sSp + a.max_local;
  uint8_t *sFlag = reinterpret_cast<uint8_t *>(sCol + kMaxColorsDev + 1);  // kind | own << 4
  R *sPhi = TDK == 2 ? reinterpret_cast<R *>((reinterpret_cast<uintptr_t>(sFlag + a.max_local) + 15) &
                                             ~uintptr_t(15))
                     : nullptr;
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  const int4 *h4 = reinterpret_cast<const int4 *>(a.chunk_hdr) + (size_t)c * 4;
  const int4 h0 = __ldg(h4), h1 = __ldg(h4 + 1), h2 = __ldg(h4 + 2), h3 = __ldg(h4 + 3);
  const int elem_off = h0.x, n_elem = h0.y, int_start = h0.w, n_int = h1.x, sp_off = h1.y, n_sp = h1.z,
            n_col = h1.w;
  const int n_int_pad = (n_int + 7) & ~7;
  const int cof[9] = {0, h2.x, h2.y, h2.z, h2.w, h3.x, h3.y, h3.z, h3.w};
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    fence_proxy_async();
    const uint32_t nbytes = (uint32_t)(n_int_pad * sizeof(R));
    const uint32_t sbytes = (uint32_t)(((n_sp + 3) & ~3) * 4);
    mbar_expect_tx(bar, (uint32_t)(a.Qvol ? 3 : 2) * nbytes + sbytes);
    if (nbytes) {
      bulk_g2s(sT, a.T + int_start, nbytes, bar);
      bulk_g2s(sCoef, a.coef + int_start, nbytes, bar);
      if (a.Qvol) bulk_g2s(sQ, a.Qvol + int_start, nbytes, bar);
    }
    if (sbytes) bulk_g2s(sSp, a.sp_list + sp_off, sbytes, bar);
  }
  // element records of the run, in registers (<= 8 colours of <= kThreads elements)
  CT cc[8];
  R pp[8][6];
  unsigned vmask = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int e = NPE == 8 ? cof[k] + tid : k * kThreads + tid;
    if (NPE == 8 ? (k < n_col && e < cof[k + 1]) : e < n_elem) {
      vmask |= 1u << k;
      cc[k] = __ldg(gconn + elem_off + e);
#pragma unroll
      for (int q = 0; q < 6; ++q) pp[k][q] = __ldg(a.P + (size_t)q * a.n_slots + elem_off + e);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // shared nodes: T, coef, Q, kind and ownership into shared memory
  for (int l = tid; l < n_sp; l += kThreads) {
    const int s = sSp[l];
    R t = R(0), cf = R(0), q = R(0);
    uint8_t fl = 0xff;
    if (s >= 0) {
      t = a.T[a.N_int + s];
      cf = a.coef[a.N_int + s];
      if (a.Qvol) q = a.Qvol[a.N_int + s];
      fl = (uint8_t)(a.sp_kind[s] | (r.sp_own[sp_off + l] << 4));
    }
    sT[n_int_pad + l] = t;
    sCoef[n_int_pad + l] = cf;
    sQ[n_int_pad + l] = q;
    sFlag[l] = fl;
  }
  __syncthreads();
  __shared__ unsigned int sAbort;
  for (int j = 0; j < r.n_steps; ++j) {
    const long long g = r.g0 + j;
    if (j > 0) {
      // wait until every neighbouring chunk finished step g-1 (bounded by a.wait_ns)
      const int q0 = __ldg(r.nbr_ptr + c), q1 = __ldg(r.nbr_ptr + c + 1);
      for (int q = q0 + tid; q < q1; q += kThreads) {
        const unsigned long long *d = r.done + __ldg(r.nbr + q);
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_gpu(d) < (unsigned long long)g) {
          if (*(volatile unsigned int *)r.abort) break;
          if (globaltimer_ns() - t0 > a.wait_ns) {
            atomicOr(r.err, 1u);
            atomicExch(r.abort, 1u);
            break;
          }
          __nanosleep(64);
        }
      }
      if (tid == 0) sAbort = *(volatile unsigned int *)r.abort;
      __syncthreads();
      if (sAbort) return;  // uniform across the CTA
      // shared-node update to step g from the complete loads of step g-1
      const R *Fp = r.F3 + (size_t)((g - 1) % 3) * r.f3_stride;
      R *Fn = r.F3 + (size_t)((g + 1) % 3) * r.f3_stride;
      for (int l = tid; l < n_sp; l += kThreads) {
        const int s = sSp[l];
        if (s < 0) continue;
        const uint8_t fl = sFlag[l];
        const R T0 = sT[n_int_pad + l];
        R Tn;
        if ((fl & 15) == 2) {
          Tn = a.sp_dirT[s];  // Dirichlet held (Eq. 3)
        } else {
          R Q = sQ[n_int_pad + l];
          if ((fl & 15) == 1) Q += face_load(a, s, T0);
          Tn = explicit_update<R, TDK>(a, T0, __ldcg(Fp + s), Q, sCoef[n_int_pad + l]);
          if (!(rabs(Tn) <= a.T_abort)) atomicMin(a.fail_step, (unsigned long long)(*a.step_base + j - 1));
        }
        sT[n_int_pad + l] = Tn;
        if (fl >> 4) {
          a.T[a.N_int + s] = Tn;
          Fn[s] = R(0);
        }
      }
    }
    for (int l = tid; l < n_int_pad + n_sp; l += kThreads) sF[l] = R(0);
    __syncthreads();
    if constexpr (TDK == 2) {
      phi_pass<R>(a, sT, sPhi, n_int_pad + n_sp, tid, nullptr);
      __syncthreads();
    }
    if constexpr (NPE == 8) {
      // colour phases (plain shared-memory read-modify-write, one barrier per colour)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < n_col) {
          if (vmask & (1u << k)) {
            int idx[8];
            CR::unpack(cc[k], idx);
            R t[8], f[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) t[q] = sm_at(sT, idx[q]);
            elem_forces<R, TDK, 8>(a, t, idx, sPhi, pp[k], f);
#pragma unroll
            for (int q = 0; q < 8; ++q) sm_at(sF, idx[q]) += f[q];
          }
          __syncthreads();
        }
      }
    } else {
      // one phase, compare-and-swap adds (tets need more than 8 colours per chunk)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (vmask & (1u << k)) {
          int idx[NPE];
          CR::unpack(cc[k], idx);
          R t[NPE], f[NPE];
#pragma unroll
          for (int q = 0; q < NPE; ++q) t[q] = sm_at(sT, idx[q]);
          elem_forces<R, TDK, NPE>(a, t, idx, sPhi, pp[k], f);
#pragma unroll
          for (int q = 0; q < NPE; ++q) smem_add(&sm_at(sF, idx[q]), f[q]);
        }
      }
      __syncthreads();
    }
    // interior nodes: Eq. 16 in shared memory; shared nodes: partial loads to F[g % 3]
    for (int l = tid; l < n_int; l += kThreads) {
      const R Tn = explicit_update<R, TDK>(a, sT[l], sF[l], a.Qvol ? sQ[l] : R(0), sCoef[l]);
      if (!(rabs(Tn) <= a.T_abort)) atomicMin(a.fail_step, (unsigned long long)(*a.step_base + j));
      sT[l] = Tn;
    }
    R *Fc = r.F3 + (size_t)(g % 3) * r.f3_stride;
    for (int l = tid; l < n_sp; l += kThreads) {
      const int s = sSp[l];
      if (s >= 0) red_add(Fc + s, sF[n_int_pad + l]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_gpu(r.done + c, (unsigned long long)g + 1ull);
  }
  // interior temperatures back to HBM (shared nodes: owners stored them; the last
  // step's shared-node update is the finalize pass)
  for (int l = tid; l < n_int; l += kThreads) a.T[int_start + l] = sT[l];
}


// ---------------------------------------------------------------- utilities
// caller-order output: out[node_global[i]] = T[i] (alignment padding skipped)
template <typename R>
__global__ void to_caller_kernel(const R *T, const int32_t *node_global, const uint8_t *owned, double *out,
                                 int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && owned[i]) out[node_global[i]] = (double)T[i];
}
// caller-order input: T[i] = in[node_global[i]]; Dirichlet values re-applied by the caller
template <typename R>
__global__ void from_caller_kernel(const double *in, const int32_t *node_global, R *T, int64_t n,
                                   unsigned int *bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int32_t g = node_global[i];
    double v = g >= 0 ? in[g] : 0.0;
    if (!isfinite(v)) atomicOr(bad, 1u);
    T[i] = (R)v;
  }
}
// multi-rank readout: this rank's owned nodes, packed in its caller-id order
template <typename R>
__global__ void pack_owned_kernel(const R *T, const int32_t *pack, double *send, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) send[i] = (double)T[pack[i]];
}
// all ranks' packed slices (rank r at recv + r * stride) to caller order
struct RankOffsets { int64_t off[65]; int nranks; };
__global__ void unpack_gathered_kernel(const double *recv, const int32_t *ids, RankOffsets ro, int64_t stride,
                                       double *out, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int r = 0;
  while (r + 1 < ro.nranks && j >= ro.off[r + 1]) ++r;
  out[ids[j]] = recv[(int64_t)r * stride + (j - ro.off[r])];
}
template <typename R>
__global__ void apply_dirichlet_kernel(R *T, const uint8_t *sp_kind, const R *sp_dirT, int64_t N_int, int64_t n_sp) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_sp && sp_kind[s] == 2) T[N_int + s] = sp_dirT[s];
}


}  // namespace fed
