// fed_api.cu -- C ABI of libfed.so (include/fed.h): context, device memory,
// step launch schedule (CUDA graphs, streams), NCCL interface exchange.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fed.h"
#include "fed_kernels.cuh"
#include "fed_plan.h"

// ----------------------------------------------------------------- NCCL (dlopen)
// Minimal NCCL declarations (ABI of libnccl.so.2); loaded lazily so that the
// library has no link-time dependency on NCCL for single-GPU use.
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclUint8_ = 1, ncclUint32_ = 3, ncclFloat32_ = 7, ncclFloat64_ = 8, ncclSum_ = 0, ncclMax_ = 2 };

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
      api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
               api.GroupEnd && api.AllReduce && api.AllGather && api.GetErrorString;
    }
  }
  return api;
}

// ----------------------------------------------------------------- errors
static thread_local std::string g_err;
static fed_status fail(fed_status st, const std::string &msg) {
  g_err = msg;
  return st;
}
#define CU(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) return fail(FED_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define NC(x)                                                                                          \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != 0) return fail(FED_ERR_NCCL, std::string(#x ": ") + nccl().GetErrorString(r_));         \
  } while (0)

// ----------------------------------------------------------------- context
struct fed_ctx {
  fed::Plan pl;
  bool dry = true;
  int device = -1;
  cudaStream_t stream = nullptr, comm = nullptr;
  bool own_stream = false;
  size_t bytes = 0;
  struct Alloc { void *p; size_t bytes; bool hooked; };
  std::vector<Alloc> allocs;
  // device-memory hook (fed_options.dev_alloc / dev_free / alloc_ctx)
  void *(*hook_alloc)(size_t, int32_t, void *) = nullptr;
  void (*hook_free)(void *, size_t, int32_t, void *) = nullptr;
  void *hook_ctx = nullptr;
  unsigned long long wait_ns = 10000000000ull;  // device-side wait bound (fed_options.wait_timeout_s)
  bool skip_barrier = false;                     // create failed across ranks: no barrier in destroy
  bool free_run = false;                         // fed_debug_time_rank: PEER waits skipped
  bool pdl = true;                               // step kernels launched as programmatic dependents
  float l2_stream = 1.0f;                        // L2 evict_first fraction for streamed-once loads
  bool spoiled = false;                          // field undefined after fed_debug_time_rank
  unsigned int *d_scratch = nullptr;             // [4] words for NCCL barriers / rendezvous
  unsigned int *d_check = nullptr;               // checked build: failed device checks
  // multi-rank readout (fed_get_temperature): own packed slice, all ranks' slices
  int32_t *d_pack = nullptr, *d_gather_ids = nullptr;
  double *d_gsend = nullptr, *d_grecv = nullptr;
  // typed device buffers (R = float or double, stored as void*)
  void *T = nullptr, *F = nullptr, *coef = nullptr, *Qvol = nullptr, *P = nullptr, *Frx = nullptr;
  void *bc_coef = nullptr, *bc_tinf = nullptr, *sp_dirT = nullptr;
  void *kt = nullptr, *ct = nullptr;  // NEXT-2 tables [T | v | slope]
  int8_t *bc_ekind = nullptr;
  uint4 *conn16 = nullptr;
  uint4 *rec12 = nullptr;   // fp32 streaming hex: 12-bit packed connectivity + P_xx per slot
  int4 *conn32 = nullptr;
  int32_t *cp_list = nullptr, *g_ptr = nullptr, *g_list = nullptr;  // scatter baselines
  void *vbuf = nullptr;                                              // GATHER: v[3][n_slots]
  int32_t *chunk_hdr = nullptr, *color_off = nullptr, *sp_list = nullptr, *bc_ptr = nullptr,
          *node_global = nullptr;
  uint8_t *sp_kind = nullptr, *owned = nullptr;
  long long *d_step = nullptr;
  unsigned int *d_dTmax = nullptr;   // steady-state monitor (NEXT-4)
  bool monitor = false;
  unsigned long long *d_fail = nullptr;
  double *d_caller = nullptr;      // [N_glob] caller-order fp64 staging (lazy)
  unsigned int *d_bad = nullptr;
  // schedule
  int64_t step = 0;
  int graph_steps = 0;
  cudaGraphExec_t graph = nullptr;
  int graph_len = 0;
  cudaEvent_t ev_if = nullptr, ev_comm = nullptr;
  // timing
  bool timing = false;
  fed_timing tacc{};
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> trec;               // pending (kind, start, stop) pairs
  std::vector<cudaEvent_t> tpool;      // reusable events
  // interface exchange (nranks > 1)
  int transport = FED_TRANSPORT_NCCL;
  void *peer_blk = nullptr;            // PEER: [sig u64 x2 | pad to 256 B | Fif R x 2 n_if]
  void *Fif = nullptr;
  unsigned long long *sig = nullptr;
  unsigned int *if_done = nullptr, *peer_err = nullptr;
  const void *pF_lo = nullptr, *pF_hi = nullptr;
  int64_t pstride_lo = 0, pstride_hi = 0;
  unsigned long long *psig_lo = nullptr, *psig_hi = nullptr;
  std::vector<void *> ipc_opened;      // neighbour blocks mapped with cudaIpcOpenMemHandle
  // resident mode (fed_options.resident)
  bool resident = false;
  size_t res_smem = 0;
  int32_t *nbr_ptr = nullptr, *nbr = nullptr;
  uint8_t *sp_own = nullptr;
  unsigned long long *d_done = nullptr;
  void *F3 = nullptr;
  unsigned int *d_res_err = nullptr;   // [0] timeout bits, [1] abort
  // local rank group (fed_options.local_ranks > 1): this ctx owns the slabs
  std::vector<fed_ctx *> sub;
  bool is_sub = false;
  // nccl
  ncclComm_t ncomm = nullptr;
  int64_t launches_per_step = 0;
  int64_t launches_total = 0;     // kernels of this library launched by fed_step
  int graph_kernels = 0;          // kernels per graph replay
};

namespace {

// Device allocation owned by the context: the caller's hook when one is set
// (fed_options.dev_alloc), cudaMalloc otherwise or when `cuda_only` (memory
// shared by CUDA IPC must be an allocation of its own).  Sizes are rounded up to
// 256 bytes so every buffer keeps cudaMalloc's alignment under any hook.
template <typename T>
fed_status dalloc(fed_ctx *c, T **p, size_t count, bool cuda_only = false) {
  *p = nullptr;
  if (count == 0) count = 1;
  const size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
  void *q = nullptr;
  const bool hooked = c->hook_alloc && !cuda_only;
  if (hooked) {
    q = c->hook_alloc(bytes, c->device, c->hook_ctx);
    if (!q) return fail(FED_ERR_NOMEM, "dev_alloc hook returned NULL for " + std::to_string(bytes) + " bytes");
    if (((uintptr_t)q & 255) != 0) {
      c->hook_free(q, bytes, c->device, c->hook_ctx);
      return fail(FED_ERR_NOMEM, "dev_alloc hook returned a pointer that is not 256-byte aligned");
    }
  } else {
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) return fail(FED_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  c->allocs.push_back({q, bytes, hooked});
  c->bytes += bytes;
  *p = static_cast<T *>(q);
  return FED_OK;
}

template <typename T>
fed_status upload(fed_ctx *c, T **p, const std::vector<T> &v) {
  fed_status st = dalloc(c, p, v.size());
  if (st != FED_OK) return st;
  if (!v.empty()) CU(cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return FED_OK;
}

template <typename R>
fed_status upload_real(fed_ctx *c, void **p, const std::vector<double> &v) {
  std::vector<R> h(v.begin(), v.end());
  R *q = nullptr;
  fed_status st = upload(c, &q, h);
  *p = q;
  return st;
}

// row stride of the [3][.] shared-node load buffers (16-byte aligned rows)
int64_t f3_stride(const fed::Plan &pl) { return std::max<int64_t>(8, (pl.N_sp + 7) & ~(int64_t)7); }

template <typename R>
fed::StepArgs<R> make_args(fed_ctx *c) {
  const fed::Plan &pl = c->pl;
  fed::StepArgs<R> a;
  a.T = (R *)c->T;
  a.F = (R *)c->F;
  a.coef = (const R *)c->coef;
  a.Qvol = (const R *)c->Qvol;
  a.conn16 = c->conn16;
  a.rec12 = c->rec12;
  a.conn32 = c->conn32;
  a.P = (const R *)c->P;
  a.n_slots = pl.n_slots;
  a.chunk_hdr = c->chunk_hdr;
  a.color_off = c->color_off;
  a.sp_list = c->sp_list;
  a.bc_ptr = c->bc_ptr;
  a.bc_coef = (const R *)c->bc_coef;
  a.bc_tinf = (const R *)c->bc_tinf;
  a.bc_ekind = c->bc_ekind;
  a.sp_kind = c->sp_kind;
  a.sp_dirT = (const R *)c->sp_dirT;
  a.Frx = (const R *)c->Frx;
  a.n_if = pl.n_if;
  a.n_if_lo = pl.n_if_lo;
  a.N_int = pl.N_int;
  a.N_loc = pl.N_loc;
  a.N_sp = pl.N_sp;
  a.beta_k = (R)pl.beta_k;
  a.beta_c = (R)pl.beta_c;
  a.T_abort = (R)pl.T_abort;
  a.c0 = (R)pl.c0;
  a.kl_lo = (R)pl.kl[0]; a.kl_hi = (R)pl.kl[1]; a.kl_v0 = (R)pl.kl[2]; a.kl_s = (R)pl.kl[3]; a.kl_T0 = (R)pl.kl[4];
  a.cl_lo = (R)pl.cl[0]; a.cl_hi = (R)pl.cl[1]; a.cl_v0 = (R)pl.cl[2]; a.cl_s = (R)pl.cl[3]; a.cl_T0 = (R)pl.cl[4];
  a.kt = (const R *)c->kt;
  a.ct = (const R *)c->ct;
  a.n_kt = (int)pl.k_tab_T.size();
  a.n_ct = (int)pl.c_tab_T.size();
  a.max_local = pl.max_local_used;
  a.max_int = pl.max_int_used;
  a.max_sp = pl.max_sp_used;
  a.chunk_cap = pl.chunk_elems;
  a.step_base = c->d_step;
  a.k_off = 0;
  a.fail_step = c->d_fail;
  a.dTmax = c->monitor ? c->d_dTmax : nullptr;
  a.Fif = (R *)c->Fif;
  a.pF_lo = (const R *)c->pF_lo;
  a.pF_hi = (const R *)c->pF_hi;
  a.pstride_lo = c->pstride_lo;
  a.pstride_hi = c->pstride_hi;
  a.psig_lo = c->psig_lo;
  a.psig_hi = c->psig_hi;
  a.sig = c->sig;
  a.if_done = nullptr;  // set for the launch holding the interface chunks only
  a.n_sig_ctas = 0;
  a.peer_err = c->peer_err;
  a.wait_ns = c->wait_ns;
  a.free_run = c->free_run ? 1 : 0;
  a.check_err = c->d_check;
  a.l2_stream = c->l2_stream;
  return a;
}

// shared memory of the streaming element kernel (compact layout, runtime stride)
size_t stream_smem(const fed::Plan &pl) {
  const bool staged = pl.scatter == FED_SCATTER_CHUNK || pl.scatter == FED_SCATTER_CHUNK_CAS;
  const bool phi = pl.td == 2;
  return pl.precision == 32
             ? fed::stream_smem_bytes<float>(pl.chunk_elems, pl.max_local_used, pl.max_int_used, pl.max_sp_used, staged, phi)
             : fed::stream_smem_bytes<double>(pl.chunk_elems, pl.max_local_used, pl.max_int_used, pl.max_sp_used, staged, phi);
}

// The dynamic shared-memory limit is a per-function attribute of each device
// (set on the current device): only ever raise it, so contexts with smaller
// chunks keep working next to larger ones; the cache is keyed by (device, kernel)
template <typename K>
fed_status raise_smem_limit(K *fn, int smem, bool max_carveout = false) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, int> applied;
  int dev = -1;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int &cur = applied[{dev, (const void *)fn}];
  if (smem <= cur) return FED_OK;
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // tabulated k/c: 7 CTAs of ~29 KB need the 228 KB carveout (the default choice stops
  // at 6); the others keep the driver's choice, which leaves more L1 for loads in flight
  if (max_carveout)
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  cur = smem;
  return FED_OK;
}

template <typename R, int TDK>
fed_status set_kernel_attrs(fed_ctx *c) {
  int smem = (int)stream_smem(c->pl);
  fed_status st = FED_OK;
  if (c->pl.npe == 8) {
    if ((st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 0, 8>, smem)) != FED_OK) return st;
    if ((st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 1, 8>, smem)) != FED_OK) return st;
    if ((st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 2, 8>, smem)) != FED_OK) return st;
    st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 3, 8>, smem, TDK == 2 && sizeof(R) == 4 && FED_TDK2_CTAS > 6);
  } else {
    if ((st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 2, 4>, smem)) != FED_OK) return st;
    st = raise_smem_limit(fed::element_chunk_kernel<R, TDK, 3, 4>, smem);
  }
  return st;
}

// Launch of a step kernel, as a programmatic dependent of the previous kernel in
// the stream when c->pdl (cudaLaunchAttributeProgrammaticStreamSerialization; the
// kernels order their dependent accesses after griddepcontrol.wait, fed_kernels.cuh)
template <typename... KArgs, typename... Args>
cudaError_t launch_step_kernel(const fed_ctx *c, void (*kernel)(KArgs...), unsigned grid, unsigned block,
                               size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename R, int TDK>
void launch_chunks(fed_ctx *c, const fed::StepArgs<R> &a, unsigned n, int base, size_t smem, cudaStream_t s) {
  const int sc = c->pl.scatter;
  void (*k)(fed::StepArgs<R>, int);
  if (c->pl.npe == 4)
    k = sc == FED_SCATTER_CHUNK_REGC ? fed::element_chunk_kernel<R, TDK, 3, 4> : fed::element_chunk_kernel<R, TDK, 2, 4>;
  else if (sc == FED_SCATTER_CHUNK_CAS)
    k = fed::element_chunk_kernel<R, TDK, 1, 8>;
  else if (sc == FED_SCATTER_CHUNK_REG)
    k = fed::element_chunk_kernel<R, TDK, 2, 8>;
  else if (sc == FED_SCATTER_CHUNK_REGC)
    k = fed::element_chunk_kernel<R, TDK, 3, 8>;
  else
    k = fed::element_chunk_kernel<R, TDK, 0, 8>;
  launch_step_kernel(c, k, n, fed::kThreads, smem, s, a, base);
}

enum { K_ELEM = 0, K_NODE = 1, K_XCHG = 2 };

cudaEvent_t pool_get(fed_ctx *c) {
  if (!c->tpool.empty()) {
    cudaEvent_t e = c->tpool.back();
    c->tpool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// start a timed region of `kind` on stream s (no-op unless timing is on)
int tbegin(fed_ctx *c, int kind, cudaStream_t s) {
  if (!c->timing) return -1;
  fed_ctx::Rec r{kind, pool_get(c), pool_get(c)};
  cudaEventRecord(r.a, s);
  c->trec.push_back(r);
  return (int)c->trec.size() - 1;
}
void tend(fed_ctx *c, int idx, cudaStream_t s) {
  if (idx >= 0) cudaEventRecord(c->trec[idx].b, s);
}

bool is_multi(const fed_ctx *c) { return c->pl.nranks > 1 && !c->pl.nbr_rank.empty(); }

// Phase 1 of a step: element loads of the interface chunks (all chunks when there is
// no neighbour).  PEER transport: ONE launch of all chunks, interface chunks first;
// the last interface CTA to finish raises the neighbours' flags.
template <typename R, int TDK>
fed_status enqueue_elem_first(fed_ctx *c, int k_off) {
  const fed::Plan &pl = c->pl;
  fed::StepArgs<R> a = make_args<R>(c);
  a.k_off = k_off;
  cudaStream_t s = c->stream;
  if (pl.scatter == FED_SCATTER_ATOMIC) {
    int ti = tbegin(c, K_ELEM, s);
    unsigned grid = (unsigned)((pl.n_slots + 255) / 256);
    if (pl.npe == 4)
      fed::element_atomic_kernel<R, TDK, 4><<<grid, 256, 0, s>>>(a);
    else
      fed::element_atomic_kernel<R, TDK, 8><<<grid, 256, 0, s>>>(a);
    CU(cudaGetLastError());
    c->launches_total++;
    tend(c, ti, s);
    return FED_OK;
  }
  if (fed::atomic_family(pl.scatter)) {  // measured baselines (single rank)
    int ti = tbegin(c, K_ELEM, s);
    const bool tet = pl.npe == 4;
    if (pl.scatter == FED_SCATTER_ATOMIC_WARP) {
      unsigned grid = (unsigned)((pl.n_slots + 255) / 256);
      fed::element_scatter_kernel<R, TDK, 8, 1><<<grid, 256, 0, s>>>(a, nullptr, 0, pl.n_slots, (R *)nullptr);
      c->launches_total++;
    } else if (pl.scatter == FED_SCATTER_COLOR_PASSES) {
      for (int k = 0; k < fed::kMaxColors; ++k) {
        const int64_t b0 = pl.cp_off[k], b1 = pl.cp_off[k + 1];
        if (b1 <= b0) continue;
        unsigned grid = (unsigned)((b1 - b0 + 255) / 256);
        if (tet)
          fed::element_scatter_kernel<R, TDK, 4, 2><<<grid, 256, 0, s>>>(a, c->cp_list, b0, b1, (R *)nullptr);
        else
          fed::element_scatter_kernel<R, TDK, 8, 2><<<grid, 256, 0, s>>>(a, c->cp_list, b0, b1, (R *)nullptr);
        c->launches_total++;
      }
    } else {  // GATHER
      unsigned grid = (unsigned)((pl.n_slots + 255) / 256);
      unsigned gn = (unsigned)std::max<int64_t>(1, (pl.N_loc + 255) / 256);
      if (tet) {
        fed::element_scatter_kernel<R, TDK, 4, 3><<<grid, 256, 0, s>>>(a, nullptr, 0, pl.n_slots, (R *)c->vbuf);
        fed::gather_kernel<R, 4><<<gn, 256, 0, s>>>(a, c->g_ptr, c->g_list, (const R *)c->vbuf);
      } else {
        fed::element_scatter_kernel<R, TDK, 8, 3><<<grid, 256, 0, s>>>(a, nullptr, 0, pl.n_slots, (R *)c->vbuf);
        fed::gather_kernel<R, 8><<<gn, 256, 0, s>>>(a, c->g_ptr, c->g_list, (const R *)c->vbuf);
      }
      c->launches_total += 2;
    }
    CU(cudaGetLastError());
    tend(c, ti, s);
    return FED_OK;
  }
  const bool multi = is_multi(c);
  int64_t n_first = (multi && !c->Fif) ? pl.n_chunks_if : pl.n_chunks;
  if (multi && c->Fif) {
    a.if_done = c->if_done;
    a.n_sig_ctas = (int)pl.n_chunks_if;
  }
  if (n_first > 0) {
    int ti = tbegin(c, K_ELEM, s);
    launch_chunks<R, TDK>(c, a, (unsigned)n_first, 0, stream_smem(pl), s);
    CU(cudaGetLastError());
    c->launches_total++;
    tend(c, ti, s);
  }
  return FED_OK;
}

// Phase 2: the NCCL exchange of the interface slices on the comm stream (real
// multi-process NCCL transport only), overlapping phase 3
template <typename R>
fed_status enqueue_exchange_start(fed_ctx *c) {
  const fed::Plan &pl = c->pl;
  const int wsize = (int)sizeof(R);
  if (!is_multi(c) || c->Fif || !c->ncomm) return FED_OK;
  CU(cudaEventRecord(c->ev_if, c->stream));
  CU(cudaStreamWaitEvent(c->comm, c->ev_if, 0));
  int xi = tbegin(c, K_XCHG, c->comm);
  NcclApi &N = nccl();
  int dt = wsize == 4 ? ncclFloat32_ : ncclFloat64_;
  NC(N.GroupStart());
  for (size_t i = 0; i < pl.nbr_rank.size(); ++i) {
    char *sb = (char *)c->F + (size_t)(pl.N_int + pl.nbr_off[i]) * wsize;
    char *rb = (char *)c->Frx + (size_t)pl.nbr_off[i] * wsize;
    NC(N.Send(sb, (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
    NC(N.Recv(rb, (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
  }
  NC(N.GroupEnd());
  tend(c, xi, c->comm);
  CU(cudaEventRecord(c->ev_comm, c->comm));
  return FED_OK;
}

// Phase 3: element loads of the remaining (interior) chunks
template <typename R, int TDK>
fed_status enqueue_elem_rest(fed_ctx *c, int k_off) {
  const fed::Plan &pl = c->pl;
  if (fed::atomic_family(pl.scatter) || !is_multi(c) || c->Fif) return FED_OK;
  int64_t n_rest = pl.n_chunks - pl.n_chunks_if;
  if (n_rest <= 0) return FED_OK;
  fed::StepArgs<R> a = make_args<R>(c);
  a.k_off = k_off;
  int ti = tbegin(c, K_ELEM, c->stream);
  launch_chunks<R, TDK>(c, a, (unsigned)n_rest, (int)pl.n_chunks_if, stream_smem(pl), c->stream);
  CU(cudaGetLastError());
  c->launches_total++;
  tend(c, ti, c->stream);
  return FED_OK;
}

// Phase 4: node update of shared / boundary / Dirichlet nodes (all nodes in atomic
// mode), after the exchange; PEER: the kernel itself waits for the neighbours
template <typename R, int TDK>
fed_status enqueue_node(fed_ctx *c, int k_off) {
  const fed::Plan &pl = c->pl;
  if (is_multi(c) && !c->Fif && c->ncomm) CU(cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
  fed::StepArgs<R> a = make_args<R>(c);
  a.k_off = k_off;
  int64_t start = !fed::atomic_family(pl.scatter) ? pl.N_int : 0;
  int64_t cnt = pl.N_loc - start;
  const int64_t per_block = fed::NodeShape<R>::per_block;
  unsigned grid = (unsigned)std::max<int64_t>(1, (cnt + per_block - 1) / per_block);
  int ti = tbegin(c, K_NODE, c->stream);
  CU(launch_step_kernel(c, fed::node_kernel<R, TDK>, grid, fed::NodeShape<R>::threads, 0, c->stream, a, start));
  c->launches_total++;
  tend(c, ti, c->stream);
  return FED_OK;
}

// Local rank group, NCCL transport: deliver every rank's interface slices into its
// neighbours' receive buffers exactly as ncclSend/ncclRecv would (device copies)
fed_status group_copy_exchange(fed_ctx *g, int wsize) {
  const int P = (int)g->sub.size();
  for (int r = 0; r < P; ++r) {
    fed_ctx *c = g->sub[r];
    const fed::Plan &pl = c->pl;
    for (size_t i = 0; i < pl.nbr_rank.size(); ++i) {
      const fed_ctx *o = g->sub[pl.nbr_rank[i]];
      const fed::Plan &po = o->pl;
      // the neighbour's slice shared with rank r
      int64_t off = -1, cnt = 0;
      for (size_t j = 0; j < po.nbr_rank.size(); ++j)
        if (po.nbr_rank[j] == r) { off = po.nbr_off[j]; cnt = po.nbr_cnt[j]; }
      if (off < 0 || cnt != pl.nbr_cnt[i]) return fail(FED_ERR_INVALID, "interface slices of neighbouring slabs differ");
      int xi = tbegin(c, K_XCHG, g->stream);
      const char *src = (const char *)o->F + (size_t)(po.N_int + off) * wsize;
      CU(cudaMemcpyAsync((char *)c->Frx + (size_t)pl.nbr_off[i] * wsize, src, (size_t)cnt * wsize,
                         cudaMemcpyDeviceToDevice, g->stream));
      tend(c, xi, g->stream);
    }
  }
  return FED_OK;
}

// one full time step of a context (single rank, or every slab of a local group)
template <typename R, int TDK>
fed_status enqueue_step(fed_ctx *c, int k_off) {
  fed_status st;
  if (c->sub.empty()) {
    if ((st = enqueue_elem_first<R, TDK>(c, k_off)) != FED_OK) return st;
    if ((st = enqueue_exchange_start<R>(c)) != FED_OK) return st;
    if ((st = enqueue_elem_rest<R, TDK>(c, k_off)) != FED_OK) return st;
    return enqueue_node<R, TDK>(c, k_off);
  }
  // group: every slab's interface chunks (PEER: raising their flags), then the
  // interior chunks, then the exchange, then the node kernels -- so a node kernel
  // only ever starts after the loads it reads (no kernel waits on another)
  for (fed_ctx *r : c->sub)
    if ((st = enqueue_elem_first<R, TDK>(r, k_off)) != FED_OK) return st;
  for (fed_ctx *r : c->sub)
    if ((st = enqueue_elem_rest<R, TDK>(r, k_off)) != FED_OK) return st;
  if (c->transport == FED_TRANSPORT_NCCL && (st = group_copy_exchange(c, (int)sizeof(R))) != FED_OK) return st;
  for (fed_ctx *r : c->sub)
    if ((st = enqueue_node<R, TDK>(r, k_off)) != FED_OK) return st;
  return FED_OK;
}

int64_t launches_sum(const fed_ctx *c) {
  int64_t n = c->launches_total;
  for (const fed_ctx *r : c->sub) n += r->launches_total;
  return n;
}
void launches_reset_to(fed_ctx *c, int64_t own, const std::vector<int64_t> &subs) {
  c->launches_total = own;
  for (size_t i = 0; i < c->sub.size(); ++i) c->sub[i]->launches_total = subs[i];
}

fed_status advance(fed_ctx *c, int64_t n) {
  fed::advance_step_kernel<<<1, 1, 0, c->stream>>>(c->d_step, (long long)n);
  CU(cudaGetLastError());
  c->launches_total++;
  return FED_OK;
}

// eager launches of n steps followed by one step-counter advance
// eager launches of n steps followed by one step-counter advance
template <typename R, int TDK>
fed_status eager_steps(fed_ctx *c, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    fed_status st = enqueue_step<R, TDK>(c, (int)k);
    if (st != FED_OK) return st;
  }
  return advance(c, n);
}

// ---- resident mode
template <typename R, int TDK>
void *resident_fn(const fed::Plan &pl) {
  const bool fx = pl.precision == 32 && pl.chunk_elems <= 1024 && pl.max_local_used <= fed::kLS;
  if (pl.npe == 4)
    return fx ? (void *)fed::resident_kernel<R, TDK, fed::kLS, 4> : (void *)fed::resident_kernel<R, TDK, 0, 4>;
  return fx ? (void *)fed::resident_kernel<R, TDK, fed::kLS, 8> : (void *)fed::resident_kernel<R, TDK, 0, 8>;
}

// shared memory of the resident kernel: sT/sF with the fixed stride when it applies
size_t resident_smem_bytes(const fed::Plan &pl) {
  const bool fx = pl.precision == 32 && pl.chunk_elems <= 1024 && pl.max_local_used <= fed::kLS;
  const int ls = fx ? fed::kLS : 0;
  const bool phi = pl.td == 2;
  const size_t b = pl.precision == 32 ? fed::chunk_smem_bytes<float>(pl.chunk_elems, pl.max_local_used, false, phi, ls)
                                      : fed::chunk_smem_bytes<double>(pl.chunk_elems, pl.max_local_used, false, phi, ls);
  return b + (size_t)pl.max_local_used + 32;  // + per-node flags
}

size_t resident_smem(const fed::Plan &pl) { return resident_smem_bytes(pl); }

// decide (and prepare) resident mode after upload: every chunk on the colour-phase
// fast path, all chunks co-resident, cooperative launch available
template <typename R, int TDK>
fed_status setup_resident(fed_ctx *c, int want) {
  const fed::Plan &pl = c->pl;
  c->resident = false;
  if (want < 0) return FED_OK;
  std::string why;
  bool ok = pl.nranks == 1 && !pl.chunk_nbr_ptr.empty() &&
            (pl.scatter == FED_SCATTER_CHUNK_REGC || (pl.npe == 4 && pl.scatter == FED_SCATTER_CHUNK_REG)) &&
            pl.chunk_elems <= 8 * fed::kThreads;
  if (!ok) why = "needs one rank, a register chunk scatter, chunks <= 1024 and a mesh of <= 2048 chunks";
  for (int64_t k = 0; ok && pl.npe == 8 && k < pl.n_chunks; ++k) {
    const int32_t *co = &pl.color_off[k * (fed::kMaxColors + 1)];
    if (pl.chunk_hdr[k * fed::kChunkHdr + fed::CH_N_COLORS] > 8) ok = false;
    for (int q = 0; ok && q < 8; ++q) ok = co[q + 1] - co[q] <= fed::kThreads;
    if (!ok) why = "a chunk has more than 8 colours or more than 128 elements in a colour";
  }
  int dev = c->device, coop = 0, nsm = 0, per_sm = 0;
  const size_t smem = resident_smem(pl);
  if (ok) {
    CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    void *fn = resident_fn<R, TDK>(pl);
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, fed::kThreads, smem));
    ok = coop && (int64_t)per_sm * nsm >= pl.n_chunks;
    if (!ok) why = "chunks do not all fit on the GPU at once (" + std::to_string(pl.n_chunks) + " > " +
                   std::to_string(per_sm) + " x " + std::to_string(nsm) + ")";
  }
  if (!ok) {
    if (want > 0) return fail(FED_ERR_INVALID, "resident mode not possible: " + why);
    return FED_OK;
  }
  fed_status st;
  if ((st = upload(c, &c->nbr_ptr, pl.chunk_nbr_ptr)) != FED_OK) return st;
  if ((st = upload(c, &c->nbr, pl.chunk_nbr)) != FED_OK) return st;
  if ((st = upload(c, &c->sp_own, pl.sp_own)) != FED_OK) return st;
  if ((st = dalloc(c, &c->d_done, (size_t)pl.n_chunks)) != FED_OK) return st;
  CU(cudaMemset(c->d_done, 0, sizeof(unsigned long long) * pl.n_chunks));
  {
    R *f3 = nullptr;
    if ((st = dalloc(c, &f3, (size_t)(3 * f3_stride(pl)))) != FED_OK) return st;
    CU(cudaMemset(f3, 0, sizeof(R) * 3 * f3_stride(pl)));
    c->F3 = f3;
  }
  if ((st = dalloc(c, &c->d_res_err, 2)) != FED_OK) return st;
  CU(cudaMemset(c->d_res_err, 0, 2 * sizeof(unsigned int)));
  c->res_smem = smem;
  c->resident = true;
  return FED_OK;
}

// n steps in one cooperative launch, then the last step's shared-node update
template <typename R, int TDK>
fed_status resident_steps(fed_ctx *c, int64_t n) {
  const fed::Plan &pl = c->pl;
  for (int64_t k0 = 0; k0 < n; k0 += (1 << 30)) {
    const int nk = (int)std::min<int64_t>(n - k0, 1 << 30);
    const long long g0 = (long long)(c->step + k0);
    fed::StepArgs<R> a = make_args<R>(c);
    fed::ResArgs<R> r;
    r.n_steps = nk;
    r.g0 = g0;
    r.nbr_ptr = c->nbr_ptr;
    r.nbr = c->nbr;
    r.sp_own = c->sp_own;
    r.done = c->d_done;
    r.F3 = (R *)c->F3;
    r.f3_stride = f3_stride(pl);
    r.err = c->d_res_err;
    r.abort = c->d_res_err + 1;
    void *args[] = {(void *)&a, (void *)&r};
    CU(cudaLaunchCooperativeKernel(resident_fn<R, TDK>(pl), dim3((unsigned)pl.n_chunks), dim3(fed::kThreads), args,
                                   c->res_smem, c->stream));
    c->launches_total++;
    // finalize: the shared-node update of the last step, from F[(g_last) % 3]
    const long long gl = g0 + nk - 1;
    a.F = (R *)c->F3 + (size_t)(gl % 3) * r.f3_stride - pl.N_int;  // node_kernel reads F[N_int + s]
    a.k_off = (int)(k0 + nk - 1);
    const int64_t cnt = pl.N_loc - pl.N_int;
    const int64_t per_block = fed::NodeShape<R>::per_block;
    unsigned grid = (unsigned)std::max<int64_t>(1, (cnt + per_block - 1) / per_block);
    fed::node_kernel<R, TDK><<<grid, fed::NodeShape<R>::threads, 0, c->stream>>>(a, pl.N_int);
    CU(cudaGetLastError());
    c->launches_total++;
    // the buffer of step gl-1 still holds consumed loads
    if (pl.N_sp > 0)
      CU(cudaMemsetAsync((R *)c->F3 + (size_t)((gl + 2) % 3) * r.f3_stride, 0, sizeof(R) * pl.N_sp, c->stream));
  }
  return advance(c, n);
}

template <typename R, int TDK>
fed_status run_steps(fed_ctx *c, int64_t n) {
  fed_status st;
  if (c->resident && !c->timing && !c->monitor) return resident_steps<R, TDK>(c, n);
  if (c->timing || c->graph_steps <= 0) {
    for (int64_t k = 0; k < n; k += (1 << 20)) {
      st = eager_steps<R, TDK>(c, std::min<int64_t>(n - k, 1 << 20));
      if (st != FED_OK) return st;
    }
    return FED_OK;
  }
  int64_t G = c->graph_steps;
  if (n >= G && !c->graph) {
    // capture G steps + one counter advance; replays are then position independent
    cudaGraph_t g = nullptr;
    const int64_t before = launches_sum(c);
    std::vector<int64_t> sub_before;
    for (fed_ctx *r : c->sub) sub_before.push_back(r->launches_total);
    const int64_t own_before = c->launches_total;
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    st = eager_steps<R, TDK>(c, G);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->graph_kernels = (int)(launches_sum(c) - before);
    launches_reset_to(c, own_before, sub_before);
    if (st != FED_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e != cudaSuccess) return fail(FED_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(FED_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    c->graph_len = (int)G;
  }
  int64_t k = 0;
  while (c->graph && n - k >= c->graph_len) {
    CU(cudaGraphLaunch(c->graph, c->stream));
    c->launches_total += c->graph_kernels;
    k += c->graph_len;
  }
  if (k < n) return eager_steps<R, TDK>(c, n - k);
  return FED_OK;
}

template <typename R>
fed_status upload_all(fed_ctx *c) {
  fed::Plan &pl = c->pl;
  fed_status st;
#define UP(x) \
  if ((st = (x)) != FED_OK) return st
  std::vector<R> T0(pl.T0.begin(), pl.T0.end());
  R *T = nullptr;
  UP(upload(c, &T, T0));
  c->T = T;
  R *F = nullptr;
  UP(dalloc(c, &F, (size_t)pl.N_loc));
  CU(cudaMemset(F, 0, sizeof(R) * std::max<int64_t>(1, pl.N_loc)));
  c->F = F;
  UP(upload_real<R>(c, &c->coef, pl.coef));
  if (!pl.Qvol.empty()) UP(upload_real<R>(c, &c->Qvol, pl.Qvol));
  UP(upload_real<R>(c, &c->P, pl.P));
  {
    uint16_t *q = nullptr;
    UP(upload(c, &q, pl.conn16));
    c->conn16 = reinterpret_cast<uint4 *>(q);
  }
  if (pl.npe == 8 && pl.scatter == FED_SCATTER_CHUNK_REGC && pl.precision == 32) {
    // fp32 streaming colour-phase kernel: one 16-byte record per element slot holding
    // the 8 chunk-local positions packed to 12 bits (96 bits: field q = bits
    // 12q..12q+11 of the little-endian words x, y, z) and the operator word P_xx in w;
    // the other five operator words stay in their planes.  36 B per element instead
    // of 40 B, in 6 loads instead of 7.  fp64 (no room for an 8-byte word) and the
    // resident / staged kernels keep the 16-bit byte offsets.
    const int wb = pl.precision / 8;
    std::vector<uint32_t> pr((size_t)4 * pl.n_slots);
    for (int64_t s = 0; s < pl.n_slots; ++s) {
      uint32_t w[3] = {0, 0, 0};
      for (int q = 0; q < 8; ++q) {
        const uint32_t l = pl.conn16[8 * s + q] / wb;
        if (l >= 4096u) return fail(FED_ERR_INVALID, "internal: chunk exceeds the 12-bit packed connectivity");
        const int bit = 12 * q;
        w[bit >> 5] |= l << (bit & 31);
        if ((bit & 31) > 20) w[(bit >> 5) + 1] |= l >> (32 - (bit & 31));
      }
      const float pxx = (float)pl.P[s];  // plane 0 (xx), rounded as upload_real<float> does
      uint32_t pb;
      std::memcpy(&pb, &pxx, 4);
      pr[4 * s] = w[0];
      pr[4 * s + 1] = w[1];
      pr[4 * s + 2] = w[2];
      pr[4 * s + 3] = pb;
    }
    uint32_t *q = nullptr;
    UP(upload(c, &q, pr));
    c->rec12 = reinterpret_cast<uint4 *>(q);
  }
  if (!pl.conn32.empty()) {
    int32_t *q = nullptr;
    UP(upload(c, &q, pl.conn32));
    c->conn32 = reinterpret_cast<int4 *>(q);
  }
  if (!pl.cp_list.empty()) UP(upload(c, &c->cp_list, pl.cp_list));
  if (pl.scatter == FED_SCATTER_GATHER) {
    UP(upload(c, &c->g_ptr, pl.g_ptr));
    UP(upload(c, &c->g_list, pl.g_list));
    R *vb = nullptr;
    UP(dalloc(c, &vb, (size_t)(3 * std::max<int64_t>(1, pl.n_slots))));
    c->vbuf = vb;
  }
  UP(upload(c, &c->chunk_hdr, pl.chunk_hdr));
  UP(upload(c, &c->color_off, pl.color_off));
  UP(upload(c, &c->sp_list, pl.sp_list));
  UP(upload(c, &c->bc_ptr, pl.bc_ptr));
  UP(upload_real<R>(c, &c->bc_coef, pl.bc_coef));
  // tables packed as [T_0..T_{n-1} | v_0..v_{n-1} | slopes of the n-1 segments (fp64)]
  auto pack_table = [](const std::vector<double> &Tt, const std::vector<double> &vt) {
    std::vector<double> t(Tt);
    t.insert(t.end(), vt.begin(), vt.end());
    for (size_t i = 0; i + 1 < Tt.size(); ++i) t.push_back((vt[i + 1] - vt[i]) / (Tt[i + 1] - Tt[i]));
    return t;
  };
  if (!pl.k_tab_T.empty()) UP(upload_real<R>(c, &c->kt, pack_table(pl.k_tab_T, pl.k_tab_v)));
  if (!pl.c_tab_T.empty()) UP(upload_real<R>(c, &c->ct, pack_table(pl.c_tab_T, pl.c_tab_v)));
  UP(upload_real<R>(c, &c->bc_tinf, pl.bc_tinf));
  UP(upload(c, &c->bc_ekind, pl.bc_ekind));
  UP(upload(c, &c->sp_kind, pl.sp_kind));
  UP(upload_real<R>(c, &c->sp_dirT, pl.sp_dirT));
  {
    R *q = nullptr;
    UP(dalloc(c, &q, (size_t)std::max<int64_t>(1, pl.n_if)));
    CU(cudaMemset(q, 0, sizeof(R) * std::max<int64_t>(1, pl.n_if)));
    c->Frx = q;
  }
  if (c->transport == FED_TRANSPORT_PEER && pl.nranks > 1) {
    // one allocation (one IPC handle): [sig[2] | pad | Fif[2][n_if]] (step parity)
    unsigned char *blk = nullptr;
    const size_t nb = 256 + sizeof(R) * 2 * (size_t)std::max<int64_t>(1, pl.n_if);
    UP(dalloc(c, &blk, nb, /*cuda_only=*/true));  // shared by CUDA IPC: an allocation of its own
    CU(cudaMemset(blk, 0, nb));
    c->peer_blk = blk;
    c->sig = reinterpret_cast<unsigned long long *>(blk);
    c->Fif = blk + 256;
    UP(dalloc(c, &c->if_done, 1));
    UP(dalloc(c, &c->peer_err, 1));
    CU(cudaMemset(c->if_done, 0, sizeof(unsigned int)));
    CU(cudaMemset(c->peer_err, 0, sizeof(unsigned int)));
  }
  UP(upload(c, &c->node_global, pl.node_global));
  UP(upload(c, &c->owned, pl.node_owned));
  UP(dalloc(c, &c->d_step, 1));
  UP(dalloc(c, &c->d_fail, 1));
  UP(dalloc(c, &c->d_dTmax, 1));
  UP(dalloc(c, &c->d_scratch, 4));
  CU(cudaMemset(c->d_scratch, 0, 4 * sizeof(unsigned int)));
  if (fed::kChecked) {
    UP(dalloc(c, &c->d_check, 1));
    CU(cudaMemset(c->d_check, 0, sizeof(unsigned int)));
  }
  CU(cudaMemset(c->d_step, 0, sizeof(long long)));
  CU(cudaMemset(c->d_fail, 0xff, sizeof(unsigned long long)));
  if (pl.td == 3) {
    UP((set_kernel_attrs<R, 3>(c)));
  } else if (pl.td == 2) {
    UP((set_kernel_attrs<R, 2>(c)));
  } else if (pl.td == 1) {
    UP((set_kernel_attrs<R, 1>(c)));
  } else {
    UP((set_kernel_attrs<R, 0>(c)));
  }
#undef UP
  return FED_OK;
}

// accumulate the pending timed regions (synchronises the streams)
fed_status harvest_timing(fed_ctx *c) {
  for (fed_ctx *r : c->sub) {
    fed_status st = harvest_timing(r);
    if (st != FED_OK) return st;
  }
  if (c->trec.empty()) return FED_OK;
  CU(cudaStreamSynchronize(c->stream));
  if (c->comm) CU(cudaStreamSynchronize(c->comm));
  for (const fed_ctx::Rec &r : c->trec) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, r.a, r.b));
    if (r.kind == K_ELEM) { c->tacc.element_ms += ms; c->tacc.element_launches++; }
    else if (r.kind == K_NODE) { c->tacc.node_ms += ms; c->tacc.node_launches++; }
    else { c->tacc.exchange_ms += ms; c->tacc.exchange_count++; }
    c->tpool.push_back(r.a);
    c->tpool.push_back(r.b);
  }
  c->trec.clear();
  return FED_OK;
}

}  // namespace

// ----------------------------------------------------------------- ABI
extern "C" {

void fed_options_default(fed_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->precision = 64;
  o->dt = 0.0;
  o->dt_factor = 0.9;
  o->T_lo = 0.0;
  o->T_hi = 0.0;
  o->T_abort = 1e6;
  o->device = 0;
  o->stream = nullptr;
  o->rank = 0;
  o->nranks = 1;
  o->nccl_id = nullptr;
  o->scatter = FED_SCATTER_AUTO;
  o->chunk_elems = 0;
  o->graph_steps = 0;
  o->transport = FED_TRANSPORT_NCCL;
  o->local_ranks = 0;
}

const char *fed_last_error(void) { return g_err.c_str(); }

fed_status fed_nccl_unique_id(void *out128) {
  if (!out128) return fail(FED_ERR_INVALID, "null out");
  NcclApi &N = nccl();
  if (!N.ok) return fail(FED_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NC(N.GetUniqueId(&id));
  std::memcpy(out128, &id, 128);
  return FED_OK;
}

void fed_destroy(fed_ctx *c) {
  if (!c) return;
  for (fed_ctx *r : c->sub) fed_destroy(r);
  c->sub.clear();
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (auto &r : c->trec) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (cudaEvent_t e : c->tpool) cudaEventDestroy(e);
  if (c->ev_if) cudaEventDestroy(c->ev_if);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (!c->dry) cudaDeviceSynchronize();
  if (c->ncomm && c->d_scratch && c->stream && !c->skip_barrier) {
    // all ranks past their last step before any rank unmaps or frees memory a
    // neighbour may still read (PEER transport): a one-word all-reduce as a
    // barrier (skipped when fed_create failed: the ranks agreed on the failure
    // and every rank is already on this path)
    nccl().AllReduce(c->d_scratch, c->d_scratch + 1, 1, ncclUint32_, ncclSum_, c->ncomm, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  for (void *p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->ncomm) nccl().CommDestroy(c->ncomm);
  for (const fed_ctx::Alloc &a : c->allocs) {
    if (a.hooked)
      c->hook_free(a.p, a.bytes, c->device, c->hook_ctx);
    else
      cudaFree(a.p);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->comm) cudaStreamDestroy(c->comm);
  delete c;
}

}  // extern "C"

namespace {

// PEER transport: what a rank needs to know about a neighbour's exchange block
struct PeerDesc {
  unsigned char *blk;   // [sig[2] | pad to 256 B | Fif[2][n_if]] (own device or IPC-mapped)
  int64_t n_if, n_if_lo;
};

// point this rank's flags / loads at its neighbours' blocks (lo = rank-1, hi = rank+1)
fed_status link_peers(fed_ctx *c, const PeerDesc *lo, const PeerDesc *hi) {
  const fed::Plan &pl = c->pl;
  const size_t w = pl.precision == 32 ? 4 : 8;
  const int64_t n_lo = pl.n_if_lo, n_hi = pl.n_if - pl.n_if_lo;
  if ((n_lo > 0) != (lo != nullptr) || (n_hi > 0) != (hi != nullptr))
    return fail(FED_ERR_INVALID, "peer link: neighbour set does not match the partition");
  if (lo) {
    if (lo->n_if - lo->n_if_lo != n_lo) return fail(FED_ERR_INVALID, "peer link: interface sizes differ (rank-1)");
    c->pF_lo = lo->blk + 256 + (size_t)lo->n_if_lo * w;  // rank-1's slice shared with its rank+1 (me)
    c->pstride_lo = lo->n_if;
    c->psig_lo = reinterpret_cast<unsigned long long *>(lo->blk) + 1;  // rank-1 hears from its rank+1 at [1]
  }
  if (hi) {
    if (hi->n_if_lo != n_hi) return fail(FED_ERR_INVALID, "peer link: interface sizes differ (rank+1)");
    c->pF_hi = hi->blk + 256;                                          // rank+1's slice shared with rank-1 (me)
    c->pstride_hi = hi->n_if;
    c->psig_hi = reinterpret_cast<unsigned long long *>(hi->blk) + 0;
  }
  return FED_OK;
}

// Exchange the exchange-block IPC handles over NCCL (all-gather) and map the
// neighbours'.  Collective: every rank takes part in the all-gather even when its
// own handle could not be made (its record then carries ok = 0), so a local
// failure never leaves the other ranks blocked; a rank fails if any rank failed.
fed_status setup_peer_ipc(fed_ctx *c) {
  const fed::Plan &pl = c->pl;
  struct Wire { cudaIpcMemHandle_t h; int64_t n_if, n_if_lo; int64_t ok; };
  Wire mine{};
  std::string why;
  cudaError_t he = cudaIpcGetMemHandle(&mine.h, c->peer_blk);
  if (he != cudaSuccess) why = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(he);
  mine.ok = he == cudaSuccess;
  mine.n_if = pl.n_if;
  mine.n_if_lo = pl.n_if_lo;
  const int P = pl.nranks;
  std::vector<Wire> all((size_t)P);
  unsigned char *d = nullptr;
  CU(cudaMalloc(&d, sizeof(Wire) * (size_t)(P + 1)));
  cudaMemcpy(d, &mine, sizeof(Wire), cudaMemcpyHostToDevice);
  ncclResult_t r = nccl().AllGather(d, d + sizeof(Wire), sizeof(Wire), ncclUint8_, c->ncomm, c->stream);
  cudaError_t e = r == 0 ? cudaStreamSynchronize(c->stream) : cudaSuccess;
  if (r == 0 && e == cudaSuccess) e = cudaMemcpy(all.data(), d + sizeof(Wire), sizeof(Wire) * P, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (r != 0) return fail(FED_ERR_NCCL, std::string("ncclAllGather (IPC handles): ") + nccl().GetErrorString(r));
  CU(e);
  if (!mine.ok) return fail(FED_ERR_CUDA, why);
  for (int q = 0; q < P; ++q)
    if (!all[q].ok) return fail(FED_ERR_CUDA, "PEER set-up failed on rank " + std::to_string(q));
  PeerDesc lo{}, hi{};
  const int R = pl.rank;
  auto open = [&](int q, PeerDesc &pd) -> fed_status {
    void *p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, all[q].h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    pd = PeerDesc{(unsigned char *)p, all[q].n_if, all[q].n_if_lo};
    return FED_OK;
  };
  fed_status st;
  const bool has_lo = pl.n_if_lo > 0, has_hi = pl.n_if > pl.n_if_lo;
  if (has_lo && (st = open(R - 1, lo)) != FED_OK) return st;
  if (has_hi && (st = open(R + 1, hi)) != FED_OK) return st;
  return link_peers(c, has_lo ? &lo : nullptr, has_hi ? &hi : nullptr);
}

// Multi-rank create: every rank reports whether its own set-up succeeded and all
// ranks take the same decision (max over ranks of a status word).  Returns true if
// some rank failed.  The word lives in the context's scratch buffer when it exists.
bool any_rank_failed(fed_ctx *c, bool local_failed) {
  unsigned int *w = c->d_scratch;
  bool own = false;
  if (!w) {
    if (cudaMalloc(&w, 4 * sizeof(unsigned int)) != cudaSuccess) return true;
    own = true;
  }
  unsigned int v = local_failed ? 1u : 0u, res = 1u;
  bool ok = cudaMemcpy(w + 2, &v, sizeof(v), cudaMemcpyHostToDevice) == cudaSuccess &&
            nccl().AllReduce(w + 2, w + 3, 1, ncclUint32_, ncclMax_, c->ncomm, c->stream) == 0 &&
            cudaStreamSynchronize(c->stream) == cudaSuccess &&
            cudaMemcpy(&res, w + 3, sizeof(res), cudaMemcpyDeviceToHost) == cudaSuccess;
  if (own) cudaFree(w);
  return !ok || res != 0u;
}

// plan + upload one rank (a whole problem, or one slab of a local group)
fed_status create_one(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs, const fed_options &o,
                      bool in_group, fed_ctx **out) {
  *out = nullptr;
  fed_ctx *c = new (std::nothrow) fed_ctx();
  if (!c) return fail(FED_ERR_NOMEM, "host allocation");
  std::string err;
  if (o.resident < -1 || o.resident > 1) {
    delete c;
    return fail(FED_ERR_INVALID, "resident must be -1, 0 or 1");
  }
  if (o.device >= 0) {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, o.device) == cudaSuccess && nsm > 0)
      c->pl.sm_count = nsm;
  }
  c->pl.want_gather = !in_group;
  fed_status st = fed::build_plan(mesh, mat, bcs, &o, c->pl, err);
  if (st != FED_OK) {
    delete c;
    return fail(st, err);
  }
  c->transport = o.transport;
  c->is_sub = in_group;
  if ((o.dev_alloc != nullptr) != (o.dev_free != nullptr) || std::isnan(o.wait_timeout_s)) {
    delete c;
    return fail(FED_ERR_INVALID, "dev_alloc and dev_free must be set together; wait_timeout_s must not be NaN");
  }
  c->hook_alloc = o.dev_alloc;
  c->hook_free = o.dev_free;
  c->hook_ctx = o.alloc_ctx;
  if (const char *e = std::getenv("FED_PDL")) c->pdl = std::atoi(e) != 0;  // A/B switch
  if (const char *e = std::getenv("FED_L2_STREAM")) c->l2_stream = (float)std::atof(e);  // A/B switch
  if (o.wait_timeout_s > 0)
    c->wait_ns = (unsigned long long)std::min(o.wait_timeout_s * 1e9, 1e18);
  if (c->transport == FED_TRANSPORT_PEER && c->pl.nranks > 1 && fed::atomic_family(c->pl.scatter)) {
    delete c;
    return fail(FED_ERR_INVALID, "FED_TRANSPORT_PEER needs a CHUNK scatter strategy");
  }
  c->dry = o.device < 0;
  c->device = o.device;
  c->graph_steps = o.graph_steps == 0 ? 16 : (o.graph_steps < 0 ? 0 : o.graph_steps);
  c->launches_per_step = (!fed::atomic_family(c->pl.scatter) && is_multi(c) && c->pl.n_chunks > c->pl.n_chunks_if &&
                          c->transport != FED_TRANSPORT_PEER)
                             ? 3
                             : 2;

  if (c->pl.scatter == FED_SCATTER_GATHER) c->launches_per_step = 3;
  if (c->pl.scatter == FED_SCATTER_COLOR_PASSES) {
    c->launches_per_step = 1;
    for (int k = 0; k < fed::kMaxColors; ++k) c->launches_per_step += c->pl.cp_off[k + 1] > c->pl.cp_off[k];
  }
  if (c->dry) {
    *out = c;
    return FED_OK;
  }
  auto bail = [&](fed_status s) {
    std::string m = g_err;
    fed_destroy(c);
    g_err = m;
    return s;
  };
  cudaError_t e = cudaSetDevice(o.device);
  if (e != cudaSuccess) {
    g_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return bail(FED_ERR_CUDA);
  }
  if (o.stream) {
    c->stream = (cudaStream_t)o.stream;
  } else {
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
      g_err = cudaGetErrorString(e);
      return bail(FED_ERR_CUDA);
    }
    c->own_stream = true;
  }
  const bool multi = c->pl.nranks > 1 && !in_group;
  if (multi) {
    // the communicator first: every later set-up step may fail on one rank only, and
    // the ranks then agree on the outcome over it (the plan above is a deterministic
    // function of the same global inputs on every rank, so it fails on all or none)
    NcclApi &N = nccl();
    if (!N.ok) {
      g_err = "nranks > 1 but libnccl.so.2 could not be loaded";
      return bail(FED_ERR_NCCL);
    }
    if (!o.nccl_id) {
      g_err = "nranks > 1 requires opts.nccl_id";
      return bail(FED_ERR_INVALID);
    }
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_id, 128);
    ncclResult_t r = N.CommInitRank(&c->ncomm, c->pl.nranks, id, c->pl.rank);
    if (r != 0) {
      c->ncomm = nullptr;
      g_err = std::string("ncclCommInitRank: ") + N.GetErrorString(r);
      return bail(FED_ERR_NCCL);
    }
  }
  st = c->pl.precision == 32 ? upload_all<float>(c) : upload_all<double>(c);
  if (st != FED_OK && !multi) return bail(st);
  if (!in_group && st == FED_OK) {
    const int td = c->pl.td, want = o.resident;
    if (c->pl.precision == 32)
      st = td == 3 ? setup_resident<float, 3>(c, want) : td == 2 ? setup_resident<float, 2>(c, want)
           : td == 1 ? setup_resident<float, 1>(c, want) : setup_resident<float, 0>(c, want);
    else
      st = td == 3 ? setup_resident<double, 3>(c, want) : td == 2 ? setup_resident<double, 2>(c, want)
           : td == 1 ? setup_resident<double, 1>(c, want) : setup_resident<double, 0>(c, want);
    if (st != FED_OK && !multi) return bail(st);
  }
  if (multi) {
    std::string why = st != FED_OK ? g_err : "";
    if (st == FED_OK && ((e = cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking)) != cudaSuccess ||
                         (e = cudaEventCreateWithFlags(&c->ev_if, cudaEventDisableTiming)) != cudaSuccess ||
                         (e = cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming)) != cudaSuccess)) {
      st = FED_ERR_CUDA;
      why = cudaGetErrorString(e);
    }
    // collective on every rank, whatever happened above (a failed rank's record says so)
    if (c->transport == FED_TRANSPORT_PEER) {
      fed_status sp = setup_peer_ipc(c);
      if (st == FED_OK && sp != FED_OK) {
        st = sp;
        why = g_err;
      }
    }
    if (any_rank_failed(c, st != FED_OK)) {
      c->skip_barrier = true;
      g_err = st != FED_OK ? why : "fed_create failed on another rank";
      return bail(st != FED_OK ? st : FED_ERR_STATE);
    }
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return bail(FED_ERR_CUDA);
  }
  *out = c;
  return FED_OK;
}

// local rank group: local_ranks slabs of one mesh on one device, one stream
fed_status create_group(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs, const fed_options &o,
                        fed_ctx **out) {
  const int P = o.local_ranks;
  if (o.nranks != 1 || o.rank != 0) return fail(FED_ERR_INVALID, "local_ranks > 1 requires rank 0 of nranks 1");
  if (o.transport != FED_TRANSPORT_NCCL && o.transport != FED_TRANSPORT_PEER) return fail(FED_ERR_INVALID, "bad transport");
  fed_ctx *g = new (std::nothrow) fed_ctx();
  if (!g) return fail(FED_ERR_NOMEM, "host allocation");
  auto bail = [&](fed_status s) {
    std::string m = g_err;
    fed_destroy(g);
    g_err = m;
    return s;
  };
  g->transport = o.transport;
  if ((o.dev_alloc != nullptr) != (o.dev_free != nullptr)) {
    delete g;
    return fail(FED_ERR_INVALID, "dev_alloc and dev_free must be set together");
  }
  g->hook_alloc = o.dev_alloc;
  g->hook_free = o.dev_free;
  g->hook_ctx = o.alloc_ctx;
  g->dry = o.device < 0;
  g->device = o.device;
  g->graph_steps = o.graph_steps == 0 ? 16 : (o.graph_steps < 0 ? 0 : o.graph_steps);
  cudaError_t e;
  if (!g->dry) {
    if ((e = cudaSetDevice(o.device)) != cudaSuccess) {
      g_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
      return bail(FED_ERR_CUDA);
    }
    if (o.stream) {
      g->stream = (cudaStream_t)o.stream;
    } else {
      if ((e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking)) != cudaSuccess) {
        g_err = cudaGetErrorString(e);
        return bail(FED_ERR_CUDA);
      }
      g->own_stream = true;
    }
  }
  fed_status st;
  for (int r = 0; r < P; ++r) {
    fed_options orr = o;
    orr.rank = r;
    orr.nranks = P;
    orr.local_ranks = 0;
    orr.stream = g->stream;
    orr.graph_steps = -1;  // the group captures the graphs
    fed_ctx *sc = nullptr;
    if ((st = create_one(mesh, mat, bcs, orr, true, &sc)) != FED_OK) return bail(st);
    g->sub.push_back(sc);
  }
  // the group's plan carries the problem-wide scalars used by the ABI
  const fed::Plan &p0 = g->sub[0]->pl;
  g->pl.precision = p0.precision;
  g->pl.td = p0.td;
  std::memcpy(g->pl.kl, p0.kl, sizeof(p0.kl));
  std::memcpy(g->pl.cl, p0.cl, sizeof(p0.cl));
  g->pl.npe = p0.npe;
  g->pl.scatter = p0.scatter;
  g->pl.rank = 0;
  g->pl.nranks = P;
  g->pl.dt = p0.dt;
  g->pl.dt_crit = p0.dt_crit;
  g->pl.N_glob = p0.N_glob;
  g->pl.E_glob = p0.E_glob;
  g->pl.chunk_elems = p0.chunk_elems;
  for (fed_ctx *r : g->sub) g->launches_per_step += r->launches_per_step;
  if (!g->dry) {
    // one step counter / failure word / monitor / peer-error word for the group
    fed_status s2;
    if ((s2 = dalloc(g, &g->d_step, 1)) != FED_OK || (s2 = dalloc(g, &g->d_fail, 1)) != FED_OK ||
        (s2 = dalloc(g, &g->d_dTmax, 1)) != FED_OK || (s2 = dalloc(g, &g->peer_err, 1)) != FED_OK)
      return bail(s2);
    if ((e = cudaMemset(g->d_step, 0, sizeof(long long))) != cudaSuccess ||
        (e = cudaMemset(g->d_fail, 0xff, sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMemset(g->peer_err, 0, sizeof(unsigned int))) != cudaSuccess) {
      g_err = cudaGetErrorString(e);
      return bail(FED_ERR_CUDA);
    }
    for (fed_ctx *r : g->sub) {
      r->d_step = g->d_step;
      r->d_fail = g->d_fail;
      r->d_dTmax = g->d_dTmax;
      if (r->peer_err) r->peer_err = g->peer_err;
    }
    if (g->transport == FED_TRANSPORT_PEER) {
      std::vector<PeerDesc> pd;
      for (fed_ctx *r : g->sub) pd.push_back(PeerDesc{(unsigned char *)r->peer_blk, r->pl.n_if, r->pl.n_if_lo});
      for (int r = 0; r < P; ++r) {
        const fed::Plan &pl = g->sub[r]->pl;
        const bool has_lo = pl.n_if_lo > 0, has_hi = pl.n_if > pl.n_if_lo;
        if ((st = link_peers(g->sub[r], has_lo ? &pd[r - 1] : nullptr, has_hi ? &pd[r + 1] : nullptr)) != FED_OK)
          return bail(st);
      }
    }
  }
  *out = g;
  return FED_OK;
}

// One slab of a local rank group stepped ALONE (fed_debug_time_rank): the kernel
// sequence a rank runs on its own GPU, without waiting for its neighbours (PEER
// waits skipped, NCCL slices copied from whatever the neighbours hold).  Timing only.
template <typename R, int TDK>
fed_status enqueue_rank_alone(fed_ctx *g, fed_ctx *r, int rank, int k_off) {
  fed_status st;
  if ((st = enqueue_elem_first<R, TDK>(r, k_off)) != FED_OK) return st;
  if ((st = enqueue_elem_rest<R, TDK>(r, k_off)) != FED_OK) return st;
  if (g->transport == FED_TRANSPORT_NCCL) {
    const fed::Plan &pl = r->pl;
    const int w = (int)sizeof(R);
    for (size_t i = 0; i < pl.nbr_rank.size(); ++i) {
      const fed_ctx *o = g->sub[pl.nbr_rank[i]];
      const fed::Plan &po = o->pl;
      int64_t off = 0;
      for (size_t j = 0; j < po.nbr_rank.size(); ++j)
        if (po.nbr_rank[j] == rank) off = po.nbr_off[j];
      const char *src = (const char *)o->F + (size_t)(po.N_int + off) * w;
      CU(cudaMemcpyAsync((char *)r->Frx + (size_t)pl.nbr_off[i] * w, src, (size_t)pl.nbr_cnt[i] * w,
                         cudaMemcpyDeviceToDevice, g->stream));
    }
  }
  return enqueue_node<R, TDK>(r, k_off);
}

template <typename R, int TDK>
fed_status time_rank_alone(fed_ctx *g, int rank, int64_t n, double *ms) {
  fed_ctx *r = g->sub[rank];
  r->free_run = true;
  cudaGraph_t gr = nullptr;
  cudaGraphExec_t ex = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  fed_status st = FED_OK;
  cudaError_t e = cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    for (int64_t k = 0; k < n && st == FED_OK; ++k) st = enqueue_rank_alone<R, TDK>(g, r, rank, (int)k);
    e = cudaStreamEndCapture(g->stream, &gr);
  }
  r->free_run = false;
  if (st == FED_OK && e == cudaSuccess) e = cudaGraphInstantiate(&ex, gr, 0);
  if (st == FED_OK && e == cudaSuccess) e = cudaEventCreate(&e0);
  if (st == FED_OK && e == cudaSuccess) e = cudaEventCreate(&e1);
  if (st == FED_OK && e == cudaSuccess) e = cudaGraphLaunch(ex, g->stream);  // warm-up replay
  if (st == FED_OK && e == cudaSuccess) e = cudaEventRecord(e0, g->stream);
  if (st == FED_OK && e == cudaSuccess) e = cudaGraphLaunch(ex, g->stream);
  if (st == FED_OK && e == cudaSuccess) e = cudaEventRecord(e1, g->stream);
  if (st == FED_OK && e == cudaSuccess) e = cudaEventSynchronize(e1);
  float f = 0.f;
  if (st == FED_OK && e == cudaSuccess) e = cudaEventElapsedTime(&f, e0, e1);
  if (ex) cudaGraphExecDestroy(ex);
  if (gr) cudaGraphDestroy(gr);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st != FED_OK) return st;
  if (e != cudaSuccess) return fail(FED_ERR_CUDA, std::string("fed_debug_time_rank: ") + cudaGetErrorString(e));
  *ms = (double)f / (double)n;
  return FED_OK;
}

}  // namespace

extern "C" {

fed_status fed_debug_time_rank(fed_ctx *c, int32_t rank, int64_t n_steps, double *ms_per_step) {
  if (!c || !ms_per_step) return fail(FED_ERR_INVALID, "null argument");
  if (c->sub.empty() || c->dry) return fail(FED_ERR_STATE, "fed_debug_time_rank needs a local rank group on a device");
  if (rank < 0 || rank >= (int32_t)c->sub.size() || n_steps < 1) return fail(FED_ERR_INVALID, "rank or n_steps out of range");
  CU(cudaSetDevice(c->device));
  CU(cudaStreamSynchronize(c->stream));
  c->spoiled = true;
  const int td = c->pl.td;
  if (c->pl.precision == 32)
    return td == 3 ? time_rank_alone<float, 3>(c, rank, n_steps, ms_per_step)
           : td == 2 ? time_rank_alone<float, 2>(c, rank, n_steps, ms_per_step)
           : td == 1 ? time_rank_alone<float, 1>(c, rank, n_steps, ms_per_step)
                     : time_rank_alone<float, 0>(c, rank, n_steps, ms_per_step);
  return td == 3 ? time_rank_alone<double, 3>(c, rank, n_steps, ms_per_step)
         : td == 2 ? time_rank_alone<double, 2>(c, rank, n_steps, ms_per_step)
         : td == 1 ? time_rank_alone<double, 1>(c, rank, n_steps, ms_per_step)
                   : time_rank_alone<double, 0>(c, rank, n_steps, ms_per_step);
}

fed_status fed_create(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs, const fed_options *opts,
                      fed_ctx **out) {
  if (!out) return fail(FED_ERR_INVALID, "out is null");
  *out = nullptr;
  fed_options o;
  if (opts)
    o = *opts;
  else
    fed_options_default(&o);
  if (o.transport != FED_TRANSPORT_NCCL && o.transport != FED_TRANSPORT_PEER) return fail(FED_ERR_INVALID, "bad transport");
  if (o.local_ranks > 1) return create_group(mesh, mat, bcs, o, out);
  return create_one(mesh, mat, bcs, o, false, out);
}

static fed_status check_fail(fed_ctx *c) {
  unsigned long long f = 0;
  unsigned int pe = 0;
  CU(cudaMemcpyAsync(&f, c->d_fail, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
  if (c->peer_err) CU(cudaMemcpyAsync(&pe, c->peer_err, sizeof(pe), cudaMemcpyDeviceToHost, c->stream));
  unsigned int re = 0, ck = 0;
  if (c->d_res_err) CU(cudaMemcpyAsync(&re, c->d_res_err, sizeof(re), cudaMemcpyDeviceToHost, c->stream));
  std::vector<unsigned int> cks(c->sub.size(), 0u);
  if (c->d_check) CU(cudaMemcpyAsync(&ck, c->d_check, sizeof(ck), cudaMemcpyDeviceToHost, c->stream));
  for (size_t i = 0; i < c->sub.size(); ++i)
    if (c->sub[i]->d_check) CU(cudaMemcpyAsync(&cks[i], c->sub[i]->d_check, sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (unsigned int v : cks) ck |= v;
  if (ck) return fail(FED_ERR_CUDA, "device check failed (checked build), bits " + std::to_string(ck) +
                                        " (fed_kernels.cuh FED_DCHECK codes)");
  const std::string lim = std::to_string(c->wait_ns / 1000000000.0) + " s (fed_options.wait_timeout_s)";
  if (re) return fail(FED_ERR_CUDA, "resident mode: a chunk dependency did not resolve within " + lim +
                                        "; state undefined");
  if (pe) return fail(FED_ERR_NCCL, "PEER transport: a neighbour's interface loads did not arrive within " + lim +
                                        "; state undefined");
  if (f != ULLONG_MAX) return fail(FED_ERR_UNSTABLE, "temperature became non-finite or exceeded T_abort at step " +
                                                         std::to_string((long long)f));
  return FED_OK;
}

fed_status fed_step(fed_ctx *c, int64_t n) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (n < 0) return fail(FED_ERR_INVALID, "n must be >= 0");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context (device = -1) cannot step");
  if (c->spoiled) return fail(FED_ERR_STATE, "context used by fed_debug_time_rank: field undefined");
  CU(cudaSetDevice(c->device));
  if (n == 0) return FED_OK;
  fed_status st;
  if (c->ncomm && c->Fif) {
    // PEER rendezvous: no rank's kernels of this call start before every rank has
    // entered it, so the device-side flag waits only ever cover in-call skew
    NC(nccl().AllReduce(c->d_scratch, c->d_scratch + 1, 1, ncclUint32_, ncclSum_, c->ncomm, c->stream));
  }
  const int td = c->pl.td;
  if (c->pl.precision == 32)
    st = td == 3 ? run_steps<float, 3>(c, n) : td == 2 ? run_steps<float, 2>(c, n)
         : (td == 1 ? run_steps<float, 1>(c, n) : run_steps<float, 0>(c, n));
  else
    st = td == 3 ? run_steps<double, 3>(c, n) : td == 2 ? run_steps<double, 2>(c, n)
         : (td == 1 ? run_steps<double, 1>(c, n) : run_steps<double, 0>(c, n));
  if (st != FED_OK) return st;
  c->step += n;
  if (c->timing) {
    st = harvest_timing(c);
    if (st != FED_OK) return st;
  }
  return check_fail(c);
}

fed_status fed_run_until_steady(fed_ctx *c, double tol, int64_t max_steps, int64_t check_every,
                                int64_t *steps_taken, double *last_max_dT) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!(tol > 0) || max_steps < 1 || check_every < 1) return fail(FED_ERR_INVALID, "tol > 0, max_steps >= 1, check_every >= 1");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context (device = -1) cannot step");
  CU(cudaSetDevice(c->device));
  int64_t done = 0;
  float last = INFINITY;
  fed_status st = FED_OK;
  while (done < max_steps) {
    int64_t chunk = std::min<int64_t>(check_every, max_steps - done);
    if (chunk > 1) {
      st = fed_step(c, chunk - 1);
      done += chunk - 1;
      if (st != FED_OK) break;
    }
    // one monitored step: max |T_new - T_old| over all nodes
    CU(cudaMemsetAsync(c->d_dTmax, 0, sizeof(unsigned int), c->stream));
    c->monitor = true;
    for (fed_ctx *r : c->sub) r->monitor = true;
    const int gs = c->graph_steps;
    c->graph_steps = 0;  // eager launch with the monitor pointer set
    st = fed_step(c, 1);
    c->graph_steps = gs;
    c->monitor = false;
    for (fed_ctx *r : c->sub) r->monitor = false;
    done += 1;
    if (st != FED_OK) break;
    // max over ranks so every rank takes the same decision: the word holds the bits
    // of a non-negative float, whose order is the unsigned-integer order
    if (c->ncomm) NC(nccl().AllReduce(c->d_dTmax, c->d_dTmax, 1, ncclUint32_, ncclMax_, c->ncomm, c->stream));
    unsigned int bits = 0;
    CU(cudaMemcpyAsync(&bits, c->d_dTmax, sizeof(bits), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    std::memcpy(&last, &bits, sizeof(last));
    if ((double)last <= tol) break;
  }
  if (steps_taken) *steps_taken = done;
  if (last_max_dT) *last_max_dT = (double)last;
  return st;
}

fed_status fed_get_info(fed_ctx *c, fed_info *o) {
  if (!c || !o) return fail(FED_ERR_INVALID, "null argument");
  std::memset(o, 0, sizeof(*o));
  const fed::Plan &pl = c->pl;
  o->dt = pl.dt;
  o->dt_crit = pl.dt_crit;
  o->step = c->step;
  o->t = (double)c->step * pl.dt;
  o->fail_step = -1;
  if (!c->dry) {
    unsigned long long f = ULLONG_MAX;
    CU(cudaSetDevice(c->device));
    CU(cudaMemcpy(&f, c->d_fail, sizeof(f), cudaMemcpyDeviceToHost));
    if (f != ULLONG_MAX) o->fail_step = (int64_t)f;
  }
  o->precision = pl.precision;
  o->scatter = pl.scatter;
  o->rank = pl.rank;
  o->nranks = pl.nranks;
  o->temperature_dependent = pl.td;
  o->n_nodes_global = pl.N_glob;
  o->n_elems_global = pl.E_glob;
  o->n_nodes_local = pl.N_loc;
  o->n_elems_local = pl.E_loc;
  o->n_interior = pl.N_int;
  o->n_special = pl.N_sp;
  o->n_interface = pl.n_if;
  o->n_chunks = pl.n_chunks;
  o->n_chunks_interface = pl.n_chunks_if;
  o->n_bc_entries = (int64_t)pl.bc_coef.size();
  o->max_colors = pl.max_colors_used;
  o->chunk_elems = pl.chunk_elems;
  o->kernel_launches_per_step = c->launches_per_step;
  o->kernel_launches_total = c->launches_total;
  o->device_bytes = (int64_t)c->bytes;
  o->nodes_per_elem = pl.npe;
  o->colored = pl.colored;
  o->resident = c->resident ? 1 : 0;
  if (!c->sub.empty()) {  // local rank group: totals over the slabs
    o->rank = -1;
    o->colored = 1;
    for (const fed_ctx *r : c->sub) {
      const fed::Plan &q = r->pl;
      o->n_nodes_local += q.N_loc;
      o->n_elems_local += q.E_loc;
      o->n_interior += q.N_int;
      o->n_special += q.N_sp;
      o->n_interface += q.n_if;
      o->n_chunks += q.n_chunks;
      o->n_chunks_interface += q.n_chunks_if;
      o->n_bc_entries += (int64_t)q.bc_coef.size();
      o->max_colors = std::max(o->max_colors, q.max_colors_used);
      o->kernel_launches_total += r->launches_total;
      o->device_bytes += (int64_t)r->bytes;
      o->colored = o->colored && q.colored;
    }
  }
  return FED_OK;
}

// multi-rank readout buffers (lazy; nranks > 1 only): the caller-id layout of all
// ranks' slices, this rank's pack list, send (own slice) and receive (all slices)
static fed_status ensure_gather_buffers(fed_ctx *c) {
  if (c->d_grecv) return FED_OK;
  const fed::Plan &pl = c->pl;
  if (pl.gather_off.size() != (size_t)pl.nranks + 1 || pl.nranks > 64)
    return fail(FED_ERR_STATE, "multi-rank readout layout missing");
  int64_t stride = 0;
  for (int r = 0; r < pl.nranks; ++r) stride = std::max(stride, pl.gather_off[r + 1] - pl.gather_off[r]);
  fed_status st;
  if ((st = upload(c, &c->d_gather_ids, pl.gather_ids)) != FED_OK) return st;
  if ((st = upload(c, &c->d_pack, pl.own_pack)) != FED_OK) return st;
  if ((st = dalloc(c, &c->d_gsend, (size_t)std::max<int64_t>(1, stride))) != FED_OK) return st;
  CU(cudaMemset(c->d_gsend, 0, sizeof(double) * std::max<int64_t>(1, stride)));
  return dalloc(c, &c->d_grecv, (size_t)std::max<int64_t>(1, stride * pl.nranks));
}

static fed_status ensure_caller_buffer(fed_ctx *c) {
  if (c->d_caller) return FED_OK;
  fed_status st = dalloc(c, &c->d_caller, (size_t)c->pl.N_glob);
  if (st != FED_OK) return st;
  return dalloc(c, &c->d_bad, 1);
}

}  // extern "C"

namespace {
// out[node_global[i]] = T[i] for the nodes this slab owns (caller order, fp64)
fed_status launch_to_caller(fed_ctx *c, double *d_out, cudaStream_t s) {
  const fed::Plan &pl = c->pl;
  unsigned grid = (unsigned)std::max<int64_t>(1, (pl.N_loc + 255) / 256);
  if (pl.precision == 32)
    fed::to_caller_kernel<float><<<grid, 256, 0, s>>>((const float *)c->T, c->node_global, c->owned, d_out, pl.N_loc);
  else
    fed::to_caller_kernel<double><<<grid, 256, 0, s>>>((const double *)c->T, c->node_global, c->owned, d_out,
                                                       pl.N_loc);
  CU(cudaGetLastError());
  return FED_OK;
}
// T[i] = in[node_global[i]], then the Dirichlet values again
fed_status launch_from_caller(fed_ctx *c, const double *d_in, unsigned int *d_bad, cudaStream_t s) {
  const fed::Plan &pl = c->pl;
  unsigned grid = (unsigned)std::max<int64_t>(1, (pl.N_loc + 255) / 256);
  unsigned gsp = (unsigned)std::max<int64_t>(1, (pl.N_sp + 255) / 256);
  if (pl.precision == 32) {
    fed::from_caller_kernel<float><<<grid, 256, 0, s>>>(d_in, c->node_global, (float *)c->T, pl.N_loc, d_bad);
    fed::apply_dirichlet_kernel<float><<<gsp, 256, 0, s>>>((float *)c->T, c->sp_kind, (const float *)c->sp_dirT,
                                                           pl.N_int, pl.N_sp);
  } else {
    fed::from_caller_kernel<double><<<grid, 256, 0, s>>>(d_in, c->node_global, (double *)c->T, pl.N_loc, d_bad);
    fed::apply_dirichlet_kernel<double><<<gsp, 256, 0, s>>>((double *)c->T, c->sp_kind, (const double *)c->sp_dirT,
                                                            pl.N_int, pl.N_sp);
  }
  CU(cudaGetLastError());
  return FED_OK;
}
}  // namespace

extern "C" {

fed_status fed_get_temperature(fed_ctx *c, double *out, int64_t n_nodes) {
  if (!c || !out) return fail(FED_ERR_INVALID, "null argument");
  if (n_nodes != c->pl.N_glob) return fail(FED_ERR_INVALID, "n_nodes does not match the mesh");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context has no device state");
  const fed::Plan &pl = c->pl;
  CU(cudaSetDevice(c->device));
  fed_status st = ensure_caller_buffer(c);
  if (st != FED_OK) return st;
  // permute to caller order on the device, then one D2H copy into the caller's buffer
  if (!c->sub.empty()) {
    for (fed_ctx *r : c->sub)  // every node has exactly one owning slab
      if ((st = launch_to_caller(r, c->d_caller, c->stream)) != FED_OK) return st;
  } else if (pl.nranks > 1) {
    // every rank packs the nodes it owns; one all-gather of the packed slices
    // (N_glob doubles received per rank, half the traffic of an all-reduce of the
    // whole field), then an unpack to caller order
    if ((st = ensure_gather_buffers(c)) != FED_OK) return st;
    const int P = pl.nranks;
    int64_t stride = 0;
    fed::RankOffsets ro{};
    ro.nranks = P;
    for (int r = 0; r <= P; ++r) ro.off[r] = pl.gather_off[r];
    for (int r = 0; r < P; ++r) stride = std::max(stride, pl.gather_off[r + 1] - pl.gather_off[r]);
    const int64_t mine = (int64_t)pl.own_pack.size();
    if (mine > 0) {
      unsigned gp = (unsigned)((mine + 255) / 256);
      if (pl.precision == 32)
        fed::pack_owned_kernel<float><<<gp, 256, 0, c->stream>>>((const float *)c->T, c->d_pack, c->d_gsend, mine);
      else
        fed::pack_owned_kernel<double><<<gp, 256, 0, c->stream>>>((const double *)c->T, c->d_pack, c->d_gsend, mine);
      CU(cudaGetLastError());
    }
    NC(nccl().AllGather(c->d_gsend, c->d_grecv, (size_t)stride, ncclFloat64_, c->ncomm, c->stream));
    unsigned gu = (unsigned)((pl.N_glob + 255) / 256);
    fed::unpack_gathered_kernel<<<gu, 256, 0, c->stream>>>(c->d_grecv, c->d_gather_ids, ro, stride, c->d_caller,
                                                            pl.N_glob);
    CU(cudaGetLastError());
  } else {
    if ((st = launch_to_caller(c, c->d_caller, c->stream)) != FED_OK) return st;
  }
  CU(cudaMemcpyAsync(out, c->d_caller, sizeof(double) * pl.N_glob, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return FED_OK;
}

fed_status fed_set_temperature(fed_ctx *c, const double *T, int64_t n_nodes) {
  if (!c || !T) return fail(FED_ERR_INVALID, "null argument");
  if (n_nodes != c->pl.N_glob) return fail(FED_ERR_INVALID, "n_nodes does not match the mesh");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context has no device state");
  const fed::Plan &pl = c->pl;
  CU(cudaSetDevice(c->device));
  fed_status st = ensure_caller_buffer(c);
  if (st != FED_OK) return st;
  CU(cudaMemcpyAsync(c->d_caller, T, sizeof(double) * pl.N_glob, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemsetAsync(c->d_bad, 0, sizeof(unsigned int), c->stream));
  if (!c->sub.empty()) {
    for (fed_ctx *r : c->sub)
      if ((st = launch_from_caller(r, c->d_caller, c->d_bad, c->stream)) != FED_OK) return st;
  } else if ((st = launch_from_caller(c, c->d_caller, c->d_bad, c->stream)) != FED_OK) {
    return st;
  }
  unsigned int bad = 0;
  CU(cudaMemcpyAsync(&bad, c->d_bad, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (bad) return fail(FED_ERR_INVALID, "non-finite temperature (state now undefined; set again)");
  return FED_OK;
}

fed_status fed_set_timing(fed_ctx *c, int32_t enable) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->dry) {
    CU(cudaSetDevice(c->device));
    CU(cudaStreamSynchronize(c->stream));
  }
  for (auto &r : c->trec) {
    c->tpool.push_back(r.a);
    c->tpool.push_back(r.b);
  }
  c->trec.clear();
  c->tacc = fed_timing{};
  c->timing = enable != 0;
  for (fed_ctx *r : c->sub) {
    fed_status st = fed_set_timing(r, enable);
    if (st != FED_OK) return st;
  }
  return FED_OK;
}

fed_status fed_get_timing(fed_ctx *c, fed_timing *out) {
  if (!c || !out) return fail(FED_ERR_INVALID, "null argument");
  *out = c->tacc;
  for (const fed_ctx *r : c->sub) {  // group: summed over the slabs
    out->element_ms += r->tacc.element_ms;
    out->node_ms += r->tacc.node_ms;
    out->exchange_ms += r->tacc.exchange_ms;
    out->element_launches += r->tacc.element_launches;
    out->node_launches += r->tacc.node_launches;
    out->exchange_count += r->tacc.exchange_count;
  }
  return FED_OK;
}

fed_status fed_get_rank_timing(fed_ctx *c, int32_t rank, fed_timing *out) {
  if (!c || !out) return fail(FED_ERR_INVALID, "null argument");
  if (c->sub.empty()) {
    if (rank != 0) return fail(FED_ERR_INVALID, "rank must be 0 for a single-rank context");
    *out = c->tacc;
    return FED_OK;
  }
  if (rank < 0 || rank >= (int32_t)c->sub.size()) return fail(FED_ERR_INVALID, "rank out of range");
  *out = c->sub[rank]->tacc;
  return FED_OK;
}

fed_status fed_debug_plan(fed_ctx *c, int32_t *node_map, int64_t *n_slots, int32_t *slot_chunk, int32_t *slot_color,
                          int32_t *slot_elem) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->sub.empty()) return fail(FED_ERR_STATE, "debug accessors need a single-rank context");
  const fed::Plan &pl = c->pl;
  if (n_slots) *n_slots = pl.n_slots;
  if (node_map) std::memcpy(node_map, pl.node_map.data(), sizeof(int32_t) * pl.N_glob);
  if (slot_chunk) std::memcpy(slot_chunk, pl.slot_chunk.data(), sizeof(int32_t) * pl.n_slots);
  if (slot_color) std::memcpy(slot_color, pl.slot_color.data(), sizeof(int32_t) * pl.n_slots);
  if (slot_elem) std::memcpy(slot_elem, pl.slot_elem.data(), sizeof(int32_t) * pl.n_slots);
  return FED_OK;
}

fed_status fed_debug_chunks(fed_ctx *c, int64_t *n_chunks, int32_t *hdr, int32_t *color_off, uint16_t *conn16) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->sub.empty()) return fail(FED_ERR_STATE, "debug accessors need a single-rank context");
  const fed::Plan &pl = c->pl;
  if (n_chunks) *n_chunks = pl.n_chunks;
  if (hdr)
    for (int64_t k = 0; k < pl.n_chunks; ++k)
      std::memcpy(hdr + k * fed::kChunkHdrPublic, &pl.chunk_hdr[k * fed::kChunkHdr], sizeof(int32_t) * fed::kChunkHdrPublic);
  if (color_off) std::memcpy(color_off, pl.color_off.data(), sizeof(int32_t) * pl.color_off.size());
  if (conn16)  // [n_slots][npe] chunk-local positions (stored as byte offsets)
    for (size_t i = 0; i < pl.conn16.size(); ++i) conn16[i] = (uint16_t)(pl.conn16[i] / (pl.precision / 8));
  return FED_OK;
}

fed_status fed_debug_dataflow(fed_ctx *c, int64_t *n_chunks, int64_t *n_adj, int64_t *n_sp_total, int32_t *adj_ptr,
                              int32_t *adj, int32_t *sp_list, uint8_t *sp_own) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->sub.empty()) return fail(FED_ERR_STATE, "debug accessors need a single-rank context");
  const fed::Plan &pl = c->pl;
  const bool has = !pl.chunk_nbr_ptr.empty();
  if (n_chunks) *n_chunks = has ? pl.n_chunks : 0;
  if (n_adj) *n_adj = has ? (int64_t)pl.chunk_nbr.size() : 0;
  if (n_sp_total) *n_sp_total = has ? (int64_t)pl.sp_list.size() : 0;
  if (!has) return FED_OK;
  if (adj_ptr) std::memcpy(adj_ptr, pl.chunk_nbr_ptr.data(), sizeof(int32_t) * pl.chunk_nbr_ptr.size());
  if (adj) std::memcpy(adj, pl.chunk_nbr.data(), sizeof(int32_t) * pl.chunk_nbr.size());
  if (sp_list) std::memcpy(sp_list, pl.sp_list.data(), sizeof(int32_t) * pl.sp_list.size());
  if (sp_own) std::memcpy(sp_own, pl.sp_own.data(), pl.sp_own.size());
  return FED_OK;
}

fed_status fed_debug_gather(fed_ctx *c, int32_t *nranks, int64_t *off, int32_t *ids, int32_t *own_pack) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->sub.empty()) return fail(FED_ERR_STATE, "debug accessors need a single-rank context");
  const fed::Plan &pl = c->pl;
  if (nranks) *nranks = pl.gather_off.empty() ? 0 : pl.nranks;
  if (pl.gather_off.empty()) return FED_OK;
  if (off) std::memcpy(off, pl.gather_off.data(), sizeof(int64_t) * pl.gather_off.size());
  if (ids) std::memcpy(ids, pl.gather_ids.data(), sizeof(int32_t) * pl.gather_ids.size());
  if (own_pack) std::memcpy(own_pack, pl.own_pack.data(), sizeof(int32_t) * pl.own_pack.size());
  return FED_OK;
}

fed_status fed_debug_nodal(fed_ctx *c, double *V, double *coef, int64_t n_nodes) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (!c->sub.empty()) return fail(FED_ERR_STATE, "debug accessors need a single-rank context");
  const fed::Plan &pl = c->pl;
  if (n_nodes != pl.N_glob) return fail(FED_ERR_INVALID, "n_nodes does not match the mesh");
  for (int64_t n = 0; n < n_nodes; ++n) {
    int32_t i = pl.node_map[n];
    if (V) V[n] = i >= 0 ? pl.V[i] : NAN;
    if (coef) coef[n] = i >= 0 ? pl.coef[i] : NAN;
  }
  return FED_OK;
}

}  // extern "C"
