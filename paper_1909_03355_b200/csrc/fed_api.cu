// fed_api.cu -- C ABI of libfed.so (include/fed.h): context, device memory,
// step launch schedule (CUDA graphs, streams), NCCL interface exchange.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
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
enum { ncclFloat32_ = 7, ncclFloat64_ = 8, ncclSum_ = 0 };

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
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
               api.GroupEnd && api.AllReduce && api.GetErrorString;
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
  std::vector<void *> allocs;
  // typed device buffers (R = float or double, stored as void*)
  void *T = nullptr, *F = nullptr, *coef = nullptr, *Qvol = nullptr, *P = nullptr, *Frx = nullptr;
  void *bc_coef = nullptr, *bc_tinf = nullptr, *sp_dirT = nullptr;
  void *kt_T = nullptr, *kt_v = nullptr, *ct_T = nullptr, *ct_v = nullptr;  // NEXT-2 tables
  int8_t *bc_ekind = nullptr;
  uint4 *conn16 = nullptr;
  int4 *conn32 = nullptr;
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
  // nccl
  ncclComm_t ncomm = nullptr;
  int64_t launches_per_step = 0;
  int64_t launches_total = 0;     // kernels of this library launched by fed_step
  int graph_kernels = 0;          // kernels per graph replay
};

namespace {

template <typename T>
fed_status dalloc(fed_ctx *c, T **p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) return fail(FED_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  c->allocs.push_back(q);
  c->bytes += count * sizeof(T);
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

template <typename R>
fed::StepArgs<R> make_args(fed_ctx *c) {
  const fed::Plan &pl = c->pl;
  fed::StepArgs<R> a;
  a.T = (R *)c->T;
  a.F = (R *)c->F;
  a.coef = (const R *)c->coef;
  a.Qvol = (const R *)c->Qvol;
  a.conn16 = c->conn16;
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
  a.kt_T = (const R *)c->kt_T;
  a.kt_v = (const R *)c->kt_v;
  a.ct_T = (const R *)c->ct_T;
  a.ct_v = (const R *)c->ct_v;
  a.n_kt = (int)pl.k_tab_T.size();
  a.n_ct = (int)pl.c_tab_T.size();
  a.max_local = pl.max_local_used;
  a.chunk_cap = pl.chunk_elems;
  a.step_base = c->d_step;
  a.k_off = 0;
  a.fail_step = c->d_fail;
  a.dTmax = c->monitor ? c->d_dTmax : nullptr;
  return a;
}

size_t chunk_smem(const fed::Plan &pl) {
  const bool staged = pl.scatter == FED_SCATTER_CHUNK || pl.scatter == FED_SCATTER_CHUNK_CAS;
  const bool phi = pl.td == 2;
  return pl.precision == 32 ? fed::chunk_smem_bytes<float>(pl.chunk_elems, pl.max_local_used, staged, phi)
                            : fed::chunk_smem_bytes<double>(pl.chunk_elems, pl.max_local_used, staged, phi);
}

template <typename R, int TDK>
fed_status set_kernel_attrs(fed_ctx *c) {
  int smem = (int)chunk_smem(c->pl);
  const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if (c->pl.npe == 8) {
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 0, 8>, A, smem));
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 1, 8>, A, smem));
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 2, 8>, A, smem));
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 3, 8>, A, smem));
  } else {
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 2, 4>, A, smem));
    CU(cudaFuncSetAttribute(fed::element_chunk_kernel<R, TDK, 3, 4>, A, smem));
  }
  return FED_OK;
}

template <typename R, int TDK>
void launch_chunks(fed_ctx *c, const fed::StepArgs<R> &a, unsigned n, int base, size_t smem, cudaStream_t s) {
  const int sc = c->pl.scatter;
  if (c->pl.npe == 4) {
    if (sc == FED_SCATTER_CHUNK_REGC)
      fed::element_chunk_kernel<R, TDK, 3, 4><<<n, fed::kThreads, smem, s>>>(a, base);
    else
      fed::element_chunk_kernel<R, TDK, 2, 4><<<n, fed::kThreads, smem, s>>>(a, base);
  } else if (sc == FED_SCATTER_CHUNK_CAS) {
    fed::element_chunk_kernel<R, TDK, 1, 8><<<n, fed::kThreads, smem, s>>>(a, base);
  } else if (sc == FED_SCATTER_CHUNK_REG) {
    fed::element_chunk_kernel<R, TDK, 2, 8><<<n, fed::kThreads, smem, s>>>(a, base);
  } else if (sc == FED_SCATTER_CHUNK_REGC) {
    fed::element_chunk_kernel<R, TDK, 3, 8><<<n, fed::kThreads, smem, s>>>(a, base);
  } else {
    fed::element_chunk_kernel<R, TDK, 0, 8><<<n, fed::kThreads, smem, s>>>(a, base);
  }
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

template <typename R, int TDK>
fed_status enqueue_step(fed_ctx *c, int k_off) {
  const fed::Plan &pl = c->pl;
  fed::StepArgs<R> a = make_args<R>(c);
  a.k_off = k_off;
  cudaStream_t s = c->stream;
  const bool multi = pl.nranks > 1 && !pl.nbr_rank.empty();
  if (pl.scatter != FED_SCATTER_ATOMIC) {
    size_t smem = chunk_smem(pl);
    int64_t n_first = multi ? pl.n_chunks_if : pl.n_chunks;
    if (n_first > 0) {
      int ti = tbegin(c, K_ELEM, s);
      launch_chunks<R, TDK>(c, a, (unsigned)n_first, 0, smem, s);
      CU(cudaGetLastError());
      c->launches_total++;
      tend(c, ti, s);
    }
    if (multi) {
      // exchange the interface chunks' partial loads while the interior chunks run
      CU(cudaEventRecord(c->ev_if, s));
      CU(cudaStreamWaitEvent(c->comm, c->ev_if, 0));
      int xi = tbegin(c, K_XCHG, c->comm);
      NcclApi &N = nccl();
      int dt = sizeof(R) == 4 ? ncclFloat32_ : ncclFloat64_;
      NC(N.GroupStart());
      for (size_t i = 0; i < pl.nbr_rank.size(); ++i) {
        R *sb = (R *)c->F + pl.N_int + pl.nbr_off[i];
        R *rb = (R *)c->Frx + pl.nbr_off[i];
        NC(N.Send(sb, (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
        NC(N.Recv(rb, (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
      }
      NC(N.GroupEnd());
      tend(c, xi, c->comm);
      CU(cudaEventRecord(c->ev_comm, c->comm));
      int64_t n_rest = pl.n_chunks - pl.n_chunks_if;
      if (n_rest > 0) {
        int ti = tbegin(c, K_ELEM, s);
        launch_chunks<R, TDK>(c, a, (unsigned)n_rest, (int)pl.n_chunks_if, smem, s);
        CU(cudaGetLastError());
        c->launches_total++;
        tend(c, ti, s);
      }
      CU(cudaStreamWaitEvent(s, c->ev_comm, 0));
    }
  } else {
    int ti = tbegin(c, K_ELEM, s);
    unsigned grid = (unsigned)((pl.n_slots + 255) / 256);
    if (pl.npe == 4)
      fed::element_atomic_kernel<R, TDK, 4><<<grid, 256, 0, s>>>(a);
    else
      fed::element_atomic_kernel<R, TDK, 8><<<grid, 256, 0, s>>>(a);
    CU(cudaGetLastError());
    c->launches_total++;
    tend(c, ti, s);
    if (multi) {
      CU(cudaEventRecord(c->ev_if, s));
      CU(cudaStreamWaitEvent(c->comm, c->ev_if, 0));
      int xi = tbegin(c, K_XCHG, c->comm);
      NcclApi &N = nccl();
      int dt = sizeof(R) == 4 ? ncclFloat32_ : ncclFloat64_;
      NC(N.GroupStart());
      for (size_t i = 0; i < pl.nbr_rank.size(); ++i) {
        NC(N.Send((R *)c->F + pl.N_int + pl.nbr_off[i], (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
        NC(N.Recv((R *)c->Frx + pl.nbr_off[i], (size_t)pl.nbr_cnt[i], dt, pl.nbr_rank[i], c->ncomm, c->comm));
      }
      NC(N.GroupEnd());
      tend(c, xi, c->comm);
      CU(cudaEventRecord(c->ev_comm, c->comm));
      CU(cudaStreamWaitEvent(s, c->ev_comm, 0));
    }
  }
  // node update of shared / boundary / Dirichlet nodes (all nodes in atomic mode)
  int64_t start = pl.scatter != FED_SCATTER_ATOMIC ? pl.N_int : 0;
  int64_t cnt = pl.N_loc - start;
  const int64_t per_block = fed::kNodeVec * fed::kNodeThreads;
  unsigned grid = (unsigned)std::max<int64_t>(1, (cnt + per_block - 1) / per_block);
  {
    int ti = tbegin(c, K_NODE, s);
    fed::node_kernel<R, TDK><<<grid, fed::kNodeThreads, 0, s>>>(a, start);
    CU(cudaGetLastError());
    c->launches_total++;
    tend(c, ti, s);
  }
  return FED_OK;
}

fed_status advance(fed_ctx *c, int64_t n) {
  fed::advance_step_kernel<<<1, 1, 0, c->stream>>>(c->d_step, (long long)n);
  CU(cudaGetLastError());
  c->launches_total++;
  return FED_OK;
}

// eager launches of n steps followed by one step-counter advance
template <typename R, int TDK>
fed_status eager_steps(fed_ctx *c, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    fed_status st = enqueue_step<R, TDK>(c, (int)k);
    if (st != FED_OK) return st;
  }
  return advance(c, n);
}

template <typename R, int TDK>
fed_status run_steps(fed_ctx *c, int64_t n) {
  if (c->timing || c->graph_steps <= 0) {
    for (int64_t k = 0; k < n; k += (1 << 20)) {
      fed_status st = eager_steps<R, TDK>(c, std::min<int64_t>(n - k, 1 << 20));
      if (st != FED_OK) return st;
    }
    return FED_OK;
  }
  int64_t G = c->graph_steps;
  if (n >= G && !c->graph) {
    // capture G steps + one counter advance; replays are then position independent
    cudaGraph_t g = nullptr;
    int64_t before = c->launches_total;
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    fed_status st = eager_steps<R, TDK>(c, G);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->graph_kernels = (int)(c->launches_total - before);
    c->launches_total = before;
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
  if (!pl.conn32.empty()) {
    int32_t *q = nullptr;
    UP(upload(c, &q, pl.conn32));
    c->conn32 = reinterpret_cast<int4 *>(q);
  }
  UP(upload(c, &c->chunk_hdr, pl.chunk_hdr));
  UP(upload(c, &c->color_off, pl.color_off));
  UP(upload(c, &c->sp_list, pl.sp_list));
  UP(upload(c, &c->bc_ptr, pl.bc_ptr));
  UP(upload_real<R>(c, &c->bc_coef, pl.bc_coef));
  if (!pl.k_tab_T.empty()) {
    UP(upload_real<R>(c, &c->kt_T, pl.k_tab_T));
    UP(upload_real<R>(c, &c->kt_v, pl.k_tab_v));
  }
  if (!pl.c_tab_T.empty()) {
    UP(upload_real<R>(c, &c->ct_T, pl.c_tab_T));
    UP(upload_real<R>(c, &c->ct_v, pl.c_tab_v));
  }
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
  UP(upload(c, &c->node_global, pl.node_global));
  UP(upload(c, &c->owned, pl.node_owned));
  UP(dalloc(c, &c->d_step, 1));
  UP(dalloc(c, &c->d_fail, 1));
  UP(dalloc(c, &c->d_dTmax, 1));
  CU(cudaMemset(c->d_step, 0, sizeof(long long)));
  CU(cudaMemset(c->d_fail, 0xff, sizeof(unsigned long long)));
  if (pl.td == 2) {
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
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (auto &r : c->trec) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (cudaEvent_t e : c->tpool) cudaEventDestroy(e);
  if (c->ev_if) cudaEventDestroy(c->ev_if);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->ncomm) nccl().CommDestroy(c->ncomm);
  if (!c->dry) cudaDeviceSynchronize();
  for (void *p : c->allocs) cudaFree(p);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->comm) cudaStreamDestroy(c->comm);
  delete c;
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
  fed_ctx *c = new (std::nothrow) fed_ctx();
  if (!c) return fail(FED_ERR_NOMEM, "host allocation");
  std::string err;
  fed_status st = fed::build_plan(mesh, mat, bcs, &o, c->pl, err);
  if (st != FED_OK) {
    delete c;
    return fail(st, err);
  }
  c->dry = o.device < 0;
  c->device = o.device;
  c->graph_steps = o.graph_steps == 0 ? 16 : (o.graph_steps < 0 ? 0 : o.graph_steps);
  c->launches_per_step = (c->pl.scatter != FED_SCATTER_ATOMIC && c->pl.nranks > 1 && !c->pl.nbr_rank.empty() &&
                          c->pl.n_chunks > c->pl.n_chunks_if)
                             ? 3
                             : 2;
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
  st = c->pl.precision == 32 ? upload_all<float>(c) : upload_all<double>(c);
  if (st != FED_OK) return bail(st);
  if (c->pl.nranks > 1) {
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
      g_err = std::string("ncclCommInitRank: ") + N.GetErrorString(r);
      return bail(FED_ERR_NCCL);
    }
    if ((e = cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_if, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming)) != cudaSuccess) {
      g_err = cudaGetErrorString(e);
      return bail(FED_ERR_CUDA);
    }
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return bail(FED_ERR_CUDA);
  }
  *out = c;
  return FED_OK;
}

static fed_status check_fail(fed_ctx *c) {
  unsigned long long f = 0;
  CU(cudaMemcpyAsync(&f, c->d_fail, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (f != ULLONG_MAX) return fail(FED_ERR_UNSTABLE, "temperature became non-finite or exceeded T_abort at step " +
                                                         std::to_string((long long)f));
  return FED_OK;
}

fed_status fed_step(fed_ctx *c, int64_t n) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
  if (n < 0) return fail(FED_ERR_INVALID, "n must be >= 0");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context (device = -1) cannot step");
  CU(cudaSetDevice(c->device));
  if (n == 0) return FED_OK;
  fed_status st;
  const int td = c->pl.td;
  if (c->pl.precision == 32)
    st = td == 2 ? run_steps<float, 2>(c, n) : (td == 1 ? run_steps<float, 1>(c, n) : run_steps<float, 0>(c, n));
  else
    st = td == 2 ? run_steps<double, 2>(c, n) : (td == 1 ? run_steps<double, 1>(c, n) : run_steps<double, 0>(c, n));
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
    const bool timing = c->timing;
    const int gs = c->graph_steps;
    c->graph_steps = 0;  // eager launch with the monitor pointer set
    st = fed_step(c, 1);
    c->graph_steps = gs;
    c->monitor = false;
    (void)timing;
    done += 1;
    if (st != FED_OK) break;
    unsigned int bits = 0;
    CU(cudaMemcpyAsync(&bits, c->d_dTmax, sizeof(bits), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    std::memcpy(&last, &bits, sizeof(last));
    if (c->pl.nranks > 1) {  // max over ranks so every rank takes the same decision
      float *d = nullptr;
      CU(cudaMalloc(&d, sizeof(float)));
      CU(cudaMemcpy(d, &last, sizeof(float), cudaMemcpyHostToDevice));
      NC(nccl().AllReduce(d, d, 1, 7 /* float32 */, 2 /* ncclMax */, c->ncomm, c->stream));
      CU(cudaMemcpyAsync(&last, d, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      cudaFree(d);
    }
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
  return FED_OK;
}

static fed_status ensure_caller_buffer(fed_ctx *c) {
  if (c->d_caller) return FED_OK;
  fed_status st = dalloc(c, &c->d_caller, (size_t)c->pl.N_glob);
  if (st != FED_OK) return st;
  return dalloc(c, &c->d_bad, 1);
}

fed_status fed_get_temperature(fed_ctx *c, double *out, int64_t n_nodes) {
  if (!c || !out) return fail(FED_ERR_INVALID, "null argument");
  if (n_nodes != c->pl.N_glob) return fail(FED_ERR_INVALID, "n_nodes does not match the mesh");
  if (c->dry) return fail(FED_ERR_STATE, "dry-run context has no device state");
  const fed::Plan &pl = c->pl;
  CU(cudaSetDevice(c->device));
  fed_status st = ensure_caller_buffer(c);
  if (st != FED_OK) return st;
  // permute to caller order on the device, then one D2H copy into the caller's buffer
  unsigned grid = (unsigned)((pl.N_loc + 255) / 256);
  if (pl.nranks > 1) CU(cudaMemsetAsync(c->d_caller, 0, sizeof(double) * pl.N_glob, c->stream));
  if (pl.precision == 32)
    fed::to_caller_kernel<float><<<grid, 256, 0, c->stream>>>((const float *)c->T, c->node_global, c->owned,
                                                              c->d_caller, pl.N_loc);
  else
    fed::to_caller_kernel<double><<<grid, 256, 0, c->stream>>>((const double *)c->T, c->node_global, c->owned,
                                                               c->d_caller, pl.N_loc);
  CU(cudaGetLastError());
  if (pl.nranks > 1)
    NC(nccl().AllReduce(c->d_caller, c->d_caller, (size_t)pl.N_glob, ncclFloat64_, ncclSum_, c->ncomm, c->stream));
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
  unsigned grid = (unsigned)((pl.N_loc + 255) / 256);
  unsigned gsp = (unsigned)std::max<int64_t>(1, (pl.N_sp + 255) / 256);
  if (pl.precision == 32) {
    fed::from_caller_kernel<float><<<grid, 256, 0, c->stream>>>(c->d_caller, c->node_global, (float *)c->T,
                                                                pl.N_loc, c->d_bad);
    fed::apply_dirichlet_kernel<float><<<gsp, 256, 0, c->stream>>>((float *)c->T, c->sp_kind,
                                                                   (const float *)c->sp_dirT, pl.N_int, pl.N_sp);
  } else {
    fed::from_caller_kernel<double><<<grid, 256, 0, c->stream>>>(c->d_caller, c->node_global, (double *)c->T,
                                                                 pl.N_loc, c->d_bad);
    fed::apply_dirichlet_kernel<double><<<gsp, 256, 0, c->stream>>>((double *)c->T, c->sp_kind,
                                                                    (const double *)c->sp_dirT, pl.N_int, pl.N_sp);
  }
  CU(cudaGetLastError());
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
  return FED_OK;
}

fed_status fed_get_timing(fed_ctx *c, fed_timing *out) {
  if (!c || !out) return fail(FED_ERR_INVALID, "null argument");
  *out = c->tacc;
  return FED_OK;
}

fed_status fed_debug_plan(fed_ctx *c, int32_t *node_map, int64_t *n_slots, int32_t *slot_chunk, int32_t *slot_color,
                          int32_t *slot_elem) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
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
  const fed::Plan &pl = c->pl;
  if (n_chunks) *n_chunks = pl.n_chunks;
  if (hdr) std::memcpy(hdr, pl.chunk_hdr.data(), sizeof(int32_t) * pl.chunk_hdr.size());
  if (color_off) std::memcpy(color_off, pl.color_off.data(), sizeof(int32_t) * pl.color_off.size());
  if (conn16) std::memcpy(conn16, pl.conn16.data(), sizeof(uint16_t) * pl.conn16.size());  // [n_slots][npe]
  return FED_OK;
}

fed_status fed_debug_nodal(fed_ctx *c, double *V, double *coef, int64_t n_nodes) {
  if (!c) return fail(FED_ERR_INVALID, "null context");
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
