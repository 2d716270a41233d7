/*
 * fed.h -- C ABI of the B200-native FED-FEM hot path (libfed.so).
 *
 * FED-FEM = "Fast explicit dynamics finite element algorithm for transient
 * heat transfer", Zhang & Chauhan, arXiv 1909.03355.  Citations below are
 * P:n = line n of that paper's text (/root/reference/PAPER.md, not shipped),
 * with the section / equation it falls in; readings of garbled or silent
 * passages are numbered R1..R21 in DESIGN.md ("Readings").
 *
 * The library implements the three stages of Sec. 3.5:
 *   (i)   pre-computation      -> fed_create      (host fp64, then uploaded)
 *   (ii)  initialisation       -> fed_create / fed_set_temperature
 *   (iii) time stepping        -> fed_step        (sm_100a CUDA kernels)
 * Every step is: element thermal loads F_int = sum_e G D(T) B T_e (Eqs. 11,
 * 17, 19, 20), boundary-face loads Q (Eqs. 4, 5, 7),
 * explicit nodal update T += dt / (M c(T)) (Q - F_int) (Eq. 16, sign
 * reading R1) with Dirichlet nodes held (Eq. 3; stage iii-2.3).
 *
 * General conventions
 *  - All pointers passed IN are caller-owned HOST buffers, read only during
 *    the call (deep copy); the caller may free them on return.  Output
 *    buffers are caller-owned host buffers.  The context owns every device
 *    allocation it makes and frees it in fed_destroy.
 *  - Every function returns a fed_status and never aborts; on failure
 *    fed_last_error() returns a thread-local message.
 *  - Node numbering seen by the caller is the caller's own (0-based indices
 *    into fed_mesh.xyz); internal reordering is invisible.
 *  - Temperatures are degrees Celsius, lengths metres, SI otherwise.
 *  - A context has a single owner and is not re-entrant.  With nranks > 1
 *    every rank calls every function collectively, each passing the same
 *    GLOBAL mesh; each rank keeps only its own z-slab.
 */
#ifndef FED_H_
#define FED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fed_ctx fed_ctx; /* opaque; owns all device memory */

typedef enum {
  FED_OK = 0,
  FED_ERR_INVALID = 1,  /* bad argument / option / inconsistent sizes          */
  FED_ERR_MESH = 2,     /* bad mesh: index out of range, det J <= 0, orphan node */
  FED_ERR_NOMEM = 3,    /* host or device allocation failed                    */
  FED_ERR_CUDA = 4,     /* CUDA runtime error (message has the CUDA string)    */
  FED_ERR_NCCL = 5,     /* NCCL error or NCCL unavailable with nranks > 1      */
  FED_ERR_UNSTABLE = 6, /* a temperature became non-finite or |T| > T_abort   */
  FED_ERR_STATE = 7     /* call not valid in this state (e.g. dry-run context) */
} fed_status;

/* Boundary-condition kinds of a boundary-face record. */
enum {
  FED_BC_FLUX = 1, /* Eq. 5: prescribed flux q [W/m^2], q > 0 heats the body (R11) */
  FED_BC_CONV = 2, /* Eq. 4: convection, outward flux h (T - T_inf)            */
  FED_BC_RAD = 3   /* Eq. 7: radiation, outward flux eps sigma [(T-T_z)^4 -
                      (T_inf-T_z)^4], sigma = 5.67e-8, T_z = -273.15    */
};

/* Scatter strategy of the element thermal-load loop (north_star: "chosen by
 * measurement"). */
enum {
  FED_SCATTER_AUTO = 0,   /* FED_SCATTER_CHUNK_REGC when every chunk has <= 8 colours
                             of <= 128 elements (structured-like hex meshes), else
                             FED_SCATTER_CHUNK_REG (fastest measured)  */
  FED_SCATTER_ATOMIC = 1, /* one thread per element, 8 red.global.add per element
                             into a nodal F array, separate nodal update kernel  */
  FED_SCATTER_CHUNK = 2,  /* element chunks staged in shared memory by 1-D TMA
                             (cp.async.bulk); chunk-local nodal loads accumulated
                             in shared memory by colour phases (no atomics); the
                             nodal update of chunk-interior nodes fused into the
                             element kernel; shared nodes reduced with
                             red.global.add and updated by the node kernel       */
  FED_SCATTER_CHUNK_CAS = 3, /* as CHUNK, but chunk-local accumulation by shared-
                             memory compare-and-swap adds instead of colour phases */
  FED_SCATTER_CHUNK_REG = 4, /* as CHUNK_CAS, but element records loaded straight
                             into registers instead of staged in shared memory    */
  FED_SCATTER_CHUNK_REGC = 5, /* colour phases (as CHUNK) with element records loaded
                             straight into registers, next colour prefetched      */
  /* measured baselines of the scatter choice (single rank):   */
  FED_SCATTER_ATOMIC_WARP = 6, /* as ATOMIC, elements in Morton order, the x-pair of
                             lanes (2k, 2k+1) combines the loads of its shared
                             nodes by a warp shuffle before the red.global.add    */
  FED_SCATTER_COLOR_PASSES = 7, /* mesh colouring: one launch per colour, plain
                             read-modify-write of F (no atomics); needs a globally
                             valid colouring (structured parity colours)         */
  FED_SCATTER_GATHER = 8  /* node-centric: per element the flux v_e = phi P S^T T_e
                             (3 words), then per node a gather over its incident
                             (element, corner) pairs; deterministic, no atomics   */
};

/* Interface exchange between z-slab ranks (nranks > 1 or local_ranks > 1). */
enum {
  FED_TRANSPORT_NCCL = 0, /* after the interface chunks, ncclSend/ncclRecv of the
                             interface partial loads on a second stream, overlapped
                             with the interior chunks; combined by the node kernel */
  FED_TRANSPORT_PEER = 1  /* fused exchange over peer memory: the interface-chunk
                             launch reduces into a step-parity buffer and its last
                             CTA raises a step flag in each neighbour's memory; the
                             node kernel of the neighbour waits for the flag and
                             loads the partial loads straight from this rank's
                             memory (NVLink P2P, CUDA IPC mapping made at create
                             through NCCL).  No host-side collective per step.  Needs
                             a CHUNK scatter strategy                              */
};

/* Mesh: 8-node reduced-integration hexahedra (Eq. 17, Sec. 3.2) or
 * 4-node linear tetrahedra (Eq. 18). */
typedef struct {
  int64_t n_nodes, n_elems, n_faces;
  const double *xyz;      /* [n_nodes][3] node coordinates, metres                   */
  const int32_t *conn;    /* [n_elems][nodes_per_elem] 0-based node ids.  hex8 corner
                             order: bottom face counter-clockwise seen from +zeta,
                             then the top face (natural signs (---),(+--),(++-),
                             (-+-),(--+),(+-+),(+++),(-++)); det J at the centre
                             must be > 0.  tet4: positively oriented (volume > 0). */
  const int32_t *faces;   /* [n_faces][nodes_per_face] boundary faces (planar), any
                             corner order; may be NULL if n_faces == 0             */
  const int32_t *face_bc; /* [n_faces] index into fed_bcs.face_bcs, or -1 (adiabatic,
                             Eq. 6)                                                */
  int32_t nodes_per_elem; /* 8 (hex8) or 4 (tet4); 0 means 8                        */
  int32_t nodes_per_face; /* 4 (quads) or 3 (triangles); 0 means 4 for hex8, 3 for
                             tet4.  Each face corner receives A_f / nodes_per_face */
} fed_mesh;

/* Material (Eq. 1): rho constant, c(T) and k(T) linear in T (R8).
 * c(T) = c0 (1 + beta_c T);  D(T) = D_ref (1 + beta_k T).  The element
 * conductivity is the average of the nodal values (R6); c is taken at
 * each node's own temperature (Eq. 16, R7).  beta_c = beta_k = 0 is
 * the temperature-independent (TI) path of Sec. 3.3 (Eqs. 21-24). */
typedef struct {
  double rho;      /* kg/m^3, > 0                                             */
  double c0;       /* J/(kg K), > 0                                           */
  double beta_c;   /* 1/K                                                     */
  double D_ref[6]; /* conductivity tensor xx, yy, zz, xy, yz, xz  W/(m K), SPD */
  double beta_k;   /* 1/K                                                     */
  /* Tabulated properties ("linear interpolation between points"; NEXT-2).
   * n = 0: unused.  Otherwise 1..32 points, temperatures strictly increasing
   * (degC), values > 0, linear in between, clamped to the end values outside.
   * k table: D(T) = D_ref * k_tab(T) (replaces 1 + beta_k T);
   * c table: c(T) = c_tab(T) J/(kg K) (replaces c0 (1 + beta_c T)).
   * Pointers are read during fed_create only. */
  int32_t n_k_table;
  const double *k_table_T, *k_table_val;
  int32_t n_c_table;
  const double *c_table_T, *c_table_val;
} fed_material;

typedef struct {
  int32_t kind;      /* FED_BC_FLUX | FED_BC_CONV | FED_BC_RAD                    */
  double q;          /* W/m^2           (FLUX)                                    */
  double h;          /* W/(m^2 K)       (CONV)                                    */
  double T_inf;      /* degC            (CONV, RAD)                               */
  double eps;        /* emissivity      (RAD)                                     */
  int32_t area_mode; /* 0: each face corner gets A_f / nodes_per_face (R9);
                        1: the paper's concentrated loads (NEXT-3):
                        every unique node of the record's faces gets
                        (sum of the record's face areas) / (#unique nodes)     */
} fed_face_bc;

/* Boundary conditions and initial state. */
typedef struct {
  int32_t n_face_bcs;
  const fed_face_bc *face_bcs; /* [n_face_bcs]                                   */
  int64_t n_dirichlet;
  const int32_t *dir_nodes;    /* [n_dirichlet] node ids held at dir_T (Eq. 3);
                                  Dirichlet wins over any face load (R12)         */
  const double *dir_T;         /* [n_dirichlet] degC                             */
  const double *q_vol;         /* [n_nodes] volumetric source W/m^3 at the nodes
                                  (nodal quadrature Q_n = q_vol(x_n) V_n), or NULL */
  const double *T0;            /* [n_nodes] initial field degC, or NULL (= 0)     */
} fed_bcs;

typedef struct {
  int32_t precision;     /* 32 or 64: storage and arithmetic type of the step   */
  double dt;             /* > 0: use exactly this step (seconds);
                            <= 0: dt = dt_factor * dt_crit; NaN or an infinite
                            result: FED_ERR_INVALID                               */
  double dt_factor;      /* default 0.9                                          */
  double T_lo, T_hi;     /* temperature range over which dt_crit is evaluated for
                            temperature-dependent materials (R13)                 */
  double T_abort;        /* |T| above this marks the run unstable (default 1e6)  */
  int32_t device;        /* CUDA device ordinal; -1 = dry run: plan + precompute
                            on the host only (no GPU, fed_step -> FED_ERR_STATE)  */
  void *stream;          /* cudaStream_t to launch on, or NULL (library-owned)   */
  int32_t rank, nranks;  /* z-slab domain decomposition over nranks GPUs         */
  const void *nccl_id;   /* 128-byte ncclUniqueId (from fed_nccl_unique_id on rank
                            0, broadcast by the caller), required if nranks > 1   */
  int32_t scatter;       /* FED_SCATTER_*                                        */
  int32_t chunk_elems;   /* elements per chunk (CHUNK scatter), 0 = auto         */
  int32_t graph_steps;   /* steps captured per CUDA graph, 0 = auto, <0 = off    */
  int32_t transport;     /* FED_TRANSPORT_* (default NCCL)                        */
  int32_t local_ranks;   /* > 1: ONE context holds local_ranks z-slab ranks of the
                            mesh on ONE device (requires nranks == 1) -- the
                            partitioned path of nranks = local_ranks GPUs, run on
                            one GPU for testing and per-rank timing.  Every slab is
                            planned, stored and stepped exactly as on its own GPU;
                            the exchange is a device copy of the slices ncclSend
                            would deliver (NCCL) or the same peer-load node kernel
                            on same-device pointers (PEER).  All slabs' kernels
                            run in one stream in an order where no kernel ever
                            waits for another.  0 or 1: off                     */
  int32_t resident;      /* resident mode (single rank, hex8 meshes whose chunks all
                            fit on the GPU at once): ONE cooperative launch runs all
                            n steps of fed_step; each CTA keeps its chunk's records
                            in registers and its nodes in shared memory, and steps
                            are ordered by per-chunk dataflow (a chunk waits only for
                            the chunks sharing nodes with it) instead of kernel
                            boundaries.  0 = auto (used when possible and timing is
                            off), 1 = required (fed_create fails if impossible),
                            -1 = off.  Auto chunk sizing prefers chunks that fit  */
  /* Device-memory hook (stage i data placement): when dev_alloc is
   * non-NULL every device buffer of the context is obtained from
   * dev_alloc(bytes, device, alloc_ctx) and returned with dev_free(ptr, bytes,
   * device, alloc_ctx) in fed_destroy (e.g. a PyTorch caching allocator), except
   * the PEER exchange block, which must be a cudaMalloc allocation of its own
   * because it is shared by CUDA IPC.  dev_alloc returning NULL fails the call
   * with FED_ERR_NOMEM.  Both NULL: cudaMalloc / cudaFree. */
  void *(*dev_alloc)(size_t bytes, int32_t device, void *alloc_ctx);
  void (*dev_free)(void *ptr, size_t bytes, int32_t device, void *alloc_ctx);
  void *alloc_ctx;
  double wait_timeout_s; /* bound on every device-side wait (PEER neighbour flags,
                            resident-mode chunk dependencies): a wait longer than
                            this sets an error flag instead of hanging the GPU and
                            the call returns FED_ERR_NCCL / FED_ERR_CUDA (state
                            undefined).  <= 0: 10 s                              */
  int32_t chunk_order;   /* launch order of the element chunks: 0 = layer-major (z
                            layer, y row, x of the chunk's mean cell; default: chunks
                            sharing nodes run close together, so the shared nodes'
                            lines are still in L2 for the second toucher), 1 = the
                            Morton order the chunks are cut in (measured baseline) */
} fed_options;

typedef struct {
  double dt;            /* step used                                          */
  double dt_crit;       /* element-bound critical step over [T_lo, T_hi] (R13)  */
  int64_t step;         /* steps taken so far                                 */
  double t;             /* step * dt (never summed)                     */
  int64_t fail_step;    /* first step whose update went unstable, or -1       */
  int32_t precision, scatter, rank, nranks;
  int32_t temperature_dependent;          /* 0 TI; 1 linear laws; 2 tables (> 2 points);
                                             3 tables of <= 2 points (clamped linear) */
  int64_t n_nodes_global, n_elems_global;
  int64_t n_nodes_local, n_elems_local;   /* this rank's slab                  */
  int64_t n_interior, n_special;          /* chunk-interior / shared+BC nodes   */
  int64_t n_interface;                    /* nodes shared with other ranks      */
  int64_t n_chunks, n_chunks_interface;
  int64_t n_bc_entries;                   /* (node, face-bc) pairs              */
  int32_t max_colors, chunk_elems;
  int64_t kernel_launches_per_step;       /* element + node launches per step    */
  int64_t kernel_launches_total;          /* kernels launched by fed_step so far,
                                             incl. one step-counter advance per batch */
  int64_t device_bytes;                   /* device memory owned by the context */
  int32_t nodes_per_elem;                 /* 8 (hex8) or 4 (tet4)               */
  int32_t colored;                        /* element colours valid (0: CAS only) */
  int32_t resident;                       /* 1 if fed_step runs in resident mode   */
} fed_info;

/* Per-kernel device time accumulated while timing is enabled (CUDA events on
 * the launching stream; fed_step then launches without CUDA graphs). */
typedef struct {
  double element_ms;    /* element thermal-load kernel(s), summed            */
  double node_ms;       /* node update kernel, summed                        */
  double exchange_ms;   /* interface exchange (nranks > 1), summed           */
  int64_t element_launches, node_launches, exchange_count;
} fed_timing;

/* Fill *opts with defaults: precision 64, dt = 0 (0.9 x critical), T range
 * [0, 0], T_abort 1e6, device 0, no stream, rank 0 of 1, scatter AUTO,
 * transport NCCL, no local rank group, cudaMalloc, 10 s wait bound. */
void fed_options_default(fed_options *opts);

/* Stages (i) and (ii) of Sec. 3.5: validate the mesh (index range, det J > 0
 * at every element centre, every node used by an element), compute per element
 * the compact operator P_e = (det J / 8) J^-T D_ref J^-1 (equivalent to
 * G D B of Eqs. 17/19/20), lumped volumes V_n (equal split, R3), coefficients
 * dt / (rho c0 V_n) (Eqs. 14/21), face tributary areas, the critical step
 * (Eq. 29, R13), reorder/partition/colour for the device, upload, set
 * T = T0 and Dirichlet values.  On success *out owns everything.
 * With nranks > 1 the call is collective: the NCCL communicator is created
 * first, and after every rank's fallible set-up (upload, PEER IPC mapping) the
 * ranks agree on the outcome, so either every rank succeeds or every rank
 * fails (a rank whose own set-up succeeded returns FED_ERR_STATE, "fed_create
 * failed on another rank"). */
fed_status fed_create(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs,
                      const fed_options *opts, fed_ctx **out);

/* Stage (iii): advance n >= 0 explicit steps (blocking until done).  Returns
 * FED_ERR_UNSTABLE if any update produced |T| > T_abort or a non-finite
 * value; fed_get_info reports the first such step.  With nranks > 1 the call
 * is collective; under FED_TRANSPORT_PEER it starts with a one-word NCCL
 * all-reduce on the context's stream, so no rank's kernels of this call run
 * before every rank has entered it (the per-step flag waits inside the call are
 * then bounded by the step time, not by host-side skew). */
fed_status fed_step(fed_ctx *ctx, int64_t n);

/* Steady-state mode (NEXT-4; the paper's criterion "Delta T <= 0.001 degC",
 * P:248): advance in batches of check_every steps; the last step of each batch
 * measures max_n |T_n^{k+1} - T_n^k| on the device (max over ranks); stop when
 * it is <= tol or after max_steps steps.  *steps_taken (may be NULL) receives
 * the number of steps advanced, *last_max_dT (may be NULL) the last measured
 * change (degC).  Errors as fed_step. */
fed_status fed_run_until_steady(fed_ctx *ctx, double tol, int64_t max_steps, int64_t check_every,
                                int64_t *steps_taken, double *last_max_dT);

/* Copy the current temperatures (fp64, caller numbering) into out[n_nodes]
 * (n_nodes must equal fed_mesh.n_nodes).  With nranks > 1 every rank receives
 * the full global field: each rank packs the nodes it owns (a node on a slab
 * interface belongs to the lower rank) and one ncclAllGather of the packed
 * slices delivers them to every rank (collective: all ranks must call). */
fed_status fed_get_temperature(fed_ctx *ctx, double *out, int64_t n_nodes);

/* Overwrite the temperature field from T[n_nodes] (caller numbering);
 * Dirichlet nodes keep their prescribed values. */
fed_status fed_set_temperature(fed_ctx *ctx, const double *T, int64_t n_nodes);

fed_status fed_get_info(fed_ctx *ctx, fed_info *out);

/* Enable (1) / disable (0) per-kernel CUDA-event timing and reset counters. */
fed_status fed_set_timing(fed_ctx *ctx, int32_t enable);
fed_status fed_get_timing(fed_ctx *ctx, fed_timing *out);

/* Per-rank kernel times of a local_ranks group (rank in [0, local_ranks)); for
 * a single-rank context rank must be 0 (same as fed_get_timing). */
fed_status fed_get_rank_timing(fed_ctx *ctx, int32_t rank, fed_timing *out);

/* Per-rank cost of a local rank group (timing only): replays n_steps of slab
 * `rank`'s own kernel sequence ALONE in a CUDA graph -- what that rank launches
 * on its own GPU, without waiting for its neighbours (PEER flag waits skipped;
 * NCCL slices copied from whatever the neighbours' buffers hold) -- and writes
 * the CUDA-event time per step.  The field is undefined afterwards: later
 * fed_step calls on the context fail with FED_ERR_STATE. */
fed_status fed_debug_time_rank(fed_ctx *ctx, int32_t rank, int64_t n_steps, double *ms_per_step);

/* Write a fresh 128-byte NCCL unique id into out128 (rank 0 only).  Returns
 * FED_ERR_NCCL if libnccl.so.2 cannot be loaded. */
fed_status fed_nccl_unique_id(void *out128);

/* Host-side plan inspection (valid for dry-run and device contexts), for
 * tests.  Copies out: the internal id of every caller node (-1 if not on this
 * rank) into node_map[n_nodes_global]; and for every local element slot its
 * chunk, colour and caller element id (-1 for padding) into the three arrays
 * of length n_slots (query n_slots with all pointers NULL). */
fed_status fed_debug_plan(fed_ctx *ctx, int32_t *node_map, int64_t *n_slots, int32_t *slot_chunk,
                          int32_t *slot_color, int32_t *slot_elem);

/* Chunk tables of the plan: *n_chunks, then (if non-NULL) the chunk headers
 * hdr[n_chunks][8] = {slot offset, #elements, #slots, first interior node,
 * #interior nodes, special-list offset, #special nodes, #colours}, colour
 * offsets color_off[n_chunks][33] and chunk-local connectivity
 * conn16[n_slots][nodes_per_elem]. */
fed_status fed_debug_chunks(fed_ctx *ctx, int64_t *n_chunks, int32_t *hdr, int32_t *color_off, uint16_t *conn16);

/* Multi-rank readout layout (nranks > 1, for tests): *nranks, then (if
 * non-NULL) off[nranks + 1] (slice boundaries), ids[n_nodes_global] (caller ids,
 * slice r = the nodes rank r owns, increasing), and this rank's pack list
 * own_pack[off[rank + 1] - off[rank]] (internal ids in its slice order). */
fed_status fed_debug_gather(fed_ctx *ctx, int32_t *nranks, int64_t *off, int32_t *ids, int32_t *own_pack);

/* Host-side precompute inspection: lumped volume V_n and the coefficient
 * dt/(rho c0 V_n) per caller node (nodes not on this rank: NaN). */
fed_status fed_debug_nodal(fed_ctx *ctx, double *V, double *coef, int64_t n_nodes);

/* Dataflow tables of resident mode (host-side, for tests): chunk adjacency
 * in CSR form (chunks sharing at least one node; query sizes with NULL arrays:
 * *n_chunks, *n_adj), the shared-node lists of every chunk as in the chunk header
 * (sp_list[n_sp_total], -1 = hole) and, parallel to it, sp_own (1 = the chunk
 * owns the node).  Empty (sizes 0) when the plan has no dataflow tables. */
fed_status fed_debug_dataflow(fed_ctx *ctx, int64_t *n_chunks, int64_t *n_adj, int64_t *n_sp_total,
                              int32_t *adj_ptr, int32_t *adj, int32_t *sp_list, uint8_t *sp_own);

/* Thread-local message of the last failure on this thread ("" if none). */
const char *fed_last_error(void);

/* Release everything; fed_destroy(NULL) is a no-op. */
void fed_destroy(fed_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* FED_H_ */
