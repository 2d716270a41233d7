// fed_plan.h -- host-side plan of the B200 FED-FEM path (internal header).
//
// The plan is everything fed_create computes on the host before uploading:
// validation, the fp64 pre-computation of Sec. 3.5 stage (i),
// the z-slab partition (nranks > 1), the locality reorder, element chunks +
// colours for the shared-memory scatter, and the node classification that
// lets the element kernel update chunk-interior nodes in place.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fed.h"

namespace fed {

constexpr int kMaxColors = 32;        // colours per chunk (hex: <= 27 needed)
constexpr int kChunkHdr = 16;         // int32 words per chunk header (64 B, one load per CTA)
constexpr int kChunkHdrPublic = 8;    // words per header exposed by fed_debug_chunks

// chunk header layout (int32 words); words 8..15 = colour offsets 1..8 (colour 0
// starts at slot 0), so the element kernel's fast path needs no second table load
enum { CH_ELEM_OFF = 0, CH_N_ELEM = 1, CH_N_PAD = 2, CH_INT_START = 3, CH_N_INT = 4,
       CH_SP_OFF = 5, CH_N_SP = 6, CH_N_COLORS = 7, CH_COLOR_OFF1 = 8 };

inline int max_local_nodes(int chunk) { return chunk + chunk / 2 + 128; }

// scatter strategies without chunk kernels (global node arrays, conn32)
inline bool atomic_family(int sc) {
  return sc == FED_SCATTER_ATOMIC || sc == FED_SCATTER_ATOMIC_WARP || sc == FED_SCATTER_COLOR_PASSES ||
         sc == FED_SCATTER_GATHER;
}

struct Plan {
  int sm_count = 148;     // input: SMs of the target device (auto chunk sizing)
  bool want_gather = true;  // input: build the multi-rank readout layout (not for local rank groups)
  // problem
  int precision = 64;
  int td = 0;  // 0 TI, 1 linear k(T)/c(T) laws, 2 general tables (NEXT-2), 3 clamped-linear (tables of <= 2 points)
  // td 3: k(T)/k_ref = kl[2] + kl[3] (clamp(T, kl[0], kl[1]) - kl[4]), c(T) = cl[2] + cl[3] (clamp(T, cl[0], cl[1]) - cl[4])
  double kl[5] = {0, 0, 0, 0, 0}, cl[5] = {0, 0, 0, 0, 0};
  int npe = 8, npf = 4;   // nodes per element (8 hex8 | 4 tet4) / per boundary face
  int colored = 1;        // element colours valid (0: compare-and-swap modes only)
  int rank = 0, nranks = 1;
  int scatter = FED_SCATTER_CHUNK;
  int chunk_elems = 1024;
  int max_local = 0;        // capacity used to build chunks
  int max_local_used = 8;   // max over chunks of padded local node count (sizes shared memory)
  int max_int_used = 8;     // max over chunks of the padded interior range (coef / Q staging)
  int max_sp_used = 8;      // max over chunks of the shared-node list length (4-padded, 8-rounded)
  double rho = 0, c0 = 0, beta_c = 0, beta_k = 0, D_ref[6] = {0, 0, 0, 0, 0, 0};
  double dt = 0, dt_crit = 0, T_abort = 1e6;
  std::vector<double> k_tab_T, k_tab_v, c_tab_T, c_tab_v;  // NEXT-2 tables (may be empty)
  int64_t N_glob = 0, E_glob = 0;

  // local nodes: internal ids [0, N_int) chunk-interior, [N_int, N_loc) special
  int64_t N_loc = 0, N_int = 0, N_sp = 0;
  int64_t n_if = 0, n_if_lo = 0;            // interface specials are s in [0, n_if)
  std::vector<int32_t> node_global;         // [N_loc] -> caller id
  std::vector<int32_t> node_map;            // [N_glob] caller id -> internal id or -1
  std::vector<uint8_t> node_owned;          // [N_loc] 1 if this rank reports the node
  // multi-rank readout (nranks > 1): a node belongs to the lowest rank touching it.
  // Rank r's owned caller ids in increasing order form slice r of gather_ids
  // ([gather_off[r], gather_off[r+1])); own_pack lists this rank's internal ids in
  // the order of its own slice.
  std::vector<int32_t> gather_ids;          // [N_glob]
  std::vector<int64_t> gather_off;          // [nranks + 1]
  std::vector<int32_t> own_pack;            // [gather_off[rank+1] - gather_off[rank]]

  // element slots (chunk-major, colour-sorted inside a chunk, padded)
  int64_t E_loc = 0, n_slots = 0;
  std::vector<int32_t> slot_elem;           // [n_slots] caller element id or -1
  std::vector<int32_t> slot_chunk, slot_color;
  std::vector<uint16_t> conn16;             // [n_slots][8] chunk-local node index
  std::vector<int32_t> conn32;              // [n_slots][8] internal node id (-1 pad)
  std::vector<double> P;                    // [6][n_slots] compact operator
  // FED_SCATTER_COLOR_PASSES: slots grouped by colour (cp_off[k] .. cp_off[k+1])
  std::vector<int32_t> cp_list, cp_off;
  // FED_SCATTER_GATHER: per internal node its incident (slot << 3 | corner) entries
  std::vector<int32_t> g_ptr, g_list;

  // chunks
  int64_t n_chunks = 0, n_chunks_if = 0;    // interface-touching chunks come first
  int max_colors_used = 0;
  std::vector<int32_t> chunk_hdr;           // [n_chunks][kChunkHdr]
  std::vector<int32_t> color_off;           // [n_chunks][kMaxColors+1] slot offsets
  std::vector<int32_t> sp_list;             // special indices per chunk (-1 = hole), 4-aligned per chunk

  // nodes
  std::vector<double> V;                    // [N_loc] lumped volume
  std::vector<double> coef;                 // [N_loc] dt / (rho c0 V)
  std::vector<double> Qvol;                 // [N_loc] q_vol(x) V  (empty if none)
  std::vector<double> T0;                   // [N_loc]

  // special-node boundary data
  std::vector<int32_t> bc_ptr;              // [N_sp + 1]
  std::vector<int32_t> bc_idx;              // [n_bc_entries] face-BC record
  std::vector<double> bc_area;              // [n_bc_entries] sum_f A_f / 4
  std::vector<double> bc_coef;              // [n_bc_entries] area x (q | h | eps sigma)
  std::vector<double> bc_tinf;              // [n_bc_entries]
  std::vector<int8_t> bc_ekind;             // [n_bc_entries]
  std::vector<uint8_t> sp_dir;              // [N_sp] 1 = Dirichlet
  std::vector<uint8_t> sp_kind;             // [N_sp] 0 plain, 1 face-BC entries, 2 Dirichlet
  std::vector<double> sp_dirT;              // [N_sp]
  std::vector<int32_t> bc_kind;
  std::vector<double> bc_q, bc_h, bc_Tinf, bc_eps;

  // resident mode (small meshes, one rank): chunk adjacency (chunks sharing a node) and,
  // parallel to sp_list, 1 where the chunk owns the shared node (lowest touching chunk)
  std::vector<int32_t> chunk_nbr_ptr, chunk_nbr;
  std::vector<uint8_t> sp_own;
  // neighbours (nranks > 1): specials [nbr_off[i], nbr_off[i]+nbr_cnt[i]) shared with nbr_rank[i]
  std::vector<int32_t> nbr_rank, nbr_off, nbr_cnt;
};

// Build the plan. Returns FED_OK or an error status with a message in err.
fed_status build_plan(const fed_mesh *mesh, const fed_material *mat, const fed_bcs *bcs,
                      const fed_options *opts, Plan &plan, std::string &err);

// Largest eigenvalue of a symmetric 3x3 matrix (closed trigonometric form).
double sym3_max_eig(const double a[3][3]);

}  // namespace fed
