// internal.h -- shared declarations of the product library (host plan + device runtime).
// Not part of the ABI; include/fastdog.h is.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector_types.h>
#include <string>
#include <vector>

#include "fastdog.h"

namespace fdog {

// Successor codes of the packed topology (16-bit local index into the next
// partition P_{h+1}, or a terminal).  Def. BDD P:247-254.
constexpr uint32_t kBot = 0xFFFFu;
constexpr uint32_t kTop = 0xFFFEu;
constexpr int32_t kMaxWidth = 0xFFFD;
constexpr int kLanes = 32;  // BDDs per warp tile (one BDD per lane)
// Shapes with a partition wider than this run node-parallel, one warp per BDD
// (tile kind bit 5, kernels.cu process_bdd_coop).
constexpr int kCoopWidth = 32;
constexpr int kMaxTileRows = 128;  // rows of the widest tile (4 per lane)
constexpr int kMaxElld = 8;        // ELL-D degree groups of the averaging layout

// A distinct compiled BDD topology (many rows share one: same coefficients,
// relation and right-hand side).
struct Shape {
  int32_t k = 0;                   // hops = |I_j|
  std::vector<int32_t> hop_start;  // k+1, partition P_h = [hop_start[h], hop_start[h+1])
  std::vector<uint16_t> lo, hi;    // s^0, s^1 as local index into P_{h+1} or kBot/kTop
  int32_t max_w = 0;
  // signature (for the dedupe map)
  int8_t rel = 0;
  int64_t rhs = 0;
  std::vector<int32_t> coef;
  int32_t nodes() const { return hop_start.empty() ? 0 : hop_start.back(); }
};

// Device tile descriptor: L (= lanes, 4..32) BDDs with the same number of
// partitions K, one per lane.  Per-lane arrays use the [index][L] layout.
//   kind bit 0 clear ("shared topology"): all lanes use one Shape; topology
//          entry of node n at topo[topo_base + n]  (warp-uniform load);
//   kind bit 0 set ("per-lane topology"): entry of node n, lane l at
//          topo[topo_base + n*L + l], partitions padded to the widest lane
//          with (bottom, bottom) nodes;
//   kind bit 1 set: staged through shared memory by TMA (fits the per-warp
//          budget); clear: processed from global memory (L = 32).
//   kind bit 2 set ("arc-mask tile", staged shared-topology tiles of shapes
//          whose partitions have <= 2 nodes): the stage holds the shape's hop
//          records (HopRec, at recs + 16 * rec_base) instead of topology and
//          partition offsets; the sweeps use the branch-free min-plus form.
//   kind bit 3 set (with bit 2): every partition but the first and the last
//          is a chain hop (HopRec type 1); the sweeps fold those hops.
//   kind bit 4 set (with bit 3): the first partition is a root hop (type 2)
//          and the last a join into top (type 3); folded as well.
//   kind bit 6 set (with bit 2): the hop records are not staged; the
//          kernels read them from global memory (set by the packer for tiles
//          whose stage would not fit the budget with them; a shape's records
//          are shared by its tiles, i.e. L1 / L2-resident).  Bit 4 tiles
//          never read their records and stage none either.
//   kind bit 5 set ("cooperative", shapes wider than kCoopWidth): one BDD
//          (L = 1), processed node-parallel by a whole warp from global
//          memory; its topology is two 32-bit words per node (uint2 at
//          topo[topo_base], absolute child index, top = nodes, bottom =
//          nodes + 1): no 16-bit limit on the BDD size.
// Topology entries are absolute child indices within the tile (s^0 in the low
// 16 bits, s^1 in the high 16 bits), top = nodes, bottom = nodes + 1.
// Partition offsets of the tile: hop_off[hop_base + h], h = 0..K.
// Slot (h, lane) of the tile: slot_base + h*L + lane.
struct TileDesc {
  int64_t slot_base;
  int64_t topo_base;
  int64_t dist_base;  // distances: dist[dist_base + n*L + l], n < nodes + 2 (two sentinels)
  int32_t hop_base;
  int32_t K;
  int32_t n_lanes;  // valid lanes (<= lanes)
  int32_t kind;
  int32_t nodes;    // nodes per lane (hop_off[hop_base + K])
  int32_t max_w;    // widest partition of the tile
  int32_t lanes;    // L
  int32_t rec_base; // kind bit 2: first hop record, in 16-byte units of Plan::recs
  int32_t pair_base; // tile-closed pairs: Plan::pair_list[pair_base .. + n_pairs), each
                     // (i | m << 16): tile slot offsets i < m of one variable (|J_i| = 2)
  int32_t n_pairs;   // (64 bytes: fetched as four 16-byte cp.async chunks)
};
static_assert(sizeof(TileDesc) == 64, "TileDesc layout");

#if defined(__CUDACC__)
#define FDOG_HD __host__ __device__ __forceinline__
#else
#define FDOG_HD inline
#endif

// Shared-memory layout of one warp (identical on host and device):
//   [0, 16)                   two mbarriers
//   [16, 256)                 ring of three tile descriptors (current, next, next-but-one)
//   [256, 256 + SB)           stage buffer 0: lambda | avg->delta | distances D[nodes + 2][L] |
//                             topology | partition offsets
//   [256 + SB, 256 + 2 SB)    stage buffer 1 (NB = 2 only)
//   [256 + NB SB, + DB)       relaxation buffers R[3 (W + 1)][L]
// Recompute design (Plan::rc, narrow tiles only): the stage buffers hold no
// distances (lambda | avg->delta | topology | partition offsets), and the DB
// region is the lane-private distance scratch D[nodes + 2][L].
FDOG_HD int r16(int bytes) { return (bytes + 15) & ~15; }
FDOG_HD int stage_lam_bytes(int tsz, int K, int L) { return r16(K * L * tsz); }
FDOG_HD int stage_va_bytes(int tsz, int K, int L) { return r16(K * L * tsz); }
FDOG_HD int stage_dist_bytes(int tsz, int nodes, int L) { return r16((nodes + 2) * L * tsz); }
FDOG_HD int stage_topo_bytes(int kind, int nodes, int L) { return r16(((kind & 1) ? nodes * L : nodes) * 4); }
FDOG_HD int stage_hop_bytes(int K) { return r16((K + 1) * 4); }
// Hop record of an arc-mask tile (one per partition P_h of a shape whose
// partitions have <= 2 nodes), T = build precision:
//   A[0..3]  0-arc masks, A[4..7] 1-arc masks, entry 2 i + j = 0 if the arc
//            out of node i of P_h ends in node j of P_{h+1}, else +inf.  For
//            the last partition, j = 0 is the terminal top (bottom is never a
//            target: arcs to bottom are +inf in every column);
//   n0, n1   first node of P_h and of P_{h+1} (n1 = nodes = top on the last
//            partition), so D[n1 + j] is the distance of target j -- on the
//            last partition the sentinels (0 for top, +inf).
//   w2       1 if P_h has two nodes.
//   type     0 generic; 1..3 a specialised pattern (plan.cpp append_recs,
//            kernels.cu hop_type): the kernels then skip the masks.
FDOG_HD int rec_bytes(int tsz) { return 8 * tsz + 16; }
constexpr int kKindRecGlobal = 64;  // kind bit 6
// (arc-mask tiles: the records, unless bit 4 (never read) or bit 6 (read from
// global memory) is set)
FDOG_HD int stage_tail_bytes(int tsz, int kind, int K, int nodes, int L) {
  if (kind & 4) return (kind & (16 | kKindRecGlobal)) ? 0 : r16(K * rec_bytes(tsz));
  return stage_topo_bytes(kind, nodes, L) + stage_hop_bytes(K);
}
FDOG_HD int stage_bytes(int tsz, int kind, int K, int nodes, int L) {
  return stage_lam_bytes(tsz, K, L) + stage_va_bytes(tsz, K, L) + stage_dist_bytes(tsz, nodes, L) +
         stage_tail_bytes(tsz, kind, K, nodes, L);
}
FDOG_HD int stage_bytes_rc(int tsz, int kind, int K, int nodes, int L) {
  return stage_lam_bytes(tsz, K, L) + stage_va_bytes(tsz, K, L) + stage_tail_bytes(tsz, kind, K, nodes, L);
}
// tile-closed pair list, staged after the tail (TileDesc::n_pairs entries of 4 bytes)
FDOG_HD int stage_pairs_bytes(int n_pairs) { return r16(n_pairs * 4); }
FDOG_HD int relax_slots(int W) { return 3 * (W + 1); }
FDOG_HD int relax_bytes(int tsz, int W, int L) { return r16(relax_slots(W) * L * tsz); }
constexpr int kWarpHeader = 256;
FDOG_HD int warp_bytes(int SB, int DB, int NB) { return (kWarpHeader + NB * SB + DB + 127) & ~127; }
// Warps per sweep CTA (<= wmax, the launch bounds' 4): the count that keeps
// the most warps resident on an SM with smem_sm bytes of shared memory
// (1 KB reserved per CTA), larger CTAs on ties.  (CTAs of 4 warps of 33 KB
// each left QAP128 at 4 warps per SM where 2 or 3 per CTA fit 6.)
inline int sweep_warps_per_cta(int wb, int wmax, int smem_block, int smem_sm, int *resident = nullptr) {
  int best = 1, best_res = -1;
  for (int w = std::max(1, std::min(wmax, smem_block / std::max(wb, 1))); w >= 1; --w) {
    const int res = w * (smem_sm / (w * wb + 1024));
    if (res > best_res) {
      best_res = res;
      best = w;
    }
  }
  if (resident) *resident = best_res;
  return best;
}

// One contiguous device image of everything a solver uploads (built by the
// plan, untimed; pinned host memory when a CUDA device is present), so that
// creating a solver is one allocation and one host->device copy.
enum ImageSection {
  kImTiles = 0, kImHopOff, kImTopo, kImSlotVar, kImVarPtr, kImVarSlots, kImVarXidx, kImDegList, kImEll, kImEllVar,
  kImCsrVar, kImXLocal, kImXDeg, kImLambda0, kImDist0, kImEll4, kImEll4Var, kImRecs, kImCanon, kImPairs, kImElld,
  kImElldVar, kImCount
};

struct HostImage {
  unsigned char *data = nullptr;
  size_t bytes = 0;
  bool pinned = false;
  size_t off[kImCount] = {0};
  HostImage() = default;
  HostImage(const HostImage &) = delete;
  HostImage &operator=(const HostImage &) = delete;
  ~HostImage();
};

struct Plan {
  int32_t n_vars = 0, n_cons = 0, rank = 0, world = 1;
  std::vector<double> cost;
  std::vector<int32_t> owner;      // row -> rank
  std::vector<int32_t> row_shape;  // row -> shape id (-1: empty row or not local)
  std::vector<int64_t> row_ptr;    // copy of the problem's CSR (local rows' vars)
  std::vector<int32_t> col_var;
  std::vector<Shape> shapes;
  std::vector<int32_t> local_rows;  // ascending
  std::vector<int32_t> deg_global;  // |J_i| over all ranks
  double free_term = 0.0;           // sum_{|J_i|=0} min(c_i, 0)  (A13)
  double max_abs_cost = 0.0;

  // device layout
  std::vector<TileDesc> tiles;
  std::vector<int32_t> hop_off;
  std::vector<uint32_t> topo;       // lo | hi << 16
  std::vector<unsigned char> recs;  // hop records of arc-mask shapes (build precision, 16-byte units)
  std::vector<int32_t> slot_var;    // padded device slots: variable or -1
  std::vector<int64_t> canon_slot;  // canonical local slot -> device slot
  std::vector<int32_t> canon_con, canon_pos;
  std::vector<int32_t> var_list;    // CSR part of the averaging: variables by first device slot
  std::vector<int64_t> var_ptr;     // CSR over var_list
  std::vector<int32_t> var_slots;   // device slots, j ascending within a variable
  std::vector<int32_t> var_xidx;    // per var_list entry: index into shared_vars or -1
  std::vector<int32_t> shared_vars; // ascending global ids exchanged with other ranks
  std::vector<int32_t> deg_list;    // |J_i| (global) per var_list entry
  std::vector<int32_t> ell;         // ELL part: slot pairs (second -1 if |J_i| = 1)
  std::vector<int32_t> ell_var;     // ELL part: the variables
  int64_t n_ell_open = 0;           // ELL entries [0, n_ell_open) are averaged by the kernel; the rest
                                    // are tile-closed pairs the sweep averages on chip (pair_list)
  std::vector<uint32_t> pair_list;  // per tile with closed pairs (TileDesc::pair_base, n_pairs)
  std::vector<int32_t> ell4;        // ELL-4 part (|J_i| = 3, 4): slot quads, -1 padded
  std::vector<int32_t> ell4_var;
  // ELL-D part: frequent degrees d in [5, 32] (not exchanged), one group per d,
  // slot k of variable v at elld[elld_off[g] + k * elld_n[g] + v] (column-major:
  // a warp's index loads are coalesced; k ascending = j ascending, A1)
  std::vector<int32_t> elld;
  std::vector<int32_t> elld_var;    // the variables, group by group
  std::vector<int32_t> elld_d, elld_n;
  std::vector<int64_t> elld_off;
  std::vector<int32_t> col_coef;    // copy of the rows (feasibility checks of primal labelings)
  std::vector<int8_t> rel;
  std::vector<int64_t> rhs;
  int64_t n_vars_local = 0;         // variables with local slots (ELL + CSR)
  int64_t n_vars_shared = 0;        // of those, held by another rank too (counted once per plan)
  int64_t n_free_vars = 0;          // |J_i| = 0 (A13)
  std::vector<int32_t> x_local;     // per shared var: index into var_list or -1
  std::vector<int32_t> x_deg;       // per shared var: |J_i| (global)

  // per-warp shared-memory budget the tiles were packed for (precision-specific)
  int32_t precision = 32, SB = 0, DB = 0, NB = 2;
  int32_t host_threads = 1;         // threads of the host packing phases
  bool rc = false;                  // recompute design: tiles packed for sweep_kernel<..., RC>
  int64_t n_dist = 0;               // elements of the distance array
  int64_t direct_tiles = 0;
  int64_t n_interior_tiles = 0;     // world > 1: tiles [0, n) hold no exchanged variable (swept while
                                    // the exchange runs); the boundary tiles follow
  int64_t coop_tiles = 0;           // kind bit 5 tiles (one wide BDD each)
  int32_t coop_w = 0;               // widest partition of a cooperative tile
  int32_t direct_w = 0;             // widest partition of the other unstaged tiles
  bool coop_smem = false;           // the cooperative relaxation buffers fit the DB region
  int32_t tmem_cols = 0;            // recompute design, fp32: TMEM columns per CTA holding the distance
                                    // scratch of 32-row arc-mask tiles (0: shared memory)
  bool lifted = false;              // lifted two-sided storage (fdog_options::lifted): every tile from
                                    // global memory, every variable in the CSR averaging part

  HostImage image;                  // device image (see ImageSection)

  int64_t n_nodes = 0;              // real (unpadded) nodes on this rank
  int64_t n_slots = 0;              // real slots
  int64_t tiles_shared = 0;
  int32_t max_hops = 0, max_width = 0, max_tile_nodes = 0;
};

// compiler B on the GPU (compile_gpu.cu): every shape's k, coef, rel, rhs in,
// hop_start / lo / hi / max_w out -- identical to the host compiler;
// FDOG_ETOOBIG when a shape exceeds the GPU scratch bound (compile on the host)
fdog_status gpu_compile_shapes(std::vector<Shape> &shapes, int device);

// the packer's canonical-slot and variable phases on the GPU (pack_gpu.cu,
// FDOG_GPU_PACK=1): fills canon_slot / canon_con / canon_pos, var_list,
// var_ptr, var_slots exactly as the host phases do
fdog_status gpu_pack_slots(Plan &P, const std::vector<int64_t> &row_slot, const std::vector<int32_t> &row_L,
                           int device);

// host-side helpers implemented in plan.cpp
void set_error(const char *fmt, ...);
fdog_status build_plan(const fdog_problem *p, const fdog_options *o, Plan &plan);
fdog_status build_image(Plan &plan);

// ---- device launchers (kernels.cu) -------------------------------------
enum SweepMode { kForward = 0, kBackward = 1, kEnergy = 2, kCfr = 3 };

struct SweepArgs {
  const TileDesc *tiles;
  int32_t n_tiles;
  const int32_t *hop_off;
  const uint32_t *topo;
  const unsigned char *recs;  // hop records of arc-mask tiles
  const int32_t *slot_var;
  void *lambda;          // T*
  void *delta_out;       // T*: per slot delta out
  const void *avg_in;    // T*: per slot avg_i in (== delta_out: in place; else the delta_bar buffer
                         // holding avg_i for averaged slots and delta_bar for tile-closed pairs)
  const uint32_t *pairs; // tile-closed pair lists (null: none)
  void *m0, *m1;         // T*, recorded min-marginals (may be null)
  double omega, clamp;
  float omega_f, clamp_f;  // the same, rounded once to fp32 (fp32 kernels read them as operands)
  double *lb_part;       // per tile bound contribution (reduced by lb_reduce_kernel)
  unsigned int *done_counter;
  unsigned int *tile_counter;  // dynamic tile scheduler (reset by the last CTA)
  int32_t max_nodes, max_w, max_hops;  // over all tiles (direct-mode scratch)
  void *dist;               // T*, per-node distances (store design)
  int32_t SB, DB, NB;       // per-warp stage-buffer / relaxation budgets (bytes), stage buffers
  int32_t static_sched;     // 1: round-robin tiles only (no dynamic claims)
  int32_t pdl_early;        // 1: griddepcontrol.launch_dependents after a warp's last tile
  int32_t claim_batch;      // dynamic schedule: tiles per claim (>= 1)
  int32_t snake;            // static rounds alternate direction
  int32_t spread;           // static tiles spread over CTAs (SMs) first
  void *scratch;            // T*, [warps][scratch_stride] for direct tiles
  unsigned long long *trace;  // debug (FDOG_TRACE=1): per warp {start, end, tiles, smid}, else null
  int64_t scratch_stride;   // elements per warp
  int32_t coop_bw;          // cooperative tiles: entries per relaxation buffer (two per warp)
  int32_t coop_smem;        // 1: in the warp's DB region, 0: in scratch
  int32_t tmem_cols;        // > 0: recompute-design distances of 32-row arc-mask tiles in TMEM,
                            // columns per warp (fp32; the kernel variant rw = 0)
  void *lambda0;            // T*, lifted mode: lambda^{j,0} per slot (null otherwise)
  const void *avg0;         // T*, lifted mode: the 0-side averages per slot
};

struct AvgArgs {
  int32_t n_ell;             // variables in the ELL part (|J_i| <= 2, not exchanged)
  const int2 *ell;           // their slot pairs (y = -1 if |J_i| = 1)
  int32_t n_ell4;            // variables in the ELL-4 part (|J_i| = 3, 4, not exchanged)
  const int4 *ell4;          // their slot quads (-1 padded)
  int32_t n_elld_g;          // ELL-D groups (<= kMaxElld)
  int32_t elld_d[8], elld_n[8];  // degree and variables of group g
  int64_t elld_off[8];       // first entry of group g in elld
  const int32_t *elld;       // column-major slot indices of the ELL-D part
  int32_t n;                 // variables in the CSR part
  int32_t group;             // lanes per CSR variable (power of two <= 32)
  const int64_t *var_ptr;    // CSR over the CSR part
  const int32_t *var_slots;  // device slots, ascending j within a variable
  const int32_t *var_xidx;   // may be null (world == 1)
  const int32_t *deg_l;      // |J_i| (global) per CSR entry
  const void *delta_bar;     // T*: delta of the last pass
  void *avg_slot;            // T*: avg_i written into every slot of i (the other delta buffer)
  void *xbuf;                // T* partial sums of shared variables (may be null)
  unsigned int *tile_counter;  // sweep scheduler counter, reset here for the next sweep
  int32_t ell_v;             // ELL variables per thread (1, 2, 4 or 8; the fused path uses 4)
  int32_t ell_local;         // 1: a thread's ELL variables are consecutive (else strided by the thread count)
  int32_t csr_first;         // 1: the CSR section takes the first threads (else the last)
};

// Peer-memory exchange (kernels.cu peer_finish_kernel): the W ranks' exchange
// regions as device pointers valid in this process.
constexpr int kMaxPeers = 16;
constexpr int kRegionBuf = 256;  // first partial-sum buffer of a region
struct PeerArgs {
  int32_t world, rank;
  int64_t buf_off;                          // byte offset of this pass's buffer
  unsigned long long timeout_ns;            // wait for a peer at most this long
  const unsigned char *region[kMaxPeers];
};

struct PrimalArgs {
  int32_t n_ell, n_ell4, n_csr;
  int32_t n_elld_g;           // ELL-D groups (AvgArgs), after the CSR entries
  int32_t elld_d[8], elld_n[8];
  int64_t elld_off[8];
  const int32_t *elld, *elld_var;
  const int2 *ell;
  const int32_t *ell_var;     // variable of each ELL entry
  const int4 *ell4;
  const int32_t *ell4_var;
  const int32_t *csr_var;     // variable of each CSR entry
  const int64_t *var_ptr;
  const int32_t *var_slots;
  const void *delta_bar;      // T*
  void *lambda;               // T*
  uint8_t *x;                 // per variable
  unsigned long long *undecided;
  int32_t mode;               // 0 classify, 1 perturb
  int32_t round;
  double delta;
  uint64_t seed;
};

// Non-deferred (sequential) min-marginal averaging: one
// kernel per level of the variable schedule (solver.cpp seq_schedule); thread
// q in [q0, q1) handles the q-th variable of the pass order and all its slots.
struct SeqArgs {
  const TileDesc *tiles;
  const int32_t *hop_off;
  const uint32_t *topo;
  const int32_t *slot_tile;   // device slot -> tile
  const int64_t *ptr;         // per pass-order variable: its slots [ptr[q], ptr[q+1]) in slots
  const int32_t *slots;       // device slots, j ascending within a variable
  void *lambda;               // T*
  void *dist;                 // T*, store-design distances (shp(v,T) before a forward pass, shp(r,v) before a backward one)
  void *delta;                // T*, scratch: omega * d per slot
  void *m0, *m1;              // T*, recorded min-marginals (may be null)
  double *e_lane;             // per (tile, lane): E^j, written at the BDD's last visited partition
  double omega, clamp;
  float omega_f, clamp_f;     // the same in fp32
  int32_t forward;
};
int launch_seq_level(int precision, bool record, const SeqArgs &a, int64_t q0, int64_t q1, void *stream);
// per tile: lb_part[t] = sum over the tile's valid lanes of e_lane (fixed order)
int launch_seq_bound(const TileDesc *tiles, int32_t n_tiles, const double *e_lane, double *lb_part, void *stream);
// store-design distances of every BDD from the current lambda, in global memory:
// forward = 0: shp(v, T) (before a forward pass); 1: shp(r, v) (before a backward pass)
int launch_dist_dp(int precision, const SeqArgs &a, int32_t n_tiles, int32_t forward, void *stream);

// returns the cudaError_t as int
// rc: recompute design (sweep_kernel<..., RC = true>; plan packed with Plan::rc)
// rw: the most rows per lane of any tile (1, 2, 4; TileDesc::lanes / 32); 0:
// the TMEM variant (fp32 recompute design with SweepArgs::tmem_cols > 0)
int launch_sweep(int precision, int mode, bool record, bool rc, int rw, const SweepArgs &a, int grid, int block,
                 size_t smem, void *stream);
int launch_sweep_stream(int precision, int mode, bool record, const SweepArgs &a, void *stream);
// chunked walk of rows too long to stage whole (store design; every tile an arc-mask tile)
int launch_sweep_chunk(int precision, int mode, bool record, const SweepArgs &a, void *stream);
// lifted representation (fdog_options::lifted): both averages per slot, the
// lifted final correction, lambda^1 - lambda^0 into out
int launch_avg_lifted(int precision, const AvgArgs &a, void *avg0, void *stream);
int launch_add_deferred_lifted(int precision, int64_t n, void *lam1, void *lam0, void *delta, void *stream);
int launch_lifted_diff(int precision, int64_t n, const void *lam1, const void *lam0, void *out, void *stream);
int sweep_occupancy(int precision, int mode, bool record, bool rc, int rw, int block, size_t smem, int *blocks_per_sm);
int launch_avg(int precision, const AvgArgs &a, void *stream);
int launch_peer_signal(const PeerArgs &pa, void *stream);
int preload_kernels(int precision);
int launch_peer_finish(int precision, const AvgArgs &a, int32_t n_shared, const int32_t *xlocal,
                       const int32_t *deg_x, const PeerArgs &pa, void *stream);
int launch_avg_finish(int precision, const AvgArgs &a, int32_t n_shared, const int32_t *xlocal, const int32_t *deg_x,
                      void *stream);
int launch_add_deferred(int precision, int64_t n, void *lambda, void *delta, void *stream);
int launch_lb_reduce(const double *lb_part, int32_t n, double *out, void *stream);
// lb_part[t] += sum over tile t's slots of min(delta_bar, 0) (the A7 term after an energy sweep)
int launch_lb_deferred(int precision, const TileDesc *tiles, int32_t n_tiles, const void *delta, double *lb_part,
                       void *stream);
// smem > 0: the mutable state is copied into that many bytes of shared memory
int launch_fused_small(int precision, bool record, const SweepArgs &sa, const AvgArgs &aa, int32_t n_iter,
                       int64_t n_slots, int64_t n_dist, size_t smem, void *stream);
int launch_primal(int precision, const PrimalArgs &a, void *stream);
// top / bottom sentinel slots (0 / +inf) of every tile lane's distance column
int launch_dist_sentinels(int precision, const TileDesc *tiles, int32_t n_tiles, void *dist, void *stream);
// out[q] = src[canon[q]], q < n: per-slot state in canonical (j, h) order
int launch_gather_canon(int precision, int64_t n, const int32_t *canon, const void *src, void *out, int widen,
                        void *stream);

}  // namespace fdog
