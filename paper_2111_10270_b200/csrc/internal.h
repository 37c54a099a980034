// internal.h -- shared declarations of the product library (host plan + device runtime).
// Not part of the ABI; include/fastdog.h is.
#pragma once
#include <cstdint>
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

// Device tile descriptor: 32 BDDs with the same number of hops K, one per lane.
//   kind 0 ("shared topology"): all lanes use one Shape, topology entry of node n
//          at topo[topo_base + n]  (warp-uniform load);
//   kind 1 ("per-lane topology"): entry of node n, lane l at
//          topo[topo_base + n*32 + l]  (coalesced), partitions padded to the
//          widest lane with (bot, bot) nodes.
// Partition offsets of the tile: hop_off[hop_base + h], h = 0..K.
// Slot (h, lane) of the tile: slot_base + h*32 + lane.
struct TileDesc {
  int64_t slot_base;
  int64_t topo_base;
  int32_t hop_base;
  int32_t K;
  int32_t n_lanes;
  int32_t kind;
  int32_t nodes;   // nodes per lane (hop_off[hop_base + K])
  int32_t max_w;   // widest partition of the tile
};
static_assert(sizeof(TileDesc) == 40, "TileDesc layout");

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
  std::vector<int32_t> slot_var;    // padded device slots: variable or -1
  std::vector<int64_t> canon_slot;  // canonical local slot -> device slot
  std::vector<int32_t> canon_con, canon_pos;
  std::vector<int32_t> var_list;    // variables with local slots, ascending
  std::vector<int64_t> var_ptr;     // CSR over var_list
  std::vector<int32_t> var_slots;   // device slots, j ascending within a variable
  std::vector<int32_t> var_xidx;    // per var_list entry: index into shared_vars or -1
  std::vector<int32_t> shared_vars; // ascending global ids exchanged with other ranks

  int64_t n_nodes = 0;              // real (unpadded) nodes on this rank
  int64_t n_slots = 0;              // real slots
  int64_t tiles_shared = 0;
  int32_t max_hops = 0, max_width = 0, max_tile_nodes = 0;
};

// host-side helpers implemented in plan.cpp
void set_error(const char *fmt, ...);
fdog_status build_plan(const fdog_problem *p, const fdog_options *o, Plan &plan);

// ---- device launchers (kernels.cu) -------------------------------------
enum SweepMode { kForward = 0, kBackward = 1, kEnergy = 2 };

struct SweepArgs {
  const TileDesc *tiles;
  int32_t n_tiles;
  const int32_t *hop_off;
  const uint32_t *topo;
  const int32_t *slot_var;
  void *lambda;          // T*
  const void *avg;       // T*, indexed by global variable
  void *delta_out;       // T*
  void *m0, *m1;         // T*, recorded min-marginals (may be null)
  double omega, clamp;
  double *lb_part;       // per tile
  double *lb_out;        // final (written by the last CTA)
  unsigned int *done_counter;
  int32_t max_nodes, max_w, max_hops;
};

struct AvgArgs {
  int32_t n;                 // entries of var_list
  const int32_t *var_list;
  const int64_t *var_ptr;
  const int32_t *var_slots;
  const int32_t *var_xidx;   // may be null (world == 1)
  const int32_t *deg;        // |J_i| global, indexed by variable
  const void *delta_bar;     // T*
  void *avg;                 // T*
  void *xbuf;                // T* partial sums of shared variables (may be null)
};

// returns the cudaError_t as int
int launch_sweep(int precision, int mode, bool record, const SweepArgs &a, int grid, int block,
                 size_t smem, void *stream);
int sweep_smem_bytes(int precision, int max_nodes, int max_w, int max_hops, int warps);
int sweep_occupancy(int precision, int mode, bool record, int block, size_t smem, int *blocks_per_sm);
int launch_avg(int precision, const AvgArgs &a, void *stream);
int launch_avg_finish(int precision, int32_t n_shared, const int32_t *shared_vars, const int32_t *deg,
                      const void *xbuf, void *avg, void *stream);
int launch_add_deferred(int precision, int64_t n, void *lambda, void *delta, void *stream);
int launch_fill(int precision, int64_t n, void *dst, double value, void *stream);

}  // namespace fdog
