// solver.cpp -- device runtime of the hot path and the solver half of the C ABI.
//
// fdog_iterate(n, omega) enqueues, per pass (A2):
//     avg_kernel (deferred averaging)  [+ ncclAllReduce + avg_finish, world > 1]
//  -> sweep_kernel<forward|backward>          (min-marginals, dual update, bound)
//  -> swap(delta_bar, delta_new)              (mbar <- m)
// all stream-ordered, no host synchronisation.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.h"

namespace fdog {
std::shared_ptr<const Plan> plan_of(const fdog_plan *p);
}

using namespace fdog;

namespace {

// ---- minimal NCCL surface, resolved with dlopen (world > 1 only) --------
typedef struct {
  char internal[128];
} nccl_uid;
typedef void *nccl_comm;
typedef int (*nccl_init_fn)(nccl_comm *, int, nccl_uid, int);
typedef int (*nccl_allreduce_fn)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*nccl_destroy_fn)(nccl_comm);
typedef const char *(*nccl_errstr_fn)(int);
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0;

struct Nccl {
  void *lib = nullptr;
  nccl_init_fn init = nullptr;
  nccl_allreduce_fn allreduce = nullptr;
  nccl_destroy_fn destroy = nullptr;
  nccl_errstr_fn errstr = nullptr;
  nccl_comm comm = nullptr;
};

enum KernelId { kKSweepFwd = 0, kKSweepBwd, kKEnergy, kKAvg, kKAvgFinish, kKAllreduce, kKAddDeferred, kKLbReduce, kKPrimal, kKCount };
const char *kKernelNames[kKCount] = {"sweep_forward", "sweep_backward", "sweep_energy", "avg", "avg_finish",
                                     "nccl_allreduce", "add_deferred", "lb_reduce", "primal"};

struct EventRec {
  int kernel;
  cudaEvent_t a, b;
};

}  // namespace

struct fdog_solver {
  int precision = 32;
  int device = 0;
  size_t tsz = 4;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // caller-owned device memory (fdog_options::dev_alloc); allocs come from it
  void *(*dev_alloc)(size_t, int32_t, void *, void *) = nullptr;
  void (*dev_free)(void *, int32_t, void *, void *) = nullptr;
  void *alloc_ctx = nullptr;
  std::vector<void *> own_allocs;  // cudaMalloc'ed regardless (the IPC-mapped exchange region)
  bool record_mm = false;
  bool profile = false;
  double clamp = 0.0;
  int rank = 0, world = 1;
  bool external = false;  // world > 1 without NCCL: the caller performs the exchange
  // peer-memory exchange (fdog_set_peer_regions; external mode only): this
  // rank's region (pass counter, error word, two partial-sum buffers) and the
  // peers' regions as device pointers valid in this process
  unsigned char *d_region = nullptr;
  size_t region_stride = 0;  // bytes per partial-sum buffer
  bool peer = false;
  int32_t peer_par = 0;      // parity of the next pass's buffer
  // world > 1: the exchange of a pass runs on xstream while the interior tiles
  // [0, n_int) sweep on stream; the boundary tiles wait for it
  int64_t n_int = 0;
  bool overlap_ok = true;
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  PeerArgs peer_args{};
  bool stream_mode = false;  // forward/backward passes use sweep_stream_kernel
  int rw = 1;                // most rows per lane of any tile (sweep_kernel instantiation)
  int32_t tmem_cols = 0;     // TMEM columns per sweep CTA (recompute design, fp32; Plan::tmem_cols)
  bool lifted = false;       // lifted two-sided storage: d_lambda = lambda^{j,1}
  void *d_lam0 = nullptr;    // lambda^{j,0} per device slot
  void *d_avg0 = nullptr;    // 0-side averages per device slot
  void *d_lam_out = nullptr; // lambda^1 - lambda^0 (getter scratch)
  int32_t coop_bw = 0;       // cooperative tiles: relaxation buffer entries
  bool coop_smem = false;
  int64_t n_coop = 0;
  bool chunk_mode = false;   // ... or sweep_chunk_kernel (every tile an arc-mask tile)
  bool rc = false;           // recompute design (Plan::rc): no distance traffic, no dist_state
  bool dbar_zero = true;     // delta_bar == 0 (fresh, finalized, set_state with 0, or after a _seq pass)
  int32_t ell_v = 4;         // averaging: ELL variables per thread (measured best of 1, 2, 4, 8)
  int32_t ell_local = 0;     // averaging: a thread's ELL variables strided by the thread count (consecutive: slower)
  int32_t csr_first = 1;     // averaging: CSR section in the first blocks (its chains are the longest)
  bool get_direct = true;    // getters: widen to fp64 on the device, one D2H (host widening measured slower)
  // non-deferred variant (fdog_pass_seq): level schedule, built on first use
  bool seq_ready = false;
  std::vector<int64_t> seq_lvl[2];        // [backward, forward]: level boundaries in pass order
  int64_t *d_seq_ptr[2] = {nullptr, nullptr};
  int32_t *d_seq_slots[2] = {nullptr, nullptr};
  int32_t *d_slot_tile = nullptr;
  double *d_e_lane = nullptr;
  int32_t static_sched = 0;  // TMA sweep: round-robin tiles only
  int32_t pdl_early = 0;     // sweep warps release the averaging grid when their tiles are done
  int32_t claim_batch = 1;   // dynamic schedule: tiles per atomic claim
  int32_t snake = 1;         // static rounds alternate direction
  int32_t spread = 0;        // static tiles over CTAs first (measured: no gain, QAP50 +3 %; off)

  // host copies needed by getters
  // host-side data shared with the plan (no copy; kept alive by the solver)
  std::shared_ptr<const Plan> plan;
  double free_term = 0.0;
  int64_t n_dev_slots = 0;
  int32_t n_tiles = 0, n_varlist = 0, n_shared = 0;
  int32_t max_nodes = 0, max_w = 0, max_hops = 0;
  int64_t n_vars = 0;
  fdog_stats_t st{};

  // device buffers
  TileDesc *d_tiles = nullptr;
  int32_t *d_hop_off = nullptr;
  uint32_t *d_topo = nullptr;
  int32_t *d_slot_var = nullptr;
  void *d_lambda = nullptr;
  void *d_delta[2] = {nullptr, nullptr};
  void *d_m0 = nullptr, *d_m1 = nullptr;
  int32_t *d_var_slots = nullptr, *d_var_xidx = nullptr, *d_deg_list = nullptr;
  int2 *d_ell = nullptr;
  int4 *d_ell4 = nullptr;
  const int32_t *d_elld = nullptr;  // ELL-D part of the averaging (Plan::elld)
  const int32_t *d_elld_var = nullptr;
  int32_t n_elld_g = 0, elld_d[kMaxElld] = {0}, elld_n[kMaxElld] = {0};
  int64_t elld_off[kMaxElld] = {0};
  int32_t *d_ell4_var = nullptr;
  int32_t n_ell = 0, n_ell4 = 0, csr_group = 1;
  // tile-closed pairs (Plan::n_ell_open): the sweep averages them
  // on chip; the averaging kernel writes the other averages in place into the
  // delta_bar buffer, the sweep writes delta into the other one
  int32_t n_ell_open = 0;
  const uint32_t *d_pairs = nullptr;
  bool pairs = false;
  bool avg_full = false;  // (fdog_finalize_averaged: every variable, into the other buffer)
  // primal rounding
  int32_t *d_ell_var = nullptr, *d_csr_var = nullptr;
  uint8_t *d_x = nullptr;
  unsigned long long *d_undecided = nullptr;
  int64_t n_dist = 0;
  int64_t upload_bytes = 0;  // host->device bytes of create
  bool lb_dirty = false;  // per-tile partials not reduced yet
  int64_t *d_var_ptr = nullptr;
  double *d_lb_part = nullptr, *d_lb = nullptr;
  unsigned int *d_counter = nullptr;
  void *d_xbuf = nullptr;
  int32_t *d_x_local = nullptr, *d_x_deg = nullptr;
  std::vector<void *> allocs;

  int cur = 0;        // delta_bar = d_delta[cur]
  int64_t passes = 0;
  int64_t launches = 0;
  int grid = 0, block = 0;
  size_t smem = 0;
  int32_t SB = 0, DB = 0, NB = 2;
  size_t warp_bytes = 0;
  const unsigned char *d_recs = nullptr;
  const int32_t *d_canon = nullptr;  // canonical slot -> device slot
  void *d_canon_out = nullptr;       // getters' staging buffer (T per canonical slot)
  void *d_dist = nullptr;
  int dist_state = 0;  // 0: distances hold shp(v, T); 1: shp(r, v)
  int64_t n_direct = 0, scratch_stride = 0;
  void *d_scratch = nullptr;
  unsigned long long *d_trace = nullptr;  // FDOG_TRACE=1: per-warp sweep timeline of the last sweep

  // one captured iteration (avg, forward, avg, backward), keyed by omega and
  // the parity of the delta buffers; replayed by fdog_iterate
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t seq_graph = nullptr;  // one iteration of the non-deferred variant
  double seq_graph_omega = 0.0;
  int seq_graph_cur = -1;  // the graph's scratch is d_delta[cur ^ 1] of capture time
  int64_t seq_graph_launches = 0;
  double graph_omega = 0.0;
  int graph_cur = -1;
  int64_t graph_launches = 0;
  bool use_graphs = true;
  bool use_fused = false;  // small problems: all iterations in one single-CTA launch
  size_t fused_smem = 0;   // > 0: its state is shared-memory resident

  Nccl nccl;
  std::vector<EventRec> events;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[kKCount] = {0};
  int64_t prof_n[kKCount] = {0};
  double bytes[kKCount] = {0};
};

// Device memory of a solver: the caller's allocator if it gave one, else cudaMalloc.
static cudaError_t dev_alloc(fdog_solver *s, void **p, size_t bytes) {
  if (!s->dev_alloc) return cudaMalloc(p, bytes);
  *p = s->dev_alloc(bytes, s->device, (void *)s->stream, s->alloc_ctx);
  return *p ? cudaSuccess : cudaErrorMemoryAllocation;
}

static void dev_free(fdog_solver *s, void *p) {
  if (!p) return;
  if (s->dev_alloc) {
    if (s->dev_free) s->dev_free(p, s->device, (void *)s->stream, s->alloc_ctx);
  } else {
    cudaFree(p);
  }
}


namespace {

fdog_status cuda_fail(cudaError_t e, const char *what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return FDOG_ENOMEM;
  return FDOG_ECUDA;
}

#define CK(call, what)                                 \
  do {                                                 \
    cudaError_t e__ = (cudaError_t)(call);             \
    if (e__ != cudaSuccess) return cuda_fail(e__, what); \
  } while (0)

cudaEvent_t get_event(fdog_solver *s) {
  if (!s->event_pool.empty()) {
    cudaEvent_t e = s->event_pool.back();
    s->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Timed {
  fdog_solver *s;
  int k;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Timed(fdog_solver *s_, int k_, cudaStream_t st_ = nullptr) : s(s_), k(k_), st(st_ ? st_ : s_->stream) {
    s->launches++;
    if (s->profile) {
      a = get_event(s);
      cudaEventRecord(a, st);
    }
  }
  ~Timed() {
    if (s->profile) {
      cudaEvent_t b = get_event(s);
      cudaEventRecord(b, st);
      s->events.push_back({k, a, b});
    }
  }
};

SweepArgs sweep_args(fdog_solver *s, double omega);

// one sweep over tiles [t0, t1) (default: all)
fdog_status run_sweep(fdog_solver *s, int mode, double omega, int64_t t0 = 0, int64_t t1 = -1) {
  if (t1 < 0) t1 = s->n_tiles;
  if (t1 <= t0 && s->n_tiles > 0) return FDOG_OK;
  SweepArgs a = sweep_args(s, omega);
  a.tiles += t0;
  a.lb_part += t0;
  a.n_tiles = (int32_t)(t1 - t0);
  const bool rec = s->record_mm && (mode == kForward || mode == kBackward);
  int e;
  if (t0 > 0) {
    // the second sweep of a split pass: its own claim counter
    a.tile_counter = s->d_counter + 2;
    CK(cudaMemsetAsync(s->d_counter + 2, 0, sizeof(unsigned int), s->stream), "memset");
  } else if (mode != kForward && mode != kBackward) {
    // not preceded by avg_kernel: reset the dynamic tile counter here
    CK(cudaMemsetAsync(s->d_counter + 1, 0, sizeof(unsigned int), s->stream), "memset");
  }
  {
    Timed t(s, mode == kForward ? kKSweepFwd : mode == kBackward ? kKSweepBwd : kKEnergy);
    if (s->chunk_mode && (mode == kForward || mode == kBackward))
      e = launch_sweep_chunk(s->precision, mode, rec, a, s->stream);
    else if (s->stream_mode && (mode == kForward || mode == kBackward))
      e = launch_sweep_stream(s->precision, mode, rec, a, s->stream);
    else {
      const int64_t warps = s->block / 32;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(s->grid, (a.n_tiles + warps - 1) / warps));
      e = launch_sweep(s->precision, mode, rec, s->rc, s->rw, a, grid, s->block, s->smem, s->stream);
    }
  }
  if (e) return cuda_fail((cudaError_t)e, "sweep launch");
  s->lb_dirty = true;
  return FDOG_OK;
}

SweepArgs sweep_args(fdog_solver *s, double omega) {
  SweepArgs a{};
  a.tiles = s->d_tiles;
  a.n_tiles = s->n_tiles;
  a.hop_off = s->d_hop_off;
  a.topo = s->d_topo;
  a.recs = s->d_recs;
  a.slot_var = nullptr;  // (not uploaded)
  a.lambda = s->d_lambda;
  a.delta_out = s->d_delta[s->cur ^ 1];  // delta out
  // avg_i in: in place in delta_out, or (tile-closed pairs) the delta_bar
  // buffer, where the averaging kernel wrote the other averages in place
  a.avg_in = s->pairs ? s->d_delta[s->cur] : s->d_delta[s->cur ^ 1];
  a.pairs = s->pairs ? s->d_pairs : nullptr;
  a.m0 = s->d_m0;
  a.m1 = s->d_m1;
  a.omega = omega;
  a.clamp = s->clamp;
  a.omega_f = (float)omega;
  a.clamp_f = (float)s->clamp;
  a.lb_part = s->d_lb_part;
  a.done_counter = s->d_counter;
  a.tile_counter = s->d_counter + 1;
  a.max_nodes = s->max_nodes;
  a.max_w = s->max_w;
  a.max_hops = s->max_hops;
  a.SB = s->SB;
  a.DB = s->DB;
  a.NB = s->NB;
  a.dist = s->d_dist;
  a.static_sched = s->static_sched;
  a.pdl_early = s->pdl_early;
  a.claim_batch = s->claim_batch;
  a.snake = s->snake;
  a.spread = s->spread;
  a.trace = s->d_trace;
  a.scratch = s->d_scratch;  // relaxation buffers of direct (unstaged) tiles
  a.scratch_stride = s->scratch_stride;
  a.coop_bw = s->coop_bw;
  a.coop_smem = s->coop_smem ? 1 : 0;
  a.tmem_cols = s->tmem_cols;
  a.lambda0 = s->lifted ? s->d_lam0 : nullptr;
  a.avg0 = s->lifted ? s->d_avg0 : nullptr;
  return a;
}

AvgArgs avg_args(fdog_solver *s);

fdog_status run_avg_finish(fdog_solver *s, cudaStream_t st = nullptr) {
  if (s->world <= 1 || s->n_shared <= 0) return FDOG_OK;
  if (!st) st = s->stream;
  AvgArgs a = avg_args(s);
  int e;
  {
    Timed t(s, kKAvgFinish, st);
    e = launch_avg_finish(s->precision, a, s->n_shared, s->d_x_local, s->d_x_deg, st);
  }
  if (e) return cuda_fail((cudaError_t)e, "avg_finish launch");
  return FDOG_OK;
}

// peer-memory exchange of one pass (after run_avg published this rank's
// partials): wait for the peers', sum them in rank order over NVLink, scatter
// the averages
fdog_status run_peer_exchange(fdog_solver *s, cudaStream_t st = nullptr) {
  if (!st) st = s->stream;
  AvgArgs a = avg_args(s);
  PeerArgs pa = s->peer_args;
  pa.buf_off = kRegionBuf + (int64_t)s->peer_par * (int64_t)s->region_stride;
  int e;
  {
    Timed t(s, kKAvgFinish, st);
    e = launch_peer_finish(s->precision, a, s->n_shared, s->d_x_local, s->d_x_deg, pa, st);
  }
  if (e) return cuda_fail((cudaError_t)e, "peer exchange launch");
  s->peer_par ^= 1;
  return FDOG_OK;
}

AvgArgs avg_args(fdog_solver *s) {
  AvgArgs a{};
  const bool inplace = s->pairs && !s->avg_full;
  a.n_ell = inplace ? s->n_ell_open : s->n_ell;
  a.ell = s->d_ell;
  a.n_ell4 = s->n_ell4;
  a.ell4 = s->d_ell4;
  a.n_elld_g = s->n_elld_g;
  for (int g = 0; g < s->n_elld_g; ++g) {
    a.elld_d[g] = s->elld_d[g];
    a.elld_n[g] = s->elld_n[g];
    a.elld_off[g] = s->elld_off[g];
  }
  a.elld = s->d_elld;
  a.tile_counter = s->d_counter + 1;
  a.ell_v = s->ell_v;
  a.ell_local = s->ell_local;
  a.csr_first = s->csr_first;
  a.n = s->n_varlist;
  a.group = s->csr_group;
  a.var_ptr = s->d_var_ptr;
  a.var_slots = s->d_var_slots;
  a.var_xidx = s->world > 1 ? s->d_var_xidx : nullptr;
  a.deg_l = s->d_deg_list;
  a.delta_bar = s->d_delta[s->cur];
  a.avg_slot = inplace ? s->d_delta[s->cur] : s->d_delta[s->cur ^ 1];
  a.xbuf = s->d_xbuf;
  return a;
}

fdog_status run_avg(fdog_solver *s) {
  AvgArgs a = avg_args(s);
  if (s->peer) a.xbuf = s->d_region + kRegionBuf + (size_t)s->peer_par * s->region_stride;
  if (s->world > 1 && s->n_shared > 0)  // entries of variables this rank does not hold contribute 0
    CK(cudaMemsetAsync(a.xbuf, 0, (size_t)s->n_shared * s->tsz, s->stream), "memset");
  int e;
  {
    Timed t(s, kKAvg);
    e = s->lifted ? launch_avg_lifted(s->precision, a, s->d_avg0, s->stream) : launch_avg(s->precision, a, s->stream);
  }
  if (e) return cuda_fail((cudaError_t)e, "avg launch");
  if (s->peer) {  // publish this rank's partials (the peers read them in their run_peer_exchange)
    if (s->n_shared > 0 && (e = launch_peer_signal(s->peer_args, s->stream)))
      return cuda_fail((cudaError_t)e, "peer signal launch");
    s->launches++;
    return FDOG_OK;
  }
  return FDOG_OK;
}

// the exchange step of a pass (P:641 across ranks) on stream st:
// ncclAllReduce of the shared partial sums + avg_finish, or the peer-memory
// sum + scatter
fdog_status run_exchange(fdog_solver *s, cudaStream_t st) {
  if (s->world <= 1 || s->n_shared <= 0) return FDOG_OK;
  if (s->peer) return run_peer_exchange(s, st);
  if (s->external) return run_avg_finish(s, st);  // (the caller summed the partials)
  int r;
  {
    Timed t(s, kKAllreduce, st);
    s->launches--;  // not our kernel
    r = s->nccl.allreduce(s->d_xbuf, s->d_xbuf, (size_t)s->n_shared, s->precision == 64 ? kNcclFloat64 : kNcclFloat32,
                          kNcclSum, s->nccl.comm, st);
  }
  if (r) {
    set_error("ncclAllReduce: %s", s->nccl.errstr ? s->nccl.errstr(r) : "error");
    return FDOG_ENCCL;
  }
  return run_avg_finish(s, st);
}

// the exchange overlaps the interior tiles' sweep (NCCL or peer exchange with
// boundary tiles; FDOG_OVERLAP=0 runs it first, on the solver's stream)
bool overlapped(const fdog_solver *s) {
  return s->world > 1 && s->n_shared > 0 && (s->peer || !s->external) && s->n_int > 0 && s->n_int < s->n_tiles &&
         s->overlap_ok;
}

// stage 0: conversions + averaging (partials of the exchanged variables in
// xbuf); stage 1: exchanged averages + sweep + swap.  do_pass runs both.
fdog_status pass_stage(fdog_solver *s, bool forward, double omega, int stage) {
  fdog_status st;
  if (stage == 0) {
    // the pass needs the distances of the opposite direction;
    // after an unusual call sequence recompute them first
    // (the recompute design derives them inside the pass)
    if (!s->rc && forward && s->dist_state != 0 && (st = run_sweep(s, kEnergy, omega))) return st;
    if (!s->rc && !forward && s->dist_state != 1 && (st = run_sweep(s, kCfr, omega))) return st;
    return run_avg(s);
  }
  const int mode = forward ? kForward : kBackward;
  if (overlapped(s)) {
    if (!s->xstream) {
      CK(cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking), "cudaStreamCreate");
      CK(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
      CK(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming), "cudaEventCreate");
    }
    CK(cudaEventRecord(s->ev_fork, s->stream), "cudaEventRecord");
    CK(cudaStreamWaitEvent(s->xstream, s->ev_fork, 0), "cudaStreamWaitEvent");
    if ((st = run_exchange(s, s->xstream))) return st;
    CK(cudaEventRecord(s->ev_join, s->xstream), "cudaEventRecord");
    if ((st = run_sweep(s, mode, omega, 0, s->n_int))) return st;  // interior tiles: no exchanged variable
    CK(cudaStreamWaitEvent(s->stream, s->ev_join, 0), "cudaStreamWaitEvent");
    if ((st = run_sweep(s, mode, omega, s->n_int, s->n_tiles))) return st;
  } else {
    if ((st = run_exchange(s, s->stream))) return st;
    if ((st = run_sweep(s, mode, omega))) return st;
  }
  s->dist_state = s->rc ? 2 : (forward ? 1 : 0);  // (the recompute design keeps no distances in HBM)
  s->cur ^= 1;  // mbar <- m
  s->passes++;
  s->dbar_zero = false;
  return FDOG_OK;
}

fdog_status do_pass(fdog_solver *s, bool forward, double omega) {
  fdog_status st = pass_stage(s, forward, omega, 0);
  return st ? st : pass_stage(s, forward, omega, 1);
}

fdog_status energy(fdog_solver *s) {
  fdog_status st = run_sweep(s, kEnergy, 0.5);
  if (!st) s->dist_state = s->rc ? 2 : 0;
  return st;
}

// ---- non-deferred variant ---------------------------
// Level schedule of one pass direction: level(i) = 1 + max over the rows of i
// of the level of i's predecessor (forward: the previous variable of the row;
// backward: the next one).  Variables of one level share no BDD, so a level is
// one kernel launch and the pass equals visiting the variables one by one.
fdog_status seq_schedule(fdog_solver *s) {
  if (s->seq_ready) return FDOG_OK;
  const Plan &P = *s->plan;
  const int64_t S = (int64_t)P.canon_slot.size();
  const int32_t n = P.n_vars;
  // per variable: canonical slots, j ascending
  std::vector<int64_t> vptr(n + 1, 0);
  for (int64_t q = 0; q < S; ++q) vptr[P.col_var[P.row_ptr[P.canon_con[q]] + P.canon_pos[q]] + 1]++;
  for (int32_t i = 0; i < n; ++i) vptr[i + 1] += vptr[i];
  std::vector<int64_t> vq(S), fill(vptr.begin(), vptr.end() - 1);
  for (int64_t q = 0; q < S; ++q) vq[fill[P.col_var[P.row_ptr[P.canon_con[q]] + P.canon_pos[q]]]++] = q;
  std::vector<int32_t> slot_tile(std::max<int64_t>(s->n_dev_slots, 1), 0);
  for (int32_t t = 0; t < (int32_t)P.tiles.size(); ++t) {
    const TileDesc &d = P.tiles[t];
    for (int64_t x = 0; x < (int64_t)d.K * d.lanes; ++x) slot_tile[d.slot_base + x] = t;
  }
  const size_t bytes = slot_tile.size() * 4 + 2 * ((size_t)(n + 1) * 8 + (size_t)std::max<int64_t>(S, 1) * 4) +
                       (size_t)std::max(s->n_tiles, 1) * kMaxTileRows * 8 + 8 * 256;  // + alignment of six sections
  unsigned char *base = nullptr;
  CK(dev_alloc(s, (void **)&base, bytes), "device allocation (seq schedule)");
  s->allocs.push_back(base);
  size_t at = 0;
  auto carve = [&](size_t b) {
    unsigned char *p = base + at;
    at += (b + 255) & ~(size_t)255;
    return p;
  };
  s->d_slot_tile = (int32_t *)carve(slot_tile.size() * 4);
  CK(cudaMemcpyAsync(s->d_slot_tile, slot_tile.data(), slot_tile.size() * 4, cudaMemcpyHostToDevice, s->stream), "H2D");
  for (int dir = 0; dir < 2; ++dir) {
    const bool fwd = dir == 1;
    std::vector<int32_t> lvl(n, -1);
    int32_t nl = 0;
    for (int32_t t = 0; t < n; ++t) {
      const int32_t i = fwd ? t : n - 1 - t;
      if (vptr[i] == vptr[i + 1]) continue;
      int32_t L = 0;
      for (int64_t x = vptr[i]; x < vptr[i + 1]; ++x) {
        const int64_t q = vq[x];
        const int32_t j = P.canon_con[q], pos = P.canon_pos[q];
        const int32_t k = (int32_t)(P.row_ptr[j + 1] - P.row_ptr[j]);
        const int32_t nb = fwd ? pos - 1 : pos + 1;  // the row's neighbour visited before i
        if (nb >= 0 && nb < k) L = std::max(L, lvl[P.col_var[P.row_ptr[j] + nb]] + 1);
      }
      lvl[i] = L;
      nl = std::max(nl, L + 1);
    }
    // pass order: by level, then variable (counting sort)
    std::vector<int64_t> cnt(nl + 1, 0);
    for (int32_t i = 0; i < n; ++i)
      if (lvl[i] >= 0) cnt[lvl[i] + 1]++;
    for (int32_t l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
    s->seq_lvl[dir] = cnt;
    std::vector<int32_t> order(cnt[nl]);
    std::vector<int64_t> f(cnt.begin(), cnt.end() - 1);
    for (int32_t i = 0; i < n; ++i)
      if (lvl[i] >= 0) order[f[lvl[i]]++] = i;
    std::vector<int64_t> ptr(order.size() + 1, 0);
    std::vector<int32_t> slots;
    slots.reserve(S);
    for (size_t o = 0; o < order.size(); ++o) {
      const int32_t i = order[o];
      for (int64_t x = vptr[i]; x < vptr[i + 1]; ++x) slots.push_back((int32_t)P.canon_slot[vq[x]]);
      ptr[o + 1] = (int64_t)slots.size();
    }
    s->d_seq_ptr[dir] = (int64_t *)carve(ptr.size() * 8);
    s->d_seq_slots[dir] = (int32_t *)carve(std::max<size_t>(slots.size(), 1) * 4);
    CK(cudaMemcpyAsync(s->d_seq_ptr[dir], ptr.data(), ptr.size() * 8, cudaMemcpyHostToDevice, s->stream), "H2D");
    if (!slots.empty())
      CK(cudaMemcpyAsync(s->d_seq_slots[dir], slots.data(), slots.size() * 4, cudaMemcpyHostToDevice, s->stream), "H2D");
    CK(cudaStreamSynchronize(s->stream), "sync");  // host vectors go out of scope
  }
  s->d_e_lane = (double *)carve((size_t)std::max(s->n_tiles, 1) * kMaxTileRows * 8);
  CK(cudaMemsetAsync(s->d_e_lane, 0, (size_t)std::max(s->n_tiles, 1) * kMaxTileRows * 8, s->stream), "memset");
  s->seq_ready = true;
  return FDOG_OK;
}

SeqArgs seq_args(fdog_solver *s, bool forward, double omega) {
  SeqArgs a{};
  a.tiles = s->d_tiles;
  a.hop_off = s->d_hop_off;
  a.topo = s->d_topo;
  a.slot_tile = s->d_slot_tile;
  a.ptr = s->d_seq_ptr[forward ? 1 : 0];
  a.slots = s->d_seq_slots[forward ? 1 : 0];
  a.lambda = s->d_lambda;
  a.dist = s->d_dist;
  a.delta = s->d_delta[s->cur ^ 1];  // scratch; delta_bar (d_delta[cur]) stays 0
  a.m0 = s->record_mm ? s->d_m0 : nullptr;
  a.m1 = s->record_mm ? s->d_m1 : nullptr;
  a.e_lane = s->d_e_lane;
  a.omega = omega;
  a.clamp = s->clamp;
  a.omega_f = (float)omega;
  a.clamp_f = (float)s->clamp;
  a.forward = forward ? 1 : 0;
  return a;
}

fdog_status do_pass_seq(fdog_solver *s, bool forward, double omega) {
  fdog_status st = seq_schedule(s);
  if (st) return st;
  SeqArgs a = seq_args(s, forward, omega);
  int e;
  // store-design distances of the opposite direction
  if (forward ? s->dist_state != 0 : s->dist_state != 1) {
    Timed t(s, kKEnergy);
    e = launch_dist_dp(s->precision, a, s->n_tiles, forward ? 0 : 1, s->stream);
    if (e) return cuda_fail((cudaError_t)e, "dist_dp launch");
  }
  const std::vector<int64_t> &lv = s->seq_lvl[forward ? 1 : 0];
  {
    Timed t(s, forward ? kKSweepFwd : kKSweepBwd);
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      e = launch_seq_level(s->precision, s->record_mm, a, lv[l], lv[l + 1], s->stream);
      if (e) return cuda_fail((cudaError_t)e, "seq level launch");
      s->launches++;
    }
    s->launches--;  // (Timed counts one)
  }
  e = launch_seq_bound(s->d_tiles, s->n_tiles, s->d_e_lane, s->d_lb_part, s->stream);
  if (e) return cuda_fail((cudaError_t)e, "seq bound launch");
  s->launches++;
  s->dist_state = forward ? 1 : 0;
  s->passes++;
  s->dbar_zero = true;
  s->lb_dirty = true;
  return FDOG_OK;
}

void free_solver(fdog_solver *s) {
  if (!s) return;
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (auto &e : s->events) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : s->event_pool) cudaEventDestroy(e);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->seq_graph) cudaGraphExecDestroy(s->seq_graph);
  if (s->xstream) {
    cudaStreamSynchronize(s->xstream);
    cudaStreamDestroy(s->xstream);
  }
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  for (void *p : s->allocs) dev_free(s, p);
  for (void *p : s->own_allocs) cudaFree(p);
  if (s->nccl.comm && s->nccl.destroy) s->nccl.destroy(s->nccl.comm);
  if (s->nccl.lib) dlclose(s->nccl.lib);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

fdog_status fetch_slots(fdog_solver *s, const void *dev, double *out, int64_t len) {
  const int64_t n = (int64_t)s->plan->canon_slot.size();
  if (!out || len < n) {
    set_error("output length %lld < %lld slots", (long long)len, (long long)n);
    return FDOG_EINVAL;
  }
  if (n == 0) return FDOG_OK;
  // canonical (j, h) order and the widening to fp64 on the device (gather
  // kernel), then one contiguous copy straight into the caller's buffer
  // (measured 1.1 ms for GM's 2.3 M slots vs 4.8-7.9 ms through a host buffer)
  const bool direct = s->precision == 64 || s->get_direct;
  const int e = launch_gather_canon(s->precision, n, s->d_canon, dev, s->d_canon_out, direct ? 1 : 0, s->stream);
  if (e) return cuda_fail((cudaError_t)e, "gather launch");
  s->launches++;
  if (direct) {  // fp64 values (widened on the device in fp32) straight into the caller's buffer
    CK(cudaMemcpyAsync(out, s->d_canon_out, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s->stream), "D2H");
    CK(cudaStreamSynchronize(s->stream), "sync");
  } else {
    std::vector<float> buf((size_t)n);
    CK(cudaMemcpyAsync(buf.data(), s->d_canon_out, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, s->stream), "D2H");
    CK(cudaStreamSynchronize(s->stream), "sync");
    for (int64_t q = 0; q < n; ++q) out[q] = (double)buf[q];
  }
  return FDOG_OK;
}

fdog_status put_slots(fdog_solver *s, void *dev, const double *in, int64_t len) {
  const int64_t n = (int64_t)s->plan->canon_slot.size();
  if (len != n) {
    set_error("input length %lld != %lld slots", (long long)len, (long long)n);
    return FDOG_EINVAL;
  }
  std::vector<unsigned char> buf((size_t)std::max<int64_t>(s->n_dev_slots, 1) * s->tsz);
  CK(cudaMemcpyAsync(buf.data(), dev, (size_t)s->n_dev_slots * s->tsz, cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  if (s->precision == 64) {
    double *b = (double *)buf.data();
    for (int64_t q = 0; q < n; ++q) b[s->plan->canon_slot[q]] = in[q];
  } else {
    float *b = (float *)buf.data();
    for (int64_t q = 0; q < n; ++q) b[s->plan->canon_slot[q]] = (float)in[q];
  }
  CK(cudaMemcpyAsync(dev, buf.data(), (size_t)s->n_dev_slots * s->tsz, cudaMemcpyHostToDevice, s->stream), "H2D");
  CK(cudaStreamSynchronize(s->stream), "sync");
  return FDOG_OK;
}

fdog_status init_nccl(fdog_solver *s, const fdog_options *o) {
  if (!o->nccl_unique_id) {
    set_error("world > 1 needs nccl_unique_id");
    return FDOG_EINVAL;
  }
  const char *path = o->nccl_library ? o->nccl_library : "libnccl.so.2";
  s->nccl.lib = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!s->nccl.lib) {
    set_error("dlopen(%s): %s", path, dlerror());
    return FDOG_ENCCL;
  }
  s->nccl.init = (nccl_init_fn)dlsym(s->nccl.lib, "ncclCommInitRank");
  s->nccl.allreduce = (nccl_allreduce_fn)dlsym(s->nccl.lib, "ncclAllReduce");
  s->nccl.destroy = (nccl_destroy_fn)dlsym(s->nccl.lib, "ncclCommDestroy");
  s->nccl.errstr = (nccl_errstr_fn)dlsym(s->nccl.lib, "ncclGetErrorString");
  if (!s->nccl.init || !s->nccl.allreduce || !s->nccl.destroy) {
    set_error("libnccl is missing ncclCommInitRank/ncclAllReduce/ncclCommDestroy");
    return FDOG_ENCCL;
  }
  nccl_uid uid;
  std::memcpy(uid.internal, o->nccl_unique_id, sizeof uid.internal);
  // FDOG_NCCL_SELF=1 (test knob, one GPU): a one-rank communicator even for
  // world > 1 -- the exchange's allreduce is then the identity, which the
  // tests compare with the external-exchange mode doing the same
  const char *ns = getenv("FDOG_NCCL_SELF");
  const bool self = ns && ns[0] == '1';
  int r = s->nccl.init(&s->nccl.comm, self ? 1 : s->world, uid, self ? 0 : s->rank);
  if (r) {
    set_error("ncclCommInitRank: %s", s->nccl.errstr ? s->nccl.errstr(r) : "error");
    return FDOG_ENCCL;
  }
  return FDOG_OK;
}

// FDOG_PLAN_TRACE=1: phase times of a solver's create on stderr (host time;
// device work is asynchronous until the final synchronisation)
struct CreateTimer {
  bool on = getenv("FDOG_PLAN_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char *what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[create] %-26s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

fdog_status create_impl(std::shared_ptr<const Plan> plan, const fdog_options *o, fdog_solver *s) {
  CreateTimer ctm;
  s->plan = plan;
  const Plan &P = *plan;
  s->precision = o->precision == 64 ? 64 : 32;
  if (o->precision != 32 && o->precision != 64) {
    set_error("precision must be 32 or 64");
    return FDOG_EINVAL;
  }
  s->tsz = s->precision == 64 ? 8 : 4;
  s->device = o->device;
  s->dev_alloc = o->dev_alloc;
  s->dev_free = o->dev_free;
  s->alloc_ctx = o->alloc_ctx;
  s->record_mm = o->record_mm != 0;
  s->lifted = o->lifted != 0;
  if (s->lifted != P.lifted) {
    set_error("the plan was packed %s the lifted representation; create the plan with the same option",
              P.lifted ? "for" : "without");
    return FDOG_EINVAL;
  }
  s->profile = o->profile != 0;
  if (const char *ev = getenv("FDOG_ELLV")) {  // experiment knob: ELL variables per averaging thread (1, 2, 4, 8)
    const int v = atoi(ev);
    if (v == 1 || v == 2 || v == 4 || v == 8) s->ell_v = v;
  }
  {
    const char *g = getenv("FDOG_GRAPHS");  // experiment knob: FDOG_GRAPHS=0 disables graph replay
    s->use_graphs = !(g && g[0] == '0');
    const char *ov = getenv("FDOG_OVERLAP");  // test knob: FDOG_OVERLAP=0 runs the exchange before the sweep
    s->overlap_ok = !(ov && ov[0] == '0');
  }
  s->rank = P.rank;
  s->world = P.world;
  s->clamp = o->clamp > 0 ? o->clamp : 1e4 * (1.0 + P.max_abs_cost);  // A5
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (s->device < 0 || s->device >= ndev) {
    set_error("device %d not present (%d devices)", s->device, ndev);
    return FDOG_EINVAL;
  }
  CK(cudaSetDevice(s->device), "cudaSetDevice");
  if (o->stream) {
    s->stream = (cudaStream_t)o->stream;
  } else {
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    s->own_stream = true;
  }
  s->free_term = P.rank == 0 ? P.free_term : 0.0;
  s->n_dev_slots = (int64_t)P.slot_var.size();
  s->n_tiles = (int32_t)P.tiles.size();
  s->n_int = P.world > 1 ? P.n_interior_tiles : s->n_tiles;
  s->n_varlist = (int32_t)P.var_list.size();
  s->n_shared = (int32_t)P.shared_vars.size();
  s->n_vars = P.n_vars;
  s->max_nodes = std::max(1, P.max_tile_nodes);
  s->max_w = std::max(1, P.max_width);
  s->max_hops = std::max(1, P.max_hops);

  // launch configuration: persistent grid of warps; per-warp shared-memory
  // budget chosen so that >= 16 warps fit per SM; tiles within the budget are
  // staged through TMA (kind bit 2), the rest run directly from global memory
  struct {
    int smem_sm, smem_block, sms;
  } prop;
  CK(cudaDeviceGetAttribute(&prop.smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, s->device), "attr");
  CK(cudaDeviceGetAttribute(&prop.smem_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device), "attr");
  CK(cudaDeviceGetAttribute(&prop.sms, cudaDevAttrMultiProcessorCount, s->device), "attr");
  std::vector<TileDesc> tiles = P.tiles;
  if (P.precision != s->precision) {
    set_error("plan packed for fp%d, solver asked for fp%d", P.precision, s->precision);
    return FDOG_EINVAL;
  }
  s->SB = P.SB;
  s->DB = P.DB;
  s->NB = P.NB;
  s->rc = P.rc;
  s->warp_bytes = (size_t)warp_bytes(P.SB, P.DB, P.NB);
  for (const auto &d : tiles) s->rw = std::max(s->rw, d.lanes / 32);
  s->n_direct = P.direct_tiles;
  s->n_coop = P.coop_tiles;
  {
    // all tiles narrow: the passes stream from global memory (no staging)
    bool narrow = true;
    for (const auto &d : tiles) narrow = narrow && d.max_w <= 2;
    // the TMA-staged kernel wins while every tile is staged and enough warps fit
    // per SM; long BDDs (tiles too large to stage, or only for < 8 warps per SM)
    // stream instead
    const size_t sm_bytes = (size_t)prop.smem_sm - 4096;
    const bool staged_ok = sm_bytes / std::max<size_t>(s->warp_bytes, 1) >= 8 && s->n_direct == 0;
    const char *m = getenv("FDOG_SWEEP");  // experiment knob: "tma" or "stream"
    const bool forced = m && (m[0] == 's' || m[0] == 't');
    s->stream_mode = !s->rc && narrow && (forced ? m[0] == 's' : !staged_ok);
    // rows too long to stage: walk them in chunks through shared memory when
    // every tile carries hop records (FDOG_CHUNK=0 keeps the streaming kernel)
    bool masks = true;
    for (const auto &d : tiles) masks = masks && (d.kind & 4);
    const char *ck = getenv("FDOG_CHUNK");
    s->chunk_mode = s->stream_mode && masks && !(forced && m[0] == 's') && !(ck && ck[0] == '0');
    // tiny instances (BASELINE configs[0]) are launch-latency bound: one CTA
    // runs every iteration of an fdog_iterate call (fused_small_kernel)
    const char *fz = getenv("FDOG_FUSED");  // experiment knob: 0 / 1
    const bool small = tiles.size() <= 64 && P.n_slots <= (1 << 15) && P.direct_tiles == 0;  // (long rows: chunked kernel)
    s->use_fused = !s->rc && narrow && P.world == 1 && (fz ? fz[0] == '1' : small);
    const size_t fbytes = (size_t)(3 * (int64_t)P.slot_var.size() + P.n_dist) * s->tsz;
    const char *fr = getenv("FDOG_FUSED_SMEM");  // experiment knob: 0 keeps the state in global memory
    s->fused_smem = (fbytes <= (size_t)prop.smem_block && !(fr && fr[0] == '0')) ? fbytes : 0;
    if (m && m[0] == 's' && !narrow) {
      set_error("FDOG_SWEEP=stream needs every partition <= 2 nodes wide");
      return FDOG_EINVAL;
    }
  }
  if (s->lifted) {  // every tile through sweep_kernel's lane-serial / node-parallel paths (the lifted arc costs)
    s->stream_mode = s->chunk_mode = s->use_fused = false;
  }
  if (s->rw > 1 && (s->stream_mode || s->chunk_mode || s->use_fused)) {  // (plan.cpp never packs them so)
    set_error("tiles of %d rows need the staged sweep kernel", 32 * s->rw);
    return FDOG_EINVAL;
  }
  // tile-closed pairs are averaged by sweep_kernel only (the streaming,
  // chunked and fused paths read every average from the averaging kernel)
  s->pairs = !s->lifted && P.n_ell_open < (int64_t)(P.ell.size() / 2) && !s->stream_mode && !s->chunk_mode && !s->use_fused &&
             P.direct_tiles == 0;
  // (4 warps per CTA: sweep_kernel's launch bounds; TMEM kernels below)
  const char *wpb = getenv("FDOG_WPB");  // test knob: fewer warps per sweep CTA (default and max 4)
  const size_t wmax = wpb ? std::max(1, std::min(4, atoi(wpb))) : 4;
  int warps = sweep_warps_per_cta(s->warp_bytes, (int)wmax, prop.smem_block, prop.smem_sm);
  // fewer tiles than 4 warps per SM: spread them, one warp per SM first
  // (measured: GAP's 20 wide BDDs, one warp each, 3.06 -> 2.53 ms per
  // iteration in CTAs of 1 warp instead of 4)
  if (s->n_tiles > 0 && s->n_tiles < (int64_t)prop.sms * warps)
    warps = std::max(1, std::min(warps, (int)((s->n_tiles + prop.sms - 1) / prop.sms)));
  s->tmem_cols = P.tmem_cols;
  if (s->tmem_cols > 0) {
    // TMEM variant (kernels.cu sweep_kernel<..., TM>): one CTA per SM (a kernel
    // with tcgen05 code runs one CTA per SM), warps in groups of four sharing
    // the 128 TMEM lanes, each group tmem_cols of the 512 columns
    const int by_tmem = 4 * (512 / s->tmem_cols);
    const int by_smem = (int)((size_t)prop.smem_block / s->warp_bytes);
    warps = std::min({16, by_tmem, by_smem});
    if (warps >= 4) warps &= ~3;
    s->rw = 0;
  }
  s->block = warps * 32;
  s->smem = (size_t)warps * s->warp_bytes;
  int bps = 1;
  for (int mode = 0; mode < 4; ++mode)
    for (int rec = 0; rec < 2; ++rec) {
      int b = 0;
      int e = sweep_occupancy(s->precision, mode, rec && mode != kEnergy, s->rc, s->rw, s->block, s->smem, &b);
      if (e) return cuda_fail((cudaError_t)e, "occupancy");
      if (mode == kForward && rec == (int)s->record_mm) bps = std::max(1, b);
    }
  const int64_t want = ((int64_t)s->n_tiles + warps - 1) / warps;
  s->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)prop.sms * bps));
  {
    // few tiles per warp: a plain round-robin over the cost-sorted tiles
    // (claims would sit on the critical path); many tiles per warp: dynamic
    // claims balance the load.  The single-buffered recompute design claims
    // dynamically whenever a warp has more than one tile (measured: QAP50
    // -8 %, CellTrack -11 %, GM equal)
    const char *sc = getenv("FDOG_SCHED");  // experiment knob: "static" or "dynamic"
    const int64_t warps_total = (int64_t)s->grid * warps;
    if (sc && (sc[0] == 's' || sc[0] == 'd')) s->static_sched = sc[0] == 's';
    else s->static_sched = s->n_tiles <= (s->rc ? 1 : 4) * warps_total;
    // store design with few tiles per warp: the sweep's tail is a large part
    // of it; its warps release the averaging grid as they finish, whose CTAs
    // load their (constant) slot indices on the idle SMs before waiting for
    // the sweep (measured: GM -1 %; CellTrack, QAP50, MRF (recompute design)
    // +0-2 %, so off there)
    // many tiles per warp: one claim takes several consecutive tiles, so the
    // single counter is not a serialisation point (measured: MRF, 68 tiles per
    // warp, sweeps 282 -> 219 us with 2-4 tiles per claim, 8: 226, 16: 235;
    // CellTrack, 9.5 per warp, 39.5 -> 38.8 us with 2; round 2: see below)
    const char *cb = getenv("FDOG_CLAIM");  // experiment knob: tiles per claim
    const int64_t tpw = s->n_tiles / std::max<int64_t>(warps_total, 1);
    // (64-row MRF-LP tiles, 41 per warp: 2 per claim 518, 4 per claim 526 us
    // per iteration; Potts-cut, 26 per warp, 1 / 2 equal)
    s->claim_batch = cb ? std::max(1, atoi(cb)) : (tpw >= 64 ? 4 : tpw >= 8 ? 2 : 1);
    s->pdl_early = !s->rc && s->n_tiles < 8 * warps_total ? 1 : 0;
    // (A balanced static grid -- every warp exactly ceil(tiles / warps) tiles --
    // was measured on QAP50: 6 % slower.  Warps' finish times spread over 2x
    // either way: a grid that is not a multiple of the SM count leaves SMs
    // with different warp counts, i.e. different per-tile times.)
  }
  // direct tiles: the lane-serial relaxation buffers (32 lanes); cooperative
  // tiles: two buffers of coop_w + 1 entries unless they sit in shared memory
  s->scratch_stride = std::max<int64_t>(P.direct_w > 0 ? (int64_t)relax_slots(P.direct_w) * 32 : 0,
                                        (P.coop_tiles > 0 && !P.coop_smem) ? 2 * ((int64_t)P.coop_w + 1) : 0);
  s->coop_bw = P.coop_w + 1;
  s->coop_smem = P.coop_smem;

  fdog_status st;
  s->n_dist = P.n_dist;
  s->n_ell = (int32_t)(P.ell.size() / 2);
  s->n_ell_open = (int32_t)P.n_ell_open;
  s->n_ell4 = (int32_t)(P.ell4.size() / 4);
  s->n_elld_g = (int32_t)P.elld_d.size();
  for (int g = 0; g < s->n_elld_g; ++g) {
    s->elld_d[g] = P.elld_d[g];
    s->elld_n[g] = P.elld_n[g];
    s->elld_off[g] = P.elld_off[g];
  }
  {
    int64_t maxdeg = 1;
    for (size_t q = 0; q + 1 < P.var_ptr.size(); ++q) maxdeg = std::max<int64_t>(maxdeg, P.var_ptr[q + 1] - P.var_ptr[q]);
    // lanes per CSR variable: about four slots per lane for the widest variable
    s->csr_group = 1;
    while (s->csr_group < 32 && 4 * s->csr_group < maxdeg) s->csr_group *= 2;
  }
  // one device allocation: the plan's image (one host->device copy) followed
  // by the runtime buffers (zeroed)
  const size_t slot_bytes = (size_t)std::max<int64_t>(s->n_dev_slots, 1) * s->tsz;
  const HostImage &im = P.image;
  if (!im.data) {
    set_error("plan has no device image");
    return FDOG_ESTATE;
  }
  size_t rt = 0;
  auto carve = [&](size_t bytes) {
    const size_t at = rt;
    rt += (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255;
    return at;
  };
  const size_t o_delta0 = carve(slot_bytes), o_delta1 = carve(slot_bytes);
  const size_t o_m0 = s->record_mm ? carve(slot_bytes) : 0, o_m1 = s->record_mm ? carve(slot_bytes) : 0;
  const size_t o_xbuf = carve((size_t)std::max<int32_t>(s->n_shared, 1) * s->tsz);
  const size_t o_lbp = carve((size_t)std::max(s->n_tiles, 1) * sizeof(double));
  const size_t o_lb = carve(2 * sizeof(double));
  const size_t o_ctr = carve(4 * sizeof(unsigned int));  // done, tile claims, split-pass claims
  const size_t o_scr = carve(std::max<size_t>(s->n_direct ? (size_t)s->grid * (s->block / 32) * s->scratch_stride * s->tsz : 0, 16));
  const size_t o_x = carve((size_t)std::max<int64_t>(P.n_vars, 1));
  const size_t o_und = carve(sizeof(unsigned long long));
  const size_t o_canon = carve((size_t)std::max<size_t>(P.canon_slot.size(), 1) * 8);  // (fp64 when widened)
  const size_t o_dist = carve((size_t)std::max<int64_t>(P.n_dist, 1) * s->tsz);
  // lifted representation: lambda^{j,0} (0 initially), its averages, getter scratch
  const size_t o_l0 = s->lifted ? carve(slot_bytes) : 0, o_a0 = s->lifted ? carve(slot_bytes) : 0;
  const size_t o_lo = s->lifted ? carve(slot_bytes) : 0;
  unsigned char *base = nullptr;
  ctm.mark("setup");
  CK(dev_alloc(s, (void **)&base, im.bytes + rt), "device allocation");
  s->allocs.push_back(base);
  s->st.device_bytes = (int64_t)(im.bytes + rt);
  s->upload_bytes = (int64_t)im.bytes;
  CK(cudaMemcpyAsync(base, im.data, im.bytes, cudaMemcpyHostToDevice, s->stream), "H2D");
  CK(cudaMemsetAsync(base + im.bytes, 0, rt, s->stream), "memset");
  auto sec = [&](int q) { return (void *)(base + im.off[q]); };
  s->d_tiles = (TileDesc *)sec(kImTiles);
  s->d_hop_off = (int32_t *)sec(kImHopOff);
  s->d_topo = (uint32_t *)sec(kImTopo);
  s->d_recs = (const unsigned char *)sec(kImRecs);
  s->d_pairs = (const uint32_t *)sec(kImPairs);
  s->d_canon = (const int32_t *)sec(kImCanon);
  s->d_var_ptr = (int64_t *)sec(kImVarPtr);
  s->d_var_slots = (int32_t *)sec(kImVarSlots);
  s->d_var_xidx = (int32_t *)sec(kImVarXidx);
  s->d_deg_list = (int32_t *)sec(kImDegList);
  s->d_ell = (int2 *)sec(kImEll);
  s->d_ell_var = (int32_t *)sec(kImEllVar);
  s->d_ell4 = (int4 *)sec(kImEll4);
  s->d_elld = (const int32_t *)sec(kImElld);
  s->d_elld_var = (const int32_t *)sec(kImElldVar);
  s->d_ell4_var = (int32_t *)sec(kImEll4Var);
  s->d_csr_var = (int32_t *)sec(kImCsrVar);
  s->d_x_local = (int32_t *)sec(kImXLocal);
  s->d_x_deg = (int32_t *)sec(kImXDeg);
  s->d_lambda = sec(kImLambda0);
  s->d_dist = nullptr;  // runtime region below
  unsigned char *r = base + im.bytes;
  s->d_delta[0] = r + o_delta0;
  s->d_delta[1] = r + o_delta1;
  if (s->record_mm) {
    s->d_m0 = r + o_m0;
    s->d_m1 = r + o_m1;
  }
  s->d_xbuf = r + o_xbuf;
  s->d_lb_part = (double *)(r + o_lbp);
  s->d_lb = (double *)(r + o_lb);
  s->d_counter = (unsigned int *)(r + o_ctr);
  s->d_scratch = r + o_scr;
  s->d_x = (uint8_t *)(r + o_x);
  s->d_undecided = (unsigned long long *)(r + o_und);
  s->d_canon_out = r + o_canon;
  if (s->lifted) {
    s->d_lam0 = r + o_l0;
    s->d_avg0 = r + o_a0;
    s->d_lam_out = r + o_lo;
  }
  if (const char *tr = getenv("FDOG_TRACE"); tr && tr[0] == '1') {
    void *p = nullptr;
    CK(dev_alloc(s, &p, (size_t)s->grid * (s->block / 32) * 4 * 8), "device allocation (trace)");
    s->allocs.push_back(p);
    s->d_trace = (unsigned long long *)p;
  }
  s->d_dist = r + o_dist;
  {
    // the distances' sentinels (top 0, bottom +inf) of every tile lane
    const int e = launch_dist_sentinels(s->precision, s->d_tiles, s->n_tiles, s->d_dist, s->stream);
    if (e) return cuda_fail((cudaError_t)e, "sentinel launch");
  }
  s->external = s->world > 1 && !o->nccl_unique_id;
  if (s->world > 1 && !s->external && (st = init_nccl(s, o))) return st;
  if (s->external) {
    // exchange region for the peer-memory mode (a separate allocation, so that
    // one CUDA IPC handle maps exactly it): counter, error word, two buffers
    s->region_stride = ((size_t)std::max<int32_t>(s->n_shared, 1) * s->tsz + 255) & ~(size_t)255;
    const size_t rb = kRegionBuf + 2 * s->region_stride;
    CK(cudaMalloc((void **)&s->d_region, rb), "cudaMalloc (exchange region)");
    s->own_allocs.push_back(s->d_region);
    CK(cudaMemsetAsync(s->d_region, 0, rb, s->stream), "memset");
  }
  // FDOG_NCCL_SELF=1 (test knob): a one-rank NCCL communicator for world == 1,
  // so the bound's allreduce goes through the same dlopen'ed NCCL calls as a
  // multi-GPU run (tests/test_gpu_parity.py::test_nccl_one_rank_communicator)
  if (s->world == 1 && o->nccl_unique_id) {
    const char *ns = getenv("FDOG_NCCL_SELF");
    if (ns && ns[0] == '1' && (st = init_nccl(s, o))) return st;
  }

  // algorithmic bytes per launch: per node 2 T (distance read +
  // write) + 4 B topology for per-lane-topology tiles; per slot 4 T (lambda
  // read + write, average read, delta write)
  {
    const double T = (double)s->tsz;
    const double slots = (double)P.n_slots, nv = (double)P.var_list.size(), nodes = (double)P.n_nodes;
    double lane_topo = 0;
    for (const auto &d : tiles)
      if (d.kind & 1) lane_topo += 4.0 * d.nodes * d.n_lanes;
    const double rec = s->record_mm ? 2 * T : 0.0;
    // (recompute design: no per-node distance traffic)
    const double dist = s->rc ? 0.0 : nodes * 2 * T;
    s->bytes[kKSweepFwd] = s->bytes[kKSweepBwd] = dist + lane_topo + slots * (4 * T + rec);
    s->bytes[kKEnergy] = dist + lane_topo + slots * T;
    // averaging: per slot the slot index, the delta gather and the average scatter;
    // per variable the CSR pointer and |J_i|
    s->bytes[kKAvg] = slots * (4 + 2 * T) + nv * (8 + 4);
    s->bytes[kKAvgFinish] = (double)s->n_shared * (4 + 4 + T);
    s->bytes[kKAllreduce] = (double)s->n_shared * T;
    s->bytes[kKAddDeferred] = (double)s->n_dev_slots * 4 * T;
  }
  ctm.mark("allocation, upload, launch setup");
  // stats
  s->st.bdds = (int64_t)P.local_rows.size();
  s->st.nodes = P.n_nodes;
  s->st.arcs = 2 * P.n_nodes;
  s->st.slots = P.n_slots;
  s->st.vars_local = P.n_vars_local;
  s->st.vars_shared = P.n_vars_shared;
  s->st.free_vars = P.n_free_vars;
  s->st.shapes = (int64_t)P.shapes.size();
  s->st.tiles = (int64_t)P.tiles.size();
  s->st.tiles_shared_topology = P.tiles_shared;
  s->st.padded_slots = s->n_dev_slots;
  s->st.max_hops = P.max_hops;
  s->st.max_width = P.max_width;
  s->st.staged_tiles = (int64_t)tiles.size() - s->n_direct;
  s->st.sweep_grid = s->grid;
  s->st.sweep_block = s->block;
  s->st.sweep_smem_per_warp = (int64_t)s->warp_bytes;
  s->st.sweep_streaming = s->chunk_mode ? 2 : s->stream_mode ? 1 : 0;
  s->st.h2d_bytes = s->upload_bytes;
  s->st.fused_small = s->use_fused ? (s->fused_smem ? 2 : 1) : 0;
  s->st.sweep_recompute = s->rc ? 1 : 0;
  s->st.tile_pairs = s->pairs ? (int64_t)s->n_ell - s->n_ell_open : 0;
  s->st.interior_tiles = s->n_int;
  s->st.coop_tiles = s->n_coop;
  s->st.tmem_cols = s->tmem_cols;

  ctm.mark("stats");
  // initial bound sum_j E^j(lambda) (+ free term on the host)
  if ((st = energy(s))) return st;
  CK(cudaStreamSynchronize(s->stream), "sync");
  ctm.mark("energy sweep + sync");
  return FDOG_OK;
}

}  // namespace

namespace {

PrimalArgs primal_args(fdog_solver *s, int mode, int32_t round, double delta, uint64_t seed) {
  PrimalArgs a{};
  a.n_ell = s->n_ell;
  a.n_ell4 = s->n_ell4;
  a.n_csr = s->n_varlist;
  a.ell = s->d_ell;
  a.ell_var = s->d_ell_var;
  a.ell4 = s->d_ell4;
  a.ell4_var = s->d_ell4_var;
  a.csr_var = s->d_csr_var;
  a.var_ptr = s->d_var_ptr;
  a.var_slots = s->d_var_slots;
  a.n_elld_g = s->n_elld_g;
  for (int g = 0; g < s->n_elld_g; ++g) {
    a.elld_d[g] = s->elld_d[g];
    a.elld_n[g] = s->elld_n[g];
    a.elld_off[g] = s->elld_off[g];
  }
  a.elld = s->d_elld;
  a.elld_var = s->d_elld_var;
  a.delta_bar = s->d_delta[s->cur];
  a.lambda = s->d_lambda;
  a.x = s->d_x;
  a.undecided = s->d_undecided;
  a.mode = mode;
  a.round = round;
  a.delta = delta;
  a.seed = seed;
  return a;
}

fdog_status primal_step_impl(fdog_solver *s, int32_t round, double delta, uint64_t seed, int64_t *undecided,
                             uint8_t *x) {
  CK(cudaMemsetAsync(s->d_undecided, 0, sizeof(unsigned long long), s->stream), "memset");
  int e;
  {
    Timed t(s, kKPrimal);
    e = launch_primal(s->precision, primal_args(s, 0, round, delta, seed), s->stream);
  }
  if (e) return cuda_fail((cudaError_t)e, "primal classify");
  unsigned long long u = 0;
  CK(cudaMemcpyAsync(&u, s->d_undecided, sizeof u, cudaMemcpyDeviceToHost, s->stream), "D2H");
  if (x && s->n_vars > 0) CK(cudaMemcpyAsync(x, s->d_x, (size_t)s->n_vars, cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  if (x)
    for (int64_t i = 0; i < s->n_vars; ++i)
      if (s->plan->deg_global[i] == 0) x[i] = s->plan->cost[i] < 0;  // free variables (A13)
  *undecided = (int64_t)u;
  if (u == 0) return FDOG_OK;
  {
    Timed t(s, kKPrimal);
    e = launch_primal(s->precision, primal_args(s, 1, round, delta, seed), s->stream);
  }
  if (e) return cuda_fail((cudaError_t)e, "primal perturb");
  s->dist_state = 2;  // lambda changed: distances are recomputed before the next pass
  return FDOG_OK;
}

bool labeling_feasible(const fdog_solver *s, const uint8_t *x, int64_t *bad_row) {
  const int64_t m = (int64_t)s->plan->rel.size();
  for (int64_t j = 0; j < m; ++j) {
    int64_t acc = 0;
    for (int64_t q = s->plan->row_ptr[j]; q < s->plan->row_ptr[j + 1]; ++q) acc += (int64_t)s->plan->col_coef[q] * x[s->plan->col_var[q]];
    const int8_t r = s->plan->rel[j];
    const bool ok = r < 0 ? acc <= s->plan->rhs[j] : r > 0 ? acc >= s->plan->rhs[j] : acc == s->plan->rhs[j];
    if (!ok) {
      *bad_row = j;
      return false;
    }
  }
  return true;
}

}  // namespace

extern "C" {

void fdog_default_primal_options(fdog_primal_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->delta0 = 1.0;
  o->alpha = 1.2;
  o->inner = 5;
  o->max_rounds = 100;
  o->omega = 0.5;
}

fdog_status fdog_primal_step(fdog_solver *s, int32_t round, double delta, uint64_t seed, int64_t *undecided,
                             uint8_t *x, int64_t len) {
  if (!s || !undecided || (x && len < s->n_vars)) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  if (s->lifted) {
    set_error("primal rounding reads single-sided state; not in the lifted representation");
    return FDOG_ESTATE;
  }
  if (s->world > 1) {
    set_error("primal rounding is single-GPU in this version");
    return FDOG_ESTATE;
  }
  if (s->passes == 0) {
    set_error("primal rounding needs the min-marginals of at least one pass");
    return FDOG_ESTATE;
  }
  return primal_step_impl(s, round, delta, seed, undecided, x);
}

fdog_status fdog_round_primal(fdog_solver *s, const fdog_primal_options *opts, uint8_t *x, int64_t len,
                              int32_t *rounds, double *objective) {
  if (!s || !x || !rounds || !objective || len < s->n_vars) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  if (s->lifted) {
    set_error("primal rounding reads single-sided state; not in the lifted representation");
    return FDOG_ESTATE;
  }
  fdog_primal_options def;
  fdog_default_primal_options(&def);
  const fdog_primal_options *o = opts ? opts : &def;
  if (!(o->delta0 > 0) || !(o->alpha >= 1) || o->inner < 1 || o->max_rounds < 0 || !(o->omega > 0 && o->omega <= 1)) {
    set_error("invalid primal options");
    return FDOG_EINVAL;
  }
  if (s->world > 1) {
    set_error("primal rounding is single-GPU in this version");
    return FDOG_ESTATE;
  }
  fdog_status st;
  // snapshot of the dual state (restored unless keep_state)
  const size_t sb = (size_t)std::max<int64_t>(s->n_dev_slots, 1) * s->tsz;
  const size_t db = (size_t)std::max<int64_t>(s->n_dist, 1) * s->tsz;
  std::vector<void *> snap;
  auto cleanup = [&]() {
    if (!snap.empty()) cudaStreamSynchronize(s->stream);
    for (void *p : snap) dev_free(s, p);
  };
  const int cur0 = s->cur, ds0 = s->dist_state;
  const int64_t passes0 = s->passes;
  const bool dirty0 = s->lb_dirty, dz0 = s->dbar_zero;
  const size_t pb = (size_t)std::max(s->n_tiles, 1) * sizeof(double), lbb = 2 * sizeof(double);
  // (with record_mm also the min-marginals, so fdog_min_marginals after the
  // rounding returns those of the restored state's last pass)
  std::vector<void *> live = {s->d_lambda, s->d_delta[0], s->d_delta[1], s->d_dist, s->d_lb_part, s->d_lb};
  std::vector<size_t> sz = {sb, sb, sb, db, pb, lbb};
  if (s->record_mm) {
    live.push_back(s->d_m0);
    live.push_back(s->d_m1);
    sz.push_back(sb);
    sz.push_back(sb);
  }
  if (!o->keep_state) {
    for (size_t q = 0; q < live.size(); ++q) {
      void *pq = nullptr;
      cudaError_t e = dev_alloc(s, &pq, sz[q]);
      if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "device allocation (primal snapshot)");
      }
      snap.push_back(pq);
      e = cudaMemcpyAsync(pq, live[q], sz[q], cudaMemcpyDeviceToDevice, s->stream);
      if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "snapshot");
      }
    }
  }
  auto restore = [&]() -> fdog_status {
    if (o->keep_state) return FDOG_OK;
    for (size_t q = 0; q < live.size(); ++q)
      CK(cudaMemcpyAsync(live[q], snap[q], sz[q], cudaMemcpyDeviceToDevice, s->stream), "restore");
    CK(cudaStreamSynchronize(s->stream), "sync");
    s->cur = cur0;
    s->dist_state = ds0;
    s->passes = passes0;
    s->lb_dirty = dirty0;
    s->dbar_zero = dz0;
    return FDOG_OK;
  };
  if (s->passes == 0 && (st = fdog_iterate(s, o->inner, o->omega))) {
    restore();
    cleanup();
    return st;
  }
  double delta = o->delta0;
  int32_t round = 0;
  for (;; ++round) {
    int64_t und = 0;
    if ((st = primal_step_impl(s, round, delta, o->seed, &und, x))) break;
    if (und == 0) break;
    if (round + 1 > o->max_rounds) {
      set_error("primal rounding: %lld undecided variables after %d rounds", (long long)und, round);
      st = FDOG_ENOSOLUTION;
      break;
    }
    delta *= o->alpha;
    if ((st = fdog_iterate(s, o->inner, o->omega))) break;
  }
  *rounds = round;
  double obj = 0.0;
  for (int64_t i = 0; i < s->n_vars; ++i) obj += x[i] ? s->plan->cost[i] : 0.0;
  *objective = obj;
  fdog_status rs = restore();
  cleanup();
  if (st) return st;
  if (rs) return rs;
  int64_t bad = -1;
  if (!labeling_feasible(s, x, &bad)) {
    set_error("internal: labeling with all variables decided violates row %lld", (long long)bad);
    return FDOG_ESTATE;
  }
  return FDOG_OK;
}

fdog_status fdog_create_from_plan(const fdog_plan *plan, const fdog_options *opts, fdog_solver **out) {
  if (!plan || !out) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *out = nullptr;
  fdog_options def;
  fdog_default_options(&def);
  const fdog_options *o = opts ? opts : &def;
  fdog_solver *s = nullptr;
  try {
    s = new fdog_solver();
    fdog_status st = create_impl(plan_of(plan), o, s);
    if (st) {
      free_solver(s);
      return st;
    }
  } catch (const std::bad_alloc &) {
    free_solver(s);
    set_error("host out of memory");
    return FDOG_ENOMEM;
  }
  *out = s;
  return FDOG_OK;
}

fdog_status fdog_create(const fdog_problem *p, const fdog_options *opts, fdog_solver **out) {
  fdog_plan *plan = nullptr;
  fdog_status st = fdog_plan_create(p, opts, &plan);
  if (st) return st;
  st = fdog_create_from_plan(plan, opts, out);
  fdog_plan_destroy(plan);
  return st;
}

void fdog_destroy(fdog_solver *s) { free_solver(s); }

fdog_status fdog_pass(fdog_solver *s, int32_t forward, double omega) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (s->external && !s->peer) {
    set_error("external-exchange mode: use fdog_pass_begin / fdog_pass_end");
    return FDOG_ESTATE;
  }
  if (!(omega > 0.0 && omega <= 1.0)) {
    set_error("omega %g outside (0, 1]", omega);
    return FDOG_EINVAL;
  }
  return do_pass(s, forward != 0, omega);
}

fdog_status fdog_pass_seq(fdog_solver *s, int32_t forward, double omega) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (s->lifted) {
    set_error("the non-deferred variant is single-sided; not in the lifted representation");
    return FDOG_ESTATE;
  }
  if (!(omega > 0.0 && omega <= 1.0)) {
    set_error("omega %g outside (0, 1]", omega);
    return FDOG_EINVAL;
  }
  if (s->world > 1) {
    set_error("the non-deferred variant is single-GPU");
    return FDOG_ESTATE;
  }
  if (s->n_coop > 0) {
    set_error("the non-deferred variant walks 16-bit topology codes; BDDs wider than %d nodes per partition "
              "run the deferred passes only", kCoopWidth);
    return FDOG_EINVAL;
  }
  if (!s->dbar_zero) {
    set_error("a deferred correction is pending: fdog_finalize first");
    return FDOG_ESTATE;
  }
  return do_pass_seq(s, forward != 0, omega);
}

fdog_status fdog_iterate_seq(fdog_solver *s, int32_t n_iter, double omega) {
  if (!s || n_iter < 0) {
    set_error("null solver or negative n_iter");
    return FDOG_EINVAL;
  }
  if (n_iter == 0) return FDOG_OK;
  fdog_status st = fdog_pass_seq(s, 1, omega);  // validates the state; builds the schedule
  if (!st) st = fdog_pass_seq(s, 0, omega);
  if (st || n_iter == 1) return st;
  // the remaining iterations replay a CUDA graph of one (forward, backward)
  // iteration: hundreds of small level kernels, launch-latency bound otherwise
  // (the distances are in the state a forward pass expects after a backward one)
  if (!s->use_graphs || s->profile) {
    for (int32_t t = 1; t < n_iter; ++t) {
      st = fdog_pass_seq(s, 1, omega);
      if (!st) st = fdog_pass_seq(s, 0, omega);
      if (st) return st;
    }
    return FDOG_OK;
  }
  if (!s->seq_graph || s->seq_graph_omega != omega || s->seq_graph_cur != s->cur) {
    if (s->seq_graph) {
      cudaGraphExecDestroy(s->seq_graph);
      s->seq_graph = nullptr;
    }
    const int ds0 = s->dist_state;
    const int64_t passes0 = s->passes, launches0 = s->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    st = do_pass_seq(s, true, omega);
    if (!st) st = do_pass_seq(s, false, omega);
    cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&s->seq_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    s->seq_graph_omega = omega;
    s->seq_graph_cur = s->cur;
    s->seq_graph_launches = s->launches - launches0;
    s->dist_state = ds0;  // capture recorded the work without running it
    s->passes = passes0;
    s->launches = launches0;
  }
  for (int32_t t = 1; t < n_iter; ++t) CK(cudaGraphLaunch(s->seq_graph, s->stream), "cudaGraphLaunch");
  s->launches += s->seq_graph_launches * (n_iter - 1);
  s->passes += 2 * (int64_t)(n_iter - 1);
  s->dist_state = 0;
  s->dbar_zero = true;
  s->lb_dirty = true;
  return FDOG_OK;
}

fdog_status fdog_pass_begin(fdog_solver *s, int32_t forward, double omega) {
  if (!s || !(omega > 0.0 && omega <= 1.0)) {
    set_error("null solver or omega outside (0, 1]");
    return FDOG_EINVAL;
  }
  if (!s->external) {
    set_error("fdog_pass_begin needs the external-exchange mode (world > 1, no NCCL id)");
    return FDOG_ESTATE;
  }
  return pass_stage(s, forward != 0, omega, 0);
}

fdog_status fdog_pass_end(fdog_solver *s, int32_t forward, double omega) {
  if (!s || !(omega > 0.0 && omega <= 1.0)) {
    set_error("null solver or omega outside (0, 1]");
    return FDOG_EINVAL;
  }
  if (!s->external) {
    set_error("fdog_pass_end needs the external-exchange mode (world > 1, no NCCL id)");
    return FDOG_ESTATE;
  }
  return pass_stage(s, forward != 0, omega, 1);
}

fdog_status fdog_exchange_region(const fdog_solver *s, void **region, int64_t *bytes) {
  if (!s || !region || !bytes) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  if (!s->d_region) {
    set_error("no exchange region: the solver is not in the external-exchange mode");
    return FDOG_ESTATE;
  }
  *region = s->d_region;
  *bytes = (int64_t)(kRegionBuf + 2 * s->region_stride);
  return FDOG_OK;
}

fdog_status fdog_set_peer_regions(fdog_solver *s, int32_t world, void *const *regions, double timeout_s) {
  if (!s || !regions || !(timeout_s > 0.0)) {
    set_error("null argument or timeout <= 0");
    return FDOG_EINVAL;
  }
  if (!s->d_region) {
    set_error("peer exchange needs the external-exchange mode (world > 1, no NCCL id)");
    return FDOG_ESTATE;
  }
  if (world != s->world || world > kMaxPeers) {
    set_error("world %d: the solver's is %d (at most %d peers)", world, s->world, kMaxPeers);
    return FDOG_EINVAL;
  }
  if (regions[s->rank] != (void *)s->d_region) {
    set_error("regions[rank] must be this solver's own region");
    return FDOG_EINVAL;
  }
  if (s->passes != 0) {
    set_error("fdog_set_peer_regions must precede the first pass (the pass counters start at 0 on every rank)");
    return FDOG_ESTATE;
  }
  {
    const int e = preload_kernels(s->precision);
    if (e) return cuda_fail((cudaError_t)e, "kernel preload");
  }
  PeerArgs pa{};
  pa.world = world;
  pa.rank = s->rank;
  pa.timeout_ns = (unsigned long long)(timeout_s * 1e9);
  for (int k = 0; k < world; ++k) {
    if (!regions[k]) {
      set_error("null region of rank %d", k);
      return FDOG_EINVAL;
    }
    pa.region[k] = (const unsigned char *)regions[k];
  }
  s->peer_args = pa;
  s->peer = true;
  s->peer_par = 0;
  return FDOG_OK;
}

fdog_status fdog_peer_error(fdog_solver *s, int32_t *err) {
  if (!s || !err) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *err = 0;
  if (!s->d_region) return FDOG_OK;
  unsigned v = 0;
  CK(cudaMemcpyAsync(&v, s->d_region + 4, 4, cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  *err = (int32_t)v;
  return FDOG_OK;
}

fdog_status fdog_ipc_handle(void *dev_ptr, void *handle) {
  if (!dev_ptr || !handle) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dev_ptr), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == FDOG_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  return FDOG_OK;
}

fdog_status fdog_ipc_open(const void *handle, void **dev_ptr) {
  if (!handle || !dev_ptr) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return FDOG_OK;
}

fdog_status fdog_ipc_close(void *dev_ptr) {
  if (!dev_ptr) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  CK(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  return FDOG_OK;
}

fdog_status fdog_exchange_size(const fdog_solver *s, int64_t *n) {
  if (!s || !n) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *n = s->n_shared;
  return FDOG_OK;
}

fdog_status fdog_exchange_read(fdog_solver *s, double *out, int64_t len) {
  if (!s || (len > 0 && !out) || len < s->n_shared) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  if (s->n_shared == 0) return FDOG_OK;
  std::vector<unsigned char> buf((size_t)s->n_shared * s->tsz);
  CK(cudaMemcpyAsync(buf.data(), s->d_xbuf, buf.size(), cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  for (int32_t q = 0; q < s->n_shared; ++q)
    out[q] = s->precision == 64 ? ((double *)buf.data())[q] : (double)((float *)buf.data())[q];
  return FDOG_OK;
}

fdog_status fdog_exchange_write(fdog_solver *s, const double *in, int64_t len) {
  if (!s || (len > 0 && !in) || len != s->n_shared) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  if (s->n_shared == 0) return FDOG_OK;
  std::vector<unsigned char> buf((size_t)s->n_shared * s->tsz);
  for (int32_t q = 0; q < s->n_shared; ++q) {
    if (s->precision == 64) ((double *)buf.data())[q] = in[q];
    else ((float *)buf.data())[q] = (float)in[q];
  }
  CK(cudaMemcpyAsync(s->d_xbuf, buf.data(), buf.size(), cudaMemcpyHostToDevice, s->stream), "H2D");
  CK(cudaStreamSynchronize(s->stream), "sync");
  return FDOG_OK;
}

fdog_status fdog_iterate(fdog_solver *s, int32_t n_iter, double omega) {
  if (!s || n_iter < 0) {
    set_error("null solver or negative n_iter");
    return FDOG_EINVAL;
  }
  if (s->external && !s->peer) {
    set_error("external-exchange mode: use fdog_pass_begin / fdog_pass_end");
    return FDOG_ESTATE;
  }
  if (!(omega > 0.0 && omega <= 1.0)) {
    set_error("omega %g outside (0, 1]", omega);
    return FDOG_EINVAL;
  }
  if (s->use_fused && !s->profile && s->world == 1 && s->dist_state == 0 && n_iter > 0) {
    // 2 n_iter passes in one launch; delta_bar ends in the same buffer
    const SweepArgs sa = sweep_args(s, omega);
    const AvgArgs aa = avg_args(s);
    const int e = launch_fused_small(s->precision, s->record_mm, sa, aa, n_iter, s->n_dev_slots, s->n_dist,
                                     s->fused_smem, s->stream);
    if (e) return cuda_fail((cudaError_t)e, "fused launch");
    s->launches += 1;
    s->passes += 2 * (int64_t)n_iter;
    s->lb_dirty = true;
    s->dbar_zero = false;
    return FDOG_OK;
  }
  // CUDA graph of one iteration: used when the passes alternate normally and
  // no per-kernel events are requested.  With world > 1 the graph holds the
  // exchange too (ncclAllReduce is captured, or the peer-memory kernels), forked
  // onto xstream and joined before the boundary tiles' sweep.
  const bool graphs = s->use_graphs && !s->profile && (s->rc || s->dist_state == 0) && n_iter > 0;
  if (graphs) {
    if (!s->graph || s->graph_omega != omega || s->graph_cur != s->cur) {
      if (s->graph) {
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
      }
      const int cur0 = s->cur, ds0 = s->dist_state;
      const int64_t passes0 = s->passes, launches0 = s->launches;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
      fdog_status st = do_pass(s, true, omega);
      if (!st) st = do_pass(s, false, omega);
      cudaError_t e = cudaStreamEndCapture(s->stream, &g);
      if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      e = cudaGraphInstantiate(&s->graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      s->graph_omega = omega;
      s->graph_cur = cur0;
      s->graph_launches = s->launches - launches0;
      s->cur = cur0;  // capture recorded the work without running it
      s->dist_state = ds0;
      s->passes = passes0;
      s->launches = launches0;
    }
    for (int32_t t = 0; t < n_iter; ++t) CK(cudaGraphLaunch(s->graph, s->stream), "cudaGraphLaunch");
    s->launches += s->graph_launches * n_iter;
    s->passes += 2 * (int64_t)n_iter;
    s->dist_state = 0;
    s->lb_dirty = true;  // the replayed sweeps wrote new per-tile partials
    s->dbar_zero = false;
    return FDOG_OK;
  }
  for (int32_t t = 0; t < n_iter; ++t) {
    fdog_status st = do_pass(s, true, omega);
    if (st) return st;
    st = do_pass(s, false, omega);
    if (st) return st;
  }
  return FDOG_OK;
}

fdog_status fdog_lower_bound(fdog_solver *s, double *out) {
  if (!s || !out) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  if (s->lb_dirty) {
    int e;
    {
      Timed t(s, kKLbReduce);
      e = launch_lb_reduce(s->d_lb_part, s->n_tiles, s->d_lb, s->stream);
    }
    if (e) return cuda_fail((cudaError_t)e, "lb_reduce launch");
    s->lb_dirty = false;
  }
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, s->d_lb, sizeof(double), cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  double tot = v + s->free_term;
  if ((s->world > 1 && !s->external) || s->nccl.comm) {
    // scalar allreduce of the per-rank partials (fp64)
    double *d = s->d_lb + 1;  // scratch slot for the cross-rank sum
    CK(cudaMemcpyAsync(d, &tot, sizeof(double), cudaMemcpyHostToDevice, s->stream), "H2D");
    int r = s->nccl.allreduce(d, d, 1, kNcclFloat64, kNcclSum, s->nccl.comm, s->stream);
    if (r) {
      set_error("ncclAllReduce(lb): %s", s->nccl.errstr ? s->nccl.errstr(r) : "error");
      return FDOG_ENCCL;
    }
    CK(cudaMemcpyAsync(&tot, d, sizeof(double), cudaMemcpyDeviceToHost, s->stream), "D2H");
    CK(cudaStreamSynchronize(s->stream), "sync");
  }
  *out = tot;
  return FDOG_OK;
}

fdog_status fdog_finalize(fdog_solver *s) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  int e;
  {
    Timed t(s, kKAddDeferred);
    e = s->lifted ? launch_add_deferred_lifted(s->precision, s->n_dev_slots, s->d_lambda, s->d_lam0,
                                               s->d_delta[s->cur], s->stream)
                  : launch_add_deferred(s->precision, s->n_dev_slots, s->d_lambda, s->d_delta[s->cur], s->stream);
  }
  if (e) return cuda_fail((cudaError_t)e, "add_deferred");
  s->dbar_zero = true;
  return energy(s);
}

fdog_status fdog_finalize_averaged(fdog_solver *s) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (s->lifted) {
    set_error("the averaged final correction is not defined for the lifted representation");
    return FDOG_ESTATE;
  }
  if (s->external && !s->peer) {
    set_error("fdog_finalize_averaged needs world == 1, the NCCL or the peer-memory exchange");
    return FDOG_ESTATE;
  }
  // the averaging kernel (+ exchange) writes avg_i into every slot of the other
  // delta buffer; lambda += that buffer, then both buffers are zero
  s->avg_full = true;
  fdog_status st = run_avg(s);
  if (!st) st = run_exchange(s, s->stream);
  s->avg_full = false;
  if (st) return st;
  int e;
  {
    Timed t(s, kKAddDeferred);
    e = launch_add_deferred(s->precision, s->n_dev_slots, s->d_lambda, s->d_delta[s->cur ^ 1], s->stream);
  }
  if (e) return cuda_fail((cudaError_t)e, "add_deferred");
  CK(cudaMemsetAsync(s->d_delta[s->cur], 0, (size_t)std::max<int64_t>(s->n_dev_slots, 1) * s->tsz, s->stream), "memset");
  s->dbar_zero = true;
  return energy(s);
}

fdog_status fdog_num_slots(const fdog_solver *s, int64_t *out) {
  if (!s || !out) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *out = (int64_t)s->plan->canon_slot.size();
  return FDOG_OK;
}

fdog_status fdog_slot_index(const fdog_solver *s, int32_t *con, int32_t *pos, int64_t len) {
  if (!s || !con || !pos || len < (int64_t)s->plan->canon_slot.size()) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  std::copy(s->plan->canon_con.begin(), s->plan->canon_con.end(), con);
  std::copy(s->plan->canon_pos.begin(), s->plan->canon_pos.end(), pos);
  return FDOG_OK;
}

fdog_status fdog_get_lambda(fdog_solver *s, double *out, int64_t len) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (s->lifted) {  // the original-space lambda = lambda^1 - lambda^0
    const int e = launch_lifted_diff(s->precision, s->n_dev_slots, s->d_lambda, s->d_lam0, s->d_lam_out, s->stream);
    if (e) return cuda_fail((cudaError_t)e, "lifted diff");
    s->launches++;
    return fetch_slots(s, s->d_lam_out, out, len);
  }
  return fetch_slots(s, s->d_lambda, out, len);
}

fdog_status fdog_get_lifted(fdog_solver *s, double *lam0, double *lam1, int64_t len) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (!s->lifted) {
    set_error("fdog_get_lifted needs the lifted representation (fdog_options::lifted)");
    return FDOG_ESTATE;
  }
  fdog_status st = fetch_slots(s, s->d_lam0, lam0, len);
  return st ? st : fetch_slots(s, s->d_lambda, lam1, len);
}

fdog_status fdog_get_deferred(fdog_solver *s, double *out, int64_t len) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  return fetch_slots(s, s->d_delta[s->cur], out, len);
}

fdog_status fdog_min_marginals(fdog_solver *s, double *m0, double *m1, int64_t len) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (!s->record_mm || s->passes == 0) {
    set_error("min_marginals needs record_mm and at least one pass");
    return FDOG_ESTATE;
  }
  fdog_status st = fetch_slots(s, s->d_m0, m0, len);
  return st ? st : fetch_slots(s, s->d_m1, m1, len);
}

fdog_status fdog_set_state(fdog_solver *s, const double *lambda, const double *delta, int64_t len) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  if (s->lifted) {
    set_error("fdog_set_state takes single-sided lambda; not in the lifted representation");
    return FDOG_ESTATE;
  }
  fdog_status st;
  if (lambda && (st = put_slots(s, s->d_lambda, lambda, len))) return st;
  if (delta && (st = put_slots(s, s->d_delta[s->cur], delta, len))) return st;
  if (delta) {
    bool z = true;
    for (int64_t q = 0; q < len && z; ++q) z = delta[q] == 0.0;
    s->dbar_zero = z;
  }
  if ((st = energy(s))) return st;
  if (!s->dbar_zero) {
    // the lifted bound (A7) keeps the outstanding sum_slots min(delta_bar, 0)
    Timed t(s, kKLbReduce);
    const int e = launch_lb_deferred(s->precision, s->d_tiles, s->n_tiles, s->d_delta[s->cur], s->d_lb_part, s->stream);
    if (e) return cuda_fail((cudaError_t)e, "lb_deferred launch");
  }
  return FDOG_OK;
}

fdog_status fdog_debug_trace(fdog_solver *s, uint64_t *out, int64_t cap, int64_t *n) {
  if (!s || !n) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *n = s->d_trace ? (int64_t)s->grid * (s->block / 32) : 0;
  if (!out || !s->d_trace) return FDOG_OK;
  if (cap < *n) {
    set_error("capacity %lld < %lld warps", (long long)cap, (long long)*n);
    return FDOG_EINVAL;
  }
  CK(cudaMemcpyAsync(out, s->d_trace, (size_t)*n * 32, cudaMemcpyDeviceToHost, s->stream), "D2H");
  CK(cudaStreamSynchronize(s->stream), "sync");
  return FDOG_OK;
}

fdog_status fdog_stats(const fdog_solver *s, fdog_stats_t *out) {
  if (!s || !out) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  *out = s->st;
  out->launches = s->launches;
  return FDOG_OK;
}

fdog_status fdog_profile(fdog_solver *s, fdog_kernel_time *out, int32_t cap, int32_t *n) {
  if (!s || !n) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  CK(cudaStreamSynchronize(s->stream), "sync");
  for (auto &e : s->events) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e.a, e.b), "cudaEventElapsedTime");
    s->prof_ms[e.kernel] += ms;
    s->prof_n[e.kernel] += 1;
    s->event_pool.push_back(e.a);
    s->event_pool.push_back(e.b);
  }
  s->events.clear();
  int32_t k = 0;
  for (int q = 0; q < kKCount; ++q) {
    if (!s->prof_n[q]) continue;
    if (out && k < cap) out[k] = {kKernelNames[q], s->prof_ms[q], s->prof_n[q], s->bytes[q]};
    ++k;
  }
  *n = k;
  return FDOG_OK;
}

fdog_status fdog_profile_enable(fdog_solver *s, int32_t on) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  CK(cudaStreamSynchronize(s->stream), "sync");
  s->profile = on != 0;
  return FDOG_OK;
}

fdog_status fdog_profile_reset(fdog_solver *s) {
  if (!s) {
    set_error("null solver");
    return FDOG_EINVAL;
  }
  CK(cudaStreamSynchronize(s->stream), "sync");
  for (auto &e : s->events) {
    s->event_pool.push_back(e.a);
    s->event_pool.push_back(e.b);
  }
  s->events.clear();
  for (int q = 0; q < kKCount; ++q) {
    s->prof_ms[q] = 0;
    s->prof_n[q] = 0;
  }
  return FDOG_OK;
}

}  // extern "C"
