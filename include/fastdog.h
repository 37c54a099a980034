/*
 * fastdog.h -- C ABI of the B200-native hot path of FastDOG (arXiv 2111.10270):
 * Alg. "Parallel Deferred Min-Marginal Averaging" over one
 * quasi-reduced ordered BDD per constraint (Def. BDD).
 *
 * Citations "P:n" are lines of the paper text; readings A1..A16 of
 * ambiguous passages are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Every function returns fdog_status; no C++ exception crosses the ABI.
 *     On error, fdog_last_error() returns a thread-local message.
 *   - Input arrays are HOST pointers borrowed for the duration of the call
 *     (copied).  Output arrays are caller-allocated HOST arrays with an
 *     explicit length; a length that is too small returns FDOG_EINVAL.
 *   - A solver handle owns all of its device memory (obtained through
 *     opts.dev_alloc when given, e.g. torch's caching allocator) and its
 *     NCCL communicator when world > 1; fdog_destroy frees them.  A handle is
 *     not thread-safe.  Device work is stream-ordered on opts.stream;
 *     getters synchronise that stream.
 *   - Slot = one multiplier lambda_i^j, i.e. one (constraint j, position h
 *     in I_j) pair.  Getters return slots in canonical order: j ascending,
 *     h ascending, over the BDDs held by this rank.
 */
#ifndef FASTDOG_H
#define FASTDOG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDOG_OK = 0,
  FDOG_EINVAL = 1,      /* bad argument / length / omega outside (0,1] (A14)       */
  FDOG_EINFEASIBLE = 2, /* some row has an empty feasible set X_j           */
  FDOG_ENOMEM = 3,      /* host or device allocation failed                         */
  FDOG_ECUDA = 4,       /* CUDA runtime error (message in fdog_last_error)          */
  FDOG_ENCCL = 5,       /* NCCL error (multi-GPU)                                   */
  FDOG_ESTATE = 6,      /* call not valid in this state (e.g. min_marginals w/o record_mm) */
  FDOG_ETOOBIG = 7,     /* a BDD exceeds the kernels' on-chip limits                */
  FDOG_ENOSOLUTION = 8  /* primal rounding: no consensus within max_rounds           */
} fdog_status;

/* Binary program (BP) P:555-565 in the row form of Example ILP P:567-577.
 * Row j: sum_{p in [row_ptr[j], row_ptr[j+1])} col_coef[p] * x[col_var[p]]  rel[j]  rhs[j].
 * col_var strictly ascending within a row (the BDD variable order, A12);
 * col_coef nonzero; rel: -1 "<=", 0 "==", +1 ">=".  Layout: CSR, host memory. */
typedef struct {
  int32_t n_vars;
  const double *cost;      /* c, length n_vars                         */
  int32_t n_cons;
  const int64_t *row_ptr;  /* length n_cons + 1                        */
  const int32_t *col_var;  /* length row_ptr[n_cons]                   */
  const int32_t *col_coef; /* length row_ptr[n_cons]                   */
  const int8_t *rel;       /* length n_cons                            */
  const int64_t *rhs;      /* length n_cons                            */
} fdog_problem;

typedef struct {
  int32_t precision;        /* 32 (fp32 sweeps, fp64 bound accumulation) or 64  */
  int32_t device;           /* CUDA device ordinal                              */
  double clamp;             /* C substituted for an infinite m1-m0 (A5); <= 0:
                               default 1e4 * (1 + max_i |c_i|)                  */
  int32_t record_mm;        /* 1: store m0, m1 per slot each pass (parity)     */
  int32_t profile;          /* 1: CUDA events around every launch (fdog_profile) */
  int32_t rank, world;      /* BDD shard of this process; world == 1: no NCCL   */
  const void *nccl_unique_id; /* 128-byte ncclUniqueId, required if world > 1   */
  const char *nccl_library; /* path of libnccl.so.2 to dlopen (NULL: default)   */
  void *stream;             /* cudaStream_t to run on; NULL: solver-owned stream */
  int32_t host_threads;     /* threads for host BDD compilation (<= 0: all)    */
  const int32_t *row_owner; /* optional (world > 1): rank of every row, length
                               n_cons, identical on every rank; NULL: the
                               locality-aware sharder (bundles of rows joined by
                               |J_i| = 2 variables, ordered by their shared
                               variables, cut by BDD node count) */
  int32_t lifted;           /* 1: lifted two-sided storage: per slot
                               lambda^{j,0} (0-arcs) and lambda^{j,1} (1-arcs),
                               updated by reading A8; the bound is the plain sum
                               of per-BDD shortest paths (no sum min(delta_bar, 0)
                               term: exact with forced variables, A5).  world 1;
                               every tile runs from global memory (lane-serial or
                               node-parallel); no primal rounding, non-deferred
                               passes, set_state or averaged finalize.          */
  /* Caller-owned device memory (north_star: "PyTorch is used only for device
     memory, streams and process groups").  If dev_alloc is set, every device
     buffer a solver holds -- the plan image with the runtime state, the
     non-deferred schedule, the primal-rounding snapshot -- is obtained by
     dev_alloc(bytes, device, stream, alloc_ctx) (stream: the solver's stream,
     the caller's opts.stream or the solver-owned one; first used on it after
     the call returns), and returned by dev_free(ptr, device, stream,
     alloc_ctx) only after that stream has been synchronised (fdog_destroy,
     end of fdog_round_primal), so the allocator may hand the memory to any
     stream afterwards.  A NULL
     return fails the call with FDOG_ENOMEM.  The one exception is the
     peer-exchange region (external-exchange mode), a cudaMalloc of its own
     so that one CUDA IPC handle maps exactly it.  dev_alloc NULL: cudaMalloc
     / cudaFree.  The Python binding passes torch's caching allocator. */
  void *(*dev_alloc)(size_t bytes, int32_t device, void *stream, void *alloc_ctx);
  void (*dev_free)(void *ptr, int32_t device, void *stream, void *alloc_ctx);
  void *alloc_ctx;
} fdog_options;

/* Sizes of this rank's part of the problem. */
typedef struct {
  int64_t bdds;          /* BDDs (non-empty rows) on this rank                        */
  int64_t nodes;         /* non-terminal BDD nodes (A12)                              */
  int64_t arcs;          /* 2 * nodes (arcs to bottom included)                */
  int64_t slots;         /* multipliers lambda_i^j                                    */
  int64_t vars_local;    /* variables with >= 1 slot on this rank                     */
  int64_t vars_shared;   /* of those, variables also held by another rank             */
  int64_t free_vars;     /* |J_i| = 0 (A13)                                           */
  int64_t shapes;        /* distinct compiled BDD topologies                          */
  int64_t tiles;         /* 32-BDD warp tiles                                         */
  int64_t tiles_shared_topology; /* tiles whose 32 BDDs share one topology           */
  int64_t padded_slots;  /* device slots incl. padding lanes                          */
  int64_t device_bytes;  /* device memory held by the solver                          */
  int64_t launches;      /* kernels launched by this handle so far                    */
  int32_t max_hops;      /* max |I_j|                                                 */
  int32_t max_width;     /* max partition size |P_h|                                  */
  int64_t staged_tiles;  /* tiles staged on chip by TMA (the rest run from global)    */
  int32_t sweep_grid, sweep_block; /* persistent sweep launch configuration           */
  int64_t sweep_smem_per_warp;     /* bytes of shared memory per warp                 */
  int32_t sweep_streaming;         /* 1: passes use the streaming sweep kernel;
                                      2: the chunked kernel (rows too long to stage)    */
  int64_t h2d_bytes;               /* host->device bytes copied by create             */
  int32_t fused_small;             /* 1: fdog_iterate runs all its iterations in one
                                      single-CTA launch (small narrow problems);
                                      2: same, state resident in shared memory         */
  int32_t sweep_recompute;         /* 1: the passes recompute the opposite-direction
                                      distances on chip (no per-node HBM traffic)     */
  int64_t tile_pairs;              /* variables with |J_i| = 2 whose two slots share a
                                      tile: averaged on chip by the sweep (solver: only
                                      when the sweep path supports it; plan: eligible) */
  int64_t interior_tiles;          /* world > 1: tiles holding no exchanged variable,
                                      swept while the exchange runs (= tiles if world 1) */
  int64_t coop_tiles;              /* one-BDD tiles swept node-parallel by a warp
                                      (a partition wider than 32 nodes)              */
  int32_t tmem_cols;               /* > 0: the recompute design keeps the distances of
                                      its 32-row tiles in tensor memory (columns per
                                      sweep CTA); 0: shared memory                    */
} fdog_stats_t;

typedef struct fdog_plan fdog_plan;     /* host-side compiled + packed problem */
typedef struct fdog_solver fdog_solver; /* device-resident solver state        */

void fdog_default_options(fdog_options *opts);

/* ---- host setup (no GPU needed) -------------------------------------- */
/* Compile every row of this rank's shard into a quasi-reduced ordered BDD
 * (host compiler "B") and pack them into
 * the device layout.  Only opts->rank, world, host_threads, row_owner are read. */
fdog_status fdog_plan_create(const fdog_problem *p, const fdog_options *opts, fdog_plan **out);
void fdog_plan_destroy(fdog_plan *plan);
fdog_status fdog_plan_stats(const fdog_plan *plan, fdog_stats_t *out);
/* Export BDD j (global row index) if held by this plan: hop_start[k+1],
 * lo[n], hi[n] with successor codes node index within the BDD, -1 bottom,
 * -2 top.  *k and *n_nodes are always written; arrays only if cap_nodes >= n
 * and cap_hops >= k (otherwise FDOG_EINVAL after writing the sizes). */
fdog_status fdog_plan_bdd(const fdog_plan *plan, int32_t j, int32_t *k, int32_t *n_nodes,
                          int32_t *hop_start, int32_t *lo, int32_t *hi, int32_t cap_hops,
                          int32_t cap_nodes);
/* Device slot of every canonical slot (j ascending, h ascending) of this rank
 * (layout inspection; len >= the rank's slot count). */
fdog_status fdog_plan_slot_map(const fdog_plan *plan, int64_t *dev_slot, int64_t len);
/* Tile descriptors for inspection: 6 values per tile (kind bits -- 0 per-lane
 * topology, 1 staged, 2 arc-mask records, 3 chain middle, 4 root/join ends --,
 * partitions K, lanes L, valid lanes, nodes per lane, first device slot);
 * *n = number of tiles; desc may be NULL to query *n; cap in tiles. */
fdog_status fdog_plan_tiles(const fdog_plan *plan, int64_t *desc, int64_t cap, int64_t *n);
/* 64-bit FNV-1a digest of every packed array and the device image (plans
 * are deterministic: the same problem and options give the same digest for
 * any host thread count). */
fdog_status fdog_plan_digest(const fdog_plan *plan, uint64_t *out);
/* Global row -> owning rank for every row (length n_cons). */
fdog_status fdog_plan_owner(const fdog_plan *plan, int32_t *owner, int64_t len);
/* Ascending global indices of the variables exchanged between ranks (held by
 * >= 2 ranks; identical on every rank).  *n = their number; vars is written
 * if cap >= *n (may be NULL to query the size). */
fdog_status fdog_plan_shared_vars(const fdog_plan *plan, int32_t *vars, int64_t cap, int64_t *n);

/* ---- device solver ------------------------------------------------------ */
/* fdog_create = fdog_plan_create + fdog_create_from_plan + fdog_plan_destroy.
 * Initialises lambda_i^j = c_i/|J_i| (A9), mbar = 0 and the
 * lower bound sum_j E^j(lambda^j) + sum_free min(c_i, 0). */
fdog_status fdog_create(const fdog_problem *p, const fdog_options *opts, fdog_solver **out);
/* Upload a plan (host -> device copies inside) and initialise.  The plan may
 * be destroyed afterwards. */
fdog_status fdog_create_from_plan(const fdog_plan *plan, const fdog_options *opts,
                                  fdog_solver **out);
void fdog_destroy(fdog_solver *s);

/* n_iter x [averaging -> forward pass -> mbar<-m -> averaging -> backward pass
 * -> mbar<-m] (A2); asynchronous on the stream.  omega in (0,1]. */
fdog_status fdog_iterate(fdog_solver *s, int32_t n_iter, double omega);
/* One pass only: forward (1, ascending) or backward (0). */
fdog_status fdog_pass(fdog_solver *s, int32_t forward, double omega);
/* Non-deferred (sequential) min-marginal averaging, P:660-661 ("if mbar <- m,
 * (dual_update) matches the update from [lange2021efficient]"):
 * variables are visited in ascending (forward) / descending (backward) global
 * order; at variable i every j in J_i computes m_ij at its current lambda^j and
 * all update at once, lambda_i^j += -omega d_ij + mean_k omega d_ik.  Run as a
 * level schedule (variables of one level share no BDD): one kernel per level,
 * the schedule built on the first call.  Single-GPU (FDOG_ESTATE if world > 1);
 * needs delta_bar = 0 (fresh solver, after fdog_finalize, or after another _seq
 * pass; else FDOG_ESTATE).  Leaves delta_bar = 0 and lower_bound = sum_j E^j.
 * fdog_iterate_seq: n x (forward, backward). */
fdog_status fdog_pass_seq(fdog_solver *s, int32_t forward, double omega);
fdog_status fdog_iterate_seq(fdog_solver *s, int32_t n_iter, double omega);
/* External exchange (world > 1 with nccl_unique_id == NULL): the caller sums
 * the exchange vectors across ranks itself (e.g. torch.distributed, or several
 * rank solvers in one process).  A pass is then two calls:
 *   fdog_pass_begin  -- deferred averaging; this rank's partial sums of the
 *                       exchanged variables are in the exchange vector;
 *   (caller: exchange vector <- sum over ranks, via fdog_exchange_read/write)
 *   fdog_pass_end    -- averages of the exchanged variables + the sweep.
 * fdog_iterate returns FDOG_ESTATE in this mode (unless the peer exchange
 * below is set), and fdog_lower_bound returns this rank's part of the bound
 * (the caller sums it). */
fdog_status fdog_pass_begin(fdog_solver *s, int32_t forward, double omega);
fdog_status fdog_pass_end(fdog_solver *s, int32_t forward, double omega);
/* Number of exchanged variables (identical on every rank), and host copies of
 * the exchange vector (fdog_plan_shared_vars order) as double. */
fdog_status fdog_exchange_size(const fdog_solver *s, int64_t *n);
fdog_status fdog_exchange_read(fdog_solver *s, double *out, int64_t len);
fdog_status fdog_exchange_write(fdog_solver *s, const double *in, int64_t len);

/* Peer-memory exchange (external-exchange mode; SURVEY §8(a) a4 without NCCL):
 * the ranks exchange the partial sums of the shared variables through each
 * other's device memory over NVLink instead of an allreduce.
 *   fdog_exchange_region  -- this solver's exchange region (device memory,
 *       one allocation of *bytes: pass counter at byte 0, error word at 4,
 *       two partial-sum buffers from byte 256).  Share it with the peers: in
 *       one process as the plain pointer, across processes through
 *       fdog_ipc_handle / fdog_ipc_open.
 *   fdog_set_peer_regions -- regions[k] = rank k's region as a device pointer
 *       valid in this process (regions[rank] = the own one), before the first
 *       pass.  From then on fdog_pass / fdog_iterate do the whole pass on the
 *       device: averaging, publish (system-scope release of the pass
 *       counter), wait until every peer has published the same pass, sum the
 *       peers' partials in rank order (every rank gets bit-identical averages),
 *       sweep.  A peer that does not publish within timeout_s seconds sets the
 *       error word (fdog_peer_error) instead of hanging the device; the
 *       results of that pass are then invalid.  fdog_pass_begin publishes,
 *       fdog_pass_end waits, so one thread may drive several ranks of one
 *       process by calling every begin before any end.  fdog_lower_bound
 *       still returns this rank's part.
 * Ownership: the region belongs to the solver and is freed by fdog_destroy;
 * a rank may destroy its solver only after every peer has finished its last
 * pass (e.g. a barrier), and an importer closes its mappings with
 * fdog_ipc_close.  fdog_set_peer_regions also loads every kernel a pass can
 * launch (a lazy first-launch load would wait for the device, where a peer's
 * kernel may be spinning).
 * Errors: FDOG_ESTATE outside the external-exchange mode or after a pass;
 * FDOG_EINVAL for a wrong world size (at most 16), a null region or a foreign
 * own region. */
#define FDOG_IPC_HANDLE_BYTES 64
fdog_status fdog_exchange_region(const fdog_solver *s, void **region, int64_t *bytes);
fdog_status fdog_set_peer_regions(fdog_solver *s, int32_t world, void *const *regions, double timeout_s);
/* *err = 1 if a peer-exchange wait timed out (synchronises the stream). */
fdog_status fdog_peer_error(fdog_solver *s, int32_t *err);
/* CUDA IPC of a device allocation (handle: FDOG_IPC_HANDLE_BYTES bytes);
 * fdog_ipc_open maps a handle of another process (peer access enabled). */
fdog_status fdog_ipc_handle(void *dev_ptr, void *handle);
fdog_status fdog_ipc_open(const void *handle, void **dev_ptr);
fdog_status fdog_ipc_close(void *dev_ptr);

/* Lower bound of the last completed pass (A7): sum_j E^j(lambda^j) +
 * sum_slots min(delta_bar, 0) + sum_free min(c_i, 0); summed over ranks.
 * Synchronises the stream. */
fdog_status fdog_lower_bound(fdog_solver *s, double *out);
/* Final correction P:650-652 (per slot, A11): lambda += delta_bar,
 * delta_bar = 0; the bound becomes sum_j E^j(lambda^j). */
fdog_status fdog_finalize(fdog_solver *s);
/* Final correction read as "a min-marginal averaging step" (P:673 prose, the
 * alternative of reading A11): lambda_i^j += (1/|J_i|) sum_k delta_bar_ik,
 * delta_bar = 0.  Also dual feasible.  world == 1, NCCL or peer-memory mode
 * (a collective: every rank calls it). */
fdog_status fdog_finalize_averaged(fdog_solver *s);

fdog_status fdog_num_slots(const fdog_solver *s, int64_t *out);
/* (j, h) of every canonical slot. */
fdog_status fdog_slot_index(const fdog_solver *s, int32_t *con, int32_t *pos, int64_t len);
/* Current lambda_i^j (not finalized), canonical slot order. */
fdog_status fdog_get_lambda(fdog_solver *s, double *out, int64_t len);
/* delta_bar = omega * clamp(mbar1 - mbar0) of the last pass (A10). */
fdog_status fdog_get_deferred(fdog_solver *s, double *out, int64_t len);
/* m0, m1 (Eq. MM) recorded during the last pass; needs record_mm. */
fdog_status fdog_min_marginals(fdog_solver *s, double *m0, double *m1, int64_t len);
/* Overwrite (lambda, delta_bar) -- checkpoint/resume; either may be NULL. */
fdog_status fdog_set_state(fdog_solver *s, const double *lambda, const double *delta, int64_t len);
/* Lifted mode only: lambda^{j,0} and lambda^{j,1} per slot, canonical order
 * (fdog_get_lambda returns lambda^1 - lambda^0).  FDOG_ESTATE
 * without opts.lifted; FDOG_EINVAL if len < slots. */
fdog_status fdog_get_lifted(fdog_solver *s, double *lam0, double *lam1, int64_t len);
fdog_status fdog_stats(const fdog_solver *s, fdog_stats_t *out);
/* Debug (solver created with FDOG_TRACE=1): per warp of the TMA-staged sweep,
 * {start, end (globaltimer ns), tiles processed, SM id} of the last sweep;
 * *n = warps (0 without tracing); cap in warps. */
fdog_status fdog_debug_trace(fdog_solver *s, uint64_t *out, int64_t cap, int64_t *n);

/* Per-kernel device time (opts.profile = 1): names[i] (static strings),
 * total milliseconds and launch counts since the last reset.  Synchronises. */
typedef struct {
  const char *name;
  double ms;
  int64_t launches;
  double bytes_per_launch; /* algorithmic bytes of one launch */
} fdog_kernel_time;
fdog_status fdog_profile(fdog_solver *s, fdog_kernel_time *out, int32_t cap, int32_t *n);
fdog_status fdog_profile_reset(fdog_solver *s);
/* Turn the per-launch CUDA events on (1) or off (0).  With events on,
 * fdog_iterate launches kernels one by one; with events off (and world == 1)
 * it replays a CUDA graph of one iteration. */
fdog_status fdog_profile_enable(fdog_solver *s, int32_t on);

/* ---- primal rounding: Alg. "Perturbation Primal Rounding" --
 * Signs of m1 - m0 are read from the min-marginals of the last pass
 * (delta_bar = omega * clamp(m1 - m0)).  The loop runs while some variable is
 * undecided -- its subproblems do not all strictly favour one value (reading
 * R1) -- perturbing lambda per variable by +delta / -delta /
 * r*delta / sign(d_i)|r|delta, r ~ U[-delta, delta] from the
 * counter-based generator splitmix64(seed, round, i), delta *= alpha,
 * then `inner` iterations of Alg. 1.  Defaults delta0 = 1.0,
 * alpha = 1.2, inner = 5, max_rounds = 100, omega = 0.5.  world == 1. */
typedef struct {
  double delta0;
  double alpha;
  int32_t inner;
  int32_t max_rounds;
  uint64_t seed;
  double omega;
  int32_t keep_state;  /* 0: restore the dual state (lambda, delta_bar, bound) afterwards */
} fdog_primal_options;
void fdog_default_primal_options(fdog_primal_options *opts);
/* One classification (+ perturbation when *undecided > 0) step.  x: length
 * n_vars host array receiving x_i = 1 iff m1 < m0 in every subproblem
 * (free variables: x_i = [c_i < 0]). */
fdog_status fdog_primal_step(fdog_solver *s, int32_t round, double delta, uint64_t seed, int64_t *undecided,
                             uint8_t *x, int64_t len);
/* The full rounding loop.  On success x is a labeling that satisfies every
 * constraint (checked on the host), *objective = <c, x>, *rounds = the number
 * of perturbation rounds.  FDOG_ENOSOLUTION: no consensus within max_rounds
 * (x holds the last labeling). */
fdog_status fdog_round_primal(fdog_solver *s, const fdog_primal_options *opts, uint8_t *x, int64_t len,
                              int32_t *rounds, double *objective);

const char *fdog_last_error(void);
int32_t fdog_version(void);

#ifdef __cplusplus
}
#endif
#endif
