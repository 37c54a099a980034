// plan.cpp -- host setup of the hot path (untimed):
//   * compiler "B": linear row -> quasi-reduced ordered BDD (Def. BDD P:241-257,
//     canonical form P:273-277, reading A12) by canonical residual classes
//     computed from the suffix-sum sets (a different algorithm from the
//     oracle's compiler "A");
//   * sharder: contiguous row ranges per rank balanced by row length;
//   * packer: rows -> 32-lane warp tiles in the hop-major SoA layout of
//     DESIGN.md §5 (partition-contiguous per BDD, made tile-local),
//     slot arrays, CSR variable -> slots (J_i).
#include <algorithm>
#include <numeric>
#include <array>
#include <initializer_list>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>

#include <cuda_runtime.h>

#include "internal.h"

namespace fdog {

static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

const char *last_error() { return g_err.c_str(); }

// ---- host parallelism of the packing phases.  Work over [0, n) is split into
// a fixed number of contiguous chunks (par_chunks); every step below writes a
// result that does not depend on the chunking, so plans are identical for
// any thread count.
static int par_chunks(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(threads, (n + (1 << 16) - 1) >> 16));
}
template <typename F>
static void par_for(int64_t n, int threads, F f) {  // f(chunk, begin, end)
  const int T = par_chunks(n, threads);
  if (T == 1) {
    f(0, (int64_t)0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back([&f, t, T, n] { f(t, n * t / T, n * (t + 1) / T); });
  f(0, (int64_t)0, n / T);
  for (auto &th : pool) th.join();
}
// Sort with a strict total order (ties impossible), chunks sorted in parallel
// and merged pairwise: the same result as std::sort for any thread count.
template <typename V, typename C>
static void par_sort(std::vector<V> &v, int threads, C cmp) {
  const int64_t n = (int64_t)v.size();
  const int T = par_chunks(n, threads);
  if (T == 1) {
    std::sort(v.begin(), v.end(), cmp);
    return;
  }
  std::vector<int64_t> b(T + 1);
  for (int t = 0; t <= T; ++t) b[t] = n * t / T;
  par_for(n, threads, [&](int c, int64_t, int64_t) { std::sort(v.begin() + b[c], v.begin() + b[c + 1], cmp); });
  std::vector<V> tmp(v.size());
  for (int w = 1; w < T; w *= 2) {
    const int pairs = (T + 2 * w - 1) / (2 * w);
    std::vector<std::thread> pool;
    for (int k = 0; k < pairs; ++k)
      pool.emplace_back([&, k] {
        const int64_t lo = b[std::min(T, 2 * w * k)], mid = b[std::min(T, 2 * w * k + w)],
                      hi = b[std::min(T, 2 * w * k + 2 * w)];
        std::merge(v.begin() + lo, v.begin() + mid, v.begin() + mid, v.begin() + hi, tmp.begin() + lo, cmp);
      });
    for (auto &th : pool) th.join();
    v.swap(tmp);
  }
}
static inline void atomic_min32(int32_t *p, int32_t v) {
  int32_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (v < cur && !__atomic_compare_exchange_n(p, &cur, v, true, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
  }
}


// ---------------------------------------------------------------------------
// Compiler B.
//
// For row sum_h a_h x_h (rel) b, let T_h be the set of achievable suffix sums
// sum_{t>=h} a_t x_t (T_k = {0}).  A top-down state at partition h is the
// residual r = b - sum_{t<h} a_t x_t; its set of feasible completions is
// {x : sum_{t>=h} a_t x_t in R(r)} with R(r) = (-inf, r], [r, inf) or {r}.
// Two residuals have the same completion set iff they select the same subset
// of T_h, so the canonical node of r is the representative
//   <= : max{t in T_h : t <= r}     >= : min{t in T_h : t >= r}     == : r if r in T_h
// (none: dead -> bottom).  Nodes of P_h are the distinct representatives
// reached from the root; the children of representative r are the
// representatives of r (x_h = 0) and r - a_h (x_h = 1) in T_{h+1}.
// ---------------------------------------------------------------------------
static bool representative(const std::vector<int64_t> &T, int rel, int64_t r, int64_t *out) {
  if (rel < 0) {
    auto it = std::upper_bound(T.begin(), T.end(), r);
    if (it == T.begin()) return false;
    *out = *(it - 1);
    return true;
  }
  if (rel > 0) {
    auto it = std::lower_bound(T.begin(), T.end(), r);
    if (it == T.end()) return false;
    *out = *it;
    return true;
  }
  if (!std::binary_search(T.begin(), T.end(), r)) return false;
  *out = r;
  return true;
}

static fdog_status compile_B(int32_t k, const int32_t *a, int rel, int64_t b, Shape &out) {
  const size_t kMaxSums = size_t(1) << 22;
  std::vector<std::vector<int64_t>> T(k + 1);
  T[k] = {0};
  for (int32_t h = k - 1; h >= 0; --h) {
    const auto &nx = T[h + 1];
    std::vector<int64_t> shifted(nx.size());
    for (size_t q = 0; q < nx.size(); ++q) shifted[q] = nx[q] + a[h];
    T[h].resize(nx.size() * 2);
    auto e = std::set_union(nx.begin(), nx.end(), shifted.begin(), shifted.end(), T[h].begin());
    T[h].resize(e - T[h].begin());
    if (T[h].size() > kMaxSums) {
      set_error("row with %d variables has more than %zu distinct suffix sums", k, kMaxSums);
      return FDOG_ETOOBIG;
    }
  }
  int64_t r0;
  if (k == 0 || !representative(T[0], rel, b, &r0)) return FDOG_EINFEASIBLE;
  out.k = k;
  out.hop_start.assign(1, 0);
  out.lo.clear();
  out.hi.clear();
  out.max_w = 0;
  std::vector<int64_t> level = {r0}, next;
  std::unordered_map<int64_t, int32_t> index;
  for (int32_t h = 0; h < k; ++h) {
    next.clear();
    index.clear();
    for (int64_t r : level) {
      int64_t res[2] = {r, r - a[h]};
      uint32_t code[2];
      for (int beta = 0; beta < 2; ++beta) {
        if (h == k - 1) {
          int64_t q;
          code[beta] = representative(T[k], rel, res[beta], &q) ? kTop : kBot;
        } else {
          int64_t q;
          if (!representative(T[h + 1], rel, res[beta], &q)) {
            code[beta] = kBot;
          } else {
            auto it = index.find(q);
            if (it == index.end()) {
              int32_t id = (int32_t)next.size();
              index.emplace(q, id);
              next.push_back(q);
              code[beta] = (uint32_t)id;
            } else {
              code[beta] = (uint32_t)it->second;
            }
          }
        }
      }
      out.lo.push_back((uint16_t)code[0]);
      out.hi.push_back((uint16_t)code[1]);
    }
    out.max_w = std::max<int32_t>(out.max_w, (int32_t)level.size());
    if ((int64_t)next.size() > kMaxWidth) {
      set_error("BDD partition wider than %d nodes", kMaxWidth);
      return FDOG_ETOOBIG;
    }
    out.hop_start.push_back(out.hop_start.back() + (int32_t)level.size());
    level.swap(next);
  }
  return FDOG_OK;
}

// 64-bit FNV-1a over the row signature (relation, rhs, coefficients).
static uint64_t signature_hash(int32_t k, const int32_t *a, int8_t rel, int64_t rhs) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int q = 0; q < 8; ++q) {
      h ^= (v >> (8 * q)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  mix((uint64_t)(uint8_t)rel);
  mix((uint64_t)rhs);
  mix((uint64_t)k);
  for (int32_t q = 0; q < k; ++q) mix((uint64_t)(uint32_t)a[q]);
  return h;
}

static fdog_status validate(const fdog_problem *p, int threads) {
  if (!p || p->n_vars < 0 || p->n_cons < 0) {
    set_error("null problem or negative sizes");
    return FDOG_EINVAL;
  }
  if ((p->n_vars > 0 && !p->cost) || (p->n_cons > 0 && (!p->row_ptr || !p->rel || !p->rhs))) {
    set_error("null problem array");
    return FDOG_EINVAL;
  }
  if (p->n_cons > 0 && p->row_ptr[0] != 0) {
    set_error("row_ptr[0] must be 0");
    return FDOG_EINVAL;
  }
  // parallel scan for the first bad row; the messages below come from it
  int32_t first_bad = p->n_cons;
  par_for(p->n_cons, threads, [&](int, int64_t j0, int64_t j1) {
    for (int64_t j = j0; j < j1; ++j) {
      const int64_t a = p->row_ptr[j], b = p->row_ptr[j + 1];
      bool bad = b < a || b - a > 0x7fffffff || p->rel[j] < -1 || p->rel[j] > 1;
      for (int64_t q = a; q < b && !bad; ++q)
        bad = p->col_var[q] < 0 || p->col_var[q] >= p->n_vars || p->col_coef[q] == 0 ||
              (q > a && p->col_var[q] <= p->col_var[q - 1]);
      if (bad) {
        atomic_min32(&first_bad, (int32_t)j);
        return;
      }
    }
  });
  for (int32_t j = first_bad; j < p->n_cons; ++j) {
    int64_t a = p->row_ptr[j], b = p->row_ptr[j + 1];
    if (b < a || b - a > 0x7fffffff) {
      set_error("row %d: bad row_ptr", j);
      return FDOG_EINVAL;
    }
    if (p->rel[j] < -1 || p->rel[j] > 1) {
      set_error("row %d: rel must be -1, 0 or 1", j);
      return FDOG_EINVAL;
    }
    for (int64_t q = a; q < b; ++q) {
      if (p->col_var[q] < 0 || p->col_var[q] >= p->n_vars) {
        set_error("row %d: variable index out of range", j);
        return FDOG_EINVAL;
      }
      if (p->col_coef[q] == 0) {
        set_error("row %d: zero coefficient", j);
        return FDOG_EINVAL;
      }
      if (q > a && p->col_var[q] <= p->col_var[q - 1]) {
        set_error("row %d: variables must be strictly ascending", j);
        return FDOG_EINVAL;
      }
    }
  }
  for (int32_t i = 0; i < p->n_vars; ++i)
    if (!std::isfinite(p->cost[i])) {
      set_error("cost[%d] is not finite", i);
      return FDOG_EINVAL;
    }
  return FDOG_OK;
}

// Row bundles and their locality order (used by the sharder and by the tile
// packer).  The only coupling between BDDs is the per-variable average of
// P:641.
//  1. Bundles: rows joined by a variable held by exactly two rows (|J_i| = 2:
//     an MRF edge's or a QAP pair's y variables) are united
//     (union-find; the root of a component is its smallest row).
//  2. A bundle heavier than total / (4 world) nodes (e.g. cell tracking, where
//     transitions chain every frame to the next) is dissolved into its rows.
//  3. Units (bundles or dissolved rows) get a locality key: for a bundle the
//     smallest index of its variables with |J_i| != 2 (the variables it shares
//     with other bundles -- pixels, QAP assignment variables, graph-matching
//     labels); for a dissolved row its smallest variable index.
// unit[j]: the unit of row j (a row index); ukey[u]: the key of unit u.
static void bundle_units(const fdog_problem *p, int world, const std::vector<int32_t> &deg,
                         const std::vector<int64_t> &weight, std::vector<int32_t> &unit, std::vector<int64_t> &ukey) {
  const int32_t m = p->n_cons;
  unit.assign(m, 0);
  ukey.assign(m, INT64_MAX);
  std::vector<int32_t> parent(m);
  for (int32_t j = 0; j < m; ++j) parent[j] = j;
  auto find = [&](int32_t x) {
    while (parent[x] != x) {
      parent[x] = parent[parent[x]];
      x = parent[x];
    }
    return x;
  };
  {
    std::vector<int32_t> first(p->n_vars, -1);
    for (int32_t j = 0; j < m; ++j)
      for (int64_t q = p->row_ptr[j]; q < p->row_ptr[j + 1]; ++q) {
        const int32_t i = p->col_var[q];
        if (deg[i] != 2) continue;
        if (first[i] < 0) {
          first[i] = j;
          continue;
        }
        int32_t a = find(first[i]), b = find(j);
        if (a == b) continue;
        if (a > b) std::swap(a, b);
        parent[b] = a;  // the smaller row is the root
      }
  }
  std::vector<int32_t> root(m);
  std::vector<int64_t> compw(m, 0);
  int64_t total = 0;
  for (int32_t j = 0; j < m; ++j) {
    root[j] = find(j);
    compw[root[j]] += weight[j];
    total += weight[j];
  }
  const int64_t cap = std::max<int64_t>(1, total / (4 * (int64_t)std::max(world, 1)));
  std::vector<int64_t> kext(m, INT64_MAX);
  for (int32_t j = 0; j < m; ++j) {
    const bool dissolve = compw[root[j]] > cap;
    const int32_t u = dissolve ? j : root[j];
    unit[j] = u;
    for (int64_t q = p->row_ptr[j]; q < p->row_ptr[j + 1]; ++q) {
      const int32_t i = p->col_var[q];
      ukey[u] = std::min<int64_t>(ukey[u], i);
      if (!dissolve && deg[i] != 2) kext[u] = std::min<int64_t>(kext[u], i);
    }
  }
  for (int32_t u = 0; u < m; ++u)
    if (kext[u] != INT64_MAX) ukey[u] = kext[u];
}

// Locality-aware sharder: the units of
// bundle_units ordered by (key, smallest row) and cut into `world` ranges of
// equal BDD node count (the rank whose share contains a unit's midpoint owns
// it).  A bundle's |J_i| = 2 variables never cross ranks.  Deterministic:
// every rank derives the same map from the same problem.
static void shard_rows(const fdog_problem *p, int world, const std::vector<int32_t> &unit,
                       const std::vector<int64_t> &ukey, const std::vector<int64_t> &weight,
                       std::vector<int32_t> &owner) {
  owner.assign(p->n_cons, 0);
  if (world <= 1 || p->n_cons == 0) return;
  const int32_t m = p->n_cons;
  std::vector<int64_t> uw(m, 0);
  int64_t total = 0;
  for (int32_t j = 0; j < m; ++j) {
    uw[unit[j]] += weight[j];
    total += weight[j];
  }
  if (total <= 0) return;
  std::vector<int32_t> units;
  for (int32_t j = 0; j < m; ++j)
    if (unit[j] == j) units.push_back(j);
  std::sort(units.begin(), units.end(), [&](int32_t a, int32_t b) {
    return ukey[a] != ukey[b] ? ukey[a] < ukey[b] : a < b;
  });
  std::vector<int32_t> rank_of(m, 0);
  int64_t acc = 0;
  for (int32_t u : units) {
    const int64_t mid2 = 2 * acc + uw[u];  // 2 * midpoint
    const int64_t r = (mid2 * world) / (2 * total);
    rank_of[u] = (int32_t)std::min<int64_t>(std::max<int64_t>(r, 0), world - 1);
    acc += uw[u];
  }
  for (int32_t j = 0; j < m; ++j) owner[j] = rank_of[unit[j]];
}

// Pad a 4-byte array to a multiple of 16 bytes: every tile's topology and
// partition table starts 16-byte aligned and may be read in whole 16-byte
// units by the TMA bulk copies.
template <typename V>
static void pad16(std::vector<V> &v) {
  static_assert(sizeof(V) == 4, "4-byte elements");
  while (v.size() % 4) v.push_back(V(0));
}

// Device topology code of a successor: absolute node index within the tile
// (next partition starts at `next`), top = nodes, bottom = nodes + 1 (the two
// sentinel slots of the kernels' distance arrays).
static uint32_t abs_code(uint16_t rel, int32_t next, int32_t nodes) {
  if (rel == kBot) return uint32_t(nodes + 1);
  if (rel == kTop) return uint32_t(nodes);
  return uint32_t(next + rel);
}

// Arc masks of partition h of a shape whose partitions have <= 2 nodes:
// A[4 beta + 2 i + j] = 0 if the beta-arc out of node i of P_h ends in node j
// of P_{h+1} (or in top on the last partition), +inf otherwise (including
// every arc to bottom).  Returns the hop type (internal.h HopRec): 1 chain
// (0-arcs 0->0, 1->1; 1-arc 1->0), 2 root (one node; ->0, ->1), 3 join
// (0-arc 0->0; 1-arc 1->0), 0 anything else.
static int hop_masks(const Shape &S, int32_t h, double A[8]) {
  for (int q = 0; q < 8; ++q) A[q] = INFINITY;
  const int32_t w = S.hop_start[h + 1] - S.hop_start[h];
  for (int32_t i = 0; i < w; ++i) {
    const int32_t n = S.hop_start[h] + i;
    for (int beta = 0; beta < 2; ++beta) {
      const uint32_t code = beta ? S.hi[n] : S.lo[n];
      if (code == kBot) continue;
      const int j = code == kTop ? 0 : (int)code;  // top only on the last partition
      A[4 * beta + 2 * i + j] = 0.0;
    }
  }
  auto is = [&](std::initializer_list<int> zeros) {
    for (int q = 0; q < 8; ++q) {
      bool z = false;
      for (int t : zeros) z = z || t == q;
      if (z != (A[q] == 0.0)) return false;
    }
    return true;
  };
  if (w == 2 && is({0, 3, 6})) return 1;
  if (w == 1 && is({0, 5})) return 2;
  if (w == 2 && is({0, 6})) return 3;
  // (Folding the Potts-cut rows' three other patterns as well, by a dispatch
  // on this type at run time, measured no gain there and a few per cent on
  // MRF-LP from the larger kernels: they keep the general masks.)
  return 0;
}

// kind bit 3: every partition but the first and the last is a chain hop
static bool chain_shape(const Shape &S) {
  if (S.max_w > 2) return false;
  double A[8];
  for (int32_t h = 1; h + 1 < S.k; ++h)
    if (hop_masks(S, h, A) != 1) return false;
  return true;
}

// kind bit 4 (with bit 3): the first partition is a root hop (type 2) and the
// last a join into top (type 3) -- every hop of the shape is then folded
static bool ends_shape(const Shape &S) {
  if (S.max_w > 2 || S.k < 2) return false;
  double A[8];
  return hop_masks(S, 0, A) == 2 && hop_masks(S, S.k - 1, A) == 3;
}

// Hop records (layout: internal.h HopRec) of a shape whose partitions have
// <= 2 nodes, in the build precision.
static void append_recs(const Shape &S, int tsz, std::vector<unsigned char> &out) {
  for (int32_t h = 0; h < S.k; ++h) {
    double A[8];
    const int32_t type = hop_masks(S, h, A);
    const int32_t w = S.hop_start[h + 1] - S.hop_start[h];
    const size_t at = out.size();
    out.resize(at + (size_t)rec_bytes(tsz), 0);
    unsigned char *r = out.data() + at;
    for (int q = 0; q < 8; ++q) {
      if (tsz == 8) {
        const double v = A[q];
        memcpy(r + 8 * q, &v, 8);
      } else {
        const float v = (float)A[q];
        memcpy(r + 4 * q, &v, 4);
      }
    }
    const int32_t tail[4] = {S.hop_start[h], S.hop_start[h + 1], w == 2 ? 1 : 0, type};
    memcpy(r + 8 * tsz, tail, 16);
  }
  out.resize((out.size() + 15) & ~(size_t)15, 0);
}

// FDOG_PLAN_TRACE=1: per-phase wall times of build_plan on stderr
struct PhaseTimer {
  bool on = getenv("FDOG_PLAN_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char *what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[plan] %-28s %8.3f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

fdog_status build_plan(const fdog_problem *p, const fdog_options *o, Plan &P) {
  PhaseTimer tm;
  int threads = o && o->host_threads > 0 ? o->host_threads : (int)std::thread::hardware_concurrency();
  threads = std::max(1, std::min(threads, 64));
  fdog_status st = validate(p, threads);
  if (st) return st;
  const int world = o ? std::max(1, o->world) : 1;
  const int rank = o ? o->rank : 0;
  if (rank < 0 || rank >= world) {
    set_error("rank %d outside [0, %d)", rank, world);
    return FDOG_EINVAL;
  }
  P.host_threads = threads;
  P.lifted = o && o->lifted;
  if (P.lifted && world > 1) {
    set_error("the lifted representation is single-GPU (world == 1)");
    return FDOG_EINVAL;
  }

  P.n_vars = p->n_vars;
  P.n_cons = p->n_cons;
  P.rank = rank;
  P.world = world;
  P.cost.assign(p->cost, p->cost + p->n_vars);
  P.max_abs_cost = 0.0;
  for (double c : P.cost) P.max_abs_cost = std::max(P.max_abs_cost, std::fabs(c));
  P.row_ptr.assign(p->row_ptr, p->row_ptr + p->n_cons + 1);
  if (p->n_cons == 0) P.row_ptr.assign(1, 0);
  const int64_t nnz = P.row_ptr.back();
  P.col_var.resize(nnz);
  P.col_coef.resize(nnz);
  par_for(nnz, threads, [&](int, int64_t a, int64_t b) {
    memcpy(P.col_var.data() + a, p->col_var + a, (b - a) * sizeof(int32_t));
    memcpy(P.col_coef.data() + a, p->col_coef + a, (b - a) * sizeof(int32_t));
  });
  P.rel.assign(p->rel, p->rel + p->n_cons);
  P.rhs.assign(p->rhs, p->rhs + p->n_cons);

  // rows with no variable: feasible (dropped) or infeasible (error)
  for (int32_t j = 0; j < p->n_cons; ++j)
    if (p->row_ptr[j + 1] == p->row_ptr[j]) {
      int64_t b = p->rhs[j];
      bool ok = p->rel[j] < 0 ? 0 <= b : p->rel[j] > 0 ? 0 >= b : b == 0;
      if (!ok) {
        set_error("row %d has no variables and is infeasible", j);
        return FDOG_EINFEASIBLE;
      }
    }

  tm.mark("copy + validate");
  // global |J_i| and the free-variable term (A13)
  P.deg_global.assign(p->n_vars, 0);
  par_for(nnz, threads, [&](int, int64_t a, int64_t b) {
    for (int64_t q = a; q < b; ++q) __atomic_fetch_add(&P.deg_global[p->col_var[q]], 1, __ATOMIC_RELAXED);
  });
  P.free_term = 0.0;
  for (int32_t i = 0; i < p->n_vars; ++i)
    if (P.deg_global[i] == 0 && P.cost[i] < 0) P.free_term += P.cost[i];

  tm.mark("degrees");
  // dedupe every non-empty row by signature (the sharder weighs rows by node
  // count, so with world > 1 all shapes are compiled, not only local ones)
  P.row_shape.assign(p->n_cons, -1);
  P.local_rows.clear();
  std::unordered_map<uint64_t, std::vector<int32_t>> sig;
  for (int32_t j = 0; j < p->n_cons; ++j) {
    int64_t a = p->row_ptr[j];
    int32_t k = (int32_t)(p->row_ptr[j + 1] - a);
    if (k == 0) continue;
    const int32_t *c = p->col_coef + a;
    uint64_t h = signature_hash(k, c, p->rel[j], p->rhs[j]);
    auto &cands = sig[h];
    int32_t id = -1;
    for (int32_t s : cands) {
      const Shape &S = P.shapes[s];
      if (S.rel == p->rel[j] && S.rhs == p->rhs[j] && (int32_t)S.coef.size() == k &&
          std::equal(c, c + k, S.coef.begin())) {
        id = s;
        break;
      }
    }
    if (id < 0) {
      id = (int32_t)P.shapes.size();
      P.shapes.emplace_back();
      Shape &S = P.shapes.back();
      S.rel = p->rel[j];
      S.rhs = p->rhs[j];
      S.coef.assign(c, c + k);
      cands.push_back(id);
    }
    P.row_shape[j] = id;
  }
  // FDOG_GPU_COMPILE=1: compile the distinct shapes on the GPU (compile_gpu.cu,
  // identical results); falls back to the host compiler when a shape's
  // suffix-sum sets may exceed the GPU scratch bound or no device is present
  bool compiled = false;
  // the device steps of the plan (compile here, the slot / variable phases of
  // the packer below; identical plans): default for problems of >= 10^7
  // nonzeros when a device is present, FDOG_GPU_COMPILE / FDOG_GPU_PACK = 0 / 1
  // override (measured on the 16-thread GPU host: MRF-LP 9.4 -> 6.8 s; QAP50
  // 0.48 -> 0.65 s, where the transfers cost more than they save)
  auto gpu_step = [&](const char *knob) {
    const char *v = getenv(knob);
    if (v) return v[0] == '1';
    return P.row_ptr.back() >= 10000000;
  };
  if (gpu_step("FDOG_GPU_COMPILE")) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
      const int dev = o ? o->device : 0;
      const fdog_status r = gpu_compile_shapes(P.shapes, dev >= 0 && dev < ndev ? dev : 0);
      if (r == FDOG_EINFEASIBLE) {
        set_error("a constraint has an empty feasible set");
        return r;
      }
      if (r == FDOG_ECUDA) return r;
      compiled = r == FDOG_OK;
    } else {
      cudaGetLastError();
    }
  }
  if (!compiled) {
    std::atomic<int64_t> next{0};
    std::atomic<int> bad{0};
    std::mutex mu;
    std::string err;
    auto work = [&]() {
      for (;;) {
        int64_t s = next.fetch_add(1);
        if (s >= (int64_t)P.shapes.size()) break;
        Shape &S = P.shapes[s];
        fdog_status r = compile_B((int32_t)S.coef.size(), S.coef.data(), S.rel, S.rhs, S);
        if (r != FDOG_OK) {
          std::lock_guard<std::mutex> g(mu);
          if (!bad.load()) {
            bad = (int)r;
            err = r == FDOG_EINFEASIBLE ? "a constraint has an empty feasible set" : last_error();
          }
        }
      }
    };
    int nt = (int)std::min<int64_t>(threads, (int64_t)P.shapes.size());
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &t : pool) t.join();
    if (bad.load()) {
      set_error("%s", err.c_str());
      return (fdog_status)bad.load();
    }
  }

  tm.mark("dedupe + compile");
  if (o && o->row_owner && world > 1) {  // caller-supplied row -> rank map
    P.owner.assign(o->row_owner, o->row_owner + p->n_cons);
    for (int32_t j = 0; j < p->n_cons; ++j)
      if (P.owner[j] < 0 || P.owner[j] >= world) {
        set_error("row_owner[%d] = %d outside [0, %d)", j, P.owner[j], world);
        return FDOG_EINVAL;
      }
  }
  // bundles + locality keys: the sharder's units, and the row order inside a
  // shape's tiles (rows of one bundle in consecutive lanes, so that a bundle's
  // |J_i| = 2 variables have both slots in one tile: the sweep averages them
  // on chip)
  std::vector<int32_t> unit;
  std::vector<int64_t> ukey;
  {
    std::vector<int64_t> wt(p->n_cons, 0);
    for (int32_t j = 0; j < p->n_cons; ++j)
      if (P.row_shape[j] >= 0) wt[j] = P.shapes[P.row_shape[j]].nodes();
    bundle_units(p, world, P.deg_global, wt, unit, ukey);
    if (!(o && o->row_owner && world > 1)) shard_rows(p, world, unit, ukey, wt, P.owner);
  }
  for (int32_t j = 0; j < p->n_cons; ++j)
    if (P.row_shape[j] >= 0) {
      if (P.owner[j] == rank) P.local_rows.push_back(j);
      else P.row_shape[j] = -1;
    }
  tm.mark("shard");
  // variables held by two or more ranks (the exchange vector, below) and the
  // "boundary" rows that hold one: their tiles are swept after the others, so
  // that the exchange of a pass overlaps the sweep of the interior tiles
  //
  std::vector<uint8_t> multi(world > 1 ? p->n_vars : 0, 0);
  std::vector<uint8_t> boundary_row(world > 1 ? p->n_cons : 0, 0);
  if (world > 1) {
    std::vector<int32_t> first(p->n_vars, -1);
    for (int32_t j = 0; j < p->n_cons; ++j)
      for (int64_t q = P.row_ptr[j]; q < P.row_ptr[j + 1]; ++q) {
        const int32_t i = P.col_var[q];
        if (first[i] < 0) first[i] = P.owner[j];
        else if (first[i] != P.owner[j]) multi[i] = 1;
      }
    for (int32_t j : P.local_rows)
      for (int64_t q = P.row_ptr[j]; q < P.row_ptr[j + 1]; ++q)
        if (multi[P.col_var[q]]) boundary_row[j] = 1;
  }
  // ---------------------------------------------------------------- packing
  P.max_hops = 0;
  P.max_width = 0;
  P.n_nodes = 0;
  P.n_slots = 0;
  for (int32_t j : P.local_rows) {
    const Shape &S = P.shapes[P.row_shape[j]];
    P.max_hops = std::max(P.max_hops, S.k);
    P.max_width = std::max(P.max_width, S.max_w);
    P.n_nodes += S.nodes();
    P.n_slots += S.k;
  }
  // group rows by shape (ascending j inside a group), or in bundle order --
  // (bundle key, bundle, j): a bundle's rows of one shape in consecutive lanes
  // -- when that closes at least 90 % of the shape's slots of |J_i| = 2
  // variables, i.e. puts both slots of those variables into one 32-row tile
  // (their averages are then computed on chip by the sweep; e.g. MRF-LP: 16
  // marginalisation rows per edge, two edges per tile).  Otherwise the j order is kept: the generators'
  // families there put a variable's two slots at the same lane of two tiles,
  // which the averaging kernel reads coalesced (GM, QAP).
  std::vector<std::vector<int32_t>> by_shape(P.shapes.size());
  std::vector<int32_t> coop_rows;  // rows of shapes wider than kCoopWidth: one cooperative tile each
  for (int32_t j : P.local_rows) {
    if (P.shapes[P.row_shape[j]].max_w > kCoopWidth) coop_rows.push_back(j);
    else by_shape[P.row_shape[j]].push_back(j);
  }
  // Rows per lane (kernels.cu mask_tile): staged arc-mask tiles of a short
  // shape hold 32 R rows, lane l the rows l + 32 k.  The per-tile work (claim,
  // descriptor, TMA issue, bound partial) and the per-hop tail, addresses and
  // loop control are shared by the R rows, and the R hop chains are
  // independent.  R = 4 for K <= 4 (fp32), 2 for K <= 16 (when the shape fills
  // such a tile), when the budget model below prefers them; not for small
  // problems (fused path) or the streaming kernel.  FDOG_WIDE=0 / 1 (tests and
  // A/B runs): never / whenever eligible.
  const char *sw = getenv("FDOG_SWEEP");
  const char *fz = getenv("FDOG_FUSED");
  const char *wd = getenv("FDOG_WIDE");
  const bool wide_force = wd && wd[0] == '1';
  // (measured, same box: MRF-LP 0.650 -> 0.579 ms per iteration, Potts-cut
  // 0.701 -> 0.593; with a few tiles per warp -- GM-worms 6 k tiles, cell
  // tracking 17 k -- the longer tiles cost more in the tail than they save:
  // GM 40.9 -> 45.7 us.  So: problems of at least 10^6 rows.)
  const bool wide_ok = !P.lifted && (wide_force || P.local_rows.size() >= 1000000) && P.n_slots > (1 << 15) && !(sw && sw[0] == 's') && !(fz && fz[0] == '1') && !(wd && wd[0] == '0');
  const char *r4k = getenv("FDOG_R4K");  // experiment knob: longest rows with four rows per lane (default 4)
  const int r4_max_k = r4k ? atoi(r4k) : 4;
  auto rows_per_lane = [&](size_t sh) -> int {
    const Shape &S = P.shapes[sh];
    if (!wide_ok || S.max_w > 2) return 1;
    int R = (S.k <= r4_max_k && !(o && o->precision == 64)) ? 4 : S.k <= 16 ? 2 : 1;  // (fp64: at most 2)
    while (R > 1 && by_shape[sh].size() < (size_t)(32 * R)) R /= 2;
    return R;
  };
  std::vector<char> pair_room(P.shapes.size(), 0);  // bundle order: stages reserve room for a pair list
  {
    const char *pe = getenv("FDOG_PAIRS");
    const bool pairs_ok = !(pe && pe[0] == '0') && !P.lifted;
    std::vector<int64_t> seen(pairs_ok ? p->n_vars : 0, -1);  // first (row position / 32) of a |J_i| = 2 variable
    for (size_t sh = 0; sh < by_shape.size() && pairs_ok; ++sh) {
      auto &rows = by_shape[sh];
      if (rows.size() < 2) continue;
      std::vector<int32_t> b = rows;
      par_sort(b, threads, [&](int32_t x, int32_t y) {
        const int32_t ux = unit[x], uy = unit[y];
        if (ukey[ux] != ukey[uy]) return ukey[ux] < ukey[uy];
        return ux != uy ? ux < uy : x < y;
      });
      int64_t slots2 = 0, same = 0;  // the shape's slots of |J_i| = 2 variables; variables closed in one tile
      const int64_t tag = (int64_t)sh << 40;
      for (size_t r = 0; r < b.size(); ++r)
        for (int64_t q = p->row_ptr[b[r]]; q < p->row_ptr[b[r] + 1]; ++q) {
          const int32_t i = p->col_var[q];
          if (P.deg_global[i] != 2) continue;
          slots2++;
          const int64_t code = tag | (int64_t)(r / (32 * rows_per_lane(sh)));
          if (seen[i] >= 0 && (seen[i] >> 40) == (int64_t)sh) same += seen[i] == code;
          else seen[i] = code;
        }
      // (measured on cell tracking: a shape whose pair partners mostly sit in
      // other shapes gains nothing from the bundle order, and the order breaks
      // the averaging kernel's coalesced pair layout: avg 32 -> 71 us)
      if (slots2 > 0 && 2 * same >= 0.9 * slots2) {
        rows.swap(b);
        pair_room[sh] = 1;
      }
    }
  }

  // ---- per-warp shared-memory budget: every tile's stage buffer
  // must fit SB and its distance arrays DB; a shape whose BDDs are too long for
  // 32 lanes is packed into tiles of 16, 8 or 4 lanes instead.  The budget is
  // chosen by a cost model: per-lane sequential chain (latency) over resident
  // warps vs. issued instructions over the SMs.
  const int tsz = (o && o->precision == 64) ? 8 : 4;
  P.precision = tsz * 8;
  // stage buffers per warp: the recompute design runs single-buffered (more
  // resident warps hide the TMA latency; measured faster on every BASELINE
  // workload), and so does the L2-resident store design of narrow shapes; see
  // the design choice below.  FDOG_NBUF = 1 | 2 overrides.
  const char *nbuf = getenv("FDOG_NBUF");
  // (world > 1: a shape's boundary rows after its interior rows, stable)
  if (world > 1)
    for (auto &rows : by_shape)
      std::stable_partition(rows.begin(), rows.end(), [&](int32_t j) { return !boundary_row[j]; });
  struct PendingTile {
    int kind;                    // bit 0 per-lane topology, bit 1 staged
    int32_t shape;               // kind 0
    int L;
    std::vector<int32_t> rows;   // lanes
    int64_t cost;
    bool boundary = false;       // holds a row with an exchanged variable
  };
  // pack(rc): budget + tiles for the store design (rc = false) or the
  // recompute design (rc = true, narrow shapes only); returns the tiles in
  // launch order
  // Recompute design, fp32: the distance scratch of 32-row arc-mask tiles can
  // live in tensor memory (kernels.cu TmemD; columns = the next power of two
  // >= nodes + 2, <= 512 per SM).  tm: pack for it -- such tiles need no DB
  // region, and a narrow shape's leftover rows go to a partly filled 32-row
  // tile of the shape (idle lanes) instead of the per-lane-topology pool.
  // (not with rows-per-lane tiles: the TMEM kernel variant has one row per lane)
  const char *tmv = getenv("FDOG_TMEM");
  int tm_cols = 32;
  bool tm_rows_ok = true;
  for (size_t sh = 0; sh < P.shapes.size(); ++sh)
    if (!by_shape[sh].empty() && P.shapes[sh].max_w <= 2) {
      while (tm_cols < P.shapes[sh].nodes() + 2) tm_cols *= 2;
      tm_rows_ok = tm_rows_ok && rows_per_lane(sh) == 1;
    }
  bool tm_packed = false, tm_allow = true;
  const bool tm_trace = getenv("FDOG_PLAN_TRACE") != nullptr;
  const char *rg = getenv("FDOG_RECS");  // test knob: FDOG_RECS=global reads every tile's records from global memory
  const bool recs_global = rg && rg[0] == 'g';
  auto pack = [&](bool rc, int nb) {
    std::vector<PendingTile> pend;
    P.NB = nbuf ? (atoi(nbuf) == 1 ? 1 : 2) : nb;
    const bool tm = tm_allow && rc && tsz == 4 && !P.lifted && tm_cols <= 512 && tm_rows_ok && !(tmv && tmv[0] == '0');
    tm_packed = tm;
    // pr: the tile may carry a pair list (at most K L / 2 pairs)
    auto fits = [&](int kind, int K, int nodes, int W, int L, int SB, int DB, bool pr = false) {
      if (P.lifted) return false;  // (lifted mode: every tile from global memory)
      const int pb = pr ? stage_pairs_bytes(K * L / 2) : 0;
      if (rc)
        return stage_bytes_rc(tsz, kind, K, nodes, L) + pb <= SB &&
               ((tm && (kind & 4) && L == 32) || stage_dist_bytes(tsz, nodes, L) <= DB);
      // (arc-mask tiles never use the relaxation buffers)
      return stage_bytes(tsz, kind, K, nodes, L) + pb <= SB && ((kind & 4) || relax_bytes(tsz, W, L) <= DB);
    };
    auto lanes_for = [&](int kind, int K, int nodes, int W, int SB, int DB, bool pr = false, int Lmax = 32) {
      for (int L = Lmax; L >= 4; L /= 2)
        if (fits(kind, K, nodes, W, L, SB, DB, pr)) return L;
      return 0;
    };
    {
      int maxW = 1;
      for (size_t s = 0; s < P.shapes.size(); ++s)
        if (!by_shape[s].empty()) maxW = std::max(maxW, P.shapes[s].max_w);
      // store design: DB holds the relaxation buffers of the widest partition;
      // recompute design: DB = SB holds the distance scratch (for partitions of
      // <= 2 nodes the distances of a tile are about as large as its stage)
      const int DB0 = relax_bytes(tsz, std::min(maxW, 64), 32);
      const int cands[] = {6, 7, 8, 9, 10, 11, 12, 14, 16, 18, 20, 22, 24, 28, 32, 40, 48, 56, 72, 96, 112};
      double best = 1e300;
      int bestSB = 0, bestDB = DB0;
      std::vector<std::array<double, 4>> cand_t;  // (modelled time, warps per SM, SB, DB)
      for (int kb : cands) {
        const int SB = tm ? ((kb * 1024 - 16 - 64) / P.NB) & ~15
                          : rc ? ((kb * 1024 - 16) / (P.NB + 1)) & ~15 : ((kb * 1024 - 16 - DB0) / P.NB) & ~15;
        const int DB = rc ? SB : DB0;
        if (SB <= 0) continue;
        double chain = 0, instr = 0;
        int usedSB = 16, usedDB = 16;
        for (size_t s = 0; s < P.shapes.size(); ++s) {
          if (by_shape[s].empty()) continue;
          const Shape &S = P.shapes[s];
          const int k0 = (S.max_w <= 2 && !P.lifted) ? 4 : 0;  // arc-mask tiles for narrow shapes
          const int kb0 = k0 ? k0 | kKindRecGlobal : 0;  // (sized without records: they may stay in global memory)
          const bool pr = k0 && pair_room[s];
          int L = lanes_for(kb0, S.k, S.nodes(), S.max_w, SB, DB, pr, 32 * rows_per_lane(s));
          double pen = (wide_force && L > 0 && L < 32 * rows_per_lane(s)) ? 1e6 : 1.0;
          if (L == 0) {  // direct from global memory: latency-bound
            L = 32;
            // (the recompute design cannot run direct tiles at all: a budget
            // that leaves any is a fallback to the store design)
            pen = rc ? 1e6 : 10.0;
          } else {
            usedSB = std::max(usedSB, (rc ? stage_bytes_rc(tsz, kb0, S.k, S.nodes(), L) : stage_bytes(tsz, kb0, S.k, S.nodes(), L)) +
                                          (pr ? stage_pairs_bytes(S.k * L / 2) : 0));
            if (rc && !(tm && k0 && L == 32)) usedDB = std::max(usedDB, stage_dist_bytes(tsz, S.nodes(), L));
          }
          const double tiles = std::ceil((double)by_shape[s].size() / L);
          const double R = L > 32 ? L / 32 : 1;  // rows per lane: R chains per tile
          // per-tile sequential chain and issued instructions (the recompute
          // design adds the on-chip distance pass)
          const double cn = rc ? 70.0 : 50.0, ck = rc ? 160.0 : 120.0, in = rc ? 30.0 : 20.0, ik = rc ? 50.0 : 35.0;
          // (R chains per lane overlap: ~1 + 0.4 (R - 1) of one chain's
          // latency; the per-tile instructions -- claim, descriptor, TMA
          // issue, bound partial, ~500 per tile on MRF-LP -- are shared)
          chain += pen * tiles * ((1.0 + 0.4 * (R - 1)) * (cn * S.nodes() + ck * S.k) + (P.NB == 1 ? 1500.0 : 0.0));
          instr += tiles * (500.0 + R * 0.55 * (in * S.nodes() + ik * S.k));
        }
        if (!rc) usedDB = DB;
        const int wb = warp_bytes(usedSB, usedDB, P.NB);
        double warps = std::min(tm ? 4.0 * (512 / tm_cols) : 32.0, std::floor(226.0 * 1024 / wb));
        if (tm) warps = std::floor(warps / 4) * 4;  // (the TMEM kernel's CTAs: groups of 4 warps)
        if (warps < 1) continue;
        const double t = std::max(chain / (148.0 * warps), instr / (148.0 * 2.0));
        if (tm_trace) fprintf(stderr, "[plan] budget rc=%d tm=%d kb=%d SB=%d usedSB=%d usedDB=%d warps=%.0f chain=%.3g instr=%.3g t=%.4g\n",
                              (int)rc, (int)tm, kb, SB, usedSB, usedDB, warps, chain, instr, t);
        cand_t.push_back({t, warps, (double)usedSB, (double)usedDB});
      }
      // the candidate with the most resident warps among those within 0.5 % of
      // the best modelled time (the model is issue-bound for most problems,
      // and more warps hide more of the latency it does not model); ties: the
      // first, i.e. the smallest budget
      for (const auto &c : cand_t) best = std::min(best, c[0]);
      double best_w = -1;
      for (const auto &c : cand_t)
        if (c[0] <= 1.005 * best && c[1] > best_w) {
          best_w = c[1];
          bestSB = (int)c[2];
          bestDB = (int)c[3];
        }
      P.SB = std::max(bestSB, 64);
      P.DB = rc ? std::max(bestDB, 64) : DB0;
    }

    std::vector<int32_t> pool;  // rows for per-lane tiles
    for (size_t s = 0; s < P.shapes.size(); ++s) {
      auto &rows = by_shape[s];
      const Shape &S = P.shapes[s];
      const int k0 = (S.max_w <= 2 && !P.lifted) ? 4 : 0;
      int L = lanes_for(k0 ? k0 | kKindRecGlobal : 0, S.k, S.nodes(), S.max_w, P.SB, P.DB, k0 && pair_room[s],
                        32 * rows_per_lane(s));
      const bool staged = L > 0;
      if (!staged) L = 32;
      // (rows too long to stage, of a narrow shape: the last tile keeps the
      // shape's records even if partly filled -- the chunked path walks them;
      // other leftovers are pooled into per-lane-topology tiles)
      // (rows of a narrow shape with at least one full tile: the rest go to a
      // partly filled tile of the same shape, with the smallest lane count
      // that holds them, instead of a per-lane-topology tile -- that path
      // walks the topology node by node and its tile became the last to
      // finish: QAP50 36 us against 28 for every other warp)
      // (tiles of 32 R rows: the rest of the shape in 32-row tiles, then as above)
      size_t full = rows.size() / L * L;
      const size_t wide_end = full;
      if (L > 32) full += (rows.size() - full) / 32 * 32;
      if (k0 && (!staged || (tm && L == 32)))
        full = rows.size();
      for (size_t q = 0; q < full;) {
        PendingTile t;
        const bool ch = k0 && chain_shape(S);
        t.kind = (staged ? 2 : 0) | k0 | (ch ? 8 : 0) | (ch && ends_shape(S) ? 16 : 0);  // records also serve the streaming kernel
        t.shape = (int32_t)s;
        t.L = q < wide_end ? L : std::min(L, 32);
        const size_t nrow = std::min(rows.size() - q, (size_t)t.L);
        if (staged && nrow < (size_t)t.L && !(tm && t.L == 32)) {  // (TMEM tiles stay 32 rows wide)
          t.L = 4;
          while ((size_t)t.L < nrow) t.L *= 2;
        }
        t.rows.assign(rows.begin() + q, rows.begin() + q + nrow);
        t.cost = (int64_t)S.nodes() + S.k;
        pend.push_back(std::move(t));
        q += nrow;
      }
      pool.insert(pool.end(), rows.begin() + full, rows.end());
    }
    // per-lane tiles: same K within a tile; similar shapes adjacent
    std::stable_sort(pool.begin(), pool.end(), [&](int32_t x, int32_t y) {
      const Shape &a = P.shapes[P.row_shape[x]], &b = P.shapes[P.row_shape[y]];
      if (a.k != b.k) return a.k < b.k;
      if (a.nodes() != b.nodes()) return a.nodes() < b.nodes();
      return P.row_shape[x] < P.row_shape[y];
    });
    auto padded = [&](const std::vector<int32_t> &rows, size_t n, int *nodes, int *W) {
      const int K = P.shapes[P.row_shape[rows[0]]].k;
      std::vector<int32_t> w(K, 0);
      for (size_t q = 0; q < n; ++q) {
        const Shape &S = P.shapes[P.row_shape[rows[q]]];
        for (int h = 0; h < K; ++h) w[h] = std::max(w[h], S.hop_start[h + 1] - S.hop_start[h]);
      }
      *nodes = 0;
      *W = 1;
      for (int h = 0; h < K; ++h) {
        *nodes += w[h];
        *W = std::max(*W, w[h]);
      }
    };
    for (size_t q = 0; q < pool.size();) {
      const int K = P.shapes[P.row_shape[pool[q]]].k;
      std::vector<int32_t> rows;
      while (q < pool.size() && rows.size() < (size_t)kLanes && P.shapes[P.row_shape[pool[q]]].k == K)
        rows.push_back(pool[q++]);
      // largest lane count whose padded tile fits the budget
      int L = 0, nodes = 0, W = 1;
      for (int Lc = 32; Lc >= 4; Lc /= 2) {
        size_t n = std::min(rows.size(), (size_t)Lc);
        padded(rows, n, &nodes, &W);
        if (fits(1, K, nodes, W, Lc, P.SB, P.DB)) {
          L = Lc;
          break;
        }
      }
      PendingTile t;
      t.shape = -1;
      if (L == 0) {
        t.kind = 1;  // direct
        t.L = 32;
      } else {
        t.kind = 3;
        t.L = L;
        if (rows.size() > (size_t)L) {  // give the surplus back to the pool
          q -= rows.size() - L;
          rows.resize(L);
        }
      }
      t.rows = rows;
      int c = 0;
      for (int32_t j : t.rows) c = std::max(c, P.shapes[P.row_shape[j]].nodes());
      t.cost = c + K;
      pend.push_back(std::move(t));
    }
    for (int32_t j : coop_rows) {
      PendingTile t;
      t.kind = 32;
      t.shape = P.row_shape[j];
      t.L = 1;
      t.rows = {j};
      t.cost = (int64_t)P.shapes[t.shape].nodes() / 8 + P.shapes[t.shape].k;  // (32 lanes split the nodes)
      pend.push_back(std::move(t));
    }
    // direct tiles first (slowest), then expensive tiles, so the dynamic
    // scheduler does not leave them for the tail
    if (world > 1)
      for (auto &t : pend)
        for (int32_t j : t.rows) t.boundary = t.boundary || boundary_row[j];
    std::stable_sort(pend.begin(), pend.end(), [](const PendingTile &a, const PendingTile &b) {
      if (a.boundary != b.boundary) return b.boundary;  // interior tiles first
      const bool da = !(a.kind & 2), db = !(b.kind & 2);
      if (da != db) return da;
      // (a tile of L < 32 rows takes about as long as a full one; a tile of
      // 32 R rows about R times as long)
      auto key = [](const PendingTile &t) { return t.L >= 32 ? t.cost * t.L / 32 : t.cost * 32 / t.L; };
      return key(a) > key(b);
    });

    return pend;
  };
  tm.mark("group by shape");
  bool narrow = coop_rows.empty();
  for (size_t s = 0; s < P.shapes.size(); ++s)
    if (!by_shape[s].empty()) narrow = narrow && P.shapes[s].max_w <= 2;
  // design choice (experiment knobs: FDOG_SWEEP = rc | tma | stream; FDOG_FUSED)
  // The recompute design halves the HBM bytes of a pass at ~30 % more
  // instructions.  When the store design's per-pass working set (distances +
  // slot data) stays resident in the 126 MB L2 across the four kernels of an
  // iteration, the bytes are cheap and the instructions are not: keep the
  // store design there (measured: GM-worms-like, 73 MB, store 4 % faster;
  // CellTrack 160 MB / QAP50 195 MB / MRF 2.2 GB, recompute 6-27 % faster).
  const double store_bytes = (double)P.n_nodes * 2 * tsz + (double)P.n_slots * 4 * tsz;
  const bool l2_resident = store_bytes <= 0.75 * 126e6;
  bool rc = !P.lifted && narrow && !(sw && (sw[0] == 't' || sw[0] == 's')) && !(fz && fz[0] == '1') &&
            (!l2_resident || (sw && sw[0] == 'r'));
  // stage buffers: single-buffered for the recompute design and for the
  // L2-resident store design of narrow shapes (its stages come from L2: more
  // resident warps beat prefetching one tile ahead; measured GM 42.4 -> 39.9 us
  // per iteration), double-buffered otherwise
  std::vector<PendingTile> pend = pack(rc, (rc || (narrow && l2_resident)) ? 1 : 2);
  if (rc) {
    bool direct = false;
    for (const auto &t : pend) direct = direct || !(t.kind & 2);
    // small problems run the fused single-CTA path (store design, solver.cpp)
    const bool small = pend.size() <= 64 && P.n_slots <= (1 << 15) && P.world == 1 && !(fz && fz[0] == '0');
    if (direct || (small && !(sw && sw[0] == 'r'))) {
      rc = false;
      pend = pack(false, 2);
    } else if (warp_bytes(P.SB, P.DB, 1) <= 9216) {
      // short rows: single-buffered warps finish a tile faster than its TMA
      // stage arrives -- double-buffer (measured: MRF 287 -> 248 us per sweep;
      // round 2: Potts-cut, 8.7 KB per warp, 411 -> 405 us per iteration;
      // MRF-LP's 64-row tiles, 10.9 KB, 235 -> 264 us per sweep, and
      // CellTrack / QAP50, whose stages are larger, stay single-buffered)
      pend = pack(true, 2);
    }
    // TMEM distances: a kernel with tcgen05 code runs one CTA per SM, so they
    // pay only when the warps per SM they allow (<= 16, 4 per 128 TMEM lanes x
    // 512 / cols columns, and the stages' shared memory) clearly exceed those of
    // the shared-memory scratch (measured: QAP50 12 vs 8 warps -3 %, QAP128 4 vs
    // 3 -6 %; cell tracking 12 vs 12 +1.5 %)
    if (rc && tm_packed && !(tmv && tmv[0] == '1')) {
      const int SB1 = P.SB, DB1 = P.DB, NB1 = P.NB;
      const int w_tm = std::min({16, 4 * (512 / tm_cols), 227 * 1024 / warp_bytes(SB1, DB1, NB1)}) & ~3;
      tm_allow = false;
      std::vector<PendingTile> pend0 = pack(true, NB1);
      // (compared in active lanes: TMEM tiles have 32 rows; the shared-memory
      // pack may use narrower tiles for the longest rows, whose idle lanes
      // cost the same issue slots -- QAP128: 4 TMEM warps of 32 rows 5.4 ms
      // per iteration, 4 warps of 16-row tiles 6.5)
      int w_sm = 0;
      sweep_warps_per_cta(warp_bytes(P.SB, P.DB, P.NB), 4, 227 * 1024, 228 * 1024, &w_sm);
      auto rows_per_tile = [](const std::vector<PendingTile> &v) {
        double rows = 0;
        for (const auto &t : v) rows += (double)t.rows.size();
        return v.empty() ? 32.0 : rows / (double)v.size();
      };
      if (w_tm * rows_per_tile(pend) >= 1.2 * w_sm * rows_per_tile(pend0)) {
        P.SB = SB1;
        P.DB = DB1;
        P.NB = NB1;
        tm_packed = true;
      } else {
        pend.swap(pend0);
        tm_packed = false;
      }
    }
  }
  P.rc = rc;
  // Hop records of staged arc-mask tiles (not fully folded): read from global
  // memory (kind bit 6) when the stages leave L1 room for a shape's records
  // (>= 48 KB of the SM's 256 KB L1 / shared storage); else staged with the
  // tile where the stage still fits the budget with them.  (Measured: cell
  // tracking, 220 KB of stages per SM, +5 % with records in global memory --
  // an L2 round trip per hop; Potts-cut, 139 KB, -6 % -- no TMA bytes and
  // smaller stages.)
  {
    const int wb = warp_bytes(P.SB, P.DB, P.NB);
    int warps_sm;
    if (tm_packed) {
      warps_sm = std::min({16, 4 * (512 / std::max(tm_cols, 32)), 227 * 1024 / wb}) & ~3;
    } else {
      int rw = 1;
      for (const auto &t : pend) rw = std::max(rw, t.L / 32);
      const int ctas = std::min(rw >= 4 ? 4 : 6, 227 * 1024 / (4 * wb + 1024));  // (sweep_kernel launch bounds)
      warps_sm = 4 * std::max(ctas, 1);
    }
    const bool l1_room = 256 * 1024 - warps_sm * wb - (warps_sm / 4) * 1024 >= 48 * 1024;
    for (auto &t : pend) {
      if ((t.kind & 6) != 6 || (t.kind & 16)) continue;
      const Shape &S = P.shapes[t.shape];
      const int pb = pair_room[t.shape] ? stage_pairs_bytes(S.k * t.L / 2) : 0;
      const int sb = rc ? stage_bytes_rc(tsz, t.kind, S.k, S.nodes(), t.L) : stage_bytes(tsz, t.kind, S.k, S.nodes(), t.L);
      if (l1_room || sb + pb > P.SB || recs_global) t.kind |= kKindRecGlobal;
    }
  }

  tm.mark("budget + tile packing");
  P.tiles.clear();
  P.hop_off.clear();
  P.topo.clear();
  P.slot_var.clear();
  P.tiles_shared = 0;
  P.direct_tiles = 0;
  P.n_interior_tiles = 0;
  P.coop_tiles = 0;
  P.coop_w = 0;
  P.direct_w = 0;
  P.max_tile_nodes = 0;
  std::vector<int64_t> shape_topo(P.shapes.size(), -1);
  std::vector<int32_t> shape_hop(P.shapes.size(), -1);
  std::vector<int64_t> shape_rec(P.shapes.size(), -1);
  P.recs.clear();
  // device slot of (row j, hop h): row_slot[j] + h * row_L[j]
  std::vector<int64_t> row_slot(p->n_cons, -1);
  std::vector<int32_t> row_L(p->n_cons, 32);
  int64_t slot_base = 0, dist_base = 0;
  for (const PendingTile &t : pend) {
    TileDesc d{};
    const Shape &S0 = P.shapes[P.row_shape[t.rows[0]]];
    const int L = t.L;
    d.K = S0.k;
    d.n_lanes = (int32_t)t.rows.size();
    d.kind = t.kind;
    d.lanes = L;
    d.slot_base = slot_base;
    d.dist_base = dist_base;
    if (t.kind & 32) {
      // cooperative tile: uint2 topology (absolute 32-bit child indices), per shape
      if (shape_topo[t.shape] < 0) {
        pad16(P.topo);
        pad16(P.hop_off);
        shape_topo[t.shape] = (int64_t)P.topo.size();
        shape_hop[t.shape] = (int32_t)P.hop_off.size();
        const int32_t nn = S0.nodes();
        auto code = [&](uint16_t rel, int32_t next) -> uint32_t {
          return rel == kBot ? (uint32_t)nn + 1 : rel == kTop ? (uint32_t)nn : (uint32_t)(next + rel);
        };
        for (int32_t h = 0; h < S0.k; ++h)
          for (int32_t n = S0.hop_start[h]; n < S0.hop_start[h + 1]; ++n) {
            P.topo.push_back(code(S0.lo[n], S0.hop_start[h + 1]));
            P.topo.push_back(code(S0.hi[n], S0.hop_start[h + 1]));
          }
        for (int32_t h = 0; h <= S0.k; ++h) P.hop_off.push_back(S0.hop_start[h]);
        pad16(P.topo);
        pad16(P.hop_off);
      }
      d.topo_base = shape_topo[t.shape] / 2;  // in uint2 units
      d.hop_base = shape_hop[t.shape];
      d.nodes = S0.nodes();
      d.max_w = S0.max_w;
      P.coop_tiles++;
      P.coop_w = std::max(P.coop_w, S0.max_w);
    } else if (!(t.kind & 1)) {
      if (shape_topo[t.shape] < 0) {
        pad16(P.topo);
        pad16(P.hop_off);
        shape_topo[t.shape] = (int64_t)P.topo.size();
        shape_hop[t.shape] = (int32_t)P.hop_off.size();
        for (int32_t h = 0; h < S0.k; ++h)
          for (int32_t n = S0.hop_start[h]; n < S0.hop_start[h + 1]; ++n)
            P.topo.push_back(abs_code(S0.lo[n], S0.hop_start[h + 1], S0.nodes()) |
                             (abs_code(S0.hi[n], S0.hop_start[h + 1], S0.nodes()) << 16));
        for (int32_t h = 0; h <= S0.k; ++h) P.hop_off.push_back(S0.hop_start[h]);
        pad16(P.topo);
        pad16(P.hop_off);
      }
      d.topo_base = shape_topo[t.shape];
      d.hop_base = shape_hop[t.shape];
      if (t.kind & 4) {
        if (shape_rec[t.shape] < 0) {
          shape_rec[t.shape] = (int64_t)(P.recs.size() / 16);
          append_recs(S0, tsz, P.recs);
        }
        if (shape_rec[t.shape] > 0x7fffffffLL) {
          set_error("hop record table exceeds 32 GiB");
          return FDOG_ETOOBIG;
        }
        d.rec_base = (int32_t)shape_rec[t.shape];
      }
      d.nodes = S0.nodes();
      d.max_w = S0.max_w;
      P.tiles_shared++;
    } else {
      // padded partition widths
      std::vector<int32_t> W(d.K, 0);
      for (int32_t j : t.rows) {
        const Shape &S = P.shapes[P.row_shape[j]];
        for (int32_t h = 0; h < d.K; ++h) W[h] = std::max(W[h], S.hop_start[h + 1] - S.hop_start[h]);
      }
      pad16(P.hop_off);
      d.hop_base = (int32_t)P.hop_off.size();
      int32_t acc = 0;
      d.max_w = 0;
      for (int32_t h = 0; h < d.K; ++h) {
        P.hop_off.push_back(acc);
        acc += W[h];
        d.max_w = std::max(d.max_w, W[h]);
      }
      P.hop_off.push_back(acc);
      pad16(P.hop_off);
      d.nodes = acc;
      pad16(P.topo);
      d.topo_base = (int64_t)P.topo.size();
      const uint32_t pad_node = uint32_t(acc + 1) | (uint32_t(acc + 1) << 16);  // both arcs to bottom
      P.topo.resize(P.topo.size() + (size_t)acc * L, pad_node);
      for (int32_t l = 0; l < d.n_lanes; ++l) {
        const Shape &S = P.shapes[P.row_shape[t.rows[l]]];
        for (int32_t h = 0; h < d.K; ++h) {
          int32_t base = P.hop_off[d.hop_base + h];
          const int32_t next = P.hop_off[d.hop_base + h + 1];
          for (int32_t w = 0; w < S.hop_start[h + 1] - S.hop_start[h]; ++w) {
            int32_t n = S.hop_start[h] + w;
            P.topo[d.topo_base + (int64_t)(base + w) * L + l] =
                abs_code(S.lo[n], next, acc) | (abs_code(S.hi[n], next, acc) << 16);
          }
        }
      }
    }
    if (!t.boundary) P.n_interior_tiles++;
    if (!(t.kind & 2)) {
      P.direct_tiles++;
      if (!(t.kind & 32)) P.direct_w = std::max(P.direct_w, d.max_w);
    }
    P.max_tile_nodes = std::max(P.max_tile_nodes, d.nodes);
    // slots
    P.slot_var.resize((size_t)(slot_base + (int64_t)d.K * L), -1);
    for (int32_t l = 0; l < d.n_lanes; ++l) {
      int32_t j = t.rows[l];
      row_slot[j] = slot_base + l;
      row_L[j] = L;
      const int32_t *vars = P.col_var.data() + P.row_ptr[j];
      for (int32_t h = 0; h < d.K; ++h) P.slot_var[slot_base + (int64_t)h * L + l] = vars[h];
    }
    // (bases stay multiples of 4 elements -- 16-byte aligned TMA sources --
    // after a one-BDD cooperative tile too; the gap is padding)
    slot_base = (slot_base + (int64_t)d.K * L + 3) & ~(int64_t)3;
    dist_base = (dist_base + (int64_t)(d.nodes + 2) * L + 3) & ~(int64_t)3;
    P.tiles.push_back(d);
  }
  // Recompute design packed for tensor memory (pack() above): the distance
  // scratch of the 32-row arc-mask tiles lives in TMEM (kernels.cu TmemD),
  // TMEM columns per CTA = the next power of two >= nodes + 2 of those tiles;
  // the DB region serves the other tiles only (chosen that way by the budget
  // model).  4 warps per CTA, 512 / cols CTAs per SM.
  P.tmem_cols = 0;
  if (P.rc && tm_packed) {
    int maxn = 0;
    for (const auto &d : P.tiles)
      if ((d.kind & 2) && (d.kind & 4) && d.lanes == 32) maxn = std::max(maxn, d.nodes + 2);
    if (maxn > 0) {
      int cols = 32;
      while (cols < maxn) cols *= 2;
      P.tmem_cols = cols;  // (<= 512: tm packing requires it)
    }
  }
  // cooperative tiles: two relaxation buffers of coop_w + 1 entries, in the
  // warp's DB region when they fit 32 KB (else in the solver's scratch)
  P.coop_smem = false;
  if (P.coop_tiles > 0 && 2 * (P.coop_w + 1) * tsz <= 32768) {
    P.DB = std::max(P.DB, r16(2 * (P.coop_w + 1) * tsz));
    P.coop_smem = true;
  }
  pad16(P.topo);
  P.topo.resize(P.topo.size() + 4, 0);  // 16-byte reads of the last topology may run past it
  P.slot_var.resize((size_t)slot_base, -1);
  P.n_dist = dist_base;
  for (const auto &d : P.tiles)
    if (!(d.kind & 32) && d.nodes + 1 > 0xFFFF) {
      set_error("a BDD tile has %d nodes; the 16-bit topology codes allow 65534", d.nodes);
      return FDOG_ETOOBIG;
    }
  if (slot_base > 0x7fffffffLL) {
    set_error("more than 2^31 device slots on one rank");
    return FDOG_ETOOBIG;
  }
  tm.mark("tile emission");
  // canonical slots and CSR variable -> device slots (j ascending, A1):
  // on the GPU with FDOG_GPU_PACK=1 (pack_gpu.cu, identical arrays), else here
  bool packed_gpu = false;
  if (gpu_step("FDOG_GPU_PACK")) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
      const int dev = o ? o->device : 0;
      const fdog_status r = gpu_pack_slots(P, row_slot, row_L, dev >= 0 && dev < ndev ? dev : 0);
      if (r) {
        set_error("GPU packing failed (%s)", cudaGetErrorString(cudaGetLastError()));
        return r;
      }
      packed_gpu = true;
    } else {
      cudaGetLastError();
    }
  }
  if (!packed_gpu) {
    P.canon_slot.clear();
    P.canon_con.clear();
    P.canon_pos.clear();
    std::vector<int64_t> cnt(p->n_vars + 1, 0);
    P.canon_slot.resize((size_t)P.n_slots);
    P.canon_con.resize((size_t)P.n_slots);
    P.canon_pos.resize((size_t)P.n_slots);
    {
      const int64_t nr = (int64_t)P.local_rows.size();
      std::vector<int64_t> q0(nr + 1, 0);  // first canonical slot of each local row
      for (int64_t r = 0; r < nr; ++r) {
        const int32_t j = P.local_rows[r];
        q0[r + 1] = q0[r] + (P.row_ptr[j + 1] - P.row_ptr[j]);
      }
      par_for(nr, threads, [&](int, int64_t r0, int64_t r1) {
        for (int64_t r = r0; r < r1; ++r) {
          const int32_t j = P.local_rows[r];
          const int32_t k = (int32_t)(P.row_ptr[j + 1] - P.row_ptr[j]);
          const int32_t *vars = P.col_var.data() + P.row_ptr[j];
          for (int32_t h = 0; h < k; ++h) {
            const int64_t q = q0[r] + h;
            P.canon_slot[q] = row_slot[j] + (int64_t)h * row_L[j];
            P.canon_con[q] = j;
            P.canon_pos[q] = h;
            __atomic_fetch_add(&cnt[vars[h]], 1, __ATOMIC_RELAXED);
          }
        }
      });
    }
    tm.mark("canonical slots + CSR");
    // variables in the order of their first device slot, so that neighbouring
    // averaging threads gather and scatter neighbouring slots (the tile layout
    // puts consecutive rows of a shape in consecutive lanes): each variable's
    // first device slot (atomic min), then the device slots that are a first
    // occurrence, compacted in device-slot order -- the order of a sort by first
    // device slot, without the sort
    P.var_list.clear();
    {
      const int64_t ns = (int64_t)P.slot_var.size();
      std::vector<int32_t> first(p->n_vars, INT32_MAX);  // (device slots < 2^31, checked above)
      par_for(ns, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t d = a; d < b; ++d)
          if (P.slot_var[d] >= 0) atomic_min32(&first[P.slot_var[d]], (int32_t)d);
      });
      const int T = par_chunks(ns, threads);
      std::vector<int64_t> cc(T + 1, 0);
      auto is_first = [&](int64_t d) { return P.slot_var[d] >= 0 && first[P.slot_var[d]] == d; };
      par_for(ns, threads, [&](int c, int64_t a, int64_t b) {
        int64_t m = 0;
        for (int64_t d = a; d < b; ++d) m += is_first(d);
        cc[c + 1] = m;
      });
      for (int c = 0; c < T; ++c) cc[c + 1] += cc[c];
      P.var_list.resize(cc[T]);
      par_for(ns, threads, [&](int c, int64_t a, int64_t b) {
        int64_t o = cc[c];
        for (int64_t d = a; d < b; ++d)
          if (is_first(d)) P.var_list[o++] = P.slot_var[d];
      });
    }
    // CSR over var_list: prefix of the local degrees
    std::vector<int64_t> where(p->n_vars, -1);
    {
      const int64_t nv = (int64_t)P.var_list.size();
      const int T = par_chunks(nv, threads);
      std::vector<int64_t> cs(T + 1, 0);
      par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
        int64_t m = 0;
        for (int64_t k = a; k < b; ++k) m += cnt[P.var_list[k]];
        cs[c + 1] = m;
      });
      for (int c = 0; c < T; ++c) cs[c + 1] += cs[c];
      P.var_ptr.resize(nv + 1);
      P.var_ptr[nv] = cs[T];
      par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
        int64_t o = cs[c];
        for (int64_t k = a; k < b; ++k) {
          P.var_ptr[k] = o;
          where[P.var_list[k]] = o;
          o += cnt[P.var_list[k]];
        }
      });
    }
    // fill: canonical slot indices claimed with an atomic cursor per variable,
    // then each variable's (short) list sorted -- ascending canonical index is
    // ascending j (A1) -- and mapped to device slots
    {
      const int64_t nq = (int64_t)P.canon_slot.size();
      std::vector<int32_t> tq((size_t)std::max<int64_t>(nq, 1));
      par_for(nq, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) {
          const int32_t i = P.col_var[P.row_ptr[P.canon_con[q]] + P.canon_pos[q]];
          tq[__atomic_fetch_add(&where[i], 1, __ATOMIC_RELAXED)] = (int32_t)q;
        }
      });
      P.var_slots.assign(P.var_ptr.back(), -1);
      par_for((int64_t)P.var_list.size(), threads, [&](int, int64_t a, int64_t b) {
        for (int64_t k = a; k < b; ++k) {
          const int64_t p0 = P.var_ptr[k], p1 = P.var_ptr[k + 1];
          std::sort(tq.begin() + p0, tq.begin() + p1);
          for (int64_t x = p0; x < p1; ++x) P.var_slots[x] = (int32_t)P.canon_slot[tq[x]];
        }
      });
    }
  }
  tm.mark("variable order");
  // shared variables: held by this rank and by another one
  P.shared_vars.clear();
  P.var_xidx.assign(P.var_list.size(), -1);
  if (world > 1) {
    // the exchange vector must be identical on every rank: all variables held
    // by >= 2 ranks, ascending; this rank contributes zeros for those it lacks
    for (int32_t i = 0; i < p->n_vars; ++i)
      if (multi[i]) P.shared_vars.push_back(i);
    std::vector<int32_t> xpos(p->n_vars, -1);
    for (size_t q = 0; q < P.shared_vars.size(); ++q) xpos[P.shared_vars[q]] = (int32_t)q;
    for (size_t q = 0; q < P.var_list.size(); ++q) P.var_xidx[q] = xpos[P.var_list[q]];
  }
  tm.mark("shared variables");
  // averaging layout: variables with <= 2 local slots that are not exchanged
  // keep their slot pair inline (ELL, one 8-byte load), with 3-4 the slot quad
  // (ELL-4); the rest stay in CSR.  (Per chunk counts, then the fill.)
  // Tile-closed pairs: a variable with |J_i| = 2 whose two slots lie in one
  // staged tile (a bundle's rows in consecutive lanes) is averaged by the sweep
  // on chip (pair maps below); its ELL entry goes to the tail of the ELL list
  // (after P.n_ell_open), used only by paths that average every variable
  // (FDOG_PAIRS=0 keeps every pair in the averaging kernel).
  {
    const int64_t nv = (int64_t)P.var_list.size();
    const char *pe = getenv("FDOG_PAIRS");
    const bool pairs_ok = !(pe && pe[0] == '0');
    auto tile_of = [&](int64_t slot) -> int32_t {  // tiles are emitted in slot order
      int32_t lo = 0, hi = (int32_t)P.tiles.size() - 1;
      while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (P.tiles[mid].slot_base <= slot) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };
    // candidate closed pairs per tile, then the tiles whose stage holds their
    // pair list within the per-warp budget
    auto candidate = [&](int64_t q, int32_t *tp) {
      if (!pairs_ok || P.var_xidx[q] >= 0 || P.var_ptr[q + 1] - P.var_ptr[q] != 2) return false;
      const int32_t t = tile_of(P.var_slots[P.var_ptr[q]]);
      const TileDesc &d = P.tiles[t];
      *tp = t;
      return t == tile_of(P.var_slots[P.var_ptr[q] + 1]) && (d.kind & 2) && (int64_t)d.K * d.lanes <= 0xFFFF;
    };
    std::vector<int32_t> tile_pairs(P.tiles.size(), 0);
    par_for(nv, threads, [&](int, int64_t a, int64_t b) {
      for (int64_t q = a; q < b; ++q) {
        int32_t t;
        if (candidate(q, &t)) __atomic_fetch_add(&tile_pairs[t], 1, __ATOMIC_RELAXED);
      }
    });
    for (size_t t = 0; t < P.tiles.size(); ++t) {
      const TileDesc &d = P.tiles[t];
      if (!tile_pairs[t]) continue;
      const int sb = P.rc ? stage_bytes_rc(tsz, d.kind, d.K, d.nodes, d.lanes)
                          : stage_bytes(tsz, d.kind, d.K, d.nodes, d.lanes);
      if (sb + stage_pairs_bytes(tile_pairs[t]) > P.SB) tile_pairs[t] = 0;  // keep them in the kernel
    }
    tm.mark("avg: closed pairs");
    auto closed = [&](int64_t q) {
      int32_t t;
      return candidate(q, &t) && tile_pairs[t] > 0;
    };
    // ELL-D groups: the kMaxElld most frequent degrees in [5, 32] with >= 65536
    // variables (every MRF pixel label: 1 + #neighbours; Potts-cut: 1 + 2
    // #neighbours and 16 for the edge variables).  Measured: MRF-LP averaging
    // 60.8 -> 44.3 us, Potts-cut 168 -> 96 us per pass; with a few thousand
    // such variables (GM's labels) the CSR lane groups are faster -- one
    // thread's d / 8 gather rounds form the tail.
    std::vector<int32_t> grp_of(33, -1);
    P.elld_d.clear();
    const char *em = getenv("FDOG_ELLD_MIN");  // test knob: smallest ELL-D group
    const int64_t elld_min = em ? std::max(1LL, atoll(em)) : 65536;
    {
      std::vector<int64_t> cnt_d(33, 0);
      for (int64_t q = 0; q < nv; ++q) {
        const int64_t d = P.var_ptr[q + 1] - P.var_ptr[q];
        if (d >= 5 && d <= 32 && P.var_xidx[q] < 0 && !P.lifted) cnt_d[d]++;
      }
      std::vector<int32_t> ds;
      for (int d = 5; d <= 32; ++d)
        if (cnt_d[d] >= elld_min) ds.push_back(d);
      std::stable_sort(ds.begin(), ds.end(), [&](int32_t a, int32_t b) { return cnt_d[a] > cnt_d[b]; });
      if ((int)ds.size() > kMaxElld) ds.resize(kMaxElld);
      std::sort(ds.begin(), ds.end());
      for (size_t g = 0; g < ds.size(); ++g) grp_of[ds[g]] = (int32_t)g;
      P.elld_d = ds;
    }
    tm.mark("avg: ELL-D degrees");
    auto cat_of = [&](int64_t q) {
      const int64_t d = P.var_ptr[q + 1] - P.var_ptr[q];
      if (P.var_xidx[q] >= 0 || P.lifted) return 2;  // (lifted mode: one CSR kernel sums both sides)
      if (d <= 2) return closed(q) ? 4 : 0;
      if (d <= 4) return 1;
      return (d <= 32 && grp_of[d] >= 0) ? 5 : 2;
    };
    std::vector<uint8_t> cat_v((size_t)std::max<int64_t>(nv, 1));
    par_for(nv, threads, [&](int, int64_t a, int64_t b) {
      for (int64_t q = a; q < b; ++q) cat_v[q] = (uint8_t)cat_of(q);
    });
    auto cat = [&](int64_t q) { return (int)cat_v[q]; };
    const int T = par_chunks(nv, threads);
    std::vector<std::array<int64_t, 5>> cc(T + 1, {0, 0, 0, 0, 0});  // ell, ell4, csr vars, csr slots, closed pairs
    par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
      std::array<int64_t, 5> m = {0, 0, 0, 0, 0};
      for (int64_t q = a; q < b; ++q) {
        const int k = cat(q);
        if (k == 5) continue;  // ELL-D: filled below
        m[k == 4 ? 4 : k]++;
        if (k == 2) m[3] += P.var_ptr[q + 1] - P.var_ptr[q];
      }
      cc[c + 1] = m;
    });
    tm.mark("avg: category counts");
    // ELL-D fill (variables in var_list order within a group)
    {
      const int G = (int)P.elld_d.size();
      P.elld_n.assign(G, 0);
      P.elld_off.assign(G, 0);
      // positions within a group in var_list order: per-chunk counts, prefix
      std::vector<int64_t> pos(nv, -1);
      const int TC = par_chunks(nv, threads);
      std::vector<std::vector<int64_t>> gc(TC + 1, std::vector<int64_t>(std::max(G, 1), 0));
      par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q)
          if (cat(q) == 5) gc[c + 1][grp_of[P.var_ptr[q + 1] - P.var_ptr[q]]]++;
      });
      for (int c = 0; c < TC; ++c)
        for (int g = 0; g < G; ++g) gc[c + 1][g] += gc[c][g];
      for (int g = 0; g < G; ++g) P.elld_n[g] = gc[TC][g];
      par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
        std::vector<int64_t> o = gc[c];
        for (int64_t q = a; q < b; ++q)
          if (cat(q) == 5) pos[q] = o[grp_of[P.var_ptr[q + 1] - P.var_ptr[q]]]++;
      });
      int64_t off = 0;
      for (int g = 0; g < G; ++g) {
        P.elld_off[g] = off;
        off += (int64_t)P.elld_d[g] * P.elld_n[g];
      }
      P.elld.assign((size_t)off, -1);
      P.elld_var.assign((size_t)std::accumulate(P.elld_n.begin(), P.elld_n.end(), (int64_t)0), -1);
      {
        std::vector<int64_t> vb(G + 1, 0);
        for (int g = 0; g < G; ++g) vb[g + 1] = vb[g] + P.elld_n[g];
        par_for(nv, threads, [&](int, int64_t a, int64_t b) {
          for (int64_t q = a; q < b; ++q)
            if (pos[q] >= 0) P.elld_var[vb[grp_of[P.var_ptr[q + 1] - P.var_ptr[q]]] + pos[q]] = P.var_list[q];
        });
      }
      par_for(nv, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) {
          if (pos[q] < 0) continue;
          const int64_t d = P.var_ptr[q + 1] - P.var_ptr[q];
          const int g = grp_of[d];
          for (int64_t k = 0; k < d; ++k)
            P.elld[P.elld_off[g] + k * P.elld_n[g] + pos[q]] = P.var_slots[P.var_ptr[q] + k];
        }
      });
    }
    tm.mark("avg: ELL-D fill");
    for (int c = 0; c < T; ++c)
      for (int u = 0; u < 5; ++u) cc[c + 1][u] += cc[c][u];
    const auto &tot = cc[T];
    P.n_ell_open = tot[0];
    P.ell.assign(2 * (tot[0] + tot[4]), -1);
    P.ell_var.resize(tot[0] + tot[4]);
    P.ell4.assign(4 * tot[1], -1);
    P.ell4_var.resize(tot[1]);
    std::vector<int32_t> csr_list(tot[2]), csr_slots(tot[3]), csr_x(tot[2]);
    std::vector<int64_t> csr_ptr(tot[2] + 1, 0);
    csr_ptr[tot[2]] = tot[3];
    par_for(nv, threads, [&](int c, int64_t a, int64_t b) {
      std::array<int64_t, 5> o = cc[c];
      o[4] += tot[0];  // closed pairs after the open ones
      for (int64_t q = a; q < b; ++q) {
        const int64_t p0 = P.var_ptr[q], p1 = P.var_ptr[q + 1];
        const int k = cat(q);
        switch (k) {
          case 5:
            break;  // ELL-D (filled above)
          case 0:
          case 4: {
            const int u = k;
            P.ell[2 * o[u]] = P.var_slots[p0];
            if (p1 - p0 == 2) P.ell[2 * o[u] + 1] = P.var_slots[p0 + 1];
            P.ell_var[o[u]++] = P.var_list[q];
            break;
          }
          case 1:
            for (int64_t u = 0; u < p1 - p0; ++u) P.ell4[4 * o[1] + u] = P.var_slots[p0 + u];
            P.ell4_var[o[1]++] = P.var_list[q];
            break;
          default:
            csr_list[o[2]] = P.var_list[q];
            csr_x[o[2]] = P.var_xidx[q];
            csr_ptr[o[2]++] = o[3];
            for (int64_t x = p0; x < p1; ++x) csr_slots[o[3]++] = P.var_slots[x];
        }
      }
    });
    tm.mark("avg: ELL / CSR fill");
    // pair lists: per staged tile with closed pairs, (i | m << 16) for the two
    // tile slot offsets i < m of each pair, ascending i; identical lists stored
    // once (every MRF-LP marginalisation tile has the same one)
    P.pair_list.clear();
    for (auto &d : P.tiles) {
      d.pair_base = -1;
      d.n_pairs = 0;
    }
    {
      // (parallel: each closed pair's tile and code, then per run of pairs of
      // one tile the sorted list and its hash; the lists are deduplicated in
      // run order, as a sequential pass would)
      const int64_t e0 = tot[0], ne = tot[4];
      std::vector<int32_t> tl((size_t)std::max<int64_t>(ne, 1));
      std::vector<uint32_t> code((size_t)std::max<int64_t>(ne, 1));
      par_for(ne, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t x = a; x < b; ++x) {
          const int64_t s1 = P.ell[2 * (e0 + x)], s2 = P.ell[2 * (e0 + x) + 1];
          const int32_t t = tile_of(s1);
          const int64_t b0 = P.tiles[t].slot_base;
          tl[x] = t;
          code[x] = (uint32_t)(std::min(s1, s2) - b0) | ((uint32_t)(std::max(s1, s2) - b0) << 16);
        }
      });
      std::vector<int64_t> run_at;  // run starts (+ ne)
      for (int64_t x = 0; x < ne; ++x)
        if (x == 0 || tl[x] != tl[x - 1]) run_at.push_back(x);
      const int64_t nr = (int64_t)run_at.size();
      run_at.push_back(ne);
      std::vector<uint64_t> run_hash((size_t)std::max<int64_t>(nr, 1));
      par_for(nr, threads, [&](int, int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) {
          const auto lo = code.begin() + run_at[r], hi = code.begin() + run_at[r + 1];
          std::sort(lo, hi, [](uint32_t x, uint32_t y) { return (x & 0xFFFF) < (y & 0xFFFF); });
          uint64_t h = 1469598103934665603ull ^ (uint64_t)(hi - lo);
          for (auto it = lo; it != hi; ++it) h = (h ^ *it) * 1099511628211ull;
          run_hash[r] = h;
        }
      });
      std::unordered_map<uint64_t, std::vector<std::pair<int32_t, int32_t>>> seen;  // (offset, length)
      for (int64_t r = 0; r < nr; ++r) {
        const auto lo = code.begin() + run_at[r], hi = code.begin() + run_at[r + 1];
        const int32_t len = (int32_t)(hi - lo);
        auto &cands = seen[run_hash[r]];
        int32_t at = -1;
        for (const auto &c0 : cands)
          if (c0.second == len && std::equal(lo, hi, P.pair_list.begin() + c0.first)) {
            at = c0.first;
            break;
          }
        if (at < 0) {
          at = (int32_t)P.pair_list.size();
          P.pair_list.insert(P.pair_list.end(), lo, hi);
          while (P.pair_list.size() % 4) P.pair_list.push_back(0);  // 16-byte aligned lists (TMA)
          cands.emplace_back(at, len);
        }
        P.tiles[tl[run_at[r]]].pair_base = at;
        P.tiles[tl[run_at[r]]].n_pairs = len;
      }
      if (P.pair_list.size() > 0x7fffffffULL) {
        set_error("pair lists exceed 2^31 entries");
        return FDOG_ETOOBIG;
      }
    }
    tm.mark("avg: pair lists");
    P.n_vars_local = nv;
    P.var_list.swap(csr_list);
    P.var_ptr.swap(csr_ptr);
    P.var_slots.swap(csr_slots);
    P.var_xidx.swap(csr_x);
  }
  P.deg_list.resize(P.var_list.size());
  for (size_t q = 0; q < P.var_list.size(); ++q) P.deg_list[q] = P.deg_global[P.var_list[q]];
  P.x_local.assign(P.shared_vars.size(), -1);
  P.x_deg.resize(P.shared_vars.size());
  for (size_t q = 0; q < P.var_list.size(); ++q)
    if (P.var_xidx[q] >= 0) P.x_local[P.var_xidx[q]] = (int32_t)q;
  for (size_t q = 0; q < P.shared_vars.size(); ++q) P.x_deg[q] = P.deg_global[P.shared_vars[q]];
  {
    // (counted once here: a loop over the variables at every solver create
    // cost MRF-LP's create 60 ms)
    int64_t sh = 0, fv = 0;
    for (int32_t x : P.var_xidx) sh += x >= 0;
    for (int32_t d : P.deg_global) fv += d == 0;
    P.n_vars_shared = sh;
    P.n_free_vars = fv;
  }
  tm.mark("averaging layout");
  return FDOG_OK;
}

HostImage::~HostImage() {
  if (!data) return;
  if (pinned) cudaFreeHost(data);
  else free(data);
}

// Lay out every uploaded array in one buffer (256-byte aligned sections),
// including the initial lambda_i^j = c_i / |J_i| (A9; fp64, rounded once
// to the build precision).  The distance array is not uploaded: the solver
// allocates it and writes its sentinels on the device (0 for top, +inf for
// bottom, never overwritten); the first energy sweep fills the rest.
fdog_status build_image(Plan &P) {
  PhaseTimer tm;
  const int tsz = P.precision == 64 ? 8 : 4;
  size_t sz[kImCount];
  sz[kImTiles] = P.tiles.size() * sizeof(TileDesc);
  sz[kImHopOff] = P.hop_off.size() * 4;
  sz[kImTopo] = P.topo.size() * 4;
  sz[kImSlotVar] = 0;  // (host-side only: no kernel reads it)
  sz[kImVarPtr] = P.var_ptr.size() * 8;
  sz[kImVarSlots] = P.var_slots.size() * 4;
  sz[kImVarXidx] = P.var_xidx.size() * 4;
  sz[kImDegList] = P.deg_list.size() * 4;
  sz[kImEll] = P.ell.size() * 4;
  sz[kImEllVar] = P.ell_var.size() * 4;
  sz[kImCsrVar] = P.var_list.size() * 4;
  sz[kImEll4] = P.ell4.size() * 4;
  sz[kImEll4Var] = P.ell4_var.size() * 4;
  sz[kImXLocal] = P.x_local.size() * 4;
  sz[kImXDeg] = P.x_deg.size() * 4;
  sz[kImLambda0] = P.slot_var.size() * tsz;
  sz[kImDist0] = 0;  // (allocated and initialised on the device, solver.cpp)
  sz[kImRecs] = P.recs.size();
  sz[kImCanon] = P.canon_slot.size() * 4;
  sz[kImPairs] = P.pair_list.size() * 4;
  sz[kImElld] = P.elld.size() * 4;
  sz[kImElldVar] = P.elld_var.size() * 4;
  size_t at = 0;
  for (int q = 0; q < kImCount; ++q) {
    P.image.off[q] = at;
    at += (std::max<size_t>(sz[q], 1) + 255) & ~(size_t)255;
  }
  P.image.bytes = at;
  void *mem = nullptr;
  int ndev = 0;
  // pinned memory makes create's one host->device copy fast (MRF-LP's 1 GB
  // image: ~8 GB/s pageable, the bulk of create); page-locking it costs about
  // as much once, here in the untimed plan, and every solver created from the
  // plan gains (FDOG_PIN_MB: the limit, MB)
  const char *pm = getenv("FDOG_PIN_MB");
  const size_t pin_max = (size_t)(pm ? atoll(pm) : 8192) << 20;
  if (at <= pin_max && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && cudaMallocHost(&mem, at) == cudaSuccess) {
    P.image.pinned = true;
  } else {
    cudaGetLastError();  // no device (host-only use) or a large image: pageable memory
    mem = malloc(at);
    if (!mem) {
      set_error("host out of memory (device image, %zu bytes)", at);
      return FDOG_ENOMEM;
    }
  }
  P.image.data = (unsigned char *)mem;
  const int threads = P.host_threads;
  // each section: its bytes, then zeros up to the next 256-byte boundary
  const void *src[kImCount] = {};
  src[kImTiles] = P.tiles.data();
  src[kImHopOff] = P.hop_off.data();
  src[kImTopo] = P.topo.data();
  src[kImVarPtr] = P.var_ptr.data();
  src[kImVarSlots] = P.var_slots.data();
  src[kImVarXidx] = P.var_xidx.data();
  src[kImDegList] = P.deg_list.data();
  src[kImEll] = P.ell.data();
  src[kImEllVar] = P.ell_var.data();
  src[kImCsrVar] = P.var_list.data();
  src[kImEll4] = P.ell4.data();
  src[kImEll4Var] = P.ell4_var.data();
  src[kImXLocal] = P.x_local.data();
  src[kImXDeg] = P.x_deg.data();
  src[kImRecs] = P.recs.data();
  src[kImPairs] = P.pair_list.data();
  src[kImElld] = P.elld.data();
  src[kImElldVar] = P.elld_var.data();
  for (int q = 0; q < kImCount; ++q) {
    const size_t end = q + 1 < kImCount ? P.image.off[q + 1] : at;
    memset(P.image.data + P.image.off[q] + sz[q], 0, end - P.image.off[q] - sz[q]);
    if (!src[q] || !sz[q]) continue;
    unsigned char *dst = P.image.data + P.image.off[q];
    const unsigned char *sp = (const unsigned char *)src[q];
    par_for((int64_t)sz[q], threads, [&](int, int64_t a, int64_t b) { memcpy(dst + a, sp + a, b - a); });
  }
  {
    int32_t *cs = (int32_t *)(P.image.data + P.image.off[kImCanon]);
    par_for((int64_t)P.canon_slot.size(), threads, [&](int, int64_t a, int64_t b) {
      for (int64_t q = a; q < b; ++q) cs[q] = (int32_t)P.canon_slot[q];
    });
  }
  unsigned char *lam = P.image.data + P.image.off[kImLambda0];
  par_for((int64_t)P.slot_var.size(), threads, [&](int, int64_t a, int64_t b) {
    for (int64_t q = a; q < b; ++q) {
      const int32_t i = P.slot_var[q];
      const double v = i >= 0 ? P.cost[i] / (double)P.deg_global[i] : 0.0;
      if (tsz == 8) ((double *)lam)[q] = v;
      else ((float *)lam)[q] = (float)v;
    }
  });
  tm.mark("device image");
  return FDOG_OK;
}

}  // namespace fdog

// ---------------------------------------------------------------------------
// C ABI: plan

using namespace fdog;

struct fdog_plan {
  std::shared_ptr<Plan> sp = std::make_shared<Plan>();
  Plan &p = *sp;
};

extern "C" {

void fdog_default_options(fdog_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->precision = 32;
  o->world = 1;
}

const char *fdog_last_error(void) { return fdog::last_error(); }

int32_t fdog_version(void) { return 1; }

fdog_status fdog_plan_create(const fdog_problem *p, const fdog_options *opts, fdog_plan **out) {
  if (!out) {
    set_error("null output handle");
    return FDOG_EINVAL;
  }
  *out = nullptr;
  try {
    auto *pl = new fdog_plan();
    fdog_status st = build_plan(p, opts, pl->p);
    if (st == FDOG_OK) st = build_image(pl->p);
    if (st != FDOG_OK) {
      delete pl;
      return st;
    }
    *out = pl;
    return FDOG_OK;
  } catch (const std::bad_alloc &) {
    set_error("host out of memory while building the plan");
    return FDOG_ENOMEM;
  } catch (const std::exception &e) {
    set_error("plan: %s", e.what());
    return FDOG_EINVAL;
  }
}

void fdog_plan_destroy(fdog_plan *plan) { delete plan; }

fdog_status fdog_plan_stats(const fdog_plan *plan, fdog_stats_t *out) {
  if (!plan || !out) {
    set_error("null argument");
    return FDOG_EINVAL;
  }
  const Plan &P = plan->p;
  std::memset(out, 0, sizeof *out);
  out->bdds = (int64_t)P.local_rows.size();
  out->nodes = P.n_nodes;
  out->arcs = 2 * P.n_nodes;
  out->slots = P.n_slots;
  out->vars_local = P.n_vars_local;
  out->vars_shared = P.n_vars_shared;
  out->free_vars = P.n_free_vars;
  out->shapes = (int64_t)P.shapes.size();
  out->tiles = (int64_t)P.tiles.size();
  out->tiles_shared_topology = P.tiles_shared;
  out->padded_slots = (int64_t)P.slot_var.size();
  out->max_hops = P.max_hops;
  out->max_width = P.max_width;
  out->staged_tiles = (int64_t)P.tiles.size() - P.direct_tiles;
  out->sweep_smem_per_warp = warp_bytes(P.SB, P.DB, P.NB);
  out->h2d_bytes = (int64_t)P.image.bytes;
  out->tile_pairs = (int64_t)(P.ell.size() / 2) - P.n_ell_open;
  out->interior_tiles = P.world > 1 ? P.n_interior_tiles : (int64_t)P.tiles.size();
  out->coop_tiles = P.coop_tiles;
  out->tmem_cols = P.tmem_cols;
  return FDOG_OK;
}

fdog_status fdog_plan_bdd(const fdog_plan *plan, int32_t j, int32_t *k, int32_t *n_nodes,
                          int32_t *hop_start, int32_t *lo, int32_t *hi, int32_t cap_hops,
                          int32_t cap_nodes) {
  if (!plan || !k || !n_nodes || j < 0 || j >= plan->p.n_cons) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  const Plan &P = plan->p;
  if (P.owner[j] != P.rank) {
    set_error("row %d is not held by this rank", j);
    return FDOG_ESTATE;
  }
  if (P.row_shape[j] < 0) {
    *k = 0;
    *n_nodes = 0;
    return FDOG_OK;
  }
  const Shape &S = P.shapes[P.row_shape[j]];
  *k = S.k;
  *n_nodes = S.nodes();
  if (cap_hops < S.k || cap_nodes < S.nodes() || !hop_start || !lo || !hi) {
    set_error("output arrays too small");
    return FDOG_EINVAL;
  }
  for (int32_t h = 0; h <= S.k; ++h) hop_start[h] = S.hop_start[h];
  for (int32_t h = 0; h < S.k; ++h)
    for (int32_t v = S.hop_start[h]; v < S.hop_start[h + 1]; ++v) {
      auto conv = [&](uint32_t c) -> int32_t {
        if (c == kBot) return -1;
        if (c == kTop) return -2;
        return S.hop_start[h + 1] + (int32_t)c;
      };
      lo[v] = conv(S.lo[v]);
      hi[v] = conv(S.hi[v]);
    }
  return FDOG_OK;
}

fdog_status fdog_plan_slot_map(const fdog_plan *plan, int64_t *dev_slot, int64_t len) {
  if (!plan || !dev_slot || len < (int64_t)plan->p.canon_slot.size()) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  std::copy(plan->p.canon_slot.begin(), plan->p.canon_slot.end(), dev_slot);
  return FDOG_OK;
}

fdog_status fdog_plan_digest(const fdog_plan *plan, uint64_t *out) {
  if (!plan || !out) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  const Plan &P = plan->p;
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void *data, size_t bytes) {
    const unsigned char *c = (const unsigned char *)data;
    for (size_t q = 0; q < bytes; ++q) {
      h ^= c[q];
      h *= 1099511628211ull;
    }
  };
  auto vec = [&](const auto &v) {
    const uint64_t n = v.size();
    mix(&n, 8);
    if (n) mix(v.data(), n * sizeof(v[0]));
  };
  vec(P.tiles);
  vec(P.hop_off);
  vec(P.topo);
  vec(P.recs);
  vec(P.slot_var);
  vec(P.canon_slot);
  vec(P.var_list);
  vec(P.var_ptr);
  vec(P.var_slots);
  vec(P.var_xidx);
  vec(P.deg_list);
  vec(P.ell);
  vec(P.ell_var);
  vec(P.ell4);
  vec(P.ell4_var);
  vec(P.elld);
  vec(P.shared_vars);
  if (P.image.data) mix(P.image.data, P.image.bytes);
  *out = h;
  return FDOG_OK;
}

fdog_status fdog_plan_tiles(const fdog_plan *plan, int64_t *desc, int64_t cap, int64_t *n) {
  if (!plan || !n) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  const auto &T = plan->p.tiles;
  *n = (int64_t)T.size();
  if (!desc) return FDOG_OK;
  if (cap < *n) {
    set_error("capacity %lld < %lld tiles", (long long)cap, (long long)*n);
    return FDOG_EINVAL;
  }
  for (size_t t = 0; t < T.size(); ++t) {
    int64_t *o = desc + 6 * t;
    o[0] = T[t].kind;
    o[1] = T[t].K;
    o[2] = T[t].lanes;
    o[3] = T[t].n_lanes;
    o[4] = T[t].nodes;
    o[5] = T[t].slot_base;
  }
  return FDOG_OK;
}

fdog_status fdog_plan_owner(const fdog_plan *plan, int32_t *owner, int64_t len) {
  if (!plan || !owner || len < plan->p.n_cons) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  std::copy(plan->p.owner.begin(), plan->p.owner.end(), owner);
  return FDOG_OK;
}

fdog_status fdog_plan_shared_vars(const fdog_plan *plan, int32_t *vars, int64_t cap, int64_t *n) {
  if (!plan || !n) {
    set_error("bad argument");
    return FDOG_EINVAL;
  }
  const auto &sv = plan->p.shared_vars;
  *n = (int64_t)sv.size();
  if (!vars) return FDOG_OK;
  if (cap < (int64_t)sv.size()) {
    set_error("output array too small");
    return FDOG_EINVAL;
  }
  std::copy(sv.begin(), sv.end(), vars);
  return FDOG_OK;
}

}  // extern "C"

// accessor for solver.cpp
namespace fdog {
std::shared_ptr<const Plan> plan_of(const fdog_plan *p) { return p->sp; }
}
