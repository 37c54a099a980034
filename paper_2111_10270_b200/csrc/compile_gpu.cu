// compile_gpu.cu -- compiler B on the GPU: one CTA per
// distinct row signature ("shape"), layer-parallel inside the CTA.
//
// Same construction as plan.cpp compile_B, step for step, so the result is
// identical (FDOG_GPU_COMPILE=1; tests/test_gpu_compile.py compares plan
// digests):
//   * bottom-up, the sorted suffix-sum sets T_h = T_{h+1} u (T_{h+1} + a_h):
//     a merge of two sorted arrays (positions by binary search), then the
//     duplicates dropped by a block-wide scan;
//   * top-down, partition h's nodes are residuals r; the children of r are the
//     canonical representatives (reading A12) of r and r - a_h in
//     T_{h+1} (<=: max t <= r; >=: min t >= r; ==: r itself) or bottom; on the
//     last partition top / bottom.  New nodes of P_{h+1} are numbered in order
//     of first appearance in (lo of node 0, hi of node 0, lo of node 1, ...):
//     each appearance atomically lowers a per-representative "first position",
//     and a block-wide scan over the first positions numbers them.
#include <cuda_runtime.h>
#include <cub/block/block_scan.cuh>

#include <climits>
#include <vector>

#include "internal.h"

namespace fdog {
namespace {

constexpr int kCB = 256;                   // threads per CTA
constexpr int64_t kLevelCap = int64_t(1) << 22;  // largest suffix-sum set per level (as compile_B)

struct CompileArgs {
  int32_t n;               // shapes
  const int32_t *k;        // per shape: |I_j|
  const int64_t *coef_off; // per shape: first coefficient
  const int32_t *coef;
  const int8_t *rel;
  const int64_t *rhs;
  const int64_t *lvl_off;  // per shape: first of its k + 1 level offsets (into t_off)
  const int64_t *t_off;    // per level: offset of T_h in tbuf (capacity between consecutive offsets)
  int64_t *tbuf;           // suffix-sum sets
  int32_t *tsize;          // per level: |T_h| (indexed like t_off)
  const int64_t *work_off; // per shape: scratch of 8 * (largest level capacity) values / ints
  int64_t *wv;             // scratch values (merge buffer / node residuals)
  int32_t *wi;             // scratch ints (flags, first positions, codes)
  const int64_t *out_off;  // per shape: first output node
  int32_t *out_lo, *out_hi;  // child codes: local index, -1 bottom, -2 top
  int32_t *out_w;          // per level: |P_h| (indexed like t_off, first k entries)
  int32_t *status;         // per shape: 0 ok, 2 infeasible, 5 too big
};

using BlockScan = cub::BlockScan<int32_t, kCB>;

// exclusive scan of flags[0, n) -> pos; returns the total
__device__ int32_t block_exclusive_scan(const int32_t *flags, int32_t *pos, int64_t n,
                                        typename BlockScan::TempStorage &tmp) {
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += kCB) {
    const int64_t i = base + threadIdx.x;
    const int32_t v = i < n ? flags[i] : 0;
    int32_t ex, tot;
    BlockScan(tmp).ExclusiveSum(v, ex, tot);
    if (i < n) pos[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  return carry;
}

__device__ __forceinline__ int64_t lower_bound(const int64_t *a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound(const int64_t *a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] <= x) lo = m + 1;
    else hi = m;
  }
  return lo;
}
// index of the canonical representative of residual r in T (or -1: bottom)
__device__ __forceinline__ int64_t rep_index(const int64_t *T, int64_t n, int rel, int64_t r) {
  if (rel < 0) return upper_bound(T, n, r) - 1;
  const int64_t i = lower_bound(T, n, r);
  if (rel > 0) return i < n ? i : -1;
  return (i < n && T[i] == r) ? i : -1;
}

__global__ void __launch_bounds__(kCB) compile_kernel(const CompileArgs a) {
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ int32_t total;
  const int s = blockIdx.x;
  const int tid = threadIdx.x;
  const int32_t k = a.k[s];
  const int32_t *coef = a.coef + a.coef_off[s];
  const int rel = a.rel[s];
  const int64_t b = a.rhs[s];
  const int64_t *toff = a.t_off + a.lvl_off[s];
  int32_t *tsz = a.tsize + a.lvl_off[s];
  int32_t *wsz = a.out_w + a.lvl_off[s];
  int64_t *wv = a.wv + a.work_off[s];
  int32_t *wi = a.wi + a.work_off[s];
  const int64_t mx = (a.work_off[s + 1] - a.work_off[s]) / 8;  // largest level capacity

  // ---- bottom-up: T_k = {0}, T_h = T_{h+1} u (T_{h+1} + a_h)
  if (tid == 0) {
    a.tbuf[toff[k]] = 0;
    tsz[k] = 1;
  }
  __syncthreads();
  for (int h = k - 1; h >= 0; --h) {
    const int64_t *A = a.tbuf + toff[h + 1];
    const int64_t m = tsz[h + 1], d = coef[h];
    // merge A and A + d (A first on ties) into wv[0, 2m)
    for (int64_t i = tid; i < m; i += kCB) {
      wv[i + lower_bound(A, m, A[i] - d)] = A[i];       // #{j : A[j] + d < A[i]}
      wv[i + upper_bound(A, m, A[i] + d)] = A[i] + d;   // #{j : A[j] <= A[i] + d}
    }
    __syncthreads();
    for (int64_t p = tid; p < 2 * m; p += kCB) wi[p] = (p == 0 || wv[p] != wv[p - 1]) ? 1 : 0;
    __syncthreads();
    const int32_t n = block_exclusive_scan(wi, wi + 2 * mx, 2 * m, tmp);  // flags [0, 2mx), positions after
    if (n > toff[h + 1] - toff[h]) {  // (capacities bound every level; never taken)
      if (tid == 0) a.status[s] = 5;
      return;
    }
    int64_t *out = a.tbuf + toff[h];
    for (int64_t p = tid; p < 2 * m; p += kCB)
      if (p == 0 || wv[p] != wv[p - 1]) out[wi[2 * mx + p]] = wv[p];
    if (tid == 0) tsz[h] = n;
    __syncthreads();
  }

  // ---- top-down.  Node residuals of the current partition in wv[0, mx),
  // the next partition's in wv[2 mx, 3 mx); ints: first positions (by
  // representative) in wi[0, mx), representative indices [mx, 3mx), new flags
  // [3mx, 5mx), new ids [5mx, 7mx).
  int64_t *cur = wv, *nxt = wv + 2 * mx;
  {
    const int64_t *T0 = a.tbuf + toff[0];
    const int64_t i = rep_index(T0, tsz[0], rel, b);
    if (i < 0) {
      if (tid == 0) a.status[s] = 2;  // empty feasible set
      return;
    }
    if (tid == 0) cur[0] = T0[i];
  }
  int64_t W = 1, node0 = 0;
  int32_t *first = wi, *flag = wi + mx, *isnew = wi + 3 * mx, *nid = wi + 5 * mx;
  __syncthreads();
  for (int h = 0; h < k; ++h) {
    const int64_t d = coef[h];
    int32_t *lo = a.out_lo + a.out_off[s] + node0, *hi = a.out_hi + a.out_off[s] + node0;
    if (h == k - 1) {
      for (int64_t p = tid; p < 2 * W; p += kCB) {
        const int64_t r = cur[p >> 1] - ((p & 1) ? d : 0);
        const bool ok = rel < 0 ? 0 <= r : rel > 0 ? 0 >= r : r == 0;  // representative in T_k = {0}
        ((p & 1) ? hi : lo)[p >> 1] = ok ? -2 : -1;
      }
      if (tid == 0) wsz[h] = (int32_t)W;
      break;
    }
    const int64_t *Tn = a.tbuf + toff[h + 1];
    const int64_t mn = tsz[h + 1];
    for (int64_t q = tid; q < mn; q += kCB) first[q] = INT_MAX;
    __syncthreads();
    for (int64_t p = tid; p < 2 * W; p += kCB) {
      const int64_t i = rep_index(Tn, mn, rel, cur[p >> 1] - ((p & 1) ? d : 0));
      flag[p] = (int32_t)i;  // (representative index for now)
      if (i >= 0) atomicMin(&first[i], (int32_t)p);
    }
    __syncthreads();
    for (int64_t p = tid; p < 2 * W; p += kCB) isnew[p] = (flag[p] >= 0 && first[flag[p]] == p) ? 1 : 0;
    __syncthreads();
    const int32_t n = block_exclusive_scan(isnew, nid, 2 * W, tmp);
    if (tid == 0) total = n;
    for (int64_t p = tid; p < 2 * W; p += kCB)
      if (isnew[p]) nxt[nid[p]] = Tn[flag[p]];
    __syncthreads();
    for (int64_t p = tid; p < 2 * W; p += kCB) {
      const int32_t code = flag[p] < 0 ? -1 : nid[first[flag[p]]];
      ((p & 1) ? hi : lo)[p >> 1] = code;
    }
    if (tid == 0) wsz[h] = (int32_t)W;
    __syncthreads();
    node0 += W;
    W = total;
    int64_t *t = cur;
    cur = nxt;
    nxt = t;
    __syncthreads();
  }
}

#define GCK(x)                                        \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) {                          \
      set_error("GPU compile: %s", cudaGetErrorString(e_)); \
      for (void *p_ : mem) cudaFree(p_);              \
      return FDOG_ECUDA;                              \
    }                                                 \
  } while (0)

}  // namespace

// Compile every shape (k, coef, rel, rhs set; the rest is filled) on the GPU.
// FDOG_ETOOBIG: some level may exceed kLevelCap (the caller compiles on the host).
fdog_status gpu_compile_shapes(std::vector<Shape> &shapes, int device) {
  const int32_t n = (int32_t)shapes.size();
  if (n == 0) return FDOG_OK;
  std::vector<void *> mem;
  // per-level capacities: |T_h| <= min(2^(k-h), sum_{t>=h} |a_t| + 1); |P_h| <= |T_h|
  std::vector<int32_t> hk(n);
  std::vector<int64_t> hcoef_off(n + 1, 0), hlvl(n + 1, 0), hwork(n + 1, 0), hout(n + 1, 0), htoff, hrhs(n);
  std::vector<int32_t> hcoef;
  std::vector<int8_t> hrel(n);
  int64_t tcap = 0;
  for (int32_t s = 0; s < n; ++s) {
    const Shape &S = shapes[s];
    const int32_t k = (int32_t)S.coef.size();
    hk[s] = k;
    hrel[s] = S.rel;
    hrhs[s] = S.rhs;
    hcoef.insert(hcoef.end(), S.coef.begin(), S.coef.end());
    hcoef_off[s + 1] = (int64_t)hcoef.size();
    std::vector<int64_t> cap(k + 1);
    int64_t sum = 0, mx = 1, nodes = 0;
    for (int32_t h = k; h >= 0; --h) {
      if (h < k) sum += S.coef[h] < 0 ? -(int64_t)S.coef[h] : S.coef[h];
      const int64_t pw = (k - h) < 62 ? (int64_t(1) << (k - h)) : INT64_MAX;
      cap[h] = std::min(pw, sum + 1);
      if (cap[h] > kLevelCap) return FDOG_ETOOBIG;
      mx = std::max(mx, cap[h]);
    }
    hlvl[s + 1] = hlvl[s] + k + 1;
    for (int32_t h = 0; h <= k; ++h) {
      htoff.push_back(tcap);
      tcap += cap[h];
      if (h < k) nodes += cap[h];
    }
    hwork[s + 1] = hwork[s] + 8 * mx;
    hout[s + 1] = hout[s] + nodes;
  }
  int prev = -1;
  cudaGetDevice(&prev);
  GCK(cudaSetDevice(device));
  auto up = [&](const void *src, size_t bytes) -> void * {
    void *d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    mem.push_back(d);
    if (bytes && cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return d;
  };
  auto alloc = [&](size_t bytes) -> void * {
    void *d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    mem.push_back(d);
    cudaMemset(d, 0, std::max<size_t>(bytes, 16));
    return d;
  };
  CompileArgs a{};
  a.n = n;
  a.k = (const int32_t *)up(hk.data(), hk.size() * 4);
  a.coef_off = (const int64_t *)up(hcoef_off.data(), hcoef_off.size() * 8);
  a.coef = (const int32_t *)up(hcoef.data(), hcoef.size() * 4);
  a.rel = (const int8_t *)up(hrel.data(), hrel.size());
  a.rhs = (const int64_t *)up(hrhs.data(), hrhs.size() * 8);
  a.lvl_off = (const int64_t *)up(hlvl.data(), hlvl.size() * 8);
  a.t_off = (const int64_t *)up(htoff.data(), htoff.size() * 8);
  a.tbuf = (int64_t *)alloc((size_t)tcap * 8);
  a.tsize = (int32_t *)alloc(htoff.size() * 4);
  a.work_off = (const int64_t *)up(hwork.data(), hwork.size() * 8);
  a.wv = (int64_t *)alloc((size_t)hwork[n] * 8);
  a.wi = (int32_t *)alloc((size_t)hwork[n] * 4);
  a.out_off = (const int64_t *)up(hout.data(), hout.size() * 8);
  a.out_lo = (int32_t *)alloc((size_t)hout[n] * 4);
  a.out_hi = (int32_t *)alloc((size_t)hout[n] * 4);
  a.out_w = (int32_t *)alloc(htoff.size() * 4);
  a.status = (int32_t *)alloc((size_t)n * 4);
  for (void *p : mem)
    if (!p) GCK(cudaErrorMemoryAllocation);
  if (!a.k || !a.coef || !a.tbuf || !a.wv || !a.wi || !a.out_lo || !a.out_hi || !a.status) GCK(cudaErrorMemoryAllocation);
  compile_kernel<<<n, kCB>>>(a);
  GCK(cudaGetLastError());
  GCK(cudaDeviceSynchronize());
  std::vector<int32_t> st(n), w(htoff.size()), lo(hout[n]), hi(hout[n]);
  GCK(cudaMemcpy(st.data(), a.status, (size_t)n * 4, cudaMemcpyDeviceToHost));
  GCK(cudaMemcpy(w.data(), a.out_w, w.size() * 4, cudaMemcpyDeviceToHost));
  GCK(cudaMemcpy(lo.data(), a.out_lo, lo.size() * 4, cudaMemcpyDeviceToHost));
  GCK(cudaMemcpy(hi.data(), a.out_hi, hi.size() * 4, cudaMemcpyDeviceToHost));
  for (void *p : mem) cudaFree(p);
  if (prev >= 0) cudaSetDevice(prev);
  for (int32_t s = 0; s < n; ++s) {
    if (st[s] == 2) return FDOG_EINFEASIBLE;
    if (st[s] != 0) return FDOG_ETOOBIG;
    Shape &S = shapes[s];
    const int32_t k = hk[s];
    S.k = k;
    S.hop_start.assign(1, 0);
    S.lo.clear();
    S.hi.clear();
    S.max_w = 0;
    int64_t node = hout[s];
    for (int32_t h = 0; h < k; ++h) {
      const int32_t W = w[hlvl[s] + h];
      if (W > kMaxWidth) return FDOG_ETOOBIG;
      for (int32_t q = 0; q < W; ++q, ++node) {
        const int32_t l = lo[node], r = hi[node];
        S.lo.push_back(l == -1 ? (uint16_t)kBot : l == -2 ? (uint16_t)kTop : (uint16_t)l);
        S.hi.push_back(r == -1 ? (uint16_t)kBot : r == -2 ? (uint16_t)kTop : (uint16_t)r);
      }
      S.max_w = std::max(S.max_w, W);
      S.hop_start.push_back(S.hop_start.back() + W);
    }
  }
  return FDOG_OK;
}

}  // namespace fdog
