// kernels.cu -- sm_100a kernels of the deferred min-marginal averaging hot path.
//
//   sweep_kernel<T, MODE, REC, RC> one pass (forward P:627-645 / backward P:647-648)
//                                  over all BDD tiles, TMA-staged; MODE kEnergy =
//                                  sum_j E^j only, kCfr = shp(r, .) only.
//   sweep_stream_kernel<T, MODE, REC> the same pass streamed from global memory
//                                  (store design, narrow tiles; FDOG_SWEEP=stream).
//   avg_kernel<T>                  deferred averaging avg_i = mean_{k in J_i} delta_bar_ik
//                                  (P:641 second term, readings A1/A10).
//   avg_finish_kernel<T>           shared variables after the NCCL exchange.
//   peer_signal_kernel, peer_finish_kernel<T>  the exchange over peer memory instead.
//   add_deferred_kernel<T>         final correction lambda += delta_bar.
//   fused_small_kernel<T, REC>     every iteration of a small problem in one CTA.
//   primal_kernel<T>               Alg. 2 classify / perturb steps.
//
// Thread mapping: one warp per tile of L <= 32 BDDs, one BDD per
// lane.  Each lane walks its BDD's partitions sequentially (the hop recursion
// P:317-342 is sequential); distances live in the lane's private column of
// shared memory ([node][lane] layout: conflict-free, no cross-lane
// communication, no atomics, no barriers inside a pass).  Two designs for the
// distances of the opposite direction:
//   * recompute (RC, default for narrow problems): rebuilt on chip at the start
//     of every pass from the current lambda -- equal to the stored distances of
//     P:315-316 exactly, since lambda has not changed since they were computed
//     -- so HBM traffic is per-slot data only;
//   * store: kept in HBM per node and converted in place by each pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "internal.h"

namespace fdog {

template <typename T>
__device__ __forceinline__ T t_inf();
template <>
__device__ __forceinline__ float t_inf<float>() { return __int_as_float(0x7f800000); }
template <>
__device__ __forceinline__ double t_inf<double>() { return __longlong_as_double(0x7ff0000000000000ll); }

// IEEE round-to-nearest products (no FMA contraction in the dual update, so the
// arithmetic matches the oracle's (lambda - omega*d) + avg order).
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// m1 - m0 with an infinite side replaced by +-clamp (reading A5): the IEEE
// difference is +inf exactly when m1 is infinite, -inf when m0 is, finite
// otherwise (both infinite -- NaN -- only on padding lanes, whose results are
// discarded), so one test of |m1 - m0| and a copysign give the reading.
__device__ __forceinline__ float copysign_t(float c, float s) { return copysignf(c, s); }
__device__ __forceinline__ double copysign_t(double c, double s) { return copysign(c, s); }
// omega and the clamp of a launch in the kernel's precision (T(double) rounds
// once; the fp32 copies are the same values, read straight from the
// parameter bank instead of converted per use)
template <typename T, class A>
__device__ __forceinline__ T arg_omega(const A &a) {
  if constexpr (sizeof(T) == 4) return a.omega_f;
  else return a.omega;
}
template <typename T, class A>
__device__ __forceinline__ T arg_clamp(const A &a) {
  if constexpr (sizeof(T) == 4) return a.clamp_f;
  else return a.clamp;
}

template <typename T>
__device__ __forceinline__ T mm_difference(T m1, T m0, T clamp) {
  const T d = sub_rn(m1, m0);
  return fabs(d) < t_inf<T>() ? d : copysign_t(clamp, d);
}

// ---- Programmatic dependent launch: a kernel launched with the PDL attribute
// may start while its predecessor drains; it waits here before reading the
// predecessor's outputs (or touching the tile counter it resets).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// (An early griddepcontrol.launch_dependents at the end of each sweep warp's
// tile loop (SweepArgs::pdl_early) only pays with few tiles per warp, where the
// averaging grid's CTAs prefetch their slot indices during the sweep's tail;
// with many (MRF) the dependent CTAs get in the sweep's way: 15 % slower.)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Bound of the last pass (A7): the per-tile partials summed in a fixed order
// (deterministic for any tile-to-warp assignment); one CTA, launched on demand
// by fdog_lower_bound.
__global__ void __launch_bounds__(1024) lb_reduce_kernel(const double *__restrict__ lb_part, int n, double *out) {
  __shared__ double red[32];
  pdl_wait();
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int q0 = threadIdx.x * chunk, q1 = min(n, q0 + chunk);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int q = q0;
  for (; q + 3 < q1; q += 4) {
    s0 += lb_part[q];
    s1 += lb_part[q + 1];
    s2 += lb_part[q + 2];
    s3 += lb_part[q + 3];
  }
  for (; q < q1; ++q) s0 += lb_part[q];
  double s = (s0 + s1) + (s2 + s3);
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (warp == 0) {
    double v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) *out = v;
  }
}

// ---- PTX helpers: mbarrier + TMA bulk copies (sm_90+/sm_100a) and cp.async
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// TMA 1D bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// TMA 1D bulk copy shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src) {
  if (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One lane's BDD, one pass (store design).  Pointers are
// per-lane (column offset applied) with a stride of L elements per
// partition/node; they point to shared memory (staged tiles) or global memory
// (direct tiles).  Topology words hold the ABSOLUTE child index within the
// tile (s^0 low 16 bits, s^1 high 16 bits); top = nodes and bottom = nodes + 1
// index two constant sentinel slots of D (0 and +inf), so a child lookup is a
// single load.
//   D   : per node, on entry shp(v, T) (kForward) or shp(r, v) (kBackward);
//         on exit the other one (the pass converts it in place, hop by hop).
//         kEnergy writes shp(v, T), kCfr writes shp(r, v) (no update).
//   lam : lambda_h at lam[h*L], updated in place
//   va  : per partition: the deferred average avg_i of its variable in (written
//         by avg_kernel), delta_h = omega (m1 - m0) out (kForward / kBackward)
//   R   : 3 * (rw + 1) scratch entries (forward relaxation buffers)
// Returns the lane's bound contribution E^j + sum_h min(delta_h, 0) (A7), or E^j.
template <typename T, int MODE, bool REC>
__device__ __forceinline__ double process_bdd(const int K, const int nodes, const int32_t *ho, const uint32_t *tp,
                                              const int ts, const int L, T *lam, T *va, T *D, T *R, const int rw,
                                              const bool valid, const T omega, const T clamp, T *m0g, T *m1g,
                                              T *l0 = nullptr, const T *v0 = nullptr) {
  // l0 != null: lifted mode -- 0-arcs cost lambda^{j,0} = l0[h L]
  // (else 0); v0: the 0-side averages; lam / va: lambda^{j,1} and its average
  const T inf = t_inf<T>();
  const bool lifted = l0 != nullptr;
  double acc = 0.0;
  auto emit = [&](int h, T lam_new, T delta, T m0, T m1) {
    if (!valid) {
      va[h * L] = T(0);
      return;
    }
    lam[h * L] = lam_new;
    va[h * L] = delta;
    if (REC) {
      m0g[h * L] = m0;
      m1g[h * L] = m1;
    }
  };
  // dual update of partition h (lifted: reading A8, both sides);
  // returns (lambda^0, lambda^1) of the hop after it
  auto update = [&](int h, T m0r, T m1r, T &o0, T &o1) {
    const T l = lam[h * L];
    const T z = lifted ? l0[h * L] : T(0);
    const T m0 = lifted ? z + m0r : m0r;
    const T m1 = l + m1r;  // Eq. (min-marginal-via-shortest-path) P:312
    const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
    if (!lifted) {
      o1 = add_rn(sub_rn(l, delta), va[h * L]);
      o0 = T(0);
      emit(h, o1, delta, m0, m1);
      if (valid) acc += (double)fmin(delta, T(0));
      return;
    }
    o1 = add_rn(sub_rn(l, fmax(delta, T(0))), va[h * L]);
    o0 = add_rn(sub_rn(z, fmax(-delta, T(0))), v0[h * L]);
    emit(h, o1, delta, m0, m1);
    if (valid) l0[h * L] = o0;
  };
  if constexpr (MODE == kEnergy) {
    // shp(v, T) for all nodes under the current lambda
#pragma unroll 1
    for (int h = K - 1; h >= 0; --h) {
      const T l = lam[h * L];
      const T z = lifted ? l0[h * L] : T(0);
      const int n1 = ho[h + 1];
#pragma unroll 1
      for (int n = ho[h]; n < n1; ++n) {
        const uint32_t e = tp[n * ts];
        D[n * L] = fmin(lifted ? z + D[(e & 0xFFFFu) * L] : D[(e & 0xFFFFu) * L], l + D[(e >> 16) * L]);
      }
    }
    return valid ? (double)D[0] : 0.0;  // E^j = shp(r, T)
  }
  if constexpr (MODE == kCfr) {
    // shp(r, v) for all nodes under the current lambda, relaxed
    // through the R buffers (no writes into the sentinels)
    T *cur = R, *nlo = R + (rw + 1) * L, *nhi = R + 2 * (rw + 1) * L;
    cur[0] = T(0);
#pragma unroll 1
    for (int h = 0; h < K; ++h) {
      const int n0 = ho[h], n1 = ho[h + 1];
      const int Wn = h == K - 1 ? 0 : ho[h + 2] - n1;
#pragma unroll 1
      for (int w = 0; w < Wn; ++w) {
        nlo[w * L] = inf;
        nhi[w * L] = inf;
      }
      T e_min = inf;
      const T l = lam[h * L];
      const T z = lifted ? l0[h * L] : T(0);
#pragma unroll 1
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = tp[n * ts];
        const int lo = (int)(e & 0xFFFFu), hi = (int)(e >> 16);
        const T cf = cur[(n - n0) * L];
        D[n * L] = cf;
        const int rl = min(lo - n1, rw), rh = min(hi - n1, rw);
        nlo[rl * L] = fmin(nlo[rl * L], cf);
        nhi[rh * L] = fmin(nhi[rh * L], cf);
        if (h == K - 1) e_min = fmin(e_min, fmin((lifted ? cf + z : cf) + D[lo * L], cf + l + D[hi * L]));
      }
#pragma unroll 1
      for (int w = 0; w < Wn; ++w) cur[w * L] = fmin(lifted ? nlo[w * L] + z : nlo[w * L], nhi[w * L] + l);
      if (h == K - 1 && valid) acc = (double)e_min;
    }
    return acc;
  }
  if constexpr (MODE == kForward) {
    // forward pass with updates (Alg. forward_pass_mm): D holds
    // shp(v, T) from the previous pass, valid for P_{h+1} at hop h;
    // R holds shp(r, .) of P_h (cur) and the 0-/1-arc relaxations into P_{h+1}
    // (nlo, nhi), each rw + 1 entries (the last is a sink for arcs to bottom).
    T *cur = R, *nlo = R + (rw + 1) * L, *nhi = R + 2 * (rw + 1) * L;
    cur[0] = T(0);  // shp(r, r)
#pragma unroll 1
    for (int h = 0; h < K; ++h) {
      const int n0 = ho[h], n1 = ho[h + 1];
      const bool last = h == K - 1;
      const int Wn = last ? 0 : ho[h + 2] - n1;
#pragma unroll 1
      for (int w = 0; w < Wn; ++w) {
        nlo[w * L] = inf;
        nhi[w * L] = inf;
      }
      T m0 = inf, m1r = inf;  // m1r = min(shp(r,v) + shp(s1 v, T)); lambda added below
#pragma unroll 1
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = tp[n * ts];
        const int lo = (int)(e & 0xFFFFu), hi = (int)(e >> 16);
        const T cf = cur[(n - n0) * L];
        D[n * L] = cf;  // shp(v, T) of P_h is no longer needed: keep shp(r, v)
        m0 = fmin(m0, cf + D[lo * L]);
        m1r = fmin(m1r, cf + D[hi * L]);
        const int rl = min(lo - n1, rw), rh = min(hi - n1, rw);
        nlo[rl * L] = fmin(nlo[rl * L], cf);
        nhi[rh * L] = fmin(nhi[rh * L], cf);
      }
      T z_new, lam_new;
      update(h, m0, m1r, z_new, lam_new);
      if (!last) {
        // shp(r, v), v in P_{h+1}: 1-arcs priced with the updated lambda_h (A4)
#pragma unroll 1
        for (int w = 0; w < Wn; ++w)
          cur[w * L] = fmin(lifted ? nlo[w * L] + z_new : nlo[w * L], nhi[w * L] + lam_new);
      } else if (valid) {
        acc += (double)fmin(lifted ? z_new + m0 : m0, lam_new + m1r);  // E^j at the updated lambda
      }
    }
    return acc;
  }
  if constexpr (MODE == kBackward) {
    // MODE == kBackward (Alg. backward_pass_mm): D holds shp(r, v)
    // from the forward pass, valid for P_h at hop h; shp(v, T) of P_{h+1} was
    // written into D by the previous hop of this pass.
#pragma unroll 1
    for (int h = K - 1; h >= 0; --h) {
      const int n0 = ho[h], n1 = ho[h + 1];
      T m0 = inf, m1r = inf;
#pragma unroll 1
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = tp[n * ts];
        const T cf = D[n * L];
        m0 = fmin(m0, cf + D[(e & 0xFFFFu) * L]);
        m1r = fmin(m1r, cf + D[(e >> 16) * L]);
      }
      T z_new, lam_new;
      update(h, m0, m1r, z_new, lam_new);
      // shp(v, T), v in P_h, with the updated lambda_h
#pragma unroll 1
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = tp[n * ts];
        D[n * L] = fmin(lifted ? z_new + D[(e & 0xFFFFu) * L] : D[(e & 0xFFFFu) * L], lam_new + D[(e >> 16) * L]);
      }
    }
    if (valid) acc += (double)D[0];  // E^j = shp(r, T)
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Wide BDDs (a partition wider than kCoopWidth nodes, e.g. knapsack rows):
// node-parallel, the way P:345-347 parallelises a hop over v in P_i.  One warp
// per BDD; at every hop the 32 lanes split the partition's nodes, the min-
// marginals m^0, m^1 are warp-shuffle min reductions (exact: min is
// order-independent), every lane applies the same dual update, and the
// forward relaxation into P_{h+1} is a shared-/global-memory atomic min
// on an order-preserving integer image of the distances (exact as well; for
// either order of the arcs, min(c + lambda) = min(c) + lambda under monotone
// rounding, so every value equals the lane-serial process_bdd bit for bit).
// Topology: two 32-bit absolute child indices per node (uint2), top = nodes,
// bottom = nodes + 1 (the sentinels of D) -- no 16-bit limit on BDD size.
// Single BDD per tile (L = 1): lambda / va / D are contiguous per hop / node.
template <typename T>
struct OrdOf;
template <>
struct OrdOf<float> {
  using U = uint32_t;
};
template <>
struct OrdOf<double> {
  using U = unsigned long long;
};
// order-preserving map T -> unsigned (a < b <=> ord(a) < ord(b); -0 < +0)
__device__ __forceinline__ uint32_t t_ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float t_unord(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ unsigned long long t_ord(double f) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(f);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double t_unord(unsigned long long u) {
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// buf: two relaxation buffers of `bw` entries (shared or global memory).
// Returns the BDD's bound contribution on lane 0 (0 on the other lanes).
// Every node loop runs in blocks of CB nodes per lane (lane l: nodes n0 + l +
// 32 q), loads first and stores after, so a lane has 2 CB independent distance
// gathers in flight (the BDD is in global memory / L2: latency-bound otherwise).
template <typename T, int MODE, bool REC>
__device__ __noinline__ double process_bdd_coop(const int K, const int nodes, const int32_t *ho, const uint2 *tp,
                                                T *lam, T *va, T *D, typename OrdOf<T>::U *buf, const int bw,
                                                const int lane, const T omega, const T clamp, T *m0g, T *m1g,
                                                T *l0, const T *v0) {
  // l0 != null: lifted mode, 0-arcs cost lambda^{j,0}_h = l0[h]
  using U = typename OrdOf<T>::U;
  constexpr int CB = 4;
  const T inf = t_inf<T>();
  const U uinf = t_ord(inf);
  double acc = 0.0;
  const bool lifted = l0 != nullptr;
  // dual update of partition h from the reduced min-marginals (
  // lifted: reading A8); z = lambda^{j,0}_h after it (0 unless lifted)
  auto update = [&](int h, T m0r, T m1r, T &z) -> T {
    const T l = lam[h];
    const T z0 = lifted ? l0[h] : T(0);
    const T m0 = lifted ? z0 + m0r : m0r;
    const T m1 = l + m1r;
    const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
    const T lam_new = lifted ? add_rn(sub_rn(l, fmax(delta, T(0))), va[h]) : add_rn(sub_rn(l, delta), va[h]);
    z = lifted ? add_rn(sub_rn(z0, fmax(-delta, T(0))), v0[h]) : T(0);
    __syncwarp();  // every lane has read lam[h] / va[h] / l0[h]
    if (lane == 0) {
      lam[h] = lam_new;
      va[h] = delta;
      if (lifted) l0[h] = z;
      if (REC) {
        m0g[h] = m0;
        m1g[h] = m1;
      }
      if (!lifted) acc += (double)fmin(delta, T(0));
    }
    return lam_new;
  };
  if (MODE == kEnergy || MODE == kBackward) {
    // backward: D holds shp(r, v) (forward pass); shp(v, T) of P_{h+1} is
    // written by the previous hop.  kEnergy: shp(v, T) only.
#pragma unroll 1
    for (int h = K - 1; h >= 0; --h) {
      const int n0 = ho[h], n1 = ho[h + 1];
      T l = lam[h];
      T z = lifted ? l0[h] : T(0);
      if (MODE == kBackward) {
        T m0 = inf, m1r = inf;
#pragma unroll 1
        for (int nb = n0 + lane; nb < n1; nb += 32 * CB) {
          uint2 e[CB];
          T cf[CB], x0[CB], x1[CB];
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            const bool ok = nb + 32 * q < n1;
            e[q] = ok ? tp[nb + 32 * q] : make_uint2(nodes + 1, nodes + 1);
            cf[q] = ok ? D[nb + 32 * q] : inf;
          }
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            x0[q] = D[e[q].x];
            x1[q] = D[e[q].y];
          }
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            m0 = fmin(m0, cf[q] + x0[q]);
            m1r = fmin(m1r, cf[q] + x1[q]);
          }
        }
        l = update(h, warp_min(m0), warp_min(m1r), z);
      }
#pragma unroll 1
      for (int nb = n0 + lane; nb < n1; nb += 32 * CB) {
        uint2 e[CB];
        T v[CB];
#pragma unroll
        for (int q = 0; q < CB; ++q) e[q] = nb + 32 * q < n1 ? tp[nb + 32 * q] : make_uint2(nodes + 1, nodes + 1);
#pragma unroll
        for (int q = 0; q < CB; ++q) v[q] = fmin(lifted ? z + D[e[q].x] : D[e[q].x], l + D[e[q].y]);
#pragma unroll
        for (int q = 0; q < CB; ++q)
          if (nb + 32 * q < n1) D[nb + 32 * q] = v[q];
      }
      __syncwarp();  // the next hop reads these as children
    }
    if (lane == 0) acc += (double)D[0];  // E^j = shp(r, T)
    return acc;
  }
  // forward / kCfr: shp(r, .) of P_h in buffer `cur` (ord images), relaxed into
  // `nxt` for P_{h+1}; D of P_h is overwritten with shp(r, v) (store design).
  U *cur = buf, *nxt = buf + bw;
  if (lane == 0) cur[0] = t_ord(T(0));  // shp(r, r)
  __syncwarp();
#pragma unroll 1
  for (int h = 0; h < K; ++h) {
    const int n0 = ho[h], n1 = ho[h + 1];
    const bool last = h == K - 1;
    const int Wn = last ? 0 : ho[h + 2] - n1;
    for (int w = lane; w < Wn; w += 32) nxt[w] = uinf;
    T m0 = inf, m1r = inf;
    if (MODE == kForward || last) {  // min-marginals against shp(., T) of P_{h+1}; kCfr: E^j only
#pragma unroll 1
      for (int nb = n0 + lane; nb < n1; nb += 32 * CB) {
        uint2 e[CB];
        T cf[CB], x0[CB], x1[CB];
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          const bool ok = nb + 32 * q < n1;
          e[q] = ok ? tp[nb + 32 * q] : make_uint2(nodes + 1, nodes + 1);
          cf[q] = ok ? t_unord(cur[nb + 32 * q - n0]) : inf;
        }
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          x0[q] = D[e[q].x];
          x1[q] = D[e[q].y];
        }
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          m0 = fmin(m0, cf[q] + x0[q]);
          m1r = fmin(m1r, cf[q] + x1[q]);
        }
      }
      m0 = warp_min(m0);
      m1r = warp_min(m1r);
    }
    T l = lam[h];
    T z = lifted ? l0[h] : T(0);
    if (MODE == kForward) l = update(h, m0, m1r, z);
    __syncwarp();  // nxt initialised; the reads of D of P_{h+1} are done
    // D of P_h <- shp(r, v); relax into P_{h+1} (A4: 1-arcs priced with the updated lambda_h)
#pragma unroll 1
    for (int nb = n0 + lane; nb < n1; nb += 32 * CB) {
      uint2 e[CB];
      T cf[CB];
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const bool ok = nb + 32 * q < n1;
        e[q] = ok ? tp[nb + 32 * q] : make_uint2(nodes + 1, nodes + 1);
        cf[q] = ok ? t_unord(cur[nb + 32 * q - n0]) : inf;
      }
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        if (nb + 32 * q >= n1) continue;
        D[nb + 32 * q] = cf[q];
        if (!last) {
          if ((int)e[q].x < n1 + Wn) atomicMin(&nxt[e[q].x - n1], t_ord(lifted ? cf[q] + z : cf[q]));  // 0-arc
          if ((int)e[q].y < n1 + Wn) atomicMin(&nxt[e[q].y - n1], t_ord(cf[q] + l));  // 1-arc
        }
      }
    }
    __syncwarp();
    if (!last) {
      U *t = cur;
      cur = nxt;
      nxt = t;
    } else if (lane == 0) {
      acc += (double)fmin(lifted ? z + m0 : m0, l + m1r);  // E^j = shp(r, T) (at the updated lambda)
    }
  }
  return acc;
}

// Narrow tiles (every partition has <= 2 nodes -- all one-hot, at-most-one and
// marginalisation rows of the BASELINE workloads).  Same arithmetic and the
// same D / va conventions as process_bdd, with the per-partition values of the
// sweep direction in registers and no loops over nodes.
template <typename T, int MODE, bool REC, int LC>
__device__ __forceinline__ double process_bdd_w2(const int K, const int32_t *ho, const uint32_t *tp, const int ts_rt,
                                                 const int L_rt, T *lam, T *va, T *D, const bool valid, const T omega,
                                                 const T clamp, T *m0g, T *m1g) {
  // LC = 32: full shared-topology tile, compile-time strides (shifts and
  // immediate shared-memory offsets); LC = 0: runtime lane count / stride
  const int L = LC ? LC : L_rt;
  const int ts = LC ? 1 : ts_rt;
  const T inf = t_inf<T>();
  double acc = 0.0;
  auto finish = [&](int h, T l, T m0, T m1r) -> T {
    const T m1 = l + m1r;
    const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
    const T lam_new = add_rn(sub_rn(l, delta), va[h * L]);
    if (valid) {
      lam[h * L] = lam_new;
      va[h * L] = delta;
      if (REC) {
        m0g[h * L] = m0;
        m1g[h * L] = m1;
      }
      acc += (double)fmin(delta, T(0));
    } else {
      va[h * L] = T(0);
    }
    return lam_new;
  };
  if constexpr (MODE == kForward) {
    T c0 = T(0), c1 = inf;  // shp(r, .) of the (up to) two nodes of P_h
    int n0 = ho[0];
#pragma unroll 1
    for (int h = 0; h < K - 1; ++h) {
      const int n1 = ho[h + 1];
      const uint32_t e0 = tp[n0 * ts];
      const int lo0 = (int)(e0 & 0xFFFFu), hi0 = (int)(e0 >> 16);
      D[n0 * L] = c0;  // shp(v, T) of P_h is no longer needed: keep shp(r, v)
      T m0 = c0 + D[lo0 * L], m1r = c0 + D[hi0 * L];
      // relaxation into P_{h+1} (nodes n1, n1 + 1); other targets are bottom
      T nl0 = lo0 == n1 ? c0 : inf, nl1 = lo0 == n1 + 1 ? c0 : inf;
      T nh0 = hi0 == n1 ? c0 : inf, nh1 = hi0 == n1 + 1 ? c0 : inf;
      if (n1 - n0 > 1) {
        const uint32_t e1 = tp[(n0 + 1) * ts];
        const int lo1 = (int)(e1 & 0xFFFFu), hi1 = (int)(e1 >> 16);
        D[(n0 + 1) * L] = c1;
        m0 = fmin(m0, c1 + D[lo1 * L]);
        m1r = fmin(m1r, c1 + D[hi1 * L]);
        if (lo1 == n1) nl0 = fmin(nl0, c1);
        if (lo1 == n1 + 1) nl1 = fmin(nl1, c1);
        if (hi1 == n1) nh0 = fmin(nh0, c1);
        if (hi1 == n1 + 1) nh1 = fmin(nh1, c1);
      }
      const T lam_new = finish(h, lam[h * L], m0, m1r);
      c0 = fmin(nl0, nh0 + lam_new);  // A4: 1-arcs priced with the updated lambda_h
      c1 = fmin(nl1, nh1 + lam_new);
      n0 = n1;
    }
    {  // last partition: successors are terminals (sentinels of D)
      const int h = K - 1;
      const uint32_t e0 = tp[n0 * ts];
      D[n0 * L] = c0;
      T m0 = c0 + D[(e0 & 0xFFFFu) * L], m1r = c0 + D[(e0 >> 16) * L];
      if (ho[K] - n0 > 1) {
        const uint32_t e1 = tp[(n0 + 1) * ts];
        D[(n0 + 1) * L] = c1;
        m0 = fmin(m0, c1 + D[(e1 & 0xFFFFu) * L]);
        m1r = fmin(m1r, c1 + D[(e1 >> 16) * L]);
      }
      const T lam_new = finish(h, lam[h * L], m0, m1r);
      if (valid) acc += (double)fmin(m0, lam_new + m1r);  // E^j at the updated lambda
    }
    return acc;
  }
  if constexpr (MODE == kBackward) {
    // kBackward
#pragma unroll 1
    for (int h = K - 1; h >= 0; --h) {
      const int n0 = ho[h], n1 = ho[h + 1];
      const uint32_t e0 = tp[n0 * ts];
      const T f0 = D[n0 * L];
      const T a0 = D[(e0 & 0xFFFFu) * L], b0 = D[(e0 >> 16) * L];
      T m0 = f0 + a0, m1r = f0 + b0;
      T a1 = inf, b1 = inf;
      const bool two = n1 - n0 > 1;
      if (two) {
        const uint32_t e1 = tp[(n0 + 1) * ts];
        const T f1 = D[(n0 + 1) * L];
        a1 = D[(e1 & 0xFFFFu) * L];
        b1 = D[(e1 >> 16) * L];
        m0 = fmin(m0, f1 + a1);
        m1r = fmin(m1r, f1 + b1);
      }
      const T lam_new = finish(h, lam[h * L], m0, m1r);
      D[n0 * L] = fmin(a0, lam_new + b0);  // shp(v, T) with the updated lambda_h
      if (two) D[(n0 + 1) * L] = fmin(a1, lam_new + b1);
    }
    if (valid) acc += (double)D[0];  // E^j = shp(r, T)
  }
  return acc;
}

// successor value: top, bottom, or a node of the next partition (held in
// registers).  The sentinels are tested first: on the last partition
// n1 == nodes == top.
template <typename T>
__device__ __forceinline__ T succ(int code, int n1, int top, T v0, T v1) {
  const T inf = t_inf<T>();
  return code == top ? T(0) : code > top ? inf : code == n1 ? v0 : code == n1 + 1 ? v1 : inf;
}

// Recompute design, narrow tiles (every partition <= 2 nodes).
// The distances of the opposite direction are not kept in HBM: phase 1
// recomputes them on chip from the current lambda -- shp(v, T) for a forward
// pass, shp(r, v) for a backward pass -- into the
// lane's column of the per-warp scratch D (two sentinel slots: D[top] = 0,
// D[bottom] = +inf).  Because lambda has not changed since the previous pass
// computed them, they are bit-identical to the stored distances of P:315-316.
// Phase 2 is the pass with updates; its own-direction distances
// are carried in registers.  HBM traffic per pass: lambda read + write, the
// average read, delta write -- nothing per node.
template <typename T, int MODE, bool REC, int LC>
__device__ __forceinline__ double process_rc_w2(const int K, const int top, const int32_t *ho, const uint32_t *tp,
                                                const int ts_rt, const int L_rt, T *lam, T *va, T *D,
                                                const bool valid, const T omega, const T clamp, T *m0g, T *m1g) {
  const int L = LC ? LC : L_rt;
  const int ts = LC ? 1 : ts_rt;
  const T inf = t_inf<T>();
  double acc = 0.0;
  auto finish = [&](int h, T l, T m0, T m1r) -> T {
    const T m1 = l + m1r;
    const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
    const T lam_new = add_rn(sub_rn(l, delta), va[h * L]);
    if (valid) {
      lam[h * L] = lam_new;
      va[h * L] = delta;
      if (REC) {
        m0g[h * L] = m0;
        m1g[h * L] = m1;
      }
      acc += (double)fmin(delta, T(0));
    } else {
      va[h * L] = T(0);
    }
    return lam_new;
  };
  if constexpr (MODE == kForward) {
    {  // phase 1: shp(v, T) for every node under the current lambda
      T x0 = inf, x1 = inf;  // shp(., T) of P_{h+1}
#pragma unroll 1
      for (int h = K - 1; h >= 0; --h) {
        const int n0 = ho[h], n1 = ho[h + 1];
        const uint32_t e0 = tp[n0 * ts];
        const T l = lam[h * L];
        const T ct0 = fmin(succ((int)(e0 & 0xFFFFu), n1, top, x0, x1), l + succ((int)(e0 >> 16), n1, top, x0, x1));
        T ct1 = inf;
        if (n1 - n0 > 1) {
          const uint32_t e1 = tp[(n0 + 1) * ts];
          ct1 = fmin(succ((int)(e1 & 0xFFFFu), n1, top, x0, x1), l + succ((int)(e1 >> 16), n1, top, x0, x1));
          D[(n0 + 1) * L] = ct1;
        }
        D[n0 * L] = ct0;
        x0 = ct0;
        x1 = ct1;
      }
    }
    // phase 2: forward pass with updates; shp(r, .) of P_h in registers
    T c0 = T(0), c1 = inf;
    int n0 = ho[0];
#pragma unroll 1
    for (int h = 0; h < K; ++h) {
      const int n1 = ho[h + 1];
      const uint32_t e0 = tp[n0 * ts];
      const int lo0 = (int)(e0 & 0xFFFFu), hi0 = (int)(e0 >> 16);
      T m0 = c0 + D[lo0 * L], m1r = c0 + D[hi0 * L];
      T nl0 = lo0 == n1 ? c0 : inf, nl1 = lo0 == n1 + 1 ? c0 : inf;
      T nh0 = hi0 == n1 ? c0 : inf, nh1 = hi0 == n1 + 1 ? c0 : inf;
      if (n1 - n0 > 1) {
        const uint32_t e1 = tp[(n0 + 1) * ts];
        const int lo1 = (int)(e1 & 0xFFFFu), hi1 = (int)(e1 >> 16);
        m0 = fmin(m0, c1 + D[lo1 * L]);
        m1r = fmin(m1r, c1 + D[hi1 * L]);
        if (lo1 == n1) nl0 = fmin(nl0, c1);
        if (lo1 == n1 + 1) nl1 = fmin(nl1, c1);
        if (hi1 == n1) nh0 = fmin(nh0, c1);
        if (hi1 == n1 + 1) nh1 = fmin(nh1, c1);
      }
      const T lam_new = finish(h, lam[h * L], m0, m1r);
      if (h == K - 1) {
        if (valid) acc += (double)fmin(m0, lam_new + m1r);  // E^j at the updated lambda
      } else {
        c0 = fmin(nl0, nh0 + lam_new);  // A4: 1-arcs priced with the updated lambda_h
        c1 = fmin(nl1, nh1 + lam_new);
      }
      n0 = n1;
    }
    return acc;
  }
  // kBackward.  Phase 1: shp(r, v) for every node under the current lambda
  // (P:319-324, 1-arcs out of P_h priced with lambda_h, reading A4).
  {
    T c0 = T(0), c1 = inf;
    int n0 = ho[0];
#pragma unroll 1
    for (int h = 0; h < K - 1; ++h) {
      const int n1 = ho[h + 1];
      const uint32_t e0 = tp[n0 * ts];
      const int lo0 = (int)(e0 & 0xFFFFu), hi0 = (int)(e0 >> 16);
      D[n0 * L] = c0;
      T nl0 = lo0 == n1 ? c0 : inf, nl1 = lo0 == n1 + 1 ? c0 : inf;
      T nh0 = hi0 == n1 ? c0 : inf, nh1 = hi0 == n1 + 1 ? c0 : inf;
      if (n1 - n0 > 1) {
        const uint32_t e1 = tp[(n0 + 1) * ts];
        const int lo1 = (int)(e1 & 0xFFFFu), hi1 = (int)(e1 >> 16);
        D[(n0 + 1) * L] = c1;
        if (lo1 == n1) nl0 = fmin(nl0, c1);
        if (lo1 == n1 + 1) nl1 = fmin(nl1, c1);
        if (hi1 == n1) nh0 = fmin(nh0, c1);
        if (hi1 == n1 + 1) nh1 = fmin(nh1, c1);
      }
      const T l = lam[h * L];
      c0 = fmin(nl0, nh0 + l);
      c1 = fmin(nl1, nh1 + l);
      n0 = n1;
    }
    D[n0 * L] = c0;
    if (ho[K] - n0 > 1) D[(n0 + 1) * L] = c1;
  }
  // phase 2: backward pass with updates; shp(., T) of P_{h+1} in registers
  T ct0 = inf, ct1 = inf;
#pragma unroll 1
  for (int h = K - 1; h >= 0; --h) {
    const int n0 = ho[h], n1 = ho[h + 1];
    const uint32_t e0 = tp[n0 * ts];
    const bool two = n1 - n0 > 1;
    const T f0 = D[n0 * L];
    const T a0 = succ((int)(e0 & 0xFFFFu), n1, top, ct0, ct1), b0 = succ((int)(e0 >> 16), n1, top, ct0, ct1);
    T m0 = f0 + a0, m1r = f0 + b0;
    T a1 = inf, b1 = inf;
    if (two) {
      const uint32_t e1 = tp[(n0 + 1) * ts];
      const T f1 = D[(n0 + 1) * L];
      a1 = succ((int)(e1 & 0xFFFFu), n1, top, ct0, ct1);
      b1 = succ((int)(e1 >> 16), n1, top, ct0, ct1);
      m0 = fmin(m0, f1 + a1);
      m1r = fmin(m1r, f1 + b1);
    }
    const T lam_new = finish(h, lam[h * L], m0, m1r);
    ct0 = fmin(a0, lam_new + b0);  // shp(v, T) with the updated lambda_h
    ct1 = two ? fmin(a1, lam_new + b1) : inf;
  }
  if (valid) acc += (double)ct0;  // E^j = shp(r, T)
  return acc;
}

// ---------------------------------------------------------------------------
// Arc-mask form of a narrow hop (tiles with kind bit 2; HopRec in internal.h).
// With the 0/+inf arc masks A of partition P_h, the hop is branch-free
// min-plus arithmetic over the (up to) two nodes i of P_h and the two targets
// j of P_{h+1} (or top on the last partition):
//   a_i = min_j (A0[i][j] + x_j),  b_i = min_j (A1[i][j] + x_j)
//     (x = shp(., T) of P_{h+1}: the distance of node i's 0-/1-successor),
//   m^0 = min_i (c_i + a_i),  m^1 = lambda_h + min_i (c_i + b_i),
//   shp(v_i, T) = min(a_i, lambda_h + b_i),
//   shp(r, v_j) = min_i min(c_i + A0[i][j], lambda_h + (c_i + A1[i][j])) (A4),
// with c = shp(r, .) of P_h.  Adding a 0 mask is exact and +inf masks
// absorb, so every value is bit-identical to the topology-walking form
// (process_bdd_w2).  The loops prefetch the next partition's record, lambda,
// average and distances while the current one is computed.
template <typename T>
struct __align__(16) HopRec {
  T A[8];
  int32_t n0, n1, w2, type;
};
static_assert(sizeof(HopRec<float>) == 48 && sizeof(HopRec<double>) == 80, "HopRec layout (internal.h rec_bytes)");

// The record's 16-byte tail (n0, n1, w2, type), one vector load.
template <typename T>
__device__ __forceinline__ int4 hop_tail(const HopRec<T> *r) {
  return *reinterpret_cast<const int4 *>(&r->n0);
}

template <typename T>
__device__ __forceinline__ void arc_mins(const HopRec<T> &r, T x0, T x1, T &a0, T &a1, T &b0, T &b1) {
  a0 = fmin(r.A[0] + x0, r.A[1] + x1);
  a1 = fmin(r.A[2] + x0, r.A[3] + x1);
  b0 = fmin(r.A[4] + x0, r.A[5] + x1);
  b1 = fmin(r.A[6] + x0, r.A[7] + x1);
}

// Hop types (plan.cpp append_recs): the masks of type 1..3 are fixed, so the
// general expressions fold to the ones below (exactly: a 0 mask adds nothing,
// an +inf mask drops the term).  The type is warp-uniform in a tile.
//   1 chain: 0-arcs 0->0, 1->1; 1-arc 1->0     (a = (x0, x1), b = (inf, x0))
//   2 root : one node; 0-arc ->0, 1-arc ->1    (a0 = x0, b0 = x1)
//   3 join : 0-arc 0->0; 1-arc 1->0            (a = (x0, inf), b = (inf, x0))
// m^0 = min_i (c_i + a_i), m^1 - lambda = min_i (c_i + b_i); c = shp(r, .) of
// P_h in a forward pass, the stored/recomputed shp(r, .) in a backward pass.
template <typename T>
__device__ __forceinline__ void hop_mm(const int type, const HopRec<T> *rp, T x0, T x1, T c0, T c1, T &m0, T &m1r) {
  if (type == 1) {
    m0 = fmin(c0 + x0, c1 + x1);
    m1r = c1 + x0;
  } else if (type == 2) {
    m0 = c0 + x0;
    m1r = c0 + x1;
  } else if (type == 3) {
    m0 = c0 + x0;
    m1r = c1 + x0;
  } else {
    const HopRec<T> r = *rp;
    T a0, a1, b0, b1;
    arc_mins(r, x0, x1, a0, a1, b0, b1);
    m0 = fmin(c0 + a0, c1 + a1);
    m1r = fmin(c0 + b0, c1 + b1);
  }
}
// shp(v_i, T) = min(a_i, lambda + b_i)
template <typename T>
__device__ __forceinline__ void hop_ctt(const int type, const HopRec<T> *rp, T x0, T x1, T lam, T &o0, T &o1) {
  if (type == 1) {
    o0 = x0;
    o1 = fmin(x1, lam + x0);
  } else if (type == 2) {
    o0 = fmin(x0, lam + x1);
    o1 = t_inf<T>();
  } else if (type == 3) {
    o0 = x0;
    o1 = lam + x0;
  } else {
    const HopRec<T> r = *rp;
    T a0, a1, b0, b1;
    arc_mins(r, x0, x1, a0, a1, b0, b1);
    o0 = fmin(a0, lam + b0);
    o1 = fmin(a1, lam + b1);
  }
}
// shp(r, v_j) of P_{h+1} = min over arcs into v_j of c_i (+ lambda on 1-arcs)
// (reading A4)
template <typename T>
__device__ __forceinline__ void hop_relax(const int type, const HopRec<T> *rp, T c0, T c1, T lam, T &o0, T &o1) {
  if (type == 1) {
    o0 = fmin(c0, lam + c1);
    o1 = c1;
  } else if (type == 2) {
    o0 = c0;
    o1 = lam + c0;
  } else if (type == 3) {
    o0 = fmin(c0, lam + c1);
    o1 = t_inf<T>();
  } else {
    const HopRec<T> r = *rp;
    o0 = fmin(fmin(c0 + r.A[0], c1 + r.A[2]), lam + fmin(c0 + r.A[4], c1 + r.A[6]));
    o1 = fmin(fmin(c0 + r.A[1], c1 + r.A[3]), lam + fmin(c0 + r.A[5], c1 + r.A[7]));
  }
}

// dual update of one slot (A5, A10); returns the new lambda_h
template <typename T, bool REC>
__device__ __forceinline__ T mask_finish(T *lam, T *va, uint32_t hL, T l, T av, T m0, T m1r, bool valid, T omega, T clamp,
                                         T *m0g, T *m1g, double &acc) {
  const T m1 = l + m1r;
  const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
  const T lam_new = add_rn(sub_rn(l, delta), av);
  // branch-free: a padding row keeps its lambda and writes delta = 0 (selects
  // instead of a branch per row and hop, whose reconvergence made the
  // compiler re-derive the lane's addresses every hop)
  const T dv = valid ? delta : T(0);
  lam[hL] = valid ? lam_new : l;
  va[hL] = dv;
  if (REC && valid) {
    m0g[hL] = m0;
    m1g[hL] = m1;
  }
  acc += (double)fmin(dv, T(0));  // (+0 for padding: acc >= +0 sums stay exact)
  return lam_new;
}

// Loops over the partitions.  Tiles with kind bit 3 ("chain tiles") have
// type-1 (chain) hops everywhere but the first and the last partition: those
// two run the general masks, the middle ones the folded chain expressions --
// no per-hop type dispatch on the dependent chain.  Other tiles run the
// general masks throughout.  Every loop prefetches the next partition's record
// tail, lambda, average and distances before computing the current one.
template <int N>
using Ty = std::integral_constant<int, N>;  // compile-time hop type (hop_mm)

// Record tail (n0, n1, w2, type) of partition h (records given from partition
// hb on).  ENDS (kind bit 4): every hop folded, and the partition sizes are
// 1, 2, 2, ..., 2 -- P_0 = {0}, P_h = {2h - 1, 2h}, top = 2K - 1 -- so the
// tail is arithmetic and the records are never read.
template <bool ENDS, typename T>
__device__ __forceinline__ int4 tail_of(const HopRec<T> *rec, int h, int hb = 0) {
  if (ENDS) return make_int4(h ? 2 * h - 1 : 0, 2 * h + 1, h ? 1 : 0, 0);
  return hop_tail(rec + (h - hb));
}

// Distance accessors of the mask loops: where the lane's distances D[node]
// live.  SmemD: a column of shared memory ([node][L] layout, stride L, row k
// of the lane at +32 k).  TmemD (fp32, one row per lane, 32-row tiles of the
// recompute design): the warp's 32 TMEM lanes (one per BDD), column = node --
// tcgen05.st / tcgen05.ld (32x32b shape) move a lane's value(s) between its
// registers and its TMEM lane; loads are waited for (tcgen05.wait::ld) only
// where their value is consumed, one hop later.
template <typename T, int R>
struct SmemD {
  T *p;
  uint32_t L;
  __device__ __forceinline__ void st(uint32_t n, int k, T v) const { p[n * L + 32u * k] = v; }
  // node n, and node n + 1 if both
  __device__ __forceinline__ void st2(uint32_t n, int k, T a, T b, bool both) const {
    p[n * L + 32u * k] = a;
    if (both) p[(n + 1) * L + 32u * k] = b;
  }
  __device__ __forceinline__ T ld(uint32_t n, int k) const { return p[n * L + 32u * k]; }
  __device__ __forceinline__ void ld2(uint32_t n, int k, T &a, T &b) const {
    a = p[n * L + 32u * k];
    b = p[(n + 1) * L + 32u * k];
  }
  __device__ __forceinline__ void wait(T &, T &) const {}
  __device__ __forceinline__ void fence_st() const {}
};

struct TmemD {
  uint32_t ta;  // TMEM address of column 0 in the warp's lane quarter
  __device__ __forceinline__ void st(uint32_t n, int, float v) const {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + n), "r"(__float_as_uint(v))
                 : "memory");
  }
  __device__ __forceinline__ void st2(uint32_t n, int, float a, float b, bool both) const {
    if (both)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta + n), "r"(__float_as_uint(a)),
                   "r"(__float_as_uint(b))
                   : "memory");
    else
      st(n, 0, a);
  }
  __device__ __forceinline__ void ld2(uint32_t n, int, float &a, float &b) const {
    uint32_t x, y;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(ta + n) : "memory");
    a = __uint_as_float(x);
    b = __uint_as_float(y);
  }
  __device__ __forceinline__ float ld(uint32_t n, int) const {
    float a, b;
    ld2(n, 0, a, b);
    wait(a, b);
    return a;
  }
  // the registers of a tcgen05.ld are valid after tcgen05.wait::ld; routing
  // them through the wait makes every use depend on it
  __device__ __forceinline__ void wait(float &a, float &b) const {
    uint32_t x = __float_as_uint(a), y = __float_as_uint(b);
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(x), "+r"(y)::"memory");
    a = __uint_as_float(x);
    b = __uint_as_float(y);
  }
  __device__ __forceinline__ void fence_st() const { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
};

// Rows per lane (R): a tile of L = 32 R rows of one shape gives lane l the rows
// l, l + 32, ..., l + 32 (R - 1); their values sit at +32 k in every [index][L]
// array.  The R chains share the hop tail, the addresses and the loop control,
// and are independent (R-fold ILP on the dependent hop chain); each one runs
// exactly the arithmetic of R = 1.

// shp(v, T) of every node under the current lambda (no update); e[k] =
// shp(r, T) = E^j.  (kEnergy; phase 1 of a recompute forward pass.)
template <typename T, int LC, bool ENDS, int R, class DA>
__device__ __forceinline__ void mask_ctt_impl(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                              const T *lam, const DA &D, T (&e)[R]) {
  const uint32_t L = LC ? LC : L_rt;  // unsigned offsets: one wide multiply-add per address
  T x0[R], x1[R], l[R];
  int4 tl = tail_of<ENDS>(rec, K - 1);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    x0[k] = T(0);
    x1[k] = t_inf<T>();
    l[k] = lam[(K - 1) * L + 32u * k];
  }
  auto step = [&](auto ch, int h) {
    const uint32_t hn = h > 0 ? h - 1 : 0;
    const int4 tn = tail_of<ENDS>(rec, hn);
    T ln[R];
#pragma unroll
    for (int k = 0; k < R; ++k) ln[k] = lam[hn * L + 32u * k];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      hop_ctt(decltype(ch)::value, rec + (uint32_t)h, x0[k], x1[k], l[k], x0[k], x1[k]);
      D.st2(tl.x, k, x0[k], x1[k], tl.z != 0);
    }
    tl = tn;
#pragma unroll
    for (int k = 0; k < R; ++k) l[k] = ln[k];
  };
  int h = K - 1;
  if (chain) {  // bit 0: chain middle; bit 1: join last, root first
    if (h > 0) {
      if (chain & 2) step(Ty<3>(), h--);
      else step(Ty<0>(), h--);
    }
#pragma unroll 1
    for (; h > 0; --h) step(Ty<1>(), h);
    if ((chain & 2) && h >= 0) step(Ty<2>(), h--);
  }
#pragma unroll 1
  for (; h >= 0; --h) step(Ty<0>(), h);
#pragma unroll
  for (int k = 0; k < R; ++k) e[k] = x0[k];
}

template <typename T, int LC, int R, class DA>
__device__ __forceinline__ void mask_ctt(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                         const T *lam, const DA &D, T (&e)[R]) {
  if (chain & 2) mask_ctt_impl<T, LC, true, R>(K, chain, rec, L_rt, lam, D, e);
  else mask_ctt_impl<T, LC, false, R>(K, chain, rec, L_rt, lam, D, e);
}

// shp(r, v) of every node under the current lambda (no update); e[k] =
// shp(r, T) = E^j.  (kCfr; phase 1 of a recompute backward pass.)
template <typename T, int LC, bool ENDS, int R, class DA>
__device__ __forceinline__ void mask_cfr_impl(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                              const T *lam, const DA &D, T (&e)[R]) {
  const uint32_t L = LC ? LC : L_rt;  // unsigned offsets: one wide multiply-add per address
  T c0[R], c1[R], l[R];
  int4 tl = tail_of<ENDS>(rec, 0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    c0[k] = T(0);
    c1[k] = t_inf<T>();
    l[k] = lam[32u * k];
  }
  auto step = [&](auto ch, int h) {
    const uint32_t hn = h + 1 < K ? h + 1 : h;
    const int4 tn = tail_of<ENDS>(rec, hn);
    T ln[R];
#pragma unroll
    for (int k = 0; k < R; ++k) ln[k] = lam[hn * L + 32u * k];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      D.st2(tl.x, k, c0[k], c1[k], tl.z != 0);
      hop_relax(decltype(ch)::value, rec + (uint32_t)h, c0[k], c1[k], l[k], c0[k], c1[k]);
    }
    tl = tn;
#pragma unroll
    for (int k = 0; k < R; ++k) l[k] = ln[k];
  };
  int h = 0;
  if (chain) {  // bit 0: chain middle; bit 1: root first, join last (kind bits 3, 4)
    if (h < K - 1) {
      if (chain & 2) step(Ty<2>(), h++);
      else step(Ty<0>(), h++);
    }
#pragma unroll 1
    for (; h < K - 1; ++h) step(Ty<1>(), h);
    if ((chain & 2) && h < K) step(Ty<3>(), h++);
  }
#pragma unroll 1
  for (; h < K; ++h) step(Ty<0>(), h);
#pragma unroll
  for (int k = 0; k < R; ++k) e[k] = c0[k];  // after the last partition: the relaxation into top
}

template <typename T, int LC, int R, class DA>
__device__ __forceinline__ void mask_cfr(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                         const T *lam, const DA &D, T (&e)[R]) {
  if (chain & 2) mask_cfr_impl<T, LC, true, R>(K, chain, rec, L_rt, lam, D, e);
  else mask_cfr_impl<T, LC, false, R>(K, chain, rec, L_rt, lam, D, e);
}

// forward pass with updates.  D holds shp(v, T) (stored by the
// previous backward pass, or recomputed by mask_ctt); STORE: D of P_h is
// overwritten with shp(r, v) for the next backward pass (P:315-316 reuse).
// vm: bit k set if row k of the lane is a real row (not padding).
template <typename T, bool STORE, bool REC, int LC, bool ENDS, int R, class DA>
__device__ __forceinline__ double mask_forward_impl(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                                    T *lam, T *va, const DA &D, const uint32_t vm, const T omega,
                                                    const T clamp, T *m0g, T *m1g) {
  const uint32_t L = LC ? LC : L_rt;  // unsigned offsets: one wide multiply-add per address
  double acc = 0.0;
  T c0[R], c1[R], l[R], av[R], x0[R], x1[R];
  int4 tl = tail_of<ENDS>(rec, 0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    c0[k] = T(0);
    c1[k] = t_inf<T>();
    l[k] = lam[32u * k];
    av[k] = va[32u * k];
    D.ld2(tl.y, k, x0[k], x1[k]);
    D.wait(x0[k], x1[k]);
  }
  auto step = [&](auto ch, int h) {
    constexpr int ty = decltype(ch)::value;
    const uint32_t hn = h + 1 < K ? h + 1 : h;
    const int4 tn = tail_of<ENDS>(rec, hn);
    T ln[R], avn[R], x0n[R], x1n[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      ln[k] = lam[hn * L + 32u * k];
      avn[k] = va[hn * L + 32u * k];
      D.ld2(tn.y, k, x0n[k], x1n[k]);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (STORE) D.st2(tl.x, k, c0[k], c1[k], tl.z != 0);
      T m0, m1r;
      hop_mm(ty, rec + (uint32_t)h, x0[k], x1[k], c0[k], c1[k], m0, m1r);
      const T lam_new = mask_finish<T, REC>(lam + 32u * k, va + 32u * k, (uint32_t)h * L, l[k], av[k], m0, m1r,
                                            (vm >> k) & 1u, omega, clamp, REC ? m0g + 32u * k : nullptr,
                                            REC ? m1g + 32u * k : nullptr, acc);
      hop_relax(ty, rec + (uint32_t)h, c0[k], c1[k], lam_new, c0[k], c1[k]);  // A4: 1-arcs priced with the updated lambda_h
    }
    tl = tn;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      D.wait(x0n[k], x1n[k]);
      l[k] = ln[k];
      av[k] = avn[k];
      x0[k] = x0n[k];
      x1[k] = x1n[k];
    }
  };
  int h = 0;
  if (chain) {  // bit 0: chain middle; bit 1: root first, join last (kind bits 3, 4)
    if (h < K - 1) {
      if (chain & 2) step(Ty<2>(), h++);
      else step(Ty<0>(), h++);
    }
#pragma unroll 1
    for (; h < K - 1; ++h) step(Ty<1>(), h);
    if ((chain & 2) && h < K) step(Ty<3>(), h++);
  }
#pragma unroll 1
  for (; h < K; ++h) step(Ty<0>(), h);
#pragma unroll
  for (int k = 0; k < R; ++k)
    if ((vm >> k) & 1u) acc += (double)c0[k];  // E^j = shp(r, T) at the updated lambda
  return acc;
}

template <typename T, bool STORE, bool REC, int LC, int R, class DA>
__device__ __forceinline__ double mask_forward(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                               T *lam, T *va, const DA &D, const uint32_t vm, const T omega,
                                               const T clamp, T *m0g, T *m1g) {
  if (chain & 2)
    return mask_forward_impl<T, STORE, REC, LC, true, R>(K, chain, rec, L_rt, lam, va, D, vm, omega, clamp, m0g, m1g);
  return mask_forward_impl<T, STORE, REC, LC, false, R>(K, chain, rec, L_rt, lam, va, D, vm, omega, clamp, m0g, m1g);
}

// backward pass with updates.  D holds shp(r, v) (stored by the
// forward pass, or recomputed by mask_cfr); STORE: D of P_h is overwritten
// with shp(v, T) for the next forward pass.
template <typename T, bool STORE, bool REC, int LC, bool ENDS, int R, class DA>
__device__ __forceinline__ double mask_backward_impl(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                                     T *lam, T *va, const DA &D, const uint32_t vm, const T omega,
                                                     const T clamp, T *m0g, T *m1g) {
  const uint32_t L = LC ? LC : L_rt;  // unsigned offsets: one wide multiply-add per address
  const T inf = t_inf<T>();
  double acc = 0.0;
  T x0[R], x1[R], l[R], av[R], f0[R], f1[R];  // x: shp(., T) of P_{h+1}; the last partition's targets: top
  int4 tl = tail_of<ENDS>(rec, K - 1);
  // (a one-node partition's second entry is not read: in global memory the
  // load would alias the store of the partition above)
#pragma unroll
  for (int k = 0; k < R; ++k) {
    x0[k] = T(0);
    x1[k] = inf;
    l[k] = lam[(K - 1) * L + 32u * k];
    av[k] = va[(K - 1) * L + 32u * k];
    D.ld2(tl.x, k, f0[k], f1[k]);  // (the second entry of a one-node partition is not used)
    D.wait(f0[k], f1[k]);
    if (!tl.z) f1[k] = inf;
  }
  auto step = [&](auto ch, int h) {
    constexpr int ty = decltype(ch)::value;
    const uint32_t hn = h > 0 ? h - 1 : 0;
    const int4 tn = tail_of<ENDS>(rec, hn);
    T ln[R], avn[R], f0n[R], f1n[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      ln[k] = lam[hn * L + 32u * k];
      avn[k] = va[hn * L + 32u * k];
      D.ld2(tn.x, k, f0n[k], f1n[k]);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      T m0, m1r;
      hop_mm(ty, rec + (uint32_t)h, x0[k], x1[k], f0[k], f1[k], m0, m1r);
      const T lam_new = mask_finish<T, REC>(lam + 32u * k, va + 32u * k, (uint32_t)h * L, l[k], av[k], m0, m1r,
                                            (vm >> k) & 1u, omega, clamp, REC ? m0g + 32u * k : nullptr,
                                            REC ? m1g + 32u * k : nullptr, acc);
      hop_ctt(ty, rec + (uint32_t)h, x0[k], x1[k], lam_new, x0[k], x1[k]);  // shp(v, T) with the updated lambda_h
      if (STORE) D.st2(tl.x, k, x0[k], x1[k], tl.z != 0);
    }
    tl = tn;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      D.wait(f0n[k], f1n[k]);
      l[k] = ln[k];
      av[k] = avn[k];
      f0[k] = f0n[k];
      f1[k] = tn.z ? f1n[k] : inf;
    }
  };
  int h = K - 1;
  if (chain) {  // bit 0: chain middle; bit 1: join last, root first
    if (h > 0) {
      if (chain & 2) step(Ty<3>(), h--);
      else step(Ty<0>(), h--);
    }
#pragma unroll 1
    for (; h > 0; --h) step(Ty<1>(), h);
    if ((chain & 2) && h >= 0) step(Ty<2>(), h--);
  }
#pragma unroll 1
  for (; h >= 0; --h) step(Ty<0>(), h);
#pragma unroll
  for (int k = 0; k < R; ++k)
    if ((vm >> k) & 1u) acc += (double)x0[k];  // E^j = shp(r, T)
  return acc;
}

template <typename T, bool STORE, bool REC, int LC, int R, class DA>
__device__ __forceinline__ double mask_backward(const int K, const int chain, const HopRec<T> *rec, const int L_rt,
                                                T *lam, T *va, const DA &D, const uint32_t vm, const T omega,
                                                const T clamp, T *m0g, T *m1g) {
  if (chain & 2)
    return mask_backward_impl<T, STORE, REC, LC, true, R>(K, chain, rec, L_rt, lam, va, D, vm, omega, clamp, m0g, m1g);
  return mask_backward_impl<T, STORE, REC, LC, false, R>(K, chain, rec, L_rt, lam, va, D, vm, omega, clamp, m0g, m1g);
}

// One arc-mask tile of one pass: the four modes over the lane's R rows.
// Returns the lane's share of the tile's bound partial.
template <typename T, int MODE, bool REC, bool RC, int LC, int R, class DA>
__device__ __forceinline__ double mask_tile(const int K, const int chain, const HopRec<T> *rec, const int L,
                                            T *lm, T *vp, const DA &D, const uint32_t vm, const T omega,
                                            const T clamp, T *m0p, T *m1p) {
  T e[R];
  double acc = 0.0;
  if (MODE == kEnergy || MODE == kCfr) {
    if (MODE == kEnergy) mask_ctt<T, LC, R>(K, chain, rec, L, lm, D, e);
    else mask_cfr<T, LC, R>(K, chain, rec, L, lm, D, e);
#pragma unroll
    for (int k = 0; k < R; ++k)
      if ((vm >> k) & 1u) acc += (double)e[k];
  } else if (MODE == kForward) {
    if (RC) {
      mask_ctt<T, LC, R>(K, chain, rec, L, lm, D, e);
      D.fence_st();  // (TMEM: the stores above complete before the loads below)
    }
    acc = mask_forward<T, !RC, REC, LC, R>(K, chain, rec, L, lm, vp, D, vm, omega, clamp, m0p, m1p);
  } else {
    if (RC) {
      mask_cfr<T, LC, R>(K, chain, rec, L, lm, D, e);
      D.fence_st();
    }
    acc = mask_backward<T, !RC, REC, LC, R>(K, chain, rec, L, lm, vp, D, vm, omega, clamp, m0p, m1p);
  }
  return acc;
}

// Stage buffer of one tile (layout: internal.h).
template <typename T>
struct Stage {
  T *lam;
  T *va;
  T *dist;
  uint32_t *topo;
  int32_t *hop;
  uint32_t *pairs;  // tile-closed pair list (after the tail)
};

// RC: recompute design, no distances in the stage buffer (internal.h)
template <typename T, bool RC>
__device__ __forceinline__ Stage<T> stage_at(unsigned char *base, const TileDesc &d) {
  constexpr int tsz = sizeof(T);
  Stage<T> s;
  unsigned char *p = base;
  s.lam = reinterpret_cast<T *>(p);
  p += stage_lam_bytes(tsz, d.K, d.lanes);
  s.va = reinterpret_cast<T *>(p);
  p += stage_va_bytes(tsz, d.K, d.lanes);
  s.dist = RC ? nullptr : reinterpret_cast<T *>(p);
  if (!RC) p += stage_dist_bytes(tsz, d.nodes, d.lanes);
  s.topo = reinterpret_cast<uint32_t *>(p);
  p += stage_topo_bytes(d.kind, d.nodes, d.lanes);
  s.hop = reinterpret_cast<int32_t *>(p);
  s.pairs = reinterpret_cast<uint32_t *>(s.topo) + stage_tail_bytes(tsz, d.kind, d.K, d.nodes, d.lanes) / 4;
  return s;
}

// One lane issues the TMA bulk copies of a tile's lambda, variables, topology
// and partition offsets; completion is counted on the stage's mbarrier.
template <typename T, int MODE, bool RC>
__device__ __forceinline__ void issue_stage(const SweepArgs &a, const TileDesc &d, const Stage<T> &s, uint64_t *bar) {
  const bool upd = MODE == kForward || MODE == kBackward;
  const uint32_t lam_b = (uint32_t)d.K * d.lanes * sizeof(T);
  const uint32_t va_b = upd ? lam_b : 0u;
  const uint32_t dist_b = RC ? 0u : (uint32_t)(d.nodes + 2) * d.lanes * sizeof(T);
  const bool masks = d.kind & 4;  // hop records instead of topology + partition offsets
  // (records: none staged for fully folded tiles, which never read them, and
  // for kind bit 6 tiles, which read them from global memory)
  const uint32_t topo_b = masks ? (uint32_t)stage_tail_bytes((int)sizeof(T), d.kind, d.K, d.nodes, d.lanes)
                                : (uint32_t)stage_topo_bytes(d.kind, d.nodes, d.lanes);
  const uint32_t hop_b = masks ? 0u : (uint32_t)stage_hop_bytes(d.K);
  const uint32_t pair_b = (upd && a.pairs && d.n_pairs > 0) ? (uint32_t)stage_pairs_bytes(d.n_pairs) : 0u;
  mbar_expect_tx(bar, lam_b + va_b + dist_b + topo_b + hop_b + pair_b);
  if (pair_b) bulk_g2s(s.pairs, a.pairs + d.pair_base, pair_b, bar);
  bulk_g2s(s.lam, reinterpret_cast<const T *>(a.lambda) + d.slot_base, lam_b, bar);
  if (va_b) bulk_g2s(s.va, reinterpret_cast<const T *>(a.avg_in) + d.slot_base, va_b, bar);
  if (!RC) bulk_g2s(s.dist, reinterpret_cast<const T *>(a.dist) + d.dist_base, dist_b, bar);
  if (masks) {
    if (topo_b) bulk_g2s(s.topo, a.recs + 16 * (int64_t)d.rec_base, topo_b, bar);
  } else {
    bulk_g2s(s.topo, a.topo + d.topo_base, topo_b, bar);
    bulk_g2s(s.hop, a.hop_off + d.hop_base, hop_b, bar);
  }
}

// One pass over all tiles.  Persistent warps claim tiles dynamically; with
// two stage buffers the next tile's TMA loads are in flight while the current
// one is processed.  lambda, delta and the distances go back with TMA bulk
// stores.
// cp.async of one 64-byte tile descriptor into shared memory (lanes 0-3)
__device__ __forceinline__ void fetch_desc(TileDesc *dst, const TileDesc *src, int lane) {
  if (lane < 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(reinterpret_cast<char *>(dst) + 16 * lane)),
                 "l"(reinterpret_cast<const char *>(src) + 16 * lane)
                 : "memory");
  cp_async_commit();
}

// RC: recompute design (narrow tiles, every tile staged): the stage buffers
// hold lambda, averages, topology and partition offsets only; the distances
// live in a per-warp scratch column per lane (the DB region) and never touch HBM.
// RW: the most rows per lane of any tile (1, 2 or 4; separate instantiations so
// that problems without wide tiles keep the register budget of RW = 1).
// TM: the recompute design's distances of 32-row tiles in tensor memory (fp32,
// RW = 1).  A kernel holding tcgen05 code runs one CTA per SM (the driver's
// rule), so TM kernels launch one CTA of up to 16 warps per SM and the others
// carry no tcgen05 code at all.
// Registers, stated: CTAs of 4 warps (solver.cpp), at least 6 resident per SM
// (<= 80 registers; 4 with four rows per lane: <= 128); TM kernels one CTA of
// up to 16 warps.  Left to ptxas, the same source compiled to 64 (spilling)
// or to 97-106 registers depending on how --split-compile partitioned the
// module, which moved MRF-LP between 5 and 4 resident CTAs per SM (541 vs 571
// us per iteration) and GM-worms between 6 and 4 (42.6 vs 45.5 us).
template <typename T, int MODE, bool REC, bool RC, int RW, bool TM>
__global__ void __launch_bounds__(TM ? 512 : 128, TM ? 1 : (RW >= 4 ? 4 : 6)) sweep_kernel(const SweepArgs a) {
  static_assert(!TM || (RC && RW == 1 && std::is_same<T, float>::value), "TMEM distances: fp32 recompute design");
  constexpr bool kUpd = MODE == kForward || MODE == kBackward;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  unsigned char *wbase = smem_raw + (size_t)warp * warp_bytes(a.SB, a.DB, a.NB);
  uint64_t *bar = reinterpret_cast<uint64_t *>(wbase);          // bar[0], bar[1]
  TileDesc *ring = reinterpret_cast<TileDesc *>(wbase + 64);    // 3 descriptors
  unsigned char *const sbuf0 = wbase + kWarpHeader;
  unsigned char *const sbuf1 = wbase + kWarpHeader + (a.NB > 1 ? a.SB : 0);
  unsigned char *const rbase = wbase + kWarpHeader + a.NB * a.SB;

  T *__restrict__ lambda = reinterpret_cast<T *>(a.lambda);
  T *__restrict__ delta_out = reinterpret_cast<T *>(a.delta_out);
  T *__restrict__ gdist = reinterpret_cast<T *>(a.dist);
  const T omega = arg_omega<T>(a), clamp = arg_clamp<T>(a);
  const int gwarp = blockIdx.x * wpb + warp;

  // TM: the distance scratch of the 32-row arc-mask tiles lives in tensor
  // memory.  The CTA allocates groups x tmem_cols columns (tmem_cols >= nodes
  // + 2 of every such tile, groups = ceil(warps / 4), rounded to a power of
  // two); warp w uses TMEM lanes [32 (w % 4), + 32) -- one per BDD -- and
  // columns [tmem_cols (w / 4), + tmem_cols), column = node.  Shared memory then
  // holds only the stages.
  uint32_t tm_base = 0, tm_alloc = 0;
  uint32_t *const tm_slot = reinterpret_cast<uint32_t *>(smem_raw + 16);  // (warp 0's header, unused bytes)
  if constexpr (TM) {
    const uint32_t groups = (uint32_t)(wpb + 3) / 4;
    tm_alloc = 32;
    while (tm_alloc < groups * (uint32_t)a.tmem_cols) tm_alloc *= 2;
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tm_slot)),
                   "r"(tm_alloc)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tm_base = *tm_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * (uint32_t)a.tmem_cols;
  }

  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  // tile schedule (tiles sorted by decreasing cost): warp w takes its tiles of
  // the first two static rounds; later tiles are claimed from a global counter
  // (reset before every sweep, claims start at 2 W), or static_sched: every
  // round static
  const int W = gridDim.x * wpb;
  // schedule index: consecutive (i.e. the costliest) static tiles go to the
  // same warp slot of consecutive CTAs, i.e. to different SMs, instead of
  // filling one CTA's warps first (FDOG_SPREAD=0: the CTA-major order)
  const int sw = a.spread ? warp * (int)gridDim.x + (int)blockIdx.x : gwarp;
  int t = sw;
  // static rounds alternate direction (round r takes tile r W + w for even r,
  // r W + W - 1 - w for odd r): the warp with the costliest tile of one round
  // gets the cheapest of the next (cost-sorted tiles; a.snake)
  auto sidx = [&](int r) -> int {
    const long long i = (long long)r * W + ((a.snake && (r & 1)) ? W - 1 - sw : sw);
    return i < a.n_tiles ? (int)i : a.n_tiles;
  };
  int rnd = 1;  // static round of tn
  int tn = sidx(1);
  // descriptors are constant: fetch them before waiting for the predecessor
  if (t < a.n_tiles) fetch_desc(&ring[0], a.tiles + t, lane);
  if (tn < a.n_tiles) fetch_desc(&ring[1], a.tiles + tn, lane);
  pdl_wait();
  unsigned long long t_start = 0;
  int n_done = 0;
  if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  // claims take claim_batch consecutive tiles per atomic (many small tiles:
  // one counter serialises the claims of every warp)
  const int CB = a.claim_batch > 1 ? a.claim_batch : 1;
  auto claim_issue = [&]() -> int { return lane == 0 ? (int)atomicAdd(a.tile_counter, (unsigned)CB) : 0; };
  auto claim_get = [&](int raw) -> int { return 2 * W + __shfl_sync(0xffffffffu, raw, 0); };
  int bnext = 0, bend = 0;  // the rest of the current batch (warp-uniform)
  // pipeline per warp: while tile t is processed, the TMA stage loads of the
  // next tile are in flight, the descriptor of the one after is being fetched
  // (cp.async), and (dynamic schedule) the claim for the tile after that.
  uint32_t phase = 0;  // bit b = parity of bar[b]
  int b = 0, rc = 0;   // stage buffer and ring slot of the current tile
  cp_async_wait_all();
  __syncwarp();
  if (t < a.n_tiles && (ring[0].kind & 2) && lane == 0)
    issue_stage<T, MODE, RC>(a, ring[0], stage_at<T, RC>(sbuf0, ring[0]), &bar[0]);
  bool pending = !a.static_sched && tn < a.n_tiles && 2 * W < a.n_tiles;  // a claim is in flight
  int raw_nn = pending ? claim_issue() : 0;
  while (t < a.n_tiles) {
    const TileDesc &d = ring[rc];
    const TileDesc &dn = ring[rc == 2 ? 0 : rc + 1];
    TileDesc &dnn = ring[rc == 0 ? 2 : rc - 1];
    const bool has_next = tn < a.n_tiles;
    const int bn = a.NB > 1 ? (b ^ 1) : 0;
    if (a.NB > 1 && has_next && (dn.kind & 2) && lane == 0) {
      bulk_wait_read_all();  // the bulk stores issued from stage bn have read their source
      issue_stage<T, MODE, RC>(a, dn, stage_at<T, RC>(bn ? sbuf1 : sbuf0, dn), &bar[bn]);
    }
    int tnn = a.n_tiles;
    if (a.static_sched) {
      tnn = sidx(++rnd);
    } else {
      if (bnext >= bend && pending) {
        bnext = claim_get(raw_nn);
        bend = bnext + CB < a.n_tiles ? bnext + CB : a.n_tiles;
        pending = false;
      }
      if (bnext < bend) tnn = bnext++;
    }
    __syncwarp();  // every lane has read dnn's slot (it held the previous tile)
    if (tnn < a.n_tiles) fetch_desc(&dnn, a.tiles + tnn, lane);  // used one tile later
    if (!a.static_sched && !pending && bnext >= bend && tnn < a.n_tiles) {
      pending = true;  // the next batch's claim, in flight while this one is used
      raw_nn = claim_issue();
    }
    const int L = d.lanes;
    const bool active = lane < L;
    const bool valid = lane < d.n_lanes;
    const int K = d.K;
    double acc = 0.0;
    if (d.kind & 2) {
      // staged tile: everything on chip
      const Stage<T> s = stage_at<T, RC>(b ? sbuf1 : sbuf0, d);
      mbar_wait(&bar[b], (phase >> b) & 1u);
      phase ^= 1u << b;
      if (kUpd && a.pairs && d.n_pairs > 0) {
        // tile-closed pairs (|J_i| = 2, both slots in this tile; plan.cpp): the
        // stage holds their delta_bar; avg_i = (delta_bar_1 + delta_bar_2) / 2
        // (A1 -- the averaging kernel's ELL arithmetic), written into
        // both slots
#pragma unroll 4
        for (int e = lane; e < d.n_pairs; e += 32) {
          const uint32_t w = s.pairs[e];
          const uint32_t i = w & 0xFFFFu, m = w >> 16;
          const T v = (s.va[i] + s.va[m]) / T(2);
          s.va[i] = v;
          s.va[m] = v;
        }
        __syncwarp();
      }
      if (d.kind & 4) {
        // arc-mask tile (narrow shape, shared topology)
        if (active) {
          // (kind bit 6: the shape's records in global memory, not staged)
          const HopRec<T> *rec = (d.kind & kKindRecGlobal)
                                     ? reinterpret_cast<const HopRec<T> *>(a.recs + 16 * (int64_t)d.rec_base)
                                     : reinterpret_cast<const HopRec<T> *>(s.topo);
          const int chain = ((d.kind & 8) ? 1 : 0) | ((d.kind & 16) ? 2 : 0);
          T *D = RC ? reinterpret_cast<T *>(rbase) + lane : s.dist + lane;
          if (RC && !(TM && L == 32))
            for (int o = 0; o < L; o += 32) {
              D[d.nodes * L + o] = T(0);              // top
              D[(d.nodes + 1) * L + o] = t_inf<T>();  // bottom
            }
          T *m0p = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
          T *m1p = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
          T *lm = s.lam + lane, *vp = s.va + lane;
          // rows per lane: tiles of 64 / 128 rows (short rows, plan.cpp)
          const uint32_t vm = (lane < d.n_lanes ? 1u : 0u) | (lane + 32 < d.n_lanes ? 2u : 0u) |
                              (lane + 64 < d.n_lanes ? 4u : 0u) | (lane + 96 < d.n_lanes ? 8u : 0u);
          if (L == 32) {
            if constexpr (TM) {  // distances in the warp's TMEM lanes (plan: Plan::tmem_cols)
              __syncwarp();        // (tcgen05 ops are warp-collective: converged after the stage wait)
              const TmemD tm{tm_base};
              tm.st2(d.nodes, 0, T(0), t_inf<T>(), true);  // top, bottom
              acc = mask_tile<T, MODE, REC, RC, 32, 1>(K, chain, rec, L, lm, vp, tm, vm, omega, clamp, m0p, m1p);
            } else {
              acc = mask_tile<T, MODE, REC, RC, 32, 1>(K, chain, rec, L, lm, vp, SmemD<T, 1>{D, 32u}, vm, omega, clamp,
                                                       m0p, m1p);
            }
          } else if (RW >= 2 && L == 64) {
            acc = mask_tile<T, MODE, REC, RC, 64, 2>(K, chain, rec, L, lm, vp, SmemD<T, 2>{D, 64u}, vm, omega, clamp,
                                                     m0p, m1p);
          } else if (RW >= 4 && L == 128) {
            acc = mask_tile<T, MODE, REC, RC, 128, 4>(K, chain, rec, L, lm, vp, SmemD<T, 4>{D, 128u}, vm, omega,
                                                      clamp, m0p, m1p);
          } else {
            acc = mask_tile<T, MODE, REC, RC, 0, 1>(K, chain, rec, L, lm, vp, SmemD<T, 1>{D, (uint32_t)L}, vm & 1u,
                                                    omega, clamp, m0p, m1p);
          }
        }
      } else if (RC) {
        if (active) {
          T *D = reinterpret_cast<T *>(rbase) + lane;  // this lane's distance column
          D[d.nodes * L] = T(0);                      // top
          D[(d.nodes + 1) * L] = t_inf<T>();          // bottom
          const uint32_t *tp = (d.kind & 1) ? s.topo + lane : s.topo;
          const int ts = (d.kind & 1) ? L : 1;
          T *m0p = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
          T *m1p = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
          if (MODE == kEnergy) {
            // sum_j E^j(lambda): shp(v, T) under the current lambda
            const int32_t *ho = s.hop;
#pragma unroll 1
            for (int h = K - 1; h >= 0; --h) {
              const T l = s.lam[h * L + lane];
              const int n1 = ho[h + 1];
#pragma unroll 1
              for (int n = ho[h]; n < n1; ++n) {
                const uint32_t e = tp[n * ts];
                D[n * L] = fmin(D[(e & 0xFFFFu) * L], l + D[(e >> 16) * L]);
              }
            }
            acc = valid ? (double)D[0] : 0.0;
          } else if (L == 32 && !(d.kind & 1)) {
            acc = process_rc_w2<T, MODE, REC, 32>(K, d.nodes, s.hop, tp, 1, 32, s.lam + lane, s.va + lane, D, valid,
                                                  omega, clamp, m0p, m1p);
          } else {
            acc = process_rc_w2<T, MODE, REC, 0>(K, d.nodes, s.hop, tp, ts, L, s.lam + lane, s.va + lane, D, valid,
                                                 omega, clamp, m0p, m1p);
          }
        }
      } else if (active) {
        const uint32_t *tp = (d.kind & 1) ? s.topo + lane : s.topo;
        T *R = reinterpret_cast<T *>(rbase) + lane;
        T *m0p = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
        T *m1p = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
        if (kUpd && d.max_w <= 2 && L == 32 && !(d.kind & 1))
          acc = process_bdd_w2<T, MODE, REC, 32>(K, s.hop, tp, 1, 32, s.lam + lane, s.va + lane, s.dist + lane, valid,
                                                 omega, clamp, m0p, m1p);
        else if (kUpd && d.max_w <= 2)
          acc = process_bdd_w2<T, MODE, REC, 0>(K, s.hop, tp, (d.kind & 1) ? L : 1, L, s.lam + lane, s.va + lane,
                                                s.dist + lane, valid, omega, clamp, m0p, m1p);
        else
          acc = process_bdd<T, MODE, REC>(K, d.nodes, s.hop, tp, (d.kind & 1) ? L : 1, L, s.lam + lane, s.va + lane,
                                          s.dist + lane, R, d.max_w, valid, omega, clamp, m0p, m1p);
      }
      fence_proxy_async();  // lanes' shared-memory writes -> visible to the TMA stores
      __syncwarp();
      if (lane == 0) {
        if (kUpd) {
          const uint32_t bytes = (uint32_t)K * L * sizeof(T);
          bulk_s2g(lambda + d.slot_base, s.lam, bytes);
          bulk_s2g(delta_out + d.slot_base, s.va, bytes);
        }
        if (!RC) bulk_s2g(gdist + d.dist_base, s.dist, (uint32_t)(d.nodes + 2) * L * sizeof(T));
        bulk_commit();
      }
    } else if (d.kind & 32) {
      // cooperative tile: one wide BDD, node-parallel over the warp
      using U = typename OrdOf<T>::U;
      U *buf = a.coop_smem ? reinterpret_cast<U *>(rbase)
                           : reinterpret_cast<U *>(a.scratch) + (size_t)gwarp * a.scratch_stride;
      T *m0p = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base : nullptr;
      T *m1p = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base : nullptr;
      acc = process_bdd_coop<T, MODE, REC>(K, d.nodes, a.hop_off + d.hop_base,
                                           reinterpret_cast<const uint2 *>(a.topo) + d.topo_base,
                                           lambda + d.slot_base, delta_out + d.slot_base, gdist + d.dist_base, buf,
                                           a.coop_bw, lane, omega, clamp, m0p, m1p,
                                           a.lambda0 ? reinterpret_cast<T *>(a.lambda0) + d.slot_base : nullptr,
                                           a.avg0 ? reinterpret_cast<const T *>(a.avg0) + d.slot_base : nullptr);
    } else {
      // direct tile (exceeds the per-warp budget; L = 32): global memory and a
      // per-warp scratch area for the relaxation buffers
      const int64_t sbase = d.slot_base + lane;
      const uint32_t *tp = (d.kind & 1) ? a.topo + d.topo_base + lane : a.topo + d.topo_base;
      T *R = reinterpret_cast<T *>(a.scratch) + (size_t)gwarp * a.scratch_stride + lane;
      T *m0p = REC ? reinterpret_cast<T *>(a.m0) + sbase : nullptr;
      T *m1p = REC ? reinterpret_cast<T *>(a.m1) + sbase : nullptr;
      acc = process_bdd<T, MODE, REC>(K, d.nodes, a.hop_off + d.hop_base, tp, (d.kind & 1) ? 32 : 1, 32,
                                      lambda + sbase, delta_out + sbase, gdist + d.dist_base + lane, R, d.max_w,
                                      valid, omega, clamp, m0p, m1p,
                                      a.lambda0 ? reinterpret_cast<T *>(a.lambda0) + sbase : nullptr,
                                      a.avg0 ? reinterpret_cast<const T *>(a.avg0) + sbase : nullptr);
    }
    acc = warp_sum(acc);
    if (lane == 0) a.lb_part[t] = acc;
    cp_async_wait_all();  // the descriptor of the tile after next has landed
    __syncwarp();
    if (a.NB == 1 && has_next && (dn.kind & 2) && lane == 0) {
      bulk_wait_read_all();  // single stage buffer: its stores must have read it
      issue_stage<T, MODE, RC>(a, dn, stage_at<T, RC>(sbuf0, dn), &bar[0]);
    }
    t = tn;
    tn = tnn;
    rc = rc == 2 ? 0 : rc + 1;
    b = bn;
    ++n_done;
  }
  if (a.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.trace && lane == 0) {
    unsigned long long t_end, smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(*reinterpret_cast<unsigned *>(&smid)));
    smid &= 0xffffffffull;
    unsigned long long *o = a.trace + 4 * (size_t)gwarp;
    o[0] = t_start;
    o[1] = t_end;
    o[2] = (unsigned long long)n_done;
    o[3] = smid;
  }
  if (lane == 0) bulk_wait_read_all();  // shared memory must outlive the TMA stores' reads
  __syncwarp();
  if constexpr (TM) {  // every warp is done with its TMEM lanes
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tm_slot), "r"(tm_alloc) : "memory");
  }
}

// ---------------------------------------------------------------------------
// Streaming sweep for narrow tiles (every partition <= 2 nodes): one warp per
// tile, no shared memory.  Each lane streams its BDD partition by partition
// straight from global memory -- per partition one coalesced 128-byte access
// per array (lambda, avg/delta, the two distances) -- with the loads of the
// next two partitions in flight (software pipeline), so occupancy is bounded
// by registers only.  Same arithmetic and D/va conventions as process_bdd_w2.
// Forward / backward pass over partitions [hb, he) of a K-partition BDD whose
// lambda, averages and hop records are given from partition hb on (chunk
// buffers) and whose distances hold rows from node r0 on; the recursion state
// (c forward, x backward) is carried in and out.  The same prefetching loops
// and hop arithmetic as mask_forward / mask_backward (store design).
template <typename T, bool REC, int LC, bool ENDS>
__device__ __forceinline__ void mask_forward_range_impl(const int hb, const int he, const int K, const int chain,
                                                   const HopRec<T> *rec, const int L_rt, T *lam, T *va, T *D,
                                                   const int r0, const bool valid, const T omega, const T clamp,
                                                   T *m0g, T *m1g, T &c0, T &c1, double &acc) {
  const uint32_t L = LC ? LC : L_rt;
  int4 tl = tail_of<ENDS>(rec, hb, hb);
  T l = lam[0], av = va[0];
  T x0 = D[(uint32_t)(tl.y - r0) * L], x1 = D[(uint32_t)(tl.y + 1 - r0) * L];
  auto step = [&](auto ch, int h) {
    constexpr int ty = decltype(ch)::value;
    const uint32_t i = h - hb, in = h + 1 < he ? i + 1 : i;
    const int4 tn = tail_of<ENDS>(rec, hb + (int)in, hb);
    const T ln = lam[in * L], avn = va[in * L];
    const T x0n = D[(uint32_t)(tn.y - r0) * L], x1n = D[(uint32_t)(tn.y + 1 - r0) * L];
    D[(uint32_t)(tl.x - r0) * L] = c0;  // keep shp(r, v) for the backward pass
    if (tl.z) D[(uint32_t)(tl.x + 1 - r0) * L] = c1;
    T m0, m1r;
    hop_mm(ty, rec + i, x0, x1, c0, c1, m0, m1r);
    const T lam_new = mask_finish<T, REC>(lam, va, i * L, l, av, m0, m1r, valid, omega, clamp, m0g, m1g, acc);
    hop_relax(ty, rec + i, c0, c1, lam_new, c0, c1);
    tl = tn;
    l = ln;
    av = avn;
    x0 = x0n;
    x1 = x1n;
  };
  int h = hb;
  if (chain) {
    if (h == 0 && h < he && K > 1) {
      if (chain & 2) step(Ty<2>(), h++);
      else step(Ty<0>(), h++);
    }
    const int hm = min(he, K - 1);
#pragma unroll 1
    for (; h < hm; ++h) step(Ty<1>(), h);
    if ((chain & 2) && h == K - 1 && h < he) step(Ty<3>(), h++);
  }
#pragma unroll 1
  for (; h < he; ++h) step(Ty<0>(), h);
}

template <typename T, bool REC, int LC>
__device__ __forceinline__ void mask_forward_range(const int hb, const int he, const int K, const int chain,
                                                   const HopRec<T> *rec, const int L_rt, T *lam, T *va, T *D,
                                                   const int r0, const bool valid, const T omega, const T clamp,
                                                   T *m0g, T *m1g, T &c0, T &c1, double &acc) {
  if (chain & 2) return mask_forward_range_impl<T, REC, LC, true>(hb, he, K, chain, rec, L_rt, lam, va, D, r0, valid, omega, clamp, m0g, m1g, c0, c1, acc);
  return mask_forward_range_impl<T, REC, LC, false>(hb, he, K, chain, rec, L_rt, lam, va, D, r0, valid, omega, clamp, m0g, m1g, c0, c1, acc);
}

template <typename T, bool REC, int LC, bool ENDS>
__device__ __forceinline__ void mask_backward_range_impl(const int hb, const int he, const int K, const int chain,
                                                    const HopRec<T> *rec, const int L_rt, T *lam, T *va, T *D,
                                                    const int r0, const bool valid, const T omega, const T clamp,
                                                    T *m0g, T *m1g, T &x0, T &x1, double &acc) {
  const uint32_t L = LC ? LC : L_rt;
  const T inf = t_inf<T>();
  const uint32_t top = he - 1 - hb;
  int4 tl = tail_of<ENDS>(rec, hb + (int)top, hb);
  T l = lam[top * L], av = va[top * L];
  T f0 = D[(uint32_t)(tl.x - r0) * L], f1 = tl.z ? D[(uint32_t)(tl.x + 1 - r0) * L] : inf;
  auto step = [&](auto ch, int h) {
    constexpr int ty = decltype(ch)::value;
    const uint32_t i = h - hb, in = h > hb ? i - 1 : i;
    const int4 tn = tail_of<ENDS>(rec, hb + (int)in, hb);
    const T ln = lam[in * L], avn = va[in * L];
    const T f0n = D[(uint32_t)(tn.x - r0) * L], f1n = tn.z ? D[(uint32_t)(tn.x + 1 - r0) * L] : inf;
    T m0, m1r;
    hop_mm(ty, rec + i, x0, x1, f0, f1, m0, m1r);
    const T lam_new = mask_finish<T, REC>(lam, va, i * L, l, av, m0, m1r, valid, omega, clamp, m0g, m1g, acc);
    hop_ctt(ty, rec + i, x0, x1, lam_new, x0, x1);  // shp(v, T) with the updated lambda_h
    D[(uint32_t)(tl.x - r0) * L] = x0;
    if (tl.z) D[(uint32_t)(tl.x + 1 - r0) * L] = x1;
    tl = tn;
    l = ln;
    av = avn;
    f0 = f0n;
    f1 = f1n;
  };
  int h = he - 1;
  if (chain) {
    if (h == K - 1 && h >= hb && K > 1) {
      if (chain & 2) step(Ty<3>(), h--);
      else step(Ty<0>(), h--);
    }
    const int hm = max(hb, 1);
#pragma unroll 1
    for (; h >= hm; --h) step(Ty<1>(), h);
    if ((chain & 2) && h == 0 && h >= hb) step(Ty<2>(), h--);
  }
#pragma unroll 1
  for (; h >= hb; --h) step(Ty<0>(), h);
}

template <typename T, bool REC, int LC>
__device__ __forceinline__ void mask_backward_range(const int hb, const int he, const int K, const int chain,
                                                    const HopRec<T> *rec, const int L_rt, T *lam, T *va, T *D,
                                                    const int r0, const bool valid, const T omega, const T clamp,
                                                    T *m0g, T *m1g, T &x0, T &x1, double &acc) {
  if (chain & 2) return mask_backward_range_impl<T, REC, LC, true>(hb, he, K, chain, rec, L_rt, lam, va, D, r0, valid, omega, clamp, m0g, m1g, x0, x1, acc);
  return mask_backward_range_impl<T, REC, LC, false>(hb, he, K, chain, rec, L_rt, lam, va, D, r0, valid, omega, clamp, m0g, m1g, x0, x1, acc);
}

// ---------------------------------------------------------------------------
// Chunked sweep for rows too long to stage whole (store design, arc-mask
// tiles; e.g. SURVEY §8(d)'s thin-hop microbench, one BDD of 10^4 partitions,
// and QAP n=128): one warp per tile walks the partitions in chunks of kChunk.
// A chunk's lambda, averages, hop records and distance rows are staged into
// the warp's shared memory by TMA bulk copies, double-buffered (the next
// chunk's loads are in flight while the current one is computed at
// shared-memory latency); lambda, delta and the chunk's own distance rows go
// back by TMA bulk stores.  The hop recursion carries its state (shp(r, .) of
// the current partition forward, shp(., T) of the partition above backward)
// in registers across chunks.  Same arithmetic as mask_forward /
// mask_backward (store design).  Chunks never overlap in what they write, and
// a chunk reads only distance rows no earlier chunk of the pass writes.
constexpr int kChunk = 32;

template <typename T>
__host__ __device__ __forceinline__ int chunk_rows() { return 2 * (kChunk + 1) + 3; }  // <= 2 nodes per partition
template <typename T>
__host__ __device__ __forceinline__ int chunk_stage_bytes() {
  return 2 * kChunk * 32 * (int)sizeof(T) + kChunk * (8 * (int)sizeof(T) + 16) + chunk_rows<T>() * 32 * (int)sizeof(T);
}
template <typename T>
__host__ __device__ __forceinline__ int chunk_warp_bytes() { return (128 + 2 * chunk_stage_bytes<T>() + 127) & ~127; }

struct ChunkSpan {
  int h0, h1, r0, rown, rend;  // hops [h0, h1); rows [r0, rend) loaded, [r0, rown) written back
};

template <typename T, int MODE>
__device__ __forceinline__ ChunkSpan chunk_span(const TileDesc &d, const HopRec<T> *grec, int c) {
  ChunkSpan sp;
  sp.h0 = c * kChunk;
  sp.h1 = min(d.K, sp.h0 + kChunk);
  sp.r0 = __ldg(&grec[sp.h0].n0);
  sp.rown = __ldg(&grec[sp.h1 - 1].n1);  // first node after the chunk (= nodes on the last)
  // forward: also the next partition (its distances are the successors'
  // shp(., T); the last chunk's are the sentinels), +1 row so the second node
  // read of a one-node next partition (masked out) stays a defined value
  sp.rend = MODE == kForward ? min(d.nodes + 2, (sp.h1 < d.K ? __ldg(&grec[sp.h1].n1) : d.nodes + 2) + 1) : sp.rown;
  return sp;
}

template <typename T>
struct ChunkStage {
  T *lam, *va, *D;
  HopRec<T> *rec;
};
template <typename T>
__device__ __forceinline__ ChunkStage<T> chunk_stage_at(unsigned char *p) {
  ChunkStage<T> st;
  st.lam = reinterpret_cast<T *>(p);
  st.va = st.lam + kChunk * 32;
  st.rec = reinterpret_cast<HopRec<T> *>(st.va + kChunk * 32);
  st.D = reinterpret_cast<T *>(st.rec + kChunk);
  return st;
}

template <typename T>
__device__ __forceinline__ void chunk_issue(const ChunkStage<T> &st, const ChunkSpan &sp, int L, const T *glam,
                                            const T *gva, const HopRec<T> *grec, const T *gD, uint64_t *bar,
                                            bool folded) {
  const int nh = sp.h1 - sp.h0;
  const uint32_t lb = (uint32_t)nh * L * sizeof(T), rb = folded ? 0u : (uint32_t)nh * sizeof(HopRec<T>);
  const uint32_t db = (uint32_t)(sp.rend - sp.r0) * L * sizeof(T);
  mbar_expect_tx(bar, 2 * lb + rb + db);
  bulk_g2s(st.lam, glam + (int64_t)sp.h0 * L, lb, bar);
  bulk_g2s(st.va, gva + (int64_t)sp.h0 * L, lb, bar);
  if (rb) bulk_g2s(st.rec, grec + sp.h0, rb, bar);
  bulk_g2s(st.D, gD + (int64_t)sp.r0 * L, db, bar);
}

template <typename T, int MODE, bool REC>
__global__ void __launch_bounds__(128) sweep_chunk_kernel(const SweepArgs a) {
  extern __shared__ __align__(128) unsigned char csm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + warp;
  if (t >= a.n_tiles) return;  // whole warps
  unsigned char *wb = csm + (size_t)warp * chunk_warp_bytes<T>();
  uint64_t *bar = reinterpret_cast<uint64_t *>(wb);  // bar[0], bar[1]
  unsigned char *sb[2] = {wb + 128, wb + 128 + chunk_stage_bytes<T>()};
  const TileDesc d = a.tiles[t];
  const int L = d.lanes, K = d.K;
  const bool valid = lane < d.n_lanes, active = lane < L;
  const int chain = ((d.kind & 8) ? 1 : 0) | ((d.kind & 16) ? 2 : 0);
  const HopRec<T> *grec = reinterpret_cast<const HopRec<T> *>(a.recs + 16 * (int64_t)d.rec_base);
  T *glam = reinterpret_cast<T *>(a.lambda) + d.slot_base;
  T *gva = reinterpret_cast<T *>(a.delta_out) + d.slot_base;
  T *gD = reinterpret_cast<T *>(a.dist) + d.dist_base;
  T *m0g = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
  T *m1g = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
  const T omega = arg_omega<T>(a), clamp = arg_clamp<T>(a), inf = t_inf<T>();
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_wait();
  const int nch = (K + kChunk - 1) / kChunk;
  auto chunk_of = [&](int ci) { return MODE == kForward ? ci : nch - 1 - ci; };
  if (lane == 0) chunk_issue(chunk_stage_at<T>(sb[0]), chunk_span<T, MODE>(d, grec, chunk_of(0)), L, glam, gva, grec, gD, &bar[0], d.kind & 16);
  uint32_t phase = 0;
  double acc = 0.0;
  T c0 = T(0), c1 = inf;  // forward: shp(r, .) of the current partition
  T x0 = T(0), x1 = inf;  // backward: shp(., T) of the partition above
  for (int ci = 0; ci < nch; ++ci) {
    const int b = ci & 1;
    const ChunkSpan sp = chunk_span<T, MODE>(d, grec, chunk_of(ci));
    if (ci + 1 < nch && lane == 0) {
      bulk_wait_read_all();  // the stores of chunk ci - 1 (same buffer as ci + 1) have read it
      chunk_issue(chunk_stage_at<T>(sb[b ^ 1]), chunk_span<T, MODE>(d, grec, chunk_of(ci + 1)), L, glam, gva, grec, gD,
                  &bar[b ^ 1], d.kind & 16);
    }
    const ChunkStage<T> st = chunk_stage_at<T>(sb[b]);
    mbar_wait(&bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const int h0 = sp.h0, h1 = sp.h1, r0 = sp.r0;
    if (active) {
      T *lam = st.lam + lane, *va = st.va + lane, *D = st.D + lane;
      T *m0c = REC ? m0g + (int64_t)h0 * L : nullptr;  // recorded min-marginals, chunk-relative
      T *m1c = REC ? m1g + (int64_t)h0 * L : nullptr;
      if (L == 32) {
        if (MODE == kForward)
          mask_forward_range<T, REC, 32>(h0, h1, K, chain, st.rec, 32, lam, va, D, r0, valid, omega, clamp, m0c, m1c,
                                         c0, c1, acc);
        else
          mask_backward_range<T, REC, 32>(h0, h1, K, chain, st.rec, 32, lam, va, D, r0, valid, omega, clamp, m0c,
                                          m1c, x0, x1, acc);
      } else {
        if (MODE == kForward)
          mask_forward_range<T, REC, 0>(h0, h1, K, chain, st.rec, L, lam, va, D, r0, valid, omega, clamp, m0c, m1c,
                                        c0, c1, acc);
        else
          mask_backward_range<T, REC, 0>(h0, h1, K, chain, st.rec, L, lam, va, D, r0, valid, omega, clamp, m0c, m1c,
                                         x0, x1, acc);
      }
    }
    fence_proxy_async();  // lanes' shared-memory writes -> visible to the TMA stores
    __syncwarp();
    if (lane == 0) {
      const uint32_t lb = (uint32_t)(h1 - h0) * L * sizeof(T);
      bulk_s2g(glam + (int64_t)h0 * L, st.lam, lb);
      bulk_s2g(gva + (int64_t)h0 * L, st.va, lb);
      bulk_s2g(gD + (int64_t)r0 * L, st.D, (uint32_t)(sp.rown - r0) * L * sizeof(T));  // the chunk's own partitions
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_read_all();  // shared memory must outlive the TMA stores' reads
  if (valid) acc += (double)(MODE == kForward ? c0 : x0);  // E^j = shp(r, T)
  acc = warp_sum(acc);
  if (lane == 0) a.lb_part[t] = acc;
}

template <typename T>
struct HopSet {
  int n0, n1, n2;   // P_h = [n0, n1), P_{h+1} = [n1, n2)
  uint32_t e0, e1;  // topology of the (up to) two nodes of P_h
  T l, av;          // lambda_h, avg_i (in va)
  T x0, x1;         // forward: shp(., T) of P_{h+1};  backward: shp(r, .) of P_h
};

template <typename T, int MODE>
__device__ __forceinline__ void load_hop(HopSet<T> &s, int h, int K, const int32_t *ho, const uint32_t *tp, int ts,
                                         int L, const T *lam, const T *va, const T *D) {
  const T inf = t_inf<T>();
  s.n0 = __ldg(ho + h);
  s.n1 = __ldg(ho + h + 1);
  s.n2 = h + 1 < K ? __ldg(ho + h + 2) : s.n1;
  s.e0 = __ldg(tp + s.n0 * ts);
  s.e1 = s.n1 - s.n0 > 1 ? __ldg(tp + (s.n0 + 1) * ts) : 0u;
  s.l = lam[h * L];
  s.av = va[h * L];
  if (MODE == kForward) {
    s.x0 = h + 1 < K ? D[s.n1 * L] : inf;
    s.x1 = (h + 1 < K && s.n2 - s.n1 > 1) ? D[(s.n1 + 1) * L] : inf;
  } else {
    s.x0 = D[s.n0 * L];
    s.x1 = s.n1 - s.n0 > 1 ? D[(s.n0 + 1) * L] : inf;
  }
}

template <typename T, int MODE, bool REC>
__global__ void __launch_bounds__(128) sweep_stream_kernel(const SweepArgs a) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= a.n_tiles) return;  // whole warps
  const TileDesc d = a.tiles[t];
  const int L = d.lanes, K = d.K;
  const bool valid = lane < d.n_lanes;
  double acc = 0.0;
  pdl_wait();
  if ((d.kind & 4) && lane < L) {
    // arc-mask tile: the same min-plus loops as the staged kernel, on global
    // memory (records are warp-uniform loads through L1)
    const HopRec<T> *rec = reinterpret_cast<const HopRec<T> *>(a.recs + 16 * (int64_t)d.rec_base);
    const int chain = ((d.kind & 8) ? 1 : 0) | ((d.kind & 16) ? 2 : 0);
    T *lam = reinterpret_cast<T *>(a.lambda) + d.slot_base + lane;
    T *va = reinterpret_cast<T *>(a.delta_out) + d.slot_base + lane;
    T *D = reinterpret_cast<T *>(a.dist) + d.dist_base + lane;
    T *m0g = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
    T *m1g = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
    const T omega = arg_omega<T>(a), clamp = arg_clamp<T>(a);
    if (L == 32) {
      acc = MODE == kForward ? mask_forward<T, true, REC, 32, 1>(K, chain, rec, 32, lam, va, SmemD<T, 1>{D, 32u}, valid,
                                                                 omega, clamp, m0g, m1g)
                             : mask_backward<T, true, REC, 32, 1>(K, chain, rec, 32, lam, va, SmemD<T, 1>{D, 32u}, valid,
                                                                  omega, clamp, m0g, m1g);
    } else {
      acc = MODE == kForward ? mask_forward<T, true, REC, 0, 1>(K, chain, rec, L, lam, va, SmemD<T, 1>{D, (uint32_t)L},
                                                                valid, omega, clamp, m0g, m1g)
                             : mask_backward<T, true, REC, 0, 1>(K, chain, rec, L, lam, va, SmemD<T, 1>{D, (uint32_t)L},
                                                                 valid, omega, clamp, m0g, m1g);
    }
  } else if (lane < L) {
    const int32_t *ho = a.hop_off + d.hop_base;
    const int ts = (d.kind & 1) ? L : 1;
    const uint32_t *tp = a.topo + d.topo_base + ((d.kind & 1) ? lane : 0);
    T *lam = reinterpret_cast<T *>(a.lambda) + d.slot_base + lane;
    T *va = reinterpret_cast<T *>(a.delta_out) + d.slot_base + lane;
    T *D = reinterpret_cast<T *>(a.dist) + d.dist_base + lane;
    T *m0g = REC ? reinterpret_cast<T *>(a.m0) + d.slot_base + lane : nullptr;
    T *m1g = REC ? reinterpret_cast<T *>(a.m1) + d.slot_base + lane : nullptr;
    const T inf = t_inf<T>();
    const T omega = arg_omega<T>(a), clamp = arg_clamp<T>(a);
    const int top = d.nodes;
    auto finish = [&](int h, T l, T av, T m0, T m1r) -> T {
      const T m1 = l + m1r;
      const T delta = mul_rn(omega, mm_difference(m1, m0, clamp));
      const T lam_new = add_rn(sub_rn(l, delta), av);
      if (valid) {
        lam[h * L] = lam_new;
        va[h * L] = delta;
        if (REC) {
          m0g[h * L] = m0;
          m1g[h * L] = m1;
        }
        acc += (double)fmin(delta, T(0));
      } else {
        va[h * L] = T(0);
      }
      return lam_new;
    };
    HopSet<T> s0, s1, s2;
    if (MODE == kForward) {
      load_hop<T, MODE>(s0, 0, K, ho, tp, ts, L, lam, va, D);
      if (K > 1) load_hop<T, MODE>(s1, 1, K, ho, tp, ts, L, lam, va, D);
      T c0 = T(0), c1 = inf;  // shp(r, .) of P_h
#pragma unroll 1
      for (int h = 0; h < K; ++h) {
        if (h + 2 < K) load_hop<T, MODE>(s2, h + 2, K, ho, tp, ts, L, lam, va, D);
        const int n0 = s0.n0, n1 = s0.n1;
        const int lo0 = (int)(s0.e0 & 0xFFFFu), hi0 = (int)(s0.e0 >> 16);
        D[n0 * L] = c0;  // keep shp(r, v) (P:315-316 reuse for the backward pass)
        T m0 = c0 + succ(lo0, n1, top, s0.x0, s0.x1), m1r = c0 + succ(hi0, n1, top, s0.x0, s0.x1);
        T nl0 = lo0 == n1 ? c0 : inf, nl1 = lo0 == n1 + 1 ? c0 : inf;
        T nh0 = hi0 == n1 ? c0 : inf, nh1 = hi0 == n1 + 1 ? c0 : inf;
        if (n1 - n0 > 1) {
          const int lo1 = (int)(s0.e1 & 0xFFFFu), hi1 = (int)(s0.e1 >> 16);
          D[(n0 + 1) * L] = c1;
          m0 = fmin(m0, c1 + succ(lo1, n1, top, s0.x0, s0.x1));
          m1r = fmin(m1r, c1 + succ(hi1, n1, top, s0.x0, s0.x1));
          if (lo1 == n1) nl0 = fmin(nl0, c1);
          if (lo1 == n1 + 1) nl1 = fmin(nl1, c1);
          if (hi1 == n1) nh0 = fmin(nh0, c1);
          if (hi1 == n1 + 1) nh1 = fmin(nh1, c1);
        }
        const T lam_new = finish(h, s0.l, s0.av, m0, m1r);
        if (h == K - 1) {
          if (valid) acc += (double)fmin(m0, lam_new + m1r);  // E^j at the updated lambda
        } else {
          c0 = fmin(nl0, nh0 + lam_new);  // A4
          c1 = fmin(nl1, nh1 + lam_new);
        }
        s0 = s1;
        s1 = s2;
      }
    } else {
      load_hop<T, MODE>(s0, K - 1, K, ho, tp, ts, L, lam, va, D);
      if (K > 1) load_hop<T, MODE>(s1, K - 2, K, ho, tp, ts, L, lam, va, D);
      T ct0 = inf, ct1 = inf;  // shp(., T) of P_{h+1}
#pragma unroll 1
      for (int h = K - 1; h >= 0; --h) {
        if (h >= 2) load_hop<T, MODE>(s2, h - 2, K, ho, tp, ts, L, lam, va, D);
        const int n0 = s0.n0, n1 = s0.n1;
        const int lo0 = (int)(s0.e0 & 0xFFFFu), hi0 = (int)(s0.e0 >> 16);
        const T a0 = succ(lo0, n1, top, ct0, ct1), b0 = succ(hi0, n1, top, ct0, ct1);
        T m0 = s0.x0 + a0, m1r = s0.x0 + b0;
        T a1 = inf, b1 = inf;
        const bool two = n1 - n0 > 1;
        if (two) {
          const int lo1 = (int)(s0.e1 & 0xFFFFu), hi1 = (int)(s0.e1 >> 16);
          a1 = succ(lo1, n1, top, ct0, ct1);
          b1 = succ(hi1, n1, top, ct0, ct1);
          m0 = fmin(m0, s0.x1 + a1);
          m1r = fmin(m1r, s0.x1 + b1);
        }
        const T lam_new = finish(h, s0.l, s0.av, m0, m1r);
        ct0 = fmin(a0, lam_new + b0);  // shp(v, T) with the updated lambda_h
        ct1 = two ? fmin(a1, lam_new + b1) : inf;
        D[n0 * L] = ct0;
        if (two) D[(n0 + 1) * L] = ct1;
        s0 = s1;
        s1 = s2;
      }
      if (valid) acc += (double)ct0;  // E^j = shp(r, T)
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) a.lb_part[t] = acc;
}

template <typename T>
__device__ __forceinline__ void ell_store(T *out, int2 p, T x, T y) {
  if (p.x < 0) return;
  if (p.y >= 0) {
    const T v = (x + y) / T(2);
    out[p.x] = v;
    out[p.y] = v;
  } else {
    out[p.x] = x;  // |J_i| = 1: the average is the value itself
  }
}

// load through the read-only path (kernel-lifetime constant data) or a plain
// load (data written earlier in the same kernel: the fused small-problem path)
template <bool NC, typename V>
__device__ __forceinline__ V ld(const V *p) {
  if (NC) return __ldg(p);
  return *p;
}

// Deferred averaging (A1).  avg_i = (sum over the slots of i, in
// ascending j, of delta_bar) / |J_i| is written into every slot of i of the
// OTHER delta buffer, where the next sweep reads it (and overwrites it with its
// own delta).  Three sections of whole warps: ELL pairs (|J_i| <= 2, four
// variables per thread), ELL-4 quads (|J_i| = 3, 4), CSR groups (the rest and
// every exchanged variable).  avg_kernel's thread 0 also resets the sweep's
// tile counter.  (Measured slower: a slot-parallel ELL section -- every slot
// gathering its partner's delta_bar, coalesced writes -- 1.5-2.3x, the
// partner gathers lose the locality of the first slot; consecutive instead of
// strided variables per thread (FDOG_AVG_LOCAL=1) 1.1-1.4x; pairs re-ordered
// by the 2^b-slot bucket of their smaller slot, then the larger, b = 4..14:
// within 1 %.)
// NC: delta_bar is read-only for the kernel's lifetime (the standalone kernel)
// V: ELL variables per thread (tid, tid + N, ..., tid + (V-1) N: every load of
// a warp stays coalesced, all 2V gathers in flight before the first use)
// CSR part: a group of G lanes per variable (gt = thread index inside the part);
// lane j sums slots j, j+G, ... in order, then a fixed-shape shuffle tree
// combines the lanes (deterministic)
template <typename T, bool NC, bool PRE = false>
__device__ __forceinline__ void avg_csr(const AvgArgs &a, const int gt) {
  const T *__restrict__ db = reinterpret_cast<const T *>(a.delta_bar);
  T *__restrict__ out = reinterpret_cast<T *>(a.avg_slot);
  const int G = a.group;
  const int q = gt / G, j = gt % G;
  const bool on = q < a.n;
  T *__restrict__ xbuf = reinterpret_cast<T *>(a.xbuf);
  int64_t p0 = 0, p1 = 0;
  if (on) {
    p0 = __ldg(a.var_ptr + q);
    p1 = __ldg(a.var_ptr + q + 1);
  }
  if (PRE) pdl_wait();
  // lane j sums slots p0 + j, p0 + j + G, ... in ascending order; four at a
  // time, all index loads and then all gathers issued before the adds (two
  // dependent memory round trips per four slots instead of two per slot)
  T s = T(0);
  for (int64_t base = p0 + j; base < p1; base += 4 * (int64_t)G) {
    int32_t q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t p = base + (int64_t)u * G;
      q[u] = p < p1 ? __ldg(a.var_slots + p) : -1;
    }
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = q[u] >= 0 ? ld<NC>(db + q[u]) : T(0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (q[u] >= 0) s += v[u];
  }
  // the group is G consecutive lanes of one warp (G divides 32, the CSR part
  // starts at a multiple of 32 threads: the sections are rounded up)
  for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
  if (!on) return;
  const int x = a.var_xidx ? __ldg(a.var_xidx + q) : -1;
  if (x >= 0) {
    if (j == 0) xbuf[x] = s;
    return;
  }
  const T v = s / T(__ldg(a.deg_l + q));
  for (int64_t p = p0 + j; p < p1; p += G) out[__ldg(a.var_slots + p)] = v;
}

// threads of the CSR part (whole warps)
__host__ __device__ __forceinline__ int64_t avg_csr_threads(const AvgArgs &a) {
  return ((int64_t)a.n * a.group + 31) & ~(int64_t)31;
}

// threads of the ELL-D part: one per variable, each group in whole warps
__host__ __device__ __forceinline__ int64_t avg_elld_threads(const AvgArgs &a) {
  int64_t t = 0;
  for (int g = 0; g < a.n_elld_g; ++g) t += ((int64_t)a.elld_n[g] + 31) & ~(int64_t)31;
  return t;
}

// ELL-D part: variable v of group g (degree d) sums its d slots in ascending j
// (k ascending), eight index loads and eight gathers in flight at a time, then
// writes the average into every slot.  Column-major indices: the k-th index
// loads of a warp are coalesced, and so are its gathers and scatters wherever
// neighbouring variables have neighbouring k-th slots (MRF pixels, Potts edges).
template <typename T, bool NC, bool PRE>
__device__ __forceinline__ void avg_elld(const AvgArgs &a, int64_t t) {
  int g = 0;
  int64_t base = 0;
  for (; g < a.n_elld_g; ++g) {
    const int64_t w = ((int64_t)a.elld_n[g] + 31) & ~(int64_t)31;
    if (t < base + w) break;
    base += w;
  }
  if (g >= a.n_elld_g) return;
  const int64_t v = t - base;
  const int n = a.elld_n[g], d = a.elld_d[g];
  if (PRE) pdl_wait();
  if (v >= n) return;
  const int32_t *ix = a.elld + a.elld_off[g] + v;
  const T *__restrict__ db = reinterpret_cast<const T *>(a.delta_bar);
  T *__restrict__ out = reinterpret_cast<T *>(a.avg_slot);
  T s = T(0);
  for (int k0 = 0; k0 < d; k0 += 8) {
    int32_t q[8];
    T x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = k0 + u < d ? __ldg(ix + (int64_t)(k0 + u) * n) : -1;
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = q[u] >= 0 ? ld<NC>(db + q[u]) : T(0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (q[u] >= 0) s += x[u];
  }
  const T avg = s / T(d);
  for (int k = 0; k < d; ++k) out[__ldg(ix + (int64_t)k * n)] = avg;
}

// PRE: the standalone kernel launched behind a sweep (PDL): the constant index
// loads of a thread are issued before griddepcontrol.wait, the gathers of
// delta_bar after it
template <typename T, bool NC, int V = 4, bool PRE = false>
__device__ __forceinline__ void avg_body(const AvgArgs &a, int tid) {
  const T *__restrict__ db = reinterpret_cast<const T *>(a.delta_bar);
  T *__restrict__ out = reinterpret_cast<T *>(a.avg_slot);
  // csr_first: the CSR part (the longest dependent chains: offsets, slots,
  // gathers, shuffle tree, slots again, stores) takes the lowest block
  // indices, so it is dispatched in the first wave instead of forming the tail
  if (a.csr_first) {
    const int64_t nc = avg_csr_threads(a);
    if (tid < nc) {
      avg_csr<T, NC, PRE>(a, tid);
      return;
    }
    tid -= (int)nc;
  }
  // ELL part: four variables per thread (tid, tid + N, tid + 2N, tid + 3N, so
  // every load of a warp stays coalesced), all eight gathers issued before use
  const int n_ell_thr = (((a.n_ell + V - 1) / V) + 31) & ~31;  // whole warps
  if (tid < n_ell_thr) {
    int2 p[V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int q = a.ell_local ? tid * V + u : tid + u * n_ell_thr;
      p[u] = q < a.n_ell ? __ldg(a.ell + q) : make_int2(-1, -1);
    }
    if (PRE) pdl_wait();
    T x[V], y[V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      x[u] = p[u].x >= 0 ? ld<NC>(db + p[u].x) : T(0);
      y[u] = p[u].y >= 0 ? ld<NC>(db + p[u].y) : T(0);
    }
#pragma unroll
    for (int u = 0; u < V; ++u) ell_store(out, p[u], x[u], y[u]);
    return;
  }
  // ELL-4 part (|J_i| = 3 or 4): two variables per thread (q, q + N; loads of
  // a warp stay coalesced), slot quads inline, all gathers in flight before
  // the sums, each summed in ascending j
  const int n_ell4_thr = (((a.n_ell4 + 1) >> 1) + 31) & ~31;
  if (tid < n_ell_thr + n_ell4_thr) {
    const int q = tid - n_ell_thr;
    int4 p[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int qq = a.ell_local ? q * 2 + u : q + u * n_ell4_thr;
      p[u] = qq < a.n_ell4 ? __ldg(a.ell4 + qq) : make_int4(-1, -1, -1, -1);
    }
    if (PRE) pdl_wait();
    T x[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      x[u][0] = p[u].x >= 0 ? ld<NC>(db + p[u].x) : T(0);
      x[u][1] = p[u].x >= 0 ? ld<NC>(db + p[u].y) : T(0);
      x[u][2] = p[u].x >= 0 ? ld<NC>(db + p[u].z) : T(0);
      x[u][3] = p[u].w >= 0 ? ld<NC>(db + p[u].w) : T(0);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (p[u].x < 0) continue;
      T s = x[u][0] + x[u][1];
      s += x[u][2];
      if (p[u].w >= 0) s += x[u][3];
      const T v = s / T(p[u].w >= 0 ? 4 : 3);
      out[p[u].x] = v;
      out[p[u].y] = v;
      out[p[u].z] = v;
      if (p[u].w >= 0) out[p[u].w] = v;
    }
    return;
  }
  const int64_t n_elld_thr = avg_elld_threads(a);
  if (tid < n_ell_thr + n_ell4_thr + n_elld_thr) {
    avg_elld<T, NC, PRE>(a, tid - n_ell_thr - n_ell4_thr);
    return;
  }
  if (a.csr_first) return;  // (past the last section: padding threads)
  avg_csr<T, NC, PRE>(a, tid - n_ell_thr - n_ell4_thr - (int)n_elld_thr);
}

template <typename T>
// (48 registers, 5 CTAs per SM: left unbounded ptxas chose 40 and spilled;
// measured, same box: Potts-cut averaging 94.9 -> 75.1 us, MRF-LP 43.2 ->
// 36.3, cell tracking and GM equal; 56 registers (4 CTAs): 84.2 / 40.4)
__global__ void __launch_bounds__(256, 5) avg_kernel(const AvgArgs a) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) {
    pdl_wait();  // the sweep before has finished with the counter
    *a.tile_counter = 0u;
  }
  if (a.ell_v == 8) avg_body<T, true, 8, true>(a, tid);
  else if (a.ell_v == 2) avg_body<T, true, 2, true>(a, tid);
  else if (a.ell_v == 1) avg_body<T, true, 1, true>(a, tid);
  else avg_body<T, true, 4, true>(a, tid);
}

// threads the averaging needs (whole warps per section)
__host__ __device__ __forceinline__ int64_t avg_threads(const AvgArgs &a) {
  const int v = (a.ell_v == 8 || a.ell_v == 2 || a.ell_v == 1) ? a.ell_v : 4;
  return (int64_t)((((a.n_ell + v - 1) / v) + 31) & ~31) + (int64_t)((((a.n_ell4 + 1) >> 1) + 31) & ~31) +
         avg_elld_threads(a) + avg_csr_threads(a);
}

// ---------------------------------------------------------------------------
// Small problems (every tile narrow, few tiles): one CTA runs n iterations in a
// single launch -- averaging and sweep phases separated by __syncthreads
// instead of kernel boundaries (latency path, e.g. BASELINE configs[0]).
// Same device code as the standalone kernels; data stays in global memory
// (L1/L2 resident at these sizes).  cur0 = parity of delta_bar on entry.
template <typename T, bool REC>
__global__ void __launch_bounds__(1024) fused_small_kernel(const SweepArgs sa, const AvgArgs aa, int32_t n_iter,
                                                           int64_t n_slots, int64_t n_dist, int32_t resident) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T *const g_dbar = const_cast<T *>(reinterpret_cast<const T *>(aa.delta_bar));  // delta[cur] on entry
  T *const g_va = reinterpret_cast<T *>(aa.avg_slot);
  T *const g_lambda = reinterpret_cast<T *>(sa.lambda);
  T *const g_dist = reinterpret_cast<T *>(sa.dist);
  T *dbar = g_dbar, *va_all = g_va, *lambda = g_lambda, *gdist = g_dist;
  const T omega = arg_omega<T>(sa), clamp = arg_clamp<T>(sa);
  extern __shared__ __align__(16) unsigned char fsm[];
  pdl_wait();
  if (resident) {
    // the whole mutable state (lambda, both delta buffers, distances) fits in
    // shared memory: same absolute indices, shared-memory latency per hop
    T *sl = reinterpret_cast<T *>(fsm), *s0 = sl + n_slots, *s1 = s0 + n_slots, *sd = s1 + n_slots;
    for (int64_t i = threadIdx.x; i < n_slots; i += blockDim.x) {
      sl[i] = g_lambda[i];
      s0[i] = g_dbar[i];
      s1[i] = g_va[i];
    }
    for (int64_t i = threadIdx.x; i < n_dist; i += blockDim.x) sd[i] = g_dist[i];
    __syncthreads();
    lambda = sl;
    dbar = s0;
    va_all = s1;
    gdist = sd;
  }
  AvgArgs a4 = aa;
  a4.ell_v = 4;  // avg_body's default V below
  const int64_t na = avg_threads(a4);
  for (int it = 0; it < 2 * n_iter; ++it) {
    AvgArgs a = a4;
    a.delta_bar = dbar;
    a.avg_slot = va_all;
    for (int64_t base = 0; base < na; base += blockDim.x) avg_body<T, false>(a, (int)(base + threadIdx.x));
    __syncthreads();
    for (int t = warp; t < sa.n_tiles; t += nw) {
      const TileDesc d = sa.tiles[t];
      const int L = d.lanes;
      const bool valid = lane < d.n_lanes;
      double acc = 0.0;
      if (lane < L) {
        const int64_t sb = d.slot_base + lane;
        const uint32_t *tp = (d.kind & 1) ? sa.topo + d.topo_base + lane : sa.topo + d.topo_base;
        const int ts = (d.kind & 1) ? L : 1;
        T *m0p = REC ? reinterpret_cast<T *>(sa.m0) + sb : nullptr;
        T *m1p = REC ? reinterpret_cast<T *>(sa.m1) + sb : nullptr;
        if (it % 2 == 0)
          acc = process_bdd_w2<T, kForward, REC, 0>(d.K, sa.hop_off + d.hop_base, tp, ts, L, lambda + sb, va_all + sb,
                                                    gdist + d.dist_base + lane, valid, omega, clamp, m0p, m1p);
        else
          acc = process_bdd_w2<T, kBackward, REC, 0>(d.K, sa.hop_off + d.hop_base, tp, ts, L, lambda + sb, va_all + sb,
                                                     gdist + d.dist_base + lane, valid, omega, clamp, m0p, m1p);
      }
      acc = warp_sum(acc);
      if (lane == 0) sa.lb_part[t] = acc;
    }
    __syncthreads();
    T *const t = dbar;  // mbar <- m
    dbar = va_all;
    va_all = t;
  }
  if (resident) {  // an even number of swaps: dbar / va_all are s0 / s1 again
    for (int64_t i = threadIdx.x; i < n_slots; i += blockDim.x) {
      g_lambda[i] = lambda[i];
      g_dbar[i] = dbar[i];
      g_va[i] = va_all[i];
    }
    for (int64_t i = threadIdx.x; i < n_dist; i += blockDim.x) g_dist[i] = gdist[i];
  }
}

// Shared variables after the NCCL exchange: average and scatter into the local slots.
// ---------------------------------------------------------------------------
// Alg. "Perturbation Primal Rounding", one kernel per step.
// Thread per variable (ELL part: slot pair inline; CSR part: slot list).  The
// signs of m1 - m0 are those of delta_bar = omega * clamp(m1 - m0) of the last
// pass.  mode 0: classify -> x (1 iff m1 < m0 in every subproblem) and the
// count of undecided variables (reading R1); mode 1: perturbation of lambda.
__device__ __forceinline__ double primal_uniform(uint64_t seed, int64_t round, int64_t i) {
  // splitmix64(seed, round, i) -> [0, 1); the oracle implements the same generator
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + (uint64_t)round * 0xBF58476D1CE4E5B9ull +
               (uint64_t)i * 0x94D049BB133111EBull + 1ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

template <typename T>
__global__ void __launch_bounds__(256) primal_kernel(const PrimalArgs a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  int n_elld = 0;
  for (int g = 0; g < a.n_elld_g; ++g) n_elld += a.elld_n[g];
  if (q >= a.n_ell + a.n_ell4 + a.n_csr + n_elld) return;
  const T *__restrict__ db = reinterpret_cast<const T *>(a.delta_bar);
  int i, sl[4] = {-1, -1, -1, -1};
  int64_t p0 = 0, p1 = 0, deg;
  const int kind = q < a.n_ell ? 0 : q < a.n_ell + a.n_ell4 ? 1 : q < a.n_ell + a.n_ell4 + a.n_csr ? 2 : 3;
  const int32_t *ed = nullptr;  // ELL-D: slot k at ed[k * en]
  int64_t en = 0;
  if (kind == 0) {
    const int2 pr = a.ell[q];
    i = a.ell_var[q];
    sl[0] = pr.x;
    sl[1] = pr.y;
    deg = pr.y >= 0 ? 2 : 1;
  } else if (kind == 1) {
    const int4 pr = a.ell4[q - a.n_ell];
    i = a.ell4_var[q - a.n_ell];
    sl[0] = pr.x;
    sl[1] = pr.y;
    sl[2] = pr.z;
    sl[3] = pr.w;
    deg = pr.w >= 0 ? 4 : 3;
  } else if (kind == 2) {
    const int c = q - a.n_ell - a.n_ell4;
    i = a.csr_var[c];
    p0 = a.var_ptr[c];
    p1 = a.var_ptr[c + 1];
    deg = p1 - p0;
  } else {
    int v = q - a.n_ell - a.n_ell4 - a.n_csr, g = 0;
    i = a.elld_var[v];
    while (v >= a.elld_n[g]) v -= a.elld_n[g++];
    ed = a.elld + a.elld_off[g] + v;
    en = a.elld_n[g];
    deg = a.elld_d[g];
  }
  auto slot_at = [&](int64_t u) -> int { return kind < 2 ? sl[u] : kind == 2 ? a.var_slots[p0 + u] : ed[u * en]; };
  bool pos = true, neg = true, zero = true;
  double dsum = 0.0;  // sign of d_i = sum_j (m1 - m0) = sign of sum_j delta_bar (omega > 0)
  for (int64_t u = 0; u < deg; ++u) {
    const T v = db[slot_at(u)];
    pos = pos && v > T(0);
    neg = neg && v < T(0);
    zero = zero && v == T(0);
    dsum += (double)v;
  }
  if (a.mode == 0) {
    a.x[i] = neg ? 1 : 0;
    if (!(pos || neg)) atomicAdd(a.undecided, 1ull);
    return;
  }
  const double delta = a.delta;
  const double r = delta * (2.0 * primal_uniform(a.seed, a.round, i) - 1.0);  // r ~ U[-delta, delta]
  double step;
  if (pos) step = delta;
  else if (neg) step = -delta;
  else if (zero) step = r * delta;
  else step = (double)((dsum > 0) - (dsum < 0)) * fabs(r) * delta;
  T *__restrict__ lam = reinterpret_cast<T *>(a.lambda);
  for (int64_t u = 0; u < deg; ++u) {
    const int s = slot_at(u);
    lam[s] = (T)((double)lam[s] + step);
  }
}

template <typename T>
__global__ void avg_finish_kernel(const AvgArgs a, int32_t n_shared, const int32_t *__restrict__ xlocal,
                                  const int32_t *__restrict__ deg_x) {
  const T *__restrict__ xbuf = reinterpret_cast<const T *>(a.xbuf);
  T *__restrict__ out = reinterpret_cast<T *>(a.avg_slot);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_shared; q += gridDim.x * blockDim.x) {
    const int l = xlocal[q];
    if (l < 0) continue;  // exchanged variable this rank does not hold
    const T v = xbuf[q] / T(deg_x[q]);
    for (int64_t p = a.var_ptr[l]; p < a.var_ptr[l + 1]; ++p) out[a.var_slots[p]] = v;
  }
}

// ---- peer-memory exchange (world > 1, fdog_set_peer_regions) ---------------
// Every rank's exchange region (its own memory; the peers' regions mapped into
// this process by CUDA IPC or, in one process, plain device pointers):
//   [0] pass counter, [4] error word, [kRegionBuf + b * buf_stride] partial
//   sums of pass parity b.  Per pass: averaging writes this rank's partials
//   into its buffer of the pass parity; peer_signal_kernel publishes them
//   (system-scope release of counter + 1); peer_finish_kernel waits until every
//   peer's counter has reached this rank's, then sums the peers' partials over
//   NVLink in rank order 0..W-1 (identical on every rank: the ranks agree bit
//   for bit) and scatters the averages into the local slots.  Two buffers:
//   a rank rewrites parity b only two passes later, after every peer has
//   published the pass in between, i.e. finished reading this one.
__global__ void peer_signal_kernel(unsigned *counter) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__global__ void peer_finish_kernel(const AvgArgs a, int32_t n_shared, const int32_t *__restrict__ xlocal,
                                   const int32_t *__restrict__ deg_x, const PeerArgs pa) {
  T *__restrict__ out = reinterpret_cast<T *>(a.avg_slot);
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const unsigned target = *reinterpret_cast<volatile const unsigned *>(pa.region[pa.rank]);
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int good = 1;
    for (int k = 0; k < pa.world && good; ++k) {
      const unsigned *c = reinterpret_cast<const unsigned *>(pa.region[k]);
      while (ld_acquire_sys(c) < target) {
        __nanosleep(256);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > pa.timeout_ns) {  // a peer never published: report, do not hang
          atomicExch(reinterpret_cast<unsigned *>(const_cast<unsigned char *>(pa.region[pa.rank]) + 4), 1u);
          good = 0;
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();
  if (!ok) return;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_shared; q += gridDim.x * blockDim.x) {
    const int l = xlocal[q];
    if (l < 0) continue;  // exchanged variable this rank does not hold
    T sum = T(0);
    for (int k = 0; k < pa.world; ++k) {
      const T *b = reinterpret_cast<const T *>(pa.region[k] + pa.buf_off);
      sum += __ldcv(b + q);  // (no stale L1 line of the peer's memory)
    }
    const T v = sum / T(deg_x[q]);
    for (int64_t p = a.var_ptr[l]; p < a.var_ptr[l + 1]; ++p) out[a.var_slots[p]] = v;
  }
}

static int grid_for(int64_t n, int block);

int launch_peer_signal(const PeerArgs &pa, void *stream) {
  peer_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<unsigned *>(const_cast<unsigned char *>(pa.region[pa.rank])));
  return (int)cudaGetLastError();
}

int launch_peer_finish(int precision, const AvgArgs &a, int32_t n_shared, const int32_t *xlocal,
                       const int32_t *deg_x, const PeerArgs &pa, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int block = 256, grid = grid_for(std::max(n_shared, 1), block);
  if (precision == 64)
    peer_finish_kernel<double><<<grid, block, 0, st>>>(a, n_shared, xlocal, deg_x, pa);
  else
    peer_finish_kernel<float><<<grid, block, 0, st>>>(a, n_shared, xlocal, deg_x, pa);
  return (int)cudaGetLastError();
}

template <typename T>
__global__ void add_deferred_kernel(int64_t n, T *__restrict__ lambda, T *__restrict__ delta) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    lambda[q] += delta[q];
    delta[q] = T(0);
  }
}

// The outstanding deferred term of the lifted bound (A7), sum over a tile's
// slots of min(delta_bar, 0), added to the tile's partial after an energy
// sweep (fdog_set_state with a non-zero delta_bar).  One warp per tile;
// padding slots hold 0.
template <typename T>
__global__ void __launch_bounds__(256) lb_deferred_kernel(const TileDesc *__restrict__ tiles, int32_t n_tiles,
                                                          const T *__restrict__ delta, double *__restrict__ lb_part) {
  const int lane = threadIdx.x & 31;
  const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (t >= n_tiles) return;
  const TileDesc d = tiles[t];
  double acc = 0.0;
  for (int64_t q = lane; q < (int64_t)d.K * d.lanes; q += 32) acc += (double)fmin(delta[d.slot_base + q], T(0));
  acc = warp_sum(acc);
  if (lane == 0) lb_part[t] += acc;
}

// ---------------------------------------------------------------------------
// Non-deferred min-marginal averaging (oracle_pass_seq).  The
// variables of a pass are ordered by a level schedule (solver.cpp): a
// variable's level is one more than the largest level of its predecessor in
// any of its BDDs, so variables of one level share no BDD and can be updated
// together -- the same result as visiting them one by one in ascending
// (descending) index.  Thread q handles one variable: the min-marginals in
// every j in J_i (store-design distances in global memory), their
// average, the dual update, and the advance of each BDD by one partition
// (forward: shp(r, .) of P_{h+1}, P:319-324 with A4; backward: shp(., T) of
// P_h).  Generic in the partition width.
struct SeqLoc {
  int32_t h, lane, L, K, nodes;
  const int32_t *ho;   // partition offsets of the tile
  const uint32_t *tp;  // topology of node n at tp[n * ts]
  int32_t ts;
  int64_t dbase;       // distance of node n: dist[dbase + n * L]
};

__device__ __forceinline__ SeqLoc seq_locate(const SeqArgs &a, int32_t ds, int32_t &t) {
  t = __ldg(a.slot_tile + ds);
  const TileDesc &d = a.tiles[t];
  SeqLoc l;
  l.L = d.lanes;
  const int64_t off = ds - d.slot_base;
  l.h = (int32_t)(off / l.L);
  l.lane = (int32_t)(off - (int64_t)l.h * l.L);
  l.K = d.K;
  l.nodes = d.nodes;
  l.ho = a.hop_off + d.hop_base;
  l.ts = (d.kind & 1) ? l.L : 1;
  l.tp = a.topo + d.topo_base + ((d.kind & 1) ? l.lane : 0);
  l.dbase = d.dist_base + l.lane;
  return l;
}

// one warp per variable, lane k handles slots k, k + 32, ... of it (every slot
// of a high-degree variable in parallel); the sum over J_i is accumulated in
// ascending j by one lane (shuffles), as the oracle does
// (Measured slower: the whole pass as one cooperative launch with a grid
// barrier between levels, 148-592 CTAs of 16 warps looping over a level's
// variables -- GM 7.7-8.6 ms per iteration against 5.4 for the CUDA graph of
// per-level launches, one warp per variable.)
template <typename T, bool REC>
__global__ void __launch_bounds__(128) seq_level_kernel(const SeqArgs a, int64_t q0, int64_t q1) {
  const int64_t q = q0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= q1) return;  // whole warps
  T *__restrict__ lam = reinterpret_cast<T *>(a.lambda);
  T *__restrict__ D = reinterpret_cast<T *>(a.dist);
  T *__restrict__ dl = reinterpret_cast<T *>(a.delta);
  const T omega = arg_omega<T>(a), clamp = arg_clamp<T>(a), inf = t_inf<T>();
  const int64_t p0 = a.ptr[q], p1 = a.ptr[q + 1];
  // min-marginals of the variable in every j in J_i
  T sum = T(0);
  for (int64_t c0 = p0; c0 < p1; c0 += 32) {
    const int64_t p = c0 + lane;
    T delta = T(0);
    if (p < p1) {
      const int32_t ds = a.slots[p];
      int32_t t;
      const SeqLoc l = seq_locate(a, ds, t);
      const int n0 = l.ho[l.h], n1 = l.ho[l.h + 1];
      if (a.forward && l.h == 0) D[l.dbase] = T(0);  // shp(r, r)
      T m0 = inf, m1r = inf;
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = l.tp[(int64_t)n * l.ts];
        const T c = D[l.dbase + (int64_t)n * l.L];
        m0 = fmin(m0, c + D[l.dbase + (int64_t)(e & 0xFFFFu) * l.L]);
        m1r = fmin(m1r, c + D[l.dbase + (int64_t)(e >> 16) * l.L]);
      }
      const T m1 = lam[ds] + m1r;
      delta = mul_rn(omega, mm_difference(m1, m0, clamp));
      dl[ds] = delta;
      if (REC) {
        reinterpret_cast<T *>(a.m0)[ds] = m0;
        reinterpret_cast<T *>(a.m1)[ds] = m1;
      }
    }
    const int cnt = p1 - c0 < 32 ? (int)(p1 - c0) : 32;
    for (int k = 0; k < cnt; ++k) sum += __shfl_sync(0xffffffffu, delta, k);  // ascending j
  }
  const T avg = sum / T(p1 - p0);
  // update every slot, then advance its BDD by one partition
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    const int32_t ds = a.slots[p];
    int32_t t;
    const SeqLoc l = seq_locate(a, ds, t);
    const T lam_new = add_rn(sub_rn(lam[ds], dl[ds]), avg);
    lam[ds] = lam_new;
    const int n0 = l.ho[l.h], n1 = l.ho[l.h + 1];
    if (a.forward) {
      if (l.h + 1 < l.K) {
        const int n2 = l.ho[l.h + 2];
        for (int v = n1; v < n2; ++v) {
          T best = inf;
          for (int n = n0; n < n1; ++n) {
            const uint32_t e = l.tp[(int64_t)n * l.ts];
            const T c = D[l.dbase + (int64_t)n * l.L];
            if ((int)(e & 0xFFFFu) == v) best = fmin(best, c);
            if ((int)(e >> 16) == v) best = fmin(best, c + lam_new);
          }
          D[l.dbase + (int64_t)v * l.L] = best;
        }
      } else {
        // last partition: E^j = shp(r, T) at the updated lambda
        T e_j = inf;
        for (int n = n0; n < n1; ++n) {
          const uint32_t e = l.tp[(int64_t)n * l.ts];
          const T c = D[l.dbase + (int64_t)n * l.L];
          e_j = fmin(e_j, fmin(c + D[l.dbase + (int64_t)(e & 0xFFFFu) * l.L],
                               c + lam_new + D[l.dbase + (int64_t)(e >> 16) * l.L]));
        }
        a.e_lane[(int64_t)t * kMaxTileRows + l.lane] = (double)e_j;
      }
    } else {
      for (int n = n0; n < n1; ++n) {
        const uint32_t e = l.tp[(int64_t)n * l.ts];
        D[l.dbase + (int64_t)n * l.L] = fmin(D[l.dbase + (int64_t)(e & 0xFFFFu) * l.L],
                                             lam_new + D[l.dbase + (int64_t)(e >> 16) * l.L]);
      }
      if (l.h == 0) a.e_lane[(int64_t)t * kMaxTileRows + l.lane] = (double)D[l.dbase];  // E^j = shp(r, T)
    }
  }
}

__global__ void __launch_bounds__(256) seq_bound_kernel(const TileDesc *tiles, int32_t n_tiles,
                                                        const double *e_lane, double *lb_part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int nl = tiles[t].n_lanes;
  double s = 0.0;
  for (int l = 0; l < nl; ++l) s += e_lane[(int64_t)t * kMaxTileRows + l];
  lb_part[t] = s;
}

template <typename T>
__device__ __forceinline__ void dist_dp_row(const SeqArgs &a, const TileDesc &d, const int lane, const int L,
                                            const int K, const int32_t forward);

// one thread per (tile, lane): the store-design distances from the current lambda
template <typename T>
__global__ void __launch_bounds__(256) dist_dp_kernel(const SeqArgs a, int32_t n_tiles, int32_t forward) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int32_t t = (int32_t)(g >> 5), lane = (int32_t)(g & 31);
  if (t >= n_tiles) return;
  const TileDesc &d = a.tiles[t];
  const int L = d.lanes, K = d.K;
  for (int l = lane; l < L; l += 32)  // (tiles of 64 / 128 rows: several rows per thread)
    dist_dp_row<T>(a, d, l, L, K, forward);
}

template <typename T>
__device__ __forceinline__ void dist_dp_row(const SeqArgs &a, const TileDesc &d, const int lane, const int L,
                                            const int K, const int32_t forward) {
  const int32_t *ho = a.hop_off + d.hop_base;
  const int ts = (d.kind & 1) ? L : 1;
  const uint32_t *tp = a.topo + d.topo_base + ((d.kind & 1) ? lane : 0);
  T *D = reinterpret_cast<T *>(a.dist) + d.dist_base + lane;
  const T *lam = reinterpret_cast<const T *>(a.lambda) + d.slot_base + lane;
  const T inf = t_inf<T>();
  if (!forward) {  // shp(v, T)
    for (int h = K - 1; h >= 0; --h) {
      const T l = lam[(int64_t)h * L];
      for (int n = ho[h]; n < ho[h + 1]; ++n) {
        const uint32_t e = tp[(int64_t)n * ts];
        D[(int64_t)n * L] = fmin(D[(int64_t)(e & 0xFFFFu) * L], l + D[(int64_t)(e >> 16) * L]);
      }
    }
  } else {  // shp(r, v), P:319-324 (A4)
    D[0] = T(0);
    for (int h = 0; h + 1 < K; ++h) {
      const T l = lam[(int64_t)h * L];
      for (int v = ho[h + 1]; v < ho[h + 2]; ++v) {
        T best = inf;
        for (int n = ho[h]; n < ho[h + 1]; ++n) {
          const uint32_t e = tp[(int64_t)n * ts];
          const T c = D[(int64_t)n * L];
          if ((int)(e & 0xFFFFu) == v) best = fmin(best, c);
          if ((int)(e >> 16) == v) best = fmin(best, c + l);
        }
        D[(int64_t)v * L] = best;
      }
    }
  }
}

// ---------------------------------------------------------------- launchers

template <typename T, bool RC, int RW, bool TM = false>
static const void *sweep_fn_rw(int mode, bool rec) {
  if (mode == kForward)
    return rec ? (const void *)sweep_kernel<T, kForward, true, RC, RW, TM>
               : (const void *)sweep_kernel<T, kForward, false, RC, RW, TM>;
  if (mode == kBackward)
    return rec ? (const void *)sweep_kernel<T, kBackward, true, RC, RW, TM>
               : (const void *)sweep_kernel<T, kBackward, false, RC, RW, TM>;
  if (mode == kCfr) return RC ? nullptr : (const void *)sweep_kernel<T, kCfr, false, false, RW, false>;
  return (const void *)sweep_kernel<T, kEnergy, false, RC, RW, TM>;
}

// rw: most rows per lane; rw == 0: the TMEM variant (fp32 recompute design)
template <typename T, bool RC>
static const void *sweep_fn(int mode, bool rec, int rw) {
  if constexpr (RC && std::is_same<T, float>::value)
    if (rw == 0) return sweep_fn_rw<T, true, 1, true>(mode, rec);
  if constexpr (sizeof(T) == 4)  // (fp64 plans stop at 2 rows per lane)
    if (rw >= 4) return sweep_fn_rw<T, RC, 4>(mode, rec);
  if (rw >= 2) return sweep_fn_rw<T, RC, 2>(mode, rec);
  return sweep_fn_rw<T, RC, 1>(mode, rec);
}

static const void *sweep_ptr(int precision, int mode, bool rec, bool rc, int rw) {
  if (precision == 64) return rc ? sweep_fn<double, true>(mode, rec, rw) : sweep_fn<double, false>(mode, rec, rw);
  return rc ? sweep_fn<float, true>(mode, rec, rw) : sweep_fn<float, false>(mode, rec, rw);
}

// The dynamic shared-memory limit is a per-function attribute shared by every
// solver in the process: raise it to the device maximum (never lower it to one
// solver's need, which would break a concurrent solver with a larger budget).
static cudaError_t allow_max_smem(const void *f) {
  int dev = 0, mx = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  // all of the unified L1 / shared storage as shared memory: without a stated
  // preference the occupancy query and the carveout the driver picks at launch
  // varied between boxes (MRF-LP sweeps at 4 or 5 CTAs per SM with the same
  // binary: 570 vs 541 us per iteration)
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  return e;
}

int sweep_occupancy(int precision, int mode, bool rec, bool rc, int rw, int block, size_t smem, int *blocks_per_sm) {
  const void *f = sweep_ptr(precision, mode, rec, rc, rw);
  if (!f) return 0;
  cudaError_t e = allow_max_smem(f);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, smem);
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute
static int launch_pdl(const void *f, dim3 grid, dim3 block, size_t smem, void *stream, void **args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelExC(&cfg, f, args);
}

template <typename T>
static const void *stream_fn(int mode, bool rec) {
  if (mode == kForward) return rec ? (const void *)sweep_stream_kernel<T, kForward, true> : (const void *)sweep_stream_kernel<T, kForward, false>;
  return rec ? (const void *)sweep_stream_kernel<T, kBackward, true> : (const void *)sweep_stream_kernel<T, kBackward, false>;
}

int launch_sweep_stream(int precision, int mode, bool rec, const SweepArgs &a, void *stream) {
  const void *f = precision == 64 ? stream_fn<double>(mode, rec) : stream_fn<float>(mode, rec);
  void *args[] = {(void *)&a};
  const int grid = (a.n_tiles + 3) / 4;
  return launch_pdl(f, dim3(grid > 0 ? grid : 1), dim3(128), 0, stream, args);
}

template <typename T>
static const void *chunk_fn(int mode, bool rec) {
  if (mode == kForward) return rec ? (const void *)sweep_chunk_kernel<T, kForward, true> : (const void *)sweep_chunk_kernel<T, kForward, false>;
  return rec ? (const void *)sweep_chunk_kernel<T, kBackward, true> : (const void *)sweep_chunk_kernel<T, kBackward, false>;
}

int launch_sweep_chunk(int precision, int mode, bool rec, const SweepArgs &a, void *stream) {
  const void *f = precision == 64 ? chunk_fn<double>(mode, rec) : chunk_fn<float>(mode, rec);
  const size_t wbytes = (size_t)(precision == 64 ? chunk_warp_bytes<double>() : chunk_warp_bytes<float>());
  const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, (227 * 1024) / wbytes));  // warps per CTA
  const cudaError_t e = allow_max_smem(f);
  if (e != cudaSuccess) return (int)e;
  void *args[] = {(void *)&a};
  const int grid = (a.n_tiles + wpb - 1) / wpb;
  return launch_pdl(f, dim3(grid > 0 ? grid : 1), dim3(32 * wpb), (size_t)wpb * wbytes, stream, args);
}

// Load every kernel a pass, a finalize or a bound can launch (CUDA lazy
// loading would otherwise load a kernel at its first launch, and loading waits
// for the device: with a peer-exchange kernel spinning on a rank that the same
// host thread has not launched yet, that first launch would never return).
int preload_kernels(int precision) {
  cudaFuncAttributes at;
  auto load = [&](const void *f) { return f ? cudaFuncGetAttributes(&at, f) : cudaSuccess; };
  cudaError_t e = cudaSuccess;
  for (int mode = 0; mode < 4 && e == cudaSuccess; ++mode)
    for (int rec = 0; rec < 2 && e == cudaSuccess; ++rec)
      for (int rc = 0; rc < 2 && e == cudaSuccess; ++rc) {
        for (int rw = 0; rw <= 4 && e == cudaSuccess; rw = rw ? 2 * rw : 1) e = load(sweep_ptr(precision, mode, rec != 0, rc != 0, rw));
        if (e == cudaSuccess && !rc)
          e = load(precision == 64 ? stream_fn<double>(mode, rec != 0) : stream_fn<float>(mode, rec != 0));
        if (e == cudaSuccess && !rc)
          e = load(precision == 64 ? chunk_fn<double>(mode, rec != 0) : chunk_fn<float>(mode, rec != 0));
      }
  const bool d = precision == 64;
  const void *fs[] = {d ? (const void *)avg_kernel<double> : (const void *)avg_kernel<float>,
                      d ? (const void *)avg_finish_kernel<double> : (const void *)avg_finish_kernel<float>,
                      d ? (const void *)peer_finish_kernel<double> : (const void *)peer_finish_kernel<float>,
                      d ? (const void *)add_deferred_kernel<double> : (const void *)add_deferred_kernel<float>,
                      (const void *)peer_signal_kernel, (const void *)lb_reduce_kernel};
  for (const void *f : fs)
    if (e == cudaSuccess) e = load(f);
  return (int)e;
}

int launch_sweep(int precision, int mode, bool rec, bool rc, int rw, const SweepArgs &a, int grid, int block,
                 size_t smem, void *stream) {
  const void *f = sweep_ptr(precision, mode, rec, rc, rw);
  if (!f) return (int)cudaErrorInvalidValue;
  void *args[] = {(void *)&a};
  return launch_pdl(f, dim3(grid), dim3(block), smem, stream, args);
}

static int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

int launch_avg(int precision, const AvgArgs &a, void *stream) {
  const int block = 256;
  const int64_t threads = avg_threads(a);
  const int grid = (int)std::max<int64_t>(1, (threads + block - 1) / block);
  void *args[] = {(void *)&a};
  const void *f = precision == 64 ? (const void *)avg_kernel<double> : (const void *)avg_kernel<float>;
  return launch_pdl(f, dim3(grid), dim3(block), 0, stream, args);
}

int launch_avg_finish(int precision, const AvgArgs &a, int32_t n_shared, const int32_t *xlocal, const int32_t *deg_x,
                      void *stream) {
  if (n_shared <= 0) return 0;
  const int block = 256, grid = grid_for(n_shared, block);
  if (precision == 64)
    avg_finish_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(a, n_shared, xlocal, deg_x);
  else
    avg_finish_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(a, n_shared, xlocal, deg_x);
  return (int)cudaGetLastError();
}

// ---- lifted representation (fdog_options::lifted) ----------------
// The two deferred averages of a variable (reading A8, j ascending, A1):
// avg1_i = (1/|J_i|) sum_k max(delta_bar_ik, 0) into every slot of i in
// avg_slot, avg0_i = (1/|J_i|) sum_k max(-delta_bar_ik, 0) into avg0.  One
// thread per variable (every variable is in the CSR part in lifted plans).
template <typename T>
__global__ void __launch_bounds__(256) avg_lifted_kernel(const AvgArgs a, T *avg0) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  pdl_wait();  // every thread: the sweep before wrote delta_bar (PDL launch)
  if (q == 0) *a.tile_counter = 0u;
  if (q >= a.n) return;
  const T *db = reinterpret_cast<const T *>(a.delta_bar);
  T *out = reinterpret_cast<T *>(a.avg_slot);
  const int64_t p0 = a.var_ptr[q], p1 = a.var_ptr[q + 1];
  T sp = T(0), sn = T(0);
  for (int64_t x = p0; x < p1; ++x) {
    const T d = db[a.var_slots[x]];
    sp = add_rn(sp, fmax(d, T(0)));
    sn = add_rn(sn, fmax(-d, T(0)));
  }
  const T deg = T(a.deg_l[q]);
  const T v1 = sp / deg, v0 = sn / deg;
  for (int64_t x = p0; x < p1; ++x) {
    out[a.var_slots[x]] = v1;
    avg0[a.var_slots[x]] = v0;
  }
}

// final correction, lifted form of P:650-652: lambda^{j,b} += max(+-delta_bar, 0)
template <typename T>
__global__ void __launch_bounds__(256) add_deferred_lifted_kernel(int64_t n, T *lam1, T *lam0, T *delta) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const T d = delta[q];
    lam1[q] = add_rn(lam1[q], fmax(d, T(0)));
    lam0[q] = add_rn(lam0[q], fmax(-d, T(0)));
    delta[q] = T(0);
  }
}

// out = lambda^1 - lambda^0 per device slot (the original-space lambda)
template <typename T>
__global__ void __launch_bounds__(256) lifted_diff_kernel(int64_t n, const T *lam1, const T *lam0, T *out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = sub_rn(lam1[q], lam0[q]);
}

int launch_avg_lifted(int precision, const AvgArgs &a, void *avg0, void *stream) {
  const int block = 256;
  const int grid = (int)std::max<int64_t>(1, ((int64_t)a.n + block - 1) / block);
  if (precision == 64) {
    void *args[] = {(void *)&a, &avg0};
    return launch_pdl((const void *)avg_lifted_kernel<double>, dim3(grid), dim3(block), 0, stream, args);
  }
  void *args[] = {(void *)&a, &avg0};
  return launch_pdl((const void *)avg_lifted_kernel<float>, dim3(grid), dim3(block), 0, stream, args);
}

int launch_add_deferred_lifted(int precision, int64_t n, void *lam1, void *lam0, void *delta, void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  if (precision == 64)
    add_deferred_lifted_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(n, (double *)lam1, (double *)lam0,
                                                                                 (double *)delta);
  else
    add_deferred_lifted_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(n, (float *)lam1, (float *)lam0,
                                                                                (float *)delta);
  return (int)cudaGetLastError();
}

int launch_lifted_diff(int precision, int64_t n, const void *lam1, const void *lam0, void *out, void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  if (precision == 64)
    lifted_diff_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(n, (const double *)lam1, (const double *)lam0,
                                                                         (double *)out);
  else
    lifted_diff_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(n, (const float *)lam1, (const float *)lam0,
                                                                        (float *)out);
  return (int)cudaGetLastError();
}

int launch_add_deferred(int precision, int64_t n, void *lambda, void *delta, void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  if (precision == 64)
    add_deferred_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(n, (double *)lambda, (double *)delta);
  else
    add_deferred_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(n, (float *)lambda, (float *)delta);
  return (int)cudaGetLastError();
}

int launch_lb_deferred(int precision, const TileDesc *tiles, int32_t n_tiles, const void *delta, double *lb_part,
                       void *stream) {
  if (n_tiles <= 0) return 0;
  const int block = 256, grid = (int)(((int64_t)n_tiles * 32 + block - 1) / block);
  if (precision == 64)
    lb_deferred_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(tiles, n_tiles, (const double *)delta, lb_part);
  else
    lb_deferred_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(tiles, n_tiles, (const float *)delta, lb_part);
  return (int)cudaGetLastError();
}

int launch_primal(int precision, const PrimalArgs &a, void *stream) {
  int n = a.n_ell + a.n_ell4 + a.n_csr;
  for (int g = 0; g < a.n_elld_g; ++g) n += a.elld_n[g];
  if (n <= 0) return 0;
  const int block = 256, grid = (n + block - 1) / block;
  if (precision == 64)
    primal_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(a);
  else
    primal_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

int launch_fused_small(int precision, bool rec, const SweepArgs &sa, const AvgArgs &aa, int32_t n_iter,
                       int64_t n_slots, int64_t n_dist, size_t smem, void *stream) {
  int32_t resident = smem > 0 ? 1 : 0;
  void *args[] = {(void *)&sa, (void *)&aa, (void *)&n_iter, (void *)&n_slots, (void *)&n_dist, (void *)&resident};
  const void *f = precision == 64 ? (rec ? (const void *)fused_small_kernel<double, true> : (const void *)fused_small_kernel<double, false>)
                                  : (rec ? (const void *)fused_small_kernel<float, true> : (const void *)fused_small_kernel<float, false>);
  if (smem > 48 * 1024) {
    const cudaError_t e = allow_max_smem(f);
    if (e != cudaSuccess) return (int)e;
  }
  return launch_pdl(f, dim3(1), dim3(1024), smem, stream, args);
}

template <typename T, typename O>
__global__ void __launch_bounds__(256) gather_canon_kernel(int64_t n, const int32_t *__restrict__ canon,
                                                          const T *__restrict__ src, O *__restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = (O)src[canon[q]];
}

// out: T per slot, or fp64 per slot (widen = 1)
int launch_gather_canon(int precision, int64_t n, const int32_t *canon, const void *src, void *out, int widen,
                        void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  cudaStream_t st = (cudaStream_t)stream;
  if (precision == 64)
    gather_canon_kernel<double, double><<<grid, block, 0, st>>>(n, canon, (const double *)src, (double *)out);
  else if (widen)
    gather_canon_kernel<float, double><<<grid, block, 0, st>>>(n, canon, (const float *)src, (double *)out);
  else
    gather_canon_kernel<float, float><<<grid, block, 0, st>>>(n, canon, (const float *)src, (float *)out);
  return (int)cudaGetLastError();
}

int launch_seq_level(int precision, bool record, const SeqArgs &a, int64_t q0, int64_t q1, void *stream) {
  if (q1 <= q0) return 0;
  const int block = 128;  // four variables (warps) per block
  const unsigned grid = (unsigned)((q1 - q0 + 3) / 4);
  cudaStream_t st = (cudaStream_t)stream;
  if (precision == 64) {
    if (record) seq_level_kernel<double, true><<<grid, block, 0, st>>>(a, q0, q1);
    else seq_level_kernel<double, false><<<grid, block, 0, st>>>(a, q0, q1);
  } else {
    if (record) seq_level_kernel<float, true><<<grid, block, 0, st>>>(a, q0, q1);
    else seq_level_kernel<float, false><<<grid, block, 0, st>>>(a, q0, q1);
  }
  return (int)cudaGetLastError();
}

int launch_seq_bound(const TileDesc *tiles, int32_t n_tiles, const double *e_lane, double *lb_part, void *stream) {
  if (n_tiles <= 0) return 0;
  seq_bound_kernel<<<(n_tiles + 255) / 256, 256, 0, (cudaStream_t)stream>>>(tiles, n_tiles, e_lane, lb_part);
  return (int)cudaGetLastError();
}

int launch_dist_dp(int precision, const SeqArgs &a, int32_t n_tiles, int32_t forward, void *stream) {
  if (n_tiles <= 0) return 0;
  const int64_t threads = (int64_t)n_tiles * 32;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  if (precision == 64)
    dist_dp_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(a, n_tiles, forward);
  else
    dist_dp_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(a, n_tiles, forward);
  return (int)cudaGetLastError();
}

template <typename T>
__global__ void __launch_bounds__(256) dist_sentinel_kernel(const TileDesc *tiles, int32_t n_tiles, T *dist) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int32_t t = (int32_t)(g >> 5), lane = (int32_t)(g & 31);
  if (t >= n_tiles) return;
  const TileDesc &d = tiles[t];
  for (int l = lane; l < d.lanes; l += 32) {
    T *top = dist + d.dist_base + (int64_t)d.nodes * d.lanes + l;
    top[0] = T(0);
    top[d.lanes] = t_inf<T>();
  }
}

int launch_dist_sentinels(int precision, const TileDesc *tiles, int32_t n_tiles, void *dist, void *stream) {
  if (n_tiles <= 0) return 0;
  const unsigned grid = (unsigned)(((int64_t)n_tiles * 32 + 255) / 256);
  if (precision == 64)
    dist_sentinel_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(tiles, n_tiles, (double *)dist);
  else
    dist_sentinel_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(tiles, n_tiles, (float *)dist);
  return (int)cudaGetLastError();
}

int launch_lb_reduce(const double *lb_part, int32_t n, double *out, void *stream) {
  void *args[] = {(void *)&lb_part, (void *)&n, (void *)&out};
  return launch_pdl((const void *)lb_reduce_kernel, dim3(1), dim3(1024), 0, stream, args);
}


}  // namespace fdog
