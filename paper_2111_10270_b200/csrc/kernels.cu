// kernels.cu -- sm_100a kernels of the deferred min-marginal averaging hot path.
//
//   sweep_kernel<T, MODE, REC>   one pass (forward P:627-645 / backward P:647-648)
//                                over all BDD tiles; MODE kEnergy = sum_j E^j only.
//   avg_kernel<T>                deferred averaging avg_i = mean_{k in J_i} delta_bar_ik
//                                (P:641 second term, readings A1/A10).
//   avg_finish_kernel<T>         shared variables after the NCCL exchange.
//   add_deferred_kernel<T>       final correction lambda += delta_bar.
//
// Thread mapping: one warp per tile of 32 BDDs, one BDD per
// lane.  Each lane walks its BDD's partitions sequentially (the hop recursion
// P:317-342 is sequential); all distances live in the lane's private column
// of shared memory ([node][lane] layout: conflict-free, no cross-lane
// communication, no atomics, no barriers inside a pass).  The distances of the
// opposite direction are RECOMPUTED on chip at the start of every pass from
// the current lambda (they equal the stored distances of P:315-316 exactly,
// because lambda has not changed since they were computed), so HBM traffic is
// topology + per-slot data only.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

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

// m1 - m0 with an infinite side replaced by +-clamp (reading A5).
template <typename T>
__device__ __forceinline__ T mm_difference(T m1, T m0, T clamp) {
  const bool i1 = isinf(m1), i0 = isinf(m0);
  if (i1 && i0) return T(0);  // only on padding lanes
  if (i1) return clamp;
  if (i0) return -clamp;
  return sub_rn(m1, m0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Last CTA reduces the per-tile bound partials in a fixed order (deterministic).
__device__ void reduce_lb_last_cta(const double *lb_part, int n, double *out, unsigned int *counter) {
  __shared__ bool is_last;
  __shared__ double red[32];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double s = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x) s += ((volatile const double *)lb_part)[q];
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (warp == 0) {
    double v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      *out = v;
      *counter = 0u;
    }
  }
}

template <typename T, int MODE, bool REC>
__global__ void __launch_bounds__(256) sweep_kernel(const SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const size_t per_warp = (size_t)(a.max_nodes + 4 * a.max_w + 2 * a.max_hops) * 32;
  T *const dist = reinterpret_cast<T *>(smem_raw) + warp * per_warp + lane;  // [node][32]
  T *const ringA = dist + (size_t)a.max_nodes * 32;                          // [2*max_w][32]
  T *const ringB = ringA + (size_t)2 * a.max_w * 32;                         // [2*max_w][32]
  T *const lam_s = ringB + (size_t)2 * a.max_w * 32;                         // [max_hops][32]
  T *const avg_s = lam_s + (size_t)a.max_hops * 32;                          // [max_hops][32]

  const T *__restrict__ avg = reinterpret_cast<const T *>(a.avg);
  T *__restrict__ lambda = reinterpret_cast<T *>(a.lambda);
  T *__restrict__ delta_out = reinterpret_cast<T *>(a.delta_out);
  const T inf = t_inf<T>();
  const T omega = T(a.omega), clamp = T(a.clamp);

  const int nwarps = gridDim.x * wpb;
  for (int t = blockIdx.x * wpb + warp; t < a.n_tiles; t += nwarps) {
    const TileDesc d = a.tiles[t];
    const bool valid = lane < d.n_lanes;
    const int32_t *__restrict__ ho = a.hop_off + d.hop_base;
    const uint32_t *__restrict__ tp;
    int ts;
    if (d.kind == 0) {
      tp = a.topo + d.topo_base;
      ts = 1;
    } else {
      tp = a.topo + d.topo_base + lane;
      ts = 32;
    }
    const int K = d.K;
    const int64_t sb = d.slot_base + lane;

    // stage lambda (and the deferred averages) of this lane's BDD
    for (int h = 0; h < K; ++h) {
      const int64_t s = sb + (int64_t)h * 32;
      lam_s[h * 32] = lambda[s];
      if (MODE != kEnergy) {
        const int v = a.slot_var[s];
        avg_s[h * 32] = v >= 0 ? __ldg(avg + v) : T(0);
      }
    }

    double acc = 0.0;
    if (MODE == kForward || MODE == kEnergy) {
      // phase 1: shp(v, T) for all nodes under the current lambda
      for (int h = K - 1; h >= 0; --h) {
        const T lam = lam_s[h * 32];
        const int n0 = ho[h], n1 = ho[h + 1];
        for (int n = n0; n < n1; ++n) {
          const uint32_t e = __ldg(tp + (size_t)n * ts);
          const uint32_t lo = e & 0xFFFFu, hi = e >> 16;
          const T c0 = lo == kBot ? inf : lo == kTop ? T(0) : dist[(size_t)(n1 + lo) * 32];
          const T c1 = hi == kBot ? inf : hi == kTop ? T(0) : dist[(size_t)(n1 + hi) * 32];
          dist[(size_t)n * 32] = fmin(c0, lam + c1);
        }
      }
      if (MODE == kEnergy) {
        acc = valid ? (double)dist[0] : 0.0;  // E^j = shp(r, T)
      } else {
        // phase 2: forward pass with updates (Alg. forward_pass_mm)
        T *cur = ringA, *nxt = ringA + (size_t)a.max_w * 32;
        T *nlo = ringB, *nhi = ringB + (size_t)a.max_w * 32;
        cur[0] = T(0);  // shp(r, r)
        for (int h = 0; h < K; ++h) {
          const int n0 = ho[h], n1 = ho[h + 1];
          const bool last = h == K - 1;
          const int Wn = last ? 0 : ho[h + 2] - n1;
          for (int w = 0; w < Wn; ++w) {
            nlo[w * 32] = inf;
            nhi[w * 32] = inf;
          }
          T m0 = inf, m1r = inf;  // m1r = min (shp(r,v) + shp(s1 v, T)), lambda added below
          for (int n = n0; n < n1; ++n) {
            const uint32_t e = __ldg(tp + (size_t)n * ts);
            const uint32_t lo = e & 0xFFFFu, hi = e >> 16;
            const T cf = cur[(n - n0) * 32];
            if (lo != kBot) {
              const T c = lo == kTop ? T(0) : dist[(size_t)(n1 + lo) * 32];
              m0 = fmin(m0, cf + c);
              if (!last) nlo[lo * 32] = fmin(nlo[lo * 32], cf);
            }
            if (hi != kBot) {
              const T c = hi == kTop ? T(0) : dist[(size_t)(n1 + hi) * 32];
              m1r = fmin(m1r, cf + c);
              if (!last) nhi[hi * 32] = fmin(nhi[hi * 32], cf);
            }
          }
          const T lam = lam_s[h * 32];
          const T m1 = lam + m1r;  // Eq. (min-marginal-via-shortest-path) P:312
          const T dd = mm_difference(m1, m0, clamp);
          const T delta = mul_rn(omega, dd);
          const T lam_new = add_rn(sub_rn(lam, delta), avg_s[h * 32]);
          if (valid) {
            const int64_t s = sb + (int64_t)h * 32;
            lambda[s] = lam_new;
            delta_out[s] = delta;
            if (REC) {
              reinterpret_cast<T *>(a.m0)[s] = m0;
              reinterpret_cast<T *>(a.m1)[s] = m1;
            }
            acc += (double)fmin(delta, T(0));
          }
          if (!last) {
            // shp(r, v) for v in P_{h+1}, 1-arcs priced with the updated lambda_h (A4)
            for (int w = 0; w < Wn; ++w) nxt[w * 32] = fmin(nlo[w * 32], nhi[w * 32] + lam_new);
            T *tmp = cur;
            cur = nxt;
            nxt = tmp;
          } else if (valid) {
            acc += (double)fmin(m0, lam_new + m1r);  // E^j at the updated lambda
          }
        }
      }
    } else {
      // phase 1: shp(r, v) for all nodes under the current lambda
      dist[0] = T(0);
      for (int h = 0; h + 1 < K; ++h) {
        const T lam = lam_s[h * 32];
        const int n0 = ho[h], n1 = ho[h + 1], n2 = ho[h + 2];
        for (int n = n1; n < n2; ++n) dist[(size_t)n * 32] = inf;
        for (int n = n0; n < n1; ++n) {
          const uint32_t e = __ldg(tp + (size_t)n * ts);
          const uint32_t lo = e & 0xFFFFu, hi = e >> 16;
          const T cf = dist[(size_t)n * 32];
          if (lo != kBot) dist[(size_t)(n1 + lo) * 32] = fmin(dist[(size_t)(n1 + lo) * 32], cf);
          if (hi != kBot) dist[(size_t)(n1 + hi) * 32] = fmin(dist[(size_t)(n1 + hi) * 32], cf + lam);
        }
      }
      // phase 2: backward pass with updates (Alg. backward_pass_mm)
      T *cur = ringA, *nxt = ringA + (size_t)a.max_w * 32;  // shp(., T) of P_{h+1}, P_h
      T *c0s = ringB, *c1s = ringB + (size_t)a.max_w * 32;
      for (int h = K - 1; h >= 0; --h) {
        const int n0 = ho[h], n1 = ho[h + 1];
        T m0 = inf, m1r = inf;
        for (int n = n0; n < n1; ++n) {
          const uint32_t e = __ldg(tp + (size_t)n * ts);
          const uint32_t lo = e & 0xFFFFu, hi = e >> 16;
          const T cf = dist[(size_t)n * 32];
          const T c0 = lo == kBot ? inf : lo == kTop ? T(0) : cur[lo * 32];
          const T c1 = hi == kBot ? inf : hi == kTop ? T(0) : cur[hi * 32];
          c0s[(n - n0) * 32] = c0;
          c1s[(n - n0) * 32] = c1;
          if (lo != kBot) m0 = fmin(m0, cf + c0);
          if (hi != kBot) m1r = fmin(m1r, cf + c1);
        }
        const T lam = lam_s[h * 32];
        const T m1 = lam + m1r;
        const T dd = mm_difference(m1, m0, clamp);
        const T delta = mul_rn(omega, dd);
        const T lam_new = add_rn(sub_rn(lam, delta), avg_s[h * 32]);
        if (valid) {
          const int64_t s = sb + (int64_t)h * 32;
          lambda[s] = lam_new;
          delta_out[s] = delta;
          if (REC) {
            reinterpret_cast<T *>(a.m0)[s] = m0;
            reinterpret_cast<T *>(a.m1)[s] = m1;
          }
          acc += (double)fmin(delta, T(0));
        }
        // shp(v, T) for v in P_h with the updated lambda_h
        for (int w = 0; w < n1 - n0; ++w) nxt[w * 32] = fmin(c0s[w * 32], lam_new + c1s[w * 32]);
        T *tmp = cur;
        cur = nxt;
        nxt = tmp;
      }
      if (valid) acc += (double)cur[0];  // E^j = shp(r, T)
    }
    acc = warp_sum(acc);
    if (lane == 0) a.lb_part[t] = acc;
  }
  reduce_lb_last_cta(a.lb_part, a.n_tiles, a.lb_out, a.done_counter);
}

template <typename T>
__global__ void __launch_bounds__(256) avg_kernel(const AvgArgs a) {
  const T *__restrict__ db = reinterpret_cast<const T *>(a.delta_bar);
  T *__restrict__ avg = reinterpret_cast<T *>(a.avg);
  T *__restrict__ xbuf = reinterpret_cast<T *>(a.xbuf);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.n; q += gridDim.x * blockDim.x) {
    const int64_t p0 = a.var_ptr[q], p1 = a.var_ptr[q + 1];
    T s = T(0);
    for (int64_t p = p0; p < p1; ++p) s += __ldg(db + a.var_slots[p]);  // k in J_i ascending
    const int x = a.var_xidx ? a.var_xidx[q] : -1;
    if (x >= 0) {
      xbuf[x] = s;
    } else {
      const int i = a.var_list[q];
      avg[i] = s / T(a.deg[i]);
    }
  }
}

template <typename T>
__global__ void avg_finish_kernel(int32_t n, const int32_t *__restrict__ vars, const int32_t *__restrict__ deg,
                                  const T *__restrict__ xbuf, T *__restrict__ avg) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = vars[q];
    avg[i] = xbuf[q] / T(deg[i]);
  }
}

template <typename T>
__global__ void add_deferred_kernel(int64_t n, T *__restrict__ lambda, T *__restrict__ delta) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    lambda[q] += delta[q];
    delta[q] = T(0);
  }
}

template <typename T>
__global__ void fill_kernel(int64_t n, T *__restrict__ dst, T v) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[q] = v;
}

// ---------------------------------------------------------------- launchers

template <typename T>
static const void *sweep_fn(int mode, bool rec) {
  if (mode == kForward) return rec ? (const void *)sweep_kernel<T, kForward, true> : (const void *)sweep_kernel<T, kForward, false>;
  if (mode == kBackward) return rec ? (const void *)sweep_kernel<T, kBackward, true> : (const void *)sweep_kernel<T, kBackward, false>;
  return (const void *)sweep_kernel<T, kEnergy, false>;
}

static const void *sweep_ptr(int precision, int mode, bool rec) {
  return precision == 64 ? sweep_fn<double>(mode, rec) : sweep_fn<float>(mode, rec);
}

int sweep_smem_bytes(int precision, int max_nodes, int max_w, int max_hops, int warps) {
  const size_t tsz = precision == 64 ? 8 : 4;
  size_t b = (size_t)warps * (size_t)(max_nodes + 4 * max_w + 2 * max_hops) * 32 * tsz;
  return b > (size_t)0x7fffffff ? 0x7fffffff : (int)b;
}

int sweep_occupancy(int precision, int mode, bool rec, int block, size_t smem, int *blocks_per_sm) {
  const void *f = sweep_ptr(precision, mode, rec);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, smem);
}

int launch_sweep(int precision, int mode, bool rec, const SweepArgs &a, int grid, int block, size_t smem,
                 void *stream) {
  const void *f = sweep_ptr(precision, mode, rec);
  void *args[] = {(void *)&a};
  return (int)cudaLaunchKernel(f, dim3(grid), dim3(block), args, smem, (cudaStream_t)stream);
}

static int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

int launch_avg(int precision, const AvgArgs &a, void *stream) {
  const int block = 256;
  const int grid = grid_for(a.n, block);
  if (precision == 64)
    avg_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(a);
  else
    avg_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

int launch_avg_finish(int precision, int32_t n, const int32_t *vars, const int32_t *deg, const void *xbuf,
                      void *avg, void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  if (precision == 64)
    avg_finish_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(n, vars, deg, (const double *)xbuf, (double *)avg);
  else
    avg_finish_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(n, vars, deg, (const float *)xbuf, (float *)avg);
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

int launch_fill(int precision, int64_t n, void *dst, double value, void *stream) {
  if (n <= 0) return 0;
  const int block = 256, grid = grid_for(n, block);
  if (precision == 64)
    fill_kernel<double><<<grid, block, 0, (cudaStream_t)stream>>>(n, (double *)dst, value);
  else
    fill_kernel<float><<<grid, block, 0, (cudaStream_t)stream>>>(n, (float *)dst, (float)value);
  return (int)cudaGetLastError();
}

}  // namespace fdog
