// Probe of the tcgen05 st/ld semantics used by kernels.cu TmemD (dev tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(float *out, int cols, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"((uint32_t)cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  // store value = warp*10000 + lane*100 + col for col in [0, 8)
  for (int c = 0; c < 8; c += 2) {
    float a = warp * 10000 + lane * 100 + c, b = a + 1;
    if (mode == 0)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta + c), "r"(__float_as_uint(a)), "r"(__float_as_uint(b)) : "memory");
    else {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(__float_as_uint(a)) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c + 1), "r"(__float_as_uint(b)) : "memory");
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int c = 0; c < 8; c += 2) {
    uint32_t x, y;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(ta + c) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(x), "+r"(y)::"memory");
    out[(threadIdx.x) * 8 + c] = __uint_as_float(x);
    out[(threadIdx.x) * 8 + c + 1] = __uint_as_float(y);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"((uint32_t)cols) : "memory");
}

int main() {
  float *d;
  const int T = 128;
  cudaMalloc(&d, T * 8 * sizeof(float));
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, T * 8 * sizeof(float));
    probe<<<2, T>>>(d, 32, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float h[T * 8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < T; ++t)
      for (int c = 0; c < 8; ++c) {
        float want = (t >> 5) * 10000 + (t & 31) * 100 + c;
        if (h[t * 8 + c] != want) {
          if (bad < 5) printf("mode %d t %d c %d got %g want %g\n", mode, t, c, h[t * 8 + c], want);
          bad++;
        }
      }
    printf("mode %d: %s, %d mismatches\n", mode, cudaGetErrorString(e), bad);
  }
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, probe, T, 0);
  printf("occupancy blocks/SM for a tcgen05 kernel of %d threads: %d\n", T, nb);
  return 0;
}
