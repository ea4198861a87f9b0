// Throughput probe: TMEM -> registers (tcgen05.ld 32x32b.x32) vs shared memory
// -> registers (LDS.128), 8 warps per SM, bytes per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) tmem_rd(int iters, unsigned long long* cyc, uint32_t* out) {
  __shared__ uint32_t tbase_s;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase_s)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase_s + ((uint32_t)((w & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    const uint32_t a = tb + (uint32_t)(((it + w) * 32) & 511);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; ++k) acc ^= r[k];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase_s), "r"(512) : "memory");
}

__global__ void __launch_bounds__(256, 1) lds_rd(int iters, unsigned long long* cyc, uint32_t* out) {
  extern __shared__ uint4 buf[];  // 64 KB
  for (int i = threadIdx.x; i < 4096; i += 256) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint4 v = buf[(((it + w) * 8 + k) * 32 + l) & 4095];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main() {
  const int iters = 4096, blocks = 148;
  unsigned long long* cyc;
  uint32_t* out;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&out, blocks * 256 * 4);
  cudaFuncSetAttribute(lds_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  unsigned long long h[148];
  for (int rep = 0; rep < 2; ++rep) {
    tmem_rd<<<blocks, 256>>>(iters, cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = 8.0 * 32 * 32 * 4 * iters;
    printf("tcgen05.ld 32x32b.x32: %s, %.1f B/clk/SM (%llu cycles)\n", cudaGetErrorString(e),
           bytes / h[0], h[0]);
    lds_rd<<<blocks, 256, 65536>>>(iters, cyc, out);
    e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    bytes = 8.0 * 32 * 8 * 16 * iters;
    printf("LDS.128: %s, %.1f B/clk/SM (%llu cycles)\n", cudaGetErrorString(e), bytes / h[0], h[0]);
  }
  return 0;
}
