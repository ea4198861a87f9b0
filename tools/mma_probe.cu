// Throughput probe: legacy warp-level mma.sync int8 / fp16 on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void probe(int iters, int* out) {
  uint32_t a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, threadIdx.x};
  int c[8][4] = {};
  float f[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (KIND == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(f[u][0]), "+f"(f[u][1]), "+f"(f[u][2]), "+f"(f[u][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      }
    }
  }
  int s = 0;
  for (int u = 0; u < 8; ++u)
    for (int k = 0; k < 4; ++k) s += c[u][k] + (int)f[u][k];
  if (s == 12345) out[0] = s;
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind) {
    for (int warps : {4, 8, 16}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&] {
        if (kind == 0) probe<0><<<sms * 2, 32 * warps>>>(iters, out);
        else probe<1><<<sms * 2, 32 * warps>>>(iters, out);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double mmas = double(sms) * 2 * warps * iters * 8;
      const double ops = mmas * (kind == 0 ? 16 * 8 * 32 * 2 : 16 * 8 * 16 * 2);
      printf("%s warps/CTA=%d: %.3f ms, %.1f TOPS\n", kind == 0 ? "mma.sync s8 m16n8k32" :
             "mma.sync f16 m16n8k16", warps, ms, ops / ms * 1e-9);
    }
  }
  return 0;
}
