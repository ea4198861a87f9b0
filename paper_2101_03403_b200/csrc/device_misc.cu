// Small device utilities: the FP64 DFMA peak probe (roofline denominator)
// and the gather that packs arbitrary result slots for one D2H copy.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fft512.cuh"
#include "kernels.cuh"
#include "sm100.cuh"

namespace cvm {

// The roofline denominator for the FFT kernel: MEASURED_PEAKS.json carries
// only HBM and bf16 figures, so the DFMA peak is measured live (8 independent
// FMA chains per thread, 148 x 8 CTAs of 256 threads).
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// Result download: slab rows (stride 632) of an arbitrary slot list packed
// into [count][631] for one D2H copy.
__global__ void __launch_bounds__(256) gather_lwe_kernel(const uint32_t* __restrict__ slab,
                                                         const uint64_t* __restrict__ slots,
                                                         uint64_t count,
                                                         uint32_t* __restrict__ out) {
  const uint64_t total = count * kLweWords;
  for (uint64_t e = uint64_t(blockIdx.x) * 256 + threadIdx.x; e < total;
       e += uint64_t(gridDim.x) * 256) {
    const uint64_t r = e / kLweWords, w = e - r * kLweWords;
    out[e] = slab[slots[r] * kLweStride + w];
  }
}

// ----------------------------------------------------------- launchers --
cudaError_t launch_gather_lwe(const uint32_t* slab, const uint64_t* slots, uint64_t count,
                              uint32_t* out, cudaStream_t s) {
  const uint64_t total = count * kLweWords;
  const unsigned blocks = unsigned(std::min<uint64_t>((total + 255) / 256, 148 * 16));
  gather_lwe_kernel<<<blocks, 256, 0, s>>>(slab, slots, count, out);
  return cudaGetLastError();
}
cudaError_t launch_fp64_peak(double* out, int blocks, int iters, cudaStream_t s) {
  fp64_peak_kernel<<<blocks, 256, 0, s>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace cvm
