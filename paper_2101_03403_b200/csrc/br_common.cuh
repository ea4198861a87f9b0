// Shared pieces of the blind-rotation kernels (blind_rotate.cu,
// blind_rotate_v4.cu): decomposition constants, the K1 prologue (gate-input
// combination, mod-switch, ACC init) and sample extraction.
#pragma once
#include <stdint.h>

#include "fft512.cuh"
#include "kernels.cuh"
#include "tfhe_params.h"

namespace cvm {

// digits: buf = c + offset; d_p = ((buf >> (25 - 7p)) & 127) - 64
constexpr uint32_t kDecompOffset =
    (1u << (kBgBit - 1)) * ((1u << 25) + (1u << 18) + (1u << 11));
constexpr double kDigitBias = 4503599627370496.0 + 64.0;  // 2^52 + Bg/2
constexpr uint32_t kRowBytes = 1024 * 16;                 // one TRGSW row, FFT domain

// K1: the gate's input sample (cst + coef0*slot0 + coef1*slot1) mod-switched
// to Z_2N, then ACC = X^{-b} (0, mu * sum X^j).
__device__ __forceinline__ void prologue(const BrJob& job, const uint32_t* slab, uint16_t* bar,
                                         uint32_t* acc0, uint32_t* acc1, int t, int nthreads,
                                         void (*sync)(int), int sync_arg) {
  for (int i = t; i < kLweWords; i += nthreads) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    bar[i] = (uint16_t)modswitch_2n(v);
  }
  sync(sync_arg);
  const int barb = bar[kN];
  for (int j = t; j < kPolyN; j += nthreads) {
    acc0[j] = 0;
    acc1[j] = (((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu);
  }
}
static __device__ void cta_sync(int) { __syncthreads(); }
static __device__ void warp_sync(int) { __syncwarp(); }

// Sample extraction: a'_0 = a_0, a'_j = -a_{N-j}, b' = b_0.
__device__ __forceinline__ void extract(const uint32_t* acc0, const uint32_t* acc1,
                                        uint32_t* out, int t, int nthreads) {
  for (int j = t; j < kPolyN; j += nthreads) out[j] = j == 0 ? acc0[0] : 0u - acc0[kPolyN - j];
  if (t == 0) out[kPolyN] = acc1[0];
}

}  // namespace cvm
