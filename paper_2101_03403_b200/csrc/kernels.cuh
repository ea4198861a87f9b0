// Device job descriptors and kernel launchers (blind_rotate.cu, key_switch.cu,
// device_misc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft512.cuh"
#include "fft512w.cuh"
#include "schedule.hpp"
#include "tfhe_params.h"

namespace cvm {

constexpr uint32_t kNoInput = 0xFFFFFFFFu;
constexpr int kKsThreads = 160;

// One blind rotation: input sample = cst*(0,1) + coef[0]*slab[slot[0]]
// + coef[1]*slab[slot[1]] (coef 0 = unused), mu = 1/8, output extracted
// sample written to xlwe[out].
struct BrJob {
  uint32_t slot[2];
  int32_t coef[2];
  uint32_t cst;
  uint32_t out;
};

// One key switch: sample = xlwe[x[0]] (+ xlwe[x[1]]) + cst*(0,1), switched
// to the LWE key and written to slab[out_slot].
struct KsJob {
  uint32_t x[2];
  uint32_t cst;
  uint32_t out_slot;
};

cudaError_t launch_bk_to_fft(const uint32_t* bk, const c64* tw1, const c64* tw2, c64* bkf,
                             cudaStream_t s);
// bkf4 / tw4: the key in the warp-FFT bin order and the per-lane twiddle
// bases of the v4 kernels (blind_rotate_v4.cu, fft512w.cuh).
cudaError_t launch_bk_to_fft_v4(const uint32_t* bk, const c64* tw4, c64* bkf4, cudaStream_t s);
// variant < 0: the process-wide setting (br_variant()).
cudaError_t launch_blind_rotate(int variant, const BrJob* jobs, int count, const uint32_t* slab,
                                const c64* bkf, const c64* tw1, const c64* tw2,
                                const c64* bkf4, const c64* tw4, uint32_t* xout,
                                cudaStream_t s);
bool valid_br_v4_variant(int v);
// Auto-selection cost model: schedule.hpp.
cudaError_t launch_blind_rotate_v4(int variant, const BrJob* jobs, int count,
                                   const uint32_t* slab, const c64* bkf4, const c64* tw4,
                                   uint32_t* xout, cudaStream_t s);
// Blind-rotation kernel variant (a pinned choice; every one is bit-identical):
// 6000 + 10*W + 5 = v4 (one bootstrap per warp on the warp-wide FFT, W warps
// per CTA on a 5-row key ring; 6085 = full waves); 5247 = v3 (four
// bootstraps per CTA, 64-thread FFT, 7-row ring: wide-level remainders);
// 9 = wide (one bootstrap per SM, the six rows transformed concurrently);
// 96 = pair (one bootstrap per 2-SM cluster).  0 = auto by level width
// (default).  Env CVM_BR_KERNEL overrides the default.
constexpr int kDefaultBrVariant = 0;
int br_variant();
void set_br_variant(int v);
bool valid_br_variant(int v);
// Key-switch kernel: the level as one INT8 tcgen05 product (one-hot digits x
// byte limbs of the KSK, TMEM accumulators); 8 = one CTA per 128 x 128 tile,
// 9 = the tiles split along the coefficients (K) into up to 16 CTAs plus a
// reduction, so a narrow level still fills the GPU; 0 = auto (9).  Env
// CVM_KS_KERNEL.
constexpr int kDefaultKsVariant = 0;
int ks_variant();
void set_ks_variant(int v);
bool valid_ks_variant(int v);
cudaError_t launch_fp64_peak(double* out, int blocks, int iters, cudaStream_t s);
cudaError_t launch_gather_lwe(const uint32_t* slab, const uint64_t* slots, uint64_t count,
                              uint32_t* out, cudaStream_t s);
// ksktc: the KSK's byte limbs pre-arranged as tcgen05 B tiles (1024
// coefficients x 5 column tiles x 4 limbs x 4 KB), built at key upload from
// the padded [i][j][v][632] KSK (freed afterwards).
cudaError_t launch_ksk_to_tc(const uint32_t* ksk, uint32_t* ksktc, cudaStream_t s);
constexpr size_t kKskTcWords = size_t(kPolyN) * 5 * 4 * 1024;
// kspart: split-K scratch of variant 9, kKsPartWords u32.
constexpr int kKsMaxSplits = 16;
constexpr size_t kKsPartWords = size_t(148 / 5) * 128 * 640;
// variant < 0: the process-wide setting (ks_variant()).
cudaError_t launch_key_switch(int variant, const KsJob* jobs, int count, const uint32_t* xlwe,
                              const uint32_t* ksktc, uint32_t* kspart, uint32_t* slab,
                              cudaStream_t s);

}  // namespace cvm
