// v4 blind rotation: one bootstrap per WARP, G bootstraps per CTA sharing a
// bulk-copy shared-memory key ring (the throughput organisation of v3, with
// the warp-wide FFT of fft512w.cuh).
//
// Why: the v3 kernel (64 threads per transform, two shared-memory exchanges
// per transform, named barriers between its two warps) is bound by the
// shared-memory pipe (LSU wavefronts 72%, profiles/r01_ncu_blind_rotate_5247.json).
// Here a transform costs one transpose (16 STS.128 + 16 LDS.128 per lane,
// 128 wavefronts per warp) plus a lane-pair swap of 8 values by shuffles,
// instead of 256 wavefronts, and the bootstrap never leaves its warp: the
// accumulator, digits, exchange buffer and every barrier are warp-local
// (__syncwarp).  Key rows are shared by the G warps; each slot is refilled by
// its last reader (per-slot counter) with the chunk S rows ahead.
//
// Key layout (bk_to_fft_v4_kernel): chunk q = 6 i + row holds the TRUE folded
// spectrum / M of both output polynomials in warp bin order,
// [slot r (16)][o (2)][lane (32)] c64 -- a lane's 32 values of a row are 32
// conflict-free LDS.128.
#include <cuda_runtime.h>

#include <cstddef>

#include "br_common.cuh"
#include "fft512w.cuh"
#include "kernels.cuh"
#include "sm100.cuh"

namespace cvm {

__device__ __forceinline__ c64 shfl_xor1(c64 v) {
  return {__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1)};
}

// A copy the compiler cannot see through: values that are loop-invariant
// (the twiddle bases, the lane's transpose addresses) are re-derived inside
// the CMux loop instead of hoisted into registers -- hoisted, the 16
// twiddles and 32 addresses spill to local memory (ptxas -v).
__device__ __forceinline__ double opaque(double x) {
  double y;
  asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ TwBasesW opaque(const TwBasesW& b) {
  return {{opaque(b.base.x), opaque(b.base.y)}, {opaque(b.w.x), opaque(b.w.y)}};
}

__device__ __forceinline__ TwBasesW load_wbases(const c64* tw4, int l) {
  return {ldg_c64(tw4 + 2 * l), ldg_c64(tw4 + 2 * l + 1)};
}

#ifdef CVM_PHASE_PROF
// Developer instrumentation (tools/v4_phases.py): per-phase clock64 sums of
// lane 0 of every warp, [cta][warp][phase].
__device__ unsigned long long g_v4_phase[148][8][8];
#define PH4(k)                                     \
  do {                                             \
    const long long now_ = clock64();              \
    ph[k] += (unsigned long long)(now_ - last_);   \
    last_ = now_;                                  \
  } while (0)
#else
#define PH4(k) \
  do {         \
  } while (0)
#endif

// ----------------------------------------------------------------- K5 v4 --
// One warp per key polynomial (i, row, o): forward warp FFT, the D factor of
// the odd lanes removed (fft512w.cuh), scaled by 1/M.
__global__ void __launch_bounds__(32) bk_to_fft_v4_kernel(const uint32_t* __restrict__ bk,
                                                          const c64* __restrict__ tw4,
                                                          c64* __restrict__ bkf4) {
  __shared__ c64 buf[512];
  const int l = threadIdx.x, e = l & 1;
  const int poly = blockIdx.x;  // ((i*6 + row)*2 + o)
  const int o = poly & 1, ir = poly >> 1;
  const uint32_t* p = bk + (size_t)poly * kPolyN;
  c64 v[16];
#pragma unroll
  for (int a = 0; a < 16; ++a)
    v[a] = {(double)(int32_t)p[l + 32 * a], (double)(int32_t)p[l + 32 * a + 512]};
  wfwd_stage1(v, load_wbases(tw4, l));
#pragma unroll
  for (int k0 = 0; k0 < 16; ++k0) buf[wpos(k0, l)] = v[k0];
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 16; ++s) v[s] = buf[wpos(l >> 1, wslot_t(e, s))];
  wfwd_stage2a(v, e);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[8 + i] = shfl_xor1(v[8 + i]);
  wfwd_stage2b(v);
  const double sc = 1.0 / kFftM;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double f = (e && (r & 1)) ? -sc : sc;
    bkf4[(size_t)ir * 1024 + (2 * r + o) * 32 + l] = {v[r].x * f, v[r].y * f};
  }
}

// ---------------------------------------------------------- K1 + K2, v4 --
// Per-bootstrap (per-warp) shared memory.
struct WarpSmem4 {
  c64 xbuf[512];                // the transpose buffer
  uint32_t acc[2][kPolyN];      // ACC (both TRLWE parts)
  uint16_t bar[kLweWords + 1];  // mod-switched input sample
};
constexpr int kV4MaxWarps = 8;
template <int S>
struct BrSmem4 {
  uint64_t full[S];
  uint32_t cnt[S];  // warps done with each slot
  alignas(128) c64 ring[S][1024];
  WarpSmem4 w[kV4MaxWarps];  // only blockDim.x / 32 of them are allocated
};
template <int S>
constexpr int v4_smem_bytes(int warps) {
  return int(offsetof(BrSmem4<S>, w) + sizeof(WarpSmem4) * warps);
}

// One CTA of blockDim.x / 32 <= 8 warps (runtime: a partial last wave runs
// with fewer bootstraps per SM instead of idle SMs), one bootstrap per warp.
// kHold: the digits of gadget levels 1 and 2 of a part are kept in registers
// (16 words, packed from the rotated differences read for level 0) instead
// of re-reading the accumulator per level.
template <int S, bool kHold>
__global__ void __launch_bounds__(32 * kV4MaxWarps, 1) blind_rotate_kernel_v4(
    const BrJob* __restrict__ jobs, int count, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf4, const c64* __restrict__ tw4, uint32_t* __restrict__ xout) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BrSmem4<S>& sm = *reinterpret_cast<BrSmem4<S>*>(smem_raw);
  const int tid = threadIdx.x;
  const int nw = blockDim.x >> 5;
  const int g = tid >> 5, l = tid & 31, e = l & 1;
  const int jidx = blockIdx.x * nw + g;
  const bool live = jidx < count;
  const BrJob job = jobs[live ? jidx : 0];
  constexpr int kChunks = kN * kRows;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      sm.cnt[s] = 0;
    }
    mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_expect_tx(&sm.full[q], kRowBytes);
      bulk_g2s(sm.ring[q], bkf4 + (size_t)q * 1024, kRowBytes, &sm.full[q]);
    }
  }
  const TwBasesW tb = load_wbases(tw4, l);
  uint32_t* acc0 = sm.w[g].acc[0];
  uint32_t* acc1 = sm.w[g].acc[1];
  uint16_t* bar = sm.w[g].bar;
  c64* xb = sm.w[g].xbuf;
  prologue(job, slab, bar, acc0, acc1, l, 32, warp_sync, 0);

  int q = 0;
#ifdef CVM_PHASE_PROF
  unsigned long long ph[8] = {};
  long long last_ = clock64();
#endif
  for (int i = 0; i < kN; ++i) {
    __syncwarp();
    const int ai = bar[i];
    c64 af[2][16];
#pragma unroll
    for (int r = 0; r < 16; ++r) af[0][r] = af[1][r] = c64{0.0, 0.0};
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const uint32_t* accp = part ? acc1 : acc0;
      // (X^ai - 1) * ACC_part at coefficients j = l + 32a and j + 512,
      // offset for the decomposition
      auto rdiff = [&](int a, uint32_t& d0, uint32_t& d1) {
        const int j = l + 32 * a;
        const int m0 = (j - ai) & (2 * kPolyN - 1);
        const int m1 = (j + 512 - ai) & (2 * kPolyN - 1);
        const uint32_t r0 = m0 < kPolyN ? accp[m0] : 0u - accp[m0 - kPolyN];
        const uint32_t r1 = m1 < kPolyN ? accp[m1] : 0u - accp[m1 - kPolyN];
        d0 = r0 - accp[j] + kDecompOffset;
        d1 = r1 - accp[j + 512] + kDecompOffset;
      };
      // kHold: level 0 reads the rotated differences and keeps the bits of
      // levels 1 and 2 (bits kLow .. kLow+13), two coefficients per register
      constexpr int kLow = 32 - kL * kBgBit;
      uint32_t pk[kHold ? 16 : 1];
#pragma unroll 1
      for (int p = 0; p < kL; ++p, ++q) {
        const int shift = 32 - (p + 1) * kBgBit;
        c64 v[16];
        if (!kHold || p == 0) {
#pragma unroll
          for (int a = 0; a < 16; ++a) {
            uint32_t d0, d1;
            rdiff(a, d0, d1);
            if constexpr (kHold)
              pk[a] = ((d0 >> kLow) & 0x3FFFu) | (((d1 >> kLow) & 0x3FFFu) << 16);
            v[a] = {u32_biased_to_double((d0 >> shift) & 127u, kDigitBias),
                    u32_biased_to_double((d1 >> shift) & 127u, kDigitBias)};
          }
        } else {
          const int sh = shift - kLow;
#pragma unroll
          for (int a = 0; a < 16; ++a)
            v[a] = {u32_biased_to_double((pk[a] >> sh) & 127u, kDigitBias),
                    u32_biased_to_double((pk[a] >> (16 + sh)) & 127u, kDigitBias)};
        }
        PH4(0);
        const int lo = opaque(l), eo = lo & 1;
        wfwd_stage1(v, opaque(tb));
#pragma unroll
        for (int k0 = 0; k0 < 16; ++k0) xb[wpos(k0, lo)] = v[k0];
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 16; ++s) v[s] = xb[wpos(lo >> 1, wslot_t(eo, s))];
        __syncwarp();  // the buffer is free for the next transpose
        wfwd_stage2a(v, e);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 + k] = shfl_xor1(v[8 + k]);
        wfwd_stage2b(v);
        PH4(1);
        const int slot = q % S;
        mbar_wait(&sm.full[slot], (q / S) & 1);
        PH4(2);
        const c64* bk = sm.ring[slot];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          af[0][r] = cmac(af[0][r], v[r], bk[(2 * r) * 32 + l]);
          af[1][r] = cmac(af[1][r], v[r], bk[(2 * r + 1) * 32 + l]);
        }
        // the slot's last reader streams the chunk S rows ahead into it.  Every
        // warp's key loads have returned (the MACs consumed them) and are
        // ordered by the fence before its count, so the bulk copy cannot
        // overwrite data still being read -- the same write-after-read
        // contract as a consumer-release / producer-acquire TMA pipeline,
        // which needs no proxy fence.
        __syncwarp();
        if (l == 0) {
          if (atom_add_release_cta(&sm.cnt[slot], 1u) == unsigned(nw - 1)) {
            sm.cnt[slot] = 0;
            if (q + S < kChunks) {
              mbar_expect_tx(&sm.full[slot], kRowBytes);
              bulk_g2s(sm.ring[slot], bkf4 + (size_t)(q + S) * 1024, kRowBytes, &sm.full[slot]);
            }
          }
        }
        PH4(3);
      }
    }
#pragma unroll 1
    for (int o = 0; o < 2; ++o) {
      c64 v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = o ? af[1][r] : af[0][r];
      winv_stage2b(v);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[8 + k] = shfl_xor1(v[8 + k]);
      winv_stage2a(v, e);
      const int lo = opaque(l), eo = lo & 1;
#pragma unroll
      for (int s = 0; s < 16; ++s) xb[wpos(lo >> 1, wslot_t(eo, s))] = v[s];
      __syncwarp();
#pragma unroll
      for (int k0 = 0; k0 < 16; ++k0) v[k0] = xb[wpos(k0, lo)];
      __syncwarp();
      winv_stage1(v, opaque(tb));
      PH4(4);
      uint32_t* accp = o ? acc1 : acc0;
#pragma unroll
      for (int a = 0; a < 16; ++a) {
        accp[l + 32 * a] += round_to_torus(v[a].x);
        accp[l + 32 * a + 512] += round_to_torus(v[a].y);
      }
      PH4(5);
    }
  }
#ifdef CVM_PHASE_PROF
  if (l == 0 && blockIdx.x < 148)
    for (int k = 0; k < 8; ++k) g_v4_phase[blockIdx.x][g][k] = ph[k];
#endif
  __syncwarp();
  if (live) extract(acc0, acc1, xout + (size_t)job.out * kXlweStride, l, 32);
}

#ifdef CVM_PHASE_PROF
extern "C" __attribute__((visibility("default"))) int cvm_debug_v4_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_v4_phase, sizeof(g_v4_phase));
}
#endif
#undef PH4

// ----------------------------------------------------------- launchers --
cudaError_t launch_bk_to_fft_v4(const uint32_t* bk, const c64* tw4, c64* bkf4, cudaStream_t s) {
  bk_to_fft_v4_kernel<<<kN * kRows * 2, 32, 0, s>>>(bk, tw4, bkf4);
  return cudaGetLastError();
}

template <int S, bool kHold>
static cudaError_t launch_v4(int warps, const BrJob* jobs, int count, const uint32_t* slab,
                             const c64* bkf4, const c64* tw4, uint32_t* xout, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  auto* kern = blind_rotate_kernel_v4<S, kHold>;
  cudaError_t e = set_smem(kern, v4_smem_bytes<S>(kV4MaxWarps), configured);
  if (e != cudaSuccess) return e;
  kern<<<(count + warps - 1) / warps, 32 * warps, v4_smem_bytes<S>(warps), s>>>(
      jobs, count, slab, bkf4, tw4, xout);
  return cudaGetLastError();
}

// 6000 + 10 * warps + 5, warps = 1..8 (held digits, 5-row key ring)
bool valid_br_v4_variant(int v) {
  const int w = (v - 6005) / 10;
  return v >= 6015 && v <= 6085 && (v - 6005) % 10 == 0 && w >= 1 && w <= kV4MaxWarps;
}

cudaError_t launch_blind_rotate_v4(int variant, const BrJob* jobs, int count,
                                   const uint32_t* slab, const c64* bkf4, const c64* tw4,
                                   uint32_t* xout, cudaStream_t s) {
  if (!valid_br_v4_variant(variant)) return cudaErrorInvalidValue;
  return launch_v4<5, true>((variant / 10) % 10, jobs, count, slab, bkf4, tw4, xout, s);
}

}  // namespace cvm
