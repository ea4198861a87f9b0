// sm_100a kernels of the batched TFHE gate-bootstrapping path.
//
//   bk_to_fft_kernel   K5  one-time: BK (time domain, u32) -> folded FFT domain,
//                          pre-scaled by 1/M, in per-thread bin order.
//   blind_rotate_kernel K1+K2 fused: gate-input combination + mod-switch
//                          prologue, 630 CMux steps (gadget decomposition,
//                          6 forward FFTs, 12 complex MACs against BK_i,
//                          2 inverse FFTs, exact rounding), sample extraction.
//   key_switch_kernel  K3+K4: (MUX combine) + LWE key switch N=1024 -> n=630.
//
// One CTA of 64 threads owns one bootstrap; the whole 630-step chain runs
// inside one launch with the accumulator resident in shared memory.  See
// DESIGN.md section 4 for the roofline of each kernel.
#include <cuda_runtime.h>

#include <type_traits>

#include "fft512.cuh"
#include "kernels.cuh"

namespace cvm {

// digits: buf = c + offset; d_p = ((buf >> (25 - 7p)) & 127) - 64
constexpr uint32_t kDecompOffset =
    (1u << (kBgBit - 1)) * ((1u << 25) + (1u << 18) + (1u << 11));
constexpr double kDigitBias = 4503599627370496.0 + 64.0;  // 2^52 + Bg/2

template <int kPattern>  // 1: fwd ex1, 2: fwd ex2 / inv exA, 3: inv exB
__device__ __forceinline__ void exchange(c64 v[8], c64* buf, int t) {
#pragma unroll
  for (int z = 0; z < 8; ++z) {
    int cell, slot;
    if (kPattern == 1) {
      cell = ex1_cell(t, z);
      slot = t >> 3;
    } else if (kPattern == 2) {
      cell = ex2_cell(t, z);
      slot = t >> 3;
    } else {
      cell = exB_cell(t, z);
      slot = t & 7;
    }
    buf[xpos(cell, slot)] = v[z];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = buf[xpos(t, s)];
}

__device__ __forceinline__ c64 ldg_c64(const c64* p) {
  double2 d = __ldg(reinterpret_cast<const double2*>(p));
  return {d.x, d.y};
}

__device__ __forceinline__ void load_twiddles(const c64* tw1, const c64* tw2,
                                              int t, c64 T1[8], c64 T2[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T1[k] = ldg_c64(tw1 + t * 8 + k);
    T2[k] = ldg_c64(tw2 + t * 8 + k);
  }
}

// ----------------------------------------------------------------- K5 --
__global__ void __launch_bounds__(64) bk_to_fft_kernel(const uint32_t* __restrict__ bk,
                                                       const c64* __restrict__ tw1,
                                                       const c64* __restrict__ tw2,
                                                       c64* __restrict__ bkf) {
  __shared__ c64 xbuf[2][512];
  const int t = threadIdx.x;
  const int poly = blockIdx.x;  // ((i*6 + row)*2 + o)
  const int o = poly & 1, ir = poly >> 1;
  c64 T1[8], T2[8];
  load_twiddles(tw1, tw2, t, T1, T2);
  const uint32_t* p = bk + (size_t)poly * kPolyN;
  c64 v[8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
    v[a] = {(double)(int32_t)p[t + 64 * a], (double)(int32_t)p[t + 64 * a + 512]};
  fwd_stage1(v, T1);
  exchange<1>(v, xbuf[0], t);
  fwd_stage2(v, T2);
  exchange<2>(v, xbuf[1], t);
  fwd_stage3(v);
  const double s = 1.0 / kFftM;
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2)
    bkf[((size_t)ir * 8 + k2) * 128 + o * 64 + t] = {v[k2].x * s, v[k2].y * s};
}

// ------------------------------------------------------------ K1 + K2 --
__global__ void __launch_bounds__(64) blind_rotate_kernel(
    const BrJob* __restrict__ jobs, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf, const c64* __restrict__ tw1,
    const c64* __restrict__ tw2, uint32_t* __restrict__ xout) {
  __shared__ uint32_t acc[2][kPolyN];
  __shared__ c64 xbuf[2][512];
  __shared__ uint16_t bar[kLweWords + 1];
  const int t = threadIdx.x;
  const BrJob job = jobs[blockIdx.x];

  c64 T1[8], T2[8];
  load_twiddles(tw1, tw2, t, T1, T2);

  // K1: combine the gate inputs and mod-switch to Z_2N.
  for (int i = t; i < kLweWords; i += 64) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    bar[i] = (uint16_t)modswitch_2n(v);
  }
  __syncthreads();
  // ACC = X^{-barb} (0, mu * sum X^j)
  {
    const int barb = bar[kN];
    for (int j = t; j < kPolyN; j += 64) {
      acc[0][j] = 0;
      acc[1][j] = (((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu);
    }
  }

  for (int i = 0; i < kN; ++i) {
    __syncthreads();
    const int ai = bar[i];
    if (ai == 0) continue;  // X^0 - 1 = 0: the CMux leaves ACC unchanged
    const c64* bk_i = bkf + (size_t)i * kBkfComplexPerStep;
    c64 af[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) af[0][k] = af[1][k] = c64{0.0, 0.0};

#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      // (X^{a_i} - 1) * ACC_part at the 16 coefficients this thread owns.
      uint32_t dif[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = t + 64 * (q & 7) + (q >> 3) * 512;
        const int m = (j - ai) & (2 * kPolyN - 1);
        const uint32_t r = m < kPolyN ? acc[part][m] : 0u - acc[part][m - kPolyN];
        dif[q] = r - acc[part][j] + kDecompOffset;
      }
#pragma unroll 1
      for (int p = 0; p < kL; ++p) {
        const int shift = 32 - (p + 1) * kBgBit;
        c64 v[8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
          v[a] = {u32_biased_to_double((dif[a] >> shift) & 127u, kDigitBias),
                  u32_biased_to_double((dif[a + 8] >> shift) & 127u, kDigitBias)};
        fwd_stage1(v, T1);
        exchange<1>(v, xbuf[0], t);
        fwd_stage2(v, T2);
        exchange<2>(v, xbuf[1], t);
        fwd_stage3(v);
        const c64* bk_r = bk_i + (size_t)(part * kL + p) * 1024;
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          const c64 b0 = ldg_c64(bk_r + k2 * 128 + t);
          const c64 b1 = ldg_c64(bk_r + k2 * 128 + 64 + t);
          af[0][k2] = cadd(af[0][k2], cmul(v[k2], b0));
          af[1][k2] = cadd(af[1][k2], cmul(v[k2], b1));
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      c64 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = af[o][k];
      inv_stageA(v);
      exchange<2>(v, xbuf[0], t);
      inv_stageB(v, T2);
      exchange<3>(v, xbuf[1], t);
      inv_stageC(v, T1);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int j = t + 64 * a;
        acc[o][j] += round_to_torus(v[a].x);
        acc[o][j + 512] += round_to_torus(v[a].y);
      }
    }
  }
  __syncthreads();
  // Sample extraction: a'_0 = a_0, a'_j = -a_{N-j}, b' = b_0.
  uint32_t* out = xout + (size_t)job.out * kXlweStride;
  for (int j = t; j < kPolyN; j += 64) out[j] = j == 0 ? acc[0][0] : 0u - acc[0][kPolyN - j];
  if (t == 0) out[kPolyN] = acc[1][0];
}

// ------------------------------------------------- K1 + K2, version 2 --
// G bootstraps per CTA (64 threads each, independent named barriers), and the
// bootstrapping key streamed through a ring of S shared-memory stages by the
// bulk-copy engine (cp.async.bulk -> SASS UBLKCP), one 16 KB TRGSW row
// (both output polynomials, all 512 bins) per stage, consumed by all G gates.
// mbarrier "full" (tx-count) / "empty" (64*G arrivals) pairs order the ring.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void group_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
// code = barrier id | (thread count << 8)
__device__ __forceinline__ void group_sync_code(int code) {
  asm volatile("bar.sync %0, %1;" ::"r"(code & 255), "r"(code >> 8) : "memory");
}

template <int kPattern>
__device__ __forceinline__ void exchange_g(c64 v[8], c64* buf, int t, int bar_id) {
#pragma unroll
  for (int z = 0; z < 8; ++z) {
    int cell, slot;
    if (kPattern == 1) {
      cell = ex1_cell(t, z);
      slot = t >> 3;
    } else if (kPattern == 2) {
      cell = ex2_cell(t, z);
      slot = t >> 3;
    } else {
      cell = exB_cell(t, z);
      slot = t & 7;
    }
    buf[xpos(cell, slot)] = v[z];
  }
  group_sync(bar_id);
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = buf[xpos(t, s)];
}

constexpr uint32_t kRowBytes = 1024 * 16;  // one TRGSW row in FFT domain

template <int G, int S, bool kTwS>
struct BrSmem {
  c64 ring[S][1024];
  c64 xbuf[G][2][512];
  c64 tw[kTwS ? 16 : 1][64];  // tw[k][t]: T1 (k 0..7), T2 (k 8..15) when kTwS
  uint32_t acc[G][2][kPolyN];
  uint16_t bar[G][kLweWords + 1];
  uint64_t full[S], empty[S];
};

// kTwS: twiddles read from shared memory instead of 64 registers;
// kMinB: CTAs per SM the register allocation must allow.
template <int G, int S, bool kTwS, int kMinB>
__global__ void __launch_bounds__(64 * G, kMinB) blind_rotate_kernel_v2(
    const BrJob* __restrict__ jobs, int count, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf, const c64* __restrict__ tw1, const c64* __restrict__ tw2,
    uint32_t* __restrict__ xout) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BrSmem<G, S, kTwS>& sm = *reinterpret_cast<BrSmem<G, S, kTwS>*>(smem_raw);
  const int tid = threadIdx.x;
  const int g = tid >> 6, t = tid & 63;
  const int bar_id = 1 + g;
  const int jidx = blockIdx.x * G + g;
  const bool live = jidx < count;
  const BrJob job = jobs[live ? jidx : 0];

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 64 * G);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr int kChunks = kN * kRows;
  if (tid == 0) {
    for (int q = 0; q < S - 1; ++q) {
      mbar_expect_tx(&sm.full[q], kRowBytes);
      bulk_g2s(sm.ring[q], bkf + (size_t)q * 1024, kRowBytes, &sm.full[q]);
    }
  }

  using TwT = std::conditional_t<kTwS, StridedTw, const c64*>;
  c64 T1r[8], T2r[8];
  TwT T1, T2;
  if constexpr (kTwS) {
    for (int e = tid; e < 64 * 8; e += 64 * G) {
      const int tt = e >> 3, k = e & 7;
      sm.tw[k][tt] = tw1[e];
      sm.tw[8 + k][tt] = tw2[e];
    }
    __syncthreads();
    T1 = StridedTw{&sm.tw[0][t]};
    T2 = StridedTw{&sm.tw[8][t]};
  } else {
    load_twiddles(tw1, tw2, t, T1r, T2r);
    T1 = T1r;
    T2 = T2r;
  }
  uint32_t* acc0 = sm.acc[g][0];
  uint32_t* acc1 = sm.acc[g][1];
  uint16_t* bar = sm.bar[g];
  for (int i = t; i < kLweWords; i += 64) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    bar[i] = (uint16_t)modswitch_2n(v);
  }
  group_sync(bar_id);
  {
    const int barb = bar[kN];
    for (int j = t; j < kPolyN; j += 64) {
      acc0[j] = 0;
      acc1[j] = (((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu);
    }
  }

  int q = 0;  // chunk sequence number = i * 6 + row
  for (int i = 0; i < kN; ++i) {
    group_sync(bar_id);
    const int ai = bar[i];
    c64 af[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) af[0][k] = af[1][k] = c64{0.0, 0.0};
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const uint32_t* accp = part ? acc1 : acc0;
      uint32_t dif[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int j = t + 64 * (x & 7) + (x >> 3) * 512;
        const int m = (j - ai) & (2 * kPolyN - 1);
        const uint32_t r = m < kPolyN ? accp[m] : 0u - accp[m - kPolyN];
        dif[x] = r - accp[j] + kDecompOffset;
      }
#pragma unroll 1
      for (int p = 0; p < kL; ++p, ++q) {
        const int shift = 32 - (p + 1) * kBgBit;
        c64 v[8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
          v[a] = {u32_biased_to_double((dif[a] >> shift) & 127u, kDigitBias),
                  u32_biased_to_double((dif[a + 8] >> shift) & 127u, kDigitBias)};
        fwd_stage1(v, T1);
        exchange_g<1>(v, sm.xbuf[g][0], t, bar_id);
        fwd_stage2(v, T2);
        exchange_g<2>(v, sm.xbuf[g][1], t, bar_id);
        fwd_stage3(v);
        // producer: refill the slot chunk q-1 used with chunk q+S-1
        if (tid == 0 && q + S - 1 < kChunks) {
          const int nq = q + S - 1, slot = nq % S;
          if (q >= 1) mbar_wait(&sm.empty[slot], ((q - 1) / S) & 1);
          mbar_expect_tx(&sm.full[slot], kRowBytes);
          bulk_g2s(sm.ring[slot], bkf + (size_t)nq * 1024, kRowBytes, &sm.full[slot]);
        }
        const int slot = q % S;
        mbar_wait(&sm.full[slot], (q / S) & 1);
        const c64* bk_r = sm.ring[slot];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          const c64 b0 = bk_r[k2 * 128 + t];
          const c64 b1 = bk_r[k2 * 128 + 64 + t];
          af[0][k2] = cadd(af[0][k2], cmul(v[k2], b0));
          af[1][k2] = cadd(af[1][k2], cmul(v[k2], b1));
        }
        mbar_arrive(&sm.empty[slot]);
      }
    }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      c64 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = af[o][k];
      inv_stageA(v);
      exchange_g<2>(v, sm.xbuf[g][0], t, bar_id);
      inv_stageB(v, T2);
      exchange_g<3>(v, sm.xbuf[g][1], t, bar_id);
      inv_stageC(v, T1);
      uint32_t* acco = o ? acc1 : acc0;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int j = t + 64 * a;
        acco[j] += round_to_torus(v[a].x);
        acco[j + 512] += round_to_torus(v[a].y);
      }
    }
  }
  group_sync(bar_id);
  if (!live) return;
  uint32_t* out = xout + (size_t)job.out * kXlweStride;
  for (int j = t; j < kPolyN; j += 64) out[j] = j == 0 ? acc0[0] : 0u - acc0[kPolyN - j];
  if (t == 0) out[kPolyN] = acc1[0];
}

// ------------------------------------------------- K1 + K2, version 3 --
// As v2, but every thread runs TWO transforms at once: the forward FFTs of
// the same gadget level of both TRLWE parts (rows p and 3+p), and the two
// inverse FFTs.  Twice the independent FP64 work between barriers, the same
// number of barriers.  Exchange buffers are single-buffered (a WAR barrier
// separates the two exchanges of a transform).  The key ring is consumed in
// pair order (rows 0,3, 1,4, 2,5 of each step).
template <int G, int S, bool kTwS = false>
struct BrSmem3 {
  c64 ring[S][1024];
  c64 xbuf[G][2][512];
  c64 tw[kTwS ? 16 : 1][64];  // tw[k][t] when kTwS
  uint32_t acc[G][2][kPolyN];
  uint16_t bar[G][kLweWords + 1];
  uint64_t full[S], empty[S];
};

// chunk q (0 .. 6n-1) -> TRGSW row offset in the FFT-domain key
__device__ __forceinline__ const c64* chunk_src(const c64* bkf, int q) {
  const int i = q / 6, k = q - 6 * (q / 6);
  const int row = (k & 1) * kL + (k >> 1);
  return bkf + ((size_t)i * kRows + row) * 1024;
}

template <int kPattern>
__device__ __forceinline__ void exchange_pair(c64 va[8], c64 vb[8], c64* ba, c64* bb, int t,
                                              int bar_id) {
#pragma unroll
  for (int z = 0; z < 8; ++z) {
    int cell, slot;
    if (kPattern == 1) {
      cell = ex1_cell(t, z);
      slot = t >> 3;
    } else if (kPattern == 2) {
      cell = ex2_cell(t, z);
      slot = t >> 3;
    } else {
      cell = exB_cell(t, z);
      slot = t & 7;
    }
    ba[xpos(cell, slot)] = va[z];
    bb[xpos(cell, slot)] = vb[z];
  }
  group_sync_code(bar_id);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    va[s] = ba[xpos(t, s)];
    vb[s] = bb[xpos(t, s)];
  }
  group_sync_code(bar_id);  // WAR: all reads done before the buffers are rewritten
}

// kIL (interleaved): warp w holds threads t = 8w..8w+7 of all four gates
// (lane = 8*g + t%8), so the key-row loads of a warp hit 8 distinct
// addresses (broadcast across gates) instead of 32; gates then advance in
// CTA-wide lockstep (bar.sync 0 over 256 threads).
// biased gadget digit u = d + Bg/2 in [0,127] -> double d: bit-pattern
// construction (no conversion unit, costs a register move) or I2F.
template <bool kI2F>
__device__ __forceinline__ double digit_to_double(uint32_t u) {
  if constexpr (kI2F) return (double)(int)(u - 64u);
  else return u32_biased_to_double(u, kDigitBias);
}

template <int G, int S, bool kTwS = false, bool kIL = false, bool kI2F = false,
          int kShift = 0>
__global__ void __launch_bounds__(64 * G) blind_rotate_kernel_v3(
    const BrJob* __restrict__ jobs, int count, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf, const c64* __restrict__ tw1, const c64* __restrict__ tw2,
    uint32_t* __restrict__ xout) {
  static_assert(S >= 4, "pairs need two chunks in flight plus prefetch");
  static_assert(!kIL || G == 4, "interleaving maps 4 gates onto a warp");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BrSmem3<G, S, kTwS>& sm = *reinterpret_cast<BrSmem3<G, S, kTwS>*>(smem_raw);
  const int tid = threadIdx.x;
  const int g = kIL ? ((tid & 31) >> 3) : (tid >> 6);
  const int t = kIL ? (8 * (tid >> 5) + (tid & 7)) : (tid & 63);
  const int bar_id = kIL ? (64 * G) << 8 : ((1 + g) | (64 << 8));
  const int jidx = blockIdx.x * G + g;
  const bool live = jidx < count;
  const BrJob job = jobs[live ? jidx : 0];
  constexpr int kChunks = kN * kRows;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 64 * G);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_expect_tx(&sm.full[q], kRowBytes);
      bulk_g2s(sm.ring[q], chunk_src(bkf, q), kRowBytes, &sm.full[q]);
    }
  }

  using TwT = std::conditional_t<kTwS, StridedTw, const c64*>;
  c64 T1r[8], T2r[8];
  TwT T1, T2;
  if constexpr (kTwS) {
    for (int e = tid; e < 64 * 8; e += 64 * G) {
      const int tt = e >> 3, k = e & 7;
      sm.tw[k][tt] = tw1[e];
      sm.tw[8 + k][tt] = tw2[e];
    }
    __syncthreads();
    T1 = StridedTw{&sm.tw[0][t]};
    T2 = StridedTw{&sm.tw[8][t]};
  } else {
    load_twiddles(tw1, tw2, t, T1r, T2r);
    T1 = T1r;
    T2 = T2r;
  }
  uint32_t* acc0 = sm.acc[g][0];
  uint32_t* acc1 = sm.acc[g][1];
  uint16_t* bar = sm.bar[g];
  c64* xa = sm.xbuf[g][0];
  c64* xb = sm.xbuf[g][1];
  for (int i = t; i < kLweWords; i += 64) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    bar[i] = (uint16_t)modswitch_2n(v);
  }
  group_sync_code(bar_id);
  {
    const int barb = bar[kN];
    for (int j = t; j < kPolyN; j += 64) {
      acc0[j] = 0;
      acc1[j] = (((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu);
    }
  }

  if constexpr (kShift > 0) {
    // Offset gates 2,3 (which share SM sub-partitions with gates 0,1) by a
    // fraction of a transform stage, so one gate's FP64 phase overlaps the
    // other's shared-memory exchange instead of contending for the same pipe.
    if (g >= 2) {
      const long long t0 = clock64();
      while (clock64() - t0 < kShift) {
      }
    }
  }
  int q = 0;  // chunk sequence number (pair order)
  for (int i = 0; i < kN; ++i) {
    group_sync_code(bar_id);
    const int ai = bar[i];
    c64 af[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) af[0][k] = af[1][k] = c64{0.0, 0.0};
#pragma unroll 1
    for (int p = 0; p < kL; ++p, q += 2) {
      const int shift = 32 - (p + 1) * kBgBit;
      c64 va[8], vb[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        // digits of (X^ai - 1) * ACC at coefficients j and j + 512, both parts
        const int j = t + 64 * x;
        const int m0 = (j - ai) & (2 * kPolyN - 1);
        const int m1 = (j + 512 - ai) & (2 * kPolyN - 1);
        const uint32_t ra0 = m0 < kPolyN ? acc0[m0] : 0u - acc0[m0 - kPolyN];
        const uint32_t ra1 = m1 < kPolyN ? acc0[m1] : 0u - acc0[m1 - kPolyN];
        const uint32_t rb0 = m0 < kPolyN ? acc1[m0] : 0u - acc1[m0 - kPolyN];
        const uint32_t rb1 = m1 < kPolyN ? acc1[m1] : 0u - acc1[m1 - kPolyN];
        const uint32_t da0 = ra0 - acc0[j] + kDecompOffset;
        const uint32_t da1 = ra1 - acc0[j + 512] + kDecompOffset;
        const uint32_t db0 = rb0 - acc1[j] + kDecompOffset;
        const uint32_t db1 = rb1 - acc1[j + 512] + kDecompOffset;
        va[x] = {digit_to_double<kI2F>((da0 >> shift) & 127u),
                 digit_to_double<kI2F>((da1 >> shift) & 127u)};
        vb[x] = {digit_to_double<kI2F>((db0 >> shift) & 127u),
                 digit_to_double<kI2F>((db1 >> shift) & 127u)};
      }
      fwd_stage1(va, T1);
      fwd_stage1(vb, T1);
      exchange_pair<1>(va, vb, xa, xb, t, bar_id);
      fwd_stage2(va, T2);
      fwd_stage2(vb, T2);
      exchange_pair<2>(va, vb, xa, xb, t, bar_id);
      fwd_stage3(va);
      fwd_stage3(vb);
      // producer: refill the slots of chunks q-2, q-1 with chunks q+S-2, q+S-1
      if (tid == 0) {
#pragma unroll
        for (int c = q - 2; c < q; ++c) {
          if (c < 0 || c + S >= kChunks) continue;
          const int slot = c % S;
          mbar_wait(&sm.empty[slot], (c / S) & 1);
          mbar_expect_tx(&sm.full[slot], kRowBytes);
          bulk_g2s(sm.ring[slot], chunk_src(bkf, c + S), kRowBytes, &sm.full[slot]);
        }
      }
      const int sa = q % S, sb = (q + 1) % S;
      mbar_wait(&sm.full[sa], (q / S) & 1);
      mbar_wait(&sm.full[sb], ((q + 1) / S) & 1);
      const c64* bka = sm.ring[sa];
      const c64* bkb = sm.ring[sb];
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        const c64 a0 = bka[k2 * 128 + t], a1 = bka[k2 * 128 + 64 + t];
        const c64 b0 = bkb[k2 * 128 + t], b1 = bkb[k2 * 128 + 64 + t];
        af[0][k2] = cadd(cadd(af[0][k2], cmul(va[k2], a0)), cmul(vb[k2], b0));
        af[1][k2] = cadd(cadd(af[1][k2], cmul(va[k2], a1)), cmul(vb[k2], b1));
      }
      mbar_arrive(&sm.empty[sa]);
      mbar_arrive(&sm.empty[sb]);
    }
    inv_stageA(af[0]);
    inv_stageA(af[1]);
    exchange_pair<2>(af[0], af[1], xa, xb, t, bar_id);
    inv_stageB(af[0], T2);
    inv_stageB(af[1], T2);
    exchange_pair<3>(af[0], af[1], xa, xb, t, bar_id);
    inv_stageC(af[0], T1);
    inv_stageC(af[1], T1);
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int j = t + 64 * a;
      acc0[j] += round_to_torus(af[0][a].x);
      acc0[j + 512] += round_to_torus(af[0][a].y);
      acc1[j] += round_to_torus(af[1][a].x);
      acc1[j + 512] += round_to_torus(af[1][a].y);
    }
  }
  group_sync_code(bar_id);
  if (!live) return;
  uint32_t* out = xout + (size_t)job.out * kXlweStride;
  for (int j = t; j < kPolyN; j += 64) out[j] = j == 0 ? acc0[0] : 0u - acc0[kPolyN - j];
  if (t == 0) out[kPolyN] = acc1[0];
}

// ---------------------------------------- K1 + K2, latency ("wide") --
// One bootstrap per CTA of 384 threads for narrow levels (the emulator's
// instruction stream averages ~90 gates per dataflow level): the six gadget
// rows of a CMux step are transformed concurrently, one 64-thread group per
// row; partial products are reduced through shared memory; groups 0 and 1
// run the two inverse transforms.  Each group streams its own 16 KB key row
// for the next step with a bulk copy as soon as it has consumed the current
// one.  Per-step latency ~ 1 forward + 1 inverse transform instead of 8.
struct WideSmem {
  c64 bkbuf[kRows][1024];   // 96 KB: this step's six TRGSW rows
  c64 xbuf[kRows][512];     // 48 KB: one exchange buffer per group
  c64 red[kL][2][8][64];    // 48 KB: partial sums [pair][o][k2][t]
  uint32_t acc[2][kPolyN];
  uint16_t bar[kLweWords + 1];
  uint64_t full[kRows];
};

__global__ void __launch_bounds__(64 * kRows, 1) blind_rotate_wide_kernel(
    const BrJob* __restrict__ jobs, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf, const c64* __restrict__ tw1, const c64* __restrict__ tw2,
    uint32_t* __restrict__ xout) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WideSmem& sm = *reinterpret_cast<WideSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int g = tid >> 6, t = tid & 63;  // group g transforms gadget row g
  const int bar_id = 1 + g;
  const int part = g / kL, p = g % kL;
  const BrJob job = jobs[blockIdx.x];

  if (tid == 0) {
    for (int r = 0; r < kRows; ++r) mbar_init(&sm.full[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(&sm.full[g], kRowBytes);
    bulk_g2s(sm.bkbuf[g], bkf + (size_t)g * 1024, kRowBytes, &sm.full[g]);
  }
  c64 T1[8], T2[8];
  load_twiddles(tw1, tw2, t, T1, T2);
  for (int i = tid; i < kLweWords; i += 64 * kRows) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    sm.bar[i] = (uint16_t)modswitch_2n(v);
  }
  __syncthreads();
  {
    const int barb = sm.bar[kN];
    for (int j = tid; j < kPolyN; j += 64 * kRows) {
      sm.acc[0][j] = 0;
      sm.acc[1][j] = (((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu);
    }
  }
  const int shift = 32 - (p + 1) * kBgBit;
  c64* xb = sm.xbuf[g];

  for (int i = 0; i < kN; ++i) {
    __syncthreads();  // ACC of the previous step complete
    const int ai = sm.bar[i];
    const uint32_t* accp = sm.acc[part];
    c64 v[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      uint32_t d[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = t + 64 * a + 512 * h;
        const int m = (j - ai) & (2 * kPolyN - 1);
        const uint32_t r = m < kPolyN ? accp[m] : 0u - accp[m - kPolyN];
        d[h] = ((r - accp[j] + kDecompOffset) >> shift) & 127u;
      }
      v[a] = {u32_biased_to_double(d[0], kDigitBias), u32_biased_to_double(d[1], kDigitBias)};
    }
    fwd_stage1(v, T1);
    exchange_g<1>(v, xb, t, bar_id);
    group_sync(bar_id);  // WAR on the single exchange buffer
    fwd_stage2(v, T2);
    exchange_g<2>(v, xb, t, bar_id);
    fwd_stage3(v);
    // partial products of this row with both output polynomials
    mbar_wait(&sm.full[g], i & 1);
    const c64* bk = sm.bkbuf[g];
    c64 pa[8], pb[8];
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      pa[k2] = cmul(v[k2], bk[k2 * 128 + t]);
      pb[k2] = cmul(v[k2], bk[k2 * 128 + 64 + t]);
    }
    group_sync(bar_id);  // the whole group has read its key row
    if (t == 0 && i + 1 < kN) {
      mbar_expect_tx(&sm.full[g], kRowBytes);
      bulk_g2s(sm.bkbuf[g], bkf + ((size_t)(i + 1) * kRows + g) * 1024, kRowBytes, &sm.full[g]);
    }
    // two-phase reduction of the six partials into three pair sums
    if (part == 1) {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        sm.red[p][0][k2][t] = pa[k2];
        sm.red[p][1][k2][t] = pb[k2];
      }
    }
    __syncthreads();
    if (part == 0) {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        sm.red[p][0][k2][t] = cadd(sm.red[p][0][k2][t], pa[k2]);
        sm.red[p][1][k2][t] = cadd(sm.red[p][1][k2][t], pb[k2]);
      }
    }
    __syncthreads();
    if (g < 2) {  // group o = g: inverse transform of output polynomial o
      const int o = g;
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2)
        v[k2] = cadd(cadd(sm.red[0][o][k2][t], sm.red[1][o][k2][t]), sm.red[2][o][k2][t]);
      inv_stageA(v);
      exchange_g<2>(v, sm.xbuf[g], t, bar_id);
      inv_stageB(v, T2);
      exchange_g<3>(v, sm.xbuf[g + 2], t, bar_id);
      inv_stageC(v, T1);
      uint32_t* acco = sm.acc[o];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int j = t + 64 * a;
        acco[j] += round_to_torus(v[a].x);
        acco[j + 512] += round_to_torus(v[a].y);
      }
    }
  }
  __syncthreads();
  uint32_t* out = xout + (size_t)job.out * kXlweStride;
  for (int j = tid; j < kPolyN; j += 64 * kRows)
    out[j] = j == 0 ? sm.acc[0][0] : 0u - sm.acc[0][kPolyN - j];
  if (tid == 0) out[kPolyN] = sm.acc[1][0];
}

static cudaError_t launch_wide(const BrJob* jobs, int count, const uint32_t* slab,
                               const c64* bkf, const c64* tw1, const c64* tw2, uint32_t* xout,
                               cudaStream_t s) {
  static bool configured = false;
  const int smem = int(sizeof(WideSmem));
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(blind_rotate_wide_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  blind_rotate_wide_kernel<<<count, 64 * kRows, smem, s>>>(jobs, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

// ------------------------------------------------------------ K3 + K4 --
__global__ void __launch_bounds__(kKsThreads) key_switch_kernel(
    const KsJob* __restrict__ jobs, const uint32_t* __restrict__ xlwe,
    const uint4* __restrict__ ksk, uint32_t* __restrict__ slab) {
  __shared__ uint32_t x[kXlweWords];
  const int t = threadIdx.x;
  const KsJob job = jobs[blockIdx.x];
  for (int i = t; i < kXlweWords; i += kKsThreads) {
    uint32_t v = xlwe[(size_t)job.x[0] * kXlweStride + i];
    if (job.x[1] != kNoInput) v += xlwe[(size_t)job.x[1] * kXlweStride + i];
    if (i == kPolyN) v += job.cst;
    x[i] = v;
  }
  __syncthreads();
  constexpr int kRowVec = kKskRowStride / 4;  // 158 uint4 per row
  if (t >= kRowVec) return;
  uint4 a = {0u, 0u, 0u, 0u};
  if (t == kN / 4) a.z = x[kPolyN];  // column 630 holds b
  const uint32_t prec = 1u << (32 - (1 + kKsBaseBit * kKsT));
#pragma unroll 2
  for (int i = 0; i < kPolyN; ++i) {
    const uint32_t abar = x[i] + prec;
    const uint4* base = ksk + (size_t)i * (kKsT * kKsBase * kRowVec) + t;
#pragma unroll
    for (int j = 0; j < kKsT; ++j) {
      const uint32_t d = (abar >> (32 - (j + 1) * kKsBaseBit)) & (kKsBase - 1);
      const uint4 r = __ldg(base + (j * kKsBase + d) * kRowVec);  // d = 0 row is zero
      a.x -= r.x;
      a.y -= r.y;
      a.z -= r.z;
      a.w -= r.w;
    }
  }
  reinterpret_cast<uint4*>(slab + (size_t)job.out_slot * kLweStride)[t] = a;
}

// ------------------------------------------------- FP64 pipe peak probe --
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

cudaError_t launch_fp64_peak(double* out, int blocks, int iters, cudaStream_t s) {
  fp64_peak_kernel<<<blocks, 256, 0, s>>>(out, iters);
  return cudaGetLastError();
}

// --------------------------------------------- K3 + K4, latency ("wide") --
// One key switch per CTA of 6 x 158 threads: the 1024 input coefficients are
// split into 6 position groups that gather concurrently, then reduced through
// shared memory -- ~6x shorter dependent load chain for narrow levels.
constexpr int kKsWidePG = 6;
constexpr int kKsWideThreads = kKsWidePG * (kKskRowStride / 4);  // 948

__global__ void __launch_bounds__(kKsWideThreads) key_switch_wide_kernel(
    const KsJob* __restrict__ jobs, const uint32_t* __restrict__ xlwe,
    const uint4* __restrict__ ksk, uint32_t* __restrict__ slab) {
  constexpr int kRowVec = kKskRowStride / 4;
  __shared__ uint32_t x[kXlweWords];
  __shared__ uint4 part[kKsWidePG - 1][kRowVec];
  const int tid = threadIdx.x;
  const int col = tid % kRowVec, pg = tid / kRowVec;
  const KsJob job = jobs[blockIdx.x];
  for (int i = tid; i < kXlweWords; i += kKsWideThreads) {
    uint32_t v = xlwe[(size_t)job.x[0] * kXlweStride + i];
    if (job.x[1] != kNoInput) v += xlwe[(size_t)job.x[1] * kXlweStride + i];
    if (i == kPolyN) v += job.cst;
    x[i] = v;
  }
  __syncthreads();
  uint4 a = {0u, 0u, 0u, 0u};
  const uint32_t prec = 1u << (32 - (1 + kKsBaseBit * kKsT));
  const int i0 = pg * kPolyN / kKsWidePG, i1 = (pg + 1) * kPolyN / kKsWidePG;
#pragma unroll 2
  for (int i = i0; i < i1; ++i) {
    const uint32_t abar = x[i] + prec;
    const uint4* base = ksk + (size_t)i * (kKsT * kKsBase * kRowVec) + col;
#pragma unroll
    for (int j = 0; j < kKsT; ++j) {
      const uint32_t d = (abar >> (32 - (j + 1) * kKsBaseBit)) & (kKsBase - 1);
      const uint4 r = __ldg(base + (j * kKsBase + d) * kRowVec);
      a.x -= r.x;
      a.y -= r.y;
      a.z -= r.z;
      a.w -= r.w;
    }
  }
  if (pg > 0) part[pg - 1][col] = a;
  __syncthreads();
  if (pg == 0) {
#pragma unroll
    for (int k = 0; k < kKsWidePG - 1; ++k) {
      const uint4 r = part[k][col];
      a.x += r.x;
      a.y += r.y;
      a.z += r.z;
      a.w += r.w;
    }
    if (col == kN / 4) a.z += x[kPolyN];  // column 630 holds b
    reinterpret_cast<uint4*>(slab + (size_t)job.out_slot * kLweStride)[col] = a;
  }
}

// ------------------------------------------------- K3 + K4, multi-gate --
// GK key switches per CTA.  For every digit position (i, j) the three
// non-zero KSK rows are loaded once (3 x 16 B per thread) and reused by all
// GK gates, whose digit selects the row with a warp-uniform branch: L1/L2
// traffic drops from 0.75*GK rows to 3 rows per position.
template <int GK>
__global__ void __launch_bounds__(kKsThreads) key_switch_multi_kernel(
    const KsJob* __restrict__ jobs, int count, const uint32_t* __restrict__ xlwe,
    const uint4* __restrict__ ksk, uint32_t* __restrict__ slab) {
  __shared__ __align__(16) uint32_t xs[kPolyN][GK];  // abar = a_i + 2^15, per gate
  __shared__ uint32_t bs[GK];
  const int t = threadIdx.x;
  const int first = blockIdx.x * GK;
  const int live = min(GK, count - first);
  for (int e = t; e < GK * kXlweWords; e += kKsThreads) {
    const int g = e / kXlweWords, i = e - g * kXlweWords;
    if (g >= live) continue;
    const KsJob& job = jobs[first + g];
    uint32_t v = xlwe[(size_t)job.x[0] * kXlweStride + i];
    if (job.x[1] != kNoInput) v += xlwe[(size_t)job.x[1] * kXlweStride + i];
    if (i == kPolyN) bs[g] = v + job.cst;
    else xs[i][g] = v + (1u << (32 - (1 + kKsBaseBit * kKsT)));
  }
  __syncthreads();
  constexpr int kRowVec = kKskRowStride / 4;
  if (t >= kRowVec) return;
  uint4 acc[GK];
#pragma unroll
  for (int g = 0; g < GK; ++g) acc[g] = make_uint4(0, 0, 0, 0);
  if (t == kN / 4) {
#pragma unroll
    for (int g = 0; g < GK; ++g) acc[g].z = g < live ? bs[g] : 0u;
  }
  for (int i = 0; i < kPolyN; ++i) {
    uint32_t ab[GK];
#pragma unroll
    for (int g = 0; g < GK; ++g) ab[g] = xs[i][g];
    const uint4* base = ksk + (size_t)i * (kKsT * kKsBase * kRowVec) + t;
#pragma unroll 2
    for (int j = 0; j < kKsT; ++j) {
      const uint4* rows = base + j * kKsBase * kRowVec;
      const uint4 r1 = __ldg(rows + 1 * kRowVec);
      const uint4 r2 = __ldg(rows + 2 * kRowVec);
      const uint4 r3 = __ldg(rows + 3 * kRowVec);
      const int sh = 32 - (j + 1) * kKsBaseBit;
#pragma unroll
      for (int g = 0; g < GK; ++g) {
        const uint32_t d = (ab[g] >> sh) & 3u;
        const uint4 r = d == 1 ? r1 : (d == 2 ? r2 : r3);
        if (d) {
          acc[g].x -= r.x;
          acc[g].y -= r.y;
          acc[g].z -= r.z;
          acc[g].w -= r.w;
        }
      }
    }
  }
#pragma unroll
  for (int g = 0; g < GK; ++g)
    if (g < live)
      reinterpret_cast<uint4*>(slab + (size_t)jobs[first + g].out_slot * kLweStride)[t] = acc[g];
}

// ----------------------------------------------------------- launchers --
cudaError_t launch_bk_to_fft(const uint32_t* bk, const c64* tw1, const c64* tw2, c64* bkf,
                             cudaStream_t s) {
  bk_to_fft_kernel<<<kN * kRows * 2, 64, 0, s>>>(bk, tw1, tw2, bkf);
  return cudaGetLastError();
}
template <int G, int S, bool kTwS = false, int kMinB = 1>
static cudaError_t launch_v2(const BrJob* jobs, int count, const uint32_t* slab, const c64* bkf,
                             const c64* tw1, const c64* tw2, uint32_t* xout, cudaStream_t s) {
  static bool configured = false;
  const int smem = int(sizeof(BrSmem<G, S, kTwS>));
  auto* kern = blind_rotate_kernel_v2<G, S, kTwS, kMinB>;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<(count + G - 1) / G, 64 * G, smem, s>>>(jobs, count, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

template <int G, int S, bool kTwS = false, bool kIL = false, bool kI2F = false,
          int kShift = 0>
static cudaError_t launch_v3(const BrJob* jobs, int count, const uint32_t* slab, const c64* bkf,
                             const c64* tw1, const c64* tw2, uint32_t* xout, cudaStream_t s) {
  static bool configured = false;
  const int smem = int(sizeof(BrSmem3<G, S, kTwS>));
  auto* kern = blind_rotate_kernel_v3<G, S, kTwS, kIL, kI2F, kShift>;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<(count + G - 1) / G, 64 * G, smem, s>>>(jobs, count, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

static int g_br_variant = -1;
int br_variant() {
  if (g_br_variant < 0) {
    const char* e = getenv("CVM_BR_KERNEL");
    g_br_variant = e ? atoi(e) : kDefaultBrVariant;
  }
  return g_br_variant;
}
void set_br_variant(int v) { g_br_variant = v; }
int default_br_variant() { return kDefaultBrVariant; }

cudaError_t launch_blind_rotate(const BrJob* jobs, int count, const uint32_t* slab,
                                const c64* bkf, const c64* tw1, const c64* tw2,
                                uint32_t* xout, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  int variant = br_variant();
  if (variant == 0) {
    // auto: narrow levels spread one bootstrap per CTA over as many SMs as
    // possible (latency); wide levels use the throughput kernel.
    variant = count <= 148 ? 9 : count <= 2 * 148 ? 13 : 3044;
  }
  switch (variant) {
    case 9: return launch_wide(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 1:
      blind_rotate_kernel<<<count, 64, 0, s>>>(jobs, slab, bkf, tw1, tw2, xout);
      return cudaGetLastError();
    case 22: return launch_v2<2, 2>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 23: return launch_v2<2, 3>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 43: return launch_v2<4, 3>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 13: return launch_v2<1, 3>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    // twiddles in shared memory, with / without a higher occupancy target
    case 123: return launch_v2<2, 3, true, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 1233: return launch_v2<2, 3, true, 3>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 143: return launch_v2<4, 3, true, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 1432: return launch_v2<4, 3, true, 2>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 2233: return launch_v2<2, 3, false, 3>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    // 12 warps per SM: 2 CTAs x 3 gates or 1 CTA x 6 gates (170 registers)
    case 322: return launch_v2<3, 2, false, 2>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 640: return launch_v2<6, 4, false, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 631: return launch_v2<6, 3, true, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 531: return launch_v2<5, 3, true, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 530: return launch_v2<5, 3, false, 1>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    // v3: paired transforms per thread
    case 3044: return launch_v3<4, 4>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3045: return launch_v3<4, 5>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3024: return launch_v3<2, 4>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3144: return launch_v3<4, 4, true>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3244: return launch_v3<4, 4, false, true>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3344: return launch_v3<4, 4, true, true>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3444:
      return launch_v3<4, 4, false, false, true>(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 3544:
      return launch_v3<4, 4, false, false, false, 400>(jobs, count, slab, bkf, tw1, tw2, xout,
                                                       s);
    case 3644:
      return launch_v3<4, 4, false, false, false, 1200>(jobs, count, slab, bkf, tw1, tw2, xout,
                                                        s);
    case 3744:
      return launch_v3<4, 4, false, false, false, 3000>(jobs, count, slab, bkf, tw1, tw2, xout,
                                                        s);
    default: return cudaErrorInvalidValue;
  }
}
cudaError_t launch_key_switch(const KsJob* jobs, int count, const uint32_t* xlwe,
                              const uint32_t* ksk, uint32_t* slab, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const uint4* k4 = reinterpret_cast<const uint4*>(ksk);
  int variant = ks_variant();
  if (variant == 0) variant = count <= 2 * 148 ? 6 : 1;  // auto by level width
  switch (variant) {
    case 1:
      key_switch_kernel<<<count, kKsThreads, 0, s>>>(jobs, xlwe, k4, slab);
      break;
    case 6:
      key_switch_wide_kernel<<<count, kKsWideThreads, 0, s>>>(jobs, xlwe, k4, slab);
      break;
    case 4:
      key_switch_multi_kernel<4><<<(count + 3) / 4, kKsThreads, 0, s>>>(jobs, count, xlwe, k4,
                                                                      slab);
      break;
    case 8:
      key_switch_multi_kernel<8><<<(count + 7) / 8, kKsThreads, 0, s>>>(jobs, count, xlwe, k4,
                                                                      slab);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

static int g_ks_variant = -1;
int ks_variant() {
  if (g_ks_variant < 0) {
    const char* e = getenv("CVM_KS_KERNEL");
    g_ks_variant = e ? atoi(e) : kDefaultKsVariant;
  }
  return g_ks_variant;
}
void set_ks_variant(int v) { g_ks_variant = v; }

}  // namespace cvm
