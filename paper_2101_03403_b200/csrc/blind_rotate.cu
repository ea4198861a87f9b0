// sm_100a blind-rotation kernels of the batched TFHE gate-bootstrapping path.
//
//   bk_to_fft_kernel        K5  one-time: BK (time domain, u32) -> folded FFT
//                               domain, pre-scaled by 1/M, per-thread bin order.
//   blind_rotate_kernel*    K1+K2 fused: gate-input combination + mod-switch
//                               prologue, 630 CMux steps (gadget decomposition,
//                               6 forward FFTs, 12 complex MACs against BK_i,
//                               2 inverse FFTs, exact rounding), sample
//                               extraction.  Organisations in this file (the
//                               64-thread FFT of fft512.cuh):
//        v3   (5247) 4 bootstraps per CTA sharing a bulk-copy shared-memory key
//             ring, two transforms in flight per thread, generated twiddles
//             (the remainder of a wide level after its full v4 waves);
//        wide (9) one bootstrap on 384 threads, the six gadget rows transformed
//             concurrently (latency, 75-148 and 223-296 bootstraps);
//        pair (96) one bootstrap on a 2-SM cluster (latency, <= 74 and 149-222
//             bootstraps: rounds of 74; schedule.hpp br_latency_pair).
//   The throughput kernel (v4, one bootstrap per warp) is blind_rotate_v4.cu.
//   Retired round-1 organisations (v1: key through L1; v2: the ring without
//   paired transforms) are measured in profiles/r01_variant_sweep.txt.
//
// All variants produce bit-identical ciphertexts (tests/test_gpu_parity.py).
// DESIGN.md section 4 gives the roofline of each kernel; measured variant
// comparisons are in profiles/r01_variant_sweep.txt.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "br_common.cuh"
#include "fft512.cuh"
#include "kernels.cuh"
#include "sm100.cuh"

namespace cvm {

__device__ __forceinline__ void load_twiddles(const c64* tw1, const c64* tw2, int t,
                                              c64 T1[8], c64 T2[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T1[k] = ldg_c64(tw1 + t * 8 + k);
    T2[k] = ldg_c64(tw2 + t * 8 + k);
  }
}

// The three exchange patterns of fft512.cuh: 1 = forward ex1, 2 = forward
// ex2 / inverse exA, 3 = inverse exB.
template <int kPattern>
__device__ __forceinline__ int ex_pos(int t, int z) {
  if (kPattern == 1) return xpos(ex1_cell(t, z), t >> 3);
  if (kPattern == 2) return xpos(ex2_cell(t, z), t >> 3);
  return xpos(exB_cell(t, z), t & 7);
}

// One exchange through a shared buffer; `sync` is __syncthreads or a named
// group barrier.  The caller guarantees the buffer is not being read.
template <int kPattern, class Sync>
__device__ __forceinline__ void exchange(c64 v[8], c64* buf, int t, Sync sync) {
#pragma unroll
  for (int z = 0; z < 8; ++z) buf[ex_pos<kPattern>(t, z)] = v[z];
  sync();
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = buf[xpos(t, s)];
}

// Two transforms exchanged together through two single buffers; the trailing
// barrier protects the buffers for the next exchange (write-after-read).
template <int kPattern>
__device__ __forceinline__ void exchange_pair(c64 va[8], c64 vb[8], c64* ba, c64* bb, int t,
                                              int bar_id) {
#pragma unroll
  for (int z = 0; z < 8; ++z) {
    const int pos = ex_pos<kPattern>(t, z);
    ba[pos] = va[z];
    bb[pos] = vb[z];
  }
  group_sync(bar_id);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    va[s] = ba[xpos(t, s)];
    vb[s] = bb[xpos(t, s)];
  }
  group_sync(bar_id);
}

// 16 digit-pairs of (X^ai - 1) * ACC_part owned by thread t (coefficients
// t + 64a and t + 64a + 512), offset for the gadget decomposition.
__device__ __forceinline__ void rotated_diff(const uint32_t* accp, int ai, int t,
                                             uint32_t dif[16]) {
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    const int j = t + 64 * (x & 7) + (x >> 3) * 512;
    const int m = (j - ai) & (2 * kPolyN - 1);
    const uint32_t r = m < kPolyN ? accp[m] : 0u - accp[m - kPolyN];
    dif[x] = r - accp[j] + kDecompOffset;
  }
}

__device__ __forceinline__ void digits(const uint32_t dif[16], int shift, c64 v[8]) {
#pragma unroll
  for (int a = 0; a < 8; ++a)
    v[a] = {u32_biased_to_double((dif[a] >> shift) & 127u, kDigitBias),
            u32_biased_to_double((dif[a + 8] >> shift) & 127u, kDigitBias)};
}

// acc += round(v) for the 16 coefficients thread t owns.
__device__ __forceinline__ void add_rounded(uint32_t* acc, const c64 v[8], int t) {
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int j = t + 64 * a;
    acc[j] += round_to_torus(v[a].x);
    acc[j + 512] += round_to_torus(v[a].y);
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
  auto sync = [] { __syncthreads(); };
  fwd_stage1(v, T1);
  exchange<1>(v, xbuf[0], t, sync);
  fwd_stage2(v, T2);
  exchange<2>(v, xbuf[1], t, sync);
  fwd_stage3(v);
  const double s = 1.0 / kFftM;
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2)
    bkf[((size_t)ir * 8 + k2) * 128 + o * 64 + t] = {v[k2].x * s, v[k2].y * s};
}

// Resident bases of the generated twiddles (kTwRec): T1[k] = t1b * t1w^k,
// T2[k] = t2w^k (see TwPow8).
struct TwBases {
  c64 t1b, t1w, t2w;
};
__device__ __forceinline__ TwBases tw_bases(const c64* tw1, int t) {
  TwBases b;
  b.t1b = ldg_c64(tw1 + t * 8);  // w^t (the fold twist), exact table value
  double s, c;
  sincospi(-double(t) / 256.0, &s, &c);  // W_512^t
  b.t1w = {c, s};
  sincospi(-double(t >> 3) / 32.0, &s, &c);  // W_512^(8 (t>>3))
  b.t2w = {c, s};
  return b;
}

// ---------------------------------------------------------- K1 + K2, v3 --
// G bootstraps per CTA share a bulk-copy key ring, and every thread runs two
// transforms at once: the forward FFTs of the same gadget level of both TRLWE
// parts (rows p and 3+p), and the two inverse FFTs -- twice the independent
// FP64 work between barriers, the same number of barriers.  Exchange buffers are single-buffered (a WAR barrier
// follows each exchange).  The key ring is consumed in pair order (rows 0,3,
// 1,4, 2,5 of each step) and the producer keeps one pair in flight.
template <int G, int S>
struct BrSmem3 {
  c64 ring[S][1024];
  c64 xbuf[G][2][512];
  uint32_t acc[G][2][kPolyN];
  uint16_t bar[G][kLweWords + 1];
  uint64_t full[S];
  uint32_t cnt[S];  // readers done with each slot
};

// chunk q (0 .. 6n-1, pair order) -> TRGSW row in the FFT-domain key
__device__ __forceinline__ const c64* chunk_src(const c64* bkf, int q) {
  const int i = q / 6, k = q - 6 * (q / 6);
  const int row = (k & 1) * kL + (k >> 1);
  return bkf + ((size_t)i * kRows + row) * 1024;
}

// The remainder kernel of wide levels (variant 5247: G = 4 bootstraps per
// CTA on a 7-row ring): twiddles generated on use (TwPow8, 12 resident
// registers instead of 64), the rotated accumulator differences held across
// the three gadget levels, and each key slot refilled by its last reader.
template <int G, int S>
__global__ void __launch_bounds__(64 * G, 1) blind_rotate_kernel_v3(
    const BrJob* __restrict__ jobs, int count, const uint32_t* __restrict__ slab,
    const c64* __restrict__ bkf, const c64* __restrict__ tw1, const c64* __restrict__ tw2,
    uint32_t* __restrict__ xout) {
  static_assert(S >= 4, "pairs need two chunks in flight plus prefetch");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BrSmem3<G, S>& sm = *reinterpret_cast<BrSmem3<G, S>*>(smem_raw);
  const int tid = threadIdx.x;
  const int g = tid >> 6, t = tid & 63;
  const int bar_id = 1 + g;
  const int jidx = blockIdx.x * G + g;
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
      bulk_g2s(sm.ring[q], chunk_src(bkf, q), kRowBytes, &sm.full[q]);
    }
  }
  // T1[k] = t1b * t1w^k, T2[k] = t2w^k
  const TwBases twb = tw_bases(tw1, t);
  const c64 t1b = twb.t1b, t1w = twb.t1w, t2w = twb.t2w;
  uint32_t* acc0 = sm.acc[g][0];
  uint32_t* acc1 = sm.acc[g][1];
  uint16_t* bar = sm.bar[g];
  c64* xa = sm.xbuf[g][0];
  c64* xb = sm.xbuf[g][1];
  prologue(job, slab, bar, acc0, acc1, t, 64, group_sync, bar_id);

  int q = 0;
  for (int i = 0; i < kN; ++i) {
    group_sync(bar_id);
    const int ai = bar[i];
    c64 af[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) af[0][k] = af[1][k] = c64{0.0, 0.0};
    // (X^ai - 1) * ACC at coefficients j and j + 512 of both parts, offset
    // for the decomposition; the 32 words are kept for the three gadget
    // levels instead of re-reading the accumulator per level
    auto rot_diff = [&](int x, uint32_t& da0, uint32_t& da1, uint32_t& db0, uint32_t& db1) {
      const int j = t + 64 * x;
      const int m0 = (j - ai) & (2 * kPolyN - 1);
      const int m1 = (j + 512 - ai) & (2 * kPolyN - 1);
      const uint32_t ra0 = m0 < kPolyN ? acc0[m0] : 0u - acc0[m0 - kPolyN];
      const uint32_t ra1 = m1 < kPolyN ? acc0[m1] : 0u - acc0[m1 - kPolyN];
      const uint32_t rb0 = m0 < kPolyN ? acc1[m0] : 0u - acc1[m0 - kPolyN];
      const uint32_t rb1 = m1 < kPolyN ? acc1[m1] : 0u - acc1[m1 - kPolyN];
      da0 = ra0 - acc0[j] + kDecompOffset;
      da1 = ra1 - acc0[j + 512] + kDecompOffset;
      db0 = rb0 - acc1[j] + kDecompOffset;
      db1 = rb1 - acc1[j + 512] + kDecompOffset;
    };
    uint32_t dh[8][4];
#pragma unroll
    for (int x = 0; x < 8; ++x) rot_diff(x, dh[x][0], dh[x][1], dh[x][2], dh[x][3]);
#pragma unroll 1
    for (int p = 0; p < kL; ++p, q += 2) {
      const int shift = 32 - (p + 1) * kBgBit;
      c64 va[8], vb[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const uint32_t da0 = dh[x][0], da1 = dh[x][1], db0 = dh[x][2], db1 = dh[x][3];
        va[x] = {u32_biased_to_double((da0 >> shift) & 127u, kDigitBias),
                 u32_biased_to_double((da1 >> shift) & 127u, kDigitBias)};
        vb[x] = {u32_biased_to_double((db0 >> shift) & 127u, kDigitBias),
                 u32_biased_to_double((db1 >> shift) & 127u, kDigitBias)};
      }
      {
        const TwPow8 w1(t1b, t1w);
        fwd_stage1(va, w1);
        fwd_stage1(vb, w1);
      }
      exchange_pair<1>(va, vb, xa, xb, t, bar_id);
      {
        const TwPow8 w2(t2w);
        fwd_stage2(va, w2);
        fwd_stage2(vb, w2);
      }
      exchange_pair<2>(va, vb, xa, xb, t, bar_id);
      fwd_stage3(va);
      fwd_stage3(vb);
      const int sa = q % S, sb = (q + 1) % S;
      mbar_wait(&sm.full[sa], (q / S) & 1);
      mbar_wait(&sm.full[sb], ((q + 1) / S) & 1);
      const c64* bka = sm.ring[sa];
      const c64* bkb = sm.ring[sb];
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        const c64 a0 = bka[k2 * 128 + t], a1 = bka[k2 * 128 + 64 + t];
        const c64 b0 = bkb[k2 * 128 + t], b1 = bkb[k2 * 128 + 64 + t];
        af[0][k2] = cmac(cmac(af[0][k2], va[k2], a0), vb[k2], b0);
        af[1][k2] = cmac(cmac(af[1][k2], va[k2], a1), vb[k2], b1);
      }
      // the slot's last reader (counted per warp) streams the chunk S ahead
      // into it at once, so no thread blocks waiting for the slowest bootstrap
      __syncwarp();
      if ((tid & 31) == 0) {
        __threadfence_block();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int slot = h ? sb : sa, c = q + h;
          if (atomicAdd(&sm.cnt[slot], 32u) == 64u * G - 32u) {
            sm.cnt[slot] = 0;
            if (c + S < kChunks) {
              mbar_expect_tx(&sm.full[slot], kRowBytes);
              bulk_g2s(sm.ring[slot], chunk_src(bkf, c + S), kRowBytes, &sm.full[slot]);
            }
          }
        }
      }
    }
    inv_stageA(af[0]);
    inv_stageA(af[1]);
    exchange_pair<2>(af[0], af[1], xa, xb, t, bar_id);
    {
      const TwPow8 w2(t2w);
      inv_stageB(af[0], w2);
      inv_stageB(af[1], w2);
    }
    exchange_pair<3>(af[0], af[1], xa, xb, t, bar_id);
    {
      const TwPow8 w1(t1b, t1w);
      inv_stageC(af[0], w1);
      inv_stageC(af[1], w1);
    }
    add_rounded(acc0, af[0], t);
    add_rounded(acc1, af[1], t);
  }
  group_sync(bar_id);
  if (live) extract(acc0, acc1, xout + (size_t)job.out * kXlweStride, t, 64);
}

// ------------------------------------------------ K1 + K2, latency: wide --
// One bootstrap per CTA of 384 threads for narrow levels (the emulator's
// instruction stream averages ~90 gates per dataflow level): the six gadget
// rows of a CMux step are transformed concurrently, one 64-thread group per
// row; partial products are reduced through shared memory; groups 0 and 1
// run the two inverse transforms.  Each group streams its own 16 KB key row
// for the next step with a bulk copy as soon as it has consumed the current
// one.  Per-step latency ~ 1 forward + 1 inverse transform instead of 8.
struct WideSmem {
  c64 bkbuf[kRows][1024];  // 96 KB: this step's six TRGSW rows
  c64 xbuf[kRows][512];    // 48 KB: one exchange buffer per group
  c64 red[kL][2][8][64];   // 48 KB: partial sums [pair][o][k2][t]
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
    mbar_init_fence();
  }
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(&sm.full[g], kRowBytes);
    bulk_g2s(sm.bkbuf[g], bkf + (size_t)g * 1024, kRowBytes, &sm.full[g]);
  }
  c64 T1[8], T2[8];
  load_twiddles(tw1, tw2, t, T1, T2);
  prologue(job, slab, sm.bar, sm.acc[0], sm.acc[1], tid, 64 * kRows, cta_sync, 0);
  const int shift = 32 - (p + 1) * kBgBit;
  c64* xb = sm.xbuf[g];
  auto sync = [bar_id] { group_sync(bar_id); };

  for (int i = 0; i < kN; ++i) {
    __syncthreads();  // ACC of the previous step complete
    const int ai = sm.bar[i];
    uint32_t dif[16];
    rotated_diff(sm.acc[part], ai, t, dif);
    c64 v[8];
    digits(dif, shift, v);
    fwd_stage1(v, T1);
    exchange<1>(v, xb, t, sync);
    group_sync(bar_id);  // WAR on the single exchange buffer
    fwd_stage2(v, T2);
    exchange<2>(v, xb, t, sync);
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
    // two-phase reduction of the six partials into three pair sums
    if (part == 1) {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        sm.red[p][0][k2][t] = pa[k2];
        sm.red[p][1][k2][t] = pb[k2];
      }
    }
    __syncthreads();  // (every group has read its key row)
    if (t == 0 && i + 1 < kN) {  // the next row lands outside every group's MAC
      mbar_expect_tx(&sm.full[g], kRowBytes);
      bulk_g2s(sm.bkbuf[g], bkf + ((size_t)(i + 1) * kRows + g) * 1024, kRowBytes, &sm.full[g]);
    }
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
      exchange<2>(v, sm.xbuf[g], t, sync);
      inv_stageB(v, T2);
      exchange<3>(v, sm.xbuf[g + 2], t, sync);
      inv_stageC(v, T1);
      add_rounded(sm.acc[o], v, t);
    }
  }
  __syncthreads();
  extract(sm.acc[0], sm.acc[1], xout + (size_t)job.out * kXlweStride, tid, 64 * kRows);
}

// ------------------------------------ K1 + K2, latency: 2-SM cluster --
// One bootstrap on a cluster of two CTAs (two SMs).  The wide kernel is bound
// by one SM's shared-memory pipe (six transforms' exchanges, six key rows,
// the partial-product reduction: LSU wavefronts 74% busy), so the work is
// split by TRLWE part: CTA r holds ACC part r, transforms its three gadget
// rows, and owns output polynomial r.  Its partial product for the other
// output polynomial goes to the peer through distributed shared memory; one
// cluster barrier per CMux step; each CTA then runs one inverse transform and
// updates its own ACC part -- no ACC broadcast is needed, because the digits
// of part r depend only on ACC part r.
#ifdef CVM_PHASE_PROF
// Developer instrumentation (tools/pair_phases.py): per-phase clock64 sums
// of thread 0 of groups 0 and 1 of every CTA, [cta][group][phase].
__device__ unsigned long long g_pair_phase[148 * 2][2][12];
#define PH(k)                                      \
  do {                                             \
    const long long now_ = clock64();              \
    ph[k] += (unsigned long long)(now_ - last_);   \
    last_ = now_;                                  \
  } while (0)
#else
#define PH(k) \
  do {        \
  } while (0)
#endif
struct PairSmem {
  c64 bkbuf[kL][1024];    // 48 KB: this CTA's three TRGSW rows
  c64 xbuf[kL][2][512];   // 48 KB: two exchange buffers per group (no WAR barrier)
  c64 red[kL][2][8][64];  // 48 KB: partial products [p][o][k2][t]
  c64 recv[2][8][64];     // 16 KB: the peer's partial for my polynomial (2 steps)
  uint32_t acc[kPolyN];   // ACC part r
  uint16_t bar[kLweWords + 1];
  uint64_t full[kL];
  uint64_t rbar[2];  // the peer's partial of step parity 0 / 1 landed
};

// The peer's partial product arrives by st.async remote stores that
// complete a transaction count on this CTA's rbar mbarrier (armed each step
// with the expected 8 KB), so the consumer waits on a local mbarrier instead
// of a cluster barrier (whose release fence, MEMBAR.ALL.GPU, and
// arrive/wait were ~15% of the pair kernel's stall samples).  The receive
// buffer alternates by step parity; the data dependence through the two
// accumulator parts keeps the peer from overwriting a buffer still being read.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 * kL, 1)
    blind_rotate_pair_kernel(const BrJob* __restrict__ jobs, const uint32_t* __restrict__ slab,
                             const c64* __restrict__ bkf, const c64* __restrict__ tw1,
                             const c64* __restrict__ tw2, uint32_t* __restrict__ xout) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int r = int(cluster.block_rank());  // TRLWE part and output polynomial
  const int tid = threadIdx.x;
  const int g = tid >> 6, t = tid & 63;  // group g: gadget level g of part r
  const int bar_id = 1 + g;
  const BrJob job = jobs[blockIdx.x >> 1];
  const int row = r * kL + g;  // TRGSW row (part * l + level)

  if (tid == 0) {
    for (int p = 0; p < kL; ++p) mbar_init(&sm.full[p], 1);
    mbar_init(&sm.rbar[0], 1);
    mbar_init(&sm.rbar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(&sm.full[g], kRowBytes);
    bulk_g2s(sm.bkbuf[g], bkf + (size_t)row * 1024, kRowBytes, &sm.full[g]);
  }
  c64 T1[8], T2[8];
  load_twiddles(tw1, tw2, t, T1, T2);
  // K1: both CTAs mod-switch the input; each initialises its own ACC part
  for (int i = tid; i < kLweWords; i += 64 * kL) {
    uint32_t v = i == kN ? job.cst : 0u;
    if (job.coef[0]) v += (uint32_t)job.coef[0] * slab[(size_t)job.slot[0] * kLweStride + i];
    if (job.coef[1]) v += (uint32_t)job.coef[1] * slab[(size_t)job.slot[1] * kLweStride + i];
    sm.bar[i] = (uint16_t)modswitch_2n(v);
  }
  __syncthreads();
  {
    const int barb = sm.bar[kN];
    for (int j = tid; j < kPolyN; j += 64 * kL)
      sm.acc[j] = r == 0 ? 0u : ((((j + barb) & (2 * kPolyN - 1)) < kPolyN) ? kMu : (0u - kMu));
  }
  uint32_t peer_recv_a, peer_rbar_a;  // shared::cluster addresses in the peer
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(peer_recv_a)
               : "r"(smem_u32(&sm.recv[0][0][0])), "r"(r ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(peer_rbar_a)
               : "r"(smem_u32(&sm.rbar[0])), "r"(r ^ 1));
  const int shift = 32 - (g + 1) * kBgBit;
  c64* xb0 = sm.xbuf[g][0];
  c64* xb1 = sm.xbuf[g][1];
  auto sync = [bar_id] { group_sync(bar_id); };
  cluster.sync();  // the peer's shared memory is live before any remote store
#ifdef CVM_PHASE_PROF
  unsigned long long ph[12] = {};
  long long last_ = clock64();
#endif

  for (int i = 0; i < kN; ++i) {
    __syncthreads();  // ACC part r of the previous step complete
    PH(0);
    if (tid == 0) mbar_expect_tx(&sm.rbar[i & 1], 8 * 64 * 16);
    const int ai = sm.bar[i];
    uint32_t dif[16];
    rotated_diff(sm.acc, ai, t, dif);
    c64 v[8];
    digits(dif, shift, v);
    PH(1);
    fwd_stage1(v, T1);
    exchange<1>(v, xb0, t, sync);
    fwd_stage2(v, T2);
    exchange<2>(v, xb1, t, sync);
    fwd_stage3(v);
    PH(2);
    mbar_wait(&sm.full[g], i & 1);
    PH(3);
    const c64* bk = sm.bkbuf[g];
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      sm.red[g][0][k2][t] = cmul(v[k2], bk[k2 * 128 + t]);
      sm.red[g][1][k2][t] = cmul(v[k2], bk[k2 * 128 + 64 + t]);
    }
    __syncthreads();  // all three levels' partial products in red (and keys read)
    PH(4);
    if (t == 0 && i + 1 < kN) {  // next row's copy lands outside every group's MAC
      mbar_expect_tx(&sm.full[g], kRowBytes);
      bulk_g2s(sm.bkbuf[g], bkf + ((size_t)(i + 1) * kRows + row) * 1024, kRowBytes,
               &sm.full[g]);
    }
    PH(5);
    {  // the peer's polynomial: sum over levels, store remotely -- every group
       // takes a share of the bins (group 0 the smallest: it owns the inverse)
      auto send = [&](int k2) {
        const c64 x = cadd(cadd(sm.red[0][r ^ 1][k2][t], sm.red[1][r ^ 1][k2][t]),
                           sm.red[2][r ^ 1][k2][t]);
        const uint32_t a = peer_recv_a + uint32_t(((i & 1) * 512 + k2 * 64 + t) * 16);
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, "
            "[%3];" ::"r"(a),
            "l"(__double_as_longlong(x.x)), "l"(__double_as_longlong(x.y)),
            "r"(peer_rbar_a + uint32_t(8 * (i & 1)))
            : "memory");
      };
      // bins k2 sent by groups 0 / 1 / 2: 2 / 3 / 3 (0 / 4 / 4: 1.428 ms per
      // 74-gate level, 1 / 4 / 3: 1.423, 2 / 3 / 3: 1.410, 3 / 3 / 2: 1.413)
      constexpr int n0 = 2, n1 = 3;
      const int first = g == 0 ? 0 : g == 1 ? n0 : n0 + n1;
      const int count = g == 0 ? n0 : g == 1 ? n1 : 8 - n0 - n1;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (kk < count) send(first + kk);
    }
    if (g == 0) {  // my polynomial: local part of the sum
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2)
        v[k2] = cadd(cadd(sm.red[0][r][k2][t], sm.red[1][r][k2][t]), sm.red[2][r][k2][t]);
    }
    PH(6);
    if (g == 0) mbar_wait(&sm.rbar[i & 1], (i >> 1) & 1);  // the peer's partial landed
    PH(7);
    if (g == 0) {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) v[k2] = cadd(v[k2], sm.recv[i & 1][k2][t]);
      inv_stageA(v);
      exchange<2>(v, sm.xbuf[1][0], t, sync);
      PH(8);
      inv_stageB(v, T2);
      exchange<3>(v, sm.xbuf[2][0], t, sync);
      PH(9);
      inv_stageC(v, T1);
      PH(10);
      add_rounded(sm.acc, v, t);
      PH(11);
    }
  }
#ifdef CVM_PHASE_PROF
  if (t == 0 && g < 2 && blockIdx.x < 148 * 2)
    for (int k = 0; k < 12; ++k) g_pair_phase[blockIdx.x][g][k] = ph[k];
#endif
  __syncthreads();
  // sample extraction: CTA 0 owns a (from ACC part 0), CTA 1 the b word
  uint32_t* out = xout + (size_t)job.out * kXlweStride;
  if (r == 0) {
    for (int j = tid; j < kPolyN; j += 64 * kL) out[j] = j == 0 ? sm.acc[0] : 0u - sm.acc[kPolyN - j];
  } else if (tid == 0) {
    out[kPolyN] = sm.acc[0];
  }
  cluster.sync();  // no CTA leaves while its shared memory may still be addressed
}

// ----------------------------------------------------------- launchers --
#ifdef CVM_PHASE_PROF
extern "C" __attribute__((visibility("default"))) int cvm_debug_pair_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_pair_phase, sizeof(g_pair_phase));
}
#endif
#undef PH

cudaError_t launch_bk_to_fft(const uint32_t* bk, const c64* tw1, const c64* tw2, c64* bkf,
                             cudaStream_t s) {
  bk_to_fft_kernel<<<kN * kRows * 2, 64, 0, s>>>(bk, tw1, tw2, bkf);
  return cudaGetLastError();
}

static cudaError_t launch_v3(const BrJob* jobs, int count, const uint32_t* slab, const c64* bkf,
                             const c64* tw1, const c64* tw2, uint32_t* xout, cudaStream_t s) {
  constexpr int G = 4, S = 7;
  static std::atomic<uint64_t> configured{0};
  auto* kern = blind_rotate_kernel_v3<G, S>;
  const int smem = int(sizeof(BrSmem3<G, S>));
  cudaError_t e = set_smem(kern, smem, configured);
  if (e != cudaSuccess) return e;
  kern<<<(count + G - 1) / G, 64 * G, smem, s>>>(jobs, count, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

static cudaError_t launch_wide(const BrJob* jobs, int count, const uint32_t* slab,
                               const c64* bkf, const c64* tw1, const c64* tw2, uint32_t* xout,
                               cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  const int smem = int(sizeof(WideSmem));
  cudaError_t e = set_smem(blind_rotate_wide_kernel, smem, configured);
  if (e != cudaSuccess) return e;
  blind_rotate_wide_kernel<<<count, 64 * kRows, smem, s>>>(jobs, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

static cudaError_t launch_pair(const BrJob* jobs, int count, const uint32_t* slab,
                               const c64* bkf, const c64* tw1, const c64* tw2, uint32_t* xout,
                               cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  const int smem = int(sizeof(PairSmem));
  cudaError_t e = set_smem(blind_rotate_pair_kernel, smem, configured);
  if (e != cudaSuccess) return e;
  blind_rotate_pair_kernel<<<2 * count, 64 * kL, smem, s>>>(jobs, slab, bkf, tw1, tw2, xout);
  return cudaGetLastError();
}

static int g_br_variant = -1;
int br_variant() {
  if (g_br_variant < 0) g_br_variant = env_or("CVM_BR_KERNEL", kDefaultBrVariant);
  return g_br_variant;
}
void set_br_variant(int v) { g_br_variant = v; }
int default_br_variant() { return kDefaultBrVariant; }
bool valid_br_variant(int v) {
  return v == 0 || v == 9 || v == 96 || v == 5247 || valid_br_v4_variant(v);
}

cudaError_t launch_blind_rotate(int variant, const BrJob* jobs, int count, const uint32_t* slab,
                                const c64* bkf, const c64* tw1, const c64* tw2,
                                const c64* bkf4, const c64* tw4, uint32_t* xout,
                                cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (variant < 0) variant = br_variant();
  if (valid_br_v4_variant(variant))
    return launch_blind_rotate_v4(variant, jobs, count, slab, bkf4, tw4, xout, s);
  if (variant == 0) {
    // auto: a very narrow level runs each bootstrap on a 2-SM cluster, a
    // narrow one on a whole SM (latency); a level of up to two bootstraps
    // per SM gives each its own CTA; wide levels use the v4 throughput
    // kernel (blind_rotate_v4.cu) with the remainder split off below.
    constexpr int kSms = kBrSms;
    if (count <= 2 * kSms) {
      // pair rounds of 74 (1.41 ms) or wide rounds of 148 (2.27 ms): pair up
      // to 74 and for 149-222 (4.18 vs 4.54 ms), wide otherwise
      variant = br_latency_pair(count) ? 96 : 9;
    } else {
      // Wide levels: the v4 kernel (one bootstrap per warp, 8 per SM) works
      // in waves of 8 x 148 bootstraps (~11.4 ms; with 5-7 warps per SM a
      // wave still takes ~11.2 ms, with 2-4 ~8.1 ms: a lone warp is
      // latency-bound), the v3 kernel (5247) in rounds of 4 x 148 (~5.9 ms),
      // the latency kernel in rounds of 148 (~2.3 ms).  Full v4 waves, then
      // the remainder on whichever finishes it first (costs in 0.1 ms,
      // tools/v4_waves.py; profiles/r01_variant_sweep.txt).
      const int full = count / kBrWave8, rest = count - full * kBrWave8;
      const int head = full * kBrWave8;
      if (head > 0) {
        cudaError_t e = launch_blind_rotate_v4(6085, jobs, head, slab, bkf4, tw4, xout, s);
        if (e != cudaSuccess || rest == 0) return e;
      }
      int b8 = 0, b4 = 0, b1 = 0;
      br_remainder_plan(rest, &b8, &b4, &b1);
      constexpr int kW8 = kBrWave8, kW4 = kBrWave4;
      int done = head;
      if (b8) {  // rest/148 warps per SM
        const int n = std::min(rest, kW8), warps = (n + kSms - 1) / kSms;
        cudaError_t e = launch_blind_rotate_v4(6005 + 10 * warps, jobs + done, n, slab, bkf4,
                                               tw4, xout, s);
        if (e != cudaSuccess) return e;
        done += n;
      }
      if (b4 && done < count) {
        const int n = std::min(count - done, b4 * kW4);
        cudaError_t e = launch_v3(jobs + done, n, slab, bkf, tw1, tw2, xout, s);
        if (e != cudaSuccess) return e;
        done += n;
      }
      if (b1 && done < count) {
        const int n = count - done;
        return br_latency_pair(n) ? launch_pair(jobs + done, n, slab, bkf, tw1, tw2, xout, s)
                                  : launch_wide(jobs + done, n, slab, bkf, tw1, tw2, xout, s);
      }
      return cudaSuccess;
    }
  }
  switch (variant) {
    case 9: return launch_wide(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 96: return launch_pair(jobs, count, slab, bkf, tw1, tw2, xout, s);
    case 5247: return launch_v3(jobs, count, slab, bkf, tw1, tw2, xout, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cvm
