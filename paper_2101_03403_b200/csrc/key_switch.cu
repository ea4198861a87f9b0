// sm_100a key switch (K3 + K4: MUX combine, LWE key switch N = 1024 ->
// n = 630) of a whole level as one integer matrix product on the tcgen05
// tensor cores:
//   out[g][col] = b_g - sum_{i,j} KSK[i][j][d_gij][col]
//              = b_g - (A x B)[g][col],  A[g][(i,j,v)] = [d_gij == v] (one-hot),
// B[(i,j,v)][col] = KSK[i][j][v][col].  B's 32-bit torus words are split into
// four byte limbs, each product exact in u8 x u8 -> s32 (a column sum is at
// most 8192 * 255 < 2^31), recombined mod 2^32 as sum_l acc_l << 8 l.
// K = 1024 coefficients x 8 digits x 4 values, one coefficient per k32 step.
// Variant 8: one CTA per 128-gate x 128-column tile; variant 9 (default):
// the same tiles split along K over up to 16 CTAs + ks_reduce_kernel.
// (Round 1's gather kernels and the mma.sync product are retired; their
// numbers are in profiles/r01_variant_sweep.txt.)  DESIGN.md section 4.4.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fft512.cuh"
#include "kernels.cuh"
#include "sm100.cuh"

namespace cvm {

// ------------------------------- K3 + K4 on tcgen05 (5th-gen tensor cores) --
// The one-hot x byte-limb product issued as tcgen05.mma kind::i8 (u8 x u8 -> s32) with the four limb accumulators in
// tensor memory: CTA tile 128 gates (M) x 128 columns (N) x 4 limbs = all 512
// TMEM columns; one k32 step per coefficient (4 MMAs, one per limb).
//   warps 0-3 (128 threads, thread = gate = TMEM lane): write the one-hot A
//             tile of each coefficient into shared memory, then run the
//             epilogue (tcgen05.ld, limb recombination, b - sum, store);
//   warp 4 lane 0: MMA issuer; warp 5 lane 0: bulk-copy producer of the B
//             tiles (16 KB per coefficient, pre-arranged in HBM in the
//             canonical no-swizzle K-major layout by ksk_to_tc_kernel).
// Operand layout (K-major, SWIZZLE_NONE): core matrices of 8 rows x 16 B;
// row r, K-chunk c at (r/8)*256 + c*128 + (r%8)*16 (LBO 128 B, SBO 256 B).
constexpr int kTcRows = 128;       // gates per CTA (M) and columns per CTA (N)
constexpr int kTcColTiles = 5;     // 640 >= 632 columns
constexpr int kTcStages = 6;
constexpr int kTcThreads = 192;
constexpr uint32_t kTcTileBytes = 4096;  // 128 rows x 32 B
static_assert(kKskTcWords == size_t(kPolyN) * kTcColTiles * 4 * (kTcTileBytes / 4));
// idesc: D s32 (c_format 2), A/B u8 (format 0), K-major, N = 128, M = 128
constexpr uint32_t kTcIdesc = (2u << 4) | (uint32_t(kTcRows >> 3) << 17) |
                              (uint32_t(kTcRows >> 4) << 24);

struct KsTcSmem {
  uint8_t a[kTcStages][kTcTileBytes];     // one-hot digits, 128 gates x 32 B
  uint8_t b[kTcStages][4][kTcTileBytes];  // KSK limbs, 128 columns x 32 B each
  uint64_t b_full[kTcStages], a_full[kTcStages], empty[kTcStages], done;
  uint32_t tmem_base;
  KsJob job[kTcRows];
  uint32_t bval[kTcRows];
};

// [i][ctile][limb][col-group 16][k-chunk 2][8 cols][4 words]: word q of
// k-chunk c is digit j = 4c + q, its bytes v = 0..3 the limb of KSK[i][j][v][col]
__global__ void __launch_bounds__(256) ksk_to_tc_kernel(const uint32_t* __restrict__ ksk,
                                                        uint32_t* __restrict__ out) {
  const size_t idx = size_t(blockIdx.x) * 256 + threadIdx.x;
  if (idx >= kKskTcWords) return;
  size_t x = idx;
  const int q = int(x % 4);
  x /= 4;
  const int rr = int(x % 8);
  x /= 8;
  const int kc = int(x % 2);
  x /= 2;
  const int ng = int(x % 16);
  x /= 16;
  const int l = int(x % 4);
  x /= 4;
  const int ct = int(x % kTcColTiles);
  const int i = int(x / kTcColTiles);
  const int col = ct * kTcRows + ng * 8 + rr;
  const int j = kc * 4 + q;
  uint32_t w = 0;
  if (col < kKskRowStride) {
#pragma unroll
    for (int v = 0; v < kKsBase; ++v) {
      const uint32_t k = ksk[((size_t(i) * kKsT + j) * kKsBase + v) * kKskRowStride + col];
      w |= ((k >> (8 * l)) & 0xFFu) << (8 * v);
    }
  }
  out[idx] = w;
}

__device__ __forceinline__ uint64_t umma_desc_kmajor(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (1ull << 46);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(kTcIdesc), "r"(accumulate)
      : "memory");
}

// Split-K (blockIdx.z, `part` non-null): CTA z multiplies coefficients
// [z*k_per, (z+1)*k_per) only and writes its partial result (mod 2^32) to
// part[z][gate][col]; ks_reduce_kernel sums the splits.  A narrow level then
// runs on 16x more CTAs (one 128-gate tile x 5 column tiles is only five).
__global__ void __launch_bounds__(kTcThreads, 1) key_switch_tc_kernel(
    const KsJob* __restrict__ jobs, int count, const uint32_t* __restrict__ xlwe,
    const uint32_t* __restrict__ ksktc, uint32_t* __restrict__ slab, int k_per,
    uint32_t* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  KsTcSmem& sm = *reinterpret_cast<KsTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g0 = blockIdx.x * kTcRows, ct = blockIdx.y;
  const int z = blockIdx.z, k0 = z * k_per, k1 = k0 + k_per;
  const uint32_t prec = 1u << (32 - (1 + kKsBaseBit * kKsT));

  if (tid < kTcRows) {
    const int g = g0 + tid;
    const KsJob jb = jobs[g < count ? g : 0];
    sm.job[tid] = jb;
    uint32_t b = xlwe[size_t(jb.x[0]) * kXlweStride + kPolyN] + jb.cst;
    if (jb.x[1] != kNoInput) b += xlwe[size_t(jb.x[1]) * kXlweStride + kPolyN];
    sm.bval[tid] = b;
  }
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&sm.b_full[s], 1);
      mbar_init(&sm.a_full[s], kTcRows);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.done, 1);
    mbar_init_fence();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp < 4) {
    // ---- A producer: one-hot digits of gate `tid` for every coefficient ----
    const KsJob& jb = sm.job[tid];
    const uint32_t* x0 = xlwe + size_t(jb.x[0]) * kXlweStride;
    const uint32_t* x1 = jb.x[1] != kNoInput ? xlwe + size_t(jb.x[1]) * kXlweStride : nullptr;
    const uint32_t row_off = uint32_t((tid >> 3) * 256 + (tid & 7) * 16);
    for (int i0 = k0; i0 < k1; i0 += 16) {
      uint32_t ab[16];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 w = *reinterpret_cast<const uint4*>(x0 + i0 + 4 * v);
        if (x1) {
          const uint4 u = *reinterpret_cast<const uint4*>(x1 + i0 + 4 * v);
          w.x += u.x;
          w.y += u.y;
          w.z += u.z;
          w.w += u.w;
        }
        ab[4 * v] = w.x + prec;
        ab[4 * v + 1] = w.y + prec;
        ab[4 * v + 2] = w.z + prec;
        ab[4 * v + 3] = w.w + prec;
      }
#pragma unroll
      for (int ii = 0; ii < 16; ++ii) {
        const int li = i0 - k0 + ii, s = li % kTcStages;
        if (li >= kTcStages) mbar_wait(&sm.empty[s], ((li / kTcStages) + 1) & 1);
        uint32_t oh[8];
#pragma unroll
        for (int j = 0; j < kKsT; ++j) oh[j] = 1u << (8 * ((ab[ii] >> (30 - 2 * j)) & 3u));
        uint4* dst = reinterpret_cast<uint4*>(sm.a[s] + row_off);
        dst[0] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
        dst[8] = make_uint4(oh[4], oh[5], oh[6], oh[7]);  // + 128 B: k-chunk 1
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&sm.a_full[s]);
      }
    }
    // ---- epilogue: TMEM -> registers, recombine the limbs, store ----
    mbar_wait(&sm.done, 0);
    tc_fence_after();
    const uint32_t lane_base = tbase + (uint32_t(32 * warp) << 16);
    const int g = g0 + tid;
    uint32_t* out = slab + size_t(sm.job[tid].out_slot) * kLweStride;
    for (int c0 = 0; c0 < kTcRows; c0 += 8) {
      uint32_t r[4][8];
#pragma unroll
      for (int l = 0; l < 4; ++l) tc_ld8(lane_base + uint32_t(l * kTcRows + c0), r[l]);
      tc_wait_ld16(r[0], r[1]);  // waits for all four; ties the registers to the wait
      tc_wait_ld16(r[2], r[3]);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = ct * kTcRows + c0 + c;
        const uint32_t sum = r[0][c] + (r[1][c] << 8) + (r[2][c] << 16) + (r[3][c] << 24);
        if (g < count && col < kKskRowStride) {
          const uint32_t v = (col == kN && z == 0 ? sm.bval[tid] : 0u) - sum;
          if (part) part[(size_t(z) * gridDim.x * kTcRows + g) * (kTcColTiles * kTcRows) + col] = v;
          else out[col] = v;
        }
      }
    }
  } else if (warp == 4) {
    // ---- MMA issuer ----
    if (lane == 0) {
      for (int li = 0; li < k_per; ++li) {
        const int s = li % kTcStages;
        const uint32_t par = (li / kTcStages) & 1;
        mbar_wait(&sm.b_full[s], par);
        mbar_wait(&sm.a_full[s], par);
        tc_fence_after();
        const uint64_t ad = umma_desc_kmajor(sm.a[s]);
#pragma unroll
        for (int l = 0; l < 4; ++l)
          umma_i8(tbase + uint32_t(l * kTcRows), ad, umma_desc_kmajor(sm.b[s][l]), li > 0);
        tc_commit(&sm.empty[s]);  // frees stage s once these MMAs have read it
      }
      tc_commit(&sm.done);
    }
    __syncwarp();
  } else {
    // ---- B producer ----
    if (lane == 0) {
      for (int i = k0; i < k1; ++i) {
        const int li = i - k0, s = li % kTcStages;
        if (li >= kTcStages) mbar_wait(&sm.empty[s], ((li / kTcStages) + 1) & 1);
        mbar_expect_tx(&sm.b_full[s], 4 * kTcTileBytes);
        bulk_g2s(sm.b[s], ksktc + (size_t(i) * kTcColTiles + ct) * (4 * kTcTileBytes / 4),
                 4 * kTcTileBytes, &sm.b_full[s]);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}

// Sum of the split-K partials of key_switch_tc_kernel into the output slots.
__global__ void __launch_bounds__(256) ks_reduce_kernel(const KsJob* __restrict__ jobs,
                                                        int count, int splits, int rows,
                                                        const uint32_t* __restrict__ part,
                                                        uint32_t* __restrict__ slab) {
  const int g = blockIdx.x;
  const size_t plane = size_t(rows) * (kTcColTiles * kTcRows);
  uint32_t* out = slab + size_t(jobs[g].out_slot) * kLweStride;
  for (int col = threadIdx.x; col < kKskRowStride; col += blockDim.x) {
    const uint32_t* p = part + size_t(g) * (kTcColTiles * kTcRows) + col;
    uint32_t v = 0;
    for (int z = 0; z < splits; ++z) v += p[z * plane];
    out[col] = v;
  }
  (void)count;
}

// ----------------------------------------------------------- launchers --
static int g_ks_variant = -1;
int ks_variant() {
  if (g_ks_variant < 0) g_ks_variant = env_or("CVM_KS_KERNEL", kDefaultKsVariant);
  return g_ks_variant;
}
void set_ks_variant(int v) { g_ks_variant = v; }
bool valid_ks_variant(int v) { return v == 0 || v == 8 || v == 9; }

cudaError_t launch_ksk_to_tc(const uint32_t* ksk, uint32_t* ksktc, cudaStream_t s) {
  ksk_to_tc_kernel<<<unsigned((kKskTcWords + 255) / 256), 256, 0, s>>>(ksk, ksktc);
  return cudaGetLastError();
}

cudaError_t launch_key_switch(int variant, const KsJob* jobs, int count, const uint32_t* xlwe,
                              const uint32_t* ksktc, uint32_t* kspart, uint32_t* slab,
                              cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (variant < 0) variant = ks_variant();
  // auto: the split-K tcgen05 product at every width (0.037 ms for a
  // 32-gate level vs 0.178 for the 6-group gather and 0.26 unsplit; equal to
  // the unsplit product on wide levels; profiles/r01_variant_sweep.txt)
  if (variant == 0) variant = 9;
  switch (variant) {
    case 8: {
      if (!ksktc) return cudaErrorInvalidValue;
      static std::atomic<uint64_t> configured{0};
      const int smem = int(sizeof(KsTcSmem));
      cudaError_t e = set_smem(key_switch_tc_kernel, smem, configured);
      if (e != cudaSuccess) return e;
      const dim3 grid((count + kTcRows - 1) / kTcRows, kTcColTiles);
      key_switch_tc_kernel<<<grid, kTcThreads, smem, s>>>(jobs, count, xlwe, ksktc, slab,
                                                           kPolyN, nullptr);
      break;
    }
    case 9: {  // split-K tcgen05 product: ~148 CTAs whatever the level width
      if (!ksktc || !kspart) return cudaErrorInvalidValue;
      static std::atomic<uint64_t> configured{0};
      const int smem = int(sizeof(KsTcSmem));
      cudaError_t e = set_smem(key_switch_tc_kernel, smem, configured);
      if (e != cudaSuccess) return e;
      const int mt = (count + kTcRows - 1) / kTcRows;
      int splits = 1;
      while (splits < kKsMaxSplits && 2 * splits * mt * kTcColTiles <= 148) splits *= 2;
      if (splits == 1) {
        key_switch_tc_kernel<<<dim3(mt, kTcColTiles), kTcThreads, smem, s>>>(
            jobs, count, xlwe, ksktc, slab, kPolyN, nullptr);
        break;
      }
      key_switch_tc_kernel<<<dim3(mt, kTcColTiles, splits), kTcThreads, smem, s>>>(
          jobs, count, xlwe, ksktc, slab, kPolyN / splits, kspart);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      ks_reduce_kernel<<<count, 256, 0, s>>>(jobs, count, splits, mt * kTcRows, kspart, slab);
      break;
    }
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cvm
