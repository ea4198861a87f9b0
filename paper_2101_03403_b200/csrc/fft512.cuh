// Negacyclic FFT for TFHE's external product, one polynomial (N = 1024,
// folded into M = 512 complex points) spread over 64 threads x 8 points.
//
// Folding: z_j = (p_j + i p_{j+512}) * w^j, w = e^{i pi/N}; Z = DFT_512(z)
// evaluates p at the 512 roots e^{i pi (4k+1)/N}; products of two real
// polynomials mod X^N+1 become point-wise products of their Z.
//
// 512 = 8 x 8 x 8 with j = 64a + 8b + c and k = k0 + 8k1 + 64k2:
//   fwd stage 1  role t = 8b+c   : DFT8 over a, x T1[k0] (= w^t W^{t k0})
//   exchange 1   (t=8b+c, k0)    -> cell 8c+k0, slot b
//   fwd stage 2  role t = 8c+k0  : DFT8 over b, x T2[k1] (= W^{8 c k1})
//   exchange 2   (t=8c+k0, k1)   -> cell 8k1+k0, slot c
//   fwd stage 3  role t = 8k1+k0 : DFT8 over c  -> bins t + 64 k2
// The inverse runs the mirror image (stage A/B/C) with conjugate twiddles
// applied on the inputs, so the thread that owns bin set {t + 64 k2} after
// the forward transform also owns it before the inverse, and the thread that
// owns coefficients {t + 64a, t + 64a + 512} before the forward owns them after
// the inverse.  No bit reversal is ever performed: the bootstrapping key is
// stored in the same per-thread bin order (tfhe_params.h kBkf*).
//
// Every function here is __host__ __device__ so tests/native/fft_emul.cpp can
// run the exact same arithmetic on the CPU with 64 emulated threads.
#pragma once
#include <stdint.h>
#include <string.h>

#include <cmath>

#include "tfhe_params.h"

namespace cvm {

struct alignas(16) c64 {
  double x, y;
};

CVM_HD c64 cmul(c64 a, c64 b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
CVM_HD c64 cmul_conj(c64 a, c64 b) {  // a * conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
CVM_HD c64 cadd(c64 a, c64 b) { return {a.x + b.x, a.y + b.y}; }
// acc + a * b as four FMAs (cadd(acc, cmul(a, b)) costs 2 MUL + 2 FMA + 2 ADD:
// without reassociation the compiler cannot fold the accumulate).
CVM_HD c64 cmac(c64 acc, c64 a, c64 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
CVM_HD c64 csub(c64 a, c64 b) { return {a.x - b.x, a.y - b.y}; }

// e^{i pi a / 16}, a = 0..7: the stride-64 part of the fold twist w^{64a}.
// (Called with compile-time a inside unrolled loops, so it folds to immediates.)
CVM_HD c64 twist_const(int a) {
  switch (a) {
    case 1: return {0.98078528040323043, 0.19509032201612826};
    case 2: return {0.92387953251128674, 0.38268343236508977};
    case 3: return {0.83146961230254524, 0.55557023301960218};
    case 4: return {0.70710678118654752, 0.70710678118654752};
    case 5: return {0.55557023301960218, 0.83146961230254524};
    case 6: return {0.38268343236508977, 0.92387953251128674};
    case 7: return {0.19509032201612826, 0.98078528040323043};
    default: return {1.0, 0.0};
  }
}

constexpr double kRsqrt2 = 0.70710678118654752440;

// In-place 8-point DFT, natural order in and out.
// kInverse=false: X_k = sum x_n e^{-2 pi i nk/8};  true: e^{+2 pi i nk/8}.
template <bool kInverse>
CVM_HD void dft8(c64 v[8]) {
  // DIT: E = DFT4(even), O = DFT4(odd).
  c64 s0 = cadd(v[0], v[4]), d0 = csub(v[0], v[4]);
  c64 s1 = cadd(v[2], v[6]), d1 = csub(v[2], v[6]);
  c64 s2 = cadd(v[1], v[5]), d2 = csub(v[1], v[5]);
  c64 s3 = cadd(v[3], v[7]), d3 = csub(v[3], v[7]);
  // multiply by -i (forward) or +i (inverse)
  auto rot = [](c64 a) -> c64 {
    return kInverse ? c64{-a.y, a.x} : c64{a.y, -a.x};
  };
  c64 e0 = cadd(s0, s1), e2 = csub(s0, s1);
  c64 t = rot(d1);
  c64 e1 = cadd(d0, t), e3 = csub(d0, t);
  c64 o0 = cadd(s2, s3), o2 = csub(s2, s3);
  c64 u = rot(d3);
  c64 o1 = cadd(d2, u), o3 = csub(d2, u);
  // odd half times W8^k; the 1/sqrt(2) scalings fuse into the final +-.
  // w1 = r*(p1, q1), w3 = r*(p3, q3) with r = 1/sqrt(2).
  double p1, q1, p3, q3;
  c64 w2;
  if (!kInverse) {
    p1 = o1.x + o1.y;
    q1 = o1.y - o1.x;
    w2 = {o2.y, -o2.x};
    p3 = o3.y - o3.x;
    q3 = -(o3.x + o3.y);
  } else {
    p1 = o1.x - o1.y;
    q1 = o1.x + o1.y;
    w2 = {-o2.y, o2.x};
    p3 = -(o3.x + o3.y);
    q3 = o3.x - o3.y;
  }
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = {fma(kRsqrt2, p1, e1.x), fma(kRsqrt2, q1, e1.y)};
  v[5] = {fma(-kRsqrt2, p1, e1.x), fma(-kRsqrt2, q1, e1.y)};
  v[2] = cadd(e2, w2);
  v[6] = csub(e2, w2);
  v[3] = {fma(kRsqrt2, p3, e3.x), fma(kRsqrt2, q3, e3.y)};
  v[7] = {fma(-kRsqrt2, p3, e3.x), fma(-kRsqrt2, q3, e3.y)};
}

// Physical position (in c64 units) of (cell, slot) in a 512-entry exchange
// buffer.  The XOR swizzle keeps every quarter-warp of 16-byte accesses on 8
// distinct bank groups for all four exchange patterns.
CVM_HD int xpos(int cell, int slot) {
  return cell * 8 + ((slot ^ cell ^ (cell >> 3)) & 7);
}

// ---------------------------------------------------------------- forward --
// Input: v[a] = p_{t+64a} + i p_{t+64a+512} (untwisted).
// TW: anything indexable by k = 0..7 (the kernels pass register arrays).
template <class TW>
CVM_HD void fwd_stage1(c64 v[8], const TW& T1) {
#pragma unroll
  for (int a = 1; a < 8; ++a) v[a] = cmul(v[a], twist_const(a));
  dft8<false>(v);
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = cmul(v[k], T1[k]);
}
template <class TW>
CVM_HD void fwd_stage2(c64 v[8], const TW& T2) {
  dft8<false>(v);
#pragma unroll
  for (int k = 1; k < 8; ++k) v[k] = cmul(v[k], T2[k]);
}
CVM_HD void fwd_stage3(c64 v[8]) { dft8<false>(v); }

// Exchange write/read helpers: cell/slot for thread role t and value index z.
CVM_HD int ex1_cell(int t, int z) { return 8 * (t & 7) + z; }   // slot = t >> 3
CVM_HD int ex2_cell(int t, int z) { return 8 * z + (t & 7); }   // slot = t >> 3
CVM_HD int exB_cell(int t, int z) { return 8 * z + (t >> 3); }  // slot = t & 7

// ---------------------------------------------------------------- inverse --
CVM_HD void inv_stageA(c64 v[8]) { dft8<true>(v); }
template <class TW>
CVM_HD void inv_stageB(c64 v[8], const TW& T2) {
#pragma unroll
  for (int k = 1; k < 8; ++k) v[k] = cmul_conj(v[k], T2[k]);
  dft8<true>(v);
}
// Output: v[a] = M * (p_{t+64a} + i p_{t+64a+512}) (scale folded into the key).
template <class TW>
CVM_HD void inv_stageC(c64 v[8], const TW& T1) {
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = cmul_conj(v[k], T1[k]);
  dft8<true>(v);
#pragma unroll
  for (int a = 1; a < 8; ++a) v[a] = cmul_conj(v[a], twist_const(a));
}

// Per-thread twiddles (host-side table builder; long double for accuracy).
//   T1[t][k] = w^t W^{t k} = e^{i pi t (1 - 4k) / 1024}
//   T2[t][k] = W^{8 (t>>3) k} = e^{-i pi (t>>3) k / 32}
inline void make_twiddles(c64 T1[64][8], c64 T2[64][8]) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < 64; ++t)
    for (int k = 0; k < 8; ++k) {
      long double a1 = pi * t * (1 - 4 * k) / 1024.0L;
      T1[t][k] = {(double)std::cos(a1), (double)std::sin(a1)};
      long double a2 = -pi * (t >> 3) * k / 32.0L;
      T2[t][k] = {(double)std::cos(a2), (double)std::sin(a2)};
    }
}

// Per-thread twiddles generated on use, T[k] = base * w^k (k = 0..7), from
// two resident complex values instead of eight: 9 (or 6 with base 1)
// complex multiplies per use, a few ulp -- inside the FFT's rounding margin
// (tests/native/fft_emul.cpp measures both modes), and
// 52 fewer live registers per thread.  Bases: T1 = (w^t, W_512^t),
// T2 = W_512^(8 (t>>3)).
struct TwPow8 {
  c64 v[8];
  CVM_HD TwPow8(c64 base, c64 w) {
    const c64 w2 = cmul(w, w), w4 = cmul(w2, w2);
    v[0] = base;
    v[1] = cmul(base, w);
    v[2] = cmul(base, w2);
    v[3] = cmul(v[2], w);
    v[4] = cmul(base, w4);
    v[5] = cmul(v[4], w);
    v[6] = cmul(v[4], w2);
    v[7] = cmul(v[6], w);
  }
  CVM_HD explicit TwPow8(c64 w) {  // base 1
    v[0] = {1.0, 0.0};
    v[1] = w;
    v[2] = cmul(w, w);
    v[3] = cmul(v[2], w);
    v[4] = cmul(v[2], v[2]);
    v[5] = cmul(v[4], w);
    v[6] = cmul(v[4], v[2]);
    v[7] = cmul(v[6], w);
  }
  CVM_HD const c64& operator[](int k) const { return v[k]; }
};

// ---------------------------------------------------- exact conversions --
// Small non-negative integer u (< 2^31) to double, exactly, without I2F:
// the bit pattern 0x43300000:u is the double 2^52 + u.
CVM_HD double u32_biased_to_double(uint32_t u, double bias) {
#if defined(__CUDA_ARCH__)
  return __hiloint2double(0x43300000, (int)u) - bias;
#else
  uint64_t bits = (uint64_t(0x43300000) << 32) | u;
  double d;
  memcpy(&d, &bits, 8);
  return d - bias;
#endif
}

// round(v) mod 2^32 for |v| < 2^51: add 1.5*2^52, keep the low mantissa word.
CVM_HD uint32_t round_to_torus(double v) {
  double t = v + 6755399441055744.0;
#if defined(__CUDA_ARCH__)
  return (uint32_t)__double2loint(t);
#else
  uint64_t bits;
  memcpy(&bits, &t, 8);
  return (uint32_t)bits;
#endif
}

}  // namespace cvm
