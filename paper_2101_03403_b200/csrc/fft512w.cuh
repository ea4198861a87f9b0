// Warp-wide negacyclic FFT for the v4 blind-rotation kernel: one polynomial
// (N = 1024, folded into M = 512 complex points, fft512.cuh) on ONE warp,
// 16 points per lane.  Compared with the 64-thread transform of fft512.cuh it
// needs one shared-memory transpose instead of two exchanges (and no named
// barrier, the transform never leaves its warp); the second exchange is a
// lane-pair swap of 8 values through shuffles.
//
// 512 = 16 x 32 with j = 32a + t (lane t, a = 0..15), k = k0 + 16 k1:
//   stage 1  (lane t)          : z_j = p'_j w^{32a} (twist), DFT16 over a,
//                                x T1[t][k0] = w^t W^{t k0}
//   transpose (smem)           : lane 2 k0 + e gets y_t of its k0 for
//                                t = 8e + i (slot i) and t = 8e + i + 16 (slot 8 + i)
//   stage 2a (lane pair)       : radix-2 DIF over t = m, m + 16:
//                                s_m = y_m + y_{m+16}, d_m = (y_m - y_{m+16}) w32^m;
//                                the even lane keeps s (m = i), the odd lane d
//                                (m = 8 + i); the other half is swapped
//   stage 2b (lane)            : DFT16 over m -> k1 = 2r + e in slot r
// The odd lane's DFT16 input is its natural sequence rotated by 8 (own
// m = 8..15 first), so its outputs carry a factor (-1)^r: the forward
// transform is D * F with D = diag((-1)^r on odd lanes).  The inverse undoes
// exactly that, so products with a key stored as the TRUE spectrum F(k)
// (bk_to_fft_v4_kernel removes D) come back right: F'^{-1}(D F(v) F(k)) = v*k.
//
// Every function is __host__ __device__; the lane-pair swap is left to the
// caller (shuffles on the device, tests/native/fft_emul.cpp on the CPU).
#pragma once
#include "fft512.cuh"

namespace cvm {

// e^{i pi a / 32}, a = 0..15: the stride-32 part of the fold twist w^{32a}.
CVM_HD c64 twist32(int a) {
  switch (a) {
    case 1: return {0.9951847266721969, 0.0980171403295606};
    case 2: return {0.9807852804032304, 0.19509032201612828};
    case 3: return {0.9569403357322088, 0.2902846772544624};
    case 4: return {0.9238795325112867, 0.3826834323650898};
    case 5: return {0.881921264348355, 0.47139673682599764};
    case 6: return {0.8314696123025452, 0.5555702330196022};
    case 7: return {0.773010453362737, 0.6343932841636455};
    case 8: return {0.7071067811865476, 0.7071067811865476};
    case 9: return {0.6343932841636455, 0.773010453362737};
    case 10: return {0.5555702330196022, 0.8314696123025452};
    case 11: return {0.47139673682599764, 0.881921264348355};
    case 12: return {0.3826834323650898, 0.9238795325112867};
    case 13: return {0.2902846772544624, 0.9569403357322088};
    case 14: return {0.19509032201612828, 0.9807852804032304};
    case 15: return {0.0980171403295606, 0.9951847266721969};
    default: return {1.0, 0.0};
  }
}

constexpr double kCos8 = 0.9238795325112867;  // cos(pi/8)
constexpr double kSin8 = 0.3826834323650898;  // sin(pi/8)

// v * e^{-+ i pi / 4} (forward: conj = false -> (1 - i)/sqrt2)
template <bool kInverse>
CVM_HD c64 mul_w8(c64 v) {
  return kInverse ? c64{kRsqrt2 * (v.x - v.y), kRsqrt2 * (v.x + v.y)}
                  : c64{kRsqrt2 * (v.x + v.y), kRsqrt2 * (v.y - v.x)};
}
// v * (c, s) for the forward twiddle (c, -s) or its inverse (c, +s)
template <bool kInverse>
CVM_HD c64 mul_cs(c64 v, double c, double s) {
  return kInverse ? c64{fma(-v.y, s, v.x * c), fma(v.x, s, v.y * c)}
                  : c64{fma(v.y, s, v.x * c), fma(-v.x, s, v.y * c)};
}

template <bool kInverse>
CVM_HD void dft4(c64& x0, c64& x1, c64& x2, c64& x3) {
  const c64 a0 = cadd(x0, x2), a1 = csub(x0, x2);
  const c64 b0 = cadd(x1, x3), d = csub(x1, x3);
  const c64 b1 = kInverse ? c64{-d.y, d.x} : c64{d.y, -d.x};  // (x1 - x3) * (-+ i)
  x0 = cadd(a0, b0);
  x2 = csub(a0, b0);
  x1 = cadd(a1, b1);
  x3 = csub(a1, b1);
}

// In-place 16-point DFT, natural order in and out (4 x 4, n = 4 n1 + n2,
// k = k1 + 4 k2).  kInverse = false: X_k = sum x_n e^{-2 pi i nk/16}.
template <bool kInverse>
CVM_HD void dft16(c64 v[16]) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<kInverse>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // Y[n2][k1] sits in v[4 k1 + n2]; twiddle w16^{n2 k1}
  v[5] = mul_cs<kInverse>(v[5], kCos8, kSin8);     // (1,1): w16
  v[9] = mul_w8<kInverse>(v[9]);                   // (1,2): w8
  v[13] = mul_cs<kInverse>(v[13], kSin8, kCos8);   // (1,3): w16^3
  v[6] = mul_w8<kInverse>(v[6]);                   // (2,1): w8
  v[10] = kInverse ? c64{-v[10].y, v[10].x} : c64{v[10].y, -v[10].x};  // (2,2): -+i
  {                                                // (2,3): w16^6 = -conj(w8)...
    const c64 u = v[14];                           // forward (-r, -r), inverse (-r, +r)
    v[14] = kInverse ? c64{-kRsqrt2 * (u.x + u.y), kRsqrt2 * (u.x - u.y)}
                     : c64{kRsqrt2 * (u.y - u.x), -kRsqrt2 * (u.x + u.y)};
  }
  v[7] = mul_cs<kInverse>(v[7], kSin8, kCos8);     // (3,1): w16^3
  {                                                // (3,2): w16^6
    const c64 u = v[11];
    v[11] = kInverse ? c64{-kRsqrt2 * (u.x + u.y), kRsqrt2 * (u.x - u.y)}
                     : c64{kRsqrt2 * (u.y - u.x), -kRsqrt2 * (u.x + u.y)};
  }
  {                                                // (3,3): w16^9 = -w16
    const c64 u = mul_cs<kInverse>(v[15], kCos8, kSin8);
    v[15] = {-u.x, -u.y};
  }
  // DFT4 over n2 for each k1: inputs v[4 k1 + n2], outputs X[k1 + 4 k2]
  c64 o[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    c64 a = v[4 * k1], b = v[4 * k1 + 1], c = v[4 * k1 + 2], d = v[4 * k1 + 3];
    dft4<kInverse>(a, b, c, d);
    o[k1] = a;
    o[k1 + 4] = b;
    o[k1 + 8] = c;
    o[k1 + 12] = d;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = o[k];
}

// T[k] = base * w^k, k = 0..15, applied in place (tree of depth 4 from
// base, w, w^2, w^4, w^8; a few ulp, inside the rounding margin measured by
// tests/native/fft_emul.cpp).  kConj multiplies by the conjugates.
template <bool kConj>
CVM_HD void apply_pow16(c64 v[16], c64 base, c64 w) {
  // each twiddle is applied as soon as it exists, so at most a few are live
  auto mul = [](c64 x, c64 t) { return kConj ? cmul_conj(x, t) : cmul(x, t); };
  const c64 w2 = cmul(w, w), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
  v[0] = mul(v[0], base);
  v[1] = mul(v[1], cmul(base, w));
  const c64 t2 = cmul(base, w2);
  v[2] = mul(v[2], t2);
  v[3] = mul(v[3], cmul(t2, w));
  const c64 t4 = cmul(base, w4);
  v[4] = mul(v[4], t4);
  v[5] = mul(v[5], cmul(t4, w));
  const c64 t6 = cmul(t4, w2);
  v[6] = mul(v[6], t6);
  v[7] = mul(v[7], cmul(t6, w));
  const c64 t8 = cmul(base, w8);
  v[8] = mul(v[8], t8);
  v[9] = mul(v[9], cmul(t8, w));
  const c64 t10 = cmul(t8, w2);
  v[10] = mul(v[10], t10);
  v[11] = mul(v[11], cmul(t10, w));
  const c64 t12 = cmul(t8, w4);
  v[12] = mul(v[12], t12);
  v[13] = mul(v[13], cmul(t12, w));
  const c64 t14 = cmul(t12, w2);
  v[14] = mul(v[14], t14);
  v[15] = mul(v[15], cmul(t14, w));
}

// Per-lane twiddle bases of stage 1: T1[t][k0] = base * w^k0 with
// base = e^{i pi t / 1024} and w = e^{-i pi 4 t / 1024}.
struct TwBasesW {
  c64 base, w;
};

// ---------------------------------------------------------------- forward --
// Input v[a] = p_{t+32a} + i p_{t+32a+512} (untwisted).
CVM_HD void wfwd_twist_dft(c64 v[16]) {
#pragma unroll
  for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], twist32(a));
  dft16<false>(v);
}
CVM_HD void wfwd_stage1(c64 v[16], const TwBasesW& b) {
  wfwd_twist_dft(v);
  apply_pow16<false>(v, b.base, b.w);
}

// Transpose position (c64 units) of (k0, t) in a 512-entry buffer; the XOR
// keeps both the stage-1 writes (fixed k0, lanes t) and the stage-2 reads
// (fixed slot, lanes 2 k0 + e) on 8 distinct 16-byte bank groups per
// quarter-warp.
CVM_HD int wpos(int k0, int t) { return k0 * 32 + (t ^ ((2 * (k0 & 3) + ((t >> 3) & 1)) & 7)); }
// the t that stage-2 lane (k0, e) holds in slot s
CVM_HD int wslot_t(int e, int s) { return 8 * e + (s & 7) + 16 * (s >> 3); }

// w32^i = e^{-i pi i / 16} (i = 0..7) times v; kInverse: the conjugate
template <bool kInverse>
CVM_HD c64 mul_w32(c64 v, int i) {
  if (i == 0) return v;
  if (i == 4) return mul_w8<kInverse>(v);
  const c64 c = twist_const(i);  // e^{+i pi i / 16}
  return kInverse ? cmul(v, c) : cmul_conj(v, c);
}

// Stage 2a (before the lane-pair swap): slots (i, 8+i) = (y_m, y_{m+16}),
// m = 8e + i.  Leaves the kept value in slot i and the one to send in 8+i.
CVM_HD void wfwd_stage2a(c64 v[16], int e) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const c64 A = v[i], B = v[8 + i];
    const c64 s = cadd(A, B);
    const c64 c = mul_w32<false>(csub(A, B), i);
    const c64 d = e ? c64{c.y, -c.x} : c;  // w32^{8e} = (-i)^e
    v[i] = e ? d : s;
    v[8 + i] = e ? s : d;
  }
}
// Stage 2b (after the swap put the partner's half in slots 8..15).
CVM_HD void wfwd_stage2b(c64 v[16]) { dft16<false>(v); }

// ---------------------------------------------------------------- inverse --
// Mirror image: stage 2b^-1, swap slots 8..15 back (caller), stage 2a^-1,
// transpose, stage 1^-1.  Output v[a] = M * (p_{t+32a} + i p_{t+32a+512}).
CVM_HD void winv_stage2b(c64 v[16]) { dft16<true>(v); }
CVM_HD void winv_stage2a(c64 v[16], int e) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const c64 keep = v[i], recv = v[8 + i];
    const c64 s = e ? recv : keep;
    const c64 d0 = e ? keep : recv;
    const c64 d = e ? c64{-d0.y, d0.x} : d0;  // times i^e
    const c64 c = mul_w32<true>(d, i);
    v[i] = cadd(s, c);
    v[8 + i] = csub(s, c);
  }
}
CVM_HD void winv_dft_untwist(c64 v[16]) {
  dft16<true>(v);
#pragma unroll
  for (int a = 1; a < 16; ++a) v[a] = cmul_conj(v[a], twist32(a));
}
CVM_HD void winv_stage1(c64 v[16], const TwBasesW& b) {
  apply_pow16<true>(v, b.base, b.w);
  winv_dft_untwist(v);
}

// Host-side exact bases for lane t (long double), shared by the device
// table builder and the CPU emulation.
inline TwBasesW make_wbases(int t) {
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double ab = pi * t / 1024.0L, aw = -pi * 4 * t / 1024.0L;
  return {{(double)std::cos(ab), (double)std::sin(ab)}, {(double)std::cos(aw), (double)std::sin(aw)}};
}

}  // namespace cvm
