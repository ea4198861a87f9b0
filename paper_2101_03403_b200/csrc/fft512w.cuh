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

// The same DFT16 with the twiddled second-stage radix-4 butterflies fused
// into FMAs (144 FP64 instructions instead of 160).  Columns k1 = 1 and 3
// factor cos(pi/8) out of their two twiddles (t = tan(pi/8)), so the
// butterfly sums become c * (P + t Q) -- one FMA per component -- and the
// final adds absorb c as FMAs; column k1 = 2 absorbs 1/sqrt2 the same way.
// The inverse is the forward transform with real and imaginary parts swapped
// on input and output (swap(z) = i conj(z), so swap o DFT o swap = IDFT):
// register renaming, no instructions.  Rounding differs from dft16 by a few ulp
// (tests/native/fft_emul.cpp checks products and the rounding margin).
constexpr double kTan8 = 0.41421356237309503;  // tan(pi/8)
template <bool kInverse>
CVM_HD void dft16f(c64 v[16]) {
  if (kInverse) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = {v[i].y, v[i].x};
  }
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<false>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // Y[n2][k1] in v[4 k1 + n2]; X[k1 + 4 k2] = output k2 of column k1
  c64 o[16];
  {  // k1 = 0: no twiddles
    c64 a = v[0], b = v[1], c = v[2], d = v[3];
    dft4<false>(a, b, c, d);
    o[0] = a, o[4] = b, o[8] = c, o[12] = d;
  }
  {  // k1 = 1: twiddles w16, w8, w16^3
    const c64 Y0 = v[4], Y1 = v[5], Y2 = v[6], Y3 = v[7];
    const double px = Y2.x + Y2.y, py = Y2.y - Y2.x;  // w8 Y2 = r p
    const c64 a0 = {fma(kRsqrt2, px, Y0.x), fma(kRsqrt2, py, Y0.y)};
    const c64 a1 = {fma(-kRsqrt2, px, Y0.x), fma(-kRsqrt2, py, Y0.y)};
    const double A = Y1.x + Y3.y, B = Y1.y + Y3.x, C = Y1.y - Y3.x, D = Y3.y - Y1.x;
    const double P1 = fma(kTan8, B, A), P2 = fma(kTan8, D, C);
    const double P3 = fma(kTan8, C, -D), P4 = fma(-kTan8, A, B);
    o[1] = {fma(kCos8, P1, a0.x), fma(kCos8, P2, a0.y)};
    o[9] = {fma(-kCos8, P1, a0.x), fma(-kCos8, P2, a0.y)};
    o[5] = {fma(kCos8, P4, a1.x), fma(-kCos8, P3, a1.y)};
    o[13] = {fma(-kCos8, P4, a1.x), fma(kCos8, P3, a1.y)};
  }
  {  // k1 = 2: twiddles w8, -i, w8^3
    const c64 Y0 = v[8], Y1 = v[9], Y2 = v[10], Y3 = v[11];
    const c64 a0 = {Y0.x + Y2.y, Y0.y - Y2.x}, a1 = {Y0.x - Y2.y, Y0.y + Y2.x};
    const double E = Y1.x + Y1.y, F = Y1.y - Y1.x, G = Y3.y - Y3.x, H = Y3.y + Y3.x;
    const double b0x = E + G, b0y = F - H, dx = E - G, dy = F + H;  // b0, d / r
    o[2] = {fma(kRsqrt2, b0x, a0.x), fma(kRsqrt2, b0y, a0.y)};
    o[10] = {fma(-kRsqrt2, b0x, a0.x), fma(-kRsqrt2, b0y, a0.y)};
    o[6] = {fma(kRsqrt2, dy, a1.x), fma(-kRsqrt2, dx, a1.y)};
    o[14] = {fma(-kRsqrt2, dy, a1.x), fma(kRsqrt2, dx, a1.y)};
  }
  {  // k1 = 3: twiddles w16^3, w8^3, w16^9
    const c64 Y0 = v[12], Y1 = v[13], Y2 = v[14], Y3 = v[15];
    const double px = Y2.y - Y2.x, q = Y2.x + Y2.y;  // w8^3 Y2 = r (px, -q)
    const c64 a0 = {fma(kRsqrt2, px, Y0.x), fma(-kRsqrt2, q, Y0.y)};
    const c64 a1 = {fma(-kRsqrt2, px, Y0.x), fma(kRsqrt2, q, Y0.y)};
    const double A = Y1.x + Y3.y, B = Y1.y + Y3.x, C = Y1.y - Y3.x, E = Y1.x - Y3.y;
    const double P1 = fma(kTan8, E, C), P2 = fma(kTan8, B, -A);
    const double P3 = fma(kTan8, A, B), P4 = fma(kTan8, C, -E);
    o[3] = {fma(kCos8, P1, a0.x), fma(kCos8, P2, a0.y)};
    o[11] = {fma(-kCos8, P1, a0.x), fma(-kCos8, P2, a0.y)};
    o[7] = {fma(kCos8, P4, a1.x), fma(-kCos8, P3, a1.y)};
    o[15] = {fma(-kCos8, P4, a1.x), fma(kCos8, P3, a1.y)};
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = kInverse ? c64{o[k].y, o[k].x} : o[k];
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
  dft16f<false>(v);
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
CVM_HD void wfwd_stage2b(c64 v[16]) { dft16f<false>(v); }

// ---------------------------------------------------------------- inverse --
// Mirror image: stage 2b^-1, swap slots 8..15 back (caller), stage 2a^-1,
// transpose, stage 1^-1.  Output v[a] = M * (p_{t+32a} + i p_{t+32a+512}).
CVM_HD void winv_stage2b(c64 v[16]) { dft16f<true>(v); }
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
  dft16f<true>(v);
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
