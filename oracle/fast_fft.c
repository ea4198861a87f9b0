/*
 * Double-precision negacyclic FFT for the oracle's OR_MODE_FFT (the CPU speed
 * baseline; test infrastructure only -- see tfhe_oracle.h).
 *
 * This is the TFHE library's own method for the external product (a real
 * polynomial mod X^N+1 folded into N/2 complex points, twisted by the 2N-th
 * root of unity, one N/2-point complex FFT), restated on split real/imaginary
 * arrays so the compiler vectorises the butterflies (AVX2 with
 * -march=x86-64-v3):
 *   forward = twist + decimation-in-frequency radix-2 (natural in,
 *             bit-reversed out), last two stages fused into a multiply-free
 *             radix-4 pass;
 *   inverse = the mirror decimation-in-time pass (bit-reversed in, natural
 *             out) + untwist.
 * Point-wise products do not care about bin order, so no bit reversal is ever
 * performed.  N = 1024, M = N/2 = 512.  Spectra are stored split:
 * re[0..511], im[0..511].
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

#define N 1024
#define M 512

static double tw_re[M], tw_im[M];  /* fold twist omega^j = e^{i pi j / N}       */
static double st_re[M], st_im[M];  /* stage twiddles: [h + j] = e^{-i pi j / h} */
static pthread_once_t once = PTHREAD_ONCE_INIT;

static void init(void) {
  for (int j = 0; j < M; ++j) {
    tw_re[j] = cos(M_PI * j / N);
    tw_im[j] = sin(M_PI * j / N);
  }
  for (int h = 1; h < M; h <<= 1)
    for (int j = 0; j < h; ++j) {
      st_re[h + j] = cos(M_PI * j / h);
      st_im[h + j] = -sin(M_PI * j / h);
    }
}

void ff_init(void) { pthread_once(&once, init); }

/* Forward DIF, stages h = 256 .. 4 with twiddles, then a fused radix-4 pass
 * for h = 2 (twiddles 1, -i) and h = 1 (twiddle 1). */
static void fft_dif(double* restrict re, double* restrict im) {
  for (int h = M / 2; h >= 4; h >>= 1) {
    const double* wr = st_re + h;
    const double* wi = st_im + h;
    for (int i = 0; i < M; i += 2 * h) {
      double* ur = re + i;
      double* ui = im + i;
      double* vr = re + i + h;
      double* vi = im + i + h;
      for (int j = 0; j < h; ++j) {
        const double ar = ur[j] - vr[j], ai = ui[j] - vi[j];
        ur[j] += vr[j];
        ui[j] += vi[j];
        vr[j] = ar * wr[j] - ai * wi[j];
        vi[j] = ar * wi[j] + ai * wr[j];
      }
    }
  }
  for (int i = 0; i < M; i += 4) {
    const double x0r = re[i], x1r = re[i + 1], x2r = re[i + 2], x3r = re[i + 3];
    const double x0i = im[i], x1i = im[i + 1], x2i = im[i + 2], x3i = im[i + 3];
    /* h = 2: (x0,x2), (x1,x3)*(-i) on the difference */
    const double a0r = x0r + x2r, a0i = x0i + x2i, a2r = x0r - x2r, a2i = x0i - x2i;
    const double a1r = x1r + x3r, a1i = x1i + x3i;
    const double d3r = x1r - x3r, d3i = x1i - x3i;
    const double a3r = d3i, a3i = -d3r; /* times -i */
    /* h = 1 */
    re[i] = a0r + a1r;
    im[i] = a0i + a1i;
    re[i + 1] = a0r - a1r;
    im[i + 1] = a0i - a1i;
    re[i + 2] = a2r + a3r;
    im[i + 2] = a2i + a3i;
    re[i + 3] = a2r - a3r;
    im[i + 3] = a2i - a3i;
  }
}

/* Inverse DIT (conjugate twiddles, unscaled): the exact mirror of fft_dif. */
static void fft_dit_inv(double* restrict re, double* restrict im) {
  for (int i = 0; i < M; i += 4) {
    const double y0r = re[i], y1r = re[i + 1], y2r = re[i + 2], y3r = re[i + 3];
    const double y0i = im[i], y1i = im[i + 1], y2i = im[i + 2], y3i = im[i + 3];
    /* h = 1 */
    const double a0r = y0r + y1r, a0i = y0i + y1i, a1r = y0r - y1r, a1i = y0i - y1i;
    const double a2r = y2r + y3r, a2i = y2i + y3i, e3r = y2r - y3r, e3i = y2i - y3i;
    /* h = 2: second of each pair times +i */
    const double a3r = -e3i, a3i = e3r;
    re[i] = a0r + a2r;
    im[i] = a0i + a2i;
    re[i + 2] = a0r - a2r;
    im[i + 2] = a0i - a2i;
    re[i + 1] = a1r + a3r;
    im[i + 1] = a1i + a3i;
    re[i + 3] = a1r - a3r;
    im[i + 3] = a1i - a3i;
  }
  for (int h = 4; h < M; h <<= 1) {
    const double* wr = st_re + h;
    const double* wi = st_im + h;
    for (int i = 0; i < M; i += 2 * h) {
      double* ur = re + i;
      double* ui = im + i;
      double* vr = re + i + h;
      double* vi = im + i + h;
      for (int j = 0; j < h; ++j) {
        const double br = vr[j] * wr[j] + vi[j] * wi[j];  /* v * conj(w) */
        const double bi = vi[j] * wr[j] - vr[j] * wi[j];
        vr[j] = ur[j] - br;
        vi[j] = ui[j] - bi;
        ur[j] += br;
        ui[j] += bi;
      }
    }
  }
}

static void forward_d(const double* p, double* out) {
  double* re = out;
  double* im = out + M;
  for (int j = 0; j < M; ++j) {
    const double x = p[j], y = p[j + M];
    re[j] = x * tw_re[j] - y * tw_im[j];
    im[j] = x * tw_im[j] + y * tw_re[j];
  }
  fft_dif(re, im);
}

void ff_forward_int(const int32_t* in, double* out) {
  double p[N];
  for (int j = 0; j < N; ++j) p[j] = (double)in[j];
  forward_d(p, out);
}

void ff_forward_u32(const uint32_t* in, double* out) {
  double p[N];
  for (int j = 0; j < N; ++j) p[j] = (double)(int32_t)in[j];
  forward_d(p, out);
}

/* round(v) mod 2^32 for |v| < 2^51 (round half to even, like llrint): add
 * 1.5 * 2^52 and keep the low mantissa word -- vectorisable, unlike llrint. */
static inline uint32_t round_torus(double v) {
  const double t = v + 6755399441055744.0;
  uint64_t bits;
  memcpy(&bits, &t, 8);
  return (uint32_t)bits;
}

void ff_inverse_round(const double* in, uint32_t* out) {
  double re[M], im[M];
  memcpy(re, in, sizeof(re));
  memcpy(im, in + M, sizeof(im));
  fft_dit_inv(re, im);
  const double s = 1.0 / M;
  for (int j = 0; j < M; ++j) {
    const double zr = re[j] * s, zi = im[j] * s;
    const double wr = zr * tw_re[j] + zi * tw_im[j];
    const double wi = zi * tw_re[j] - zr * tw_im[j];
    out[j] = round_torus(wr);
    out[j + M] = round_torus(wi);
  }
}
