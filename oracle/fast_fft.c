/*
 * Double-precision negacyclic FFT for the oracle's OR_MODE_FFT (the CPU speed
 * baseline; test infrastructure only -- see tfhe_oracle.h).
 *
 * This is the TFHE library's own method for the external product (a real
 * polynomial mod X^N+1 folded into N/2 complex points, twisted by the 2N-th
 * root of unity, one N/2-point complex FFT), restated as an iterative radix-2
 * FFT on split real/imaginary arrays with contiguous per-stage twiddles so the
 * compiler vectorises the butterflies (AVX2 with -march=x86-64-v3).
 * N = 1024, M = N/2 = 512.  Spectra are stored split: re[0..511], im[0..511].
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

#define N 1024
#define M 512

static double tw_re[M], tw_im[M];   /* fold twist omega^j = e^{i pi j / N}        */
static double st_re[M], st_im[M];   /* stage twiddles: [h + j] = e^{-i pi j / h}  */
static int rev9[M];
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
  for (int i = 0; i < M; ++i) {
    int r = 0;
    for (int b = 0; b < 9; ++b)
      if (i & (1 << b)) r |= 1 << (8 - b);
    rev9[i] = r;
  }
}

void ff_init(void) { pthread_once(&once, init); }

/* In-place DIT FFT on split arrays; inverse uses conjugate twiddles (unscaled). */
static void fft512(double* restrict re, double* restrict im, int inverse) {
  for (int i = 0; i < M; ++i) {
    const int r = rev9[i];
    if (i < r) {
      double t = re[i];
      re[i] = re[r];
      re[r] = t;
      t = im[i];
      im[i] = im[r];
      im[r] = t;
    }
  }
  const double sgn = inverse ? -1.0 : 1.0;
  for (int h = 1; h < M; h <<= 1) {
    const double* wr = st_re + h;
    const double* wi = st_im + h;
    for (int i = 0; i < M; i += 2 * h) {
      double* ur = re + i;
      double* ui = im + i;
      double* vr = re + i + h;
      double* vi = im + i + h;
      for (int j = 0; j < h; ++j) {
        const double c = wr[j], s = sgn * wi[j];
        const double xr = vr[j] * c - vi[j] * s;
        const double xi = vr[j] * s + vi[j] * c;
        vr[j] = ur[j] - xr;
        vi[j] = ui[j] - xi;
        ur[j] += xr;
        ui[j] += xi;
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
  fft512(re, im, 0);
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

void ff_inverse_round(const double* in, uint32_t* out) {
  double re[M], im[M];
  memcpy(re, in, sizeof(re));
  memcpy(im, in + M, sizeof(im));
  fft512(re, im, 1);
  const double s = 1.0 / M;
  for (int j = 0; j < M; ++j) {
    const double zr = re[j] * s, zi = im[j] * s;
    const double wr = zr * tw_re[j] + zi * tw_im[j];
    const double wi = zi * tw_re[j] - zr * tw_im[j];
    out[j] = (uint32_t)(int64_t)llrint(wr);
    out[j + M] = (uint32_t)(int64_t)llrint(wi);
  }
}
