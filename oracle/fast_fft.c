/*
 * Double-precision negacyclic FFT for the oracle's OR_MODE_FFT (the CPU speed
 * baseline; test infrastructure only -- see tfhe_oracle.h).
 *
 * This is the TFHE library's own method for the external product (a real
 * polynomial mod X^N+1 folded into N/2 complex points, twisted by the 2N-th
 * root of unity, one N/2-point complex FFT), restated as a plain iterative
 * radix-2 FFT.  N = 1024, M = N/2 = 512.  Complex arrays are interleaved
 * (re, im) doubles.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>

#define N 1024
#define M 512

static double tw_re[M], tw_im[M];      /* twist omega^j = e^{i pi j / N}     */
static double rt_re[M / 2], rt_im[M / 2]; /* e^{-2 pi i k / M}               */
static int rev9[M];
static pthread_once_t once = PTHREAD_ONCE_INIT;

static void init(void) {
  for (int j = 0; j < M; ++j) {
    tw_re[j] = cos(M_PI * j / N);
    tw_im[j] = sin(M_PI * j / N);
  }
  for (int k = 0; k < M / 2; ++k) {
    rt_re[k] = cos(2.0 * M_PI * k / M);
    rt_im[k] = -sin(2.0 * M_PI * k / M);
  }
  for (int i = 0; i < M; ++i) {
    int r = 0;
    for (int b = 0; b < 9; ++b)
      if (i & (1 << b)) r |= 1 << (8 - b);
    rev9[i] = r;
  }
}

void ff_init(void) { pthread_once(&once, init); }

/* In-place forward (sign = -1) or inverse-unscaled (sign = +1) FFT. */
static void fft512(double* a, int inverse) {
  for (int i = 0; i < M; ++i)
    if (i < rev9[i]) {
      double t0 = a[2 * i], t1 = a[2 * i + 1];
      a[2 * i] = a[2 * rev9[i]];
      a[2 * i + 1] = a[2 * rev9[i] + 1];
      a[2 * rev9[i]] = t0;
      a[2 * rev9[i] + 1] = t1;
    }
  for (int len = 2; len <= M; len <<= 1) {
    const int half = len >> 1, step = M / len;
    for (int i = 0; i < M; i += len)
      for (int j = 0; j < half; ++j) {
        const double wr = rt_re[j * step];
        const double wi = inverse ? -rt_im[j * step] : rt_im[j * step];
        double* u = a + 2 * (i + j);
        double* v = a + 2 * (i + j + half);
        const double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
        v[0] = u[0] - vr;
        v[1] = u[1] - vi;
        u[0] += vr;
        u[1] += vi;
      }
  }
}

static void forward_d(const double* p, double* out) {
  for (int j = 0; j < M; ++j) {
    const double x = p[j], y = p[j + M];
    out[2 * j] = x * tw_re[j] - y * tw_im[j];
    out[2 * j + 1] = x * tw_im[j] + y * tw_re[j];
  }
  fft512(out, 0);
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
  double a[N];
  for (int q = 0; q < N; ++q) a[q] = in[q];
  fft512(a, 1);
  const double s = 1.0 / M;
  for (int j = 0; j < M; ++j) {
    const double zr = a[2 * j] * s, zi = a[2 * j + 1] * s;
    const double wr = zr * tw_re[j] + zi * tw_im[j];
    const double wi = zi * tw_re[j] - zr * tw_im[j];
    out[j] = (uint32_t)(int64_t)llrint(wr);
    out[j + M] = (uint32_t)(int64_t)llrint(wi);
  }
}
