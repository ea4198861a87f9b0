/*
 * CPU restatement of TFHE gate bootstrapping (parity oracle).  See
 * tfhe_oracle.h for scope, provenance and the test-infrastructure-only rule.
 *
 * Compiled with -ffp-contract=off so the Box-Muller noise sampler gives the
 * same doubles as the product's host keygen.
 */
#define _GNU_SOURCE
#include "tfhe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define N OR_N_POLY
#define NL OR_N_LWE

/* ------------------------------------------------------------------ RNG --
 * splitmix64 seeding + xoshiro256**; streams keep keys / encryption apart. */
typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix64(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void rng_init(rng_t* r, uint64_t seed, uint64_t stream) {
  uint64_t x = seed ^ (stream * 0xD1B54A32D192ED03ull);
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(rng_t* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
  s[2] ^= t; s[3] = rotl(s[3], 45);
  return result;
}
static uint32_t rng_u32(rng_t* r) { return (uint32_t)(rng_next(r) >> 32); }
static int32_t rng_bit(rng_t* r) { return (int32_t)(rng_next(r) >> 63); }
/* Torus32 Gaussian of standard deviation sigma (as a fraction of the torus). */
static uint32_t rng_gauss_t32(rng_t* r, double sigma) {
  double u1 = (double)((rng_next(r) >> 11) + 1) * 0x1.0p-53;
  double u2 = (double)(rng_next(r) >> 11) * 0x1.0p-53;
  double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  double x = g * sigma * 4294967296.0;
  return (uint32_t)(int32_t)(int64_t)floor(x + 0.5);
}

#define KS_STDEV 0x1.0p-15
#define BK_STDEV 0x1.0p-25
#define STREAM_KEYS 1
#define STREAM_ENC 2
#define MU (1u << 29)

/* Negacyclic product with a binary key polynomial: out = a * z mod X^N+1. */
static void mul_binary_key(const uint32_t* a, const int32_t* z, uint32_t* out) {
  memset(out, 0, N * sizeof(uint32_t));
  for (int k = 0; k < N; ++k) {
    if (!z[k]) continue;
    /* X^k * a */
    for (int j = 0; j < N; ++j) {
      int d = j + k;
      if (d < N) out[d] += a[j];
      else out[d - N] -= a[j];
    }
  }
}

void oracle_keygen(uint64_t seed, int32_t* lwe_key, int32_t* tlwe_key,
                   uint32_t* bk, uint32_t* ksk) {
  rng_t r;
  rng_init(&r, seed, STREAM_KEYS);
  for (int i = 0; i < NL; ++i) lwe_key[i] = rng_bit(&r);
  for (int i = 0; i < N; ++i) tlwe_key[i] = rng_bit(&r);
  /* BK_i = TRGSW(s_i) under z: 6 TRLWE rows of (a, b = a*z + e), plus
   * s_i * h_p on the `part` polynomial's constant coefficient
   * (h_p = 2^(32 - (p+1)*Bgbit)). */
  uint32_t e[N];
  for (int i = 0; i < NL; ++i) {
    for (int row = 0; row < 6; ++row) {
      uint32_t* a = bk + ((size_t)(i * 6 + row) * 2 + 0) * N;
      uint32_t* b = bk + ((size_t)(i * 6 + row) * 2 + 1) * N;
      for (int j = 0; j < N; ++j) a[j] = rng_u32(&r);
      for (int j = 0; j < N; ++j) e[j] = rng_gauss_t32(&r, BK_STDEV);
      mul_binary_key(a, tlwe_key, b);
      for (int j = 0; j < N; ++j) b[j] += e[j];
      const int part = row / OR_L, p = row % OR_L;
      const uint32_t h = 1u << (32 - (p + 1) * OR_BGBIT);
      if (lwe_key[i]) {
        if (part == 0) a[0] += h;
        else b[0] += h;
      }
    }
  }
  /* KSK[i][j][v] = LWE_s(z_i * v * 2^(32-(j+1)*basebit)), v = 0 is zero. */
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < OR_KS_T; ++j) {
      for (int v = 0; v < 4; ++v) {
        uint32_t* row = ksk + ((size_t)(i * OR_KS_T + j) * 4 + v) * OR_LWE_WORDS;
        if (v == 0) {
          memset(row, 0, OR_LWE_WORDS * sizeof(uint32_t));
          continue;
        }
        uint32_t acc = 0;
        for (int k = 0; k < NL; ++k) {
          row[k] = rng_u32(&r);
          acc += row[k] * (uint32_t)lwe_key[k];
        }
        uint32_t msg = (uint32_t)tlwe_key[i] * (uint32_t)v *
                       (1u << (32 - (j + 1) * OR_KS_BASEBIT));
        row[NL] = acc + rng_gauss_t32(&r, KS_STDEV) + msg;
      }
    }
  }
}

void oracle_encrypt(uint64_t seed, const int32_t* lwe_key, int count,
                    const uint8_t* bits, uint32_t* out) {
  rng_t r;
  rng_init(&r, seed, STREAM_ENC);
  for (int g = 0; g < count; ++g) {
    uint32_t* c = out + (size_t)g * OR_LWE_WORDS;
    uint32_t acc = 0;
    for (int k = 0; k < NL; ++k) {
      c[k] = rng_u32(&r);
      acc += c[k] * (uint32_t)lwe_key[k];
    }
    c[NL] = acc + rng_gauss_t32(&r, KS_STDEV) + (bits[g] ? MU : (uint32_t)-MU);
  }
}

static int32_t phase_of(const uint32_t* c, const int32_t* key, int n) {
  uint32_t acc = 0;
  for (int k = 0; k < n; ++k) acc += c[k] * (uint32_t)key[k];
  return (int32_t)(c[n] - acc);
}

void oracle_decrypt(const int32_t* lwe_key, int count, const uint32_t* in,
                    uint8_t* bits, int32_t* phases) {
  for (int g = 0; g < count; ++g) {
    int32_t ph = phase_of(in + (size_t)g * OR_LWE_WORDS, lwe_key, NL);
    if (bits) bits[g] = ph > 0;
    if (phases) phases[g] = ph;
  }
}

/* Extracted samples are keyed by the TRLWE key coefficients. */
void oracle_decrypt_x(const int32_t* tlwe_key, int count, const uint32_t* in,
                      uint8_t* bits, int32_t* phases) {
  for (int g = 0; g < count; ++g) {
    int32_t ph = phase_of(in + (size_t)g * OR_XLWE_WORDS, tlwe_key, N);
    if (bits) bits[g] = ph > 0;
    if (phases) phases[g] = ph;
  }
}

/* ------------------------------------------- exact NTT mod 2^64-2^32+1 -- */
static const uint64_t P = 0xFFFFFFFF00000001ull;
static const uint64_t EPS = 0xFFFFFFFFull; /* 2^64 mod P */

static inline uint64_t add_p(uint64_t a, uint64_t b) {
  uint64_t r = a + b;
  if (r < a) r += EPS;
  else if (r >= P) r -= P;
  return r;
}
static inline uint64_t sub_p(uint64_t a, uint64_t b) {
  uint64_t r = a - b;
  if (a < b) r += P;
  return r;
}
static inline uint64_t mul_p(uint64_t a, uint64_t b) {
  unsigned __int128 x = (unsigned __int128)a * b;
  uint64_t lo = (uint64_t)x, hi = (uint64_t)(x >> 64);
  uint64_t hh = hi >> 32, hl = hi & EPS;
  uint64_t t0 = lo - hh;
  if (lo < hh) t0 -= EPS;
  uint64_t t1 = hl * EPS;
  uint64_t r = t0 + t1;
  if (r < t1) r += EPS;
  if (r >= P) r -= P;
  return r;
}
static uint64_t pow_p(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mul_p(r, b);
    b = mul_p(b, b);
    e >>= 1;
  }
  return r;
}

typedef struct {
  uint64_t psi[N], psi_inv[N]; /* psi^j, psi^-j * N^-1 */
  uint64_t w[N], w_inv[N];     /* omega^k for the cyclic stages */
  int rev[N];
} ntt_tables;
static ntt_tables g_ntt;
static pthread_once_t g_ntt_once = PTHREAD_ONCE_INIT;

static void ntt_init(void) {
  /* 7 generates Z_P^*; psi = 7^((P-1)/2N) has order 2N = 2048. */
  uint64_t psi = pow_p(7, (P - 1) / (2 * N));
  uint64_t psi_i = pow_p(psi, 2 * N - 1);
  uint64_t n_inv = pow_p(N, P - 2);
  uint64_t a = 1, b = n_inv;
  for (int j = 0; j < N; ++j) {
    g_ntt.psi[j] = a;
    g_ntt.psi_inv[j] = b;
    a = mul_p(a, psi);
    b = mul_p(b, psi_i);
  }
  uint64_t om = mul_p(psi, psi), om_i = pow_p(om, N - 1);
  a = 1;
  b = 1;
  for (int k = 0; k < N; ++k) {
    g_ntt.w[k] = a;
    g_ntt.w_inv[k] = b;
    a = mul_p(a, om);
    b = mul_p(b, om_i);
  }
  for (int i = 0; i < N; ++i) {
    int r = 0;
    for (int bit = 0; bit < 10; ++bit)
      if (i & (1 << bit)) r |= 1 << (9 - bit);
    g_ntt.rev[i] = r;
  }
}

static void ntt_cyclic(uint64_t* a, const uint64_t* w) {
  for (int i = 0; i < N; ++i)
    if (i < g_ntt.rev[i]) {
      uint64_t t = a[i];
      a[i] = a[g_ntt.rev[i]];
      a[g_ntt.rev[i]] = t;
    }
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1, step = N / len;
    for (int i = 0; i < N; i += len)
      for (int j = 0; j < half; ++j) {
        uint64_t u = a[i + j], v = mul_p(a[i + j + half], w[j * step]);
        a[i + j] = add_p(u, v);
        a[i + j + half] = sub_p(u, v);
      }
  }
}
static void ntt_fwd(uint64_t* a) {
  for (int j = 0; j < N; ++j) a[j] = mul_p(a[j], g_ntt.psi[j]);
  ntt_cyclic(a, g_ntt.w);
}
static void ntt_inv(uint64_t* a) {
  ntt_cyclic(a, g_ntt.w_inv);
  for (int j = 0; j < N; ++j) a[j] = mul_p(a[j], g_ntt.psi_inv[j]);
}
static inline uint64_t to_p(int64_t v) { return v >= 0 ? (uint64_t)v : P - (uint64_t)(-v); }
/* centred lift to Z, then mod 2^32 */
static inline uint32_t from_p(uint64_t v) {
  return v > P / 2 ? (uint32_t)(0u - (uint32_t)(P - v)) : (uint32_t)v;
}

/* ------------------------------------------------------- FFT mode hooks -- */
void ff_init(void);
void ff_forward_int(const int32_t* in, double* out);     /* 512 complex */
void ff_forward_u32(const uint32_t* in, double* out);    /* signed view */
void ff_inverse_round(const double* in, uint32_t* out);  /* scaled, rounded */

/* ------------------------------------------------------------ key tables -- */
struct oracle_keys {
  int mode;
  const uint32_t* bk;   /* time domain (schoolbook mode); caller-owned copy */
  uint32_t* bk_copy;
  uint64_t* bk_ntt;     /* [i][row][poly][N] */
  double* bk_fft;       /* [i][row][poly][512 complex] */
  uint32_t* ksk;
};

oracle_keys* oracle_keys_load(const uint32_t* bk, const uint32_t* ksk, int mode) {
  oracle_keys* k = (oracle_keys*)calloc(1, sizeof(*k));
  k->mode = mode;
  k->ksk = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)OR_KSK_WORDS);
  memcpy(k->ksk, ksk, sizeof(uint32_t) * (size_t)OR_KSK_WORDS);
  const size_t npoly = (size_t)NL * 6 * 2;
  if (mode == OR_MODE_NTT) {
    pthread_once(&g_ntt_once, ntt_init);
    k->bk_ntt = (uint64_t*)malloc(sizeof(uint64_t) * npoly * N);
    for (size_t p = 0; p < npoly; ++p) {
      uint64_t* d = k->bk_ntt + p * N;
      for (int j = 0; j < N; ++j) d[j] = to_p((int32_t)bk[p * N + j]);
      ntt_fwd(d);
    }
  } else if (mode == OR_MODE_FFT) {
    ff_init();
    k->bk_fft = (double*)malloc(sizeof(double) * npoly * N);
    for (size_t p = 0; p < npoly; ++p) ff_forward_u32(bk + p * N, k->bk_fft + p * N);
  } else {
    k->bk_copy = (uint32_t*)malloc(sizeof(uint32_t) * npoly * N);
    memcpy(k->bk_copy, bk, sizeof(uint32_t) * npoly * N);
    k->bk = k->bk_copy;
  }
  return k;
}

void oracle_keys_free(oracle_keys* k) {
  if (!k) return;
  free(k->bk_copy);
  free(k->bk_ntt);
  free(k->bk_fft);
  free(k->ksk);
  free(k);
}

static void schoolbook(const int32_t* d, const uint32_t* p, uint32_t* out) {
  memset(out, 0, N * sizeof(uint32_t));
  for (int i = 0; i < N; ++i) {
    if (!d[i]) continue;
    const uint32_t di = (uint32_t)d[i];
    for (int j = 0; j < N; ++j) {
      int t = i + j;
      if (t < N) out[t] += di * p[j];
      else out[t - N] -= di * p[j];
    }
  }
}

void oracle_negacyclic_mul(int mode, const int32_t* digits, const uint32_t* poly,
                           uint32_t* out) {
  if (mode == OR_MODE_SCHOOLBOOK) {
    schoolbook(digits, poly, out);
  } else if (mode == OR_MODE_NTT) {
    pthread_once(&g_ntt_once, ntt_init);
    uint64_t a[N], b[N];
    for (int j = 0; j < N; ++j) {
      a[j] = to_p(digits[j]);
      b[j] = to_p((int32_t)poly[j]);
    }
    ntt_fwd(a);
    ntt_fwd(b);
    for (int j = 0; j < N; ++j) a[j] = mul_p(a[j], b[j]);
    ntt_inv(a);
    for (int j = 0; j < N; ++j) out[j] = from_p(a[j]);
  } else {
    ff_init();
    double a[N], b[N], c[N];
    ff_forward_int(digits, a);
    ff_forward_u32(poly, b);
    for (int k = 0; k < N / 2; ++k) {  /* split spectra: re[0..511], im[512..] */
      double ar = a[k], ai = a[k + N / 2], br = b[k], bi = b[k + N / 2];
      c[k] = ar * br - ai * bi;
      c[k + N / 2] = ar * bi + ai * br;
    }
    ff_inverse_round(c, out);
  }
}

/* ------------------------------------------------------- bootstrapping -- */
uint32_t oracle_modswitch(uint32_t phase) {
  /* round(phase * 2N / 2^32) mod 2N  ==  ((u64)phase<<32 + 2^52) >> 53 */
  return (uint32_t)((((uint64_t)phase << 32) + (1ull << 52)) >> 53) & (2 * N - 1);
}

/* out = X^a * in, a in [0, 2N) */
static void mul_xai(uint32_t* out, int a, const uint32_t* in) {
  /* coefficient j takes in[(j - a) mod 2N], negated when that index >= N */
  if (a < N) {
    for (int j = 0; j < a; ++j) out[j] = 0u - in[j - a + N];
    for (int j = a; j < N; ++j) out[j] = in[j - a];
  } else {
    const int b = a - N;
    for (int j = 0; j < b; ++j) out[j] = in[j - b + N];
    for (int j = b; j < N; ++j) out[j] = 0u - in[j - b];
  }
}

/* Signed gadget decomposition (bk_l=3, Bgbit=7): offset trick, truncating. */
static void decompose(const uint32_t* c, int32_t d[OR_L][N]) {
  const uint32_t half = 1u << (OR_BGBIT - 1), mask = (1u << OR_BGBIT) - 1;
  uint32_t offset = 0;
  for (int p = 0; p < OR_L; ++p) offset += 1u << (32 - (p + 1) * OR_BGBIT);
  offset *= half;
  for (int j = 0; j < N; ++j) {
    const uint32_t buf = c[j] + offset;
    for (int p = 0; p < OR_L; ++p)
      d[p][j] = (int32_t)((buf >> (32 - (p + 1) * OR_BGBIT)) & mask) - (int32_t)half;
  }
}

typedef struct {
  uint64_t nt[2][N];   /* NTT-domain accumulators */
  double ff[2][N];     /* FFT-domain accumulators */
  uint64_t tmp[N];
  double ftmp[N];
  uint32_t t32[N];
} scratch_t;

/* acc += ExtProd(BK_i, diff) where diff = (X^a - 1) acc. */
static void cmux_step(const oracle_keys* k, int i, uint32_t acc[2][N],
                      int bara, scratch_t* s) {
  uint32_t diff[2][N];
  int32_t dig[2][OR_L][N];
  for (int part = 0; part < 2; ++part) {
    mul_xai(diff[part], bara, acc[part]);
    for (int j = 0; j < N; ++j) diff[part][j] -= acc[part][j];
    decompose(diff[part], dig[part]);
  }
  if (k->mode == OR_MODE_SCHOOLBOOK) {
    for (int part = 0; part < 2; ++part)
      for (int p = 0; p < OR_L; ++p) {
        const int row = part * OR_L + p;
        for (int out = 0; out < 2; ++out) {
          schoolbook(dig[part][p], k->bk + ((size_t)(i * 6 + row) * 2 + out) * N, s->t32);
          for (int j = 0; j < N; ++j) acc[out][j] += s->t32[j];
        }
      }
    return;
  }
  if (k->mode == OR_MODE_NTT) {
    memset(s->nt, 0, sizeof(s->nt));
    for (int part = 0; part < 2; ++part)
      for (int p = 0; p < OR_L; ++p) {
        const int row = part * OR_L + p;
        for (int j = 0; j < N; ++j) s->tmp[j] = to_p(dig[part][p][j]);
        ntt_fwd(s->tmp);
        for (int out = 0; out < 2; ++out) {
          const uint64_t* b = k->bk_ntt + ((size_t)(i * 6 + row) * 2 + out) * N;
          for (int j = 0; j < N; ++j)
            s->nt[out][j] = add_p(s->nt[out][j], mul_p(s->tmp[j], b[j]));
        }
      }
    for (int out = 0; out < 2; ++out) {
      ntt_inv(s->nt[out]);
      for (int j = 0; j < N; ++j) acc[out][j] += from_p(s->nt[out][j]);
    }
    return;
  }
  /* FFT mode */
  memset(s->ff, 0, sizeof(s->ff));
  for (int part = 0; part < 2; ++part)
    for (int p = 0; p < OR_L; ++p) {
      const int row = part * OR_L + p;
      ff_forward_int(dig[part][p], s->ftmp);
      for (int out = 0; out < 2; ++out) {
        const double* restrict br = k->bk_fft + ((size_t)(i * 6 + row) * 2 + out) * N;
        const double* restrict bi = br + N / 2;
        double* restrict ar = s->ff[out];
        double* restrict ai = ar + N / 2;
        const double* restrict xr = s->ftmp;
        const double* restrict xi = s->ftmp + N / 2;
        for (int q = 0; q < N / 2; ++q) {
          ar[q] += xr[q] * br[q] - xi[q] * bi[q];
          ai[q] += xr[q] * bi[q] + xi[q] * br[q];
        }
      }
    }
  for (int out = 0; out < 2; ++out) {
    ff_inverse_round(s->ff[out], s->t32);
    for (int j = 0; j < N; ++j) acc[out][j] += s->t32[j];
  }
}

void oracle_blind_rotate_extract(const oracle_keys* k, const uint32_t* lwe,
                                 uint32_t mu, uint32_t* out) {
  if (k->mode == OR_MODE_NTT) pthread_once(&g_ntt_once, ntt_init);
  scratch_t* s = (scratch_t*)malloc(sizeof(scratch_t));
  uint32_t acc[2][N], tv[N];
  for (int j = 0; j < N; ++j) tv[j] = mu;
  const int barb = (int)oracle_modswitch(lwe[NL]);
  memset(acc[0], 0, sizeof(acc[0]));
  mul_xai(acc[1], (2 * N - barb) % (2 * N), tv);
  for (int i = 0; i < NL; ++i) {
    const int bara = (int)oracle_modswitch(lwe[i]);
    if (bara == 0) continue;
    cmux_step(k, i, acc, bara, s);
  }
  out[0] = acc[0][0];
  for (int j = 1; j < N; ++j) out[j] = 0u - acc[0][N - j];
  out[N] = acc[1][0];
  free(s);
}

void oracle_key_switch(const oracle_keys* k, const uint32_t* x, uint32_t* out) {
  memset(out, 0, OR_LWE_WORDS * sizeof(uint32_t));
  out[NL] = x[N];
  const uint32_t prec = 1u << (32 - (1 + OR_KS_BASEBIT * OR_KS_T));
  for (int i = 0; i < N; ++i) {
    const uint32_t abar = x[i] + prec;
    for (int j = 0; j < OR_KS_T; ++j) {
      const uint32_t v = (abar >> (32 - (j + 1) * OR_KS_BASEBIT)) & 3u;
      if (!v) continue;
      const uint32_t* row = k->ksk + ((size_t)(i * OR_KS_T + j) * 4 + v) * OR_LWE_WORDS;
      for (int q = 0; q < OR_LWE_WORDS; ++q) out[q] -= row[q];
    }
  }
}

/* (const, coeff_a, coeff_b) of each bootstrapped binary gate. */
static int gate_combo(int kind, uint32_t* c, int* ca, int* cb) {
  const uint32_t e = 1u << 29, q = 1u << 30; /* 1/8, 1/4 */
  switch (kind) {
    case OR_NAND:  *c = e;      *ca = -1; *cb = -1; return 0;
    case OR_AND:   *c = 0u - e; *ca = 1;  *cb = 1;  return 0;
    case OR_OR:    *c = e;      *ca = 1;  *cb = 1;  return 0;
    case OR_XOR:   *c = q;      *ca = 2;  *cb = 2;  return 0;
    case OR_XNOR:  *c = 0u - q; *ca = -2; *cb = -2; return 0;
    case OR_NOR:   *c = 0u - e; *ca = -1; *cb = -1; return 0;
    case OR_ANDNY: *c = 0u - e; *ca = -1; *cb = 1;  return 0;
    case OR_ANDYN: *c = 0u - e; *ca = 1;  *cb = -1; return 0;
    case OR_ORNY:  *c = e;      *ca = -1; *cb = 1;  return 0;
    case OR_ORYN:  *c = e;      *ca = 1;  *cb = -1; return 0;
    default: return -1;
  }
}

static void combine(uint32_t c, int ca, const uint32_t* a, int cb,
                    const uint32_t* b, uint32_t* out) {
  for (int q = 0; q < OR_LWE_WORDS; ++q)
    out[q] = (uint32_t)ca * a[q] + (uint32_t)cb * b[q];
  out[NL] += c;
}

static int one_gate(const oracle_keys* k, int kind, const uint32_t* a,
                    const uint32_t* b, const uint32_t* c, uint32_t* out) {
  uint32_t t[OR_LWE_WORDS], x1[OR_XLWE_WORDS], x2[OR_XLWE_WORDS];
  if (kind == OR_MUX) {
    const uint32_t e = 1u << 29;
    combine(0u - e, 1, a, 1, b, t);       /* AND(sel, on_true)        */
    oracle_blind_rotate_extract(k, t, MU, x1);
    combine(0u - e, -1, a, 1, c, t);      /* AND(NOT sel, on_false)   */
    oracle_blind_rotate_extract(k, t, MU, x2);
    for (int q = 0; q < OR_XLWE_WORDS; ++q) x1[q] += x2[q];
    x1[N] += e;                           /* + (0, 1/8)               */
    oracle_key_switch(k, x1, out);
    return 0;
  }
  uint32_t cst;
  int ca, cb;
  if (gate_combo(kind, &cst, &ca, &cb)) return -1;
  combine(cst, ca, a, cb, b, t);
  oracle_blind_rotate_extract(k, t, MU, x1);
  oracle_key_switch(k, x1, out);
  return 0;
}

typedef struct {
  const oracle_keys* k;
  int count, stride, start;
  const uint8_t* kinds;
  const uint32_t *a, *b, *c;
  uint32_t* out;
  int err;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  for (int g = j->start; g < j->count; g += j->stride) {
    const size_t o = (size_t)g * OR_LWE_WORDS;
    if (one_gate(j->k, j->kinds[g], j->a + o, j->b + o, j->c ? j->c + o : NULL,
                 j->out + o))
      j->err = -1;
  }
  return NULL;
}

/* ---- batched lockstep evaluation (the CPU speed baseline) ----------------
 * The per-gate worker above streams the whole bootstrapping key (62 MB in FFT
 * domain) once per gate per thread, so many threads are DRAM-bound.  Batched
 * the way the GPU runs a level: every bootstrap of the batch advances one CMux
 * step at a time, all threads on the same key row (96 KB, cache-resident
 * across the thread's bootstraps), one barrier per step. */
typedef struct {
  uint32_t acc[2][N];
  uint16_t bar[NL + 1];
} brstate_t;

typedef struct {
  const oracle_keys* k;
  brstate_t* st;
  int nboot, tid, nthreads;
  pthread_barrier_t* barrier;
  /* epilogue: gates g = tid, tid + nthreads, ... (first[g] = its bootstrap) */
  int count;
  const uint8_t* kinds;
  const int* first;
  uint32_t* out;
} lockstep_t;

static void lockstep_extract(const brstate_t* st, uint32_t* out);

static void* lockstep_worker(void* arg) {
  lockstep_t* L = (lockstep_t*)arg;
  scratch_t* s = (scratch_t*)malloc(sizeof(scratch_t));
  for (int i = 0; i < NL; ++i) {
    for (int j = L->tid; j < L->nboot; j += L->nthreads) {
      const int a = L->st[j].bar[i];
      if (a) cmux_step(L->k, i, L->st[j].acc, a, s);
    }
    pthread_barrier_wait(L->barrier);
  }
  free(s);
  /* extraction + key switch (MUX: both extractions + (0, 1/8)) */
  for (int g = L->tid; g < L->count; g += L->nthreads) {
    uint32_t x1[OR_XLWE_WORDS], x2[OR_XLWE_WORDS];
    const int j = L->first[g];
    lockstep_extract(&L->st[j], x1);
    if (L->kinds[g] == OR_MUX) {
      lockstep_extract(&L->st[j + 1], x2);
      for (int q = 0; q < OR_XLWE_WORDS; ++q) x1[q] += x2[q];
      x1[N] += 1u << 29;
    }
    oracle_key_switch(L->k, x1, L->out + (size_t)g * OR_LWE_WORDS);
  }
  return NULL;
}

static void lockstep_init(brstate_t* st, const uint32_t* lwe) {
  uint32_t tv[N];
  for (int j = 0; j < N; ++j) tv[j] = MU;
  for (int i = 0; i <= NL; ++i) st->bar[i] = (uint16_t)oracle_modswitch(lwe[i]);
  memset(st->acc[0], 0, sizeof(st->acc[0]));
  mul_xai(st->acc[1], (2 * N - st->bar[NL]) % (2 * N), tv);
}

static void lockstep_extract(const brstate_t* st, uint32_t* out) {
  out[0] = st->acc[0][0];
  for (int j = 1; j < N; ++j) out[j] = 0u - st->acc[0][N - j];
  out[N] = st->acc[1][0];
}

static int gates_lockstep(const oracle_keys* k, int count, const uint8_t* kinds,
                          const uint32_t* in_a, const uint32_t* in_b, const uint32_t* in_c,
                          uint32_t* out, int threads) {
  int nboot = 0;
  int* first = (int*)malloc(sizeof(int) * (size_t)(count > 0 ? count : 1));
  if (!first) return -1;
  for (int g = 0; g < count; ++g) {
    first[g] = nboot;
    nboot += kinds[g] == OR_MUX ? 2 : 1;
  }
  brstate_t* st = (brstate_t*)malloc(sizeof(brstate_t) * (size_t)(nboot > 0 ? nboot : 1));
  if (!st) {
    free(first);
    return -1;
  }
  uint32_t t[OR_LWE_WORDS];
  for (int g = 0, j = 0; g < count; ++g) {
    const size_t o = (size_t)g * OR_LWE_WORDS;
    if (kinds[g] == OR_MUX) {
      const uint32_t e = 1u << 29;
      combine(0u - e, 1, in_a + o, 1, in_b + o, t);
      lockstep_init(&st[j++], t);
      combine(0u - e, -1, in_a + o, 1, in_c + o, t);
      lockstep_init(&st[j++], t);
    } else {
      uint32_t cst;
      int ca, cb;
      gate_combo(kinds[g], &cst, &ca, &cb);
      combine(cst, ca, in_a + o, cb, in_b + o, t);
      lockstep_init(&st[j++], t);
    }
  }
  if (threads > nboot) threads = nboot > 0 ? nboot : 1;
  if (threads > 256) threads = 256;
  pthread_barrier_t barrier;
  pthread_barrier_init(&barrier, NULL, (unsigned)threads);
  pthread_t tid[256];
  lockstep_t L[256];
  for (int i = 0; i < threads; ++i) {
    L[i] = (lockstep_t){k, st, nboot, i, threads, &barrier, count, kinds, first, out};
    if (i > 0) pthread_create(&tid[i], NULL, lockstep_worker, &L[i]);
  }
  lockstep_worker(&L[0]);
  for (int i = 1; i < threads; ++i) pthread_join(tid[i], NULL);
  pthread_barrier_destroy(&barrier);
  free(st);
  free(first);
  return 0;
}

int oracle_gates(const oracle_keys* k, int count, const uint8_t* kinds,
                 const uint32_t* in_a, const uint32_t* in_b,
                 const uint32_t* in_c, uint32_t* out, int threads) {
  if (k->mode == OR_MODE_NTT) pthread_once(&g_ntt_once, ntt_init);
  if (k->mode == OR_MODE_FFT) ff_init();
  for (int g = 0; g < count; ++g)
    if (kinds[g] < OR_NAND || kinds[g] > OR_MUX || (kinds[g] == OR_MUX && !in_c))
      return -1;
  if (k->mode == OR_MODE_FFT && count > 1)
    return gates_lockstep(k, count, kinds, in_a, in_b, in_c, out, threads < 1 ? 1 : threads);
  if (threads < 1) threads = 1;
  if (threads > count) threads = count > 0 ? count : 1;
  pthread_t tid[256];
  job_t jobs[256];
  if (threads > 256) threads = 256;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){k, count, threads, t, kinds, in_a, in_b, in_c, out, 0};
    if (t > 0) pthread_create(&tid[t], NULL, worker, &jobs[t]);
  }
  worker(&jobs[0]);
  int err = jobs[0].err;
  for (int t = 1; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    err |= jobs[t].err;
  }
  return err;
}
