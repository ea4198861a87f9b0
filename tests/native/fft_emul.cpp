// CPU emulation of the 64-thread negacyclic FFT in
// paper_2101_03403_b200/csrc/fft512.cuh: runs the same __host__ __device__
// stage functions, exchange-buffer permutations and swizzle with 64 emulated
// threads and checks products of random (digit, torus32) polynomials against
// the exact negacyclic product.  Also checks the swizzle is bank-conflict-free.
// Two twiddle modes: the host tables (make_twiddles) and the generated
// twiddles of the kTwRec kernels (TwPow8 from two bases per thread) on the
// digit side; the key side always uses the tables (bk_to_fft_kernel).  The
// largest distance of an un-rounded output to the nearest integer is printed
// per mode -- the rounding margin (a flip needs 0.5).
//
// Build+run by tests/test_fft_emul.py:  g++ -O2 -std=c++17 -I<csrc> fft_emul.cpp
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "fft512.cuh"
#include "fft512w.cuh"

using namespace cvm;

static c64 T1[64][8], T2[64][8];
static c64 B1b[64], B1w[64], B2w[64];  // TwPow8 bases per thread
static bool g_rec = false;             // digit side uses generated twiddles

struct TabTw {
  const c64* p;
  const c64& operator[](int k) const { return p[k]; }
};

// forward: coefficient poly (as doubles) -> bins[t][k2]
static void forward(const double* p, c64 bins[64][8], bool rec) {
  c64 v[64][8];
  c64 buf[512];
  for (int t = 0; t < 64; ++t)
    for (int a = 0; a < 8; ++a) v[t][a] = {p[t + 64 * a], p[t + 64 * a + 512]};
  for (int t = 0; t < 64; ++t) {
    if (rec) fwd_stage1(v[t], TwPow8(B1b[t], B1w[t]));
    else fwd_stage1(v[t], TabTw{T1[t]});
  }
  for (int t = 0; t < 64; ++t)
    for (int z = 0; z < 8; ++z) buf[xpos(ex1_cell(t, z), t >> 3)] = v[t][z];
  for (int t = 0; t < 64; ++t)
    for (int s = 0; s < 8; ++s) v[t][s] = buf[xpos(t, s)];
  for (int t = 0; t < 64; ++t) {
    if (rec) fwd_stage2(v[t], TwPow8(B2w[t]));
    else fwd_stage2(v[t], TabTw{T2[t]});
  }
  for (int t = 0; t < 64; ++t)
    for (int z = 0; z < 8; ++z) buf[xpos(ex2_cell(t, z), t >> 3)] = v[t][z];
  for (int t = 0; t < 64; ++t)
    for (int s = 0; s < 8; ++s) v[t][s] = buf[xpos(t, s)];
  for (int t = 0; t < 64; ++t) {
    fwd_stage3(v[t]);
    for (int k = 0; k < 8; ++k) bins[t][k] = v[t][k];
  }
}

static void inverse(c64 bins[64][8], uint32_t* out, double* worst) {
  c64 v[64][8];
  c64 buf[512];
  for (int t = 0; t < 64; ++t)
    for (int k = 0; k < 8; ++k) v[t][k] = bins[t][k];
  for (int t = 0; t < 64; ++t) inv_stageA(v[t]);
  for (int t = 0; t < 64; ++t)
    for (int z = 0; z < 8; ++z) buf[xpos(ex2_cell(t, z), t >> 3)] = v[t][z];
  for (int t = 0; t < 64; ++t)
    for (int s = 0; s < 8; ++s) v[t][s] = buf[xpos(t, s)];
  for (int t = 0; t < 64; ++t) {
    if (g_rec) inv_stageB(v[t], TwPow8(B2w[t]));
    else inv_stageB(v[t], TabTw{T2[t]});
  }
  for (int t = 0; t < 64; ++t)
    for (int z = 0; z < 8; ++z) buf[xpos(exB_cell(t, z), t & 7)] = v[t][z];
  for (int t = 0; t < 64; ++t)
    for (int s = 0; s < 8; ++s) v[t][s] = buf[xpos(t, s)];
  for (int t = 0; t < 64; ++t) {
    if (g_rec) inv_stageC(v[t], TwPow8(B1b[t], B1w[t]));
    else inv_stageC(v[t], TabTw{T1[t]});
    for (int a = 0; a < 8; ++a) {
      for (double x : {v[t][a].x, v[t][a].y}) {
        const double d = std::fabs(x - std::nearbyint(x));
        if (d > *worst) *worst = d;
      }
      out[t + 64 * a] = round_to_torus(v[t][a].x);
      out[t + 64 * a + 512] = round_to_torus(v[t][a].y);
    }
  }
}

static bool check_swizzle() {
  // For each exchange pattern, every quarter-warp (8 consecutive threads)
  // writing value z, and reading slot s, must touch 8 distinct 16-B bank groups.
  auto distinct = [](int* g) {
    int seen = 0;
    for (int i = 0; i < 8; ++i) {
      if (seen & (1 << g[i])) return false;
      seen |= 1 << g[i];
    }
    return true;
  };
  int g[8];
  for (int q = 0; q < 8; ++q)
    for (int z = 0; z < 8; ++z) {
      for (int i = 0; i < 8; ++i) g[i] = xpos(ex1_cell(8 * q + i, z), q) & 7;
      if (!distinct(g)) return false;
      for (int i = 0; i < 8; ++i) g[i] = xpos(ex2_cell(8 * q + i, z), q) & 7;
      if (!distinct(g)) return false;
      for (int i = 0; i < 8; ++i) g[i] = xpos(exB_cell(8 * q + i, z), i) & 7;
      if (!distinct(g)) return false;
      for (int i = 0; i < 8; ++i) g[i] = xpos(8 * q + i, z) & 7;  // reads
      if (!distinct(g)) return false;
    }
  return true;
}

static int run(int trials, bool rec, double* worst) {
  g_rec = rec;
  std::mt19937_64 rng(7);
  for (int trial = 0; trial < trials; ++trial) {
    // 6 digit polys x 6 key polys summed, like one external-product output.
    std::vector<uint32_t> exact(1024, 0);
    c64 acc[64][8] = {};
    for (int r = 0; r < 6; ++r) {
      std::vector<int32_t> d(1024);
      std::vector<uint32_t> b(1024);
      for (auto& x : d) x = int32_t(rng() % 128) - 64;
      for (auto& x : b) x = uint32_t(rng());
      for (int i = 0; i < 1024; ++i)
        for (int j = 0; j < 1024; ++j) {
          uint32_t prod = uint32_t(d[i]) * b[j];
          if (i + j < 1024) exact[i + j] += prod;
          else exact[i + j - 1024] -= prod;
        }
      std::vector<double> dd(1024), bd(1024);
      for (int i = 0; i < 1024; ++i) {
        dd[i] = d[i];
        bd[i] = double(int32_t(b[i])) / 512.0;
      }
      c64 D[64][8], B[64][8];
      forward(dd.data(), D, rec);   // digit side: kernel's twiddle mode
      forward(bd.data(), B, false);  // key side: tables (bk_to_fft_kernel)
      for (int t = 0; t < 64; ++t)
        for (int k = 0; k < 8; ++k) acc[t][k] = cadd(acc[t][k], cmul(D[t][k], B[t][k]));
    }
    std::vector<uint32_t> got(1024);
    inverse(acc, got.data(), worst);
    for (int i = 0; i < 1024; ++i)
      if (got[i] != exact[i]) {
        printf("FAIL (%s) trial %d coef %d got %u want %u\n", rec ? "rec" : "table", trial, i,
               got[i], exact[i]);
        return 1;
      }
  }
  return 0;
}

// ------------------------------------------------ warp FFT (fft512w.cuh) --
// 32 emulated lanes; the lane-pair swap of slots 8..15 stands in for the
// kernel's shuffles.
static void wswap(c64 v[32][16]) {
  for (int l = 0; l < 32; l += 2)
    for (int i = 8; i < 16; ++i) std::swap(v[l][i], v[l + 1][i]);
}

static void wforward(const double* p, c64 bins[32][16], bool key) {
  c64 v[32][16];
  c64 buf[512];
  for (int t = 0; t < 32; ++t) {
    for (int a = 0; a < 16; ++a) v[t][a] = {p[t + 32 * a], p[t + 32 * a + 512]};
    wfwd_stage1(v[t], make_wbases(t));
    for (int k0 = 0; k0 < 16; ++k0) buf[wpos(k0, t)] = v[t][k0];
  }
  for (int l = 0; l < 32; ++l) {
    for (int s = 0; s < 16; ++s) v[l][s] = buf[wpos(l >> 1, wslot_t(l & 1, s))];
    wfwd_stage2a(v[l], l & 1);
  }
  wswap(v);
  for (int l = 0; l < 32; ++l) {
    wfwd_stage2b(v[l]);
    for (int r = 0; r < 16; ++r) {
      c64 x = v[l][r];
      if (key && (l & 1) && (r & 1)) x = {-x.x, -x.y};  // the key side stores F, not D F
      bins[l][r] = x;
    }
  }
}

static void winverse(c64 bins[32][16], uint32_t* out, double* worst) {
  c64 v[32][16];
  c64 buf[512];
  for (int l = 0; l < 32; ++l) {
    for (int r = 0; r < 16; ++r) v[l][r] = bins[l][r];
    winv_stage2b(v[l]);
  }
  wswap(v);
  for (int l = 0; l < 32; ++l) {
    winv_stage2a(v[l], l & 1);
    for (int s = 0; s < 16; ++s) buf[wpos(l >> 1, wslot_t(l & 1, s))] = v[l][s];
  }
  for (int t = 0; t < 32; ++t) {
    for (int k0 = 0; k0 < 16; ++k0) v[t][k0] = buf[wpos(k0, t)];
    winv_stage1(v[t], make_wbases(t));
    for (int a = 0; a < 16; ++a) {
      for (double x : {v[t][a].x, v[t][a].y}) {
        const double d = std::fabs(x - std::nearbyint(x));
        if (d > *worst) *worst = d;
      }
      out[t + 32 * a] = round_to_torus(v[t][a].x);
      out[t + 32 * a + 512] = round_to_torus(v[t][a].y);
    }
  }
}

static bool check_wswizzle() {
  for (int q = 0; q < 4; ++q)
    for (int z = 0; z < 16; ++z) {
      int seen_w = 0, seen_r = 0;
      for (int i = 0; i < 8; ++i) {
        const int gw = wpos(z, 8 * q + i) & 7;                             // stage-1 write
        const int l = 8 * q + i, gr = wpos(l >> 1, wslot_t(l & 1, z)) & 7;  // stage-2 read
        if ((seen_w >> gw) & 1 || (seen_r >> gr) & 1) return false;
        seen_w |= 1 << gw;
        seen_r |= 1 << gr;
      }
    }
  // the transpose is a bijection onto the 512 entries
  int hit[512] = {};
  for (int k0 = 0; k0 < 16; ++k0)
    for (int t = 0; t < 32; ++t) ++hit[wpos(k0, t)];
  for (int i = 0; i < 512; ++i)
    if (hit[i] != 1) return false;
  return true;
}

static int run_w(int trials, double* worst) {
  std::mt19937_64 rng(11);
  for (int trial = 0; trial < trials; ++trial) {
    std::vector<uint32_t> exact(1024, 0);
    c64 acc[32][16] = {};
    for (int r = 0; r < 6; ++r) {
      std::vector<int32_t> d(1024);
      std::vector<uint32_t> b(1024);
      for (auto& x : d) x = int32_t(rng() % 128) - 64;
      for (auto& x : b) x = uint32_t(rng());
      for (int i = 0; i < 1024; ++i)
        for (int j = 0; j < 1024; ++j) {
          uint32_t prod = uint32_t(d[i]) * b[j];
          if (i + j < 1024) exact[i + j] += prod;
          else exact[i + j - 1024] -= prod;
        }
      std::vector<double> dd(1024), bd(1024);
      for (int i = 0; i < 1024; ++i) {
        dd[i] = d[i];
        bd[i] = double(int32_t(b[i])) / 512.0;
      }
      c64 D[32][16], B[32][16];
      wforward(dd.data(), D, false);
      wforward(bd.data(), B, true);
      for (int l = 0; l < 32; ++l)
        for (int k = 0; k < 16; ++k) acc[l][k] = cadd(acc[l][k], cmul(D[l][k], B[l][k]));
    }
    std::vector<uint32_t> got(1024);
    winverse(acc, got.data(), worst);
    for (int i = 0; i < 1024; ++i)
      if (got[i] != exact[i]) {
        printf("FAIL (warp) trial %d coef %d got %u want %u\n", trial, i, got[i], exact[i]);
        return 1;
      }
  }
  return 0;
}

int main(int argc, char** argv) {
  int trials = argc > 1 ? atoi(argv[1]) : 20;
  make_twiddles(T1, T2);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < 64; ++t) {
    B1b[t] = T1[t][0];
    B1w[t] = {double(std::cos(-pi * t / 256.0L)), double(std::sin(-pi * t / 256.0L))};
    B2w[t] = {double(std::cos(-pi * (t >> 3) / 32.0L)), double(std::sin(-pi * (t >> 3) / 32.0L))};
  }
  if (!check_swizzle()) {
    printf("FAIL swizzle conflict\n");
    return 1;
  }
  if (!check_wswizzle()) {
    printf("FAIL warp transpose conflict\n");
    return 1;
  }
  double worst_tab = 0, worst_rec = 0, worst_w = 0;
  if (run(trials, false, &worst_tab) || run(trials, true, &worst_rec) || run_w(trials, &worst_w))
    return 1;
  printf("OK %d trials bit-exact (table twiddles: max distance to integer %.4g; "
         "generated twiddles: %.4g; warp FFT: %.4g)\n", trials, worst_tab, worst_rec, worst_w);
  return 0;
}
