// Key-owner operations on the host: key generation, bit encryption and
// decryption.  These stay on the CPU exactly as in the reference, where they
// are Backend::encrypt_bit / decrypt_bit (gates.hpp:120-121) and the Word
// helpers (word.cpp:42-86); only cloud keys (BK, KSK) go to the device.
//
// Deterministic spec, shared with the CPU oracle so a
// seed names one key set: splitmix64-seeded xoshiro256** per stream, Box-Muller
// Gaussians rounded to torus32.  Compiled with -ffp-contract=off.
#include <cmath>
#include <cstring>
#include <vector>

#include "cvm_internal.hpp"

namespace cvm {

namespace {

class Xoshiro {
 public:
  Xoshiro(uint64_t seed, uint64_t stream) {
    uint64_t x = seed ^ (stream * 0xD1B54A32D192ED03ull);
    for (uint64_t& w : s_) w = mix(x);
  }
  uint64_t next() {
    const uint64_t r = rotl(s_[1] * 5, 7) * 9;
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return r;
  }
  uint32_t u32() { return uint32_t(next() >> 32); }
  int32_t bit() { return int32_t(next() >> 63); }
  // Gaussian torus32 sample of standard deviation `sigma` (torus fraction).
  uint32_t gauss(double sigma) {
    const double u1 = double((next() >> 11) + 1) * 0x1.0p-53;
    const double u2 = double(next() >> 11) * 0x1.0p-53;
    const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    const double x = g * sigma * 4294967296.0;
    return uint32_t(int32_t(int64_t(std::floor(x + 0.5))));
  }

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  static uint64_t mix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  uint64_t s_[4];
};

constexpr uint64_t kStreamKeys = 1, kStreamEnc = 2;

// b += a * z  (mod X^N + 1, z binary)
void add_mul_binary(const uint32_t* a, const int32_t* z, uint32_t* b) {
  for (int k = 0; k < kPolyN; ++k) {
    if (!z[k]) continue;
    const int n = kPolyN - k;
    for (int j = 0; j < n; ++j) b[k + j] += a[j];
    for (int j = n; j < kPolyN; ++j) b[j - n] -= a[j];
  }
}

}  // namespace

KeySet::KeySet(uint64_t seed)
    : lwe_key(kN), tlwe_key(kPolyN), bk(kBkWords), ksk(kKskWords) {
  Xoshiro rng(seed, kStreamKeys);
  for (auto& s : lwe_key) s = rng.bit();
  for (auto& z : tlwe_key) z = rng.bit();
  // BK_i: TRGSW encryption of s_i; row = part*l + p, part 0 -> a, 1 -> b.
  std::vector<uint32_t> e(kPolyN);
  for (int i = 0; i < kN; ++i) {
    for (int row = 0; row < kRows; ++row) {
      uint32_t* a = &bk[(size_t(i) * kRows + row) * 2 * kPolyN];
      uint32_t* b = a + kPolyN;
      for (int j = 0; j < kPolyN; ++j) a[j] = rng.u32();
      for (int j = 0; j < kPolyN; ++j) e[j] = rng.gauss(kBkStdev);
      std::memcpy(b, e.data(), kPolyN * sizeof(uint32_t));
      add_mul_binary(a, tlwe_key.data(), b);
      if (lwe_key[i]) {
        const uint32_t h = 1u << (32 - (row % kL + 1) * kBgBit);
        (row / kL == 0 ? a : b)[0] += h;
      }
    }
  }
  // KSK[i][j][v]: LWE encryption of z_i * v / 4^(j+1); v = 0 left zero.
  for (int i = 0; i < kPolyN; ++i)
    for (int j = 0; j < kKsT; ++j)
      for (int v = 0; v < kKsBase; ++v) {
        uint32_t* row = &ksk[((size_t(i) * kKsT + j) * kKsBase + v) * kLweWords];
        if (v == 0) {
          std::memset(row, 0, kLweWords * sizeof(uint32_t));
          continue;
        }
        uint32_t dot = 0;
        for (int k = 0; k < kN; ++k) {
          row[k] = rng.u32();
          dot += row[k] * uint32_t(lwe_key[k]);
        }
        const uint32_t msg =
            uint32_t(tlwe_key[i]) * uint32_t(v) * (1u << (32 - (j + 1) * kKsBaseBit));
        row[kN] = dot + rng.gauss(kKsStdev) + msg;
      }
}

void KeySet::encrypt(uint64_t seed, size_t count, const uint8_t* bits,
                     uint32_t* out) const {
  Xoshiro rng(seed, kStreamEnc);
  for (size_t g = 0; g < count; ++g) {
    uint32_t* c = out + g * kLweWords;
    uint32_t dot = 0;
    for (int k = 0; k < kN; ++k) {
      c[k] = rng.u32();
      dot += c[k] * uint32_t(lwe_key[k]);
    }
    c[kN] = dot + rng.gauss(kKsStdev) + (bits[g] ? kMu : 0u - kMu);
  }
}

int32_t KeySet::phase(const uint32_t* c) const {
  uint32_t dot = 0;
  for (int k = 0; k < kN; ++k) dot += c[k] * uint32_t(lwe_key[k]);
  return int32_t(c[kN] - dot);
}

}  // namespace cvm
