// TFHE gate-bootstrapping parameter set and device data layout.
//
// The parameter set is BASELINE.json configs[0]: the TFHE library's default
// 110-bit gate-bootstrapping set (n=630, N=1024, k=1, bk_l=3, bk_Bgbit=7,
// ks_t=8, ks_basebit=2, torus32).  See DESIGN.md section 3 for the algorithm
// and oracle/tfhe_oracle.h for its provenance.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CVM_HD __host__ __device__ __forceinline__
#else
#define CVM_HD inline
#endif

namespace cvm {

constexpr int kN = 630;            // LWE dimension n
constexpr int kPolyN = 1024;       // ring degree N (X^N + 1)
constexpr int kFftM = kPolyN / 2;  // folded complex length
constexpr int kL = 3;              // gadget levels
constexpr int kBgBit = 7;          // log2 Bg
constexpr int kRows = 2 * kL;      // TRGSW rows (k+1)*l
constexpr int kKsT = 8;            // key-switch digits
constexpr int kKsBaseBit = 2;      // key-switch base 4
constexpr int kKsBase = 1 << kKsBaseBit;

constexpr int kLweWords = kN + 1;        // a[0..629], b
constexpr int kLweStride = 632;          // padded slot stride (16-B aligned)
constexpr int kXlweWords = kPolyN + 1;   // extracted sample a[0..1023], b
constexpr int kXlweStride = 1028;        // padded stride (16-B aligned)
constexpr int kKskRowStride = 632;       // KSK row (631 used + 1 zero pad)

constexpr uint32_t kMu = 1u << 29;       // 1/8 on the torus
constexpr double kBkStdev = 0x1.0p-25;
constexpr double kKsStdev = 0x1.0p-15;

// Sizes of the host key arrays (time domain) exchanged at the C ABI.
constexpr size_t kBkWords = size_t(kN) * kRows * 2 * kPolyN;            // u32
constexpr size_t kKskWords = size_t(kPolyN) * kKsT * kKsBase * kLweWords;  // u32

// Device bootstrapping key in FFT domain: per CMux step i, per TRGSW row,
// per k2 (0..7), per output poly o (0..1), per thread t (0..63): one complex
// double = the folded-FFT bin t + 64*k2 of BK[i][row][o], pre-scaled by 1/M
// (thread-contiguous, so 16-byte loads from the shared ring are conflict-free).
constexpr size_t kBkfComplexPerStep = size_t(kRows) * 8 * 64 * 2;  // 6144
constexpr size_t kBkfBytes = size_t(kN) * kBkfComplexPerStep * 16;  // 61,931,520

// mod-switch a torus32 phase to Z_{2N}: round(phase * 2N / 2^32) mod 2N.
CVM_HD uint32_t modswitch_2n(uint32_t phase) {
  return ((phase + (1u << 20)) >> 21) & (2 * kPolyN - 1);
}

// Gate input combination (const + ca*a + cb*b) of each bootstrapped gate,
// indexed by cryptovm::GateKind (gates.hpp:31-46); kinds 0..2 and 13 unused.
struct GateCombo {
  uint32_t c;
  int32_t ca, cb;
};

}  // namespace cvm
