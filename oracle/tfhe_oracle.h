/*
 * CPU restatement of TFHE gate bootstrapping -- the PARITY ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the CPU timing baseline -- never as the product path.
 *
 * What it restates.  The reference (/root/reference/proj) ships no TFHE code:
 * its only backend, SimBackend, evaluates cleartext booleans
 * (proj/core/src/sim_backend.cpp:25-51).  The arithmetic CryptoEmu runs under
 * every gate lives in the third-party TFHE library (cited as `tfhe2020`,
 * PAPER.md:43,67-112; called as bootsAND/bootsXOR/bootsMUX/... PAPER.md:215,
 * 296-303,474-491), which is neither vendored nor version-pinned (the
 * bibliography is not shipped).  This file restates the PUBLISHED TFHE gate
 * bootstrapping algorithm (Chillotti-Gama-Georgieva-Izabachene, "TFHE: fast
 * fully homomorphic encryption over the torus", J. Cryptology 2020, and the
 * library's default 110-bit gate-bootstrapping parameter set):
 *     n=630, N=1024, k=1, bk_l=3, bk_Bgbit=7, ks_t=8, ks_basebit=2, torus32,
 *     ks_stdev=2^-15 (fresh LWE and KS key), bk_stdev=2^-25 (bootstrapping key).
 *
 * Semantics it follows from the reference:
 *   gate set / asymmetric gates   proj/core/include/cryptovm/gates.hpp:31-46
 *   truth tables, MUX order       proj/core/src/sim_backend.cpp:25-51,98-106
 *   bootstrap counts              gates.cpp:35-50 (MUX = 2 bootstraps)
 *
 * Parity status.  Decrypted bits / integers: PINNED against the reference's own
 * SimBackend run here (tests/golden/, produced by oracle/ref_golden.cpp).
 * Raw torus32 coefficients: "parity unpinned" against the TFHE library itself
 * (absent from /root/reference and this container); pinned instead by the
 * exact-integer known-answer tests in tests/test_oracle.py (NTT product ==
 * schoolbook product, bootstrapping noise/decryption over many seeds).
 *
 * The negacyclic products are EXACT: an NTT over the prime 2^64-2^32+1 (|sum| <
 * 2^50 so the centred lift is exact), or O(N^2) schoolbook for the KATs.
 * A second, double-precision FFT mode (the TFHE library's own method) serves as
 * the CPU speed baseline.
 */
#ifndef TFHE_ORACLE_H_
#define TFHE_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_N_LWE 630        /* n   */
#define OR_N_POLY 1024      /* N   */
#define OR_L 3              /* bk_l */
#define OR_BGBIT 7          /* bk_Bgbit */
#define OR_KS_T 8           /* ks_t */
#define OR_KS_BASEBIT 2     /* ks_basebit */
#define OR_LWE_WORDS 631    /* a[0..629], b */
#define OR_XLWE_WORDS 1025  /* extracted LWE: a[0..1023], b */
#define OR_BK_WORDS (630 * 6 * 2 * 1024)
#define OR_KSK_WORDS (1024 * 8 * 4 * 631)

/* Gate kind codes = cryptovm::GateKind enumerators (gates.hpp:31-46). */
enum {
  OR_CONSTANT = 0, OR_NOT, OR_COPY, OR_NAND, OR_AND, OR_OR, OR_XOR, OR_XNOR,
  OR_NOR, OR_ANDNY, OR_ANDYN, OR_ORNY, OR_ORYN, OR_MUX
};

enum { OR_MODE_NTT = 0, OR_MODE_FFT = 1, OR_MODE_SCHOOLBOOK = 2 };

/* Deterministic key generation from one seed (spec in DESIGN.md section 3).
 * bk[i][row][poly][coef] (row = part*3 + level), ksk[i][j][v][631]. */
void oracle_keygen(uint64_t seed, int32_t* lwe_key, int32_t* tlwe_key,
                   uint32_t* bk, uint32_t* ksk);
void oracle_encrypt(uint64_t seed, const int32_t* lwe_key, int count,
                    const uint8_t* bits, uint32_t* out);
void oracle_decrypt(const int32_t* lwe_key, int count, const uint32_t* in,
                    uint8_t* bits, int32_t* phases);
void oracle_decrypt_x(const int32_t* tlwe_key, int count, const uint32_t* in,
                      uint8_t* bits, int32_t* phases);

typedef struct oracle_keys oracle_keys;
oracle_keys* oracle_keys_load(const uint32_t* bk, const uint32_t* ksk, int mode);
void oracle_keys_free(oracle_keys* k);

/* Bootstrapped gates, `count` independent ones, on `threads` host threads.
 * kinds: OR_NAND..OR_MUX.  in_c only read for MUX (sel=a, on_true=b,
 * on_false=c).  Ciphertexts are 631 u32 each. */
int oracle_gates(const oracle_keys* k, int count, const uint8_t* kinds,
                 const uint32_t* in_a, const uint32_t* in_b,
                 const uint32_t* in_c, uint32_t* out, int threads);

/* Pieces, for known-answer tests. */
void oracle_blind_rotate_extract(const oracle_keys* k, const uint32_t* lwe,
                                 uint32_t mu, uint32_t* out_xlwe);
void oracle_key_switch(const oracle_keys* k, const uint32_t* xlwe,
                       uint32_t* out_lwe);
void oracle_negacyclic_mul(int mode, const int32_t* digits,
                           const uint32_t* poly, uint32_t* out);
uint32_t oracle_modswitch(uint32_t phase);

#ifdef __cplusplus
}
#endif
#endif
