// Runs the REFERENCE's own functional units and emulator (compiled from
// /root/reference/proj/core/src into oracle/_ref) on the B200 path through
// cryptovm::GpuBackend, with verify=true so every decryption is also checked
// against the shadow SimBackend.  Exit code 0 = all results correct.
#include <cstdio>
#include <filesystem>
#include <memory>
#include <random>

#include "cryptovm/alu.hpp"
#include "cryptovm/emulator.hpp"
#include "cryptovm/isa.hpp"
#include "cryptovm/keyservice.hpp"
#include "cryptovm/word.hpp"
#include "cryptovm/errors.hpp"
#include "cryptovm_ct_image.hpp"
#include "cryptovm_gpu_backend.hpp"

using namespace cryptovm;

int main() {
  cvm_keyset* ks = nullptr;
  cvm_ctx* ctx = nullptr;
  if (cvm_keyset_generate(5, &ks) || cvm_ctx_create(0, &ctx) || cvm_upload_keyset(ctx, ks)) {
    std::fprintf(stderr, "setup failed: %s\n", cvm_last_error());
    return 2;
  }
  int bad = 0;
  {
    GpuBackend bk(ctx, ks, /*verify=*/true);
    std::mt19937_64 rng(11);  // the seed of alu_add_test.cc's random adds
    // 1) alu::add, 16 bits, 8 independent adders recorded before one flush.
    std::vector<std::uint64_t> av, bv;
    std::vector<alu::AddResult> sums;
    for (int i = 0; i < 8; ++i) {
      av.push_back(rng() & 0xFFFF);
      bv.push_back(rng() & 0xFFFF);
      Word a = Word::encrypt(bk, av.back(), 16), b = Word::encrypt(bk, bv.back(), 16);
      sums.push_back(alu::add(bk, a, b));
    }
    for (int i = 0; i < 8; ++i) {
      const std::uint64_t got = decrypt_word(bk, sums[i].sum);
      const bool carry = bk.decrypt_bit(sums[i].carry_out);
      const std::uint64_t want = av[i] + bv[i];
      if (got != (want & 0xFFFF) || carry != ((want >> 16) & 1)) ++bad;
    }
    std::printf("add16 x8: %s\n", bad ? "FAIL" : "ok");
    // 2) alu::mul_unsigned and div_unsigned, 8 bits.
    for (int i = 0; i < 2; ++i) {
      const std::uint64_t x = rng() & 0xFF, y = (rng() & 0xFF) | 1;
      Word a = Word::encrypt(bk, x, 8), b = Word::encrypt(bk, y, 8);
      Word p = alu::mul_unsigned(bk, a, b);
      Word q = alu::div_unsigned(bk, a, b);
      const bool ok = decrypt_word(bk, p) == x * y && decrypt_word(bk, q) == x / y;
      bad += !ok;
      std::printf("mul8/div8 %llu,%llu: %s\n", (unsigned long long)x, (unsigned long long)y,
                  ok ? "ok" : "FAIL");
    }
    // 3) the emulator with a branchy program (emulator_test.cc LoopPrograms):
    //    branches resolve through LocalBranchOracle -> decrypt_bit (a flush).
    LocalBranchOracle oracle(bk);
    Machine m(bk, {.word_size = 16}, std::make_unique<BufferMemory>(16, std::vector<Word>{}),
              oracle);
    Program p = assemble(
        ".word_size 16\nMOV R0 0\nMOV R1 13\nMOV R2 11\nagain:\nADD R0 R0 R1\n"
        "SUBS R2 R2 1\nB_NE again\nHALT\n");
    m.run(p, 1000);
    const std::uint64_t r0 = decrypt_word(bk, m.reg(0));
    const bool ok = r0 == 143 && m.stats().branch_queries == 11;
    bad += !ok;
    std::printf("machine 13*11 loop: R0=%llu branches=%llu %s\n", (unsigned long long)r0,
                (unsigned long long)m.stats().branch_queries, ok ? "ok" : "FAIL");
    // 4) ciphertext-sized memory image + NZCV branch payload (SURVEY f-2):
    //    the emulator LOADs/STOREs 2,524-B LWE blobs through the image file,
    //    and a branch query carrying the four flag ciphertexts is resolved.
    {
      const std::string path =
          (std::filesystem::temp_directory_path() / "cvm_ct_image_demo.bin").string();
      encrypt_ct_file(bk, {5, 9, 1000, 0xFFFF}, 16, path);
      LocalBranchOracle oracle2(bk);
      auto mem = std::make_unique<CiphertextFileMemory>(bk, path);
      const std::size_t blob = mem->blob_bytes();
      Machine m2(bk, {.word_size = 16}, std::move(mem), oracle2);
      m2.run(assemble(".word_size 16\nLOAD R0 0\nLOAD R1 1\nADD R2 R0 R1\nSTORE R2 3\n"
                      "LOAD R3 2\nSUBS R4 R3 R0\nSTORE R4 0\nHALT\n"),
             100);
      const MemoryImage img = decrypt_ct_file(bk, path);
      bool ok = blob == CVM_LWE_WORDS * 4 && img.width == 16 &&
                img.values == std::vector<std::uint64_t>{995, 9, 1000, 14};
      BranchQuery q;
      q.cond = CondCode::Hi;  // unsigned higher: C set and Z clear (1000 > 5)
      q.nzcv_payload = serialize_flags(bk, m2.flags());
      q.target = 7;
      q.fallthrough = 3;
      const BranchReply r = resolve_branch_ct(q, bk, /*user_controlled=*/true);
      ok = ok && q.nzcv_payload.size() == 4 * blob && r.next_pc == 7u;
      bool rejected = false;
      try {
        resolve_branch(q, bk);  // the reference's 1-byte-per-flag check
      } catch (const ProtocolError&) {
        rejected = true;
      }
      ok = ok && rejected;
      std::filesystem::remove(path);
      bad += !ok;
      std::printf("ciphertext image + branch payload (%zu-B blobs): %s\n", blob,
                  ok ? "ok" : "FAIL");
    }
    const cvm_backend_stats st = bk.stats();
    std::printf("stats: nodes=%llu bootstrapped=%llu levels=%llu flushes=%llu mismatches=%llu\n",
                (unsigned long long)st.nodes, (unsigned long long)st.bootstrapped,
                (unsigned long long)st.levels_run, (unsigned long long)st.flushes,
                (unsigned long long)bk.mismatches());
  }
  cvm_ctx_destroy(ctx);
  cvm_keyset_destroy(ks);
  std::printf("%s\n", bad ? "ADAPTER FAIL" : "ADAPTER OK");
  return bad ? 1 : 0;
}
