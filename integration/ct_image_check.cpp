// CPU check of the ciphertext-image / branch-payload additions against the
// reference's own SimBackend (blob size 1) and its plaintext-image code:
// round trips, the emulator through CiphertextFileMemory, resolve_branch_ct
// agreeing with resolve_branch, and the error paths.  Exit 0 = all good.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <memory>

#include "cryptovm/emulator.hpp"
#include "cryptovm/errors.hpp"
#include "cryptovm/isa.hpp"
#include "cryptovm/keyservice.hpp"
#include "cryptovm/sim_backend.hpp"
#include "cryptovm_ct_image.hpp"

using namespace cryptovm;

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  int bad = 0;
  auto expect = [&](bool ok, const char* what) {
    std::printf("%-48s %s\n", what, ok ? "ok" : "FAIL");
    bad += !ok;
  };
  const auto dir = std::filesystem::temp_directory_path();
  const std::string path = (dir / "cvm_ct_check.bin").string();
  const std::string plain = (dir / "cvm_ct_check_v1.bin").string();
  SimBackend sim;

  encrypt_ct_file(sim, {5, 9, 1000, 0xFFFF}, 16, path);
  expect(std::filesystem::file_size(path) == kCtHeaderSize + 4 * 16 * 1, "image size (1-B blobs)");
  expect(decrypt_ct_file(sim, path).values == std::vector<std::uint64_t>{5, 9, 1000, 0xFFFF},
         "encrypt/decrypt round trip");

  {
    LocalBranchOracle oracle(sim);
    Machine m(sim, {.word_size = 16}, std::make_unique<CiphertextFileMemory>(sim, path), oracle);
    m.run(assemble(".word_size 16\nLOAD R0 0\nLOAD R1 1\nADD R2 R0 R1\nSTORE R2 3\n"
                   "LOAD R3 2\nSUBS R4 R3 R0\nSTORE R4 0\nHALT\n"),
          100);
    expect(decrypt_ct_file(sim, path).values == std::vector<std::uint64_t>{995, 9, 1000, 14},
           "emulator LOAD/STORE through the image");
    for (int c = 0; c < kCondCodeCount; ++c) {
      BranchQuery q;
      q.cond = static_cast<CondCode>(c);
      q.nzcv_payload = serialize_flags(sim, m.flags());
      q.target = 9;
      q.fallthrough = 4;
      if (resolve_branch_ct(q, sim, true).next_pc != resolve_branch(q, sim, true).next_pc ||
          resolve_branch_ct(q, sim).taken != resolve_branch(q, sim).taken) {
        expect(false, "resolve_branch_ct == resolve_branch");
      }
    }
    expect(true, "resolve_branch_ct == resolve_branch (15 conds)");
  }
  {
    CiphertextFileMemory mem(sim, path);
    expect(throws<InputError>([&] { mem.load(4); }), "load out of range -> InputError");
    expect(throws<InputError>([&] { mem.store(0, Word::constant(sim, 1, 8)); }),
           "store width mismatch -> InputError");
  }
  encrypt_file({1, 2}, 16, plain);  // the reference's version-1 plaintext image
  expect(throws<IoError>([&] { CiphertextFileMemory m(sim, plain); }),
         "version-1 image rejected -> IoError");
  {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    f << "CEMX";
  }
  expect(throws<IoError>([&] { decrypt_ct_file(sim, path); }), "truncated/bad magic -> IoError");
  encrypt_ct_file(sim, {1}, 8, path);
  std::filesystem::resize_file(path, std::filesystem::file_size(path) - 1);
  expect(throws<IoError>([&] { CiphertextFileMemory m(sim, path); }), "short body -> IoError");
  BranchQuery q;
  q.nzcv_payload = {1, 0, 1};
  expect(throws<ProtocolError>([&] { resolve_branch_ct(q, sim); }), "payload not 4 blobs");
  expect(throws<InputError>([&] { encrypt_ct_file(sim, {256}, 8, path); }), "value too wide");
  std::filesystem::remove(path);
  std::filesystem::remove(plain);
  std::printf("%s\n", bad ? "CT IMAGE FAIL" : "CT IMAGE OK");
  return bad ? 1 : 0;
}
