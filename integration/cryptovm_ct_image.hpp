// Ciphertext-sized memory images and branch payloads.
//
// The reference's wire and file formats assume a backend whose export_bit
// blob is ONE byte (SimBackend, sim_backend.cpp:118-128):
//   * the CEMU memory image packs each word LSB-first into ceil(N/8) bytes
//     and FileMemory::load/store round-trips bits through 1-byte blobs
//     (keyservice.cpp:440-484, esp. :456, :474-476);
//   * resolve_branch requires a 4-byte NZCV payload (keyservice.cpp:123-144),
//     while serialize_flags (:113-121) already concatenates whatever
//     export_bit returns.
// With real ciphertexts every bit is an LWE sample (631 x u32 = 2,524 B), so
// both need a ciphertext-sized variant.  These are the additions a maintainer
// would make next to keyservice.cpp; they use only the public Backend API, so
// they work with cryptovm::GpuBackend (and with SimBackend, blob size 1).
//
// Image layout (version 2, little endian):
//   "CEMU" | u8 version = 2 | u16 width | u32 count | u32 blob_bytes |
//   count * width blobs, word-major, bit 0 (LSB) first.
// Version 1 files (the reference's plaintext layout) are rejected with the
// same IoError the reference raises for an unknown version.
#ifndef CRYPTOVM_CT_IMAGE_HPP_
#define CRYPTOVM_CT_IMAGE_HPP_

#include <cstdint>
#include <string>
#include <vector>

#include "cryptovm/emulator.hpp"
#include "cryptovm/gates.hpp"
#include "cryptovm/keyservice.hpp"

namespace cryptovm {

constexpr std::uint8_t kCtImageVersion = 2;
constexpr std::size_t kCtHeaderSize = 4 + 1 + 2 + 4 + 4;

// Key owner: encrypt `values` (width bits each) into a ciphertext image.
void encrypt_ct_file(Backend& key, const std::vector<std::uint64_t>& values, unsigned width,
                     const std::string& path);
// Key owner: decrypt a ciphertext image.
MemoryImage decrypt_ct_file(Backend& key, const std::string& path);

// File-backed data memory over a ciphertext image: every load imports the
// word's blobs, every store exports the stored bits (an evaluation point).
class CiphertextFileMemory final : public DataMemory {
 public:
  CiphertextFileMemory(Backend& backend, const std::string& path);

  Word load(std::size_t address) override;
  void store(std::size_t address, const Word& word) override;
  std::size_t size() const override { return count_; }
  unsigned word_size() const override { return width_; }
  std::size_t blob_bytes() const { return blob_; }

 private:
  std::streamoff offset_of(std::size_t address) const;

  Backend& backend_;
  std::string path_;
  unsigned width_ = 0;
  std::size_t count_ = 0;
  std::size_t blob_ = 0;
};

// resolve_branch for ciphertext payloads: the NZCV payload is four equal
// export_bit blobs (what serialize_flags produces for any backend).
BranchReply resolve_branch_ct(const BranchQuery& query, Backend& key,
                              bool user_controlled = false);

}  // namespace cryptovm

#endif  // CRYPTOVM_CT_IMAGE_HPP_
