// cryptovm::GpuBackend -- the shim a maintainer adds to the reference tree
// (/root/reference/proj/core) to run CryptoEmu's unchanged functional units
// and emulator on the B200 path through include/cvm_gpu.h.
//
// It implements the abstract cryptovm::Backend (gates.hpp:109-132).  BitHandle
// can only be minted by SimBackend (gates.hpp:88-100, `friend class
// SimBackend`), so the shim composes a SimBackend that mints the handles and
// records the DAG; every gate is mirrored into a cvm_backend whose node ids
// follow the same dense numbering.  decrypt_bit returns the GPU ciphertext's
// decryption, never the shadow's clear bit; with verify=true every decryption
// is also compared against the shadow (a free per-gate oracle).
#ifndef CRYPTOVM_GPU_BACKEND_HPP_
#define CRYPTOVM_GPU_BACKEND_HPP_

#include <cstdint>
#include <mutex>
#include <vector>

#include "cryptovm/gates.hpp"
#include "cryptovm/sim_backend.hpp"
#include "cryptovm/word.hpp"
#include "cvm_gpu.h"

namespace cryptovm {

class GpuBackend final : public Backend {
 public:
  // `ctx` must already hold the cloud keys (cvm_upload_keyset); `owner` is the
  // key owner's keyset used by encrypt_bit / decrypt_bit.
  //
  // Evaluation is demand-driven: a decrypt_bit / export_bit evaluates only the
  // cone of influence of that bit, so gates whose results are never read (the
  // high half of the emulator's MUL product, overwritten registers, replaced
  // flags) never run.  The reference decrypts words bit by bit
  // (word.cpp:70-77); a caller that knows which bits it will read next calls
  // evaluate() on all of them first -- one flush, one batch of launches --
  // and the decryptions after it only download.  flush_all = true restores
  // "evaluate everything pending at the first decrypt".
  GpuBackend(cvm_ctx* ctx, const cvm_keyset* owner, bool verify = false,
             std::uint64_t enc_seed = 1, bool flush_all = false);
  ~GpuBackend() override;
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;

  BitHandle constant(bool value) override;
  BitHandle unary_gate(GateKind kind, BitHandle a) override;
  BitHandle binary_gate(GateKind kind, BitHandle a, BitHandle b) override;
  BitHandle mux_gate(BitHandle sel, BitHandle on_true, BitHandle on_false) override;

  BitHandle encrypt_bit(bool value) override;
  bool decrypt_bit(BitHandle bit) override;
  std::vector<std::uint8_t> export_bit(BitHandle bit) override;
  BitHandle import_bit(const std::vector<std::uint8_t>& blob) override;

  void push_region(std::string_view name) override;
  void pop_region() override;
  void fence() override;

  // Evaluate everything recorded so far (one batched launch pair per level).
  void flush();
  // Evaluate the cone of influence of `bits` now (one flush).
  void evaluate(const std::vector<BitHandle>& bits);
  void evaluate(const Word& word) { evaluate(word.bits()); }
  const GateDag& dag() const { return shadow_.dag(); }
  cvm_backend_stats stats() const;
  std::uint64_t mismatches() const { return mismatches_; }

 private:
  cvm_handle mapped(BitHandle h, const char* what) const;
  BitHandle bind(BitHandle shadow, cvm_handle gpu);

  SimBackend shadow_;
  cvm_backend* gpu_ = nullptr;
  const cvm_keyset* owner_;
  bool verify_;
  std::vector<cvm_handle> map_;  // shadow node id -> cvm handle
  std::uint64_t mismatches_ = 0;
  mutable std::mutex mu_;
};

}  // namespace cryptovm

#endif  // CRYPTOVM_GPU_BACKEND_HPP_
