// Backend selection for the reference CLI's `run` (SURVEY f-4): `--backend
// sim` keeps the reference's SimBackend, `--backend gpu` runs the same
// Machine on the B200 through cryptovm::GpuBackend.  The session owns the
// GPU stack (key owner's keyset, device context with the cloud keys
// uploaded) and exposes the recorded GateDag either way (SimBackend's, or the
// shim's shadow), so --trace and the schedule report keep working.
// cli_backend_gpu.patch wires it into tools/cryptovm.cpp.
#ifndef CRYPTOVM_BACKEND_SELECT_HPP_
#define CRYPTOVM_BACKEND_SELECT_HPP_

#include <cstdint>
#include <memory>
#include <string>

#include "cryptovm/dag.hpp"
#include "cryptovm/gates.hpp"

namespace cryptovm {

class BackendSession {
 public:
  virtual ~BackendSession() = default;
  // kind: "sim" or "gpu" (InputError otherwise; Error when no sm_100a GPU).
  static std::unique_ptr<BackendSession> make(const std::string& kind, const CostTable& costs,
                                              std::uint64_t key_seed = 1, int device = 0);
  virtual Backend& backend() = 0;
  virtual const GateDag& dag() const = 0;
  // Whether bits are real ciphertexts (export_bit blobs are not 1 byte), so
  // the 1-byte-per-bit FileMemory image cannot hold them.
  virtual bool ciphertexts() const = 0;
};

}  // namespace cryptovm

#endif  // CRYPTOVM_BACKEND_SELECT_HPP_
