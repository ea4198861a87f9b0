// See cryptovm_backend_select.hpp.
#include "cryptovm_backend_select.hpp"

#include "cryptovm/errors.hpp"
#include "cryptovm/sim_backend.hpp"
#include "cryptovm_gpu_backend.hpp"

namespace cryptovm {

namespace {

class SimSession final : public BackendSession {
 public:
  explicit SimSession(const CostTable& costs) : sim_(costs) {}
  Backend& backend() override { return sim_; }
  const GateDag& dag() const override { return sim_.dag(); }
  bool ciphertexts() const override { return false; }

 private:
  SimBackend sim_;
};

class GpuSession final : public BackendSession {
 public:
  GpuSession(std::uint64_t key_seed, int device) {
    auto fail = [](const char* what) {
      throw Error(std::string(what) + ": " + cvm_last_error());
    };
    if (cvm_keyset_generate(key_seed, &ks_) != CVM_OK) fail("cvm_keyset_generate");
    if (cvm_ctx_create(device, &ctx_) != CVM_OK) {
      cvm_keyset_destroy(ks_);
      fail("cvm_ctx_create");
    }
    if (cvm_upload_keyset(ctx_, ks_) != CVM_OK) {
      cvm_ctx_destroy(ctx_);
      cvm_keyset_destroy(ks_);
      fail("cvm_upload_keyset");
    }
    gpu_ = std::make_unique<GpuBackend>(ctx_, ks_);
  }
  ~GpuSession() override {
    gpu_.reset();
    cvm_ctx_destroy(ctx_);
    cvm_keyset_destroy(ks_);
  }
  Backend& backend() override { return *gpu_; }
  const GateDag& dag() const override { return gpu_->dag(); }
  bool ciphertexts() const override { return true; }

 private:
  cvm_keyset* ks_ = nullptr;
  cvm_ctx* ctx_ = nullptr;
  std::unique_ptr<GpuBackend> gpu_;
};

}  // namespace

std::unique_ptr<BackendSession> BackendSession::make(const std::string& kind,
                                                     const CostTable& costs,
                                                     std::uint64_t key_seed, int device) {
  if (kind == "sim") return std::make_unique<SimSession>(costs);
  if (kind == "gpu") return std::make_unique<GpuSession>(key_seed, device);
  throw InputError("--backend must be sim or gpu");
}

}  // namespace cryptovm
