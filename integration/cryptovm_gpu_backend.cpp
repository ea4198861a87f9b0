// See cryptovm_gpu_backend.hpp.  Status codes of the C ABI become the
// reference's exceptions: CVM_E_INPUT -> InputError, anything else -> Error
// (errors.hpp:24-58).
#include "cryptovm_gpu_backend.hpp"

#include <string>

#include "cryptovm/errors.hpp"

namespace cryptovm {

namespace {
void check(int rc, const char* what) {
  if (rc == CVM_OK) return;
  std::string msg = std::string(what) + ": " + cvm_last_error();
  if (rc == CVM_E_INPUT) throw InputError(msg);
  throw Error(msg);
}
}  // namespace

GpuBackend::GpuBackend(cvm_ctx* ctx, const cvm_keyset* owner, bool verify,
                       std::uint64_t enc_seed, bool flush_all)
    : owner_(owner), verify_(verify) {
  check(cvm_backend_create(ctx, owner, enc_seed, &gpu_), "cvm_backend_create");
  check(cvm_backend_set_flush_policy(gpu_, flush_all ? CVM_FLUSH_ALL : CVM_FLUSH_CONE),
        "set_flush_policy");
  map_.push_back(0);  // node id 0 is the invalid handle
}

GpuBackend::~GpuBackend() { cvm_backend_destroy(gpu_); }

cvm_handle GpuBackend::mapped(BitHandle h, const char* what) const {
  if (!h.valid() || h.node() >= map_.size())
    throw InputError(std::string("invalid bit handle passed to ") + what);
  return map_[h.node()];
}

BitHandle GpuBackend::bind(BitHandle shadow, cvm_handle gpu) {
  if (map_.size() <= shadow.node()) map_.resize(shadow.node() + 1, 0);
  map_[shadow.node()] = gpu;
  return shadow;
}

BitHandle GpuBackend::constant(bool value) {
  std::lock_guard<std::mutex> lock(mu_);
  cvm_handle g;
  check(cvm_backend_constant(gpu_, value ? 1 : 0, &g), "constant");
  return bind(shadow_.constant(value), g);
}

BitHandle GpuBackend::unary_gate(GateKind kind, BitHandle a) {
  std::lock_guard<std::mutex> lock(mu_);
  const cvm_handle ga = mapped(a, "unary_gate");
  BitHandle s = shadow_.unary_gate(kind, a);  // validates the kind first
  cvm_handle g;
  check(cvm_backend_unary_gate(gpu_, static_cast<uint32_t>(kind), ga, &g), "unary_gate");
  return bind(s, g);
}

BitHandle GpuBackend::binary_gate(GateKind kind, BitHandle a, BitHandle b) {
  std::lock_guard<std::mutex> lock(mu_);
  const cvm_handle ga = mapped(a, "binary_gate"), gb = mapped(b, "binary_gate");
  BitHandle s = shadow_.binary_gate(kind, a, b);
  cvm_handle g;
  check(cvm_backend_binary_gate(gpu_, static_cast<uint32_t>(kind), ga, gb, &g),
        "binary_gate");
  return bind(s, g);
}

BitHandle GpuBackend::mux_gate(BitHandle sel, BitHandle on_true, BitHandle on_false) {
  std::lock_guard<std::mutex> lock(mu_);
  const cvm_handle gs = mapped(sel, "mux_gate"), gt = mapped(on_true, "mux_gate"),
                   gf = mapped(on_false, "mux_gate");
  BitHandle s = shadow_.mux_gate(sel, on_true, on_false);
  cvm_handle g;
  check(cvm_backend_mux_gate(gpu_, gs, gt, gf, &g), "mux_gate");
  return bind(s, g);
}

BitHandle GpuBackend::encrypt_bit(bool value) {
  std::lock_guard<std::mutex> lock(mu_);
  cvm_handle g;
  check(cvm_backend_encrypt_bit(gpu_, value ? 1 : 0, &g), "encrypt_bit");
  return bind(shadow_.encrypt_bit(value), g);
}

bool GpuBackend::decrypt_bit(BitHandle bit) {
  std::lock_guard<std::mutex> lock(mu_);
  const cvm_handle g = mapped(bit, "decrypt_bit");
  int v = 0;
  check(cvm_backend_decrypt_bit(gpu_, g, &v), "decrypt_bit");  // flushes
  const bool shadow = shadow_.decrypt_bit(bit);                // keeps decrypt_count
  if (verify_ && shadow != (v != 0)) {
    ++mismatches_;
    throw Error("GPU decryption differs from the shadow SimBackend at node " +
                std::to_string(bit.node()));
  }
  return v != 0;
}

std::vector<std::uint8_t> GpuBackend::export_bit(BitHandle bit) {
  std::lock_guard<std::mutex> lock(mu_);
  std::vector<std::uint8_t> blob(CVM_LWE_WORDS * 4);
  check(cvm_backend_export_bit(gpu_, mapped(bit, "export_bit"), blob.data(), blob.size()),
        "export_bit");
  return blob;
}

BitHandle GpuBackend::import_bit(const std::vector<std::uint8_t>& blob) {
  std::lock_guard<std::mutex> lock(mu_);
  cvm_handle g;
  check(cvm_backend_import_bit(gpu_, blob.data(), blob.size(), &g), "import_bit");
  // The shadow records an input node.  Only in verify mode (a test harness
  // holding the owner key) does it learn the clear bit, so later decryptions
  // of gates over imported bits can still be checked against it.
  std::uint8_t clear = 0;
  if (verify_) {
    check(cvm_decrypt_bits(owner_, 1, reinterpret_cast<const uint32_t*>(blob.data()), &clear,
                           nullptr),
          "import_bit (verify)");
  }
  return bind(shadow_.import_bit({clear}), g);
}

void GpuBackend::push_region(std::string_view name) {
  std::lock_guard<std::mutex> lock(mu_);
  shadow_.push_region(name);
  check(cvm_backend_push_region(gpu_, std::string(name).c_str()), "push_region");
}

void GpuBackend::pop_region() {
  std::lock_guard<std::mutex> lock(mu_);
  shadow_.pop_region();
  check(cvm_backend_pop_region(gpu_), "pop_region");
}

void GpuBackend::fence() {
  std::lock_guard<std::mutex> lock(mu_);
  shadow_.fence();
  check(cvm_backend_fence(gpu_), "fence");
}

void GpuBackend::flush() {
  std::lock_guard<std::mutex> lock(mu_);
  check(cvm_backend_flush(gpu_), "flush");
}

void GpuBackend::evaluate(const std::vector<BitHandle>& bits) {
  std::lock_guard<std::mutex> lock(mu_);
  std::vector<cvm_handle> hs;
  hs.reserve(bits.size());
  for (const BitHandle& b : bits) hs.push_back(mapped(b, "evaluate"));
  check(cvm_backend_evaluate(gpu_, hs.size(), hs.data()), "evaluate");
}

cvm_backend_stats GpuBackend::stats() const {
  cvm_backend_stats s{};
  check(cvm_backend_stats_get(gpu_, &s), "stats");
  return s;
}

}  // namespace cryptovm
