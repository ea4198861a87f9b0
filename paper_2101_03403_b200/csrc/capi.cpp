// extern "C" wrappers (include/cvm_gpu.h).  Exceptions become status codes
// and a thread-local message, mirroring the reference's InputError / Error
// split (errors.hpp:24-58).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "cvm_internal.hpp"

using namespace cvm;

struct cvm_keyset {
  KeySet ks;
  explicit cvm_keyset(uint64_t seed) : ks(seed) {}
};
struct cvm_ctx {
  Context* ctx;
  uint64_t enc_seed = 1;
};
struct cvm_backend {
  std::unique_ptr<Backend> impl;
  GpuBackend* gpu = nullptr;      // set for the device backend
  ClearBackend* clear = nullptr;  // set for the cleartext recorder
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return CVM_OK;
  } catch (const InputError& e) {
    g_err = e.what();
    return CVM_E_INPUT;
  } catch (const StateError& e) {
    g_err = e.what();
    return CVM_E_STATE;
  } catch (const DeviceError& e) {
    g_err = e.what();
    return CVM_E_DEVICE;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return CVM_E_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CVM_E_DEVICE;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw InputError(std::string("null ") + what);
}

GateKind kind_of(uint32_t k) {
  if (k > uint32_t(GateKind::Mux)) throw InputError("unknown gate kind " + std::to_string(k));
  return GateKind(k);
}


}  // namespace

extern "C" {

const char* cvm_last_error(void) { return g_err.c_str(); }
const char* cvm_version(void) { return "cvm_b200 0.1 (sm_100a, FP64-FFT blind rotation)"; }

// ------------------------------------------------------------- key owner --
int cvm_keyset_generate(uint64_t seed, cvm_keyset** out) {
  return guard([&] {
    need(out, "out");
    *out = new cvm_keyset(seed);
  });
}
void cvm_keyset_destroy(cvm_keyset* ks) { delete ks; }
int cvm_keyset_export(const cvm_keyset* k, int32_t* lwe_key, int32_t* tlwe_key, uint32_t* bk,
                      uint32_t* ksk) {
  return guard([&] {
    need(k, "keyset");
    if (lwe_key) std::memcpy(lwe_key, k->ks.lwe_key.data(), kN * 4);
    if (tlwe_key) std::memcpy(tlwe_key, k->ks.tlwe_key.data(), kPolyN * 4);
    if (bk) std::memcpy(bk, k->ks.bk.data(), kBkWords * 4);
    if (ksk) std::memcpy(ksk, k->ks.ksk.data(), kKskWords * 4);
  });
}
int cvm_encrypt_bits(const cvm_keyset* k, uint64_t seed, size_t count, const uint8_t* bits,
                     uint32_t* out) {
  return guard([&] {
    need(k, "keyset");
    if (count) {
      need(bits, "bits");
      need(out, "out");
    }
    k->ks.encrypt(seed, count, bits, out);
  });
}
int cvm_decrypt_bits(const cvm_keyset* k, size_t count, const uint32_t* lwe, uint8_t* bits,
                     int32_t* phases) {
  return guard([&] {
    need(k, "keyset");
    if (count) need(lwe, "lwe");
    for (size_t i = 0; i < count; ++i) {
      const int32_t ph = k->ks.phase(lwe + i * kLweWords);
      if (bits) bits[i] = ph > 0;
      if (phases) phases[i] = ph;
    }
  });
}

// ----------------------------------------------------------- device ctx --
int cvm_ctx_create(int device, cvm_ctx** out) {
  return guard([&] {
    need(out, "out");
    *out = new cvm_ctx{context_create(device)};
  });
}
void cvm_ctx_destroy(cvm_ctx* c) {
  if (!c) return;
  context_destroy(c->ctx);
  delete c;
}
int cvm_upload_keys(cvm_ctx* c, const uint32_t* bk, const uint32_t* ksk) {
  return guard([&] {
    need(c, "ctx");
    context_upload_keys(c->ctx, bk, ksk);
  });
}
int cvm_upload_keyset(cvm_ctx* c, const cvm_keyset* k) {
  return guard([&] {
    need(c, "ctx");
    need(k, "keyset");
    context_upload_keys(c->ctx, k->ks.bk.data(), k->ks.ksk.data());
  });
}
int cvm_slots_reserve(cvm_ctx* c, uint64_t n) {
  return guard([&] {
    need(c, "ctx");
    context_reserve(c->ctx, n);
  });
}
int cvm_slots_alloc(cvm_ctx* c, uint64_t n, uint64_t* first) {
  return guard([&] {
    need(c, "ctx");
    need(first, "first");
    *first = context_alloc_slots(c->ctx, n);
    context_reserve(c->ctx, context_slots_used(c->ctx));
  });
}
uint64_t cvm_slots_capacity(const cvm_ctx* c) { return c ? context_capacity(c->ctx) : 0; }
int cvm_upload_lwe(cvm_ctx* c, uint64_t slot, uint64_t count, const uint32_t* lwe) {
  return guard([&] {
    need(c, "ctx");
    context_upload(c->ctx, slot, count, lwe);
  });
}
int cvm_download_lwe(cvm_ctx* c, uint64_t slot, uint64_t count, uint32_t* lwe) {
  return guard([&] {
    need(c, "ctx");
    context_download(c->ctx, slot, count, lwe);
  });
}
int cvm_submit_level(cvm_ctx* c, const cvm_gate* gates, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    context_submit_level(c->ctx, gates, count);
  });
}
int cvm_sync(cvm_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    context_sync(c->ctx);
  });
}
int cvm_ctx_set_profiling(cvm_ctx* c, int on) {
  return guard([&] {
    need(c, "ctx");
    context_set_profiling(c->ctx, on != 0);
  });
}
int cvm_ctx_kernel_stats(cvm_ctx* c, cvm_kernel_stats* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    *out = context_stats(c->ctx);
  });
}
int cvm_ctx_reset_stats(cvm_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    context_reset_stats(c->ctx);
  });
}
int cvm_ctx_flush_l2(cvm_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    context_flush_l2(c->ctx);
  });
}
int cvm_ctx_event_record(cvm_ctx* c, int which) {
  return guard([&] {
    need(c, "ctx");
    context_event(c->ctx, which);
  });
}
int cvm_ctx_event_elapsed_ms(cvm_ctx* c, double* ms) {
  return guard([&] {
    need(c, "ctx");
    need(ms, "ms");
    *ms = context_event_elapsed(c->ctx);
  });
}

int cvm_ctx_fp64_peak(cvm_ctx* c, int reps, double* tflops) {
  return guard([&] {
    need(c, "ctx");
    need(tflops, "tflops");
    *tflops = context_fp64_peak(c->ctx, reps < 1 ? 1 : reps);
  });
}
int cvm_ctx_sm_count(cvm_ctx* c, int* sms) {
  return guard([&] {
    need(c, "ctx");
    need(sms, "sms");
    *sms = context_sm_count(c->ctx);
  });
}

int cvm_set_br_variant(int v) {
  return guard([&] {
    if (!cvm::valid_br_variant(v))
      throw InputError("unknown blind-rotation kernel variant " + std::to_string(v));
    cvm::set_br_variant(v);
  });
}
int cvm_get_br_variant(void) { return cvm::br_variant(); }
int cvm_set_level_packing(int on) {
  return guard([&] {
    if (on != 0 && on != 1) throw InputError("level packing is 0 or 1");
    cvm::set_level_packing(on != 0);
  });
}
int cvm_get_level_packing(void) { return cvm::level_packing() ? 1 : 0; }
int cvm_set_ks_variant(int v) {
  return guard([&] {
    if (!cvm::valid_ks_variant(v))
      throw InputError("unknown key-switch kernel variant " + std::to_string(v));
    cvm::set_ks_variant(v);
  });
}
int cvm_get_ks_variant(void) { return cvm::ks_variant(); }
int cvm_ctx_set_kernels(cvm_ctx* c, int br_variant, int ks_variant, int level_packing) {
  return guard([&] {
    need(c, "ctx");
    if (br_variant != -1 && !valid_br_variant(br_variant))
      throw InputError("unknown blind-rotation variant " + std::to_string(br_variant));
    if (ks_variant != -1 && !valid_ks_variant(ks_variant))
      throw InputError("unknown key-switch variant " + std::to_string(ks_variant));
    if (level_packing < -1 || level_packing > 1) throw InputError("level_packing is -1, 0 or 1");
    context_set_kernels(c->ctx, br_variant, ks_variant, level_packing);
  });
}
int cvm_ctx_get_kernels(cvm_ctx* c, int* br_variant, int* ks_variant, int* level_packing) {
  return guard([&] {
    need(c, "ctx");
    context_get_kernels(c->ctx, br_variant, ks_variant, level_packing);
  });
}

// -------------------------------------------------------------- backend --
int cvm_backend_create(cvm_ctx* c, const cvm_keyset* owner, uint64_t enc_seed,
                       cvm_backend** out) {
  return guard([&] {
    need(out, "out");
    auto b = std::make_unique<cvm_backend>();
    if (c) {
      auto g = std::make_unique<GpuBackend>(c->ctx, owner ? &owner->ks : nullptr, enc_seed);
      b->gpu = g.get();
      b->impl = std::move(g);
    } else {
      auto r = std::make_unique<ClearBackend>();
      b->clear = r.get();
      b->impl = std::move(r);
    }
    *out = b.release();
  });
}
void cvm_backend_destroy(cvm_backend* b) { delete b; }
int cvm_backend_constant(cvm_backend* b, int v, cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->impl->constant(v != 0);
  });
}
int cvm_backend_unary_gate(cvm_backend* b, uint32_t kind, cvm_handle a, cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->impl->unary_gate(kind_of(kind), a);
  });
}
int cvm_backend_binary_gate(cvm_backend* b, uint32_t kind, cvm_handle x, cvm_handle y,
                            cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->impl->binary_gate(kind_of(kind), x, y);
  });
}
int cvm_backend_mux_gate(cvm_backend* b, cvm_handle s, cvm_handle t, cvm_handle f,
                         cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->impl->mux_gate(s, t, f);
  });
}
int cvm_backend_encrypt_bit(cvm_backend* b, int v, cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->impl->encrypt_bit(v != 0);
  });
}
int cvm_backend_decrypt_bit(cvm_backend* b, cvm_handle h, int* v) {
  return guard([&] {
    need(b, "backend");
    need(v, "out");
    *v = b->impl->decrypt_bit(h) ? 1 : 0;
  });
}
int cvm_backend_decrypt_bits(cvm_backend* b, size_t n, const cvm_handle* hs, uint8_t* out) {
  return guard([&] {
    need(b, "backend");
    if (n) {
      need(hs, "handles");
      need(out, "out");
    }
    if (b->gpu) b->gpu->decrypt_bits(n, hs, out);
    else
      for (size_t i = 0; i < n; ++i) out[i] = b->impl->decrypt_bit(hs[i]) ? 1 : 0;
  });
}
int cvm_backend_import_lwe(cvm_backend* b, size_t n, const uint32_t* lwe, cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    if (!b->gpu) throw InputError("the cleartext recorder holds no ciphertexts");
    if (n) need(out, "out");
    b->gpu->import_lwe(n, lwe, out);
  });
}
int cvm_backend_export_lwe(cvm_backend* b, size_t n, const cvm_handle* hs, uint32_t* lwe) {
  return guard([&] {
    need(b, "backend");
    if (!b->gpu) throw InputError("the cleartext recorder holds no ciphertexts");
    if (n) {
      need(hs, "handles");
      need(lwe, "out");
    }
    b->gpu->export_lwe(n, hs, lwe);
  });
}
int cvm_backend_export_bit(cvm_backend* b, cvm_handle h, uint8_t* blob, size_t size) {
  return guard([&] {
    need(b, "backend");
    need(blob, "blob");
    if (size != kLweWords * 4) throw InputError("bit ciphertexts are 2524-byte blobs");
    if (!b->gpu) throw InputError("the cleartext recorder holds no ciphertexts");
    uint32_t c[kLweWords];
    b->gpu->export_lwe(1, &h, c);
    std::memcpy(blob, c, sizeof(c));  // little-endian host
  });
}
int cvm_backend_import_bit(cvm_backend* b, const uint8_t* blob, size_t size, cvm_handle* out) {
  return guard([&] {
    need(b, "backend");
    need(blob, "blob");
    need(out, "out");
    if (size != kLweWords * 4) throw InputError("bit ciphertexts are 2524-byte blobs");
    if (!b->gpu) throw InputError("the cleartext recorder holds no ciphertexts");
    uint32_t c[kLweWords];
    std::memcpy(c, blob, sizeof(c));
    b->gpu->import_lwe(1, c, out);
  });
}
int cvm_backend_push_region(cvm_backend* b, const char* name) {
  return guard([&] {
    need(b, "backend");
    need(name, "name");
    b->impl->push_region(name);
  });
}
int cvm_backend_pop_region(cvm_backend* b) {
  return guard([&] {
    need(b, "backend");
    b->impl->pop_region();
  });
}
int cvm_backend_fence(cvm_backend* b) {
  return guard([&] {
    need(b, "backend");
    b->impl->fence();
  });
}
int cvm_backend_flush(cvm_backend* b) {
  return guard([&] {
    need(b, "backend");
    if (b->gpu) b->gpu->flush();
  });
}
int cvm_backend_set_flush_policy(cvm_backend* b, int policy) {
  return guard([&] {
    need(b, "backend");
    if (policy != CVM_FLUSH_CONE && policy != CVM_FLUSH_ALL)
      throw InputError("unknown flush policy");
    if (b->gpu) b->gpu->set_cone_only(policy == CVM_FLUSH_CONE);
  });
}
int cvm_backend_stats_get(const cvm_backend* b, cvm_backend_stats* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->gpu ? b->gpu->stats() : b->clear->stats();
  });
}
int cvm_backend_region_count(const cvm_backend* b, uint64_t* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    if (!b->gpu) throw InputError("the cleartext recorder keeps no region attribution");
    *out = b->gpu->region_count();
  });
}
int cvm_backend_region_info(const cvm_backend* b, uint64_t idx, char* name, size_t name_size,
                            uint64_t* recorded, uint64_t* executed) {
  return guard([&] {
    need(b, "backend");
    if (!b->gpu) throw InputError("the cleartext recorder keeps no region attribution");
    std::string n;
    b->gpu->region_info(idx, &n, recorded, executed);
    if (name && name_size) {
      const size_t k = std::min(n.size(), name_size - 1);
      std::memcpy(name, n.data(), k);
      name[k] = 0;
    }
  });
}
int cvm_backend_node_count(const cvm_backend* b, uint64_t* out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    *out = b->gpu ? b->gpu->nodes().size() : b->clear->nodes().size();
  });
}
int cvm_backend_nodes(const cvm_backend* b, uint64_t first, uint64_t count, int64_t* rows) {
  return guard([&] {
    need(b, "backend");
    const std::vector<Node>& ns = b->gpu ? b->gpu->nodes() : b->clear->nodes();
    if (first + count > ns.size()) throw InputError("node range out of bounds");
    if (count) need(rows, "rows");
    for (uint64_t i = 0; i < count; ++i) {
      const Node& n = ns[first + i];
      int64_t* r = rows + i * 7;
      r[0] = int64_t(n.kind);
      r[1] = n.input;
      r[2] = n.ndeps;
      r[3] = int64_t(n.dep[0]);
      r[4] = int64_t(n.dep[1]);
      r[5] = int64_t(n.dep[2]);
      r[6] = n.const_value;
    }
  });
}

int cvm_backend_capture_plan(cvm_backend* b, cvm_plan** out) {
  return guard([&] {
    need(b, "backend");
    need(out, "out");
    if (!b->gpu) throw InputError("the cleartext recorder cannot capture device plans");
    *out = reinterpret_cast<cvm_plan*>(b->gpu->capture_plan());
  });
}
int cvm_plan_run(cvm_ctx* c, cvm_plan* p, int use_graph) {
  return guard([&] {
    need(c, "ctx");
    need(p, "plan");
    context_run_plan(c->ctx, reinterpret_cast<Plan*>(p), use_graph != 0);
  });
}
int cvm_plan_info(const cvm_plan* p, uint64_t* levels, uint64_t* gates, uint64_t* boots) {
  return guard([&] {
    need(p, "plan");
    const Plan* q = reinterpret_cast<const Plan*>(p);
    if (levels) *levels = q->levels.size();
    if (gates) *gates = q->gates;
    if (boots) *boots = q->bootstraps;
  });
}
void cvm_plan_destroy(cvm_plan* p) { delete reinterpret_cast<Plan*>(p); }
int cvm_backend_handle_slot(const cvm_backend* b, cvm_handle h, int64_t* slot, int32_t* sign,
                            uint32_t* constant) {
  return guard([&] {
    need(b, "backend");
    const std::vector<Node>& ns = b->gpu ? b->gpu->nodes() : b->clear->nodes();
    if (h == 0 || h > ns.size()) throw InputError("invalid bit handle");
    const Node& n = ns[h - 1];
    if (slot) *slot = n.slot;
    if (sign) *sign = n.sign;
    if (constant) *constant = n.constant;
  });
}

// --------------------------------------------------------------- circuits --
int cvm_backend_replay_dag(cvm_backend* b, const cvm_dag_node* nodes, uint64_t n,
                           const cvm_handle* inputs, uint64_t n_inputs, cvm_handle* handles) {
  return guard([&] {
    need(b, "backend");
    if (n_inputs) need(inputs, "inputs");
    replay_dag(*b->impl, nodes, n, inputs, n_inputs, handles);
  });
}
int cvm_backend_set_dag_regions(cvm_backend* b, const char* const* names, uint64_t n) {
  return guard([&] {
    need(b, "backend");
    if (n) need(names, "names");
    if (b->gpu) b->gpu->set_dag_regions(names, n);
  });
}
int cvm_backend_evaluate(cvm_backend* b, size_t n, const cvm_handle* hs) {
  return guard([&] {
    need(b, "backend");
    if (n) need(hs, "handles");
    if (b->gpu) b->gpu->evaluate(n, hs);
  });
}

int cvm_dag_batch(cvm_ctx* c, const cvm_dag_node* nodes, uint64_t n_nodes,
                  const uint64_t* outputs, uint64_t n_outputs, uint64_t batch,
                  const uint32_t* in_lwe, uint64_t in_words, uint32_t* out_lwe,
                  uint64_t out_words, cvm_backend_stats* stats) {
  return cvm_dag_batch_regions(c, nodes, n_nodes, nullptr, 0, outputs, n_outputs, batch, in_lwe,
                               in_words, out_lwe, out_words, stats);
}

int cvm_dag_batch_regions(cvm_ctx* c, const cvm_dag_node* nodes, uint64_t n_nodes,
                          const char* const* region_names, uint64_t n_regions,
                          const uint64_t* outputs, uint64_t n_outputs, uint64_t batch,
                          const uint32_t* in_lwe, uint64_t in_words, uint32_t* out_lwe,
                          uint64_t out_words, cvm_backend_stats* stats) {
  return guard([&] {
    need(c, "ctx");
    uint64_t n_in = 0;
    validate_dag(nodes, n_nodes, &n_in);
    if (n_outputs) need(outputs, "outputs");
    for (uint64_t o = 0; o < n_outputs; ++o)
      if (outputs[o] == 0 || outputs[o] > n_nodes) throw InputError("output id out of range");
    const uint64_t kMaxBits = UINT64_MAX / kLweWords;
    if (batch && (n_in > kMaxBits / batch || n_outputs > kMaxBits / batch))
      throw InputError("batch too large");
    if (in_words != batch * n_in * kLweWords)
      throw InputError("in_lwe holds " + std::to_string(in_words) + " words, the batch needs " +
                       std::to_string(batch * n_in * kLweWords));
    if (out_words != batch * n_outputs * kLweWords)
      throw InputError("out_lwe holds " + std::to_string(out_words) + " words, the batch needs " +
                       std::to_string(batch * n_outputs * kLweWords));
    if (in_words) need(in_lwe, "in_lwe");
    if (out_words) need(out_lwe, "out_lwe");
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    GpuBackend bk(c->ctx, nullptr, 0);
    if (n_regions) {
      need(region_names, "region_names");
      bk.set_dag_regions(region_names, n_regions);
    }
    std::vector<Bit> in(batch * n_in), handles(n_nodes), outs(batch * n_outputs);
    // Inputs are DMA'd straight from the caller's buffers; every path out of
    // this call synchronises the stream first, so they may be released after.
    auto t1 = t0, t2 = t0;
    try {
      bk.import_lwe_direct(in.size(), in_lwe, in.data());
      t1 = clk::now();
      for (uint64_t i = 0; i < batch; ++i) {
        replay_dag(bk, nodes, n_nodes, in.data() + i * n_in, n_in, handles.data());
        for (uint64_t o = 0; o < n_outputs; ++o)
          outs[i * n_outputs + o] = handles[outputs[o] - 1];
      }
      t2 = clk::now();
      bk.export_lwe(outs.size(), outs.data(), out_lwe);  // synchronises
      bk.release_slots();  // the batch's slots are scratch: reuse them next call
    } catch (...) {
      context_sync(c->ctx);
      bk.release_slots();  // the batch's scratch slots are not leaked on failure
      throw;
    }
    if (stats) *stats = bk.stats();
    if (std::getenv("CVM_DAG_TIMING")) {
      const auto ms = [](auto a, auto b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
      };
      std::fprintf(stderr, "cvm_dag_batch: import %.2f ms, record %.2f ms, run+export %.2f ms\n",
                   ms(t0, t1), ms(t1, t2), ms(t2, clk::now()));
    }
  });
}

}  // extern "C"
