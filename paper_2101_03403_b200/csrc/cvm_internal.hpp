// Internal C++ interfaces behind the C ABI (include/cvm_gpu.h).
#pragma once
#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/cvm_gpu.h"
#include "schedule.hpp"
#include "tfhe_params.h"

namespace cvm {

// Error taxonomy of the reference (errors.hpp:24-58): InputError for
// precondition violations, Error for everything else (here: device failures).
struct InputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- key owner --
struct KeySet {
  explicit KeySet(uint64_t seed);
  void encrypt(uint64_t seed, size_t count, const uint8_t* bits, uint32_t* out) const;
  int32_t phase(const uint32_t* lwe) const;
  bool decrypt(const uint32_t* lwe) const { return phase(lwe) > 0; }

  std::vector<int32_t> lwe_key, tlwe_key;
  std::vector<uint32_t> bk, ksk;
};

// ------------------------------------------------------------ device ctx --
class Context;
struct BrJob;
struct KsJob;

// Captured gate levels with device-resident job tables (cvm_plan).
struct Plan {
  struct Level {
    const BrJob* br;
    uint64_t n_br;
    const KsJob* ks;
    uint64_t n_ks;
  };
  ~Plan();
  std::vector<Level> levels;
  uint64_t gates = 0, bootstraps = 0, max_br = 0;
  void* dmem = nullptr;
  void* exec = nullptr;  // cudaGraphExec_t
  const void* graph_slab = nullptr;
  const void* graph_xlwe = nullptr;
  const Context* owner = nullptr;  // the context whose slots and memory it uses
  std::shared_ptr<std::atomic<bool>> ran;  // set by the first cvm_plan_run
};
Context* context_create(int device);
void context_destroy(Context* c);
void context_upload_keys(Context* c, const uint32_t* bk, const uint32_t* ksk);
void context_reserve(Context* c, uint64_t n);
uint64_t context_alloc_slots(Context* c, uint64_t n);  // returns first slot id
uint64_t context_slots_used(const Context* c);
bool context_release_slots(Context* c, uint64_t first, uint64_t end);
uint64_t context_capacity(const Context* c);
void context_upload(Context* c, uint64_t slot, uint64_t count, const uint32_t* lwe);
void context_download(Context* c, uint64_t slot, uint64_t count, uint32_t* lwe);
// Any slot list -> one contiguous [count][631] host block (device gather).
void context_gather_download(Context* c, const uint64_t* slots, uint64_t count,
                             uint32_t* lwe);
void context_submit_level(Context* c, const cvm_gate* gates, uint64_t count);
void context_sync(Context* c);
Plan* context_make_plan(Context* c, const std::vector<std::vector<cvm_gate>>& levels);
void context_run_plan(Context* c, Plan* p, bool graph);
bool context_has_keys(const Context* c);
void context_set_profiling(Context* c, bool on);
cvm_kernel_stats context_stats(Context* c);
void context_reset_stats(Context* c);
void context_flush_l2(Context* c);
void context_event(Context* c, int which);
double context_event_elapsed(Context* c);
double context_fp64_peak(Context* c, int reps);
int context_sm_count(const Context* c);
// Per-context kernel choices (-1 = follow the process-wide setting).
void context_set_kernels(Context* c, int br, int ks, int pack);
void context_get_kernels(Context* c, int* br, int* ks, int* pack);
bool context_level_packing(Context* c);

// --------------------------------------------------------------- backend --
// Mirror of cryptovm::Backend (gates.hpp:109-132) with handles as dense node
// ids (0 = invalid).
using Bit = uint64_t;

enum class GateKind : uint8_t {
  Constant, Not, Copy, Nand, And, Or, Xor, Xnor, Nor, AndNY, AndYN, OrNY, OrYN, Mux
};
int bootstrap_count(GateKind k);

class Backend {
 public:
  virtual ~Backend() = default;
  virtual Bit constant(bool value) = 0;
  virtual Bit unary_gate(GateKind kind, Bit a) = 0;
  virtual Bit binary_gate(GateKind kind, Bit a, Bit b) = 0;
  virtual Bit mux_gate(Bit sel, Bit on_true, Bit on_false) = 0;
  virtual Bit encrypt_bit(bool value) = 0;
  virtual bool decrypt_bit(Bit bit) = 0;
  virtual void push_region(std::string_view name) = 0;
  virtual void pop_region() = 0;
  virtual void fence() = 0;
};

// Node record (the reference DagNode, dag.hpp:33-42, minus cost/region).
// Wave packing of the levelizer (backend.cpp); process-wide, default on
// (env CVM_PACK=0 turns it off).
bool level_packing();
void set_level_packing(bool on);

struct Node {
  GateKind kind;
  bool input;
  bool const_value;
  uint8_t ndeps;
  uint32_t level;       // dataflow level (bootstrapped depth), 0 = available
  uint32_t gate_idx;    // GpuBackend: index of the recorded cvm_gate
  Bit dep[3];
  // Linear form of the node's ciphertext: sign * slab[slot] + constant.
  int64_t slot;         // -1: pure constant
  int32_t sign;
  uint32_t constant;
  uint32_t plan;        // 1-based index of the captured plan producing it, 0 = none
  uint32_t region;      // region path index at recording (GpuBackend::region_name)
};

class GpuBackend final : public Backend {
 public:
  GpuBackend(Context* ctx, const KeySet* owner, uint64_t enc_seed);
  Bit constant(bool value) override;
  Bit unary_gate(GateKind kind, Bit a) override;
  Bit binary_gate(GateKind kind, Bit a, Bit b) override;
  Bit mux_gate(Bit sel, Bit on_true, Bit on_false) override;
  Bit encrypt_bit(bool value) override;
  bool decrypt_bit(Bit bit) override;
  void push_region(std::string_view name) override;
  void pop_region() override;
  void fence() override;

  void decrypt_bits(size_t n, const Bit* hs, uint8_t* out);
  // a validated recorded table (dag.cpp) re-issued under one lock
  void replay(const cvm_dag_node* nodes, uint64_t n, const Bit* inputs, Bit* handles);
  // region names of the replayed tables' node.region indices
  void set_dag_regions(const char* const* names, uint64_t n);
  void import_lwe(size_t n, const uint32_t* lwe, Bit* out);
  void import_lwe_direct(size_t n, const uint32_t* lwe, Bit* out);
  void export_lwe(size_t n, const Bit* hs, uint32_t* out);
  // Give every slot this backend took back to the context if they are the
  // allocator's top run (call only after the work is synchronised and the
  // backend will not be used again).  Returns whether they were released.
  bool release_slots();
  void flush();                             // everything pending
  void flush_for(size_t n, const Bit* hs);  // cone of influence of hs only (validated)
  // flush_for + one download of the requested gate outputs into a host cache:
  // the key owner's bit-by-bit decryptions that follow (word.cpp:70-77) are
  // then served without a device round trip each (cvm_backend_evaluate).
  void evaluate(size_t n, const Bit* hs);
  // Flush policy of decrypt/export: the requested cone only (default) or
  // everything pending (for callers that decrypt bit by bit, like the
  // reference's decrypt_word loop, word.cpp:70-77).
  void set_cone_only(bool on) { cone_only_ = on; }
  Plan* capture_plan();
  cvm_backend_stats stats() const;
  // Region attribution (the reference's region labels, GateDag::intern_region
  // / bootstrapped_in_region, dag.hpp): path "a/b" of the region stack at
  // each gate; index 0 = outside any region.
  size_t region_count() const;
  void region_info(size_t idx, std::string* name, uint64_t* recorded, uint64_t* executed) const;
  const std::vector<Node>& nodes() const { return nodes_; }

 private:
  const Node& node(Bit h, const char* what) const;
  Bit constant_nl(bool value);  // the gate calls without taking mu_
  Bit unary_gate_nl(GateKind kind, Bit a);
  Bit binary_gate_nl(GateKind kind, Bit a, Bit b);
  Bit mux_gate_nl(Bit sel, Bit on_true, Bit on_false);
  Bit add_node(Node n);
  Bit record_gate(Node n, const cvm_gate& g);
  cvm_operand operand(Bit h) const;
  uint64_t take_slot();
  void stage_uploads();
  // launches of the selected gates; `ids_out` (optional) gets each launch's
  // node ids in the same order
  std::vector<std::vector<cvm_gate>> levels_of(const std::vector<Bit>& ids,
                                               std::vector<std::vector<Bit>>* ids_out) const;
  std::vector<std::vector<cvm_gate>> pack_levels(std::vector<Bit> ids, uint32_t depth,
                                                 std::vector<std::vector<Bit>>* ids_out) const;
  std::string level_label(size_t k, size_t n, const std::vector<Bit>& ids) const;
  void run(const std::vector<Bit>& ids);
  void retire(const std::vector<Bit>& done);
  void flush_locked();
  void flush_for_locked(size_t n, const Bit* hs);
  void check_captured(const Node& n) const;

  std::mutex mu_;
  Context* ctx_;
  const KeySet* owner_;
  uint64_t enc_seed_;
  uint64_t enc_counter_ = 0;
  std::vector<Node> nodes_;          // nodes_[id - 1]
  uint64_t next_slot_ = 0, chunk_end_ = 0, chunk_ = 4096;  // slot chunk from ctx
  std::vector<std::pair<uint64_t, uint64_t>> runs_;  // slot runs taken [first, end)
  // pending uploads (fresh encryptions / imports) and recorded gates
  std::vector<uint32_t> pending_upload_;
  uint64_t pending_upload_slot_ = 0;
  std::vector<cvm_gate> gates_;     // every recorded gate (node.gate_idx)
  std::vector<Bit> pending_;        // not yet evaluated gate nodes, id order
  uint64_t first_pending_ = UINT64_MAX;
  bool cone_only_ = true;
  std::vector<uint32_t> region_stack_;        // indices of the open regions
  std::vector<std::string> region_names_{""};  // interned paths
  std::vector<uint64_t> region_recorded_{0}, region_executed_{0};
  std::vector<uint32_t> dag_region_;  // replayed table's region index -> region id
  uint32_t intern_region(const std::string& path);
  uint64_t fences_ = 0;
  cvm_backend_stats stats_{};
  std::vector<std::shared_ptr<std::atomic<bool>>> plans_;  // captured plans: ran yet?
  // Host copies of evaluated gate outputs (slot -> 631 words).  Only slots a
  // flush of this backend wrote: gate outputs are never rewritten (a plan's
  // and an input's slots are, so they are never cached); cleared when the
  // backend returns its slots.
  std::vector<uint8_t> slot_evaluated_;  // by slot - slot_base_
  uint64_t slot_base_ = 0;
  std::unordered_map<int64_t, std::vector<uint32_t>> cache_;
};

// Cleartext recorder: the SimBackend semantics (sim_backend.cpp:25-154) with
// the same node table as GpuBackend.  It holds no ciphertexts and cannot run
// the bootstrapping path; it exists so the host logic (circuits, levelisation,
// DAG identity with the reference) is testable without a GPU, and as the
// shadow that GPU results are checked against.
class ClearBackend final : public Backend {
 public:
  Bit constant(bool value) override;
  Bit unary_gate(GateKind kind, Bit a) override;
  Bit binary_gate(GateKind kind, Bit a, Bit b) override;
  Bit mux_gate(Bit sel, Bit on_true, Bit on_false) override;
  Bit encrypt_bit(bool value) override;
  bool decrypt_bit(Bit bit) override;
  void push_region(std::string_view name) override;
  void pop_region() override;
  void fence() override;
  cvm_backend_stats stats() const { return stats_; }
  const std::vector<Node>& nodes() const { return nodes_; }

 private:
  Bit add(Node n, bool value);
  bool value(Bit h, const char* what) const;
  std::mutex mu_;
  std::vector<Node> nodes_;
  std::vector<uint8_t> values_;
  size_t regions_ = 0;
  cvm_backend_stats stats_{};
};

// ---------------------------------------------------------- circuit replay --
// A recorded circuit (cvm_dag_node table, the reference GateDag's node shape)
// re-issued as Backend calls; handles[i] receives node i+1's handle.  Inputs
// are consumed in node order by the table's input nodes (dag.cpp).
void validate_dag(const cvm_dag_node* nodes, uint64_t n, uint64_t* n_inputs);
void replay_dag(Backend& bk, const cvm_dag_node* nodes, uint64_t n, const Bit* inputs,
                uint64_t n_inputs, Bit* handles);

}  // namespace cvm

namespace cvm {
// Blind-rotation kernel variant selection (kernels.cu).
int br_variant();
void set_br_variant(int v);
int default_br_variant();
bool valid_br_variant(int v);
int ks_variant();
void set_ks_variant(int v);
bool valid_ks_variant(int v);
}  // namespace cvm
