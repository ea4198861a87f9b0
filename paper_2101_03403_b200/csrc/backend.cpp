// GpuBackend: the cryptovm::Backend contract (gates.hpp:109-132) over the
// device context, with lazy recording, dataflow levelisation and
// demand-driven evaluation.
//
// Reference behaviour kept:
//  * every gate call returns a handle immediately; handles are dense 1-based
//    node ids as in GateDag::append (dag.cpp:57-73), 0 is invalid;
//  * invalid handles / wrong kinds raise InputError before anything is
//    enqueued (sim_backend.cpp:47-57,80-83);
//  * CONSTANT, NOT and COPY are not bootstrapped (gates.cpp:35-50): here they
//    are folded into a linear form (sign * slot + constant) consumed by the
//    next bootstrapped gate's input combination, so they cost nothing;
//  * regions and fences are recorded, but a fence is only a latency-model
//    annotation (dag.hpp:44-48): gates are pure, so evaluation
//    follows dataflow -- the level of a gate is 1 + the deepest level among
//    its not-yet-evaluated inputs.
// Evaluation happens at flush points.  A decrypt / export evaluates only the
// cone of influence of the requested handles (everything else stays pending
// and runs if and when something needs it): gates are pure, so results are
// unchanged, and circuits whose outputs are partly discarded -- the
// emulator's MUL keeps the low half of a 2N-bit product (emulator.cpp:271-285),
// registers get overwritten, CMP flags get replaced -- skip their dead gates
// (SURVEY.md section 8 f-3).  cvm_backend_flush evaluates everything pending.
// Each level becomes one cvm_submit_level (two launches).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "cvm_internal.hpp"

namespace cvm {

int bootstrap_count(GateKind k) {
  switch (k) {
    case GateKind::Constant:
    case GateKind::Not:
    case GateKind::Copy:
      return 0;
    case GateKind::Mux:
      return 2;
    default:
      return 1;
  }
}

namespace {
bool is_gate(GateKind k) { return k >= GateKind::Nand; }
}  // namespace

GpuBackend::GpuBackend(Context* ctx, const KeySet* owner, uint64_t enc_seed)
    : ctx_(ctx), owner_(owner), enc_seed_(enc_seed) {
  if (!ctx_) throw InputError("backend needs a device context");
  if (!context_has_keys(ctx_)) throw StateError("upload keys before creating a backend");
  nodes_.reserve(1 << 16);
}

const Node& GpuBackend::node(Bit h, const char* what) const {
  if (h == 0 || h > nodes_.size())
    throw InputError(std::string("invalid bit handle passed to ") + what);
  return nodes_[h - 1];
}

Bit GpuBackend::add_node(Node n) {
  nodes_.push_back(n);
  stats_.nodes = nodes_.size();
  return nodes_.size();
}

cvm_operand GpuBackend::operand(Bit h) const {
  const Node& n = nodes_[h - 1];
  return cvm_operand{n.slot, n.sign, n.constant};
}

Bit GpuBackend::record_gate(Node n, const cvm_gate& g) {
  n.gate_idx = uint32_t(gates_.size());
  n.region = region_stack_.empty() ? 0u : region_stack_.back();
  region_recorded_[n.region]++;
  gates_.push_back(g);
  const Bit id = add_node(n);
  pending_.push_back(id);
  first_pending_ = std::min<uint64_t>(first_pending_, id);
  stats_.bootstrapped++;
  stats_.bootstraps += uint64_t(bootstrap_count(n.kind));
  return id;
}

Bit GpuBackend::constant(bool value) {
  std::lock_guard<std::mutex> lock(mu_);
  return constant_nl(value);
}
Bit GpuBackend::constant_nl(bool value) {
  Node n{};
  n.kind = GateKind::Constant;
  n.const_value = value;
  n.slot = -1;
  n.sign = 1;
  n.constant = value ? kMu : 0u - kMu;  // trivial sample (0, +-1/8)
  return add_node(n);
}

Bit GpuBackend::unary_gate(GateKind kind, Bit a) {
  std::lock_guard<std::mutex> lock(mu_);
  return unary_gate_nl(kind, a);
}
Bit GpuBackend::unary_gate_nl(GateKind kind, Bit a) {
  if (kind != GateKind::Not && kind != GateKind::Copy)
    throw InputError("not a unary gate");
  const Node& in = node(a, "unary_gate");
  Node n = in;
  n.kind = kind;
  n.input = false;
  n.const_value = false;
  n.ndeps = 1;
  n.dep[0] = a;
  n.dep[1] = n.dep[2] = 0;
  if (kind == GateKind::Not) {
    n.sign = -in.sign;
    n.constant = 0u - in.constant;
  }
  return add_node(n);
}

Bit GpuBackend::binary_gate(GateKind kind, Bit a, Bit b) {
  std::lock_guard<std::mutex> lock(mu_);
  return binary_gate_nl(kind, a, b);
}
Bit GpuBackend::binary_gate_nl(GateKind kind, Bit a, Bit b) {
  const Node& na = node(a, "binary_gate");
  const Node& nb = node(b, "binary_gate");
  if (bootstrap_count(kind) != 1) throw InputError("not a bootstrapped binary gate");
  Node n{};
  n.kind = kind;
  n.ndeps = 2;
  n.dep[0] = a;
  n.dep[1] = b;
  n.level = std::max(na.level, nb.level) + 1;
  n.slot = int64_t(take_slot());
  n.sign = 1;
  cvm_gate g{};
  g.kind = uint32_t(kind);
  g.in[0] = operand(a);
  g.in[1] = operand(b);
  g.in[2] = cvm_operand{-1, 1, 0};
  g.out_slot = uint64_t(n.slot);
  return record_gate(n, g);
}

Bit GpuBackend::mux_gate(Bit sel, Bit on_true, Bit on_false) {
  std::lock_guard<std::mutex> lock(mu_);
  return mux_gate_nl(sel, on_true, on_false);
}
Bit GpuBackend::mux_gate_nl(Bit sel, Bit on_true, Bit on_false) {
  const Node& ns = node(sel, "mux_gate");
  const Node& nt = node(on_true, "mux_gate");
  const Node& nf = node(on_false, "mux_gate");
  Node n{};
  n.kind = GateKind::Mux;
  n.ndeps = 3;
  n.dep[0] = sel;
  n.dep[1] = on_true;
  n.dep[2] = on_false;
  n.level = std::max({ns.level, nt.level, nf.level}) + 1;
  n.slot = int64_t(take_slot());
  n.sign = 1;
  cvm_gate g{};
  g.kind = uint32_t(GateKind::Mux);
  g.in[0] = operand(sel);
  g.in[1] = operand(on_true);
  g.in[2] = operand(on_false);
  g.out_slot = uint64_t(n.slot);
  return record_gate(n, g);
}

// A recorded table replayed under one lock (dag.cpp validates it first).
void GpuBackend::replay(const cvm_dag_node* nodes, uint64_t n, const Bit* inputs,
                        Bit* handles) {
  std::lock_guard<std::mutex> lock(mu_);
  if (!dag_region_.empty())  // region indices checked before anything is recorded
    for (uint64_t i = 0; i < n; ++i)
      if (nodes[i].region >= dag_region_.size())
        throw InputError("dag region index out of range at dag node " + std::to_string(i + 1));
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const cvm_dag_node& d = nodes[i];
    const GateKind kind = GateKind(d.kind);
    Bit h;
    if (d.input) h = inputs[k++];
    else if (kind == GateKind::Constant) h = constant_nl(d.value != 0);
    else if (kind == GateKind::Not || kind == GateKind::Copy)
      h = unary_gate_nl(kind, handles[d.dep[0] - 1]);
    else if (kind == GateKind::Mux)
      h = mux_gate_nl(handles[d.dep[0] - 1], handles[d.dep[1] - 1], handles[d.dep[2] - 1]);
    else h = binary_gate_nl(kind, handles[d.dep[0] - 1], handles[d.dep[1] - 1]);
    handles[i] = h;
    // attribute the gate to the table's region (recorded as the stack's top
    // otherwise)
    if (!dag_region_.empty() && d.region && is_gate(kind) && !d.input) {
      Node& nd = nodes_[h - 1];
      region_recorded_[nd.region]--;
      nd.region = dag_region_[d.region];
      region_recorded_[nd.region]++;
    }
  }
}

Bit GpuBackend::encrypt_bit(bool value) {
  if (!owner_) throw StateError("encrypt_bit needs the key owner's keyset");
  uint32_t c[kLweWords];
  const uint8_t bit = value ? 1 : 0;
  {
    std::lock_guard<std::mutex> lock(mu_);
    owner_->encrypt(enc_seed_ * 0x9E3779B97F4A7C15ull + enc_counter_++, 1, &bit, c);
  }
  Bit h;
  import_lwe(1, c, &h);
  return h;
}

void GpuBackend::import_lwe(size_t count, const uint32_t* lwe, Bit* out) {
  std::lock_guard<std::mutex> lock(mu_);
  if (count && !lwe) throw InputError("import: null ciphertexts");
  for (size_t i = 0; i < count; ++i) {
    const uint64_t s = take_slot();
    // Staged uploads form one contiguous slot run; start a new run otherwise.
    if (!pending_upload_.empty() &&
        pending_upload_slot_ + pending_upload_.size() / kLweWords != s)
      stage_uploads();
    if (pending_upload_.empty()) pending_upload_slot_ = s;
    pending_upload_.insert(pending_upload_.end(), lwe + i * kLweWords,
                           lwe + (i + 1) * kLweWords);
    Node n{};
    n.kind = GateKind::Constant;
    n.input = true;
    n.slot = int64_t(s);
    n.sign = 1;
    out[i] = add_node(n);
  }
}

// Zero-copy import for synchronous batch entry points (cvm_fu_batch): one
// contiguous slot run uploaded straight from the caller's buffer (a direct
// DMA when it is pinned, one staging copy otherwise).  The caller keeps `lwe`
// alive until the context is synchronised.
void GpuBackend::import_lwe_direct(size_t count, const uint32_t* lwe, Bit* out) {
  std::lock_guard<std::mutex> lock(mu_);
  if (count == 0) return;
  if (!lwe) throw InputError("import: null ciphertexts");
  stage_uploads();  // keep earlier staged uploads ordered before this one
  const uint64_t first = context_alloc_slots(ctx_, count);
  runs_.push_back({first, first + count});
  context_reserve(ctx_, context_slots_used(ctx_));
  context_upload(ctx_, first, count, lwe);
  for (size_t i = 0; i < count; ++i) {
    Node n{};
    n.kind = GateKind::Constant;
    n.input = true;
    n.slot = int64_t(first + i);
    n.sign = 1;
    out[i] = add_node(n);
  }
}

bool GpuBackend::release_slots() {
  std::lock_guard<std::mutex> lock(mu_);
  if (runs_.empty()) return true;
  auto r = runs_;
  std::sort(r.begin(), r.end());
  for (size_t i = 1; i < r.size(); ++i)
    if (r[i].first != r[i - 1].second) return false;  // another user interleaved
  if (!context_release_slots(ctx_, r.front().first, r.back().second)) return false;
  runs_.clear();
  next_slot_ = chunk_end_ = 0;
  cache_.clear();
  slot_evaluated_.clear();
  return true;
}

uint64_t GpuBackend::take_slot() {
  if (next_slot_ == chunk_end_) {
    next_slot_ = context_alloc_slots(ctx_, chunk_);
    chunk_end_ = next_slot_ + chunk_;
    runs_.push_back({next_slot_, chunk_end_});
    chunk_ = std::min<uint64_t>(chunk_ * 2, uint64_t(1) << 20);
  }
  return next_slot_++;
}

// Copies the staged run into pinned memory and enqueues its upload.
void GpuBackend::stage_uploads() {
  if (pending_upload_.empty()) return;
  context_reserve(ctx_, context_slots_used(ctx_));
  context_upload(ctx_, pending_upload_slot_, pending_upload_.size() / kLweWords,
                 pending_upload_.data());
  pending_upload_.clear();
}

// Below this many gates every level runs on the latency kernels, whose cost
// does not reward reshaping.
constexpr int kPackMinGates = 2 * 148;

static std::atomic<int> g_pack{-1};
bool level_packing() {
  if (g_pack.load() < 0) {
    const char* e = getenv("CVM_PACK");
    g_pack.store(e && e[0] == '0' ? 0 : 1);
  }
  return g_pack.load() == 1;
}
void set_level_packing(bool on) { g_pack.store(on ? 1 : 0); }

// Groups the selected pending gates into launches (their pending inputs are
// selected too, so levels stay consistent): by dataflow level, or -- the
// default -- wave-packed (pack_levels).
std::vector<std::vector<cvm_gate>> GpuBackend::levels_of(
    const std::vector<Bit>& ids, std::vector<std::vector<Bit>>* ids_out) const {
  uint32_t depth = 0;
  for (Bit id : ids) depth = std::max(depth, nodes_[id - 1].level);
  if (context_level_packing(ctx_) && depth > 1 && ids.size() > size_t(kPackMinGates))
    return pack_levels(ids, depth, ids_out);
  std::vector<std::vector<cvm_gate>> lv;
  std::vector<std::vector<Bit>> li;
  for (Bit id : ids) {
    const Node& n = nodes_[id - 1];
    if (lv.size() < n.level) lv.resize(n.level), li.resize(n.level);
    lv[n.level - 1].push_back(gates_[n.gate_idx]);
    li[n.level - 1].push_back(id);
  }
  lv.erase(std::remove_if(lv.begin(), lv.end(), [](const auto& v) { return v.empty(); }),
           lv.end());
  li.erase(std::remove_if(li.begin(), li.end(), [](const auto& v) { return v.empty(); }),
           li.end());
  if (ids_out) *ids_out = std::move(li);
  return lv;
}

// Wave packing (schedule.hpp): the number of launches stays the critical
// path, but a gate may run in any launch between its earliest (ASAP) and
// latest (ALAP) level, and launches are filled to the widths the
// blind-rotation planner runs most efficiently: e.g. a 256 x ADD16 batch runs
// as five launches of exactly six full v4 waves instead of ASAP widths 8192,
// 8192, 7680, 7424, 6656 (each with a partial wave).  Gates are pure, so
// results are unchanged (tests/test_gpu_parity.py compares packed and plain
// runs; tests/native/schedule_test.cpp checks the schedule's invariants).
std::vector<std::vector<cvm_gate>> GpuBackend::pack_levels(
    std::vector<Bit> ids, uint32_t depth, std::vector<std::vector<Bit>>* ids_out) const {
  std::sort(ids.begin(), ids.end());  // node ids are a topological order
  const size_t G = ids.size();
  const Bit lo = ids.front(), hi = ids.back();
  std::vector<int32_t> local(hi - lo + 1, -1);
  for (size_t i = 0; i < G; ++i) local[ids[i] - lo] = int32_t(i);
  // the selected gate a dependency stands for (NOT / COPY are folded)
  auto src = [&](Bit id) -> int32_t {
    while (id) {
      const Node& n = nodes_[id - 1];
      if (n.input || (n.kind != GateKind::Not && n.kind != GateKind::Copy)) break;
      id = n.dep[0];
    }
    return (id >= lo && id <= hi) ? local[id - lo] : -1;
  };
  std::vector<int32_t> pred(3 * G, -1);
  std::vector<uint8_t> boots(G);
  for (size_t i = 0; i < G; ++i) {
    const Node& n = nodes_[ids[i] - 1];
    boots[i] = n.kind == GateKind::Mux ? 2 : 1;
    for (int d = 0; d < n.ndeps; ++d) {
      const int32_t s = src(n.dep[d]);
      bool dup = false;
      for (int e = 0; e < d; ++e) dup |= pred[3 * i + e] == s;
      if (s >= 0 && !dup) pred[3 * i + d] = s;
    }
  }
  const std::vector<uint32_t> launch = pack_schedule(pred, boots);
  std::vector<std::vector<cvm_gate>> out(depth);
  std::vector<std::vector<Bit>> li(depth);
  for (size_t i = 0; i < G; ++i) {
    out[launch[i] - 1].push_back(gates_[nodes_[ids[i] - 1].gate_idx]);
    li[launch[i] - 1].push_back(ids[i]);
  }
  out.erase(std::remove_if(out.begin(), out.end(), [](const auto& v) { return v.empty(); }),
            out.end());
  li.erase(std::remove_if(li.begin(), li.end(), [](const auto& v) { return v.empty(); }),
           li.end());
  if (ids_out) *ids_out = std::move(li);
  return out;
}

// After the gates in `done` became resident: recompute the levels of what is
// still pending (node ids are a topological order) and drop `done`.
void GpuBackend::retire(const std::vector<Bit>& done) {
  for (Bit id : done) nodes_[id - 1].level = 0;
  if (done.size() == pending_.size()) {
    pending_.clear();
    for (uint64_t i = first_pending_; i <= nodes_.size(); ++i) nodes_[i - 1].level = 0;
    first_pending_ = UINT64_MAX;
    return;
  }
  std::vector<Bit> still;
  still.reserve(pending_.size() - done.size());
  for (Bit id : pending_)
    if (nodes_[id - 1].level != 0) still.push_back(id);
  pending_.swap(still);
  const uint64_t from = pending_.empty() ? nodes_.size() + 1 : pending_.front();
  for (uint64_t i = first_pending_; i <= nodes_.size(); ++i) {
    Node& n = nodes_[i - 1];
    if (n.level == 0) continue;
    uint32_t lv = 0;
    for (int d = 0; d < n.ndeps; ++d) lv = std::max(lv, nodes_[n.dep[d] - 1].level);
    n.level = is_gate(n.kind) ? lv + 1 : lv;
  }
  first_pending_ = from;
}

void GpuBackend::run(const std::vector<Bit>& ids) {
  context_reserve(ctx_, context_slots_used(ctx_));
  stage_uploads();
  std::vector<std::vector<Bit>> lids;
  const auto lv = levels_of(ids, &lids);
  for (Bit id : ids) {
    const Node& n = nodes_[id - 1];
    region_executed_[n.region]++;
    if (slot_evaluated_.empty()) slot_base_ = uint64_t(n.slot);
    if (uint64_t(n.slot) < slot_base_) {
      slot_evaluated_.insert(slot_evaluated_.begin(), slot_base_ - uint64_t(n.slot), 0);
      slot_base_ = uint64_t(n.slot);
    }
    const uint64_t k = uint64_t(n.slot) - slot_base_;
    if (k >= slot_evaluated_.size()) slot_evaluated_.resize(k + 1, 0);
    slot_evaluated_[k] = 1;
  }
  // NVTX ranges per launch (nsys / ncu timelines), labelled with the
  // regions of its gates; built only when a tool is attached or CVM_NVTX=1
  static const bool nvtx = getenv("CUDA_INJECTION64_PATH") || getenv("CVM_NVTX");
  if (nvtx) nvtxRangePushA(("cvm flush: " + std::to_string(ids.size()) + " gates, " +
                            std::to_string(lv.size()) + " launches").c_str());
  uint64_t gates = 0, boots = 0;
  for (size_t k = 0; k < lv.size(); ++k) {
    const auto& level = lv[k];
    if (nvtx) nvtxRangePushA(level_label(k, lv.size(), lids[k]).c_str());
    context_submit_level(ctx_, level.data(), level.size());
    if (nvtx) nvtxRangePop();
    gates += level.size();
    for (const auto& g : level) boots += g.kind == uint32_t(GateKind::Mux) ? 2 : 1;
    stats_.max_level_width = std::max<uint64_t>(stats_.max_level_width, level.size());
  }
  context_sync(ctx_);
  if (nvtx) nvtxRangePop();
  stats_.flushes++;
  stats_.levels_run += lv.size();
  stats_.last_flush_levels = lv.size();
  stats_.last_flush_gates = gates;
  stats_.executed += gates;
  stats_.executed_bootstraps += boots;
  retire(ids);
}

void GpuBackend::flush() {
  std::lock_guard<std::mutex> lock(mu_);
  flush_locked();
}

void GpuBackend::flush_locked() {
  for (Bit id : pending_) {
    const Node& n = nodes_[id - 1];
    for (int d = 0; d < n.ndeps; ++d)
      if (nodes_[n.dep[d] - 1].level == 0) check_captured(nodes_[n.dep[d] - 1]);
  }
  if (pending_.empty()) {
    stage_uploads();
    return;
  }
  const std::vector<Bit> all = pending_;
  run(all);
}

// A handle whose value a captured plan produces is readable only once that
// plan has run (capture marks its gates resident up front).
void GpuBackend::check_captured(const Node& n) const {
  if (n.plan && !plans_[n.plan - 1]->load())
    throw StateError("handle is produced by a captured plan that has not run yet");
}

// Evaluates the cone of influence of `hs` only.
void GpuBackend::flush_for(size_t count, const Bit* hs) {
  std::lock_guard<std::mutex> lock(mu_);
  for (size_t i = 0; i < count; ++i) node(hs[i], "evaluate");
  flush_for_locked(count, hs);
}

void GpuBackend::flush_for_locked(size_t count, const Bit* hs) {
  std::vector<Bit> need, stack;
  std::vector<uint8_t> seen;
  for (size_t i = 0; i < count; ++i) {
    const Node& n = nodes_[hs[i] - 1];
    if (n.level != 0) stack.push_back(hs[i]);
    else check_captured(n);
  }
  if (stack.empty()) {
    stage_uploads();
    return;
  }
  seen.assign(nodes_.size() - first_pending_ + 1, 0);
  while (!stack.empty()) {
    const Bit id = stack.back();
    stack.pop_back();
    const Node& n = nodes_[id - 1];
    if (n.level == 0) {
      check_captured(n);
      continue;
    }
    if (seen[id - first_pending_]) continue;
    seen[id - first_pending_] = 1;
    if (is_gate(n.kind)) need.push_back(id);
    for (int d = 0; d < n.ndeps; ++d) stack.push_back(n.dep[d]);
  }
  std::sort(need.begin(), need.end());
  run(need);
}

// Moves every pending level into a replayable plan (uploads are enqueued now).
// Its gates count as resident from here on, but reading one (export, decrypt,
// or a flush of a gate built on it) throws StateError until the plan has run.
Plan* GpuBackend::capture_plan() {
  std::lock_guard<std::mutex> lock(mu_);
  context_reserve(ctx_, context_slots_used(ctx_));
  stage_uploads();
  const std::vector<Bit> all = pending_;
  const auto lv = levels_of(all, nullptr);
  Plan* p = context_make_plan(ctx_, lv);
  p->ran = std::make_shared<std::atomic<bool>>(all.empty());
  plans_.push_back(p->ran);
  for (Bit id : all) nodes_[id - 1].plan = uint32_t(plans_.size());
  for (const auto& level : lv)
    stats_.max_level_width = std::max<uint64_t>(stats_.max_level_width, level.size());
  stats_.last_flush_levels = lv.size();
  stats_.last_flush_gates = p->gates;
  if (!all.empty()) retire(all);  // resident once the plan has run
  return p;
}

void GpuBackend::evaluate(size_t count, const Bit* hs) {
  std::lock_guard<std::mutex> lock(mu_);
  for (size_t i = 0; i < count; ++i) node(hs[i], "evaluate");
  flush_for_locked(count, hs);
  std::vector<uint64_t> sl;
  for (size_t i = 0; i < count; ++i) {
    const int64_t slot = nodes_[hs[i] - 1].slot;
    if (slot < 0 || uint64_t(slot) < slot_base_) continue;
    const uint64_t k = uint64_t(slot) - slot_base_;
    if (k < slot_evaluated_.size() && slot_evaluated_[k] == 1) {
      slot_evaluated_[k] = 2;  // queued / cached
      sl.push_back(uint64_t(slot));
    }
  }
  if (sl.empty()) return;
  std::vector<uint32_t> buf(sl.size() * kLweWords);
  context_gather_download(ctx_, sl.data(), sl.size(), buf.data());
  for (size_t q = 0; q < sl.size(); ++q)
    cache_[int64_t(sl[q])].assign(buf.begin() + q * kLweWords, buf.begin() + (q + 1) * kLweWords);
}

void GpuBackend::export_lwe(size_t count, const Bit* hs, uint32_t* out) {
  std::lock_guard<std::mutex> lock(mu_);
  for (size_t i = 0; i < count; ++i) node(hs[i], "export");
  // served from the host cache when every requested value is there
  bool cached = !cache_.empty();
  for (size_t i = 0; i < count && cached; ++i) {
    const Node& n = nodes_[hs[i] - 1];
    cached = n.slot < 0 || (n.level == 0 && cache_.count(n.slot));
  }
  if (cached) {
    for (size_t q = 0; q < count; ++q) {
      const Node& n = nodes_[hs[q] - 1];
      uint32_t* o = out + q * kLweWords;
      if (n.slot < 0) {
        std::memset(o, 0, kLweWords * 4);
      } else {
        const uint32_t* src = cache_.at(n.slot).data();
        for (int w = 0; w < kLweWords; ++w) o[w] = n.sign > 0 ? src[w] : 0u - src[w];
      }
      o[kN] += n.constant;
    }
    return;
  }
  if (cone_only_) {
    flush_for_locked(count, hs);
  } else {
    for (size_t i = 0; i < count; ++i)
      if (nodes_[hs[i] - 1].level == 0) check_captured(nodes_[hs[i] - 1]);
    flush_locked();
  }
  // One device gather of the requested slots (in request order) and one
  // download, then the linear forms (NOT / COPY / CONSTANT) applied on the host.
  std::vector<uint64_t> sl;
  sl.reserve(count);
  for (size_t q = 0; q < count; ++q)
    if (nodes_[hs[q] - 1].slot >= 0) sl.push_back(uint64_t(nodes_[hs[q] - 1].slot));
  const bool direct = sl.size() == count;  // gather straight into `out`
  std::vector<uint32_t> buf(direct ? 0 : sl.size() * kLweWords);
  uint32_t* base = direct ? out : buf.data();
  context_gather_download(ctx_, sl.data(), sl.size(), base);
  size_t k = 0;
  for (size_t q = 0; q < count; ++q) {
    const Node& n = nodes_[hs[q] - 1];
    uint32_t* o = out + q * kLweWords;
    if (n.slot < 0) {
      std::memset(o, 0, kLweWords * 4);
    } else {
      const uint32_t* src = base + (k++) * kLweWords;
      if (n.sign > 0) {
        if (src != o) std::memcpy(o, src, kLweWords * 4);
      } else {
        for (int w = 0; w < kLweWords; ++w) o[w] = 0u - src[w];
      }
    }
    o[kN] += n.constant;
  }
}

bool GpuBackend::decrypt_bit(Bit bit) {
  uint8_t v;
  decrypt_bits(1, &bit, &v);
  return v != 0;
}

void GpuBackend::decrypt_bits(size_t count, const Bit* hs, uint8_t* out) {
  if (!owner_) throw StateError("decrypt needs the key owner's keyset");
  std::vector<uint32_t> c(count * kLweWords);
  export_lwe(count, hs, c.data());
  for (size_t i = 0; i < count; ++i) out[i] = owner_->decrypt(&c[i * kLweWords]) ? 1 : 0;
  std::lock_guard<std::mutex> lock(mu_);
  stats_.decrypts += count;
}

uint32_t GpuBackend::intern_region(const std::string& path) {
  for (size_t i = 1; i < region_names_.size(); ++i)
    if (region_names_[i] == path) return uint32_t(i);
  region_names_.push_back(path);
  region_recorded_.push_back(0);
  region_executed_.push_back(0);
  return uint32_t(region_names_.size() - 1);
}

void GpuBackend::push_region(std::string_view name) {
  std::lock_guard<std::mutex> lock(mu_);
  const std::string path = region_stack_.empty()
                               ? std::string(name)
                               : region_names_[region_stack_.back()] + "/" + std::string(name);
  region_stack_.push_back(path.empty() ? 0u : intern_region(path));
}

void GpuBackend::set_dag_regions(const char* const* names, uint64_t n) {
  std::lock_guard<std::mutex> lock(mu_);
  dag_region_.assign(n, 0);
  for (uint64_t k = 0; k < n; ++k) {
    if (!names[k]) throw InputError("null region name");
    const std::string path(names[k]);
    dag_region_[k] = path.empty() ? 0u : intern_region(path);
  }
}

void GpuBackend::pop_region() {
  std::lock_guard<std::mutex> lock(mu_);
  if (region_stack_.empty()) throw InputError("pop_region without a matching push_region");
  region_stack_.pop_back();
}

size_t GpuBackend::region_count() const { return region_names_.size(); }
void GpuBackend::region_info(size_t idx, std::string* name, uint64_t* recorded,
                             uint64_t* executed) const {
  if (idx >= region_names_.size()) throw InputError("region index out of range");
  if (name) *name = region_names_[idx];
  if (recorded) *recorded = region_recorded_[idx];
  if (executed) *executed = region_executed_[idx];
}

// NVTX label of launch k of n: its width and the regions its gates come from
// (most gates first), e.g. "cvm level 3/9: 7104 gates [adder/carry 6656, ...]".
std::string GpuBackend::level_label(size_t k, size_t n, const std::vector<Bit>& ids) const {
  std::vector<std::pair<uint64_t, uint32_t>> hist;
  for (Bit id : ids) {
    const uint32_t r = nodes_[id - 1].region;
    auto it = std::find_if(hist.begin(), hist.end(), [r](const auto& h) { return h.second == r; });
    if (it == hist.end()) hist.push_back({1, r});
    else ++it->first;
  }
  std::sort(hist.begin(), hist.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  std::string s = "cvm level " + std::to_string(k + 1) + "/" + std::to_string(n) + ": " +
                  std::to_string(ids.size()) + " gates [";
  for (size_t i = 0; i < hist.size() && i < 3; ++i)
    s += (i ? ", " : "") + (region_names_[hist[i].second].empty()
                                ? std::string("-")
                                : region_names_[hist[i].second]) +
         " " + std::to_string(hist[i].first);
  return s + (hist.size() > 3 ? ", ...]" : "]");
}

void GpuBackend::fence() {
  std::lock_guard<std::mutex> lock(mu_);
  ++fences_;
}

cvm_backend_stats GpuBackend::stats() const {
  cvm_backend_stats s = stats_;
  s.pending = pending_.size();
  return s;
}

}  // namespace cvm
