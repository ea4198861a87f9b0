// Cleartext recorder (see cvm_internal.hpp): boolean semantics of every gate
// kind as in SimBackend::eval_binary (sim_backend.cpp:25-51), MUX argument
// order sel ? on_true : on_false (sim_backend.cpp:98-106), plus the node
// table and dataflow-level statistics the GPU backend would produce.
#include <algorithm>

#include "cvm_internal.hpp"

namespace cvm {

namespace {
bool eval(GateKind k, bool a, bool b) {
  switch (k) {
    case GateKind::Nand: return !(a && b);
    case GateKind::And: return a && b;
    case GateKind::Or: return a || b;
    case GateKind::Xor: return a != b;
    case GateKind::Xnor: return a == b;
    case GateKind::Nor: return !(a || b);
    case GateKind::AndNY: return !a && b;
    case GateKind::AndYN: return a && !b;
    case GateKind::OrNY: return !a || b;
    case GateKind::OrYN: return a || !b;
    default: throw InputError("not a bootstrapped binary gate");
  }
}
}  // namespace

bool ClearBackend::value(Bit h, const char* what) const {
  if (h == 0 || h > nodes_.size())
    throw InputError(std::string("invalid bit handle passed to ") + what);
  return values_[h - 1] != 0;
}

Bit ClearBackend::add(Node n, bool v) {
  nodes_.push_back(n);
  values_.push_back(v ? 1 : 0);
  stats_.nodes = nodes_.size();
  if (bootstrap_count(n.kind) > 0 && !n.input) {
    stats_.bootstrapped++;
    stats_.bootstraps += bootstrap_count(n.kind);
    stats_.levels_run = std::max<uint64_t>(stats_.levels_run, n.level);
  }
  return nodes_.size();
}

Bit ClearBackend::constant(bool v) {
  std::lock_guard<std::mutex> lock(mu_);
  Node n{};
  n.kind = GateKind::Constant;
  n.const_value = v;
  n.slot = -1;
  n.sign = 1;
  return add(n, v);
}

Bit ClearBackend::encrypt_bit(bool v) {
  std::lock_guard<std::mutex> lock(mu_);
  Node n{};
  n.kind = GateKind::Constant;
  n.input = true;
  n.slot = -1;
  n.sign = 1;
  return add(n, v);
}

Bit ClearBackend::unary_gate(GateKind kind, Bit a) {
  std::lock_guard<std::mutex> lock(mu_);
  if (kind != GateKind::Not && kind != GateKind::Copy) throw InputError("not a unary gate");
  const bool va = value(a, "unary_gate");
  Node n{};
  n.kind = kind;
  n.ndeps = 1;
  n.dep[0] = a;
  n.level = nodes_[a - 1].level;
  n.slot = -1;
  n.sign = 1;
  return add(n, kind == GateKind::Not ? !va : va);
}

Bit ClearBackend::binary_gate(GateKind kind, Bit a, Bit b) {
  std::lock_guard<std::mutex> lock(mu_);
  const bool va = value(a, "binary_gate"), vb = value(b, "binary_gate");
  const bool r = eval(kind, va, vb);
  Node n{};
  n.kind = kind;
  n.ndeps = 2;
  n.dep[0] = a;
  n.dep[1] = b;
  n.level = std::max(nodes_[a - 1].level, nodes_[b - 1].level) + 1;
  n.slot = -1;
  n.sign = 1;
  return add(n, r);
}

Bit ClearBackend::mux_gate(Bit s, Bit t, Bit f) {
  std::lock_guard<std::mutex> lock(mu_);
  const bool vs = value(s, "mux_gate"), vt = value(t, "mux_gate"), vf = value(f, "mux_gate");
  Node n{};
  n.kind = GateKind::Mux;
  n.ndeps = 3;
  n.dep[0] = s;
  n.dep[1] = t;
  n.dep[2] = f;
  n.level = std::max({nodes_[s - 1].level, nodes_[t - 1].level, nodes_[f - 1].level}) + 1;
  n.slot = -1;
  n.sign = 1;
  return add(n, vs ? vt : vf);
}

bool ClearBackend::decrypt_bit(Bit h) {
  std::lock_guard<std::mutex> lock(mu_);
  stats_.decrypts++;
  return value(h, "decrypt_bit");
}

void ClearBackend::push_region(std::string_view) {
  std::lock_guard<std::mutex> lock(mu_);
  ++regions_;
}
void ClearBackend::pop_region() {
  std::lock_guard<std::mutex> lock(mu_);
  if (!regions_) throw InputError("pop_region without a matching push_region");
  --regions_;
}
void ClearBackend::fence() {}

}  // namespace cvm
