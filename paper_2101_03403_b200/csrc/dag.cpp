// Circuit replay: a gate table in the shape of the reference's GateDag
// (DagNode, proj/core/include/cryptovm/dag.hpp:33-42; ids assigned by
// GateDag::append, dag.cpp:57-73) is re-issued, node by node, as Backend calls
// on the device backend.  The circuits themselves are recorded by the
// reference's own functional units / emulator on the reference side of the
// boundary (integration/) -- this library holds no copy of
// them.
#include <string>

#include "cvm_internal.hpp"

namespace cvm {

void validate_dag(const cvm_dag_node* nodes, uint64_t n, uint64_t* n_inputs) {
  if (n && !nodes) throw InputError("null dag nodes");
  uint64_t inputs = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const cvm_dag_node& d = nodes[i];
    const std::string at = " at dag node " + std::to_string(i + 1);
    if (d.kind > uint8_t(GateKind::Mux)) throw InputError("unknown gate kind" + at);
    if (d.input) {
      if (d.ndeps) throw InputError("input node with dependencies" + at);
      ++inputs;
      continue;
    }
    const GateKind k = GateKind(d.kind);
    const unsigned want = k == GateKind::Constant                        ? 0
                          : (k == GateKind::Not || k == GateKind::Copy) ? 1
                          : k == GateKind::Mux                          ? 3
                                                                        : 2;
    if (d.ndeps != want) throw InputError("wrong dependency count" + at);
    for (unsigned j = 0; j < want; ++j)
      if (d.dep[j] == 0 || d.dep[j] > i) throw InputError("dependency out of order" + at);
  }
  if (n_inputs) *n_inputs = inputs;
}

void replay_dag(Backend& bk, const cvm_dag_node* nodes, uint64_t n, const Bit* inputs,
                uint64_t n_inputs, Bit* handles) {
  uint64_t need = 0;
  validate_dag(nodes, n, &need);
  if (need != n_inputs)
    throw InputError("dag has " + std::to_string(need) + " input nodes, " +
                     std::to_string(n_inputs) + " inputs given");
  if (n && !handles) throw InputError("null handle output");
  if (auto* gpu = dynamic_cast<GpuBackend*>(&bk)) {
    gpu->replay(nodes, n, inputs, handles);  // one lock for the whole table
    return;
  }
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const cvm_dag_node& d = nodes[i];
    const GateKind kind = GateKind(d.kind);
    Bit h;
    if (d.input) {
      h = inputs[k++];
    } else if (kind == GateKind::Constant) {
      h = bk.constant(d.value != 0);
    } else if (kind == GateKind::Not || kind == GateKind::Copy) {
      h = bk.unary_gate(kind, handles[d.dep[0] - 1]);
    } else if (kind == GateKind::Mux) {
      h = bk.mux_gate(handles[d.dep[0] - 1], handles[d.dep[1] - 1], handles[d.dep[2] - 1]);
    } else {
      h = bk.binary_gate(kind, handles[d.dep[0] - 1], handles[d.dep[1] - 1]);
    }
    handles[i] = h;
  }
}

}  // namespace cvm
