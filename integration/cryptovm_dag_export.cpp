// See cryptovm_dag_export.hpp.
#include "cryptovm_dag_export.hpp"

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "cryptovm/alu.hpp"
#include "cryptovm/emulator.hpp"
#include "cryptovm/errors.hpp"
#include "cryptovm/isa.hpp"
#include "cryptovm/keyservice.hpp"
#include "cryptovm/word.hpp"
#include "cryptovm_gpu_backend.hpp"

namespace cryptovm {

BitHandle DagRecorder::constant(bool value) {
  BitHandle h = sim_.constant(value);
  if (const_value_.size() <= h.node()) const_value_.resize(h.node() + 1, 0);
  const_value_[h.node()] = value ? 1 : 0;
  return h;
}
BitHandle DagRecorder::unary_gate(GateKind kind, BitHandle a) { return sim_.unary_gate(kind, a); }
BitHandle DagRecorder::binary_gate(GateKind kind, BitHandle a, BitHandle b) {
  return sim_.binary_gate(kind, a, b);
}
BitHandle DagRecorder::mux_gate(BitHandle s, BitHandle t, BitHandle f) {
  return sim_.mux_gate(s, t, f);
}
BitHandle DagRecorder::encrypt_bit(bool value) { return sim_.encrypt_bit(value); }
bool DagRecorder::decrypt_bit(BitHandle bit) { return sim_.decrypt_bit(bit); }
std::vector<std::uint8_t> DagRecorder::export_bit(BitHandle bit) { return sim_.export_bit(bit); }
BitHandle DagRecorder::import_bit(const std::vector<std::uint8_t>& blob) {
  return sim_.import_bit(blob);
}
void DagRecorder::push_region(std::string_view name) { sim_.push_region(name); }
void DagRecorder::pop_region() { sim_.pop_region(); }
void DagRecorder::fence() { sim_.fence(); }

std::vector<cvm_dag_node> DagRecorder::table() const {
  const GateDag& dag = sim_.dag();
  std::vector<cvm_dag_node> t(dag.size());
  for (std::size_t i = 0; i < dag.size(); ++i) {
    const DagNode& n = dag.node_at(i);
    cvm_dag_node& d = t[i];
    d.kind = static_cast<std::uint8_t>(n.kind);
    d.input = n.input ? 1 : 0;
    d.ndeps = n.dep_count;
    d.value = n.id < const_value_.size() ? const_value_[n.id] : 0;
    d.region = n.region;
    for (int j = 0; j < 3; ++j) d.dep[j] = n.dep[j];
  }
  return t;
}

}  // namespace cryptovm

using namespace cryptovm;

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
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CVM_E_INPUT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CVM_E_DEVICE;
  }
}

bool uses_c(const std::string& op) { return op == "add_cin" || op == "addsub"; }

// One functional-unit instance on `bk` over operands already entered (the
// calls the reference's own tests and emulator make).
std::vector<BitHandle> build_fu(Backend& bk, const std::string& op, unsigned width,
                                const Word& a, const Word& b, BitHandle c) {
  std::vector<BitHandle> out;
  auto append = [&](const Word& w) { out.insert(out.end(), w.bits().begin(), w.bits().end()); };
  auto add_result = [&](const alu::AddResult& r) {
    append(r.sum);
    out.push_back(r.carry_out);
  };
  if (op == "add") {
    add_result(alu::add(bk, a, b));
  } else if (op == "add_cin") {
    add_result(alu::add(bk, a, b, c));
  } else if (op == "sub") {
    add_result(alu::sub(bk, a, b));
  } else if (op == "addsub") {
    add_result(alu::add_sub_select(bk, a, b, c));
  } else if (op == "cmp") {
    // SUBS / CMP as the emulator issues it (emulator.cpp:258-270, 168-175):
    // subtraction, then NZCV with the complemented b sign.
    const alu::AddResult r = alu::sub(bk, a, b);
    bk.fence();
    const BitHandle b_sign = not_gate(bk, b.msb());
    const alu::Flags f = alu::flags(bk, r.sum, r.carry_out, a.msb(), b_sign);
    append(r.sum);
    out.insert(out.end(), {f.n, f.z, f.c, f.v});
  } else if (op == "and" || op == "orr" || op == "eor" || op == "orn") {
    const alu::BitwiseKind k = op == "and"   ? alu::BitwiseKind::And
                               : op == "orr" ? alu::BitwiseKind::Or
                               : op == "eor" ? alu::BitwiseKind::Xor
                                             : alu::BitwiseKind::OrNot;
    append(alu::bitwise(bk, k, a, b));
  } else if (op == "lsl" || op == "lsr" || op == "asr") {
    const alu::ShiftKind k = op == "lsl"   ? alu::ShiftKind::LogicalLeft
                             : op == "lsr" ? alu::ShiftKind::LogicalRight
                                           : alu::ShiftKind::ArithmeticRight;
    append(alu::shift_reg(bk, a, k, b));
  } else if (op == "umul") {
    append(alu::mul_unsigned(bk, a, b));
  } else if (op == "smul") {
    append(alu::mul_signed(bk, a, b));
  } else if (op == "mul_lo") {
    // MUL as the emulator issues it: the low half of the product
    // (emulator.cpp:271-285).
    const Word p = alu::mul_unsigned(bk, a, b);
    out.assign(p.bits().begin(), p.bits().begin() + width);
  } else if (op == "udiv") {
    append(alu::div_unsigned(bk, a, b));
  } else if (op == "udiv_exact") {
    append(alu::div_unsigned(bk, a, b, alu::DivAccumulator::Exact));
  } else {
    throw InputError("unknown functional-unit op '" + op + "'");
  }
  return out;
}

void fill(const DagRecorder& rec, const std::vector<BitHandle>& outs, cvmref_dag* out) {
  const std::vector<cvm_dag_node> t = rec.table();
  auto* nodes = static_cast<cvm_dag_node*>(std::malloc(sizeof(cvm_dag_node) * (t.size() + 1)));
  auto* outputs = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (outs.size() + 1)));
  if (!nodes || !outputs) {
    std::free(nodes);
    std::free(outputs);
    throw std::bad_alloc();
  }
  out->n_nodes = t.size();
  out->nodes = nodes;
  out->n_outputs = outs.size();
  out->outputs = outputs;
  std::memcpy(out->nodes, t.data(), sizeof(cvm_dag_node) * t.size());
  out->n_inputs = 0;
  for (const cvm_dag_node& n : t) out->n_inputs += n.input;
  const auto names = rec.dag().regions();
  out->n_regions = names.size();
  out->regions = static_cast<char**>(std::calloc(names.size() + 1, sizeof(char*)));
  if (!out->regions) throw std::bad_alloc();
  for (std::size_t k = 0; k < names.size(); ++k) {
    out->regions[k] = static_cast<char*>(std::malloc(names[k].size() + 1));
    if (!out->regions[k]) throw std::bad_alloc();
    std::memcpy(out->regions[k], names[k].c_str(), names[k].size() + 1);
  }
  for (std::size_t i = 0; i < outs.size(); ++i) out->outputs[i] = outs[i].node();
}

Program to_program(unsigned word_size, const cvmref_insn* p, uint64_t n) {
  Program prog;
  prog.word_size = word_size;
  for (uint64_t i = 0; i < n; ++i) {
    const cvmref_insn& x = p[i];
    Instruction insn;
    const std::string op(x.op, strnlen(x.op, sizeof(x.op)));
    const auto code = opcode_from_name(op);
    if (!code) throw InputError("unknown opcode '" + op + "'");
    insn.op = *code;
    const std::string cond(x.cond, strnlen(x.cond, sizeof(x.cond)));
    if (!cond.empty()) {
      const auto cc = cond_from_name(cond);
      if (!cc) throw InputError("unknown condition '" + cond + "'");
      insn.cond = *cc;
    }
    insn.rd = x.rd;
    insn.rn = x.rn;
    insn.rm = x.rm;
    if (x.has_imm) insn.imm = x.imm;
    if (x.has_imm2) insn.imm2 = x.imm2;
    if (x.has_target) insn.target = x.target;
    insn.sets_flags = x.sets_flags != 0;
    prog.instructions.push_back(insn);
  }
  return prog;
}

// Refuses branch queries: recording runs without the key owner.
class NoBranches final : public BranchOracle {
 public:
  BranchDecision resolve(CondCode, const alu::Flags&, std::uint32_t, std::uint32_t) override {
    throw InputError("branches need the key owner's oracle; record straight-line programs");
  }
};

}  // namespace

extern "C" {

const char* cvmref_last_error(void) { return g_err.c_str(); }

int cvmref_record_fu(const char* op, unsigned width, cvmref_dag* out) {
  return guard([&] {
    if (!op || !out) throw InputError("null argument");
    if (width == 0 || width > 64) throw InputError("width must be 1..64");
    DagRecorder rec;
    const std::string o(op);
    const Word a = Word::encrypt(rec, 0, width);
    const Word b = Word::encrypt(rec, 0, width);
    const BitHandle c = uses_c(o) ? rec.encrypt_bit(false) : BitHandle{};
    fill(rec, build_fu(rec, o, width, a, b, c), out);
  });
}

int cvmref_record_program(unsigned word_size, unsigned register_count, uint64_t n_mem,
                          const cvmref_insn* program, uint64_t n_insn, cvmref_dag* out) {
  return guard([&] {
    if (!out || (n_insn && !program)) throw InputError("null argument");
    const Program prog = to_program(word_size, program, n_insn);
    DagRecorder rec;
    std::vector<Word> words;
    for (uint64_t i = 0; i < n_mem; ++i) words.push_back(Word::encrypt(rec, 0, word_size));
    NoBranches oracle;
    Machine m(rec, {.word_size = word_size, .register_count = register_count},
              std::make_unique<BufferMemory>(word_size, std::move(words)), oracle);
    m.run(prog, prog.instructions.size() + 1);
    std::vector<BitHandle> outs;
    for (unsigned r = 0; r < register_count; ++r) {
      const Word& w = m.reg(r);
      outs.insert(outs.end(), w.bits().begin(), w.bits().end());
    }
    const alu::Flags& f = m.flags();
    outs.insert(outs.end(), {f.n, f.z, f.c, f.v});
    fill(rec, outs, out);
  });
}

void cvmref_dag_free(cvmref_dag* d) {
  if (!d) return;
  std::free(d->nodes);
  std::free(d->outputs);
  if (d->regions)
    for (uint64_t k = 0; k < d->n_regions; ++k) std::free(d->regions[k]);
  std::free(d->regions);
  d->nodes = nullptr;
  d->outputs = nullptr;
  d->regions = nullptr;
}

int cvmref_sim_program(unsigned word_size, unsigned register_count, const uint64_t* mem,
                       uint64_t n_mem, const cvmref_insn* program, uint64_t n_insn,
                       uint64_t max_steps, uint64_t* regs_out, uint8_t* nzcv_out) {
  return guard([&] {
    if ((n_mem && !mem) || (n_insn && !program) || !regs_out || !nzcv_out)
      throw InputError("null argument");
    const Program prog = to_program(word_size, program, n_insn);
    SimBackend bk;
    std::vector<Word> words;
    for (uint64_t i = 0; i < n_mem; ++i) words.push_back(Word::encrypt(bk, mem[i], word_size));
    LocalBranchOracle oracle(bk);
    Machine m(bk, {.word_size = word_size, .register_count = register_count},
              std::make_unique<BufferMemory>(word_size, std::move(words)), oracle);
    m.run(prog, max_steps);
    for (unsigned r = 0; r < register_count; ++r) regs_out[r] = decrypt_word(bk, m.reg(r));
    const alu::Flags& f = m.flags();
    nzcv_out[0] = bk.decrypt_bit(f.n);
    nzcv_out[1] = bk.decrypt_bit(f.z);
    nzcv_out[2] = bk.decrypt_bit(f.c);
    nzcv_out[3] = bk.decrypt_bit(f.v);
  });
}

int cvmref_sim_fu_batch(const char* op, unsigned width, uint64_t batch, const uint64_t* a,
                        const uint64_t* b, const uint64_t* c, uint64_t* out, double* seconds,
                        uint64_t* nodes) {
  return guard([&] {
    if (!op || (batch && (!a || !b || !out))) throw InputError("null argument");
    const std::string o(op);
    if (uses_c(o) && batch && !c) throw InputError("null carry / select operand");
    const auto t0 = std::chrono::steady_clock::now();
    SimBackend bk;
    for (uint64_t i = 0; i < batch; ++i) {
      const Word x = Word::encrypt(bk, a[i], width), y = Word::encrypt(bk, b[i], width);
      const BitHandle z = uses_c(o) ? bk.encrypt_bit(c[i] != 0) : BitHandle{};
      const std::vector<BitHandle> r = build_fu(bk, o, width, x, y, z);
      if (r.size() > 64) throw InputError("output wider than 64 bits");
      out[i] = decrypt_word(bk, Word(r));
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (nodes) *nodes = bk.dag().size();
  });
}

int cvmref_add_batch_gpu(cvm_ctx* ctx, const cvm_keyset* owner, unsigned width, uint64_t batch,
                         const uint64_t* a, const uint64_t* b, uint64_t* sums, uint8_t* carries,
                         cvm_backend_stats* stats) {
  return guard([&] {
    if (!ctx || !owner || (batch && (!a || !b || !sums))) throw InputError("null argument");
    GpuBackend bk(ctx, owner);
    std::vector<alu::AddResult> res;
    res.reserve(batch);
    std::vector<BitHandle> all;
    for (uint64_t i = 0; i < batch; ++i) {
      const Word x = Word::encrypt(bk, a[i], width), y = Word::encrypt(bk, b[i], width);
      res.push_back(alu::add(bk, x, y));
      all.insert(all.end(), res.back().sum.bits().begin(), res.back().sum.bits().end());
      all.push_back(res.back().carry_out);
    }
    bk.evaluate(all);  // one demand-driven flush for every result bit
    for (uint64_t i = 0; i < batch; ++i) {
      sums[i] = decrypt_word(bk, res[i].sum);
      const bool c = bk.decrypt_bit(res[i].carry_out);
      if (carries) carries[i] = c ? 1 : 0;
    }
    if (stats) *stats = bk.stats();
  });
}

int cvmref_run_program_gpu(cvm_ctx* ctx, const cvm_keyset* owner, unsigned word_size,
                           unsigned register_count, const uint64_t* mem, uint64_t n_mem,
                           const cvmref_insn* program, uint64_t n_insn, uint64_t max_steps,
                           uint64_t* regs_out, uint8_t* nzcv_out, cvm_backend_stats* stats,
                           uint64_t* branch_queries) {
  return guard([&] {
    if (!ctx || !owner || (n_mem && !mem) || (n_insn && !program))
      throw InputError("null argument");
    const Program prog = to_program(word_size, program, n_insn);
    GpuBackend bk(ctx, owner);
    std::vector<Word> words;
    for (uint64_t i = 0; i < n_mem; ++i) words.push_back(Word::encrypt(bk, mem[i], word_size));
    LocalBranchOracle oracle(bk);
    Machine m(bk, {.word_size = word_size, .register_count = register_count},
              std::make_unique<BufferMemory>(word_size, std::move(words)), oracle);
    m.run(prog, max_steps);
    std::vector<BitHandle> live;
    for (unsigned r = 0; r < register_count; ++r) {
      const Word& w = m.reg(r);
      live.insert(live.end(), w.bits().begin(), w.bits().end());
    }
    const alu::Flags& f = m.flags();
    live.insert(live.end(), {f.n, f.z, f.c, f.v});
    bk.evaluate(live);  // the key owner's reads: one flush of their cone
    for (unsigned r = 0; r < register_count; ++r)
      if (regs_out) regs_out[r] = decrypt_word(bk, m.reg(r));
    if (nzcv_out) {
      nzcv_out[0] = bk.decrypt_bit(f.n);
      nzcv_out[1] = bk.decrypt_bit(f.z);
      nzcv_out[2] = bk.decrypt_bit(f.c);
      nzcv_out[3] = bk.decrypt_bit(f.v);
    }
    if (stats) *stats = bk.stats();
    if (branch_queries) *branch_queries = m.stats().branch_queries;
  });
}

}  // extern "C"
