// Golden-vector driver: runs the UNMODIFIED reference core (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref) and prints
// the gate DAGs and cleartext results its SimBackend produces.
//
// Test infrastructure only -- consumed by tests/golden/make_golden.py, never by
// the product.  Output is a line-oriented text format:
//
//   DAG <op> <width>                       one functional-unit instance
//   N <kind> <input> <ndeps> <d0> <d1> <d2> <const>  one line per DAG node,
//                                          id = line index+1
//   OUT <id> ...                            output node ids (LSB first)
//   VEC <op> <width> <a> <b> <c> <result>   seeded / fixed cleartext vectors
//   PROG <seed> ...                         config-5 program + final state
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "cryptovm/alu.hpp"
#include "cryptovm/emulator.hpp"
#include "cryptovm/isa.hpp"
#include "cryptovm/keyservice.hpp"
#include "cryptovm/sim_backend.hpp"
#include "cryptovm/word.hpp"

using namespace cryptovm;

namespace {

// Forwards every call to a SimBackend and remembers the value of each
// CONSTANT node (the DAG itself does not store it, dag.hpp:33-42).
class Tap final : public Backend {
 public:
  SimBackend sim;
  std::vector<int> const_value;  // indexed by node id
  BitHandle constant(bool value) override {
    BitHandle h = sim.constant(value);
    note(h, value);
    return h;
  }
  BitHandle unary_gate(GateKind kind, BitHandle a) override {
    return sim.unary_gate(kind, a);
  }
  BitHandle binary_gate(GateKind kind, BitHandle a, BitHandle b) override {
    return sim.binary_gate(kind, a, b);
  }
  BitHandle mux_gate(BitHandle s, BitHandle t, BitHandle f) override {
    return sim.mux_gate(s, t, f);
  }
  BitHandle encrypt_bit(bool value) override { return sim.encrypt_bit(value); }
  bool decrypt_bit(BitHandle bit) override { return sim.decrypt_bit(bit); }
  std::vector<std::uint8_t> export_bit(BitHandle bit) override {
    return sim.export_bit(bit);
  }
  BitHandle import_bit(const std::vector<std::uint8_t>& blob) override {
    return sim.import_bit(blob);
  }
  void push_region(std::string_view name) override { sim.push_region(name); }
  void pop_region() override { sim.pop_region(); }
  void fence() override { sim.fence(); }
  const GateDag& dag() const { return sim.dag(); }

 private:
  void note(BitHandle h, bool v) {
    if (const_value.size() <= h.node()) const_value.resize(h.node() + 1, 0);
    const_value[h.node()] = v ? 1 : 0;
  }
};

void dump_dag(const Tap& tap) {
  const GateDag& dag = tap.dag();
  for (const DagNode& n : dag.nodes()) {
    int value = n.id < tap.const_value.size() ? tap.const_value[n.id] : 0;
    std::printf("N %d %d %d %llu %llu %llu %d\n", static_cast<int>(n.kind),
                n.input ? 1 : 0, n.dep_count,
                static_cast<unsigned long long>(n.dep[0]),
                static_cast<unsigned long long>(n.dep[1]),
                static_cast<unsigned long long>(n.dep[2]), value);
  }
}

void dump_out(const std::vector<BitHandle>& bits) {
  std::printf("OUT");
  for (const BitHandle& b : bits) {
    std::printf(" %llu", static_cast<unsigned long long>(b.node()));
  }
  std::printf("\n");
}

std::uint64_t mask_of(unsigned w) {
  return w >= 64 ? ~0ull : ((1ull << w) - 1);
}

// Builds one FU instance on `bk` with operands (a, b, c) already encrypted.
std::vector<BitHandle> build(Backend& bk, const std::string& op, const Word& a,
                             const Word& b, BitHandle c) {
  std::vector<BitHandle> out;
  auto append = [&](const Word& w) {
    out.insert(out.end(), w.bits().begin(), w.bits().end());
  };
  if (op == "add") {
    auto r = alu::add(bk, a, b);
    append(r.sum);
    out.push_back(r.carry_out);
  } else if (op == "add_cin") {
    auto r = alu::add(bk, a, b, c);
    append(r.sum);
    out.push_back(r.carry_out);
  } else if (op == "sub") {
    auto r = alu::sub(bk, a, b);
    append(r.sum);
    out.push_back(r.carry_out);
  } else if (op == "addsub") {
    auto r = alu::add_sub_select(bk, a, b, c);
    append(r.sum);
    out.push_back(r.carry_out);
  } else if (op == "cmp") {
    // SUBS/CMP as the emulator issues it (emulator.cpp:258-270,168-175).
    auto r = alu::sub(bk, a, b);
    bk.fence();
    BitHandle b_sign = not_gate(bk, b.msb());
    alu::Flags f = alu::flags(bk, r.sum, r.carry_out, a.msb(), b_sign);
    append(r.sum);
    out.push_back(f.n);
    out.push_back(f.z);
    out.push_back(f.c);
    out.push_back(f.v);
  } else if (op == "and" || op == "orr" || op == "eor" || op == "orn") {
    alu::BitwiseKind k = op == "and"   ? alu::BitwiseKind::And
                         : op == "orr" ? alu::BitwiseKind::Or
                         : op == "eor" ? alu::BitwiseKind::Xor
                                       : alu::BitwiseKind::OrNot;
    append(alu::bitwise(bk, k, a, b));
  } else if (op == "lsl" || op == "lsr" || op == "asr") {
    alu::ShiftKind k = op == "lsl"   ? alu::ShiftKind::LogicalLeft
                       : op == "lsr" ? alu::ShiftKind::LogicalRight
                                     : alu::ShiftKind::ArithmeticRight;
    append(alu::shift_reg(bk, a, k, b));
  } else if (op == "umul") {
    append(alu::mul_unsigned(bk, a, b));
  } else if (op == "smul") {
    append(alu::mul_signed(bk, a, b));
  } else if (op == "udiv") {
    append(alu::div_unsigned(bk, a, b));
  } else if (op == "udiv_exact") {
    append(alu::div_unsigned(bk, a, b, alu::DivAccumulator::Exact));
  } else {
    std::fprintf(stderr, "unknown op %s\n", op.c_str());
    std::exit(2);
  }
  return out;
}

bool uses_c(const std::string& op) { return op == "add_cin" || op == "addsub"; }

void cmd_dag(const std::string& op, unsigned w) {
  Tap bk;
  Word a = Word::encrypt(bk, 0, w);
  Word b = Word::encrypt(bk, 0, w);
  BitHandle c = uses_c(op) ? bk.encrypt_bit(false) : BitHandle{};
  std::vector<BitHandle> out = build(bk, op, a, b, c);
  std::printf("DAG %s %u %zu\n", op.c_str(), w, bk.dag().size());
  dump_dag(bk);
  dump_out(out);
}

void cmd_vectors(const std::string& op, unsigned w, std::uint64_t seed,
                 int count, bool exhaustive) {
  std::mt19937_64 rng(seed);
  const std::uint64_t m = mask_of(w);
  auto run_one = [&](std::uint64_t av, std::uint64_t bv, std::uint64_t cv) {
    SimBackend bk;
    Word a = Word::encrypt(bk, av, w);
    Word b = Word::encrypt(bk, bv, w);
    BitHandle c = uses_c(op) ? bk.encrypt_bit(cv != 0) : BitHandle{};
    std::vector<BitHandle> out = build(bk, op, a, b, c);
    std::printf("VEC %s %u %llu %llu %llu", op.c_str(), w,
                static_cast<unsigned long long>(av),
                static_cast<unsigned long long>(bv),
                static_cast<unsigned long long>(cv));
    // Results as bit string (LSB first), outputs may exceed 64 bits.
    std::printf(" ");
    for (const BitHandle& h : out) std::printf("%d", bk.decrypt_bit(h) ? 1 : 0);
    std::printf("\n");
  };
  if (exhaustive) {
    for (std::uint64_t av = 0; av <= m; ++av)
      for (std::uint64_t bv = 0; bv <= m; ++bv)
        for (std::uint64_t cv = 0; cv <= (uses_c(op) ? 1u : 0u); ++cv)
          run_one(av, bv, cv);
    return;
  }
  for (int i = 0; i < count; ++i) {
    std::uint64_t av = rng() & m, bv = rng() & m, cv = rng() & 1;
    run_one(av, bv, cv);
  }
}

// Config 5 (BASELINE.json configs[4]): 8 encrypted 16-bit registers loaded
// from a seeded BufferMemory, 64 instructions uniform over
// {ADD, SUB, AND, ORR, EOR, LSL, LSR, MUL, CMP}, then one UDIV whose divisor
// register is nonzero (chosen from a cleartext pre-run on SimBackend).
void cmd_program(std::uint64_t seed, int count) {
  const unsigned w = 16;
  std::mt19937_64 rng(seed);
  std::vector<std::uint64_t> mem(8);
  for (auto& v : mem) v = rng() & 0xFFFF;
  Program p;
  p.word_size = w;
  for (int r = 0; r < 8; ++r) {
    Instruction insn;
    insn.op = Opcode::Load;
    insn.rd = r;
    insn.imm = static_cast<std::uint64_t>(r);
    p.instructions.push_back(insn);
  }
  const Opcode ops[9] = {Opcode::Add, Opcode::Sub, Opcode::And,
                         Opcode::Or,  Opcode::Xor, Opcode::Lls,
                         Opcode::Lrs, Opcode::Mul, Opcode::Cmp};
  for (int i = 0; i < count; ++i) {
    Instruction insn;
    insn.op = ops[rng() % 9];
    int rd = static_cast<int>(rng() % 8);
    int rn = static_cast<int>(rng() % 8);
    int rm = static_cast<int>(rng() % 8);
    if (insn.op != Opcode::Cmp) insn.rd = rd;
    insn.rn = rn;
    insn.rm = rm;
    insn.sets_flags = opcode_sets_flags(insn.op);
    p.instructions.push_back(insn);
  }
  auto make_mem = [&](Backend& bk) {
    std::vector<Word> words;
    for (auto v : mem) words.push_back(Word::encrypt(bk, v, w));
    return std::make_unique<BufferMemory>(w, std::move(words));
  };
  // Cleartext pre-run to pick a nonzero divisor register.
  std::vector<std::uint64_t> pre(8);
  {
    SimBackend bk;
    LocalBranchOracle oracle(bk);
    Machine m(bk, {.word_size = w, .register_count = 8}, make_mem(bk), oracle);
    m.run(p, p.instructions.size() + 1);
    for (unsigned r = 0; r < 8; ++r) pre[r] = decrypt_word(bk, m.reg(r));
  }
  std::vector<int> nonzero;
  for (int r = 0; r < 8; ++r)
    if (pre[r] != 0) nonzero.push_back(r);
  Instruction div;
  div.op = Opcode::Udiv;
  div.rd = static_cast<int>(rng() % 8);
  div.rn = static_cast<int>(rng() % 8);
  div.rm = nonzero.empty() ? 0 : nonzero[rng() % nonzero.size()];
  div.sets_flags = false;
  p.instructions.push_back(div);

  Tap bk;
  LocalBranchOracle oracle(bk);
  Machine m(bk, {.word_size = w, .register_count = 8}, make_mem(bk), oracle);
  m.run(p, p.instructions.size() + 1);
  std::printf("PROG %llu %zu\n", static_cast<unsigned long long>(seed),
              p.instructions.size());
  std::printf("MEM");
  for (auto v : mem) std::printf(" %llu", static_cast<unsigned long long>(v));
  std::printf("\n");
  for (const Instruction& insn : p.instructions) {
    std::printf("I %s %d %d %d %lld %d\n", std::string(opcode_name(insn.op)).c_str(),
                insn.rd, insn.rn, insn.rm,
                insn.imm ? static_cast<long long>(*insn.imm) : -1LL,
                insn.sets_flags ? 1 : 0);
  }
  std::printf("REGS");
  std::vector<BitHandle> outs;
  for (unsigned r = 0; r < 8; ++r) {
    const Word& reg = m.reg(r);
    std::printf(" %llu", static_cast<unsigned long long>(decrypt_word(bk, reg)));
    outs.insert(outs.end(), reg.bits().begin(), reg.bits().end());
  }
  std::printf("\n");
  const alu::Flags& f = m.flags();
  std::printf("NZCV %d %d %d %d\n", bk.decrypt_bit(f.n), bk.decrypt_bit(f.z),
              bk.decrypt_bit(f.c), bk.decrypt_bit(f.v));
  outs.push_back(f.n);
  outs.push_back(f.z);
  outs.push_back(f.c);
  outs.push_back(f.v);
  std::printf("DAG program %u %zu\n", w, bk.dag().size());
  dump_dag(bk);
  dump_out(outs);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: ref_golden dag OP W | vec OP W SEED COUNT | exh OP W | one OP W A B C "
                 "| prog SEED COUNT\n");
    return 2;
  }
  std::string cmd = argv[1];
  if (cmd == "dag" && argc == 4) {
    cmd_dag(argv[2], static_cast<unsigned>(std::atoi(argv[3])));
  } else if (cmd == "vec" && argc == 6) {
    cmd_vectors(argv[2], static_cast<unsigned>(std::atoi(argv[3])),
                std::strtoull(argv[4], nullptr, 10), std::atoi(argv[5]), false);
  } else if (cmd == "one" && argc == 7) {
    // one fixed example: ref_golden one OP W A B C
    const std::string op = argv[2];
    const unsigned w = static_cast<unsigned>(std::atoi(argv[3]));
    SimBackend bk;
    Word a = Word::encrypt(bk, std::strtoull(argv[4], nullptr, 10), w);
    Word b = Word::encrypt(bk, std::strtoull(argv[5], nullptr, 10), w);
    BitHandle c = uses_c(op) ? bk.encrypt_bit(std::atoi(argv[6]) != 0) : BitHandle{};
    std::vector<BitHandle> out = build(bk, op, a, b, c);
    std::printf("VEC %s %u %s %s %s ", op.c_str(), w, argv[4], argv[5], argv[6]);
    for (const BitHandle& h : out) std::printf("%d", bk.decrypt_bit(h) ? 1 : 0);
    std::printf("\n");
  } else if (cmd == "exh" && argc == 4) {
    cmd_vectors(argv[2], static_cast<unsigned>(std::atoi(argv[3])), 0, 0, true);
  } else if (cmd == "prog" && argc == 4) {
    cmd_program(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]));
  } else {
    std::fprintf(stderr, "bad arguments\n");
    return 2;
  }
  return 0;
}
