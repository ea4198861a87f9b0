// Straight-line CryptoEmu machine (reference Machine, emulator.cpp:82-369):
// encrypted registers created lazily as CONSTANT-zero words, the opcode
// dispatch onto the functional units, NZCV updates, and a fence after every
// instruction.  Branches need the key owner's oracle (keyservice.cpp:146-155)
// and are rejected here; config 5 (BASELINE.json configs[4]) is branch-free.
#include <bit>
#include <string>

#include "cvm_internal.hpp"

namespace cvm {

namespace {

// cryptovm::Opcode enumerators (isa.hpp:27-55)
enum Op : uint32_t {
  Load, Store, Mov, Add, Adds, Sub, Subs, Mul, Muls, Smul, Smuls, Udiv, Lls, Lrs, Ars,
  And, Or, Xor, Orn, Not, Bfc, Bfi, Rbit, Rev, Cmp, B, Halt
};

const char* op_name(uint32_t op) {
  static const char* names[] = {"LOAD", "STORE", "MOV", "ADD", "ADDS", "SUB", "SUBS",
                                "MUL", "MULS", "SMUL", "SMULS", "UDIV", "LLS", "LRS",
                                "ARS", "AND", "OR", "XOR", "ORN", "NOT", "BFC", "BFI",
                                "RBIT", "REV", "CMP", "B", "HALT"};
  return op <= Halt ? names[op] : "?";
}

class Machine {
 public:
  Machine(Backend& bk, unsigned ws, unsigned nregs, std::vector<Word> mem)
      : bk_(bk), ws_(ws), regs_(nregs), mem_(std::move(mem)) {
    if (!std::has_single_bit(ws) || ws < 4 || ws > 64)
      throw InputError("word size must be a power of two in [4, 64]");
    if (nregs == 0) throw InputError("register count must be positive");
    for (const Word& w : mem_)
      if (w.size() != ws) throw InputError("data memory word size does not match the machine");
    Region r(bk_, "init");
    f_.n = bk_.constant(false);
    f_.z = bk_.constant(false);
    f_.c = bk_.constant(false);
    f_.v = bk_.constant(false);
  }

  const Word& reg(int i) {
    if (i < 0 || size_t(i) >= regs_.size()) throw InputError("register index out of range");
    if (regs_[i].empty()) {
      Region r(bk_, "init");
      regs_[i] = alu::constant_word(bk_, 0, ws_);
    }
    return regs_[i];
  }
  void write(int i, Word w) {
    if (i < 0 || size_t(i) >= regs_.size()) throw InputError("register index out of range");
    regs_[i] = std::move(w);
  }
  Word operand(const cvm_insn& in) {
    if (in.rm >= 0) return reg(in.rm);
    if (in.imm < 0) throw InputError("instruction is missing an operand");
    Region r(bk_, "imm");
    return alu::constant_word(bk_, uint64_t(in.imm), ws_);
  }
  Word copies(const Word& w) {
    Word o(w.size());
    for (size_t i = 0; i < w.size(); ++i) o[i] = copy_gate(bk_, w[i]);
    return o;
  }
  void flags_add(const alu::AddResult& r, const Word& a, const Word& b, bool subtraction) {
    Bit bs = subtraction ? not_gate(bk_, b.back()) : b.back();
    f_ = alu::flags(bk_, r.sum, r.carry_out, a.back(), bs);
  }

  void step(const cvm_insn& in) {
    execute(in);
    bk_.fence();
  }

  void execute(const cvm_insn& in) {
    Region r(bk_, op_name(in.op));
    switch (in.op) {
      case Halt:
        return;
      case B:
        throw InputError("branches need a branch oracle; straight-line programs only");
      case Load: {
        if (in.imm < 0 || size_t(in.imm) >= mem_.size()) throw InputError("load address out of range");
        write(in.rd, copies(mem_[size_t(in.imm)]));
        return;
      }
      case Store: {
        if (in.imm < 0 || size_t(in.imm) >= mem_.size()) throw InputError("store address out of range");
        Word w = copies(reg(in.rn));
        mem_[size_t(in.imm)] = std::move(w);
        return;
      }
      case Mov:
        if (in.imm >= 0) write(in.rd, alu::constant_word(bk_, uint64_t(in.imm), ws_));
        else write(in.rd, copies(reg(in.rn)));
        return;
      case Add:
      case Adds: {
        Word a = reg(in.rn);
        Word b = operand(in);
        alu::AddResult res = alu::add(bk_, a, b);
        write(in.rd, res.sum);
        if (in.sets_flags) {
          bk_.fence();
          flags_add(res, a, b, false);
        }
        return;
      }
      case Sub:
      case Subs:
      case Cmp: {
        Word a = reg(in.rn);
        Word b = operand(in);
        alu::AddResult res = alu::sub(bk_, a, b);
        if (in.op != Cmp) write(in.rd, res.sum);
        if (in.sets_flags) {
          bk_.fence();
          flags_add(res, a, b, true);
        }
        return;
      }
      case Mul:
      case Muls:
      case Smul:
      case Smuls: {
        Word a = reg(in.rn);
        Word b = operand(in);
        const bool sgn = in.op == Smul || in.op == Smuls;
        Word p = sgn ? alu::mul_signed(bk_, a, b) : alu::mul_unsigned(bk_, a, b);
        Word low(p.begin(), p.begin() + ws_);
        write(in.rd, low);
        if (in.sets_flags) {
          bk_.fence();
          Region fr(bk_, "flags");
          f_.n = copy_gate(bk_, low.back());
          f_.z = not_gate(bk_, alu::or_reduce(bk_, low));
        }
        return;
      }
      case Udiv: {
        Word a = reg(in.rn);
        Word b = operand(in);
        write(in.rd, alu::div_unsigned(bk_, a, b));
        return;
      }
      case Lls:
      case Lrs:
      case Ars: {
        const alu::ShiftKind k = in.op == Lls   ? alu::ShiftKind::LogicalLeft
                                 : in.op == Lrs ? alu::ShiftKind::LogicalRight
                                                : alu::ShiftKind::ArithmeticRight;
        Word v = reg(in.rn);
        if (in.rm >= 0) {
          Word amt = reg(in.rm);
          write(in.rd, alu::shift_reg(bk_, v, k, amt));
        } else {
          if (in.imm < 0) throw InputError("shift is missing an amount");
          write(in.rd, alu::shift_imm(bk_, v, k, unsigned(in.imm)));
        }
        return;
      }
      case And:
      case Or:
      case Xor:
      case Orn: {
        const alu::BitwiseKind k = in.op == And  ? alu::BitwiseKind::And
                                   : in.op == Or ? alu::BitwiseKind::Or
                                   : in.op == Xor ? alu::BitwiseKind::Xor
                                                  : alu::BitwiseKind::OrNot;
        Word a = reg(in.rn);
        Word b = operand(in);
        write(in.rd, alu::bitwise(bk_, k, a, b));
        return;
      }
      case Not:
        write(in.rd, alu::not_word(bk_, reg(in.rn)));
        return;
      // Data movement (alu.cpp:387-452): COPY / CONSTANT only, no bootstraps.
      case Bfc:
      case Bfi: {
        if (in.imm < 0 || in.imm2 < 0) throw InputError("BFC/BFI is missing its field operands");
        const size_t lsb = size_t(in.imm), width = size_t(in.imm2);
        const Word dst = reg(in.rd);
        const Word src = in.op == Bfi ? reg(in.rn) : Word{};
        if (width == 0 || lsb + width > ws_) throw InputError("bit field out of range");
        Region fr(bk_, in.op == Bfc ? "bfc" : "bfi");
        Word out(ws_);
        for (size_t i = 0; i < ws_; ++i) {
          const bool field = i >= lsb && i < lsb + width;
          if (in.op == Bfc) out[i] = field ? bk_.constant(false) : copy_gate(bk_, dst[i]);
          else out[i] = field ? copy_gate(bk_, src[i - lsb]) : copy_gate(bk_, dst[i]);
        }
        write(in.rd, out);
        return;
      }
      case Rbit:
      case Rev: {
        const Word w = reg(in.rn);
        if (in.op == Rev && ws_ % 8) throw InputError("rev: width must be a multiple of 8");
        Region fr(bk_, in.op == Rbit ? "rbit" : "rev");
        Word out(ws_);
        for (size_t i = 0; i < ws_; ++i) {
          const size_t src = in.op == Rbit ? ws_ - 1 - i : (ws_ / 8 - 1 - i / 8) * 8 + i % 8;
          out[i] = copy_gate(bk_, w[src]);
        }
        write(in.rd, out);
        return;
      }
      default:
        throw InputError("unknown opcode " + std::to_string(in.op));
    }
  }

  std::vector<Word> regs_out() {
    std::vector<Word> out;
    for (size_t i = 0; i < regs_.size(); ++i) out.push_back(reg(int(i)));
    return out;
  }
  const alu::Flags& nzcv() const { return f_; }

 private:
  Backend& bk_;
  unsigned ws_;
  std::vector<Word> regs_;
  std::vector<Word> mem_;
  alu::Flags f_{};
};

}  // namespace

void machine_run(Backend& bk, unsigned word_size, unsigned register_count,
                 const std::vector<Word>& memory, const cvm_insn* program, uint32_t count,
                 std::vector<Word>* regs, alu::Flags* nzcv) {
  Machine m(bk, word_size, register_count, memory);
  for (uint32_t i = 0; i < count; ++i) {
    if (program[i].op == Halt) break;
    m.step(program[i]);
  }
  if (regs) *regs = m.regs_out();
  if (nzcv) *nzcv = m.nzcv();
}

}  // namespace cvm
