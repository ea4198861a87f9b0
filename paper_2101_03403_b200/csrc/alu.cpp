// Functional units: the CryptoEmu ALU circuits (reference alu.hpp:68-136)
// built from Backend gate calls.  They emit the same gates, in the same
// order, with the same regions and fences as the reference circuits
// (proj/core/src/alu.cpp), so a recorded DAG is node-for-node identical to
// the reference SimBackend's (checked against tests/golden/dags.npz), and a
// GpuBackend levelises them into batched launches.
#include <bit>
#include <optional>
#include <string>

#include "cvm_internal.hpp"

namespace cvm {
namespace alu {

namespace {

struct GP {  // per-bit (generate, propagate)
  Bit g, p;
};

void same_width(const Word& a, const Word& b, const char* op) {
  if (a.empty() || b.empty()) throw InputError(std::string(op) + ": words must be non-empty");
  if (a.size() != b.size()) throw InputError(std::string(op) + ": width mismatch");
}

unsigned log2_exact(const Word& w, const char* op) {
  if (!std::has_single_bit(w.size()))
    throw InputError(std::string(op) + ": width must be a power of two");
  return unsigned(std::countr_zero(w.size()));
}

GP gp(Backend& bk, Bit a, Bit b) {
  Bit g = and_gate(bk, a, b);
  Bit p = xor_gate(bk, a, b);
  return {g, p};
}

// (g,p) o (g',p') = (g | p&g', p&p')   -- alu.cpp:110-115
GP combine(Backend& bk, const GP& hi, const GP& lo) {
  Bit through = and_gate(bk, hi.p, lo.g);
  Bit g = or_gate(bk, hi.g, through);
  Bit p = and_gate(bk, hi.p, lo.p);
  return {g, p};
}

// Kogge-Stone: gp stage, optional carry-in fold, log2(n) scan levels, sum.
AddResult kogge_stone(Backend& bk, const Word& a, const Word& b, std::optional<Bit> cin) {
  same_width(a, b, "add");
  const size_t n = a.size();
  Region adder(bk, "adder");
  std::vector<GP> pre(n);
  {
    Region st(bk, "gp");
    for (size_t i = 0; i < n; ++i) pre[i] = gp(bk, a[i], b[i]);
  }
  if (cin) {
    bk.fence();
    Region st(bk, "cin");
    Bit t = and_gate(bk, pre[0].p, *cin);
    pre[0].g = or_gate(bk, pre[0].g, t);
  }
  Word prop(n);
  for (size_t i = 0; i < n; ++i) prop[i] = pre[i].p;
  unsigned level = 1;
  for (size_t d = 1; d < n; d <<= 1, ++level) {
    bk.fence();
    Region st(bk, "carry/level" + std::to_string(level));
    std::vector<GP> nxt = pre;
    for (size_t i = d; i < n; ++i) nxt[i] = combine(bk, pre[i], pre[i - d]);
    pre.swap(nxt);
  }
  bk.fence();
  Word sum(n);
  {
    Region st(bk, "sum");
    Bit c0 = cin ? *cin : bk.constant(false);
    sum[0] = xor_gate(bk, prop[0], c0);
    for (size_t i = 1; i < n; ++i) sum[i] = xor_gate(bk, prop[i], pre[i - 1].g);
  }
  return {sum, pre[n - 1].g};
}

// One right shift of the [carry, acc, low] register chain (mul loops).
void shift_chain(Backend& bk, Word& low, Word& acc, const AddResult& partial) {
  Region st(bk, "shift");
  const size_t n = low.size();
  Word nl(n), na(n);
  for (size_t i = 0; i + 1 < n; ++i) {
    nl[i] = copy_gate(bk, low[i + 1]);
    na[i] = copy_gate(bk, partial.sum[i + 1]);
  }
  nl[n - 1] = copy_gate(bk, partial.sum[0]);
  na[n - 1] = copy_gate(bk, partial.carry_out);
  low.swap(nl);
  acc.swap(na);
}

Word concat(const Word& lo, const Word& hi) {
  Word w(lo);
  w.insert(w.end(), hi.begin(), hi.end());
  return w;
}

}  // namespace

AddResult add(Backend& bk, const Word& a, const Word& b) {
  return kogge_stone(bk, a, b, std::nullopt);
}
AddResult add(Backend& bk, const Word& a, const Word& b, Bit carry_in) {
  return kogge_stone(bk, a, b, carry_in);
}

AddResult sub(Backend& bk, const Word& a, const Word& b) {
  same_width(a, b, "sub");
  Region r(bk, "sub");
  Word nb;
  {
    Region st(bk, "not");
    nb = not_word(bk, b);
  }
  Bit one = bk.constant(true);
  return add(bk, a, nb, one);
}

AddResult add_sub_select(Backend& bk, const Word& a, const Word& b, Bit subtract) {
  same_width(a, b, "add_sub_select");
  Region r(bk, "addsub");
  Word sel;
  sel.reserve(b.size());
  {
    Region st(bk, "select");
    for (Bit x : b) sel.push_back(xor_gate(bk, x, subtract));
  }
  return add(bk, a, sel, subtract);
}

Word shift_imm(Backend& bk, const Word& w, ShiftKind kind, unsigned amount) {
  const size_t n = w.size();
  if (amount > n) throw InputError("shift_imm: amount out of range");
  Region r(bk, "shift_imm");
  Word out(n);
  for (size_t i = 0; i < n; ++i) {
    switch (kind) {
      case ShiftKind::LogicalLeft:
        out[i] = i < amount ? bk.constant(false) : copy_gate(bk, w[i - amount]);
        break;
      case ShiftKind::LogicalRight:
        out[i] = i + amount < n ? copy_gate(bk, w[i + amount]) : bk.constant(false);
        break;
      case ShiftKind::ArithmeticRight:
        out[i] = i + amount < n ? copy_gate(bk, w[i + amount]) : copy_gate(bk, w.back());
        break;
    }
  }
  return out;
}

// Barrel shifter, stage k muxes by 2^(k-1) under amount bit k-1.
Word shift_reg(Backend& bk, const Word& w, ShiftKind kind, const Word& amount) {
  same_width(w, amount, "shift_reg");
  const size_t n = w.size();
  const unsigned stages = log2_exact(w, "shift_reg");
  Region r(bk, "barrel");
  const Bit sign = w.back();
  Word cur = w;
  for (unsigned k = 1; k <= stages; ++k) {
    Region st(bk, "stage" + std::to_string(k));
    const size_t d = size_t(1) << (k - 1);
    const Bit fill = kind == ShiftKind::ArithmeticRight ? sign : bk.constant(false);
    const Bit sel = amount[k - 1];
    Word nxt(n);
    for (size_t i = 0; i < n; ++i) {
      Bit moved;
      if (kind == ShiftKind::LogicalLeft) moved = i >= d ? cur[i - d] : fill;
      else moved = i + d < n ? cur[i + d] : fill;
      nxt[i] = bk.mux_gate(sel, moved, cur[i]);
    }
    cur.swap(nxt);
  }
  return cur;
}

Word mul_unsigned(Backend& bk, const Word& a, const Word& b) {
  same_width(a, b, "mul_unsigned");
  const size_t n = a.size();
  Region r(bk, "umul");
  Word acc(n);
  {
    Region st(bk, "init");
    for (auto& x : acc) x = bk.constant(false);
  }
  Word low = b;
  for (size_t it = 0; it < n; ++it) {
    Region ri(bk, "iter" + std::to_string(it));
    Word row(n);
    {
      Region st(bk, "row");
      for (size_t i = 0; i < n; ++i) row[i] = and_gate(bk, a[i], low[0]);
    }
    AddResult partial = add(bk, acc, row);
    shift_chain(bk, low, acc, partial);
    bk.fence();
  }
  return concat(low, acc);
}

Word mul_signed(Backend& bk, const Word& a, const Word& b) {
  same_width(a, b, "mul_signed");
  const size_t n = a.size();
  if (n < 2) throw InputError("mul_signed: width must be at least 2");
  Region r(bk, "smul");
  Word acc(n);
  {
    Region st(bk, "init");
    for (auto& x : acc) x = bk.constant(false);
  }
  Word low = b;
  for (size_t it = 0; it < n; ++it) {
    Region ri(bk, "iter" + std::to_string(it));
    Word row(n);
    {
      // complemented sign-position partial products (Baugh-Wooley style)
      Region st(bk, "row");
      const bool last = it == n - 1;
      for (size_t i = 0; i < n; ++i) {
        const bool inv = last ? i != n - 1 : i == n - 1;
        row[i] = inv ? nand_gate(bk, a[i], low[0]) : and_gate(bk, a[i], low[0]);
      }
    }
    AddResult partial = add(bk, acc, row);
    shift_chain(bk, low, acc, partial);
    bk.fence();
  }
  {
    Region st(bk, "correction");
    Word off = constant_word(bk, uint64_t(1) | (uint64_t(1) << (n - 1)), unsigned(n));
    acc = add(bk, acc, off).sum;
  }
  bk.fence();
  return concat(low, acc);
}

// Non-restoring division over an (n+2)-bit (Widened) or n-bit accumulator.
Word div_unsigned(Backend& bk, const Word& dividend, const Word& divisor,
                  DivAccumulator mode) {
  same_width(dividend, divisor, "div_unsigned");
  const size_t n = dividend.size();
  const size_t aw = mode == DivAccumulator::Widened ? n + 2 : n;
  Region r(bk, "udiv");
  Word acc(aw);
  Word dext = divisor;
  {
    Region st(bk, "init");
    for (auto& x : acc) x = bk.constant(false);
    for (size_t i = n; i < aw; ++i) dext.push_back(bk.constant(false));
  }
  Word q = dividend;
  for (size_t it = 0; it < n; ++it) {
    Region ri(bk, "iter" + std::to_string(it));
    Word na(aw), nq(n);
    {
      Region st(bk, "shift");
      na[0] = copy_gate(bk, q[n - 1]);
      for (size_t i = 1; i < aw; ++i) na[i] = copy_gate(bk, acc[i - 1]);
      for (size_t i = 1; i < n; ++i) nq[i] = copy_gate(bk, q[i - 1]);
    }
    Bit subtract = not_gate(bk, na[aw - 1]);
    acc = add_sub_select(bk, na, dext, subtract).sum;
    nq[0] = not_gate(bk, acc[aw - 1]);
    q.swap(nq);
    bk.fence();
  }
  return q;
}

Word bitwise(Backend& bk, BitwiseKind kind, const Word& a, const Word& b) {
  same_width(a, b, "bitwise");
  GateKind g = kind == BitwiseKind::And   ? GateKind::And
               : kind == BitwiseKind::Or  ? GateKind::Or
               : kind == BitwiseKind::Xor ? GateKind::Xor
                                          : GateKind::OrYN;
  Region r(bk, "bitwise");
  Word out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = bk.binary_gate(g, a[i], b[i]);
  return out;
}

Word not_word(Backend& bk, const Word& a) {
  Word out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = not_gate(bk, a[i]);
  return out;
}

Word constant_word(Backend& bk, uint64_t value, unsigned width) {
  if (width < 1 || width > 64) throw InputError("word width must be in [1, 64]");
  if (width < 64 && (value >> width) != 0) throw InputError("value does not fit");
  Word w(width);
  for (unsigned i = 0; i < width; ++i) w[i] = bk.constant((value >> i) & 1);
  return w;
}

Bit or_reduce(Backend& bk, const Word& w) {
  if (w.empty()) throw InputError("or_reduce: empty word");
  Word layer = w;
  while (layer.size() > 1) {
    Word nxt;
    nxt.reserve((layer.size() + 1) / 2);
    for (size_t i = 0; i + 1 < layer.size(); i += 2) nxt.push_back(or_gate(bk, layer[i], layer[i + 1]));
    if (layer.size() % 2) nxt.push_back(layer.back());
    layer.swap(nxt);
  }
  return layer[0];
}

Flags flags(Backend& bk, const Word& result, Bit carry_out, Bit a_msb, Bit b_msb) {
  Region r(bk, "flags");
  Flags f;
  f.n = copy_gate(bk, result.back());
  f.c = copy_gate(bk, carry_out);
  {
    Region st(bk, "z");
    f.z = not_gate(bk, or_reduce(bk, result));
  }
  {
    Region st(bk, "v");
    const Bit s = result.back();
    Bit both_neg = and_gate(bk, a_msb, b_msb);
    // GCC evaluates these two argument NOTs right to left (b first), which
    // fixes the node order the reference records.
    Bit nb = not_gate(bk, b_msb);
    Bit na = not_gate(bk, a_msb);
    Bit both_pos = and_gate(bk, na, nb);
    Bit pos_ov = and_gate(bk, both_pos, s);
    Bit ns = not_gate(bk, s);
    Bit neg_ov = and_gate(bk, both_neg, ns);
    f.v = or_gate(bk, pos_ov, neg_ov);
  }
  return f;
}

}  // namespace alu

int fu_out_width(uint32_t op, uint32_t w) {
  switch (op) {
    case CVM_FU_ADD:
    case CVM_FU_ADD_CIN:
    case CVM_FU_SUB:
    case CVM_FU_ADDSUB:
      return int(w) + 1;
    case CVM_FU_CMP:
      return int(w) + 4;
    case CVM_FU_UMUL:
    case CVM_FU_SMUL:
      return 2 * int(w);
    case CVM_FU_AND:
    case CVM_FU_ORR:
    case CVM_FU_EOR:
    case CVM_FU_ORN:
    case CVM_FU_LSL:
    case CVM_FU_LSR:
    case CVM_FU_ASR:
    case CVM_FU_UDIV:
    case CVM_FU_UDIV_EXACT:
    case CVM_FU_MUL_LO:
      return int(w);
    default:
      return -1;
  }
}

Word fu_apply(Backend& bk, uint32_t op, const Word& a, const Word& b, Bit c) {
  using namespace alu;
  auto with_carry = [](const AddResult& r) {
    Word w = r.sum;
    w.push_back(r.carry_out);
    return w;
  };
  switch (op) {
    case CVM_FU_ADD: return with_carry(add(bk, a, b));
    case CVM_FU_ADD_CIN: return with_carry(add(bk, a, b, c));
    case CVM_FU_SUB: return with_carry(sub(bk, a, b));
    case CVM_FU_ADDSUB: return with_carry(add_sub_select(bk, a, b, c));
    case CVM_FU_CMP: {
      // SUBS / CMP as the emulator issues them (emulator.cpp:258-270,168-175)
      AddResult r = sub(bk, a, b);
      bk.fence();
      Bit b_sign = not_gate(bk, b.back());
      Flags f = flags(bk, r.sum, r.carry_out, a.back(), b_sign);
      Word w = r.sum;
      w.insert(w.end(), {f.n, f.z, f.c, f.v});
      return w;
    }
    case CVM_FU_AND: return bitwise(bk, BitwiseKind::And, a, b);
    case CVM_FU_ORR: return bitwise(bk, BitwiseKind::Or, a, b);
    case CVM_FU_EOR: return bitwise(bk, BitwiseKind::Xor, a, b);
    case CVM_FU_ORN: return bitwise(bk, BitwiseKind::OrNot, a, b);
    case CVM_FU_LSL: return shift_reg(bk, a, ShiftKind::LogicalLeft, b);
    case CVM_FU_LSR: return shift_reg(bk, a, ShiftKind::LogicalRight, b);
    case CVM_FU_ASR: return shift_reg(bk, a, ShiftKind::ArithmeticRight, b);
    case CVM_FU_UMUL: return mul_unsigned(bk, a, b);
    case CVM_FU_SMUL: return mul_signed(bk, a, b);
    case CVM_FU_UDIV: return div_unsigned(bk, a, b, DivAccumulator::Widened);
    case CVM_FU_UDIV_EXACT: return div_unsigned(bk, a, b, DivAccumulator::Exact);
    case CVM_FU_MUL_LO: {
      Word p = mul_unsigned(bk, a, b);
      p.resize(a.size());  // the high half's gates are recorded but dead
      return p;
    }
    default: throw InputError("unknown functional-unit op " + std::to_string(op));
  }
}

}  // namespace cvm
