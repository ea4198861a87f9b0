// Reference-side circuit recording: the reference's own functional units
// (alu.hpp) and emulator (emulator.hpp) issue their gates once into a
// DagRecorder -- a cryptovm::Backend that forwards to a SimBackend, so node
// ids are exactly the GateDag's -- and the recorded table is handed to the
// B200 library (cvm_dag_batch / cvm_backend_replay_dag, include/cvm_gpu.h).
// The B200 library therefore holds no copy of the circuits.
//
// Also the C entry points (cvmref_*) the Python tests and bench.py bind with
// ctypes: record a functional unit or a program, and run the reference API
// end to end on the GPU through cryptovm::GpuBackend.
#ifndef CRYPTOVM_DAG_EXPORT_HPP_
#define CRYPTOVM_DAG_EXPORT_HPP_

#include <cstdint>
#include <vector>

#include "cvm_gpu.h"

#ifdef __cplusplus
#include "cryptovm/gates.hpp"
#include "cryptovm/sim_backend.hpp"

namespace cryptovm {

// Forwards every call to a SimBackend (which mints the handles and records
// the GateDag) and remembers each CONSTANT's value, which DagNode does not
// store (dag.hpp:33-42).
class DagRecorder final : public Backend {
 public:
  BitHandle constant(bool value) override;
  BitHandle unary_gate(GateKind kind, BitHandle a) override;
  BitHandle binary_gate(GateKind kind, BitHandle a, BitHandle b) override;
  BitHandle mux_gate(BitHandle sel, BitHandle on_true, BitHandle on_false) override;
  BitHandle encrypt_bit(bool value) override;
  bool decrypt_bit(BitHandle bit) override;
  std::vector<std::uint8_t> export_bit(BitHandle bit) override;
  BitHandle import_bit(const std::vector<std::uint8_t>& blob) override;
  void push_region(std::string_view name) override;
  void pop_region() override;
  void fence() override;

  const GateDag& dag() const { return sim_.dag(); }
  // The recorded DAG as the C ABI's node table.
  std::vector<cvm_dag_node> table() const;

 private:
  SimBackend sim_;
  std::vector<std::uint8_t> const_value_;  // by node id
};

}  // namespace cryptovm
extern "C" {
#endif

#define CVMREF_API __attribute__((visibility("default")))

/* A recorded circuit: node table + output node ids (LSB first). */
typedef struct cvmref_dag {
  cvm_dag_node* nodes;
  uint64_t n_nodes;
  uint64_t* outputs;
  uint64_t n_outputs;
  uint64_t n_inputs;
  char** regions;  /* GateDag::regions(): path of each node.region index */
  uint64_t n_regions;
} cvmref_dag;

/* One instruction of a straight-line or branching program (isa.hpp:87-97).
 * op / cond are the reference's names (opcode_from_name / cond_from_name);
 * cond "" = unconditional; has_* flag the optional fields. */
typedef struct cvmref_insn {
  char op[8];
  char cond[4];
  int32_t rd, rn, rm;
  int32_t sets_flags;
  int32_t has_imm, has_imm2, has_target;
  uint32_t target;
  uint64_t imm, imm2;
} cvmref_insn;

CVMREF_API const char* cvmref_last_error(void);
/* The functional unit `op` at `width` bits as the reference records it:
 * inputs a (width bits), b (width bits) and, for add_cin / addsub, c; ops
 * add, add_cin, sub, addsub, cmp (SUBS/CMP: sub + NZCV as the emulator issues
 * it, emulator.cpp:168-175), and, orr, eor, orn, lsl, lsr, asr, umul, smul,
 * udiv, udiv_exact, mul_lo (MUL as the emulator issues it: the low half). */
CVMREF_API int cvmref_record_fu(const char* op, unsigned width, cvmref_dag* out);
/* A program on the reference Machine (emulator.cpp) over a BufferMemory of
 * `n_mem` encrypted words (the inputs, word by word); outputs are the final
 * registers then N, Z, C, V.  Branches need the key owner and are rejected. */
CVMREF_API int cvmref_record_program(unsigned word_size, unsigned register_count,
                                     uint64_t n_mem, const cvmref_insn* program,
                                     uint64_t n_insn, cvmref_dag* out);
CVMREF_API void cvmref_dag_free(cvmref_dag* dag);

/* The reference Machine on SimBackend (cleartext; LocalBranchOracle) over a
 * BufferMemory holding mem[0..n_mem): the expected final registers and NZCV
 * of a program, for cross-checks of the GPU against the reference. */
CVMREF_API int cvmref_sim_program(unsigned word_size, unsigned register_count,
                                  const uint64_t* mem, uint64_t n_mem,
                                  const cvmref_insn* program, uint64_t n_insn,
                                  uint64_t max_steps, uint64_t* regs_out, uint8_t* nzcv_out);

/* The reference's own CPU path on the same circuit: `batch` instances of `op`
 * on SimBackend (cleartext booleans, sim_backend.cpp -- not FHE work),
 * operands a[i], b[i] (and c[i] for add_cin / addsub); results decrypted as
 * words of the output width (<= 64 bits) into out[i]; wall seconds of the
 * recording + evaluation in *seconds, and the total DAG node count. */
CVMREF_API int cvmref_sim_fu_batch(const char* op, unsigned width, uint64_t batch,
                                   const uint64_t* a, const uint64_t* b, const uint64_t* c,
                                   uint64_t* out, double* seconds, uint64_t* nodes);

/* The reference API end to end on the B200 through cryptovm::GpuBackend:
 * `batch` x alu::add on Word::encrypt'ed operands, one evaluation of every
 * sum, decrypt_word per result (word.cpp:42-86). */
CVMREF_API int cvmref_add_batch_gpu(cvm_ctx* ctx, const cvm_keyset* owner, unsigned width,
                                    uint64_t batch, const uint64_t* a, const uint64_t* b,
                                    uint64_t* sums, uint8_t* carries,
                                    cvm_backend_stats* stats);
/* The reference Machine (branches through LocalBranchOracle) on the B200 over
 * encrypted memory `mem`; the final registers and NZCV are evaluated in one
 * demand-driven flush, then decrypted. */
CVMREF_API int cvmref_run_program_gpu(cvm_ctx* ctx, const cvm_keyset* owner,
                                      unsigned word_size, unsigned register_count,
                                      const uint64_t* mem, uint64_t n_mem,
                                      const cvmref_insn* program, uint64_t n_insn,
                                      uint64_t max_steps, uint64_t* regs_out,
                                      uint8_t* nzcv_out, cvm_backend_stats* stats,
                                      uint64_t* branch_queries);

#ifdef __cplusplus
}
#endif
#endif  // CRYPTOVM_DAG_EXPORT_HPP_
