// `cryptovm run` with backend selection, without CLI11 (absent in this
// image): the flow of the reference CLI's cmd_run (tools/cryptovm.cpp:142-254)
// -- assemble, encrypt the memory words, Machine::run with the local branch
// oracle, decrypt, schedule report -- over BackendSession, so `--backend gpu`
// executes on the B200.  cli_backend_gpu.patch makes the same change inside
// the reference CLI; this driver is the part that compiles and runs here.
//
//   cryptovm_run PROGRAM.s [--backend sim|gpu] [--mem 5,9,...] [--width 16]
//                [--regs 16] [--max-steps N] [--workers 1,48]
// Prints one JSON document: run status, instructions, branch queries, the
// final registers (decrypted), the reference's schedule report of the DAG.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "cryptovm/emulator.hpp"
#include "cryptovm/errors.hpp"
#include "cryptovm/isa.hpp"
#include "cryptovm/keyservice.hpp"
#include "cryptovm/sched.hpp"
#include "cryptovm/word.hpp"
#include "cryptovm_backend_select.hpp"

using namespace cryptovm;

namespace {

std::vector<std::uint64_t> split_u64(const std::string& s) {
  std::vector<std::uint64_t> out;
  std::stringstream in(s);
  std::string item;
  while (std::getline(in, item, ','))
    if (!item.empty()) out.push_back(std::stoull(item, nullptr, 0));
  return out;
}

int run(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: cryptovm_run PROGRAM.s [--backend sim|gpu] [--mem a,b,..] "
                 "[--width W] [--regs R] [--max-steps N] [--workers 1,48]\n");
    return 2;
  }
  std::string path = argv[1], kind = "sim", mem, workers_spec = "1,48";
  unsigned width = 32, regs = 16;
  bool width_given = false;
  std::uint64_t max_steps = 1000000;
  for (int i = 2; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--backend") kind = v;
    else if (k == "--mem") mem = v;
    else if (k == "--width") width = unsigned(std::stoul(v)), width_given = true;
    else if (k == "--regs") regs = unsigned(std::stoul(v));
    else if (k == "--max-steps") max_steps = std::stoull(v);
    else if (k == "--workers") workers_spec = v;
    else throw InputError("unknown option " + k);
  }
  std::ifstream in(path);
  if (!in) throw IoError("cannot open " + path);
  std::stringstream src;
  src << in.rdbuf();
  AssembleOptions options;
  options.default_word_size = width;
  options.register_count = regs;
  Program program = assemble(src.str(), options);
  if (width_given && program.word_size != width)
    throw InputError(path + " selects a different word size than --width");
  width = program.word_size;

  std::unique_ptr<BackendSession> session = BackendSession::make(kind, CostTable());
  Backend& backend = session->backend();
  std::vector<Word> words;
  for (std::uint64_t v : split_u64(mem)) words.push_back(Word::encrypt(backend, v, width));
  LocalBranchOracle oracle(backend);
  MachineConfig config;
  config.word_size = width;
  config.register_count = regs;
  Machine machine(backend, config, std::make_unique<BufferMemory>(width, std::move(words)),
                  oracle);
  StopReason reason = StopReason::Halted;
  std::string failure;
  try {
    reason = machine.run(program, max_steps);
  } catch (const Error& e) {
    failure = e.what();
  }
  std::ostringstream out;
  out << "{\"backend\": \"" << kind << "\", \"status\": \""
      << (!failure.empty() ? "error" : reason == StopReason::Halted ? "halted" : "step_limit")
      << "\", \"instructions\": " << machine.stats().instructions
      << ", \"branch_queries\": " << machine.stats().branch_queries << ", \"registers\": [";
  for (unsigned r = 0; r < regs; ++r)
    out << (r ? ", " : "") << decrypt_word(backend, machine.reg(r));
  out << "]";
  if (!session->dag().empty()) {
    std::vector<std::uint32_t> workers;
    for (std::uint64_t w : split_u64(workers_spec)) workers.push_back(std::uint32_t(w));
    out << ", \"schedule\": " << report_to_json(analyze(session->dag(), workers));
  }
  if (!failure.empty()) out << ", \"error\": \"" << failure << "\"";
  out << "}";
  std::cout << out.str() << std::endl;
  return failure.empty() ? (reason == StopReason::Halted ? 0 : 2) : 1;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
