// Feeds a measured B200 cost table (paper_2101_03403_b200/costs.py) to the
// REFERENCE's own pricing and scheduling code: CostTable::load_file
// (gates.cpp:136-140) -> SimBackend(costs) (cryptovm.cpp:147-151) -> analyze
// (sched.cpp:188-233), on the functional-unit DAGs of the benchmark configs.
// Links only the reference core objects; no GPU needed.
//
//   cost_check <cost-table> [workers ...]     -> one JSON object per DAG
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "cryptovm/alu.hpp"
#include "cryptovm/sched.hpp"
#include "cryptovm/sim_backend.hpp"
#include "cryptovm/word.hpp"

using namespace cryptovm;

static void report(const char* name, const SimBackend& bk, const std::vector<std::uint32_t>& w) {
  const ScheduleReport r = analyze(bk.dag(), w);
  std::printf("{\"dag\": \"%s\", \"report\": %s}\n", name, report_to_json(r).c_str());
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <cost-table> [workers ...]\n", argv[0]);
    return 2;
  }
  try {
    const CostTable costs = CostTable::load_file(argv[1]);
    std::vector<std::uint32_t> workers{1};
    for (int i = 2; i < argc; ++i) workers.push_back(std::strtoul(argv[i], nullptr, 10));
    std::mt19937_64 rng(2);
    {  // C2: 256 independent 16-bit adders
      SimBackend bk(costs);
      for (int i = 0; i < 256; ++i) {
        Word a = Word::encrypt(bk, rng() & 0xFFFF, 16), b = Word::encrypt(bk, rng() & 0xFFFF, 16);
        alu::add(bk, a, b);
      }
      report("c2_add16_x256", bk, workers);
    }
    {  // C2 batch 1: one adder (the latency case)
      SimBackend bk(costs);
      Word a = Word::encrypt(bk, rng() & 0xFFFF, 16), b = Word::encrypt(bk, rng() & 0xFFFF, 16);
      alu::add(bk, a, b);
      report("c2_add16_x1", bk, workers);
    }
    {  // C4: one 16-bit multiplier (full product, every gate recorded)
      SimBackend bk(costs);
      Word a = Word::encrypt(bk, rng() & 0xFFFF, 16), b = Word::encrypt(bk, rng() & 0xFFFF, 16);
      alu::mul_unsigned(bk, a, b);
      report("c4_mul16_x1", bk, workers);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "cost_check: %s\n", e.what());
    return 1;
  }
  return 0;
}
