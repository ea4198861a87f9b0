// Invariants of the wave-packing schedule (csrc/schedule.cpp), on the CPU:
//   * every gate runs after all its predecessors;
//   * every gate runs between its ASAP and ALAP level, so the number of
//     launches is the critical path;
//   * the planner cost of the packed launches is never above that of the
//     plain ASAP levels (checked on the DAG given, and on random DAGs).
// Input (optional file): "G" then G lines "p0 p1 p2 boots" (-1 = no pred);
// "batch B" as a first line replicates the DAG B times (independent copies).
// Build + run: tests/test_schedule.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "schedule.hpp"

using namespace cvm;

struct Dag {
  std::vector<int32_t> pred;
  std::vector<uint8_t> boots;
};

static int check(const Dag& d, const char* name, bool print_widths) {
  const size_t G = d.boots.size();
  std::vector<uint32_t> asap(G, 1), tail(G, 0);
  uint32_t depth = 1;
  for (size_t i = 0; i < G; ++i) {
    for (int k = 0; k < 3; ++k) {
      const int32_t p = d.pred[3 * i + k];
      if (p >= int32_t(i)) {
        printf("FAIL %s: predecessor %d of gate %zu is not earlier\n", name, p, i);
        return 1;
      }
      if (p >= 0) asap[i] = std::max(asap[i], asap[p] + 1);
    }
    depth = std::max(depth, asap[i]);
  }
  for (size_t i = G; i-- > 0;)
    for (int k = 0; k < 3; ++k)
      if (d.pred[3 * i + k] >= 0)
        tail[d.pred[3 * i + k]] = std::max(tail[d.pred[3 * i + k]], tail[i] + 1);
  const std::vector<uint32_t> launch = pack_schedule(d.pred, d.boots);
  std::vector<int> wp(depth + 1, 0), wa(depth + 1, 0);
  for (size_t i = 0; i < G; ++i) {
    const uint32_t alap = depth - tail[i];
    if (launch[i] < asap[i] || launch[i] > alap) {
      printf("FAIL %s: gate %zu in launch %u outside [%u, %u]\n", name, i, launch[i], asap[i],
             alap);
      return 1;
    }
    for (int k = 0; k < 3; ++k) {
      const int32_t p = d.pred[3 * i + k];
      if (p >= 0 && launch[p] >= launch[i]) {
        printf("FAIL %s: gate %zu (launch %u) not after predecessor %d (launch %u)\n", name, i,
               launch[i], p, launch[p]);
        return 1;
      }
    }
    wp[launch[i]] += d.boots[i];
    wa[asap[i]] += d.boots[i];
  }
  long cp = 0, ca = 0;
  for (uint32_t k = 1; k <= depth; ++k) {
    cp += br_level_cost(wp[k]) + (wp[k] ? 3 : 0);
    ca += br_level_cost(wa[k]) + (wa[k] ? 3 : 0);
  }
  if (cp > ca) {
    printf("FAIL %s: packed cost %ld above plain levels %ld\n", name, cp, ca);
    return 1;
  }
  if (print_widths) {
    printf("%s: depth %u, cost %.1f ms packed vs %.1f ms plain; widths", name, depth, cp / 10.0,
           ca / 10.0);
    for (uint32_t k = 1; k <= depth; ++k) printf(" %d", wp[k]);
    printf(" (plain");
    for (uint32_t k = 1; k <= depth; ++k) printf(" %d", wa[k]);
    printf(")\n");
  }
  return 0;
}

static Dag random_dag(std::mt19937& rng, int G, int window) {
  Dag d;
  d.pred.assign(3 * size_t(G), -1);
  d.boots.resize(G);
  for (int i = 0; i < G; ++i) {
    d.boots[i] = rng() % 10 == 0 ? 2 : 1;
    const int np = d.boots[i] == 2 ? 3 : 2;
    for (int k = 0; k < np; ++k) {
      if (i == 0 || rng() % 4 == 0) continue;  // an input or resident operand
      const int lo = std::max(0, i - window);
      int p = lo + int(rng() % uint32_t(i - lo));
      bool dup = false;
      for (int e = 0; e < k; ++e) dup |= d.pred[3 * size_t(i) + e] == p;
      if (!dup) d.pred[3 * size_t(i) + k] = p;
    }
  }
  return d;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    FILE* f = fopen(argv[1], "r");
    if (!f) return 2;
    int batch = 1, G = 0;
    char word[16];
    if (fscanf(f, "%15s", word) == 1 && std::string(word) == "batch") {
      if (fscanf(f, "%d %d", &batch, &G) != 2) return 2;
    } else {
      G = atoi(word);
    }
    Dag one;
    one.pred.assign(3 * size_t(G), -1);
    one.boots.resize(G);
    for (int i = 0; i < G; ++i) {
      int p[3], b;
      if (fscanf(f, "%d %d %d %d", &p[0], &p[1], &p[2], &b) != 4) return 2;
      for (int k = 0; k < 3; ++k) one.pred[3 * size_t(i) + k] = p[k];
      one.boots[i] = uint8_t(b);
    }
    fclose(f);
    // independent copies, one after the other (as a batch records them:
    // adder after adder), so indices stay topological
    Dag d;
    d.pred.assign(3 * size_t(G) * batch, -1);
    d.boots.resize(size_t(G) * batch);
    for (int c = 0; c < batch; ++c)
      for (int i = 0; i < G; ++i) {
        const size_t j = size_t(c) * G + i;
        d.boots[j] = one.boots[i];
        for (int k = 0; k < 3; ++k) {
          const int32_t p = one.pred[3 * size_t(i) + k];
          d.pred[3 * j + k] = p < 0 ? -1 : int32_t(size_t(c) * G + p);
        }
      }
    if (check(d, argv[1], true)) return 1;
  }
  std::mt19937 rng(5);
  for (int t = 0; t < 40; ++t) {
    const int G = 200 + int(rng() % 20000), window = 5 + int(rng() % 3000);
    if (check(random_dag(rng, G, window), "random", false)) return 1;
  }
  printf("OK\n");
  return 0;
}
