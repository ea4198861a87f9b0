// Blind-rotation cost model and wave packing (schedule.hpp).
#include "schedule.hpp"

#include <algorithm>

namespace cvm {

int br_latency_cost(int n) {
  if (n <= 0) return 0;
  const int pair = (n + kBrPair - 1) / kBrPair * kBrTP, wide = (n + kBrSms - 1) / kBrSms * kBrT1;
  return std::min(pair, wide);
}
bool br_latency_pair(int n) {
  return (n + kBrPair - 1) / kBrPair * kBrTP < (n + kBrSms - 1) / kBrSms * kBrT1;
}

int br_remainder_plan(int rest, int* n8, int* n4, int* n1) {
  int best = rest > 0 ? 1 << 30 : 0, b8 = 0, b4 = 0, b1 = 0;
  for (int a = 0; a <= 1 && rest > 0; ++a)
    for (int b = 0; b <= 2; ++b) {
      const int left = std::max(0, rest - a * kBrWave8 - b * kBrWave4);
      if (left > 4 * kBrSms) continue;
      const int cost = a * kBrT8 + b * kBrT4 + br_latency_cost(left);
      if (cost < best) best = cost, b8 = a, b4 = b, b1 = left;
    }
  if (n8) *n8 = b8, *n4 = b4, *n1 = b1;
  return best;
}

int br_level_cost(int boots) {
  if (boots <= 0) return 0;
  if (boots <= 2 * kBrSms) return br_latency_cost(boots);
  const int full = boots / kBrWave8;
  return full * kBrT8 + br_remainder_plan(boots - full * kBrWave8, nullptr, nullptr, nullptr);
}

std::vector<uint32_t> pack_schedule(const std::vector<int32_t>& pred,
                                    const std::vector<uint8_t>& boots, int launch_cost) {
  const size_t G = boots.size();
  std::vector<uint32_t> launch(G, 0);
  if (G == 0) return launch;
  // successors (CSR), in-degrees and the ASAP depth
  std::vector<uint32_t> off(G + 1, 0), indeg(G, 0), asap(G, 1);
  uint32_t depth = 1;
  for (size_t i = 0; i < G; ++i)
    for (int d = 0; d < 3; ++d) {
      const int32_t p = pred[3 * i + d];
      if (p < 0) continue;
      ++off[p + 1];
      ++indeg[i];
      asap[i] = std::max(asap[i], asap[p] + 1);
    }
  for (size_t i = 0; i < G; ++i) {
    off[i + 1] += off[i];
    depth = std::max(depth, asap[i]);
  }
  std::vector<uint32_t> succ(off[G]), fill(off.begin(), off.end() - 1);
  for (size_t i = 0; i < G; ++i)
    for (int d = 0; d < 3; ++d)
      if (pred[3 * i + d] >= 0) succ[fill[pred[3 * i + d]]++] = uint32_t(i);
  // ALAP level: depth minus the longest gate chain after the gate
  std::vector<uint32_t> tail(G, 0), alap(G);
  for (size_t i = G; i-- > 0;)
    for (uint32_t e = off[i]; e < off[i + 1]; ++e) tail[i] = std::max(tail[i], tail[succ[e]] + 1);
  for (size_t i = 0; i < G; ++i) alap[i] = depth - tail[i];

  std::vector<uint32_t> ready, next;
  for (size_t i = 0; i < G; ++i)
    if (indeg[i] == 0) ready.push_back(uint32_t(i));
  auto urgent = [&](uint32_t a, uint32_t b) {
    return alap[a] != alap[b] ? alap[a] < alap[b] : a < b;
  };
  for (uint32_t k = 1; k <= depth; ++k) {
    std::sort(ready.begin(), ready.end(), urgent);
    int must = 0, avail = 0;
    for (uint32_t i : ready) {
      avail += int(boots[i]);
      if (alap[i] <= k) must += int(boots[i]);
    }
    // the most efficient width in [must, avail]; the cost model steps at
    // multiples of 74 bootstraps, so only those (and avail) are candidates
    int width = avail;
    if (k < depth && avail > must) {
      double best = -1.0;
      width = 0;
      auto consider = [&](int w) {
        if (w < std::max(must, 1) || w > avail) return;
        const double eff = double(w) / double(br_level_cost(w) + launch_cost);
        if (eff > best + 1e-12 || (eff > best - 1e-12 && w > width)) best = eff, width = w;
      };
      consider(avail);
      for (int w = 74; w <= avail; w += 74) consider(w);
      consider(must);
    }
    size_t taken = 0;
    int used = 0;
    for (; taken < ready.size(); ++taken) {
      const uint32_t i = ready[taken];
      if (alap[i] > k && used + int(boots[i]) > width) break;
      used += int(boots[i]);
      launch[i] = k;
      for (uint32_t e = off[i]; e < off[i + 1]; ++e)
        if (--indeg[succ[e]] == 0) next.push_back(succ[e]);
    }
    ready.erase(ready.begin(), ready.begin() + taken);
    ready.insert(ready.end(), next.begin(), next.end());
    next.clear();
  }
  return launch;
}

}  // namespace cvm
