// Host-only scheduling pieces shared by the kernel launcher (blind_rotate.cu)
// and the levelizer (backend.cpp), CUDA-free so tests/native/schedule_test.cpp
// builds them with g++ alone:
//   * the blind-rotation cost model of the auto selection (measured wave
//     times, tools/v4_waves.py);
//   * wave packing: the launch of every gate of a flushed DAG.
#pragma once
#include <cstdint>
#include <vector>

namespace cvm {

// A v4 wave of 8 x 148 bootstraps, a v3 round of 4 x 148, a wide-kernel round
// of 148 (one bootstrap per SM) and a pair-kernel round of 74 (one bootstrap
// per 2-SM cluster), in 0.1 ms.
constexpr int kBrSms = 148, kBrWave8 = 8 * kBrSms, kBrWave4 = 4 * kBrSms;
constexpr int kBrPair = kBrSms / 2;
constexpr int kBrT8 = 113, kBrT4 = 58, kBrT1 = 23, kBrTP = 14;

// Latency kernels for n bootstraps: rounds of the pair kernel or of the wide
// kernel, whichever finishes first (pair for n <= 74 and 149-222: measured
// 1.41 / 4.18 ms vs wide 2.27 / 4.54 ms).
int br_latency_cost(int n);
bool br_latency_pair(int n);

// The remainder of a wide level after its full v4 waves: at most one more v4
// wave, two v3 rounds and up to 592 bootstraps on the latency kernels, the
// cheapest combination that covers `rest`.  Returns its cost (0.1 ms); the v4
// waves / v3 rounds / latency bootstraps go to n8/n4/n1 if non-null.
int br_remainder_plan(int rest, int* n8, int* n4, int* n1);

// Device time (0.1 ms) of one level of `boots` bootstraps under the
// blind-rotation auto selection (blind_rotate.cu).
int br_level_cost(int boots);

// Wave packing.  Gates 0..G-1 in topological order; pred[3i+d] (d < 3) are
// the gate's predecessors among them (-1: none), boots[i] its bootstrap
// count (1, or 2 for MUX).  Returns the launch (1..depth, depth = the longest
// dependency chain) of every gate: each gate runs after all its
// predecessors and no later than its ALAP level; launch k takes every ready
// gate whose ALAP level is k, then the most urgent other ready gates (ALAP
// level, then index) up to the width with the most bootstraps per unit of
// br_level_cost(width) + launch_cost.  The number of launches stays depth.
std::vector<uint32_t> pack_schedule(const std::vector<int32_t>& pred,
                                    const std::vector<uint8_t>& boots, int launch_cost = 3);

}  // namespace cvm
