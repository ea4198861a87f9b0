// Device context: resident keys, LWE slot slab, level submission.
//
// A level (a set of mutually independent bootstrapped gates, e.g. one carry
// scan level of 256 adders, alu.cpp:80-89 in the reference) becomes exactly
// two launches on the context stream: blind_rotate_kernel over every
// bootstrap of the level (MUX contributes two), then key_switch_kernel over
// every gate.  Job descriptors travel through a pinned staging arena and a
// device job arena that are recycled at each cvm_sync.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "cvm_internal.hpp"
#include "kernels.cuh"

namespace cvm {

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Bump allocator over chunks; reset() recycles everything (call after sync).
template <bool kPinned>
class Arena {
 public:
  ~Arena() {
    for (auto& c : chunks_) kPinned ? (void)cudaFreeHost(c.ptr) : (void)cudaFree(c.ptr);
  }
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    for (; cur_ < chunks_.size(); ++cur_, off_ = 0) {
      if (chunks_[cur_].size - off_ >= bytes) {
        void* p = static_cast<char*>(chunks_[cur_].ptr) + off_;
        off_ += bytes;
        return p;
      }
    }
    size_t sz = std::max(bytes, size_t(16) << 20);
    void* p = nullptr;
    if (kPinned) check(cudaMallocHost(&p, sz), "cudaMallocHost(arena)");
    else check(cudaMalloc(&p, sz), "cudaMalloc(arena)");
    chunks_.push_back({p, sz});
    cur_ = chunks_.size() - 1;
    off_ = bytes;
    return p;
  }
  void reset() {
    cur_ = 0;
    off_ = 0;
  }

 private:
  struct Chunk {
    void* ptr;
    size_t size;
  };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0, off_ = 0;
};

}  // namespace

class Context {
 public:
  explicit Context(int device) : device_(device) {
    int count = 0;
    check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) throw DeviceError("no such CUDA device");
    cudaDeviceProp prop{};
    check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
      throw DeviceError("libcvm_b200 is built for sm_100a only (found sm_" +
                        std::to_string(prop.major * 10 + prop.minor) + ")");
    sm_count_ = prop.multiProcessorCount;
    check(cudaSetDevice(device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    // twiddle tables
    c64 T1[64][8], T2[64][8];
    make_twiddles(T1, T2);
    check(cudaMalloc(&tw1_, sizeof(T1)), "cudaMalloc(tw1)");
    check(cudaMalloc(&tw2_, sizeof(T2)), "cudaMalloc(tw2)");
    check(cudaMemcpy(tw1_, T1, sizeof(T1), cudaMemcpyHostToDevice), "tw1");
    check(cudaMemcpy(tw2_, T2, sizeof(T2), cudaMemcpyHostToDevice), "tw2");
    c64 T4[64];  // warp FFT (v4): per-lane twiddle bases [32][2]
    for (int l = 0; l < 32; ++l) {
      const TwBasesW b = make_wbases(l);
      T4[2 * l] = b.base;
      T4[2 * l + 1] = b.w;
    }
    check(cudaMalloc(&tw4_, sizeof(T4)), "cudaMalloc(tw4)");
    check(cudaMemcpy(tw4_, T4, sizeof(T4), cudaMemcpyHostToDevice), "tw4");
    check(cudaEventCreate(&ev_user_[0]), "event");
    check(cudaEventCreate(&ev_user_[1]), "event");
  }
  ~Context() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    for (auto& p : prof_) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    cudaEventDestroy(ev_user_[0]);
    cudaEventDestroy(ev_user_[1]);
    cudaFree(tw1_);
    cudaFree(tw2_);
    cudaFree(tw4_);
    cudaFree(bkf_);
    cudaFree(bkf4_);
    cudaFree(ksktc_);
    cudaFree(kspart_);
    cudaFree(slab_);
    cudaFree(xlwe_);
    cudaFree(flush_buf_);
    cudaStreamDestroy(stream_);
  }

  void upload_keys(const uint32_t* bk, const uint32_t* ksk) {
    if (!bk || !ksk) throw InputError("upload_keys: null key pointer");
    check(cudaSetDevice(device_), "cudaSetDevice");
    if (!bkf_) check(cudaMalloc(&bkf_, kBkfBytes), "cudaMalloc(bkf)");
    const size_t ksk_rows = size_t(kPolyN) * kKsT * kKsBase;
    uint32_t* ksk_pad = nullptr;  // staging only: the tcgen05 tiles are built from it
    check(cudaMalloc(&ksk_pad, ksk_rows * kKskRowStride * 4), "cudaMalloc(ksk)");
    uint32_t* bk_tmp = nullptr;
    check(cudaMalloc(&bk_tmp, kBkWords * 4), "cudaMalloc(bk tmp)");
    check(cudaMemcpyAsync(bk_tmp, bk, kBkWords * 4, cudaMemcpyHostToDevice, stream_),
          "upload bk");
    check(launch_bk_to_fft(bk_tmp, tw1_, tw2_, bkf_, stream_), "bk_to_fft");
    ++stats_.other_launches;
    // the same key in the warp-FFT bin order of the v4 throughput kernel
    if (!bkf4_) check(cudaMalloc(&bkf4_, kBkfBytes), "cudaMalloc(bkf4)");
    check(launch_bk_to_fft_v4(bk_tmp, tw4_, bkf4_, stream_), "bk_to_fft_v4");
    ++stats_.other_launches;
    // KSK rows padded 631 -> 632 words (pad word zero)
    check(cudaMemsetAsync(ksk_pad, 0, ksk_rows * kKskRowStride * 4, stream_), "memset ksk");
    check(cudaMemcpy2DAsync(ksk_pad, kKskRowStride * 4, ksk, kLweWords * 4, kLweWords * 4,
                            ksk_rows, cudaMemcpyHostToDevice, stream_),
          "upload ksk");
    if (!ksktc_) check(cudaMalloc(&ksktc_, kKskTcWords * 4), "cudaMalloc(ksktc)");
    if (!kspart_) check(cudaMalloc(&kspart_, kKsPartWords * 4), "cudaMalloc(kspart)");
    check(launch_ksk_to_tc(ksk_pad, ksktc_, stream_), "ksk_to_tc");
    ++stats_.other_launches;
    check(cudaStreamSynchronize(stream_), "sync(upload_keys)");
    cudaFree(bk_tmp);
    cudaFree(ksk_pad);
    has_keys_ = true;
  }

  void reserve(uint64_t n) {
    if (n <= cap_) return;
    check(cudaSetDevice(device_), "cudaSetDevice");
    uint64_t cap = std::max<uint64_t>(n, cap_ * 2);
    cap = std::max<uint64_t>(cap, 1024);
    uint32_t* p = nullptr;
    check(cudaMalloc(&p, cap * kLweStride * 4), "cudaMalloc(slab)");
    check(cudaMemsetAsync(p, 0, cap * kLweStride * 4, stream_), "memset slab");
    if (slab_) {
      check(cudaMemcpyAsync(p, slab_, cap_ * kLweStride * 4, cudaMemcpyDeviceToDevice,
                            stream_),
            "grow slab");
      check(cudaStreamSynchronize(stream_), "sync(grow)");
      cudaFree(slab_);
    }
    slab_ = p;
    cap_ = cap;
  }
  uint64_t capacity() const { return cap_; }
  // Slot ids are handed out by a bump allocator so several backends (and the
  // raw level API) can share one slab; capacity follows at the next reserve.
  uint64_t alloc_slots(uint64_t n) {
    std::lock_guard<std::mutex> lock(alloc_mu_);
    const uint64_t base = used_;
    used_ += n;
    return base;
  }
  uint64_t slots_used() const { return used_; }
  // Return the top run [first, end) to the allocator if nothing was handed out
  // after it (stack discipline; a temporary backend's slots after its work
  // has been synchronised).
  bool release_slots(uint64_t first, uint64_t end) {
    std::lock_guard<std::mutex> lock(alloc_mu_);
    if (end != used_ || first > end) return false;
    used_ = first;
    return true;
  }

  void upload(uint64_t slot, uint64_t count, const uint32_t* lwe) {
    if (count == 0) return;
    if (!lwe) throw InputError("upload_lwe: null pointer");
    if (slot + count > cap_) throw InputError("upload_lwe: slot range beyond capacity");
    check(cudaSetDevice(device_), "cudaSetDevice");
    const void* src = lwe;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, lwe) != cudaSuccess ||
        attr.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      void* staged = host_arena_.alloc(count * kLweWords * 4);
      std::memcpy(staged, lwe, count * kLweWords * 4);
      src = staged;
    }
    check(cudaMemcpy2DAsync(slab_ + slot * kLweStride, kLweStride * 4, src, kLweWords * 4,
                            kLweWords * 4, count, cudaMemcpyHostToDevice, stream_),
          "upload_lwe");
  }

  void download(uint64_t slot, uint64_t count, uint32_t* lwe) {
    if (count == 0) return;
    if (!lwe) throw InputError("download_lwe: null pointer");
    if (slot + count > cap_) throw InputError("download_lwe: slot range beyond capacity");
    check(cudaSetDevice(device_), "cudaSetDevice");
    check(cudaMemcpy2DAsync(lwe, kLweWords * 4, slab_ + slot * kLweStride, kLweStride * 4,
                            kLweWords * 4, count, cudaMemcpyDeviceToHost, stream_),
          "download_lwe");
    sync();
  }

  // Download an arbitrary slot list as one contiguous [count][631] block: a
  // device gather into the arena, one D2H copy (straight into `lwe` when it
  // is pinned), one synchronisation.
  void gather_download(const uint64_t* slots, uint64_t count, uint32_t* lwe) {
    if (count == 0) return;
    if (!lwe || !slots) throw InputError("gather_download: null pointer");
    for (uint64_t i = 0; i < count; ++i)
      if (slots[i] >= cap_) throw InputError("gather_download: slot beyond capacity");
    check(cudaSetDevice(device_), "cudaSetDevice");
    const size_t bytes = count * kLweWords * 4;
    uint64_t* h_slots = static_cast<uint64_t*>(host_arena_.alloc(count * 8));
    std::memcpy(h_slots, slots, count * 8);
    uint64_t* d_slots = static_cast<uint64_t*>(dev_arena_.alloc(count * 8));
    uint32_t* d_out = static_cast<uint32_t*>(dev_arena_.alloc(bytes));
    check(cudaMemcpyAsync(d_slots, h_slots, count * 8, cudaMemcpyHostToDevice, stream_),
          "upload gather slots");
    check(launch_gather_lwe(slab_, d_slots, count, d_out, stream_), "gather_lwe");
    ++stats_.other_launches;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, lwe) == cudaSuccess &&
                        attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    void* dst = pinned ? static_cast<void*>(lwe) : host_arena_.alloc(bytes);
    check(cudaMemcpyAsync(dst, d_out, bytes, cudaMemcpyDeviceToHost, stream_), "download");
    check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    if (!pinned) std::memcpy(lwe, dst, bytes);
    sync();
  }

  // Validates a level and returns its number of blind rotations.
  uint64_t count_br(const cvm_gate* gates, uint64_t count) const {
    if (!gates && count) throw InputError("submit_level: null gates");
    uint64_t n_br = 0;
    for (uint64_t g = 0; g < count; ++g) {
      const uint32_t k = gates[g].kind;
      if (k < uint32_t(GateKind::Nand) || k > uint32_t(GateKind::Mux))
        throw InputError("submit_level: not a bootstrapped gate kind: " + std::to_string(k));
      if (gates[g].out_slot >= cap_) throw InputError("submit_level: out_slot beyond capacity");
      n_br += k == uint32_t(GateKind::Mux) ? 2 : 1;
    }
    return n_br;
  }

  // Expands gates into blind-rotation jobs (MUX: two) and key-switch jobs.
  void expand(const cvm_gate* gates, uint64_t count, BrJob* br, KsJob* ks) const {
    uint64_t b = 0;
    for (uint64_t g = 0; g < count; ++g) {
      const cvm_gate& gt = gates[g];
      const GateKind kind = GateKind(gt.kind);
      if (kind == GateKind::Mux) {
        // AND(sel, t) and AND(NOT sel, f) without key switch, + 1/8, one KS
        const cvm_operand& s = gt.in[0];
        make_br(br[b], 0u - kMu, 1, s, 1, gt.in[1], b);
        make_br(br[b + 1], 0u - kMu, -1, s, 1, gt.in[2], b + 1);
        ks[g] = {{uint32_t(b), uint32_t(b + 1)}, kMu, uint32_t(gt.out_slot)};
        b += 2;
      } else {
        const GateCombo c = combo(kind);
        make_br(br[b], c.c, c.ca, gt.in[0], c.cb, gt.in[1], b);
        ks[g] = {{uint32_t(b), kNoInput}, 0u, uint32_t(gt.out_slot)};
        b += 1;
      }
    }
  }

  void launch_level(const BrJob* d_br, uint64_t n_br, const KsJob* d_ks, uint64_t n_ks) {
    Prof* p = begin_prof(0);
    check(launch_blind_rotate(br_variant, d_br, int(n_br), slab_, bkf_, tw1_, tw2_, bkf4_, tw4_,
                              xlwe_, stream_),
          "blind_rotate_kernel");
    end_prof(p);
    p = begin_prof(1);
    check(launch_key_switch(ks_variant, d_ks, int(n_ks), xlwe_, ksktc_, kspart_, slab_, stream_),
          "key_switch_kernel");
    end_prof(p);
    stats_.br_launches++;
    stats_.br_jobs += n_br;
    stats_.ks_launches++;
    stats_.ks_jobs += n_ks;
  }

  void submit_level(const cvm_gate* gates, uint64_t count) {
    if (count == 0) return;
    if (!has_keys_) throw StateError("submit_level before upload_keys");
    check(cudaSetDevice(device_), "cudaSetDevice");
    const uint64_t n_br = count_br(gates, count);
    if (n_br > xcap_) grow_xlwe(n_br);
    BrJob* br = static_cast<BrJob*>(host_arena_.alloc(n_br * sizeof(BrJob)));
    KsJob* ks = static_cast<KsJob*>(host_arena_.alloc(count * sizeof(KsJob)));
    expand(gates, count, br, ks);
    BrJob* d_br = static_cast<BrJob*>(dev_arena_.alloc(n_br * sizeof(BrJob)));
    KsJob* d_ks = static_cast<KsJob*>(dev_arena_.alloc(count * sizeof(KsJob)));
    check(cudaMemcpyAsync(d_br, br, n_br * sizeof(BrJob), cudaMemcpyHostToDevice, stream_),
          "upload br jobs");
    check(cudaMemcpyAsync(d_ks, ks, count * sizeof(KsJob), cudaMemcpyHostToDevice, stream_),
          "upload ks jobs");
    launch_level(d_br, n_br, d_ks, count);
  }

  // A captured sequence of levels with device-resident job tables; replayed
  // as plain launches or as one CUDA graph.
  Plan* make_plan(const std::vector<std::vector<cvm_gate>>& levels) {
    if (!has_keys_) throw StateError("plan before upload_keys");
    check(cudaSetDevice(device_), "cudaSetDevice");
    auto plan = std::make_unique<Plan>();
    plan->owner = this;
    size_t bytes = 0;
    std::vector<uint64_t> nbr(levels.size());
    for (size_t l = 0; l < levels.size(); ++l) {
      nbr[l] = count_br(levels[l].data(), levels[l].size());
      bytes += nbr[l] * sizeof(BrJob) + levels[l].size() * sizeof(KsJob) + 512;
      plan->gates += levels[l].size();
      plan->bootstraps += nbr[l];
      plan->max_br = std::max(plan->max_br, nbr[l]);
    }
    std::vector<char> host(bytes);
    check(cudaMalloc(&plan->dmem, bytes ? bytes : 1), "cudaMalloc(plan)");
    size_t off = 0;
    for (size_t l = 0; l < levels.size(); ++l) {
      Plan::Level lv;
      lv.n_br = nbr[l];
      lv.n_ks = levels[l].size();
      const size_t br_off = off, ks_off = (off + nbr[l] * sizeof(BrJob) + 255) & ~size_t(255);
      off = (ks_off + lv.n_ks * sizeof(KsJob) + 255) & ~size_t(255);
      expand(levels[l].data(), lv.n_ks, reinterpret_cast<BrJob*>(host.data() + br_off),
             reinterpret_cast<KsJob*>(host.data() + ks_off));
      lv.br = reinterpret_cast<BrJob*>(static_cast<char*>(plan->dmem) + br_off);
      lv.ks = reinterpret_cast<KsJob*>(static_cast<char*>(plan->dmem) + ks_off);
      plan->levels.push_back(lv);
    }
    check(cudaMemcpy(plan->dmem, host.data(), bytes, cudaMemcpyHostToDevice), "upload plan");
    return plan.release();
  }

  void run_plan(Plan* p, bool graph) {
    // job tables and slots live on the context that captured the plan
    if (p->owner != this) throw InputError("plan_run: plan was captured on another context");
    check(cudaSetDevice(device_), "cudaSetDevice");
    if (p->max_br > xcap_) grow_xlwe(p->max_br);
    if (!graph || profiling) {
      for (const auto& lv : p->levels) launch_level(lv.br, lv.n_br, lv.ks, lv.n_ks);
      return;
    }
    if (!p->exec || p->graph_slab != slab_ || p->graph_xlwe != xlwe_) {
      if (p->exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(p->exec));
      p->exec = nullptr;
      cudaGraph_t g;
      check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
      const cvm_kernel_stats saved = stats_;
      for (const auto& lv : p->levels) launch_level(lv.br, lv.n_br, lv.ks, lv.n_ks);
      stats_ = saved;
      check(cudaStreamEndCapture(stream_, &g), "end capture");
      cudaGraphExec_t ex = nullptr;
      check(cudaGraphInstantiate(&ex, g, 0), "cudaGraphInstantiate");
      p->exec = ex;
      cudaGraphDestroy(g);
      p->graph_slab = slab_;
      p->graph_xlwe = xlwe_;
    }
    check(cudaGraphLaunch(static_cast<cudaGraphExec_t>(p->exec), stream_), "cudaGraphLaunch");
    for (const auto& lv : p->levels) {
      stats_.br_launches++;
      stats_.br_jobs += lv.n_br;
      stats_.ks_launches++;
      stats_.ks_jobs += lv.n_ks;
    }
  }

  void sync() {
    check(cudaSetDevice(device_), "cudaSetDevice");
    check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    for (size_t i = 0; i < prof_used_; ++i) {
      float ms = 0;
      check(cudaEventElapsedTime(&ms, prof_[i].a, prof_[i].b), "cudaEventElapsedTime");
      (prof_[i].which == 0 ? stats_.br_ms : stats_.ks_ms) += ms;
    }
    prof_used_ = 0;
    host_arena_.reset();
    dev_arena_.reset();
  }

  void flush_l2() {
    check(cudaSetDevice(device_), "cudaSetDevice");
    const size_t bytes = size_t(256) << 20;  // 2x the 126 MB L2
    if (!flush_buf_) check(cudaMalloc(&flush_buf_, bytes), "cudaMalloc(flush)");
    check(cudaMemsetAsync(flush_buf_, flush_val_++ & 0xFF, bytes, stream_), "flush l2");
    ++stats_.other_launches;
  }

  // Measured DFMA throughput in TFLOP/s (2 flops per FMA), best of `reps`.
  double fp64_peak(int reps) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    double* out = nullptr;
    check(cudaMalloc(&out, 8), "cudaMalloc(peak)");
    cudaEvent_t a, b;
    check(cudaEventCreate(&a), "event");
    check(cudaEventCreate(&b), "event");
    const int blocks = sm_count_ * 8, iters = 1 << 16;
    check(launch_fp64_peak(out, blocks, 1024, stream_), "fp64_peak warmup");
    double best = 0;
    for (int r = 0; r < reps; ++r) {
      check(cudaEventRecord(a, stream_), "event");
      check(launch_fp64_peak(out, blocks, iters, stream_), "fp64_peak");
      check(cudaEventRecord(b, stream_), "event");
      check(cudaEventSynchronize(b), "event sync");
      float ms = 0;
      check(cudaEventElapsedTime(&ms, a, b), "elapsed");
      const double flops = 2.0 * 8 * double(iters) * blocks * 256;
      best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    stats_.other_launches += reps + 1;
    return best;
  }

  void event(int which) {
    check(cudaEventRecord(ev_user_[which & 1], stream_), "cudaEventRecord");
  }
  double event_elapsed() {
    check(cudaEventSynchronize(ev_user_[1]), "cudaEventSynchronize");
    float ms = 0;
    check(cudaEventElapsedTime(&ms, ev_user_[0], ev_user_[1]), "cudaEventElapsedTime");
    return ms;
  }

  bool has_keys() const { return has_keys_; }
  int sm_count() const { return sm_count_; }
  bool profiling = false;
  cvm_kernel_stats stats_{};

 private:
  struct Prof {
    cudaEvent_t a, b;
    int which;
  };

  static GateCombo combo(GateKind k) {
    const uint32_t e = 1u << 29, q = 1u << 30;
    switch (k) {
      case GateKind::Nand: return {e, -1, -1};
      case GateKind::And: return {0u - e, 1, 1};
      case GateKind::Or: return {e, 1, 1};
      case GateKind::Xor: return {q, 2, 2};
      case GateKind::Xnor: return {0u - q, -2, -2};
      case GateKind::Nor: return {0u - e, -1, -1};
      case GateKind::AndNY: return {0u - e, -1, 1};
      case GateKind::AndYN: return {0u - e, 1, -1};
      case GateKind::OrNY: return {e, -1, 1};
      case GateKind::OrYN: return {e, 1, -1};
      default: throw InputError("not a bootstrapped binary gate");
    }
  }

  void make_br(BrJob& j, uint32_t c, int ca, const cvm_operand& a, int cb,
               const cvm_operand& bop, uint64_t out) const {
    j.cst = c + uint32_t(ca) * a.constant + uint32_t(cb) * bop.constant;
    set_term(j, 0, ca, a);
    set_term(j, 1, cb, bop);
    j.out = uint32_t(out);
  }
  void set_term(BrJob& j, int i, int coef, const cvm_operand& o) const {
    if (o.slot < 0) {
      j.slot[i] = 0;
      j.coef[i] = 0;
      return;
    }
    if (uint64_t(o.slot) >= cap_) throw InputError("gate operand slot beyond capacity");
    if (o.sign != 1 && o.sign != -1) throw InputError("operand sign must be +1 or -1");
    j.slot[i] = uint32_t(o.slot);
    j.coef[i] = coef * o.sign;
  }

  void grow_xlwe(uint64_t n) {
    check(cudaStreamSynchronize(stream_), "sync(grow xlwe)");
    cudaFree(xlwe_);
    xcap_ = std::max<uint64_t>(n, 4096);
    check(cudaMalloc(&xlwe_, xcap_ * kXlweStride * 4), "cudaMalloc(xlwe)");
  }

  Prof* begin_prof(int which) {
    if (!profiling) return nullptr;
    if (prof_used_ == prof_.size()) {
      Prof p{};
      check(cudaEventCreate(&p.a), "event");
      check(cudaEventCreate(&p.b), "event");
      prof_.push_back(p);
    }
    Prof* p = &prof_[prof_used_++];
    p->which = which;
    check(cudaEventRecord(p->a, stream_), "cudaEventRecord");
    return p;
  }
  void end_prof(Prof* p) {
    if (p) check(cudaEventRecord(p->b, stream_), "cudaEventRecord");
  }

  int device_;
  int sm_count_ = 0;
  cudaStream_t stream_ = nullptr;
  c64 *tw1_ = nullptr, *tw2_ = nullptr, *bkf_ = nullptr;
  c64 *tw4_ = nullptr, *bkf4_ = nullptr;  // warp-FFT twiddle bases and key (v4)
  uint32_t* ksktc_ = nullptr;  // the KSK's byte limbs as tcgen05 B tiles
  uint32_t* kspart_ = nullptr;  // split-K partials of key-switch variant 9
  uint32_t* slab_ = nullptr;
  uint64_t cap_ = 0;
  uint64_t used_ = 0;
  std::mutex alloc_mu_;
  uint32_t* xlwe_ = nullptr;
  uint64_t xcap_ = 0;
  void* flush_buf_ = nullptr;
  unsigned flush_val_ = 1;
  bool has_keys_ = false;
  Arena<true> host_arena_;
  Arena<false> dev_arena_;
  std::vector<Prof> prof_;
  size_t prof_used_ = 0;
  cudaEvent_t ev_user_[2]{};

 public:
  // Serialises the context's stream, arenas, slab and counters between the
  // backends (and raw level API callers) of several threads sharing it; each
  // entry point below holds it for its whole call.  The slot
  // allocator has its own lock (alloc_mu_).
  std::recursive_mutex mu;
  // Kernel choices of this context: -1 follows the process-wide setting
  // (cvm_set_br_variant / cvm_set_ks_variant / cvm_set_level_packing).
  int br_variant = -1, ks_variant = -1, level_packing = -1;
};

Context* context_create(int device) { return new Context(device); }
void context_destroy(Context* c) { delete c; }
using CtxLock = std::lock_guard<std::recursive_mutex>;
void context_upload_keys(Context* c, const uint32_t* bk, const uint32_t* ksk) {
  CtxLock l(c->mu);
  c->upload_keys(bk, ksk);
}
void context_reserve(Context* c, uint64_t n) {
  CtxLock l(c->mu);
  c->reserve(n);
}
uint64_t context_capacity(const Context* c) { return c->capacity(); }
uint64_t context_alloc_slots(Context* c, uint64_t n) { return c->alloc_slots(n); }
uint64_t context_slots_used(const Context* c) { return c->slots_used(); }
bool context_release_slots(Context* c, uint64_t first, uint64_t end) {
  return c->release_slots(first, end);
}
void context_upload(Context* c, uint64_t slot, uint64_t count, const uint32_t* lwe) {
  CtxLock l(c->mu);
  c->upload(slot, count, lwe);
}
void context_download(Context* c, uint64_t slot, uint64_t count, uint32_t* lwe) {
  CtxLock l(c->mu);
  c->download(slot, count, lwe);
}
void context_gather_download(Context* c, const uint64_t* slots, uint64_t count,
                             uint32_t* lwe) {
  CtxLock l(c->mu);
  c->gather_download(slots, count, lwe);
}
void context_submit_level(Context* c, const cvm_gate* g, uint64_t n) {
  CtxLock l(c->mu);
  c->submit_level(g, n);
}
void context_sync(Context* c) {
  CtxLock l(c->mu);
  c->sync();
}
Plan* context_make_plan(Context* c, const std::vector<std::vector<cvm_gate>>& levels) {
  CtxLock l(c->mu);
  return c->make_plan(levels);
}
void context_run_plan(Context* c, Plan* p, bool graph) {
  CtxLock l(c->mu);
  c->run_plan(p, graph);
  if (p->ran) p->ran->store(true);  // its results are stream-ordered before any read
}
Plan::~Plan() {
  if (exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
  cudaFree(dmem);
}
bool context_has_keys(const Context* c) { return c->has_keys(); }
void context_set_profiling(Context* c, bool on) {
  CtxLock l(c->mu);
  c->profiling = on;
}
cvm_kernel_stats context_stats(Context* c) {
  CtxLock l(c->mu);
  return c->stats_;
}
void context_reset_stats(Context* c) {
  CtxLock l(c->mu);
  c->stats_ = cvm_kernel_stats{};
}
void context_flush_l2(Context* c) {
  CtxLock l(c->mu);
  c->flush_l2();
}
void context_event(Context* c, int which) {
  CtxLock l(c->mu);
  c->event(which);
}
double context_event_elapsed(Context* c) {
  CtxLock l(c->mu);
  return c->event_elapsed();
}
double context_fp64_peak(Context* c, int reps) {
  CtxLock l(c->mu);
  return c->fp64_peak(reps);
}
int context_sm_count(const Context* c) { return c->sm_count(); }
void context_set_kernels(Context* c, int br, int ks, int pack) {
  CtxLock l(c->mu);
  c->br_variant = br;
  c->ks_variant = ks;
  c->level_packing = pack;
}
void context_get_kernels(Context* c, int* br, int* ks, int* pack) {
  CtxLock l(c->mu);
  if (br) *br = c->br_variant;
  if (ks) *ks = c->ks_variant;
  if (pack) *pack = c->level_packing;
}
bool context_level_packing(Context* c) {
  const int p = c->level_packing;
  return p < 0 ? level_packing() : p != 0;
}

}  // namespace cvm
