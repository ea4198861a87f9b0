// sm_100a device primitives shared by the kernels: shared-memory
// addressing, mbarriers, TMA bulk copies (SASS UBLKCP), named barriers,
// cp.async, tcgen05 / tensor-memory helpers, and the launch-time dynamic
// shared-memory opt-in.
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "fft512.cuh"

namespace cvm {

__device__ __forceinline__ c64 ldg_c64(const c64* p) {
  double2 d = __ldg(reinterpret_cast<const double2*>(p));
  return {d.x, d.y};
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on `bar` (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Shared-memory atomic add with release semantics at CTA scope (orders this
// thread's earlier shared-memory accesses before the increment, without a
// full fence); returns the old value.
__device__ __forceinline__ uint32_t atom_add_release_cta(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Named barrier over the 64 threads of one bootstrap (ids 1..15).
__device__ __forceinline__ void group_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// ---- tcgen05 / tensor-memory helpers ----
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor of a [rows][16 B] block, no swizzle: core
// matrices of 8 rows x 16 B are contiguous (128 B apart in both directions).
__device__ __forceinline__ uint64_t smem_desc_rows16(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | (uint64_t(128 >> 4) << 16) | (uint64_t(128 >> 4) << 32) |
         (1ull << 46);
}
// 64 rows x 128 bit smem -> TMEM, rows 0-31 to lane quarters 0 and 2, rows
// 32-63 to quarters 1 and 3: thread t of every bootstrap finds its value in
// its own lane whichever warp pair the bootstrap runs on.
__device__ __forceinline__ void tc_cp_64x128_0213(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(taddr), "l"(desc)
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 8 consecutive 32-bit columns of this thread's lane (= two complex doubles).
// The registers are written asynchronously: read them only after
// tc_wait_ld16, which takes them as operands so no use is hoisted above it.
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld16(uint32_t (&a)[8], uint32_t (&b)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]),
                 "+r"(a[6]), "+r"(a[7]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]),
                 "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
               :
               : "memory");
}
__device__ __forceinline__ c64 c64_of(const uint32_t* r) {
  return {__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2])};
}

// ---- cp.async (16-B copies, one commit group per stage) ----
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Opt a kernel into more than 48 KB of dynamic shared memory, once.
template <class K>
// The dynamic shared-memory opt-in is per device: `configured` holds one bit
// per device ordinal (ordinals >= 64 set the attribute on every launch).
inline cudaError_t set_smem(K* kern, int bytes, std::atomic<uint64_t>& configured) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (configured.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) configured.fetch_or(bit, std::memory_order_release);
  return e;
}

inline int env_or(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

}  // namespace cvm
