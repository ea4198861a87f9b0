/*
 * cvm_gpu.h -- C ABI of the B200-native batched TFHE gate-bootstrapping
 * backend (libcvm_b200.so).  Plain pointers and sizes only; no torch/CUDA types.
 *
 * Drop-in boundary.  The reference's gate seam is the abstract C++ class
 * cryptovm::Backend (/root/reference/proj/core/include/cryptovm/gates.hpp:109-132):
 * every functional unit (alu.cpp), Word helper (word.cpp) and the emulator
 * (emulator.cpp) reach gates only through it.  A GPU backend replacing
 * SimBackend (sim_backend.hpp:33-71) binds the entry points below; the shim a
 * maintainer adds to the reference tree is shown in INTEGRATION.md.  Each entry
 * point names the reference interface it replaces.
 *
 * Conventions.  Every function returns CVM_OK (0) or a negative cvm_status;
 * the message of the last failure on the calling thread is cvm_last_error().
 * CVM_E_INPUT mirrors the reference's cryptovm::InputError (bad handle, bad
 * gate kind, bad blob: sim_backend.cpp:47-49,53-57,80-83,124-126); CVM_E_DEVICE
 * mirrors cryptovm::Error for device failures (errors.hpp:24-58).  There is no
 * CPU fallback: without a usable sm_100a device, cvm_ctx_create fails.
 */
#ifndef CVM_GPU_H_
#define CVM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVM_API __attribute__((visibility("default")))

typedef enum cvm_status {
  CVM_OK = 0,
  CVM_E_INPUT = -1,       /* precondition violated (cryptovm::InputError)  */
  CVM_E_DEVICE = -2,      /* CUDA failure / no sm_100a device              */
  CVM_E_STATE = -3,       /* call out of order (e.g. gates before keys)    */
  CVM_E_NOMEM = -4
} cvm_status;

/* Parameter set (TFHE default gate bootstrapping; BASELINE.json configs[0]). */
#define CVM_LWE_N 630
#define CVM_POLY_N 1024
#define CVM_LWE_WORDS 631                    /* a[0..629], b : 2,524 B       */
#define CVM_BK_WORDS (630u * 6u * 2u * 1024u) /* bk[i][row][poly][coef] u32   */
#define CVM_KSK_WORDS (1024u * 8u * 4u * 631u) /* ksk[i][j][v][631] u32       */

/* Gate kinds = cryptovm::GateKind enumerators (gates.hpp:31-46). */
typedef enum cvm_gate_kind {
  CVM_CONSTANT = 0, CVM_NOT = 1, CVM_COPY = 2, CVM_NAND = 3, CVM_AND = 4,
  CVM_OR = 5, CVM_XOR = 6, CVM_XNOR = 7, CVM_NOR = 8, CVM_ANDNY = 9,
  CVM_ANDYN = 10, CVM_ORNY = 11, CVM_ORYN = 12, CVM_MUX = 13
} cvm_gate_kind;

CVM_API const char* cvm_last_error(void);
CVM_API const char* cvm_version(void);

/* ------------------------------------------------------------------------
 * Key owner (host).  Keygen / encrypt / decrypt stay on the host, as in the
 * reference: Backend::encrypt_bit / decrypt_bit (gates.hpp:120-121),
 * SimBackend::encrypt_bit / decrypt_bit (sim_backend.cpp:108-116),
 * Word::encrypt / decrypt_word (word.cpp:42-86).
 * ---------------------------------------------------------------------- */
typedef struct cvm_keyset cvm_keyset;
CVM_API int cvm_keyset_generate(uint64_t seed, cvm_keyset** out);
CVM_API void cvm_keyset_destroy(cvm_keyset* ks);
/* Export key material (lwe_key 630 i32, tlwe_key 1024 i32, bk, ksk u32). */
CVM_API int cvm_keyset_export(const cvm_keyset* ks, int32_t* lwe_key,
                              int32_t* tlwe_key, uint32_t* bk, uint32_t* ksk);
/* Fresh encryptions of `count` bits (one seeded noise stream per call). */
CVM_API int cvm_encrypt_bits(const cvm_keyset* ks, uint64_t seed, size_t count,
                             const uint8_t* bits, uint32_t* out_lwe);
CVM_API int cvm_decrypt_bits(const cvm_keyset* ks, size_t count,
                             const uint32_t* lwe, uint8_t* bits, int32_t* phases);

/* ------------------------------------------------------------------------
 * Device context: one CUDA stream, bootstrapping key resident in HBM in FFT
 * domain (59 MiB), key-switching key resident (79 MiB), a slab of LWE slots.
 * ---------------------------------------------------------------------- */
typedef struct cvm_ctx cvm_ctx;
CVM_API int cvm_ctx_create(int device, cvm_ctx** out);
CVM_API void cvm_ctx_destroy(cvm_ctx* ctx);
/* Upload BK (time domain, CVM_BK_WORDS) and KSK (CVM_KSK_WORDS) once; the BK
 * is transformed to the FFT domain on the device. */
CVM_API int cvm_upload_keys(cvm_ctx* ctx, const uint32_t* bk, const uint32_t* ksk);
CVM_API int cvm_upload_keyset(cvm_ctx* ctx, const cvm_keyset* ks);
/* Hand out `n` fresh slot ids (bump allocator shared by every backend on the
 * context); capacity follows at the next reserve or flush. */
CVM_API int cvm_slots_alloc(cvm_ctx* ctx, uint64_t n, uint64_t* first);
/* Ensure capacity for `n` LWE slots (slot ids 0..n-1). */
CVM_API int cvm_slots_reserve(cvm_ctx* ctx, uint64_t n);
CVM_API uint64_t cvm_slots_capacity(const cvm_ctx* ctx);
/* Host <-> device ciphertext transfer, 631 u32 per slot, stream-ordered. */
CVM_API int cvm_upload_lwe(cvm_ctx* ctx, uint64_t slot, uint64_t count,
                           const uint32_t* lwe);
CVM_API int cvm_download_lwe(cvm_ctx* ctx, uint64_t slot, uint64_t count,
                             uint32_t* lwe);

/* A gate operand is a linear form  sign * slot + constant  (torus32): NOT,
 * COPY and CONSTANT (gates.hpp:113-114, sim_backend.cpp:75-88) fold into it,
 * so only bootstrapped gates reach the device. slot < 0: pure constant. */
typedef struct cvm_operand {
  int64_t slot;
  int32_t sign;       /* +1 or -1 */
  uint32_t constant;  /* added to the b word */
} cvm_operand;

/* One bootstrapped gate: Backend::binary_gate (gates.hpp:115) for kinds
 * NAND..ORYN with in[0], in[1]; Backend::mux_gate (gates.hpp:116-118) for MUX
 * with in[0]=sel, in[1]=on_true, in[2]=on_false. */
typedef struct cvm_gate {
  uint32_t kind;
  uint32_t pad;
  cvm_operand in[3];
  uint64_t out_slot;
} cvm_gate;

/* Enqueue one dataflow level: `count` mutually independent gates whose inputs
 * are slots written by earlier levels or uploads.  Asynchronous. */
CVM_API int cvm_submit_level(cvm_ctx* ctx, const cvm_gate* gates, uint64_t count);
/* Wait for everything enqueued on the context. */
CVM_API int cvm_sync(cvm_ctx* ctx);

/* Kernel accounting: when enabled, each launch is bracketed by CUDA events on
 * the context stream; totals are resolved at cvm_sync. */
typedef struct cvm_kernel_stats {
  uint64_t br_launches, br_jobs;   /* blind rotations (bootstraps)       */
  uint64_t ks_launches, ks_jobs;   /* key switches                       */
  uint64_t other_launches;
  double br_ms, ks_ms;             /* summed event time                  */
} cvm_kernel_stats;
CVM_API int cvm_ctx_set_profiling(cvm_ctx* ctx, int enabled);
CVM_API int cvm_ctx_kernel_stats(cvm_ctx* ctx, cvm_kernel_stats* out);
CVM_API int cvm_ctx_reset_stats(cvm_ctx* ctx);
/* Device-resident scratch write larger than L2 (for cold-cache timing). */
CVM_API int cvm_ctx_flush_l2(cvm_ctx* ctx);
/* Time a region on the context stream with CUDA events. */
CVM_API int cvm_ctx_event_record(cvm_ctx* ctx, int which);  /* 0 start, 1 stop */
CVM_API int cvm_ctx_event_elapsed_ms(cvm_ctx* ctx, double* ms);
/* Measured FP64 FMA-pipe peak of this device in TFLOP/s (roofline denominator
 * of the blind-rotation kernel) and its SM count. */
CVM_API int cvm_ctx_fp64_peak(cvm_ctx* ctx, int reps, double* tflops);
CVM_API int cvm_ctx_sm_count(cvm_ctx* ctx, int* sms);
/* Blind-rotation kernel variant (process-wide default; a context may
 * override it, cvm_ctx_set_kernels).  Every variant computes bit-identical
 * ciphertexts:
 *   6000 + 10*W + 5 (W = 1..8; 6085 = 8 warps): v4, one bootstrap per warp on
 *        the warp-wide FFT, W warps per CTA sharing a 5-row key ring
 *        (throughput; full waves of wide levels);
 *   5247: v3, four bootstraps per CTA on the 64-thread FFT, 7-row key ring
 *        (remainder rounds of wide levels);
 *   9:   one bootstrap per SM, the six gadget rows transformed concurrently;
 *   96:  one bootstrap per 2-SM thread-block cluster, partial products
 *        exchanged by st.async (latency: levels up to 74 bootstraps);
 *   0:   auto (default): 96 up to 74 bootstraps, 9 up to 296, else full v4
 *        waves with the remainder on the cheapest mix of one v4 wave, 5247
 *        rounds and 9 rounds. */
CVM_API int cvm_set_br_variant(int variant);
CVM_API int cvm_get_br_variant(void);
/* Wave packing of the levelizer (process-wide, default 1; env CVM_PACK=0):
 * a flush keeps its number of launches (the critical path), but each gate may
 * run in any launch between its earliest and latest dataflow level, and the
 * launches are filled to the widths the blind-rotation kernels run most
 * efficiently.  Results are unchanged (gates are pure); 0 = plain levels. */
CVM_API int cvm_set_level_packing(int on);
CVM_API int cvm_get_level_packing(void);
/* Key-switch kernel variant (process-wide default): 8 = the level as one
 * INT8 tcgen05.mma product (one-hot digits x KSK byte limbs, TMEM
 * accumulators), one CTA per 128-gate x 128-column tile; 9 = the same tiles
 * split along K into up to 16 CTAs plus a reduction; 0 = auto (9).
 * Bit-identical. */
CVM_API int cvm_set_ks_variant(int variant);
CVM_API int cvm_get_ks_variant(void);
/* Per-context kernel choices: a blind-rotation variant, a key-switch variant
 * and wave packing on (1) / off (0); -1 follows the process-wide setting
 * (the default for a new context).  Invalid values -> CVM_E_INPUT. */
CVM_API int cvm_ctx_set_kernels(cvm_ctx* ctx, int br_variant, int ks_variant,
                                int level_packing);
CVM_API int cvm_ctx_get_kernels(cvm_ctx* ctx, int* br_variant, int* ks_variant,
                                int* level_packing);

/* ------------------------------------------------------------------------
 * Backend: the cryptovm::Backend contract (gates.hpp:109-132) over a context.
 * Gate calls return handles immediately (lazy recording); evaluation happens
 * in dataflow levels at flush points: decrypt/export, or cvm_backend_flush.
 * Handles are dense 1-based node ids like the reference's GateDag
 * (dag.cpp:57-73); 0 is the invalid handle (BitHandle::valid(), gates.hpp:95).
 * ---------------------------------------------------------------------- */
typedef struct cvm_backend cvm_backend;
typedef uint64_t cvm_handle;
CVM_API int cvm_backend_create(cvm_ctx* ctx, const cvm_keyset* owner,
                               uint64_t enc_seed, cvm_backend** out);
CVM_API void cvm_backend_destroy(cvm_backend* b);
CVM_API int cvm_backend_constant(cvm_backend* b, int value, cvm_handle* out);
CVM_API int cvm_backend_unary_gate(cvm_backend* b, uint32_t kind, cvm_handle a,
                                   cvm_handle* out);
CVM_API int cvm_backend_binary_gate(cvm_backend* b, uint32_t kind, cvm_handle a,
                                    cvm_handle c, cvm_handle* out);
CVM_API int cvm_backend_mux_gate(cvm_backend* b, cvm_handle sel, cvm_handle on_true,
                                 cvm_handle on_false, cvm_handle* out);
CVM_API int cvm_backend_encrypt_bit(cvm_backend* b, int value, cvm_handle* out);
CVM_API int cvm_backend_decrypt_bit(cvm_backend* b, cvm_handle h, int* value);
/* Batched key-owner decryption: one flush, one download. */
CVM_API int cvm_backend_decrypt_bits(cvm_backend* b, size_t count,
                                     const cvm_handle* hs, uint8_t* values);
/* Import existing ciphertexts (631 u32 each) as fresh input handles. */
CVM_API int cvm_backend_import_lwe(cvm_backend* b, size_t count,
                                   const uint32_t* lwe, cvm_handle* out);
CVM_API int cvm_backend_export_lwe(cvm_backend* b, size_t count,
                                   const cvm_handle* hs, uint32_t* lwe);
/* export_bit / import_bit: 2,524-byte little-endian blob (631 x u32). */
CVM_API int cvm_backend_export_bit(cvm_backend* b, cvm_handle h, uint8_t* blob,
                                   size_t blob_size);
CVM_API int cvm_backend_import_bit(cvm_backend* b, const uint8_t* blob,
                                   size_t blob_size, cvm_handle* out);
CVM_API int cvm_backend_push_region(cvm_backend* b, const char* name);
CVM_API int cvm_backend_pop_region(cvm_backend* b);
CVM_API int cvm_backend_fence(cvm_backend* b);
CVM_API int cvm_backend_flush(cvm_backend* b);
/* Flush policy of decrypt/export: CVM_FLUSH_CONE (default) evaluates only the
 * cone of influence of the requested handles -- dead gates are never run;
 * CVM_FLUSH_ALL evaluates everything pending at the first decrypt, for callers
 * that decrypt one bit at a time (the reference's decrypt_word, word.cpp:70-77). */
#define CVM_FLUSH_CONE 0
#define CVM_FLUSH_ALL 1
CVM_API int cvm_backend_set_flush_policy(cvm_backend* b, int policy);

/* Plans: the backend's pending (unflushed) levels moved into a reusable object
 * with device-resident job tables -- a recorded circuit that can be replayed
 * on new inputs written into the same input slots (cvm_upload_lwe), either as
 * plain launches or as one CUDA graph.  Pending uploads are enqueued at
 * capture; results land in the same slots on every run. */
typedef struct cvm_plan cvm_plan;
CVM_API int cvm_backend_capture_plan(cvm_backend* b, cvm_plan** out);
CVM_API int cvm_plan_run(cvm_ctx* ctx, cvm_plan* plan, int use_graph);
CVM_API int cvm_plan_info(const cvm_plan* plan, uint64_t* levels, uint64_t* gates,
                          uint64_t* bootstraps);
CVM_API void cvm_plan_destroy(cvm_plan* plan);
/* Slot id backing a handle (-1 for a pure constant); sign/constant of its
 * linear form (NOT/COPY/CONSTANT folding). */
CVM_API int cvm_backend_handle_slot(const cvm_backend* b, cvm_handle h, int64_t* slot,
                                    int32_t* sign, uint32_t* constant);

/* bootstrapped/bootstraps count recorded gates (MUX = 1 / 2), like
 * ScheduleReport.bootstrapped_count (sched.cpp:196-199); executed counts the
 * gates actually evaluated (decrypt/export evaluate only the cone of the
 * requested handles, so dead gates are skipped); pending = not yet evaluated. */
typedef struct cvm_backend_stats {
  uint64_t nodes, bootstrapped, bootstraps, levels_run, flushes, decrypts;
  uint64_t last_flush_levels, last_flush_gates, max_level_width;
  uint64_t executed, executed_bootstraps, pending;
} cvm_backend_stats;
CVM_API int cvm_backend_stats_get(const cvm_backend* b, cvm_backend_stats* out);
/* Region attribution (the reference's GateDag region labels, dag.hpp:55-70):
 * push_region / pop_region build a path ("adder/carry/level1"); every gate
 * records the path open at its recording.  Region 0 is "" (outside any
 * region).  recorded = bootstrapped gates recorded in the region, executed =
 * those evaluated so far (dead gates never are).  Flushes also emit NVTX
 * ranges per launch labelled with these regions (when a profiler is attached
 * or CVM_NVTX=1). */
CVM_API int cvm_backend_region_count(const cvm_backend* b, uint64_t* out);
CVM_API int cvm_backend_region_info(const cvm_backend* b, uint64_t idx, char* name,
                                    size_t name_size, uint64_t* recorded,
                                    uint64_t* executed);
/* Node table: kind, input flag, deps (0 = none), constant value per node id. */
CVM_API int cvm_backend_node_count(const cvm_backend* b, uint64_t* out);
CVM_API int cvm_backend_nodes(const cvm_backend* b, uint64_t first, uint64_t count,
                              int64_t* rows /* count x 7 */);

/* ------------------------------------------------------------------------
 * Recorded circuits.  The reference's functional units (alu.hpp:68-136) and
 * emulator (emulator.hpp:87-133) stay on the reference side of the boundary:
 * they record their gates once through cryptovm::Backend (the shim in
 * integration/ records into a SimBackend), and the recorded
 * table -- the reference GateDag's node list (DagNode, dag.hpp:33-42, ids
 * 1-based in creation order as GateDag::append assigns them, dag.cpp:57-73) --
 * is handed to the device here.  The reference DAG does not store a
 * CONSTANT's value; the recorder adds it.
 * ---------------------------------------------------------------------- */
typedef struct cvm_dag_node {
  uint8_t kind;     /* cvm_gate_kind (DagNode::kind)                       */
  uint8_t input;    /* 1: an encrypted input entering the session          */
                    /*    (DagNode::input: encrypt_bit / import_bit)       */
  uint8_t value;    /* CONSTANT: the constant bit                          */
  uint8_t ndeps;    /* DagNode::dep_count: 0 (CONSTANT, input), 1 (NOT,    */
                    /*    COPY), 2 (binary gates), 3 (MUX: sel, t, f)      */
  uint32_t region;  /* DagNode::region: index into the table's region     */
                    /*    names (GateDag::regions()), 0 = none             */
  uint64_t dep[3];  /* DagNode::dep: ids of earlier nodes                  */
} cvm_dag_node;

/* Re-issue a recorded table as Backend calls on `b`: input nodes take the
 * handles `inputs` in node order (n_inputs must equal the table's input
 * count), every other node becomes the gate call it records.  handles[i]
 * receives node i+1's handle (n_nodes entries).  Lazy like every gate call. */
CVM_API int cvm_backend_replay_dag(cvm_backend* b, const cvm_dag_node* nodes,
                                   uint64_t n_nodes, const cvm_handle* inputs,
                                   uint64_t n_inputs, cvm_handle* handles);
/* Region names of the tables replayed next on `b` (names[k] for region index
 * k of a node; names[0] is the unlabelled ""): replayed gates are then
 * attributed to those paths (cvm_backend_region_info, NVTX labels).  n = 0
 * clears them. */
CVM_API int cvm_backend_set_dag_regions(cvm_backend* b, const char* const* names,
                                        uint64_t n);
/* Evaluate the cone of influence of `count` handles now (one flush) and
 * download their values once into a host cache, so the key owner's later
 * bit-by-bit decryptions (word.cpp:70-77) need no device round trip each. */
CVM_API int cvm_backend_evaluate(cvm_backend* b, size_t count, const cvm_handle* hs);

/* `batch` independent instances of one recorded circuit through the public
 * path with host buffers: in_lwe is batch x n_inputs x 631 u32 (n_inputs =
 * the table's input count), out_lwe batch x n_outputs x 631 (outputs: node
 * ids).  The instances are recorded on a fresh backend, only the outputs'
 * cone is evaluated (dead gates never run), levelised launches fill the
 * GPU, results are downloaded; the call's scratch slots are returned.  The
 * element counts of both buffers are checked against the table. */
CVM_API int cvm_dag_batch(cvm_ctx* ctx, const cvm_dag_node* nodes, uint64_t n_nodes,
                          const uint64_t* outputs, uint64_t n_outputs, uint64_t batch,
                          const uint32_t* in_lwe, uint64_t in_words, uint32_t* out_lwe,
                          uint64_t out_words, cvm_backend_stats* stats);
/* The same with the table's region names (see cvm_backend_set_dag_regions),
 * so the batch's launches carry NVTX labels of the reference's regions. */
CVM_API int cvm_dag_batch_regions(cvm_ctx* ctx, const cvm_dag_node* nodes, uint64_t n_nodes,
                                  const char* const* region_names, uint64_t n_regions,
                                  const uint64_t* outputs, uint64_t n_outputs,
                                  uint64_t batch, const uint32_t* in_lwe, uint64_t in_words,
                                  uint32_t* out_lwe, uint64_t out_words,
                                  cvm_backend_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* CVM_GPU_H_ */
