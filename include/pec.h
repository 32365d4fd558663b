/*
 * pec.h — C ABI of the B200 Partial Experts Checkpointing (PEC) snapshot path.
 *
 * This is the drop-in boundary for the hot path of MoC-System's PEC snapshot
 * (arXiv 2408.04307).  The reference (`mocsim`, pure Python + numpy) has no
 * FFI: its path is the Python API listed beside each entry point below, and
 * the byte movement is *modelled* as bytes/bandwidth
 * (`pkg/src/mocsim/simulator.py:57-61`, `:434-438`).  Every entry point here
 * makes one piece of that path real on an sm_100a GPU.
 *
 * Conventions
 *   - All functions are `extern "C"`, take plain pointers and sizes, and
 *     return `int` (PEC_OK == 0, negative PEC_E_* on error) unless noted.
 *   - Device entry points are asynchronous on the given CUDA stream
 *     (`stream` is a `cudaStream_t`; NULL means the legacy default stream).
 *   - The caller owns every buffer.  The library keeps no global state and
 *     never allocates device memory.
 *   - Argument validation happens on the host before any launch; a bad
 *     table is rejected with PEC_E_INVAL, never discovered by a fault.
 */
#ifndef PEC_H_
#define PEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PEC_OK 0
#define PEC_E_INVAL (-1)   /* bad argument (maps to SpecValidationError / ValueError) */
#define PEC_E_CUDA (-2)    /* CUDA launch or runtime error (maps to RuntimeError)   */
#define PEC_E_RANGE (-3)   /* size exceeds a kernel limit (e.g. experts > 4096)     */
#define PEC_E_IO (-4)      /* file I/O failed (maps to OSError)                      */
#define PEC_E_CRASH (-5)   /* injected crash: write budget exhausted (CrashPoint)    */

#define PEC_ABI_VERSION 1

/* One contiguous byte copy of a gather/scatter table.  `first_chunk` is the
 * exclusive prefix sum of ceil(nbytes / 2^chunk_log2) over the table; fill it
 * with pec_plan_chunks().  Tables passed to pec_pack/pec_unpack live in
 * DEVICE memory; 32-byte entries, 8-byte aligned. */
typedef struct pec_copy_desc {
  uint64_t src;          /* device address of the first source byte       */
  uint64_t dst;          /* device address of the first destination byte  */
  uint64_t nbytes;       /* bytes to copy (0 allowed)                      */
  uint64_t first_chunk;  /* index of this descriptor's first work chunk    */
} pec_copy_desc;

/* ABI version of the loaded library (== PEC_ABI_VERSION it was built with). */
int pec_abi_version(void);

/* Human-readable text for a PEC_* return code (static storage). */
const char* pec_strerror(int code);

/* ---- (a) per-expert token counting ------------------------------------ *
 * Replaces: route_tokens' bincount + capacity cap
 *   (pkg/src/mocsim/simulator.py:88-95) and the per-iteration accumulation
 *   into the ledger and both LoadCounters tiers (simulator.py:560-567,
 *   selector.py:83-84).
 * idx       [L][n_per_layer] int32 router top-k expert ids of ONE iteration;
 *           ids outside [0, E) are ignored (dropped tokens).
 * cap       [L] int64 per-layer capacity (the ceil(cf*total/N) cap), or NULL.
 * counters  [tiers][L][E] int64, += min(count, cap) for every tier.
 * delivered [L][E] int64 or NULL, += min(count, cap).
 * scratch   [L*E + 1] uint32, all ZERO on entry; left zero on exit.
 * Limits: 1 <= E <= 4096, 1 <= L <= 65535. */
int pec_token_hist(const int32_t* idx, int L, int64_t n_per_layer, int E,
                   const int64_t* cap, int64_t* counters, int tiers,
                   int64_t* delivered, uint32_t* scratch, void* stream);

/* Same with int64 ids (torch.topk's index dtype: no conversion pass). */
int pec_token_hist_i64(const int64_t* idx, int L, int64_t n_per_layer, int E,
                       const int64_t* cap, int64_t* counters, int tiers,
                       int64_t* delivered, uint32_t* scratch, void* stream);

/* ---- (b) K_pec expert selection --------------------------------------- *
 * Replaces: select_window / select_sequential (selector.py:21-32).
 * Writes, for each layer m, the set {(m + c*stride + j) mod E : j < width}
 * (all E experts when width >= E) sorted ascending into out[m][0..W), with
 * W = min(width, E).  out is [L][W] int32 device memory. */
int pec_select_sequential(int64_t c, int L, int E, int width, int stride,
                          int32_t* out, void* stream);

/* Replaces: select_load_aware (selector.py:91-100) + LoadCounters.mark_saved
 *   (selector.py:86-88) as used by Simulation._selections / _trigger_checkpoint
 *   (simulator.py:339-354, :425-432).
 * Per layer: the min(K, |pool|) candidates with the largest counters
 * [L][E] int64 (token counts, >= 0), ties to the lowest expert id; pool
 * duplicates count once; written sorted ascending into
 * out [L][K] (unused slots = -1).  pool [L][P] int32 restricts candidates
 * (entries outside [0,E) are skipped), or NULL for all E experts.  With
 * zero_selected != 0 the selected counters are reset to 0 in place. */
int pec_select_load_aware(int64_t* counters, int L, int E, int K,
                          const int32_t* pool, int P, int32_t* out,
                          int zero_selected, void* stream);

/* ---- (c) pack: state -> contiguous staging --------------------------- *
 * Replaces: the modelled snapshot transfer_us(snap_bytes, bw)
 *   (simulator.py:57-61, :434-438) over the per-rank ranges of
 *   build_phase_assignment (planner.py:263-295).
 * descs: DEVICE table of n copies (src = state, dst = staging), chunk
 * prefix filled by pec_plan_chunks with the same chunk_log2 (12..24).
 * mode: 0 = auto (TMA bulk), 1 = vectorised LDG/STG.128 engine, 2 = TMA bulk
 * (cp.async.bulk) engine; 10-23 = bulk ring/occupancy/narrow-grid variants (benchmarking).  Ranges may be byte-granular; the fast path needs
 * src == dst (mod 16), which the staging layout guarantees. */
int pec_pack(const pec_copy_desc* descs, int n, uint64_t total_chunks,
             int chunk_log2, int mode, void* stream);

/* ---- (d) restore scatter: staging -> state ----------------------------- *
 * Replaces: the byte side of recovery, DiskStore.load_checkpoint
 *   (store.py:267-282) + resolve_recovery decisions (engine.py:231-284).
 * Same table format with src = staging, dst = state. */
int pec_unpack(const pec_copy_desc* descs, int n, uint64_t total_chunks,
               int chunk_log2, int mode, void* stream);

/* ---- device-side plan expansion (load-aware, no host round trip) ------ *
 * Replaces: the per-checkpoint build_phase_assignment (planner.py:263-295,
 * called from simulator.py:402-406 for load-aware selection) for one rank,
 * for strategies whose non-expert placement does not depend on the due set
 * (equal_pec, baseline).  tmpl is the rank's entry list with every expert
 * due (planner order); entries with layer < 0 are always saved.  sel is the
 * device selection [L][K] (pec_select_load_aware output).  Writes out[n]
 * (dropped entries get nbytes 0) and totals[0] = chunks, totals[1] = staged
 * bytes; staging offsets follow the StagingLayout rule (>= previous end,
 * == src_offset mod stage_align).  All device memory; async. */
typedef struct pec_plan_template {
  uint64_t src_offset;  /* byte offset of the range in the state arena */
  uint64_t nbytes;
  int32_t layer;        /* MoE layer, or -1 for always-saved entries */
  int32_t expert;
  uint64_t reserved;
} pec_plan_template;

int pec_expand_plan(const pec_plan_template* tmpl, int n, const int32_t* sel, int L, int K,
                    uint64_t state_base, uint64_t stage_base, int chunk_log2, int stage_align,
                    pec_copy_desc* out, uint64_t* totals, void* stream);

/* pec_pack over a device-built table whose chunk count lives in device
 * memory (*total_chunks_dev, e.g. totals[0] of pec_expand_plan); max_chunks
 * bounds the launch. */
int pec_pack_indirect(const pec_copy_desc* descs, int n, uint64_t max_chunks,
                      const uint64_t* total_chunks_dev, int chunk_log2, int mode, void* stream);

/* ---- pack with fused CRC-32C ------------------ *
 * Replaces: the host CRC of every persisted entry (store.crc32c,
 * store.py:49-70, used for the manifest at store.py:213-216).
 * Same copy as pec_pack (TMA bulk ring per warp) and, in the same pass over
 * the bytes, entry_crc[i] = CRC-32C of descriptor i's nbytes (== pec_crc32c
 * of the staged entry).  chunk_log2 must be 15; chunk_crc is device scratch
 * of total_chunks + 1 uint32 (one per 32 KiB chunk, plus the kernel's work
 * counter); entry_crc is device memory of n uint32.
 * total_chunks_dev (nullable) caps the chunk count from device memory, as in
 * pec_pack_indirect (device-expanded plans). */
int pec_pack_crc(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                 const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                 uint32_t* entry_crc, void* stream);

/* CRC-32C of device ranges without copying them: entry_crc[i] = CRC-32C of
 * [descs[i].src, +nbytes) (dst is ignored).  Same scratch and chunking as
 * pec_pack_crc.  Used to verify restored entries in device memory before
 * they are scattered into the state (store.py:267-282 verifies every entry
 * before load_checkpoint returns any bytes). */
int pec_crc_device(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                   const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                   uint32_t* entry_crc, void* stream);

/* Host helper: fill first_chunk of a HOST table in place and return the
 * total chunk count (negative PEC_E_* on bad input). */
int64_t pec_plan_chunks(pec_copy_desc* host_descs, int n, int chunk_log2);

/* ---- host CRC-32C (persist) ------------------------------------------- *
 * Replaces: store.crc32c (store.py:49-70), Castagnoli, reflected poly
 * 0x82F63B78, crc32c(data, crc) semantics identical (chainable):
 * pec_crc32c("123456789", 9, 0) == 0xE3069283, pec_crc32c(p, 0, 0) == 0. */
uint32_t pec_crc32c(const void* data, size_t n, uint32_t crc);

/* CRC of concatenation A||B from crc(A), crc(B) and len(B). */
uint32_t pec_crc32c_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b);

/* CRC-32C of n host regions [base+offs[i], +lens[i]) into out[i], using up
 * to `threads` host threads (large regions are split and combined). */
int pec_crc32c_many(const void* base, const uint64_t* offs,
                    const uint64_t* lens, int n, uint32_t* out, int threads);

/* ---- native persist writer -------------------- *
 * Replaces: the entry-file loop of DiskStore.write_version (store.py:210-216).
 * Writes file i = lens[i] bytes from host buffer bufs[i] with a pool of up to
 * `threads` threads (whole files per thread, largest first, 4 MiB pwrites;
 * with O_DIRECT, files above 64 MiB are split into 64 MiB ranges written by
 * different threads at their offsets); with crc_out != NULL also returns
 * each file's CRC-32C, computed per piece right after writing it.  flags
 * bit 0: fsync each file; bit 1: O_DIRECT (4 KiB-aligned bounce buffer, last
 * block zero-padded then truncated back; buffered where the filesystem
 * refuses O_DIRECT); bit 2: writer threads at background priority (nice
 * +10); bit 3: overwrite existing files in place (sized to the new length,
 * pages kept) instead of truncating them.  PEC_E_IO on any
 * open/write/fsync/truncate/close failure. */
int pec_write_files(const char* const* paths, const void* const* bufs, const uint64_t* lens,
                    int n, uint32_t* crc_out, int threads, int flags);

/* Crash injection on the native writer.
 * Replaces: TruncatingInjector.write over the entry-file loop
 * (store.py:124-146, 210-216).  *budget bytes are spent in the given file
 * order as the sequential writer spends them: every file that fits is
 * written whole; the first that does not keeps its first *budget bytes and
 * the files after it are not created; *budget is left at the bytes unspent
 * and PEC_E_CRASH is returned (PEC_OK when every file fit).  The surviving
 * prefix is written by the same parallel pool as pec_write_files, so the
 * partial tree is identical to the sequential writer's.  crc_out (may be
 * NULL) is filled only on PEC_OK. */
int pec_write_files_budget(const char* const* paths, const void* const* bufs,
                           const uint64_t* lens, int n, uint32_t* crc_out, int threads,
                           int flags, uint64_t* budget);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* PEC_H_ */
