// pec_crc.cu — CRC-32C of every staged entry, computed by the pack itself.
//
// the persist tier checksums each entry
// (store.crc32c, pkg/src/mocsim/store.py:49-70; the manifest column of
// store.py:149-164).  Here the pack kernel checksums the bytes on their way
// from the state arena to the staging buffer, so the host never reads the
// payload for CRC and the HBM traffic of the pack is unchanged.
//
// CRC-32C is linear over GF(2).  With the register form R (initial value 0,
// no final inversion) and little-endian 32-bit words w_0..w_{n-1} of a
// message, R(M) = XOR_i w_i * x^(32 (n - i)) mod P, R(A || B) =
// R(A) * x^(8|B|) ^ R(B), and the standard CRC is
// crc(M) = ~(R(M) ^ ~0 * x^(8|M|) mod P).
//
// pack_crc_kernel (one persistent CTA per SM, 8 warps, each warp owns whole
// 32 KiB chunks, claimed one at a time from a counter so faster SMs take more):
//   * each warp streams its chunks as 4 KiB stages through its own ring in
//     shared memory: lane 0 issues cp.async.bulk global->smem (mbarrier
//     complete_tx), then cp.async.bulk smem->global into staging — the bytes
//     never pass through registers on their way to staging;
//   * the lanes read the stage as 16-byte slots, lane l taking slot
//     l + 32 j (one 512-byte row per LDS.128: conflict-free), so lane l word
//     t of row j is message word 128 j + 4 l + t.  Each (lane, t) keeps a
//     chain S <- S * Y ^ w with Y = x^4096 (its consecutive words are 512 B
//     apart), over the 64 rows of the chunk;
//   * S * Y is four byte lookups (slicing-by-4 with tables for Y): tables
//     live in shared memory replicated 16x, tables 0/1 in banks 0-15 and
//     2/3 in banks 16-31, and the upper half-warp visits the byte positions
//     in the order 2,3,0,1 — so every lookup of a warp hits 32 distinct
//     banks.  A PRMT forms each whole lookup address (byte of S in bits 8-15,
//     the lane's bank slot in bits 0-7, the tables' 64 KiB-aligned shared
//     base in bits 16-31): 2 instructions per lookup (PRMT + LDS);
//   * per chunk, lane l joins its chains (x^(32 (4 - t))) and shifts by its
//     lane constant x^(128 (31 - l)); a XOR butterfly gives R(chunk).
//   Chunks that are partial (an entry's last) or not 16-byte aligned take a
//   byte loop per lane instead (at most one per entry for staged plans).
// crc_fold_kernel  Horner-joins the chunk registers of every entry
//   (x^(8 * 32 KiB) per chunk, one atomic per thread run).
// crc_final_kernel applies the last chunk's length, the initial value and
//   the final inversion per entry.
// Multiplication mod P (reflected, bit 31 = x^0) is the shift-and-add
// schoolbook product or, for constants, 8 lookups of 4-bit-window tables;
// every table and power (x^(2^k), chunk and byte powers) is computed by the
// compiler (constexpr make_tables) into the device image.

#include <cuda_runtime.h>
#include <stdint.h>

#include "pec.h"
#include "pec_device.cuh"

namespace {

using pecdev::as_stream;
using pecdev::launch_status;
using pecdev::sm_count;

constexpr uint32_t kPoly = 0x82F63B78u;
constexpr int kCrcLg = 15;                      // 32 KiB chunks
constexpr int kChunk = 1 << kCrcLg;
constexpr int kStageLg = 12;                    // 4 KiB stages
constexpr int kStage = 1 << kStageLg;
constexpr int kStagesPerChunk = kChunk / kStage;
constexpr int kRowsPerStage = kStage / 512;     // 512-byte rows (32 lanes x 16 B)
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kRing = 4;                        // stages per warp

__host__ __device__ constexpr uint32_t gf2_mul(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (int i = 31; i >= 0; --i) {
    if ((a >> i) & 1u) p ^= b;
    b = (b & 1u) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^nbits mod P from the x^(2^k) table
__host__ __device__ constexpr uint32_t xpow_bits(const uint32_t* x2k, uint64_t nbits) {
  uint32_t acc = 1u << 31;  // 1
  for (int k = 0; nbits; nbits >>= 1, ++k)
    if (nbits & 1u) acc = gf2_mul(x2k[k], acc);
  return acc;
}

// Every constant the CRC kernels use, computed by the compiler (constexpr)
// and stored in the device image: the kernels copy what they need into
// shared memory instead of deriving it with thousands of GF(2) products per
// launch (round-1/early round-2 kernels built them per CTA).
// The pack kernel's shared-memory tables, laid out exactly as the kernel
// uses them, so one TMA bulk copy fills them per CTA.
struct alignas(16) SmemImage {
  uint32_t ytab[256 * 64];      // entry e, table k, lane group g at word 64 e + 32 (k & 1) + 16 (k >> 1) + g
  uint32_t lanetab[8 * 16 * 32];  // lane l's 4-bit windows of x^(128 (31 - l)), [p][v][l]
  uint32_t nib4[4 * 128];       // 4-bit windows of x^(32 (4 - t)), t = 0..3
  uint32_t t8[256];             // the standard byte table (partial chunks)
  uint32_t x2k[64];             // x^(2^k) mod P
};

struct alignas(16) CrcTables {
  SmemImage img;
  uint32_t x2k[64];             // x^(2^k) mod P
  uint32_t ybase[4][256];       // slicing-by-4 tables of Y = x^4096: T_k[e] = Y * (e << 8k)
  uint32_t lanetab[8 * 16 * 32];  // lane l's 4-bit windows of x^(128 (31 - l)), [p][v][l]
  uint32_t nib4[4][128];        // 4-bit windows of x^(32 (4 - t)), t = 0..3
  uint32_t t8[256];             // the standard byte table (partial chunks)
  uint32_t chunk_nib[128];      // 4-bit windows of x^(8 * 32 KiB)
  uint32_t chunk_pw[3][256];    // x^(8 * 32 KiB * t * 256^r)
  uint32_t byte_pw[5][256];     // x^(8 * t * 256^r)
};

constexpr CrcTables make_tables() {
  CrcTables t{};
  uint32_t p = 1u << 30;  // x^1
  for (int i = 0; i < 64; ++i) {
    t.x2k[i] = p;
    p = gf2_mul(p, p);
  }
  const uint32_t y = t.x2k[12];  // x^4096
  for (int k = 0; k < 4; ++k)
    for (int e = 0; e < 256; ++e) t.ybase[k][e] = gf2_mul(y, (uint32_t)e << (8 * k));
  uint32_t lconst[32] = {};
  for (int l = 0; l < 32; ++l) lconst[l] = xpow_bits(t.x2k, 128ull * (31 - l));
  for (int idx = 0; idx < 8 * 16 * 32; ++idx) {
    const int l = idx & 31, pv = idx >> 5, pp = pv >> 4, v = pv & 15;
    t.lanetab[idx] = gf2_mul(lconst[l], (uint32_t)v << (4 * pp));
  }
  for (int c = 0; c < 4; ++c) {
    const uint32_t m = xpow_bits(t.x2k, 32ull * (4 - c));
    for (int w = 0; w < 128; ++w) t.nib4[c][w] = gf2_mul(m, (uint32_t)(w & 15) << (4 * (w >> 4)));
  }
  for (int e = 0; e < 256; ++e) {
    uint32_t c = (uint32_t)e;
    for (int b = 0; b < 8; ++b) c = (c & 1u) ? (c >> 1) ^ kPoly : c >> 1;
    t.t8[e] = c;
  }
  for (int idx = 0; idx < 256 * 64; ++idx)   // 16x replicated, tables 0/1 and 2/3 in bank halves
    t.img.ytab[idx] = t.ybase[((idx >> 5) & 1) | (((idx >> 4) & 1) << 1)][idx >> 6];
  for (int idx = 0; idx < 8 * 16 * 32; ++idx) t.img.lanetab[idx] = t.lanetab[idx];
  for (int idx = 0; idx < 4 * 128; ++idx) t.img.nib4[idx] = t.nib4[idx >> 7][idx & 127];
  for (int e = 0; e < 256; ++e) t.img.t8[e] = t.t8[e];
  for (int i = 0; i < 64; ++i) t.img.x2k[i] = t.x2k[i];
  const uint32_t chunk = xpow_bits(t.x2k, (uint64_t)kChunk * 8);
  for (int w = 0; w < 128; ++w) t.chunk_nib[w] = gf2_mul(chunk, (uint32_t)(w & 15) << (4 * (w >> 4)));
  for (int r = 0; r < 3; ++r) {
    const uint32_t base = xpow_bits(t.x2k, ((uint64_t)kChunk * 8) << (8 * r));
    uint32_t acc = 1u << 31;
    for (int e = 0; e < 256; ++e, acc = gf2_mul(acc, base)) t.chunk_pw[r][e] = acc;
  }
  for (int r = 0; r < 5; ++r) {
    const uint32_t base = xpow_bits(t.x2k, 8ull << (8 * r));
    uint32_t acc = 1u << 31;
    for (int e = 0; e < 256; ++e, acc = gf2_mul(acc, base)) t.byte_pw[r][e] = acc;
  }
  return t;
}

__device__ const CrcTables kTab = make_tables();

// x^(8 n) mod P: five byte-power lookups for n < 2^40, the x^(2^k) walk above
__device__ __forceinline__ uint32_t xpow_bytes(uint64_t n) {
  if (n >> 40) return xpow_bits(kTab.x2k, n << 3);
  uint32_t acc = __ldg(&kTab.byte_pw[0][n & 255]);
  for (int r = 1; r < 5 && (n >> (8 * r)); ++r)
    acc = gf2_mul(acc, __ldg(&kTab.byte_pw[r][(n >> (8 * r)) & 255]));
  return acc;
}

__device__ __forceinline__ uint32_t shift_bytes(uint32_t r, uint64_t n) {
  return n ? gf2_mul(xpow_bytes(n), r) : r;
}

__device__ __forceinline__ uint32_t mul_const(const uint32_t* nib, uint32_t b) {
  uint32_t r = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) r ^= nib[p * 16 + ((b >> (4 * p)) & 15u)];
  return r;
}

// ---- TMA bulk helpers (as in pec_kernels.cu) ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}"
      :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* smem, const void* gmem, uint32_t bytes,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes,
                                         uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               :: "l"(gmem), "r"(smem_u32(smem)), "r"(bytes), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- shared-memory layout of pack_crc_kernel (dynamic, bytes) --------------
// The Y tables sit at shared-window address kYtabAddr (64 KiB-aligned), so a
// lookup address is ONE PRMT of (S, slot): byte 0 the lane's bank slot,
// byte 1 byte k of S, bytes 2-3 the table base carried in the slot register,
// and the LDS needs no add (PRMT + LDS per lookup instead of PRMT + IADD + LDS).
//   smem + 0      misc: lanetab 8 x 16 windows x 32 lanes of x^(128 (31 - l))
//                 (16 KiB), nib 4 x 128 windows of x^(32 (4 - t)) (2 KiB), t8 the
//                 standard byte table (1 KiB), x2k (256 B)
//   + kMiscBytes  bars: kWarps x kRing mbarriers
//   + kPreOff     rings of warps 0 .. kPreRings-1 (kRing x 4 KiB each)
//   kYtabAddr     ytab 256 entries x 64 words: entry e, table k, lane group g
//                 at word 64 e + 32 (k & 1) + 16 (k >> 1) + g   (64 KiB)
//   + 64 KiB      rings of the other warps
constexpr int kYtabWords = 256 * 64;
constexpr int kLaneTabWords = 8 * 16 * 32;
constexpr int kNibWords = 4 * 128;
static_assert(sizeof(SmemImage) == (size_t)(kYtabWords + kLaneTabWords + kNibWords + 256 + 64) * 4,
              "shared-memory table image layout");
static_assert(sizeof(SmemImage) % 16 == 0, "TMA bulk copies move multiples of 16 bytes");
constexpr uint32_t kYtabBytes = (uint32_t)kYtabWords * 4;
constexpr uint32_t kMiscBytes = (uint32_t)sizeof(SmemImage) - kYtabBytes;
constexpr uint32_t kRingBytes = (uint32_t)kRing * kStage;
constexpr int kPreRings = 2;
constexpr uint32_t kPreOff = (kMiscBytes + (uint32_t)kWarps * kRing * 8 + 127) / 128 * 128;
constexpr uint32_t kYtabAddr = 0x10000;
static_assert(kPreOff + kPreRings * kRingBytes < kYtabAddr, "ytab placement");
// worst case (dynamic window starting at shared address 0): up to the end of the last ring
constexpr size_t kSmemBytes = (size_t)kYtabAddr + kYtabBytes + (size_t)(kWarps - kPreRings) * kRingBytes;
static_assert(kSmemBytes <= 227 * 1024 - 1024, "dynamic shared memory budget");
static_assert(kMiscBytes % 16 == 0 && kYtabBytes % 16 == 0, "bulk-copy sizes");

// One chain step S * Y ^ w: four table lookups whose shared addresses are
// formed by one PRMT each (see the layout above).
__device__ __forceinline__ uint32_t ystep(uint32_t S, uint32_t w, const uint32_t (&slot)[4],
                                          const uint32_t (&sel)[4]) {
  uint32_t a[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint32_t addr = __byte_perm(S, slot[s], sel[s]);
    asm("ld.shared.u32 %0, [%1];" : "=r"(a[s]) : "r"(addr));
  }
  return a[0] ^ a[1] ^ a[2] ^ a[3] ^ w;
}

constexpr int kQueue = 2;   // claimed chunks queued per warp (few: claims held ahead unbalance the tail)

struct QueueEntry {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t ch;
  uint32_t len;
  uint32_t fast;
};

struct ChunkRef {
  const uint8_t* src;
  uint8_t* dst;
  uint32_t len;
  bool fast;   // full 32 KiB, src and dst 16-byte aligned
};

__device__ __forceinline__ ChunkRef chunk_ref(const pec_copy_desc* __restrict__ d, int n,
                                              uint64_t ch, pecdev::DescCursor& cur) {
  ChunkRef r;
  const int i = cur.find(d, n, ch);
  const uint64_t off = (ch - __ldg(&d[i].first_chunk)) << kCrcLg;
  const uint64_t nb = __ldg(&d[i].nbytes);
  r.len = off >= nb ? 0u : (uint32_t)(nb - off < (uint64_t)kChunk ? nb - off : kChunk);
  // a chunk index past its descriptor's bytes only exists for empty rows
  PEC_DCHECK(off < nb || nb == 0 || i + 1 == n);
  r.src = reinterpret_cast<const uint8_t*>(__ldg(&d[i].src) + off);
  r.dst = reinterpret_cast<uint8_t*>(__ldg(&d[i].dst) + off);
  r.fast = r.len == (uint32_t)kChunk &&
           ((reinterpret_cast<uintptr_t>(r.src) | reinterpret_cast<uintptr_t>(r.dst)) & 15u) == 0;
  return r;
}

template <bool kStore>
__global__ void __launch_bounds__(kThreads, 1)
pack_crc_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                const uint64_t* __restrict__ total_dev, uint32_t* __restrict__ chunk_raw) {
  const uint64_t total_cap = total;       // scratch is sized for the launch bound
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  // the layout needs the dynamic window to start below kYtabAddr - kPreOff -
  // kPreRings rings (it starts after ~2 KiB of static + reserved shared memory)
  if (sbase + kPreOff + kPreRings * kRingBytes > kYtabAddr) __trap();
  uint32_t* lanetab = reinterpret_cast<uint32_t*>(smem);
  uint32_t* nib = lanetab + kLaneTabWords;
  uint32_t* t8 = nib + kNibWords;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kMiscBytes);
  uint8_t* ytab = smem + (kYtabAddr - sbase);
  __shared__ QueueEntry queue[kWarps * kQueue];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (total_dev != nullptr) {
    const uint64_t td = *total_dev;
    total = td < total ? td : total;
  }
  // ---- tables: one TMA bulk copy of the compile-time image ---------------------
  __shared__ __align__(8) uint64_t table_bar;
  if (tid == 0) {
    for (int s = 0; s < kWarps * kRing; ++s) mbar_init(&bars[s], 1);
    mbar_init(&table_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&table_bar, (uint32_t)sizeof(SmemImage));
    bulk_g2s_plain(ytab, kTab.img.ytab, kYtabBytes, &table_bar);
    bulk_g2s_plain(smem, kTab.img.lanetab, kMiscBytes, &table_bar);
  }
  mbar_wait(&table_bar, 0);

  // ---- per-lane lookup geometry ----------------------------------------------
  // step s: the lower half-warp reads byte s of S from table s, the upper
  // half byte s ^ 2 from table s ^ 2; table k sits in the 32-word block k & 1
  // at half k >> 1, so both halves of a warp always hit disjoint banks.
  const uint32_t h = (uint32_t)lane >> 4, g = (uint32_t)lane & 15u;
  uint32_t slot[4], sel[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint32_t tk = (uint32_t)s ^ (h << 1);
    slot[s] = ((tk & 1u) << 7) | ((tk >> 1) << 6) | (g << 2);
    slot[s] |= kYtabAddr;          // the table base rides in bytes 2-3
    sel[s] = 0x7604u | (tk << 4);  // byte0 <- slot, byte1 <- S.byte[tk], bytes 2-3 <- slot
  }
  const uint32_t* ltab = lanetab + lane;

  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  uint8_t* my_ring = warp < kPreRings ? smem + kPreOff + (size_t)warp * kRingBytes
                                       : ytab + kYtabBytes + (size_t)(warp - kPreRings) * kRingBytes;
  uint64_t* my_bars = bars + warp * kRing;
  QueueEntry* q = queue + warp * kQueue;
  // chunks are claimed dynamically from a counter (slot `total` of the
  // scratch, zeroed before the launch): SMs that stream faster take more.
  // Lane 0 keeps one claim in flight (`res`) so the atomic's latency hides
  // behind a whole chunk of work.
  uint32_t* claims = chunk_raw + total_cap;
  uint32_t res = 0;
  if (lane == 0) res = atomicAdd(claims, 1u);

  // ---- producer: lane 0 issues, every lane tracks the same (uniform) state ----
  // It claims chunks, queues them for the consumer (fast ones with their 8
  // stage loads, slow ones as markers), and keeps at most kRing - 2 loads
  // ahead of the stage being consumed, so a refilled stage's bulk store was
  // issued one stage earlier (wait_group.read 1 rarely waits).
  uint32_t issued = 0, consumed = 0, q_tail = 0, q_head = 0;
  int p_u = kStagesPerChunk;
  ChunkRef p_ref = {nullptr, nullptr, 0u, false};
  bool exhausted = false;
  pecdev::DescCursor p_cur;
  auto produce = [&]() {
    while (!exhausted && issued + 2 <= consumed + kRing) {
      if (p_u == kStagesPerChunk) {
        if (q_tail - q_head == (uint32_t)kQueue) return;
        const uint64_t ch = __shfl_sync(0xffffffffu, res, 0);
        PEC_DCHECK(q_tail - q_head < (uint32_t)kQueue);
        if (ch >= total) {
          exhausted = true;
          return;
        }
        if (lane == 0) res = atomicAdd(claims, 1u);
        p_ref = chunk_ref(d, n, ch, p_cur);
        if (lane == 0) {
          QueueEntry& e = q[q_tail % kQueue];
          e.src = p_ref.src;
          e.dst = p_ref.dst;
          e.ch = ch;
          e.len = p_ref.len;
          e.fast = p_ref.fast ? 1u : 0u;
        }
        ++q_tail;
        if (!p_ref.fast) continue;
        p_u = 0;
      }
      const int s = (int)(issued % kRing);
      PEC_DCHECK(issued + 2 <= consumed + kRing && p_u < kStagesPerChunk && p_ref.fast);
      if (lane == 0) {
        if (kStore) bulk_wait_read1();   // the store that last read this stage
        mbar_expect_tx(&my_bars[s], kStage);
        bulk_g2s(my_ring + (size_t)s * kStage, p_ref.src + ((size_t)p_u << kStageLg), kStage,
                 &my_bars[s], policy);
      }
      ++issued;
      ++p_u;
    }
  };

  // ---- consumer ------------------------------------------------------------------
#pragma unroll 1
  for (;;) {
    produce();
    if (q_head == q_tail) break;            // exhausted and everything consumed
    __syncwarp();                           // lane 0's queue entry is visible
    const QueueEntry& e = q[q_head % kQueue];
    const uint8_t* src = e.src;
    uint8_t* dst = e.dst;
    const uint64_t ch = e.ch;
    const uint32_t len = e.len;
    const bool fast = e.fast != 0;
    ++q_head;
    uint32_t x = 0;  // this lane's share of R(chunk)
    if (fast) {
      uint32_t S0 = 0, S1 = 0, S2 = 0, S3 = 0;
#pragma unroll 1
      for (int u = 0; u < kStagesPerChunk; ++u) {
        const int s = (int)(consumed % kRing);
        mbar_wait(&my_bars[s], (consumed / kRing) & 1u);
        const uint8_t* stage = my_ring + (size_t)s * kStage;
        if (kStore && lane == 0) {
          bulk_s2g(dst + ((size_t)u << kStageLg), stage, kStage, policy);
          bulk_commit();
        }
        const int4* rows = reinterpret_cast<const int4*>(stage) + lane;
#pragma unroll
        for (int j = 0; j < kRowsPerStage; ++j) {
          const int4 v = rows[32 * j];
          S0 = ystep(S0, (uint32_t)v.x, slot, sel);
          S1 = ystep(S1, (uint32_t)v.y, slot, sel);
          S2 = ystep(S2, (uint32_t)v.z, slot, sel);
          S3 = ystep(S3, (uint32_t)v.w, slot, sel);
        }
        __syncwarp();            // every lane has read the stage
        ++consumed;
        produce();               // refill the stage consumed one step earlier
      }
      const uint32_t c = mul_const(nib, S0) ^ mul_const(nib + 128, S1) ^
                         mul_const(nib + 256, S2) ^ mul_const(nib + 384, S3);
#pragma unroll
      for (int p = 0; p < 8; ++p) x ^= ltab[(p * 16 + ((c >> (4 * p)) & 15u)) << 5];
#pragma unroll
      for (int j = 16; j >= 1; j >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, j);
    } else if (len > 0) {
      // partial or unaligned chunk: 1 KiB per lane, byte loop, then a warp
      // tree joins the pieces (right neighbour's length as the shift)
      constexpr uint32_t kPiece = kChunk / 32;
      const uint32_t lo = (uint32_t)lane * kPiece;
      const uint32_t hi = lo + kPiece < len ? lo + kPiece : len;
      uint32_t c = 0;
      for (uint32_t b = lo; b < hi; ++b) {
        const uint8_t v = src[b];
        if (kStore) dst[b] = v;
        c = t8[(c ^ v) & 0xFFu] ^ (c >> 8);
      }
      uint32_t my_len = hi > lo ? hi - lo : 0u;
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const uint32_t oc = __shfl_down_sync(0xffffffffu, c, 1 << j);
        const uint32_t ol = __shfl_down_sync(0xffffffffu, my_len, 1 << j);
        if ((lane & ((2 << j) - 1)) == 0) {
          c = shift_bytes(c, ol) ^ oc;
          my_len += ol;
        }
      }
      x = c;
    }
    PEC_DCHECK(ch < total_cap);
    if (lane == 0) chunk_raw[ch] = x;
  }
  PEC_DCHECK(issued == consumed);
  if (kStore && lane == 0) bulk_wait_all();
}

template <bool kStore>
int launch_pack_crc(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                    const uint64_t* total_chunks_dev, uint32_t* chunk_crc, cudaStream_t st) {
  static int ready[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return PEC_E_CUDA;
  if (!ready[dev]) {
    if (cudaFuncSetAttribute(pack_crc_kernel<kStore>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSmemBytes) != cudaSuccess)
      return PEC_E_CUDA;
    ready[dev] = 1;
  }
  // the chunk-claim counter lives after the chunk registers
  if (cudaMemsetAsync(chunk_crc + total_chunks, 0, sizeof(uint32_t), st) != cudaSuccess)
    return PEC_E_CUDA;
  uint64_t grid = (uint64_t)sm_count();
  const uint64_t need = (total_chunks + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  pack_crc_kernel<kStore><<<(unsigned)grid, kThreads, kSmemBytes, st>>>(
      descs, n, total_chunks, total_chunks_dev, chunk_crc);
  return PEC_OK;
}

// Chunk registers -> entry accumulators.  Each thread takes a contiguous run
// of chunks and Horner-accumulates consecutive chunks of one entry (constant
// 32 KiB shift through 4-bit-window tables), so an entry receives one atomic
// per thread run instead of one per chunk (2 GB entries have 64 Ki chunks:
// same-address atomics would serialise).  A run is flushed shifted by the
// whole chunks that follow it, x^(8 * 32 KiB * j), a product of up to three
// 256-entry power tables built per CTA by doubling.  The entry's LAST chunk
// keeps its register in its own slot; crc_final_kernel applies the shift by
// the last chunk's length once per entry and joins it.
__global__ void __launch_bounds__(256)
crc_fold_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                const uint64_t* __restrict__ total_dev,
                const uint32_t* __restrict__ chunk_raw, uint32_t* __restrict__ entry_raw) {
  __shared__ uint32_t cnib[128];        // windows of x^(8 * 32768)
  __shared__ uint32_t pw[3][256];       // x^(8 * 32K * t * 256^r)
  const int tid = threadIdx.x;
  if (tid < 128) cnib[tid] = __ldg(&kTab.chunk_nib[tid]);
  for (int idx = tid; idx < 3 * 256; idx += blockDim.x) pw[idx >> 8][idx & 255] =
      __ldg(&kTab.chunk_pw[0][0] + idx);
  __syncthreads();
  if (total_dev != nullptr) {
    const uint64_t td = *total_dev;
    total = td < total ? td : total;
  }
  const uint64_t threads = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t per = (total + threads - 1) / threads;
  const uint64_t c0 = ((uint64_t)blockIdx.x * blockDim.x + tid) * per;
  const uint64_t c1 = c0 + per < total ? c0 + per : total;
  pecdev::DescCursor cur;
  int run_entry = -1;
  uint32_t run = 0;                 // Horner sum of the run's chunk registers
  uint64_t run_end = 0;             // entry-relative index one past the run
  uint64_t run_chunks = 0;          // chunks of the run's entry
  auto flush = [&]() {
    if (run_entry < 0) return;
    const uint64_t j = run_chunks - 1 - run_end;  // whole chunks up to the last one
    uint32_t p = pw[0][j & 255];
    if ((j >> 8) & 255) p = gf2_mul(p, pw[1][(j >> 8) & 255]);
    if (j >> 16) p = gf2_mul(p, pw[2][(j >> 16) & 255]);
    atomicXor(&entry_raw[run_entry], gf2_mul(run, p));
    run_entry = -1;
  };
  for (uint64_t ch = c0; ch < c1; ++ch) {
    const int i = cur.find(d, n, ch);
    const uint64_t kk = ch - __ldg(&d[i].first_chunk);
    const uint64_t nb = __ldg(&d[i].nbytes);
    if ((kk << kCrcLg) >= nb) continue;
    const uint64_t chunks = (nb + kChunk - 1) >> kCrcLg;
    if (run_entry >= 0 && i != run_entry) flush();
    if (kk == chunks - 1) {
      flush();                      // this entry's run (if any) ends right before it
      continue;                     // R(last chunk) is joined in crc_final_kernel
    }
    if (run_entry < 0) {
      run_entry = i;
      run = 0;
      run_chunks = chunks;
    }
    run = mul_const(cnib, run) ^ chunk_raw[ch];
    run_end = kk + 1;
  }
  flush();
}

// Per entry: R = A * x^(8 * len(last chunk)) ^ R(last chunk), then the
// initial value / final inversion: crc = ~(R ^ ~0 * x^(8 * nbytes)).
__global__ void crc_final_kernel(const pec_copy_desc* __restrict__ d, int n,
                                 const uint32_t* __restrict__ chunk_raw,
                                 uint32_t* __restrict__ entry) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t nb = d[i].nbytes;
    if (nb == 0) {
      entry[i] = 0u;
      continue;
    }
    const uint64_t chunks = (nb + kChunk - 1) >> kCrcLg;
    const uint64_t last_len = nb - ((chunks - 1) << kCrcLg);
    PEC_DCHECK(last_len > 0 && last_len <= (uint64_t)kChunk);
    const uint32_t r_last = chunk_raw[d[i].first_chunk + chunks - 1];
    const uint32_t r = shift_bytes(entry[i], last_len) ^ r_last;
    entry[i] = ~(r ^ shift_bytes(0xFFFFFFFFu, nb));
  }
}


template <bool kStore>
int crc_entries(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                uint32_t* entry_crc, void* stream) {
  if (chunk_log2 != kCrcLg || n < 0) return PEC_E_INVAL;
  if (n == 0) return PEC_OK;
  if (descs == nullptr || entry_crc == nullptr || (total_chunks > 0 && chunk_crc == nullptr))
    return PEC_E_INVAL;
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(entry_crc, 0, sizeof(uint32_t) * (size_t)n, st) != cudaSuccess)
    return PEC_E_CUDA;
  if (total_chunks > 0) {
    const int rc = launch_pack_crc<kStore>(descs, n, total_chunks, total_chunks_dev, chunk_crc,
                                           st);
    if (rc != PEC_OK) return rc;
    uint64_t fold_grid = (total_chunks + 255) / 256;
    if (fold_grid > (uint64_t)sm_count()) fold_grid = (uint64_t)sm_count();  // tables per CTA
    crc_fold_kernel<<<(unsigned)fold_grid, 256, 0, st>>>(descs, n, total_chunks, total_chunks_dev,
                                                          chunk_crc, entry_crc);
  }
  crc_final_kernel<<<(n + 63) / 64, 64, 0, st>>>(descs, n, chunk_crc, entry_crc);
  return launch_status();
}

}  // namespace

extern "C" {

int pec_pack_crc(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                 const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                 uint32_t* entry_crc, void* stream) {
  return crc_entries<true>(descs, n, total_chunks, total_chunks_dev, chunk_log2, chunk_crc,
                           entry_crc, stream);
}

int pec_crc_device(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                   const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                   uint32_t* entry_crc, void* stream) {
  return crc_entries<false>(descs, n, total_chunks, total_chunks_dev, chunk_log2, chunk_crc,
                            entry_crc, stream);
}

}  // extern "C"
