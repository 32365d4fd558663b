// pec_crc.cu — CRC-32C of every staged entry, computed by the pack itself.
//
// the persist tier checksums each entry
// (store.crc32c, pkg/src/mocsim/store.py:49-70; the manifest column of
// store.py:149-164).  Here the pack kernel checksums the bytes it already
// holds in registers on their way from the state arena to the staging
// buffer, so the host never reads the payload for CRC and the HBM traffic of
// the pack is unchanged.
//
// CRC-32C is linear over GF(2): for the register form R (initial value 0,
// no final inversion), R(A || B) = R(A) * x^(8|B|) mod P  ^  R(B), and the
// standard CRC is crc(M) = ~(R(M) ^ ~0 * x^(8|M|) mod P).  So:
//   pack_crc_kernel   one warp per 4 KiB unit: coalesced 16 B loads, stored
//                     to staging and through a swizzled per-warp tile so each
//                     lane then folds ITS contiguous 128 B in four 32-byte
//                     chains with a byte table kept in shared memory once per
//                     lane (entry e of lane l at word 32e + l: every lookup of
//                     a warp hits 32 distinct banks); each lane shifts its
//                     register to the unit end with its own constant (lane-
//                     replicated 4-bit-window tables) and a 5-step XOR
//                     butterfly gives the unit register;
//   crc_fold_kernel   one thread per 32 KiB chunk joins its 8 unit registers,
//                     shifts the result by the bytes that follow it in its
//                     entry and XORs it into the entry's register;
//   crc_final_kernel  applies the initial value / final inversion per entry.
// Multiplication mod P (reflected, bit 31 = x^0) is the shift-and-add
// schoolbook product or, for constants, 8 lookups of 4-bit-window tables;
// x^(2^k) are precomputed on the host.

#include <cuda_runtime.h>
#include <stdint.h>

#include "pec.h"
#include "pec_device.cuh"

namespace {

using pecdev::as_stream;
using pecdev::find_desc;
using pecdev::launch_status;
using pecdev::sm_count;

constexpr uint32_t kPoly = 0x82F63B78u;
constexpr int kCrcThreads = 256;
constexpr int kCrcLg = 15;                            // 32 KiB chunks
constexpr int kPerThread = (1 << kCrcLg) / kCrcThreads;  // 128 contiguous bytes
constexpr int kVecPerThread = kPerThread / 16;        // 8 x 16 B
constexpr int kTableWords = 256 * 32;                 // lane-replicated byte table

// Constant multipliers are applied through 4-bit windows: mul(a, b) =
// XOR_p N_a[p][(b >> 4p) & 15] with N_a[p][v] = a * (v << 4p): 8 shared-memory
// lookups instead of a 32-step schoolbook product (tables built per CTA).
struct CrcConsts {
  uint32_t x2k[64];         // x^(2^k) mod P
  uint32_t unit;            // x^(8 * 4096): one 4 KiB unit
};

__host__ __device__ __forceinline__ uint32_t gf2_mul(uint32_t a, uint32_t b) {
  uint32_t p = 0;
#pragma unroll 8
  for (int i = 31; i >= 0; --i) {
    p ^= b & (0u - ((a >> i) & 1u));
    b = (b >> 1) ^ (kPoly & (0u - (b & 1u)));
  }
  return p;
}

__device__ __forceinline__ uint32_t xpow_bytes(const uint32_t* x2k, uint64_t nbytes) {
  uint32_t acc = 1u << 31;  // 1
  int k = 3;                // 8 bits per byte
  while (nbytes) {
    if (nbytes & 1u) acc = gf2_mul(x2k[k], acc);
    nbytes >>= 1;
    ++k;
  }
  return acc;
}

__device__ __forceinline__ uint32_t shift_bytes(const uint32_t* x2k, uint32_t r, uint64_t n) {
  return n ? gf2_mul(xpow_bytes(x2k, n), r) : r;
}

// Byte-table lookup at the lane-replicated slot: entry e of lane l is word
// 32e + l, i.e. byte offset (e << 7) | (l << 2) from the table base, formed by
// one shift and one LOP3 ((c << 7) & 0x7F80 | lane4).  The table is a static
// shared array, so its base is an immediate of the LDS (no per-lookup add),
// and the LOP3 is opaque so the compiler cannot re-associate lane4 into a
// base register.
__device__ __forceinline__ uint32_t lut(const uint32_t* table, uint32_t c, uint32_t lane4) {
  uint32_t off;
  asm("lop3.b32 %0, %1, 0x7F80, %2, 0xEA;" : "=r"(off) : "r"(c << 7), "r"(lane4));
  return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(table) + off);
}

__device__ __forceinline__ uint32_t fold_word(const uint32_t* table, uint32_t lane4, uint32_t c,
                                              uint32_t w) {
  c ^= w;
#pragma unroll
  for (int b = 0; b < 4; ++b) c = lut(table, c, lane4) ^ (c >> 8);
  return c;
}

__device__ __forceinline__ uint32_t mul_const(const uint32_t* nib, uint32_t b) {
  uint32_t r = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) r ^= nib[p * 16 + ((b >> (4 * p)) & 15u)];
  return r;
}

// Work unit = one warp x 4 KiB (8 units per 32 KiB chunk).  Warps take
// units independently (no block barrier on the hot path): unit u of the
// launch is warp-global index + k * total_warps, so neighbouring warps stream
// neighbouring 4 KiB and every warp keeps its own loads in flight.
constexpr int kUnitLog2 = 12;
constexpr int kUnitsPerChunk = 1 << (kCrcLg - kUnitLog2);

// Multipliers the pack kernel builds 4-bit-window tables for (128 words each):
// [0] x^(8*32) joins a lane's 32-byte chains, [1] x^(8*S) joins its
// sub-blocks (S = 4096 / kSub bytes), [2..6] x^(8*P*2^j) are the warp-tree
// levels (P = 128 / kSub bytes per lane per sub-block).
constexpr int kPackMuls = 7;
constexpr int kPackMulWords = kPackMuls * 128;
constexpr int kLaneTabWords = 8 * 16 * 32;  // per-lane x^(8*P*(31-l)) windows

template <int kThreads, int kSub, bool kLaneMul>
constexpr int pack_crc_smem() {
  return ((kLaneMul ? 2 * 128 : kPackMulWords) + (kLaneMul ? kLaneTabWords : 0)) * 4 +
         (kThreads / 32) * (4096 / kSub);
}

// kSub: the 4 KiB unit is transposed through a (4096 / kSub)-byte per-warp
// tile in kSub rounds (smaller tiles: more CTAs per SM).  kLaneMul: a full
// unit's lanes shift their registers to the unit end with per-lane constant
// tables (lane l's window table at word 32 * (16 p + v) + l: conflict-free)
// and a 5-step XOR butterfly, instead of the 5-level multiply tree.
template <int kThreads, int kSub, int kMinBlocks, bool kLaneMul>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
pack_crc_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                const uint64_t* __restrict__ total_dev, CrcConsts k,
                uint32_t* __restrict__ unit_raw) {
  constexpr int kVecSub = kVecPerThread / kSub;   // 16-byte vectors per lane per round
  constexpr int kChains = 4 / kSub;               // 32-byte chains per round
  constexpr int kPiece = kPerThread / kSub;       // bytes per lane per round
  // static smem: byte table; dynamic: multiplier windows | lane windows | per-warp tiles
  constexpr int kMuls = kLaneMul ? 2 : kPackMuls;  // tree levels only without lane tables
  __shared__ __align__(16) uint32_t table[kTableWords];
  extern __shared__ __align__(16) uint32_t dyn[];
  uint32_t* nib = dyn;
  uint32_t* lanetab = nib + kMuls * 128;
  uint32_t* stage = lanetab + (kLaneMul ? kLaneTabWords : 0);
  __shared__ uint32_t mconst[kPackMuls];
  __shared__ uint32_t lconst[32];
  if (total_dev != nullptr) {
    const uint64_t td = *total_dev;
    total = td < total ? td : total;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kMuls) {
    const uint64_t bytes = tid == 0 ? 32 : tid == 1 ? 4096 / kSub
                                             : (uint64_t)kPiece << (tid - 2);
    mconst[tid] = xpow_bytes(k.x2k, bytes);
  } else if (kLaneMul && tid >= 64 && tid < 96) {
    const int l = tid - 64;
    lconst[l] = xpow_bytes(k.x2k, (uint64_t)kPiece * (31 - l));
  }
  for (int idx = tid; idx < kTableWords; idx += kThreads) {
    uint32_t c = (uint32_t)(idx >> 5);
#pragma unroll
    for (int b = 0; b < 8; ++b) c = (c & 1u) ? (c >> 1) ^ kPoly : c >> 1;
    table[idx] = c;
  }
  __syncthreads();
  for (int idx = tid; idx < kMuls * 128; idx += kThreads) {
    const int m = idx >> 7, p = (idx >> 4) & 7, v = idx & 15;
    nib[idx] = gf2_mul(mconst[m], (uint32_t)v << (4 * p));
  }
  if (kLaneMul) {
    for (int idx = tid; idx < kLaneTabWords; idx += kThreads) {
      const int l = idx & 31, pv = idx >> 5, p = pv >> 4, v = pv & 15;
      lanetab[idx] = gf2_mul(lconst[l], (uint32_t)v << (4 * p));
    }
  }
  __syncthreads();
  const uint32_t* tab = table + lane;
  const uint32_t lane4 = (uint32_t)lane << 2;
  const uint32_t* n32 = nib;
  const uint32_t* nsub = nib + 128;
  const uint32_t* lvl = nib + 256;           // tree levels, 128 words each
  const uint32_t* ltab = lanetab + lane;
  int4* tile = reinterpret_cast<int4*>(stage) + warp * (256 / kSub);

  const uint64_t units = total * kUnitsPerChunk;
  const uint64_t warps_total = (uint64_t)gridDim.x * (kThreads / 32);
  pecdev::DescCursor cur;
  for (uint64_t u = (uint64_t)blockIdx.x * (kThreads / 32) + warp; u < units;
       u += warps_total) {
    const uint64_t ch = u >> (kCrcLg - kUnitLog2);
    const int i = cur.find(d, n, ch);
    const uint64_t nb = __ldg(&d[i].nbytes);
    const uint64_t off = ((ch - __ldg(&d[i].first_chunk)) << kCrcLg) +
                         ((u & (kUnitsPerChunk - 1)) << kUnitLog2);
    const uint64_t span = 1ull << kUnitLog2;
    const uint64_t len = off >= nb ? 0 : (nb - off < span ? nb - off : span);
    if (len == 0) {
      if (lane == 0) unit_raw[u] = 0u;
      continue;
    }
    const uint8_t* s = reinterpret_cast<const uint8_t*>(__ldg(&d[i].src) + off);
    uint8_t* t = reinterpret_cast<uint8_t*>(__ldg(&d[i].dst) + off);
    const bool fast = len == span && ((reinterpret_cast<uintptr_t>(s) |
                                      reinterpret_cast<uintptr_t>(t)) & 15u) == 0;
    uint32_t c = 0;
    uint32_t my_len;
    if (fast) {
      // coalesced 16 B units (lane + 32k) -> staging, and into a swizzled tile
      // from which each lane reads back ITS contiguous piece conflict-free
      // (16-byte slot of unit x: x ^ ((x >> 3) & 7)); 32-byte CRC chains.
      const int4* vs = reinterpret_cast<const int4*>(s);
      int4* vt = reinterpret_cast<int4*>(t);
      int4 r[kVecPerThread];
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q) r[q] = __ldg(vs + lane + 32 * q);
#pragma unroll
      for (int q = 0; q < kVecPerThread; ++q) __stcs(vt + lane + 32 * q, r[q]);
#pragma unroll
      for (int sb = 0; sb < kSub; ++sb) {
#pragma unroll
        for (int q = 0; q < kVecSub; ++q) {
          const int x = lane + 32 * q;
          tile[x ^ ((x >> 3) & 7)] = r[sb * kVecSub + q];
        }
        __syncwarp();
        int4 v4[kVecSub];
#pragma unroll
        for (int j = 0; j < kVecSub; ++j) {
          const int x = lane * kVecSub + j;
          v4[j] = tile[x ^ ((x >> 3) & 7)];
        }
        __syncwarp();  // the tile is rewritten next
        uint32_t q4[kChains];
#pragma unroll
        for (int cc = 0; cc < kChains; ++cc) q4[cc] = 0u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int w = 0; w < 4; ++w) {
#pragma unroll
            for (int cc = 0; cc < kChains; ++cc) {
              const int4 v = v4[cc * 2 + h];
              const uint32_t word = w == 0 ? (uint32_t)v.x : w == 1 ? (uint32_t)v.y
                                  : w == 2 ? (uint32_t)v.z : (uint32_t)v.w;
              q4[cc] = fold_word(table, lane4, q4[cc], word);
            }
          }
        }
        uint32_t cs = q4[0];
#pragma unroll
        for (int cc = 1; cc < kChains; ++cc) cs = mul_const(n32, cs) ^ q4[cc];
        c = sb == 0 ? cs : mul_const(nsub, c) ^ cs;
      }
      my_len = kPiece;
      if (kLaneMul) {
        // shift to the unit end with this lane's constant, XOR over the warp
        uint32_t x = 0;
#pragma unroll
        for (int p = 0; p < 8; ++p) x ^= ltab[(p * 16 + ((c >> (4 * p)) & 15u)) << 5];
#pragma unroll
        for (int j = 16; j >= 1; j >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, j);
        if (lane == 0) unit_raw[u] = x;
        continue;
      }
    } else {
      // partial or unaligned unit: bytes, 128 per lane
      const uint64_t lo = (uint64_t)lane * kPerThread;
      const uint64_t hi = lo + kPerThread < len ? lo + kPerThread : len;
      for (uint64_t b = lo; b < hi; ++b) {
        const uint8_t v = s[b];
        t[b] = v;
        c = tab[((c ^ v) & 0xFFu) << 5] ^ (c >> 8);
      }
      my_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
    }
    // warp tree: lanes hold consecutive pieces; fold right neighbours in
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const uint32_t oc = __shfl_down_sync(0xffffffffu, c, 1 << j);
      const uint32_t ol = __shfl_down_sync(0xffffffffu, my_len, 1 << j);
      if ((lane & ((2 << j) - 1)) == 0) {
        c = (fast ? mul_const(lvl + j * 128, c) : shift_bytes(k.x2k, c, ol)) ^ oc;
        my_len += ol;
      }
    }
    if (lane == 0) unit_raw[u] = c;
  }
}

template <int kThreads, int kSub, int kMinBlocks, bool kLaneMul>
int launch_pack_crc(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                    const uint64_t* total_chunks_dev, const CrcConsts& consts,
                    uint32_t* chunk_crc, cudaStream_t st) {
  auto kern = pack_crc_kernel<kThreads, kSub, kMinBlocks, kLaneMul>;
  constexpr int smem = pack_crc_smem<kThreads, kSub, kLaneMul>();
  static const int per_sm = [&] {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return 0;
    int blocks = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kThreads, smem);
    return blocks < 1 ? 1 : blocks;
  }();
  if (per_sm == 0) return PEC_E_CUDA;
  uint64_t grid = (uint64_t)sm_count() * per_sm;
  const uint64_t need = (total_chunks * kUnitsPerChunk + kThreads / 32 - 1) / (kThreads / 32);
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, kThreads, smem, st>>>(descs, n, total_chunks, total_chunks_dev, consts,
                                                   chunk_crc);
  return PEC_OK;
}

// Chunk registers -> entry accumulators.  Each thread takes a contiguous run
// of chunks, joins every chunk's (up to 8) unit registers (constant 4 KiB
// shifts through 4-bit-window tables) and Horner-accumulates consecutive
// chunks of one entry (constant 32 KiB shift), so an entry receives one
// atomic per thread run instead of one per chunk (2 GB entries have 64 Ki
// chunks: same-address atomics would serialise).  A run is flushed shifted
// by the whole chunks that follow it, x^(8 * 32 KiB * j), a product of up to
// three 256-entry power tables built per CTA by doubling.  The entry's LAST
// chunk keeps its register in its own first unit slot (only this thread
// touches that chunk's slots); crc_final_kernel applies the shift by the
// last chunk's length once per entry and joins it.
__global__ void __launch_bounds__(256)
crc_fold_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                const uint64_t* __restrict__ total_dev, CrcConsts k,
                uint32_t* __restrict__ unit_raw, uint32_t* __restrict__ entry_raw) {
  __shared__ uint32_t x2k[64];
  __shared__ uint32_t unib[128];        // windows of x^(8 * 4096)
  __shared__ uint32_t cnib[128];        // windows of x^(8 * 32768)
  __shared__ uint32_t pw[3][256];       // x^(8 * 32K * t * 256^r)
  const int tid = threadIdx.x;
  if (tid < 64) x2k[tid] = k.x2k[tid];
  __syncthreads();
  if (tid < 128) {
    const int p = (tid >> 4) & 7, v = tid & 15;
    unib[tid] = gf2_mul(k.unit, (uint32_t)v << (4 * p));
  } else if (tid < 131) {
    const int r = tid - 128;
    uint32_t b = xpow_bytes(x2k, (uint64_t)(1u << kCrcLg) << (8 * r));
    pw[r][0] = 1u << 31;
    for (int l = 0; l < 8; ++l) {  // pw[r][2^l] = base^(2^l)
      pw[r][1 << l] = b;
      b = gf2_mul(b, b);
    }
  }
  __syncthreads();
  if (tid < 128) {
    const int p = (tid >> 4) & 7, v = tid & 15;
    cnib[tid] = gf2_mul(pw[0][1], (uint32_t)v << (4 * p));
  }
  for (int l = 1; l < 8; ++l) {     // pw[t] = pw[t - 2^l] * pw[2^l] for 2^l < t < 2^(l+1)
    const int span = (1 << l) - 1;
    for (int idx = tid; idx < 3 * span; idx += blockDim.x) {
      const int r = idx / span, t = (1 << l) + 1 + idx % span;
      pw[r][t] = gf2_mul(pw[r][t - (1 << l)], pw[r][1 << l]);
    }
    __syncthreads();
  }
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
    const uint64_t off = kk << kCrcLg;
    const uint64_t nb = __ldg(&d[i].nbytes);
    if (off >= nb) continue;
    const uint64_t end = off + (1ull << kCrcLg) < nb ? off + (1ull << kCrcLg) : nb;
    uint32_t acc = unit_raw[ch * kUnitsPerChunk];
    for (int w = 1; w < kUnitsPerChunk; ++w) {
      const uint64_t uoff = off + ((uint64_t)w << kUnitLog2);
      if (uoff >= end) break;
      const uint64_t ulen = end - uoff < (1ull << kUnitLog2) ? end - uoff : (1ull << kUnitLog2);
      acc = (ulen == (1ull << kUnitLog2) ? mul_const(unib, acc) : shift_bytes(x2k, acc, ulen))
            ^ unit_raw[ch * kUnitsPerChunk + w];
    }
    const uint64_t chunks = (nb + (1ull << kCrcLg) - 1) >> kCrcLg;
    if (run_entry >= 0 && i != run_entry) flush();
    if (kk == chunks - 1) {
      unit_raw[ch * kUnitsPerChunk] = acc;   // R(last chunk), joined in crc_final_kernel
      flush();                               // this entry's run (if any) ends right before it
      continue;
    }
    if (run_entry < 0) {
      run_entry = i;
      run = 0;
      run_chunks = chunks;
    }
    run = mul_const(cnib, run) ^ acc;
    run_end = kk + 1;
  }
  flush();
}

// Per entry: R = A * x^(8 * len(last chunk)) ^ R(last chunk), then the
// initial value / final inversion: crc = ~(R ^ ~0 * x^(8 * nbytes)).
__global__ void crc_final_kernel(const pec_copy_desc* __restrict__ d, int n, CrcConsts k,
                                 const uint32_t* __restrict__ unit_raw,
                                 uint32_t* __restrict__ entry) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t nb = d[i].nbytes;
    if (nb == 0) {
      entry[i] = 0u;
      continue;
    }
    const uint64_t chunks = (nb + (1ull << kCrcLg) - 1) >> kCrcLg;
    const uint64_t last_len = nb - ((chunks - 1) << kCrcLg);
    const uint32_t r_last = unit_raw[(d[i].first_chunk + chunks - 1) * kUnitsPerChunk];
    const uint32_t r = shift_bytes(k.x2k, entry[i], last_len) ^ r_last;
    entry[i] = ~(r ^ shift_bytes(k.x2k, 0xFFFFFFFFu, nb));
  }
}

CrcConsts make_consts() {
  CrcConsts k;
  uint32_t p = 1u << 30;  // x^1
  for (int i = 0; i < 64; ++i) {
    k.x2k[i] = p;
    p = gf2_mul(p, p);
  }
  auto xpow = [&](uint64_t nbytes) {
    uint32_t acc = 1u << 31;
    int b = 3;
    while (nbytes) {
      if (nbytes & 1u) acc = gf2_mul(k.x2k[b], acc);
      nbytes >>= 1;
      ++b;
    }
    return acc;
  };
  k.unit = xpow(1u << kUnitLog2);
  return k;
}

}  // namespace

extern "C" {

int pec_pack_crc(const pec_copy_desc* descs, int n, uint64_t total_chunks,
                 const uint64_t* total_chunks_dev, int chunk_log2, uint32_t* chunk_crc,
                 uint32_t* entry_crc, void* stream) {
  if (chunk_log2 != kCrcLg || n < 0) return PEC_E_INVAL;
  if (n == 0) return PEC_OK;
  if (descs == nullptr || entry_crc == nullptr || (total_chunks > 0 && chunk_crc == nullptr))
    return PEC_E_INVAL;
  static const CrcConsts consts = make_consts();
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(entry_crc, 0, sizeof(uint32_t) * (size_t)n, st) != cudaSuccess)
    return PEC_E_CUDA;
  if (total_chunks > 0) {
    // measured on B200 (profiles/r1/crc_variants.txt): lane-constant shifts
    // instead of the multiply tree, 4 KiB tiles, 2 CTAs x 8 warps per SM
    const int rc = launch_pack_crc<256, 1, 3, true>(descs, n, total_chunks, total_chunks_dev,
                                                     consts, chunk_crc, st);
    if (rc != PEC_OK) return rc;
    uint64_t fold_grid = (total_chunks + 255) / 256;
    if (fold_grid > (uint64_t)sm_count()) fold_grid = (uint64_t)sm_count();  // tables per CTA
    crc_fold_kernel<<<(unsigned)fold_grid, 256, 0, st>>>(descs, n, total_chunks, total_chunks_dev,
                                                          consts, chunk_crc, entry_crc);
  }
  crc_final_kernel<<<(n + 255) / 256, 256, 0, st>>>(descs, n, consts, chunk_crc, entry_crc);
  return launch_status();
}

}  // extern "C"
