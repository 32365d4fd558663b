// pec_kernels.cu — sm_100a kernels of the PEC snapshot path + their C ABI.
//
// Kernels (see DESIGN.md for the roofline of each):
//   token_hist_kernel        per-expert token histogram of one iteration's
//                            router ids, capacity clamp, int64 accumulation
//                            (reference: simulator.py:88-95, :560-567)
//   select_sequential_kernel window selection (selector.py:21-32)
//   select_load_aware_kernel top-K by (-unsaved, id) + mark_saved (block radix sort)
//                            (selector.py:86-100, simulator.py:339-354)
//   copy_vec_kernel          gather/scatter engine, LDG/STG.128
//   copy_bulk_kernel         gather/scatter engine, TMA bulk (cp.async.bulk)
//                            global->smem->global ring
// pack and unpack are the same engines over a table whose src/dst roles are
// swapped (pack: state -> staging, unpack: staging -> state).

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "pec.h"
#include "pec_device.cuh"

namespace {

constexpr int kMaxExperts = 4096;

using pecdev::as_stream;
using pecdev::find_desc;
using pecdev::launch_status;
using pecdev::sm_count;

// ------------------------------------------------------------------------
// (a) token histogram
// ------------------------------------------------------------------------
// grid = (blocks_per_layer, L).  Each CTA histograms a contiguous slice of
// one layer's ids into shared memory using warp aggregation (__match_any_sync
// groups the lanes holding the same id; the group leader adds the popcount),
// then folds its histogram into scratch with global atomics.  The last CTA
// to finish (ticket in scratch[L*E]) applies the per-iteration capacity
// clamp, accumulates into the int64 counters and re-zeroes scratch — one
// launch per iteration, no host round trip.
constexpr int kHistThreads = 256;
constexpr int kHistUnroll = 8;

template <typename Id>
__global__ void __launch_bounds__(kHistThreads, 1)
token_hist_kernel(const Id* __restrict__ idx, int L, int64_t n, int E,
                  const int64_t* __restrict__ cap, int64_t* __restrict__ counters,
                  int tiers, int64_t* __restrict__ delivered,
                  uint32_t* __restrict__ scratch) {
  extern __shared__ uint32_t hist[];  // E + 1 (slot E collects ignored ids)
  const int layer = blockIdx.y;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) hist[e] = 0;
  __syncthreads();

  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < n ? lo + per : n;
  const Id* row = idx + (int64_t)layer * n;
  const unsigned lane = threadIdx.x & 31u;

  // The trip count depends only on (lo, hi), uniform across the CTA, so the
  // full-mask __match_any_sync below always sees converged warps.
  for (int64_t base = lo; base < hi; base += (int64_t)kHistThreads * kHistUnroll) {
    Id v[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t i = base + (int64_t)u * kHistThreads + threadIdx.x;
      v[u] = i < hi ? __ldg(row + i) : Id(-1);
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      // ids outside [0, E) (dropped tokens, any width) go to the ignore slot
      const int key = (v[u] >= 0 && v[u] < (Id)E) ? (int)v[u] : E;
      PEC_DCHECK(key >= 0 && key <= E);
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&hist[key], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const uint32_t c = hist[e];
    if (c) atomicAdd(&scratch[(int64_t)layer * E + e], c);
  }

  // last-CTA-done: fence our atomics, take a ticket
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t total = gridDim.x * gridDim.y;
    const uint32_t t = atomicAdd(&scratch[(int64_t)L * E], 1u);
    is_last = (t == total - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int64_t le = (int64_t)L * E;
  for (int64_t j = threadIdx.x; j < le; j += blockDim.x) {
    const int64_t c = (int64_t)atomicExch(&scratch[j], 0u);  // read via L2 and clear
    const int64_t cl = cap ? (c < cap[j / E] ? c : cap[j / E]) : c;
    if (cl) {
      for (int t = 0; t < tiers; ++t) counters[(int64_t)t * le + j] += cl;
      if (delivered) delivered[j] += cl;
    }
  }
  if (threadIdx.x == 0) atomicExch(&scratch[le], 0u);
}

// ------------------------------------------------------------------------
// (b) selection
// ------------------------------------------------------------------------
__global__ void select_sequential_kernel(int64_t c, int L, int E, int width, int stride,
                                         int32_t* __restrict__ out) {
  const int W = width < E ? width : E;
  const int64_t total = (int64_t)L * W;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(t / W);
    const int j = (int)(t % W);
    int v;
    if (width >= E) {
      v = j;
    } else {
      // window {(m + c*stride + k) mod E : k < W}, emitted sorted ascending:
      // the wrapped part [0, s+W-E) first, then [s, min(E, s+W)).
      const int64_t s64 = ((int64_t)m + (c % E) * (int64_t)(stride % E)) % E;
      const int s = (int)((s64 + E) % E);
      const int wrap = s + W - E > 0 ? s + W - E : 0;
      v = j < wrap ? j : s + (j - wrap);
    }
    out[t] = v;
  }
}

// One CTA per layer.  Candidates are all E experts, or the valid distinct ids
// of the layer's pool (a shared bitmap drops duplicates and ids outside
// [0, E)).  A block radix sort of (count + 1, id) pairs — descending and
// stable, over ids in ascending order, non-candidates keyed 0 so they sort
// last — leaves ties in ascending id order, so ranks 0..K-1 are the top-K by
// (count desc, id asc); they are flagged in the bitmap and compacted in
// ascending id order with a block scan, and their counters reset when asked.
// The sort only visits the bits the layer's largest key uses (a block max
// first), and the CTA is one warp for E <= 32.  O(E log E) per layer: 4096
// experts cost one 16-item-per-thread sort (round 1 compared every candidate
// with every other, O(E^2) per lane).
template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads)
select_load_aware_kernel(int64_t* __restrict__ counters, int E, int K,
                         const int32_t* __restrict__ pool, int P,
                         int32_t* __restrict__ out, int zero_selected) {
  using Sort = cub::BlockRadixSort<unsigned long long, kThreads, kItems, int>;
  using Scan = cub::BlockScan<int, kThreads>;
  using Max = cub::BlockReduce<unsigned long long, kThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
    typename Max::TempStorage max;
  } tmp;
  __shared__ uint8_t flag[kThreads * kItems];   // candidate, then selected
  __shared__ int n_cand;
  __shared__ int end_bit;
  const int tid = threadIdx.x, layer = blockIdx.x;
  int64_t* cnt = counters + (int64_t)layer * E;
  for (int e = tid; e < kThreads * kItems; e += kThreads)
    flag[e] = (pool == nullptr && e < E) ? 1 : 0;
  if (tid == 0) n_cand = 0;
  __syncthreads();
  if (pool != nullptr) {
    for (int i = tid; i < P; i += kThreads) {
      const int e = pool[(int64_t)layer * P + i];
      if (e >= 0 && e < E) flag[e] = 1;
    }
    __syncthreads();
  }
  unsigned long long key[kItems];
  int id[kItems];
  int mine = 0;
  unsigned long long kmax = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int e = tid * kItems + j;               // blocked: ascending ids in input order
    const bool cand = e < E && flag[e];
    // counters are token counts (>= 0): count + 1 keeps every candidate above 0
    key[j] = cand ? (unsigned long long)cnt[e] + 1ull : 0ull;
    id[j] = cand ? e : -1;
    mine += cand;
    kmax = key[j] > kmax ? key[j] : kmax;
  }
  if (mine) atomicAdd(&n_cand, mine);
  const unsigned long long bmax = Max(tmp.max).Reduce(kmax, cub::Max());
  if (tid == 0) end_bit = bmax ? 64 - __clzll((long long)bmax) : 1;
  __syncthreads();
  Sort(tmp.sort).SortDescending(key, id, 0, end_bit);   // stable: ties keep id order
  __syncthreads();
  const int kk = K < n_cand ? K : n_cand;
  for (int e = tid; e < kThreads * kItems; e += kThreads) flag[e] = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int rank = tid * kItems + j;
    if (rank < kk) {
      PEC_DCHECK(id[j] >= 0 && id[j] < E);
      flag[id[j]] = 1;
    }
  }
  __syncthreads();
  int mark = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) mark += flag[tid * kItems + j];
  int pos = 0;
  Scan(tmp.scan).ExclusiveSum(mark, pos);
  int32_t* o = out + (int64_t)layer * K;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int e = tid * kItems + j;
    if (flag[e]) {
      PEC_DCHECK(pos < K);
      o[pos++] = e;
      if (zero_selected) cnt[e] = 0;
    }
  }
  for (int j = kk + tid; j < K; j += kThreads) o[j] = -1;
}

// ------------------------------------------------------------------------
// (c)/(d) gather/scatter engines
// ------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1, %2, %3, %4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Byte-exact copy of [s, s+len) -> [t, t+len) by one CTA.  Fast path when
// s == t (mod 16): <16 head bytes, a 16-byte-vector body with UNROLL loads in
// flight per thread, <16 tail bytes.  Otherwise a word or byte loop.
template <int THREADS, int UNROLL>
__device__ __forceinline__ void cta_copy(const uint8_t* __restrict__ s, uint8_t* __restrict__ t,
                                         uint64_t len) {
  const uintptr_t sa = reinterpret_cast<uintptr_t>(s);
  const uintptr_t ta = reinterpret_cast<uintptr_t>(t);
  if (((sa ^ ta) & 15u) == 0) {
    uint64_t head = (16u - (sa & 15u)) & 15u;
    if (head > len) head = len;
    if (threadIdx.x < head) t[threadIdx.x] = s[threadIdx.x];
    const int4* vs = reinterpret_cast<const int4*>(s + head);
    int4* vt = reinterpret_cast<int4*>(t + head);
    const uint64_t nv = (len - head) >> 4;
    for (uint64_t v = threadIdx.x; v < nv; v += (uint64_t)THREADS * UNROLL) {
      int4 r[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint64_t k = v + (uint64_t)u * THREADS;
        if (k < nv) r[u] = ld_stream(vs + k);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint64_t k = v + (uint64_t)u * THREADS;
        if (k < nv) st_stream(vt + k, r[u]);
      }
    }
    const uint64_t ts = head + (nv << 4);
    const uint64_t tail = len - ts;
    if (threadIdx.x < tail) t[ts + threadIdx.x] = s[ts + threadIdx.x];
  } else if (((sa ^ ta) & 3u) == 0) {
    uint64_t head = (4u - (sa & 3u)) & 3u;
    if (head > len) head = len;
    if (threadIdx.x < head) t[threadIdx.x] = s[threadIdx.x];
    const uint32_t* ws = reinterpret_cast<const uint32_t*>(s + head);
    uint32_t* wt = reinterpret_cast<uint32_t*>(t + head);
    const uint64_t nw = (len - head) >> 2;
    for (uint64_t w = threadIdx.x; w < nw; w += THREADS) wt[w] = __ldg(ws + w);
    const uint64_t ts = head + (nw << 2);
    if (threadIdx.x < len - ts) t[ts + threadIdx.x] = s[ts + threadIdx.x];
  } else {
    for (uint64_t b = threadIdx.x; b < len; b += THREADS) t[b] = s[b];
  }
}

constexpr int kVecThreads = 256;
constexpr int kVecUnroll = 8;

__global__ void __launch_bounds__(kVecThreads)
copy_vec_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                const uint64_t* __restrict__ total_dev, int lg) {
  if (total_dev != nullptr) {
    const uint64_t t = *total_dev;  // written by pec_expand_plan earlier on the stream
    total = t < total ? t : total;
  }
  pecdev::DescCursor cur;
  for (uint64_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
    const int i = cur.find(d, n, ch);
    const uint64_t off = (ch - __ldg(&d[i].first_chunk)) << lg;
    const uint64_t nb = __ldg(&d[i].nbytes);
    if (off >= nb) continue;  // empty descriptor (never for a well-formed table)
    const uint64_t span = 1ull << lg;
    const uint64_t len = nb - off < span ? nb - off : span;
    const uint8_t* s = reinterpret_cast<const uint8_t*>(__ldg(&d[i].src) + off);
    uint8_t* t = reinterpret_cast<uint8_t*>(__ldg(&d[i].dst) + off);
    cta_copy<kVecThreads, kVecUnroll>(s, t, len);
  }
}

// ---- TMA bulk engine -----------------------------------------------------
// One elected thread per CTA streams the CTA's chunks through a ring of
// kStages shared-memory stages: cp.async.bulk global->smem completes on the
// stage's mbarrier, then cp.async.bulk smem->global (bulk_group) drains it.
// A stage is refilled only after `cp.async.bulk.wait_group.read` confirms
// the store that last read it has consumed the shared memory.  The 16-byte
// aligned body of each chunk goes through TMA; its (<16 B) unaligned head and
// tail, and any chunk whose src/dst are not congruent mod 16, are copied by
// the other warps with plain loads/stores in parallel.
constexpr int kBulkThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}"
      :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gmem), "r"(smem_u32(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem, const void* gmem, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gmem, const void* smem, uint32_t bytes,
                                              uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               :: "l"(gmem), "r"(smem_u32(smem)), "r"(bytes), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct ChunkView {
  const uint8_t* s;
  uint8_t* t;
  uint64_t len;
  uint64_t head;   // bytes before the 16-byte aligned body
  uint64_t body;   // multiple of 16, 0 when not congruent
};

__device__ __forceinline__ ChunkView chunk_view(const pec_copy_desc* __restrict__ d, int n,
                                                uint64_t ch, int lg, pecdev::DescCursor& cur) {
  ChunkView v;
  const int i = cur.find(d, n, ch);
  const uint64_t off = (ch - __ldg(&d[i].first_chunk)) << lg;
  const uint64_t nb = __ldg(&d[i].nbytes);
  const uint64_t span = 1ull << lg;
  v.len = off >= nb ? 0 : (nb - off < span ? nb - off : span);
  v.s = reinterpret_cast<const uint8_t*>(__ldg(&d[i].src) + off);
  v.t = reinterpret_cast<uint8_t*>(__ldg(&d[i].dst) + off);
  const uintptr_t sa = reinterpret_cast<uintptr_t>(v.s);
  const uintptr_t ta = reinterpret_cast<uintptr_t>(v.t);
  if (((sa ^ ta) & 15u) == 0) {
    uint64_t head = (16u - (sa & 15u)) & 15u;
    if (head > v.len) head = v.len;
    v.head = head;
    v.body = (v.len - head) & ~uint64_t(15);
  } else {
    v.head = 0;
    v.body = 0;
  }
  return v;
}

// Pipeline items are pieces of <= kStageBytes of a chunk's aligned body:
// item j of this CTA is piece (j % P) of its (j / P)-th chunk, P = pieces per
// chunk, so chunk sizes above one stage simply yield more items.

struct Piece {
  const uint8_t* src;
  uint8_t* dst;
  uint32_t bytes;  // 0 => nothing to move (phase still advanced)
};

__device__ __forceinline__ Piece piece_of(const pec_copy_desc* __restrict__ d, int n, int lg,
                                          uint64_t j, uint32_t per_chunk, int piece_log2,
                                          pecdev::DescCursor& cur) {
  const uint64_t jc = j / per_chunk;
  const uint32_t jp = (uint32_t)(j % per_chunk);
  const ChunkView v = chunk_view(d, n, blockIdx.x + jc * gridDim.x, lg, cur);
  Piece p;
  const uint64_t lo = (uint64_t)jp << piece_log2;
  const uint64_t hi = lo + (1ull << piece_log2);
  const uint64_t end = hi < v.body ? hi : v.body;
  p.bytes = end > lo ? (uint32_t)(end - lo) : 0u;
  PEC_DCHECK(p.bytes <= (1u << piece_log2) && (p.bytes & 15u) == 0);
  PEC_DCHECK(v.head + v.body <= v.len);
  p.src = v.s + v.head + lo;
  p.dst = v.t + v.head + lo;
  return p;
}

template <int kStages, int kSLog2, bool kHint>
__global__ void __launch_bounds__(kBulkThreads)
copy_bulk_kernel(const pec_copy_desc* __restrict__ d, int n, uint64_t total,
                 const uint64_t* __restrict__ total_dev, int lg) {
  constexpr int kBulkStages = kStages;
  constexpr int kStageLog2 = kSLog2;
  extern __shared__ __align__(128) uint8_t ring[];  // kBulkStages * stage
  if (total_dev != nullptr) {
    const uint64_t t = *total_dev;
    total = t < total ? t : total;
  }
  __shared__ __align__(8) uint64_t bars[kBulkStages];
  const int piece_log2 = lg < kStageLog2 ? lg : kStageLog2;
  const uint32_t stage_bytes = 1u << piece_log2;
  const uint32_t per_chunk = 1u << (lg - piece_log2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    // ---- single-thread TMA driver -------------------------------------
    const uint64_t chunks = blockIdx.x < total ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t items = chunks * per_chunk;
    uint32_t bytes_of[kBulkStages];
    uint8_t* dst_of[kBulkStages];
    pecdev::DescCursor cur;  // items are issued in increasing chunk order
    uint64_t policy = 0;
    if (kHint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    auto issue = [&](uint64_t j, int s) {
      const Piece p = piece_of(d, n, lg, j, per_chunk, piece_log2, cur);
      bytes_of[s] = p.bytes;
      dst_of[s] = p.dst;
      if (p.bytes) {
        mbar_expect_tx(&bars[s], p.bytes);
        if (kHint)
          bulk_g2s_hint(ring + (uint64_t)s * stage_bytes, p.src, p.bytes, &bars[s], policy);
        else
          bulk_g2s(ring + (uint64_t)s * stage_bytes, p.src, p.bytes, &bars[s]);
      } else {
        mbar_arrive(&bars[s]);  // keep the stage's phase sequence in step
      }
    };
    const uint64_t pre = items < (uint64_t)kBulkStages ? items : (uint64_t)kBulkStages;
    for (uint64_t j = 0; j < pre; ++j) issue(j, (int)j);
    for (uint64_t j = 0; j < items; ++j) {
      const int s = (int)(j % kBulkStages);
      mbar_wait(&bars[s], (uint32_t)((j / kBulkStages) & 1u));
      if (bytes_of[s]) {
        if (kHint)
          bulk_s2g_hint(dst_of[s], ring + (uint64_t)s * stage_bytes, bytes_of[s], policy);
        else
          bulk_s2g(dst_of[s], ring + (uint64_t)s * stage_bytes, bytes_of[s]);
      }
      bulk_commit();  // one group per item (possibly empty) keeps counts exact
      // refill the stage consumed one step earlier with item j-1+kStages
      if (j >= 1 && j - 1 + kBulkStages < items) {
        bulk_wait_read<1>();  // the store of item j-1 has read its stage
        issue(j - 1 + kBulkStages, (int)((j - 1) % kBulkStages));
      }
    }
    bulk_wait_all();
  } else {
    // ---- edge workers: unaligned heads/tails and incongruent chunks -----
    const int wid = threadIdx.x - 32;  // warps 1..3 (96 threads)
    if (wid >= 0) {
      pecdev::DescCursor cur;
      for (uint64_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
        const ChunkView v = chunk_view(d, n, ch, lg, cur);
        if (v.body == 0 && v.len > 0) {
          // incongruent or tiny chunk: plain copy by the 96 edge threads
          const uintptr_t sa = reinterpret_cast<uintptr_t>(v.s);
          const uintptr_t ta = reinterpret_cast<uintptr_t>(v.t);
          if (((sa ^ ta) & 3u) == 0 && v.len >= 8) {
            const uint64_t head = (4u - (sa & 3u)) & 3u;
            if ((uint64_t)wid < head) v.t[wid] = v.s[wid];
            const uint32_t* ws = reinterpret_cast<const uint32_t*>(v.s + head);
            uint32_t* wt = reinterpret_cast<uint32_t*>(v.t + head);
            const uint64_t nw = (v.len - head) >> 2;
            for (uint64_t w = wid; w < nw; w += kBulkThreads - 32) wt[w] = __ldg(ws + w);
            const uint64_t ts = head + (nw << 2);
            if ((uint64_t)wid < v.len - ts) v.t[ts + wid] = v.s[ts + wid];
          } else {
            for (uint64_t b = wid; b < v.len; b += kBulkThreads - 32) v.t[b] = v.s[b];
          }
        } else {
          if ((uint64_t)wid < v.head) v.t[wid] = v.s[wid];
          const uint64_t ts = v.head + v.body;
          if ((uint64_t)wid < v.len - ts) v.t[ts + wid] = v.s[ts + wid];
        }
      }
    }
  }
}

// ------------------------------------------------------------------------
// device-side plan expansion (load-aware snapshots without a host round trip)
// ------------------------------------------------------------------------
// The template is the rank's entry list for "every expert due", in the
// reference's order (planner.py:263-295: owned, experts by (layer, expert),
// non-expert modules).  For any due set the rank's entries are the
// subsequence whose (layer, expert) is selected (layer < 0: always kept).
//
// Placement (the StagingLayout rule: offset >= previous end, == source mod
// A) is a scan: every placed offset is == its source mod A, so the previous
// kept entry ends at (s_prev + n_prev) mod A and entry i's pad is
// (s_i - s_prev - n_prev) mod A — known without the absolute position.
// Offsets are then an exclusive prefix sum of (pad + n), chunk starts a
// prefix sum of ceil(n / 2^lg): one block, CUB block scans over tiles of
// kExpandThreads entries with carries between tiles.
constexpr int kExpandThreads = 512;

struct PrevKept {  // scan element: index of the latest kept entry so far
  __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

__global__ void __launch_bounds__(kExpandThreads)
expand_plan_kernel(const pec_plan_template* __restrict__ tmpl, int n,
                   const int32_t* __restrict__ sel, int L, int K,
                   uint64_t state_base, uint64_t stage_base, int lg, uint64_t align,
                   pec_copy_desc* __restrict__ out, uint64_t* __restrict__ totals) {
  using ScanU = cub::BlockScan<unsigned long long, kExpandThreads>;
  using ScanI = cub::BlockScan<int, kExpandThreads>;
  __shared__ union {
    typename ScanU::TempStorage u;
    typename ScanI::TempStorage i;
  } tmp;
  __shared__ uint64_t end_mod[kExpandThreads];   // (s + n) mod A of kept entries in the tile
  __shared__ unsigned long long carry_bytes, carry_chunks;
  __shared__ uint64_t carry_end;                   // end mod A of the last kept entry so far
  __shared__ int carry_any;
  const uint64_t span = 1ull << lg;
  const uint64_t amask = align - 1;                // align is a power of two
  if (threadIdx.x == 0) {
    carry_bytes = 0;
    carry_chunks = 0;
    carry_end = 0;
    carry_any = 0;
  }
  __syncthreads();
  for (int base = 0; base < n; base += kExpandThreads) {
    const int i = base + threadIdx.x;
    bool keep = false;
    uint64_t src = 0, nb = 0;
    if (i < n) {
      const pec_plan_template t = tmpl[i];
      src = t.src_offset;
      nb = t.nbytes;
      PEC_DCHECK(t.layer < L);
      if (t.layer < 0) {
        keep = true;
      } else if (t.layer < L) {
        for (int k = 0; k < K; ++k) keep |= (sel[(int64_t)t.layer * K + k] == t.expert);
      }
    }
    // previous kept entry inside this tile (or -1 -> carried end)
    int prev = -1;
    ScanI(tmp.i).ExclusiveScan(keep ? (int)threadIdx.x : -1, prev, -1, PrevKept());
    end_mod[threadIdx.x] = (src + nb) & amask;
    __syncthreads();
    const uint64_t prev_end = prev >= 0 ? end_mod[prev] : (carry_any ? carry_end : 0);
    const uint64_t pad = keep ? ((src - prev_end) & amask) : 0;
    const unsigned long long size = keep ? (unsigned long long)(pad + nb) : 0ull;
    const unsigned long long nch = keep ? (unsigned long long)((nb + span - 1) / span) : 0ull;
    unsigned long long pos_before = 0, tile_bytes = 0;
    ScanU(tmp.u).ExclusiveSum(size, pos_before, tile_bytes);
    __syncthreads();
    unsigned long long ch_before = 0, tile_chunks = 0;
    ScanU(tmp.u).ExclusiveSum(nch, ch_before, tile_chunks);
    if (i < n) {
      pec_copy_desc d;
      d.src = state_base + src;
      d.first_chunk = carry_chunks + ch_before;
      const uint64_t off = carry_bytes + pos_before + pad;
      d.dst = stage_base + (keep ? off : carry_bytes + pos_before);
      d.nbytes = keep ? nb : 0;
      out[i] = d;
    }
    // the last thread's inclusive "latest kept" index is the tile's last kept entry
    __shared__ int tile_last;
    if (threadIdx.x == kExpandThreads - 1) tile_last = keep ? (int)threadIdx.x : prev;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (tile_last >= 0) {
        carry_end = end_mod[tile_last];
        carry_any = 1;
      }
      carry_bytes += tile_bytes;
      carry_chunks += tile_chunks;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = carry_chunks;
    totals[1] = carry_bytes;
  }
}

// Per-device launch geometry, computed once per kernel variant (attribute
// setting and occupancy queries are host round trips that would otherwise
// sit between the caller's start event and the kernel).
struct Geometry {
  int ready = 0;
  int grid = 0;
  int smem = 0;
};

template <int kStages, int kSLog2, bool kHint, int kMaxPerSM = 64, int kGridDiv = 1>
int launch_bulk(const pec_copy_desc* descs, int n, uint64_t total, const uint64_t* total_dev,
                int lg, cudaStream_t st) {
  static Geometry geo[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return PEC_E_CUDA;
  Geometry& g = geo[dev];
  auto kern = copy_bulk_kernel<kStages, kSLog2, kHint>;
  if (!g.ready) {
    g.smem = kStages << kSLog2;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem) !=
        cudaSuccess)
      return PEC_E_CUDA;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBulkThreads, g.smem);
    if (per_sm > kMaxPerSM) per_sm = kMaxPerSM;
    const int sms = sm_count() / kGridDiv;  // narrow variants leave SMs to co-running kernels
    g.grid = (sms < 1 ? 1 : sms) * (per_sm < 1 ? 1 : per_sm);
    g.ready = 1;
  }
  const int smem = kStages << (lg < kSLog2 ? lg : kSLog2);
  const uint64_t grid = (uint64_t)g.grid < total ? (uint64_t)g.grid : total;
  kern<<<(unsigned)grid, kBulkThreads, smem, st>>>(descs, n, total, total_dev, lg);
  return launch_status();
}

int launch_vec(const pec_copy_desc* descs, int n, uint64_t total, const uint64_t* total_dev,
               int lg, cudaStream_t st) {
  static Geometry geo[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return PEC_E_CUDA;
  Geometry& g = geo[dev];
  if (!g.ready) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_vec_kernel, kVecThreads, 0);
    g.grid = sm_count() * (per_sm < 1 ? 1 : per_sm);
    g.ready = 1;
  }
  const uint64_t grid = (uint64_t)g.grid < total ? (uint64_t)g.grid : total;
  copy_vec_kernel<<<(unsigned)grid, kVecThreads, 0, st>>>(descs, n, total, total_dev, lg);
  return launch_status();
}

// mode 1: vector engine; 2: TMA bulk engine (the default); 10-16: bulk-engine
// ring/occupancy variants, 17-20: on 1/2 .. 1/8 of the SMs, 21-23: two CTAs per SM, kept for
// benchmarking (tools/pack_variants.py, tools/overlap_probe.py).
int launch_copy(const pec_copy_desc* descs, int n, uint64_t total, const uint64_t* total_dev,
                int lg, int mode, void* stream) {
  if (n < 0 || lg < 12 || lg > 24) return PEC_E_INVAL;
  const bool known = (mode >= 0 && mode <= 2) || (mode >= 10 && mode <= 23);
  if (!known) return PEC_E_INVAL;
  if (total == 0 || n == 0) return PEC_OK;
  if (descs == nullptr) return PEC_E_INVAL;
  cudaStream_t st = as_stream(stream);
  switch (mode) {
    case 1: return launch_vec(descs, n, total, total_dev, lg, st);
    case 10: return launch_bulk<3, 15, false, 1>(descs, n, total, total_dev, lg, st);
    case 11: return launch_bulk<2, 15, false, 1>(descs, n, total, total_dev, lg, st);
    case 12: return launch_bulk<4, 15, false, 1>(descs, n, total, total_dev, lg, st);
    case 13: return launch_bulk<4, 14, false, 1>(descs, n, total, total_dev, lg, st);
    case 14: return launch_bulk<3, 15, true, 1>(descs, n, total, total_dev, lg, st);
    case 15: return launch_bulk<2, 16, false, 1>(descs, n, total, total_dev, lg, st);
    case 16: return launch_bulk<6, 15, false, 1>(descs, n, total, total_dev, lg, st);
    // narrow: a fraction of the SMs (overlap studies with co-running training kernels)
    case 17: return launch_bulk<3, 15, true, 1, 2>(descs, n, total, total_dev, lg, st);
    case 18: return launch_bulk<3, 15, true, 1, 4>(descs, n, total, total_dev, lg, st);
    case 19: return launch_bulk<6, 15, true, 1, 4>(descs, n, total, total_dev, lg, st);
    case 20: return launch_bulk<6, 15, true, 1, 8>(descs, n, total, total_dev, lg, st);
    // two CTAs (two independent TMA rings) per SM
    case 21: return launch_bulk<3, 15, true, 2>(descs, n, total, total_dev, lg, st);
    case 22: return launch_bulk<2, 15, true, 2>(descs, n, total, total_dev, lg, st);
    case 23: return launch_bulk<3, 14, true, 2>(descs, n, total, total_dev, lg, st);
    // default (measured best on B200, tools/pack_variants.py): one CTA per
    // SM, 3 x 32 KiB stages (two loads in flight while one stage drains),
    // L2 evict_first on both directions (streamed once; keeps L2 for the
    // training kernels the pack overlaps with)
    default: return launch_bulk<3, 15, true, 1>(descs, n, total, total_dev, lg, st);
  }
}

template <typename Id>
int launch_token_hist(const Id* idx, int L, int64_t n_per_layer, int E, const int64_t* cap,
                      int64_t* counters, int tiers, int64_t* delivered, uint32_t* scratch,
                      void* stream) {
  if (L < 1 || L > 65535 || E < 1 || n_per_layer < 0 || tiers < 0) return PEC_E_INVAL;
  if (E > kMaxExperts) return PEC_E_RANGE;
  if (scratch == nullptr || (n_per_layer > 0 && idx == nullptr)) return PEC_E_INVAL;
  if (tiers > 0 && counters == nullptr) return PEC_E_INVAL;
  const int sms = sm_count();
  // enough CTAs to fill the GPU, each with >= one full unrolled sweep of ids
  int64_t per_layer = (int64_t)sms * 4 / L;
  const int64_t sweep = (int64_t)kHistThreads * kHistUnroll;
  const int64_t need = (n_per_layer + sweep - 1) / sweep;
  if (per_layer > need) per_layer = need;
  if (per_layer < 1) per_layer = 1;
  dim3 grid((unsigned)per_layer, (unsigned)L);
  const size_t smem = (size_t)(E + 1) * sizeof(uint32_t);
  token_hist_kernel<Id><<<grid, kHistThreads, smem, as_stream(stream)>>>(
      idx, L, n_per_layer, E, cap, counters, tiers, delivered, scratch);
  return launch_status();
}

}  // namespace

// ========================================================================
// C ABI
// ========================================================================
extern "C" {

int pec_abi_version(void) { return PEC_ABI_VERSION; }

const char* pec_strerror(int code) {
  switch (code) {
    case PEC_OK: return "ok";
    case PEC_E_INVAL: return "invalid argument";
    case PEC_E_CUDA: return "CUDA launch/runtime error";
    case PEC_E_RANGE: return "size exceeds a kernel limit";
    case PEC_E_IO: return "file I/O failed";
    case PEC_E_CRASH: return "injected crash: write budget exhausted";
    default: return "unknown error";
  }
}

int pec_token_hist(const int32_t* idx, int L, int64_t n_per_layer, int E,
                   const int64_t* cap, int64_t* counters, int tiers,
                   int64_t* delivered, uint32_t* scratch, void* stream) {
  return launch_token_hist(idx, L, n_per_layer, E, cap, counters, tiers, delivered, scratch,
                           stream);
}

int pec_token_hist_i64(const int64_t* idx, int L, int64_t n_per_layer, int E,
                       const int64_t* cap, int64_t* counters, int tiers,
                       int64_t* delivered, uint32_t* scratch, void* stream) {
  return launch_token_hist(idx, L, n_per_layer, E, cap, counters, tiers, delivered, scratch,
                           stream);
}

int pec_select_sequential(int64_t c, int L, int E, int width, int stride,
                          int32_t* out, void* stream) {
  if (L < 1 || E < 1 || width < 1 || stride < 0 || c < 0 || out == nullptr) return PEC_E_INVAL;
  const int W = width < E ? width : E;
  const int64_t total = (int64_t)L * W;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  select_sequential_kernel<<<blocks, 256, 0, as_stream(stream)>>>(c, L, E, width, stride, out);
  return launch_status();
}

int pec_select_load_aware(int64_t* counters, int L, int E, int K,
                          const int32_t* pool, int P, int32_t* out,
                          int zero_selected, void* stream) {
  if (L < 1 || E < 1 || K < 1 || counters == nullptr || out == nullptr) return PEC_E_INVAL;
  if (pool != nullptr && P < 0) return PEC_E_INVAL;
  if (E > kMaxExperts) return PEC_E_RANGE;
  cudaStream_t st = as_stream(stream);
  const int p = pool ? P : 0;
  if (E <= 32)
    select_load_aware_kernel<32, 1><<<L, 32, 0, st>>>(counters, E, K, pool, p, out,
                                                      zero_selected);
  else if (E <= 256)
    select_load_aware_kernel<256, 1><<<L, 256, 0, st>>>(counters, E, K, pool, p, out,
                                                        zero_selected);
  else if (E <= 1024)
    select_load_aware_kernel<256, 4><<<L, 256, 0, st>>>(counters, E, K, pool, p, out,
                                                        zero_selected);
  else
    select_load_aware_kernel<256, 16><<<L, 256, 0, st>>>(counters, E, K, pool, p, out,
                                                         zero_selected);
  return launch_status();
}

int pec_pack(const pec_copy_desc* descs, int n, uint64_t total_chunks,
             int chunk_log2, int mode, void* stream) {
  return launch_copy(descs, n, total_chunks, nullptr, chunk_log2, mode == 0 ? 2 : mode, stream);
}

int pec_unpack(const pec_copy_desc* descs, int n, uint64_t total_chunks,
               int chunk_log2, int mode, void* stream) {
  return launch_copy(descs, n, total_chunks, nullptr, chunk_log2, mode == 0 ? 2 : mode, stream);
}

int pec_pack_indirect(const pec_copy_desc* descs, int n, uint64_t max_chunks,
                      const uint64_t* total_chunks_dev, int chunk_log2, int mode, void* stream) {
  if (total_chunks_dev == nullptr) return PEC_E_INVAL;
  return launch_copy(descs, n, max_chunks, total_chunks_dev, chunk_log2, mode == 0 ? 2 : mode,
                     stream);
}

int pec_expand_plan(const pec_plan_template* tmpl, int n, const int32_t* sel, int L, int K,
                    uint64_t state_base, uint64_t stage_base, int chunk_log2, int stage_align,
                    pec_copy_desc* out, uint64_t* totals, void* stream) {
  if (n < 0 || L < 1 || K < 1 || chunk_log2 < 12 || chunk_log2 > 24 || stage_align < 1) return PEC_E_INVAL;
  if (n > 0 && (tmpl == nullptr || out == nullptr)) return PEC_E_INVAL;
  if (sel == nullptr || totals == nullptr) return PEC_E_INVAL;
  if (stage_align & (stage_align - 1)) return PEC_E_INVAL;
  expand_plan_kernel<<<1, kExpandThreads, 0, as_stream(stream)>>>(
      tmpl, n, sel, L, K, state_base, stage_base, chunk_log2, (uint64_t)stage_align, out, totals);
  return launch_status();
}

int64_t pec_plan_chunks(pec_copy_desc* host_descs, int n, int chunk_log2) {
  if (n < 0 || chunk_log2 < 12 || chunk_log2 > 24) return PEC_E_INVAL;
  if (n > 0 && host_descs == nullptr) return PEC_E_INVAL;
  uint64_t acc = 0;
  const uint64_t span = 1ull << chunk_log2;
  for (int i = 0; i < n; ++i) {
    host_descs[i].first_chunk = acc;
    acc += (host_descs[i].nbytes + span - 1) / span;
  }
  return (int64_t)acc;
}

}  // extern "C"
