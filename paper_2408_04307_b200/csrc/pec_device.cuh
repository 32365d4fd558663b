// pec_device.cuh — helpers shared by the PEC kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pec.h"

// Device-side invariant checks, compiled into the debug library only
// (libpec_debug.so, -DPEC_DEBUG; _build.build_debug()).  compute-sanitizer
// is not available on the B200 pool, so out-of-range indices and overruns are
// caught by these checks plus guard bands around every output buffer
// (tools/guard_kernels.py).  A failed check prints and traps (the launch
// then reports an error on the next synchronisation).
#ifdef PEC_DEBUG
#include <cstdio>
#define PEC_DCHECK(cond, ...)                                                    \
  do {                                                                           \
    if (!(cond)) {                                                               \
      printf("PEC_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define PEC_DCHECK(cond, ...) \
  do {                        \
  } while (0)
#endif

namespace pecdev {

// SM count of the current device, cached per device id (a pure function of
// the device, not library state).
inline int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PEC_OK : PEC_E_CUDA;
}

// Largest i with first_chunk[i] <= ch (empty descriptors share the next
// one's first_chunk and are skipped by taking the largest such i).
__device__ __forceinline__ int find_desc(const pec_copy_desc* __restrict__ d, int n, uint64_t ch) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&d[mid].first_chunk) <= ch) lo = mid; else hi = mid - 1;
  }
  PEC_DCHECK(n > 0 && lo >= 0 && lo < n && __ldg(&d[lo].first_chunk) <= ch);
  return lo;
}

// Monotone cursor over the table for a CTA walking chunk indices upward
// (ch = blockIdx.x, + gridDim.x, ...): resumes from the previous descriptor
// instead of a fresh binary search, so the common case is one L1-resident
// load of the next descriptor's first_chunk rather than a chain of
// dependent global loads per chunk.
struct DescCursor {
  int i = -1;
  __device__ __forceinline__ int find(const pec_copy_desc* __restrict__ d, int n, uint64_t ch) {
    if (i < 0 || __ldg(&d[i].first_chunk) > ch) {
      i = find_desc(d, n, ch);
      return i;
    }
    int steps = 0;
    while (i + 1 < n && __ldg(&d[i + 1].first_chunk) <= ch) {
      if (++steps > 8) {  // far jump: binary search instead
        i = find_desc(d, n, ch);
        return i;
      }
      ++i;
    }
    PEC_DCHECK(i >= 0 && i < n && __ldg(&d[i].first_chunk) <= ch);
    return i;
  }
};

}  // namespace pecdev
