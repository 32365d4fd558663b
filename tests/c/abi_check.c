/*
 * abi_check.c — exercises include/pec.h from plain C, linked against
 * libpec.so, the way a non-Python caller would bind the boundary.
 *
 *   abi_check          host entry points only (no GPU needed)
 *   abi_check gpu      plus pec_pack / pec_unpack / pec_select_sequential /
 *                      pec_token_hist on device 0 through the CUDA runtime
 *
 * Prints one line per check; exit status 0 iff every check passed.
 * Known answers follow the reference: store.crc32c("123456789") ==
 * 0xE3069283 (pkg/src/mocsim/store.py:49-70), select_window
 * (selector.py:21-27), bincount + cap (simulator.py:88-95).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "pec.h"

static int failures = 0;

static void check(int ok, const char* what) {
  printf("%s %s\n", ok ? "ok  " : "FAIL", what);
  if (!ok) ++failures;
}

static uint32_t crc_bitwise(const uint8_t* p, size_t n, uint32_t crc) {
  crc = ~crc;
  for (size_t i = 0; i < n; ++i) {
    crc ^= p[i];
    for (int b = 0; b < 8; ++b) crc = (crc & 1u) ? (crc >> 1) ^ 0x82F63B78u : crc >> 1;
  }
  return ~crc;
}

static void host_checks(void) {
  check(pec_abi_version() == PEC_ABI_VERSION, "pec_abi_version == PEC_ABI_VERSION");
  check(pec_strerror(PEC_OK) != NULL && pec_strerror(PEC_E_INVAL) != NULL &&
            pec_strerror(PEC_E_IO) != NULL && pec_strerror(-99) != NULL,
        "pec_strerror covers every code");
  check(pec_crc32c("123456789", 9, 0) == 0xE3069283u, "pec_crc32c known answer 0xE3069283");
  check(pec_crc32c("", 0, 0) == 0u, "pec_crc32c of nothing == 0");

  enum { N = 1 << 20 };
  uint8_t* buf = (uint8_t*)malloc(N);
  uint32_t x = 12345u;
  for (int i = 0; i < N; ++i) {
    x = x * 1664525u + 1013904223u;
    buf[i] = (uint8_t)(x >> 24);
  }
  const uint32_t whole = pec_crc32c(buf, N, 0);
  check(whole == crc_bitwise(buf, N, 0), "pec_crc32c == bitwise CRC-32C on 1 MiB");
  check(pec_crc32c(buf + 1000, N - 1000, pec_crc32c(buf, 1000, 0)) == whole,
        "pec_crc32c chains like store.crc32c(data, crc)");
  check(pec_crc32c_combine(pec_crc32c(buf, 4097, 0), pec_crc32c(buf + 4097, N - 4097, 0),
                           N - 4097) == whole,
        "pec_crc32c_combine(A, B, |B|) == crc(A||B)");

  uint64_t offs[3] = {0, 17, 300000}, lens[3] = {0, 65536 + 3, N - 300000};
  uint32_t out[3];
  int rc = pec_crc32c_many(buf, offs, lens, 3, out, 4);
  check(rc == PEC_OK && out[0] == 0u && out[1] == pec_crc32c(buf + 17, lens[1], 0) &&
            out[2] == pec_crc32c(buf + 300000, lens[2], 0),
        "pec_crc32c_many over 3 regions, 4 threads");

  pec_copy_desc t[4] = {{0, 0, 0, 0}, {0, 0, 1, 0}, {0, 0, 32768, 0}, {0, 0, 32769, 0}};
  int64_t total = pec_plan_chunks(t, 4, 15);
  check(total == 4 && t[0].first_chunk == 0 && t[1].first_chunk == 0 && t[2].first_chunk == 1 &&
            t[3].first_chunk == 2,
        "pec_plan_chunks prefix (0, 1, 32768, 32769 B at 32 KiB chunks)");
  check(pec_plan_chunks(t, 4, 3) < 0, "pec_plan_chunks rejects chunk_log2 out of range");

  char dir[] = "/tmp/pec_abi_XXXXXX";
  if (mkdtemp(dir) != NULL) {
    char p0[64], p1[64];
    snprintf(p0, sizeof p0, "%s/a.bin", dir);
    snprintf(p1, sizeof p1, "%s/b.bin", dir);
    const char* paths[2] = {p0, p1};
    const void* bufs[2] = {buf, buf + 5};
    uint64_t wl[2] = {N, 123};
    uint32_t wc[2];
    rc = pec_write_files(paths, bufs, wl, 2, wc, 2, 0);
    int ok = rc == PEC_OK && wc[0] == whole && wc[1] == pec_crc32c(buf + 5, 123, 0);
    FILE* f = fopen(p1, "rb");
    uint8_t back[123];
    ok = ok && f != NULL && fread(back, 1, 123, f) == 123 && memcmp(back, buf + 5, 123) == 0;
    if (f) fclose(f);
    check(ok, "pec_write_files writes exact bytes and returns their CRCs");
    const char* bad[1] = {"/nonexistent_dir_pec/x.bin"};
    check(pec_write_files(bad, bufs, wl, 1, NULL, 1, 0) == PEC_E_IO,
          "pec_write_files reports PEC_E_IO");
    unlink(p0);
    unlink(p1);
    rmdir(dir);
  }
  free(buf);
}

#ifdef PEC_ABI_CHECK_GPU
#include <cuda_runtime.h>

static void gpu_checks(void) {
  enum { S = 8 << 20 };
  uint8_t *state, *staging;
  pec_copy_desc* dtab;
  check(cudaMalloc((void**)&state, S) == cudaSuccess && cudaMalloc((void**)&staging, S) == cudaSuccess &&
            cudaMalloc((void**)&dtab, 8 * sizeof(pec_copy_desc)) == cudaSuccess,
        "cudaMalloc state/staging/table");
  uint8_t* h = (uint8_t*)malloc(S);
  uint8_t* back = (uint8_t*)malloc(S);
  uint32_t x = 7u;
  for (int i = 0; i < S; ++i) {
    x = x * 1664525u + 1013904223u;
    h[i] = (uint8_t)(x >> 24);
  }
  cudaMemcpy(state, h, S, cudaMemcpyHostToDevice);
  cudaMemset(staging, 0, S);
  /* byte-granular ranges, staging offsets congruent to the source mod 256 */
  const uint64_t src[5] = {0, 4096 + 3, 100000, 1 << 20, 3 << 20};
  const uint64_t len[5] = {1, 70000, 1 << 19, 5, (2 << 20) + 77};
  pec_copy_desc t[5];
  uint64_t pos = 0;
  for (int i = 0; i < 5; ++i) {
    uint64_t dst = pos + ((src[i] - pos) & 255u);
    t[i].src = (uint64_t)(uintptr_t)(state + src[i]);
    t[i].dst = (uint64_t)(uintptr_t)(staging + dst);
    t[i].nbytes = len[i];
    pos = dst + len[i];
  }
  int64_t total = pec_plan_chunks(t, 5, 15);
  cudaMemcpy(dtab, t, sizeof t, cudaMemcpyHostToDevice);
  int rc = pec_pack(dtab, 5, (uint64_t)total, 15, 0, NULL);
  cudaDeviceSynchronize();
  cudaMemcpy(back, staging, S, cudaMemcpyDeviceToHost);
  int ok = rc == PEC_OK;
  for (int i = 0; i < 5 && ok; ++i)
    ok = memcmp(back + (t[i].dst - (uint64_t)(uintptr_t)staging), h + src[i], len[i]) == 0;
  check(ok, "pec_pack: 5 byte-granular ranges bit-exact");

  /* unpack into a zeroed state */
  cudaMemset(state, 0, S);
  pec_copy_desc u[5];
  for (int i = 0; i < 5; ++i) {
    u[i] = t[i];
    u[i].src = t[i].dst;
    u[i].dst = t[i].src;
  }
  total = pec_plan_chunks(u, 5, 15);
  cudaMemcpy(dtab, u, sizeof u, cudaMemcpyHostToDevice);
  rc = pec_unpack(dtab, 5, (uint64_t)total, 15, 0, NULL);
  cudaDeviceSynchronize();
  cudaMemcpy(back, state, S, cudaMemcpyDeviceToHost);
  ok = rc == PEC_OK;
  for (int i = 0; i < 5 && ok; ++i) ok = memcmp(back + src[i], h + src[i], len[i]) == 0;
  check(ok, "pec_unpack restores the ranges bit-exact");

  /* sequential selection: c=3, L=2, E=8, K=2 -> layer m: {(m+6)%8, (m+7)%8} sorted */
  int32_t* dsel;
  cudaMalloc((void**)&dsel, 4 * sizeof(int32_t));
  rc = pec_select_sequential(3, 2, 8, 2, 2, dsel, NULL);
  int32_t hsel[4];
  cudaMemcpy(hsel, dsel, sizeof hsel, cudaMemcpyDeviceToHost);
  check(rc == PEC_OK && hsel[0] == 6 && hsel[1] == 7 && hsel[2] == 0 && hsel[3] == 7,
        "pec_select_sequential == select_window(c=3, K=2, E=8)");

  /* token histogram with a cap: ids {0,0,0,1,5,-1,9} over E=8, cap 2 */
  const int32_t ids[7] = {0, 0, 0, 1, 5, -1, 9};
  const int64_t cap = 2;
  int32_t* dids;
  int64_t *dcnt, *dcap;
  uint32_t* dscr;
  cudaMalloc((void**)&dids, sizeof ids);
  cudaMalloc((void**)&dcnt, 8 * sizeof(int64_t));
  cudaMalloc((void**)&dcap, sizeof cap);
  cudaMalloc((void**)&dscr, 9 * sizeof(uint32_t));
  cudaMemcpy(dids, ids, sizeof ids, cudaMemcpyHostToDevice);
  cudaMemcpy(dcap, &cap, sizeof cap, cudaMemcpyHostToDevice);
  cudaMemset(dcnt, 0, 8 * sizeof(int64_t));
  cudaMemset(dscr, 0, 9 * sizeof(uint32_t));
  rc = pec_token_hist(dids, 1, 7, 8, dcap, dcnt, 1, NULL, dscr, NULL);
  int64_t hc[8];
  cudaMemcpy(hc, dcnt, sizeof hc, cudaMemcpyDeviceToHost);
  check(rc == PEC_OK && hc[0] == 2 && hc[1] == 1 && hc[5] == 1 && hc[2] == 0 && hc[7] == 0,
        "pec_token_hist == min(bincount, cap), out-of-range ids dropped");
  check(pec_pack(dtab, -1, 0, 15, 0, NULL) == PEC_E_INVAL, "pec_pack rejects n < 0");
  check(cudaGetLastError() == cudaSuccess, "no CUDA error");
  cudaFree(state);
  cudaFree(staging);
  cudaFree(dtab);
  cudaFree(dsel);
  cudaFree(dids);
  cudaFree(dcnt);
  cudaFree(dcap);
  cudaFree(dscr);
  free(h);
  free(back);
}
#endif

int main(int argc, char** argv) {
  host_checks();
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) {
#ifdef PEC_ABI_CHECK_GPU
    gpu_checks();
#else
    check(0, "built without PEC_ABI_CHECK_GPU");
#endif
  }
  printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
