/*
 * mmtest.c -- the paper's test program as a plain C client of the C ABI
 * (include/mm.h): no Python, no PyTorch -- cudaMalloc'd buffers and libmm_b200.so only.
 *
 *   mmtest [-O n] [-R r] [-L levels]
 *
 * C = A (8A) with A an n x n random matrix (U[0,1), reading R13; B = 8A by
 * MultiplyWithScalar), N := NaivKahan; each method runs r times
 * (defaults n = 400, r = 10) and the table reports the median time per
 * product (CUDA events) and NormInf(N - C) (the difference formed on the host: this is the test
 * program's bookkeeping, not the product path).  Strassen runs the paper's padding plan
 * (levels = -1) and, as an extra row, an explicit depth.
 *
 * Build: gcc -O2 -std=c99 -I include -I /usr/local/cuda/include tools/mmtest.c \
 *          -L paper_1106_1347_b200 -lmm_b200 -L /usr/local/cuda/lib64 -lcudart -lm \
 *          -Wl,-rpath,'$ORIGIN/../paper_1106_1347_b200' -o tools/mmtest
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mm.h"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(2);                                                                   \
    }                                                                            \
  } while (0)

static int cmp_float(const void* a, const void* b) {
  float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

/* splitmix64 -> U[0,1) doubles (53 random bits) */
static uint64_t g_state = 1106134742ull;
static double urand(void) {
  uint64_t z = (g_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

typedef struct {
  const char* name;
  int method;
  int levels;
} Row;

int main(int argc, char** argv) {
  int64_t n = 400;
  int reps = 10, lv = 2;
  for (int i = 1; i + 1 < argc; i += 2) {
    if (!strcmp(argv[i], "-O")) n = atoll(argv[i + 1]);
    else if (!strcmp(argv[i], "-R")) reps = atoi(argv[i + 1]);
    else if (!strcmp(argv[i], "-L")) lv = atoi(argv[i + 1]);
  }
  if (n < 1 || reps < 1) {
    fprintf(stderr, "usage: mmtest [-O n] [-R r] [-L levels]\n");
    return 1;
  }
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  double* hA = (double*)malloc(bytes);
  double* hB = (double*)malloc(bytes);
  double* hN = (double*)malloc(bytes);
  double* hC = (double*)malloc(bytes);
  for (int64_t i = 0; i < n * n; i++) {
    hA[i] = urand();
    hB[i] = 8.0 * hA[i]; /* B = 8A (MultiplyWithScalar, exact) */
  }
  double *A, *B, *C;
  CK(cudaMalloc((void**)&A, bytes));
  CK(cudaMalloc((void**)&B, bytes));
  CK(cudaMalloc((void**)&C, bytes));
  CK(cudaMemcpy(A, hA, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB, bytes, cudaMemcpyHostToDevice));

  Row rows[] = {{"N := NaivKahan", MM_KAHAN, 0},      {"NaivStandard", MM_NAIVE, 0},
                {"StrassenNaiv", MM_STRASSEN, -1},     {"StrassenWinograd", MM_STRASSEN_WINOGRAD, -1},
                {"WinogradOriginal", MM_WINOGRAD, 0}, {"WinogradScaled", MM_WINOGRAD_SCALED, 0},
                {"StrassenNaiv (levels L)", MM_STRASSEN, -2},
                {"StrassenWinograd (levels L)", MM_STRASSEN_WINOGRAD, -2}};
  const int nrows = (int)(sizeof(rows) / sizeof(rows[0]));

  printf("%s\n", mm_version());
  printf("+-----------------------------------------------------------------------+\n");
  printf("|            TIME TEST FOR METHODS OF MATRIX MULTIPLICATION             |\n");
  printf("| C = A*(8A), where A is a (n x n) random matrix with n = %10lld    |\n", (long long)n);
  printf("+-----------------------------------------------------------------------+\n");
  printf("| %-28s| %16s | %20s |\n", "method", "time (sec)", "NormInf( N-C )");
  printf("+-----------------------------------------------------------------------+\n");

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float* ts = (float*)malloc(sizeof(float) * (size_t)reps);
  for (int r = 0; r < nrows; r++) {
    const int levels = rows[r].levels == -2 ? lv : rows[r].levels;
    if (levels == -1 && n > 4096) { /* P:286's plan recurses to 7^k order-17..32 bases: k > 7 impractical */
      printf("| %-28s| %38s |\n", rows[r].name, "skipped (paper plan, n > 4096)");
      continue;
    }
    const size_t ws_bytes = mm_workspace_size(rows[r].method, n, n, n, levels);
    void* ws = NULL;
    if (ws_bytes) CK(cudaMalloc(&ws, ws_bytes));
    int rc = mm_gemm(rows[r].method, A, B, C, n, n, n, levels, ws, ws_bytes, NULL, 0); /* warm-up */
    if (rc != MM_OK) {
      printf("| %-28s| %38s |\n", rows[r].name, mm_status_string(rc));
      if (ws) cudaFree(ws);
      continue;
    }
    for (int k = 0; k < reps; k++) {
      CK(cudaEventRecord(e0, 0));
      mm_gemm(rows[r].method, A, B, C, n, n, n, levels, ws, ws_bytes, NULL, 0);
      CK(cudaEventRecord(e1, 0));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ts[k], e0, e1));
    }
    qsort(ts, (size_t)reps, sizeof(float), cmp_float);
    const double sec = ts[reps / 2] / 1e3;
    CK(cudaMemcpy(r == 0 ? hN : hC, C, bytes, cudaMemcpyDeviceToHost));
    if (r == 0) {
      printf("| %-28s| %16.6f | %20s |\n", rows[r].name, sec, "");
    } else {
      double dev = 0.0; /* NormInf(N - C): max row sum of |N - C| */
      for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t j = 0; j < n; j++) s += fabs(hN[i * n + j] - hC[i * n + j]);
        if (s > dev) dev = s;
      }
      printf("| %-28s| %16.6f | %20.10f |\n", rows[r].name, sec, dev);
    }
    if (ws) CK(cudaFree(ws));
  }
  printf("+-----------------------------------------------------------------------+\n");
  /* end to end from HOST memory through the ABI (mm_methods_host): the test program's six methods on
   * page-locked copies of A and B, every product landing in host memory; Kahan's must equal N */
  {
    const int ms[] = {MM_NAIVE, MM_STRASSEN, MM_WINOGRAD_SCALED, MM_WINOGRAD, MM_STRASSEN_WINOGRAD, MM_KAHAN};
    const int nm = (int)(sizeof(ms) / sizeof(ms[0]));
    double *pA, *pB, *pC[6];
    CK(cudaHostAlloc((void**)&pA, bytes, cudaHostAllocDefault));
    CK(cudaHostAlloc((void**)&pB, bytes, cudaHostAllocDefault));
    for (int i = 0; i < nm; i++) CK(cudaHostAlloc((void**)&pC[i], bytes, cudaHostAllocDefault));
    memcpy(pA, hA, bytes);
    memcpy(pB, hB, bytes);
    const size_t hws = mm_methods_host_workspace_size(ms, nm, n, n, n, lv);
    void* dws = NULL;
    CK(cudaMalloc(&dws, hws));
    int rc = mm_methods_host(ms, nm, pA, pB, pC, n, n, n, lv, 4, dws, hws, 0); /* warm-up */
    CK(cudaEventRecord(e0, 0));
    if (rc == MM_OK) rc = mm_methods_host(ms, nm, pA, pB, pC, n, n, n, lv, 4, dws, hws, 0);
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    float ms_e2e = 0.f;
    CK(cudaEventElapsedTime(&ms_e2e, e0, e1));
    const int same = rc == MM_OK && memcmp(pC[nm - 1], hN, bytes) == 0;
    printf("end to end from host memory (mm_methods_host, %d methods, levels %d): %s, %.3f ms; "
           "NaivKahan product bitwise the device call's: %s\n",
           nm, lv, mm_status_string(rc), ms_e2e, same ? "yes" : "NO");
    cudaFree(dws);
    cudaFreeHost(pA);
    cudaFreeHost(pB);
    for (int i = 0; i < nm; i++) cudaFreeHost(pC[i]);
    if (!same) return 4;
  }
  /* the C ABI's error paths, from C */
  int bad = mm_naive(NULL, B, C, n, n, n, 0);
  int alias = mm_naive(A, B, A, n, n, n, 0);
  printf("error paths: NULL A -> %s; C aliasing A -> %s\n", mm_status_string(bad), mm_status_string(alias));
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  free(hA);
  free(hB);
  free(hN);
  free(hC);
  free(ts);
  return (bad == MM_ERR_ARG && alias == MM_ERR_ALIAS) ? 0 : 3;
}
