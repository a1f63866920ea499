// cuBLASLt algorithm search for the header step's prefill-sized GEMMs (measurement tool, not
// product code): out[R][N] (f32) = x[R][K] (bf16) . W[N][K]^T (bf16), R = stacked hi/lo rows.
// Times every heuristic cuBLASLt returns (workspace up to 64 MB) with each launch reading a
// different weight copy (copies > 2x L2), against the default algorithm (heuristic #0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_lt_search tools/lt_search.cu -lcublasLt
//   tools/_lt_search [R]
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    auto e_ = (x);                                                          \
    if ((int)e_ != 0) {                                                     \
      fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)e_); \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 144;
  struct Shape { const char* name; int N, K; };
  const Shape shapes[] = {{"qkv", 6144, 4096}, {"o_proj", 4096, 4096},
                          {"gate_up", 28672, 4096}, {"down", 4096, 14336}};
  cublasLtHandle_t lt;
  CK(cublasLtCreate(&lt));
  const size_t ws_bytes = 64ull << 20;
  void* ws;
  CK(cudaMalloc(&ws, ws_bytes));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (const Shape& sh : shapes) {
    const size_t wbytes = (size_t)sh.N * sh.K * 2;
    int copies = (int)((300ull << 20) / wbytes) + 2;
    if (copies > 12) copies = 12;
    char* W;
    CK(cudaMalloc(&W, wbytes * copies));
    CK(cudaMemset(W, 0x3c, wbytes * copies));
    __nv_bfloat16* X;
    CK(cudaMalloc(&X, (size_t)R * sh.K * 2));
    CK(cudaMemset(X, 0x3c, (size_t)R * sh.K * 2));
    float* Y;
    CK(cudaMalloc(&Y, (size_t)R * sh.N * 4));
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA)));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB)));
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, sh.K, sh.N, sh.K));
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, sh.K, R, sh.K));
    CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, sh.N, R, sh.N));
    cublasLtMatmulPreference_t pref;
    CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                            &ws_bytes, sizeof(ws_bytes)));
    std::vector<cublasLtMatmulHeuristicResult_t> res(64);
    int n = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 64, res.data(), &n));
    const float one = 1.f, zero = 0.f;
    printf("== %s  R=%d N=%d K=%d  weights %.1f MB  heuristics %d\n", sh.name, R, sh.N, sh.K,
           wbytes / 1e6, n);
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      auto run = [&](int c) {
        return cublasLtMatmul(lt, op, &one, W + (size_t)c * wbytes, la, X, lb, &zero, Y, lc, Y,
                              lc, &res[i].algo, ws, ws_bytes, s);
      };
      if (run(0) != CUBLAS_STATUS_SUCCESS) continue;
      for (int w = 0; w < 3; ++w) run(w % copies);
      const int reps = 4 * copies;
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < reps; ++r) run(r % copies);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = 1e3 * ms / reps;
      int tile = -1, splitk = -1, stages = -1, cta = -1;
      size_t sz;
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile,
                                           sizeof(tile), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk,
                                           sizeof(splitk), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages,
                                           sizeof(stages), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID,
                                           &cta, sizeof(cta), &sz);
      printf("  #%2d  %8.2f us  %6.0f GB/s  ws %6.1f MB  tile %d splitk %d stages %d cluster %d\n",
             i, us, wbytes / us / 1e3, res[i].workspaceSize / 1e6, tile, splitk, stages, cta);
    }
    cudaFree(W);
    cudaFree(X);
    cudaFree(Y);
    cublasLtMatmulPreferenceDestroy(pref);
    cublasLtMatrixLayoutDestroy(la);
    cublasLtMatrixLayoutDestroy(lb);
    cublasLtMatrixLayoutDestroy(lc);
    cublasLtMatmulDescDestroy(op);
  }
  return 0;
}
