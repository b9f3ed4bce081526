// Probe (dev tool): cuBLASLt int8 x int8 -> int32 GEMM in the key-switch shape on B200.
// D[m][n'] = sum_k B[m][k] * A[n'][k]  (A: 2528 x 24576 int8 "TN" operand, B: M x 24576 int8, D: M x 2528 int32)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ks_gemm_probe tools/ks_gemm_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  const int K = 24576, NP = 2528;
  const int M = argc > 1 ? atoi(argv[1]) : 4096;
  std::vector<int8_t> hA((size_t)NP * K), hB((size_t)M * K);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
  for (auto& v : hA) v = (int8_t)(rnd() & 0xFF);
  for (auto& v : hB) v = (rnd() % 3 == 0) ? 1 : 0;
  int8_t *dA, *dB; int32_t* dD;
  CK(cudaMalloc(&dA, hA.size())); CK(cudaMalloc(&dB, hB.size())); CK(cudaMalloc(&dD, (size_t)M * NP * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  cublasLtHandle_t lt; CK(cublasLtCreate(&lt));
  cublasLtMatmulDesc_t op; CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
  cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA)));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB)));
  cublasLtMatrixLayout_t la, lb, ld;
  CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, K, NP, K));   // A col-major K x NP (op T -> NP x K)
  CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, K, M, K));    // B col-major K x M
  CK(cublasLtMatrixLayoutCreate(&ld, CUDA_R_32I, NP, M, NP)); // D col-major NP x M
  size_t ws_bytes = 64 << 20; void* ws; CK(cudaMalloc(&ws, ws_bytes));
  cublasLtMatmulPreference_t pref; CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof(ws_bytes)));
  cublasLtMatmulHeuristicResult_t h[8]; int nres = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, ld, ld, pref, 8, h, &nres));
  printf("heuristics: %d\n", nres);
  if (!nres) return 2;
  int32_t one = 1, zero = 0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int a = 0; a < nres && a < 4; a++) {
    CK(cublasLtMatmul(lt, op, &one, dA, la, dB, lb, &zero, dD, ld, dD, ld, &h[a].algo, ws, ws_bytes, 0));
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; r++)
      CK(cublasLtMatmul(lt, op, &one, dA, la, dB, lb, &zero, dD, ld, dD, ld, &h[a].algo, ws, ws_bytes, 0));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("algo %d: %.3f ms  %.1f TOPS  %.1f ns per ciphertext\n", a, ms, 2.0 * M * K * NP / (ms * 1e-3) / 1e12, ms * 1e6 / M);
  }
  std::vector<int32_t> hD((size_t)M * NP);
  CK(cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int t = 0; t < 64; t++) {
    const int m = rnd() % M, n = rnd() % NP;
    int64_t ref = 0;
    for (int k = 0; k < K; k++) ref += (int64_t)hB[(size_t)m * K + k] * hA[(size_t)n * K + k];
    if (ref != hD[(size_t)m * NP + n]) bad++;
  }
  printf("check: %d / 64 mismatches\n", bad);
  return bad != 0;
}
