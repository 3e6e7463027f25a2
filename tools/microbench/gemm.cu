// bgemm_kernel throughput on large and K-heavy shapes (TF/s)
#include <cstdio>
#include "../../paper_1803_10270_b200/csrc/tp_gemm.cuh"
namespace tp { void set_last_error(cudaError_t) {} int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : -1; } }
using namespace tp;
int main() {
  double *A, *B, *C;
  cudaMalloc(&A, 8ull << 27); cudaMalloc(&B, 8ull << 27); cudaMalloc(&C, 8ull << 27);
  cudaMemset(A, 0, 8ull << 27); cudaMemset(B, 0, 8ull << 27);
  struct S { int M, N, K, nb; } shapes[] = {{4096, 4096, 1024, 1}, {64, 64, 4096, 256}, {64, 64, 4096, 1024}, {128, 16, 128, 4}, {64, 4096, 64, 64}, {64, 64, 4096, 128}, {64, 64, 64, 16384}, {64, 64, 64, 2048}};
  double* part; cudaMalloc(&part, 8ull << 26);
  for (auto sh : shapes) {
    BGemm g = bgemm_desc(sh.M, sh.N, sh.K, A, sh.K, 1, B, sh.N, 1, C, sh.N, 1);
    g.nb1 = sh.nb; g.sA1 = 0; g.sB1 = 0; g.sC1 = (long long)sh.M * sh.N;
    g.ksplit = bgemm_pick_split(g); g.part = part;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    bgemm_launch(g, 0); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) bgemm_launch(g, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double fl = 2.0 * sh.M * sh.N * sh.K * sh.nb;
    printf("split %d M %5d N %5d K %5d batch %5d: %8.3f ms  %6.2f TF/s  (%s)\n", g.ksplit, sh.M, sh.N, sh.K, sh.nb, ms, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
