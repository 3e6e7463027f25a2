// DSMEM all-to-all throughput inside one cluster (B200): every CTA sends a block of
// B bytes to each of the other S-1 CTAs, then waits for its own S-1 blocks.
//  mode 0: warp-coalesced st.shared::cluster.v2.f64 + barrier.cluster
//  mode 1: cp.async.bulk shared::cta -> shared::cluster by one thread, mbarrier complete_tx
//  mode 2: barrier.cluster only
// Prints cycles per round (CTA 0) and bytes sent per cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__global__ void k(int mode, int S, int B, int reps, long long* out) {
  extern __shared__ __align__(128) double sm[];
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int nd = B / 8;
  double* src = sm;                  // B bytes
  double* inbox = sm + nd;           // S slots of B bytes
  uint64_t* bar = reinterpret_cast<uint64_t*>(inbox + (size_t)S * nd);
  for (int e = threadIdx.x; e < nd; e += blockDim.x) src[e] = rank + e;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cbar();
  uint32_t ph = 0;
  long long t0 = 0;
  for (int it = -2; it < reps; ++it) {
    if (it == 0) t0 = clock64();
    if (mode == 0) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int q = warp; q < S; q += nw) {
        if (q == (int)rank) continue;
        const uint32_t dst = mapa(su32(inbox + (size_t)rank * nd), q);
        for (int e = 2 * lane; e < nd; e += 64) {
          const double2 v = *reinterpret_cast<const double2*>(src + e);
          asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" :: "r"(dst + 8u * e), "d"(v.x), "d"(v.y) : "memory");
        }
      }
      cbar();
    } else if (mode == 1) {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bar)), "r"((S - 1) * B) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int q = 0; q < S; ++q) {
          if (q == (int)rank) continue;
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(mapa(su32(inbox + (size_t)rank * nd), q)), "r"(su32(src)), "r"(B), "r"(mapa(su32(bar), q)) : "memory");
        }
      }
      asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                   :: "r"(su32(bar)), "r"(ph) : "memory");
      ph ^= 1;
      cbar();   // keep rounds separate (WAR on the inbox)
    } else {
      cbar();
    }
  }
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long* d; cudaMalloc(&d, 8);
  for (int S : {16, 8, 4}) {
    const int ncl = S == 16 ? 7 : (S == 8 ? 15 : 32);
    for (int mode : {2, 0, 1}) {
      for (int B : {512, 1536, 4096, 8192}) {
        if (mode == 2 && B != 512) continue;
        if ((size_t)(S + 1) * B + 64 > 200 * 1024) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(S * ncl); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        const int reps = 200;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, mode, S, B, reps, d);
        e = e == cudaSuccess ? cudaDeviceSynchronize() : e;
        long long cyc = 0; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("S=%d mode=%d B=%d failed: %s\n", S, mode, B, cudaGetErrorString(e)); cudaGetLastError(); continue; }
        printf("S=%2d clusters=%2d mode=%d block=%5dB  %7lld cycles/round  %6.1f B/cycle sent per SM\n", S, ncl, mode, B,
               cyc, mode == 2 ? 0.0 : (double)(S - 1) * B / cyc);
      }
    }
  }
  return 0;
}
