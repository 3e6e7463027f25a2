// Shared helpers for the tpde_b200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include <map>
#include <mutex>
#include <utility>
#include <vector>
#include "../../include/tpde_b200.h"

// clock64 phase probes / phase-skipping timing hooks of the fused kernels (tp_debug_set_als_profile,
// tp_debug_set_als_skip, tp_debug_set_circ_prof): compiled in only with -DTP_ALS_PROBES=1 (TPDE_PROBES=1 build);
// the product library carries none (their code alone costs 2-3 % on the latency-bound kernels)
#ifndef TP_ALS_PROBES
#define TP_ALS_PROBES 0
#endif

#define TP_MAXD 8          // max modes of a CP tensor handled by the fused ALS kernels
#define TP_MAXD_GEN 16     // max modes of the streamed ALS, inner product, apply and contraction kernels
#define TP_RMAX 32         // max fitted rank in the warp-register Cholesky

namespace tp {

void set_last_error(cudaError_t e);
int cuda_status(cudaError_t e);  // records and maps to TP_ECUDA / TP_OK

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Host tables that never change for a given operator/shape (GEMM offset triples,
// per-mode table lists) live on the device once: the first call uploads them
// synchronously, every later call (and CUDA-graph capture) only reads them.
template <class T>
inline const T* device_table(const std::vector<T>& v) {
  static std::mutex mu;
  static std::map<std::pair<int, std::vector<char>>, void*> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<char> key(reinterpret_cast<const char*>(v.data()), reinterpret_cast<const char*>(v.data() + v.size()));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, key});
  if (it != cache.end()) return static_cast<const T*>(it->second);
  void* p = nullptr;
  if (cudaMalloc(&p, v.empty() ? 8 : v.size() * sizeof(T)) != cudaSuccess) return nullptr;
  if (!v.empty() && cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  if (cache.size() > 256) cache.clear();   // (leaks the old tables; bounded)
  cache.emplace(std::make_pair(dev, std::move(key)), p);
  return static_cast<const T*>(p);
}

// carve device workspace
struct Carver {
  char* base;
  size_t cap, used = 0;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T> T* take(size_t n) {
    size_t off = align_up(used);
    used = off + n * sizeof(T);
    return reinterpret_cast<T*>(base + off);
  }
  bool ok() const { return used <= cap; }
};

// ---- device helpers --------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// mma.sync m8n8k4 f64: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragments (PTX ISA): A: lane holds A[lane>>2][lane&3]; B: lane holds B[lane&3][lane>>2];
// C/D: lane holds C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// shared-memory load through a 32-bit shared-window address (keeps the address
// arithmetic in one register; generic pointers into dynamic shared memory are
// rematerialised from SR_CgaCtaId under register pressure)
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// ---- bulk async copies (TMA engine, non-tensor form) + mbarrier -----------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TP_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TP_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy; bytes and both addresses must be multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 32-bit shared::cluster address of the same offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

// shared (this CTA) -> shared (peer CTA of the cluster) bulk copy, completing on
// the peer's mbarrier; addresses from mapa_u32, bytes a multiple of 16
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, const void* src, uint32_t bytes, uint32_t peer_bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(peer_bar)
      : "memory");
}

// order this thread's prior generic-proxy accesses with later async-proxy (bulk copy) ones
// (all state spaces: the bulk copies read global data that other CTAs wrote with
// generic stores, and overwrite shared memory this CTA read with generic loads)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// same, for copies that write peer CTAs' shared memory
__device__ __forceinline__ void fence_proxy_async_cluster() {
  asm volatile("fence.proxy.async.shared::cluster;\n" ::: "memory");
}


// fast reciprocal: MUFU seed + 2 Newton steps (<= 1 ulp, no slow path)
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

// fast reciprocal square root: MUFU seed + 2 Newton steps (x > 0, finite)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

}  // namespace tp
