// Shared helpers for the rlra_b200 sm_100a kernels: error plumbing behind the
// C ABI, column-major indexing, a deterministic grid barrier for the
// cooperative panel kernels, and small warp utilities.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

namespace rlra {

// thread-local last error string for rlra_b200_last_error()
void set_error(const char* fmt, ...);
const char* last_error();

#define RLRA_CHECK_CUDA(expr)                                                   \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::rlra::set_error("%s failed at %s:%d: %s", #expr, __FILE__, __LINE__,    \
                        cudaGetErrorString(_e));                                \
      return -1;                                                                \
    }                                                                           \
  } while (0)

#define RLRA_REQUIRE(cond, ...)                                                 \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ::rlra::set_error(__VA_ARGS__);                                           \
      return -2;                                                                \
    }                                                                           \
  } while (0)

// Process-wide count of kernels this library launched (bench.py's gpu_launches).
void note_launch();

#define RLRA_LAUNCHED()                                                          \
  do {                                                                          \
    ::rlra::note_launch();                                                      \
    RLRA_CHECK_CUDA(cudaGetLastError());                                        \
  } while (0)

// Optional per-kernel CUDA-event timing (bench.py's roofline): while enabled
// (rlra_b200_ktimer_enable), ktimer_mark() records an event on the launch
// stream before (end=false) and after (end=true) a named kernel launch.
enum KTimerId { KT_OZ_GEMM = 0, KT_OZ_RESIDUE_A, KT_OZ_NORMS, KT_OZ_CRT, KT_OZ_RESIDUE_B, KT_COUNT };
bool ktimer_on();
void ktimer_mark(int id, cudaStream_t st, bool end);

struct DeviceInfo {
  int sm_count = 0;
  int max_smem_optin = 0;
};
const DeviceInfo& device_info();

// Column-major element access, 64-bit indices throughout (C5 A is 8.6e9 elems).
__host__ __device__ __forceinline__ int64_t cm(int64_t i, int64_t j, int64_t ld) {
  return i + j * ld;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

// Non-contracted multiply-then-subtract: a - l*u rounded twice, exactly like the
// reference's `lu[i, jj] - lu[i, j] * ujj` built with -ffp-contract=off
// (rlra/_lu_cython.pyx:52-55, pkg/setup.py:25-27).
__device__ __forceinline__ double sub_mul_nofma(double a, double l, double u) {
  return __dsub_rn(a, __dmul_rn(l, u));
}

// Sense-reversing grid barrier over global memory for cooperative launches.
// `bar[0]` = arrival counter, `bar[1]` = generation.  All CTAs of the grid must
// be co-resident (launched with cudaLaunchCooperativeKernel).
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = bar + 1;
    unsigned int gen = *vgen;
    __threadfence();
    unsigned int arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
        __nanosleep(20);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Monotonic grid barrier: every CTA adds 1 (release), then waits until the
// counter reaches `target` = (barriers so far) * gridDim (acquire).  The host
// zeroes the counter once per factorization and tracks the running base.
__device__ __forceinline__ void grid_barrier_mono(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// ---- cluster / mbarrier / bulk-copy helpers (inline PTX)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}
// local smem [src, src+bytes) -> peer smem dst (shared::cluster), completing
// `bytes` of transactions on the peer's mbarrier
__device__ __forceinline__ void bulk_push(unsigned dst_cluster, const void* src, unsigned bytes,
                                          unsigned mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}

}  // namespace rlra
