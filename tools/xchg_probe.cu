// Exchange-latency probe for the GEPP panel protocol: 16 CTAs of one cluster
// repeatedly (a) reduce a value over the CTA (one __syncthreads), (b) publish
// a 144-byte record to every peer, (c) wait for all 16 records.  Variants:
//   0: DSMEM st.async (lanes 0..15 of warp 0, 9 x 16 B each) + mbarrier tx
//   1: global staging + fence.proxy.async + one TMA multicast + mbarrier tx
//   2: DSMEM plain remote stores + barrier.cluster arrive.release/wait.acquire
//   3: like 0, but all 8 warps wait on the mbarrier (as the GEPP kernel does)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int CS = 16, RECD = 18, T = 256;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, int r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t* b, unsigned par) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}

__device__ __forceinline__ void wait_par_cluster(uint64_t* b, unsigned par) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(T, 1) probe(int variant, int iters, double* gstage,
                                                                          unsigned long long* out) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ __align__(16) double recv[2][CS][RECD];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(8) uint64_t mbar2[2];  // variant 4: 16 remote arrivals per phase, no tx bytes
  __shared__ __align__(16) double stagebuf[RECD + 2];
  __shared__ double red[8];
  const int b = cluster.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned tx = CS * RECD * 8;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar2[0], CS);
    mbar_init(&mbar2[1], CS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    expect_tx(&mbar[0], variant == 6 ? CS * 16u : tx);
    expect_tx(&mbar[1], variant == 6 ? CS * 16u : tx);
  }
  cluster.sync();
  double acc = b + tid;
  unsigned phase = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const int par = it & 1;
    // (a) a CTA reduction with one barrier
    double v = acc;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = lane < 8 ? red[lane] : -1.0;
    for (int o = 4; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    // (b) publish
    if (variant == 0 || variant == 3) {
      if (warp == 0 && lane < CS) {
        const unsigned dst = mapa(smem_u32(&recv[par][b][0]), lane), bar = mapa(smem_u32(&mbar[par]), lane);
        for (int c = 0; c < RECD; c += 2)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                           dst + 8 * c),
                       "d"(v + c), "d"(v), "r"(bar)
                       : "memory");
      }
    } else if (variant == 4) {
      if (warp == 0 && lane < CS) {
        const unsigned dst = mapa(smem_u32(&recv[par][b][0]), lane), bar = mapa(smem_u32(&mbar2[par]), lane);
        for (int c = 0; c < RECD; c += 2)
          asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(dst + 8 * c), "d"(v + c), "d"(v) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
      }
    } else if (variant == 5) {
      if (warp == 0) {
        if (lane < RECD) stagebuf[lane] = v + lane;
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane < CS) {
          const unsigned dst = mapa(smem_u32(&recv[par][b][0]), lane), bar = mapa(smem_u32(&mbar[par]), lane);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "r"(smem_u32(stagebuf)), "r"((unsigned)(RECD * 8)), "r"(bar)
              : "memory");
        }
      }
    } else if (variant == 6) {
      if (warp == 0 && lane < CS) {
        const unsigned dst = mapa(smem_u32(&recv[par][b][0]), lane), bar = mapa(smem_u32(&mbar[par]), lane);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
                     "d"(v), "d"(v), "r"(bar)
                     : "memory");
      }
    } else if (variant == 1) {
      if (tid == 0) {
        double* slot = gstage + ((size_t)par * CS + b) * RECD;
        for (int c = 0; c < RECD; c++) slot[c] = v + c;
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
            "[%3], %4;" ::"r"(smem_u32(&recv[par][b][0])),
            "l"(slot), "r"((unsigned)(RECD * 8)), "r"(smem_u32(&mbar[par])), "h"((unsigned short)0xffff)
            : "memory");
      }
    } else {
      if (warp == 0 && lane < CS) {
        double* dst = cluster.map_shared_rank(&recv[par][b][0], lane);
        for (int c = 0; c < RECD; c++) dst[c] = v + c;
      }
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    // (c) wait for all records
    if (variant == 4) {
      wait_par_cluster(&mbar2[par], (phase >> par) & 1u);
      phase ^= 1u << par;
    } else if (variant != 2) {
      if (variant == 3 || variant >= 5 || tid == 0) {
        wait_par(&mbar[par], (phase >> par) & 1u);
      }
      phase ^= 1u << par;
      if (tid == 0) expect_tx(&mbar[par], variant == 6 ? CS * 16u : tx);
      if (variant == 0 || variant == 1) __syncthreads();
    }
    double s = 0.0;
    if (lane < CS) s = recv[par][lane][1];
    acc += s * 1e-30;
  }
  unsigned long long t1 = clock64();
  if (tid == 0) out[b] = (t1 - t0) / iters;
  if (tid == 0 && acc == 12345.0) out[b + 16] = 1;
  cluster.sync();
}

int main() {
  double* g;
  unsigned long long* o;
  cudaMalloc(&g, 1 << 20);
  cudaMalloc(&o, 64 * 8);
  const char* names[] = {"st.async DSMEM + mbarrier (1 waiter)", "global + TMA multicast + mbarrier",
                         "DSMEM stores + cluster barrier", "st.async DSMEM + mbarrier (all threads wait)",
                         "remote st + remote mbarrier arrive.release", "smem stage + 16 DSMEM bulk copies",
                         "st.async key only (16 B per peer)"};
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int v = 0; v < 7; v++) {
    probe<<<16, T>>>(v, 2000, g, o);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-46s %6llu cycles/iter (CTA0) %6llu (CTA15)  %s\n", names[v], h[0], h[15], cudaGetErrorString(e));
  }
  return 0;
}
