// Latency probes on a 16-CTA cluster (B200): cluster barrier, DSMEM load,
// dependent FP64 chains, __drcp_rn, block argmax, fence.proxy.async.global.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ double ieee_div_by(double x, double d, double rcp) {
  const double ax = fabs(x), ad = fabs(d);
  if (ax > 0x1p-960 && ax < 0x1p+960 && ad > 0x1p-960 && ad < 0x1p+960) {
    const double q0 = __dmul_rn(x, rcp);
    const double rem = fma(-d, q0, x);
    return fma(rem, rcp, q0);
  }
  return x / d;
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 1) probe(unsigned long long* out, double seed) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double buf[64];
  const int tid = threadIdx.x, b = cluster.block_rank();
  if (tid < 64) buf[tid] = (double)((tid + 1) % 64);
  cluster.sync();
  unsigned long long t0, t1;
  double acc = seed;
  // (1) split cluster barrier round trip, 100 iterations
  t0 = clk();
  for (int i = 0; i < 100; i++) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  t1 = clk();
  if (tid == 0) out[b * 16 + 0] = (t1 - t0) / 100;
  // (1b) relaxed arrive
  t0 = clk();
  for (int i = 0; i < 100; i++) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  t1 = clk();
  if (tid == 0) out[b * 16 + 1] = (t1 - t0) / 100;
  // (2) dependent DSMEM loads from peer (b+1)%16
  unsigned addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(&buf[0])), "r"((b + 1) % 16));
  t0 = clk();
  int ci = 0;
  for (int i = 0; i < 100; i++) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr + ci * 8) : "memory");
    ci = (int)v;
  }
  t1 = clk();
  acc += ci;
  if (tid == 0) out[b * 16 + 2] = (t1 - t0) / 100;
  // (3) dependent DFMA chain
  double x = seed;
  t0 = clk();
  for (int i = 0; i < 100; i++) x = fma(x, 1.0000001, 1e-9);
  t1 = clk();
  acc += x;
  if (tid == 0) out[b * 16 + 3] = (t1 - t0) / 100;
  // (4) __drcp_rn chain
  t0 = clk();
  for (int i = 0; i < 100; i++) x = __drcp_rn(x + 1.0);
  t1 = clk();
  acc += x;
  if (tid == 0) out[b * 16 + 4] = (t1 - t0) / 100;
  // (5) 64-bit shuffle chain (fmax butterfly of 5 rounds), per round
  t0 = clk();
  for (int i = 0; i < 20; i++)
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  t1 = clk();
  acc += x;
  if (tid == 0) out[b * 16 + 5] = (t1 - t0) / 100;
  // (6) __syncthreads round trip
  t0 = clk();
  for (int i = 0; i < 100; i++) __syncthreads();
  t1 = clk();
  if (tid == 0) out[b * 16 + 6] = (t1 - t0) / 100;
  // (7) local smem dependent load
  t0 = clk();
  int ix = tid & 31;
  for (int i = 0; i < 100; i++) {
    double v = buf[ix];
    ix = (int)v;
  }
  t1 = clk();
  acc += ix;
  if (tid == 0) out[b * 16 + 7] = (t1 - t0) / 100;
  // (8) global store + fence.proxy.async.global
  t0 = clk();
  for (int i = 0; i < 20; i++) {
    if (tid == 0) {
      out[2048 + b] = t0 + i;
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
    }
  }
  t1 = clk();
  if (tid == 0) out[b * 16 + 8] = (t1 - t0) / 20;
  // (9) redux.min
  unsigned k = tid;
  t0 = clk();
  for (int i = 0; i < 100; i++) k = __reduce_min_sync(0xffffffffu, k + i) + (k & 1);
  t1 = clk();
  if (tid == 0) out[b * 16 + 9] = (t1 - t0) / 100;
  // (10) DMUL->DADD chain (sub_mul_nofma)
  t0 = clk();
  for (int i = 0; i < 100; i++) x = __dsub_rn(x, __dmul_rn(x, 1e-7));
  t1 = clk();
  acc += x + k;
  if (tid == 0) out[b * 16 + 10] = (t1 - t0) / 100;
  // (11) decision-like sequence by warp 0 after a cluster barrier, 16 reps
  {
    __shared__ double rec[2][18];
    __shared__ double diag[2][16];
    if (tid < 18) { rec[0][tid] = (tid == 0) ? (double)(b * 7 % 16) : (tid == 1 ? (double)b : 1.0 + tid); rec[1][tid] = rec[0][tid]; }
    if (tid < 16) { diag[0][tid] = 2.0 + tid; diag[1][tid] = 2.0 + tid; }
    cluster.sync();
    const int lane = tid & 31;
    unsigned ra, da;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&rec[0][0])), "r"(lane < 16 ? lane : 0));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(da) : "r"(smem_u32(&diag[0][(lane - 16) & 15])), "r"(0));
    unsigned long long tot = 0, tw = 0;
    for (int rep = 0; rep < 16; rep++) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      unsigned long long ta = clk();
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      unsigned long long tb = clk();
      if (tid < 32) {
        double rv = -1.0, dl = 0.0;
        if (lane < 16) asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(rv) : "r"(ra + (rep & 1) * 144) : "memory");
        if (lane >= 16) asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(dl) : "r"(da + (rep & 1) * 128) : "memory");
        double vm = rv;
        for (int o = 16; o; o >>= 1) vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
        const unsigned w = __reduce_min_sync(0xffffffffu, (rv == vm) ? (unsigned)lane : 32u);
        double ul = __shfl_sync(0xffffffffu, dl, 16 + (lane & 15));
        unsigned wa;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(wa) : "r"(smem_u32(&rec[rep & 1][2 + (lane & 15)])), "r"((int)(w & 15)));
        if (lane < 16) asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(ul) : "r"(wa) : "memory");
        buf[lane] = ul;
      }
      __syncthreads();
      unsigned long long tc = clk();
      tot += tc - tb;
      tw += tb - ta;
    }
    if (tid == 0) { out[b * 16 + 11] = tot / 16; out[b * 16 + 12] = tw / 16; }
  }
  // (13) 3 independent ieee divisions + look-ahead per thread, all 256 threads
  {
    double xs[3] = {seed + tid, seed * 2 + tid, seed * 3 + tid}, ys[3] = {1.0 + tid, 2.0, 3.0};
    const double d = 1.2345 + b, rcp = __drcp_rn(d);
    __syncthreads();
    unsigned long long ta = clk();
    for (int rep = 0; rep < 16; rep++) {
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const double l = ieee_div_by(xs[k], d, rcp);
        xs[k] = l;
        ys[k] = __dsub_rn(ys[k], __dmul_rn(l, 0.5));
      }
    }
    unsigned long long tb = clk();
    if (tid == 0) out[b * 16 + 13] = (tb - ta) / 16;
    acc += xs[0] + xs[1] + xs[2] + ys[0] + ys[1] + ys[2];
  }
  if (acc == 12345.678) out[4000] = 1;
  cluster.sync();
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 4096);
  cudaMemset(d, 0, 8 * 4096);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 2; rep++) probe<<<16, 256>>>(d, 1.0);
  cudaDeviceSynchronize();
  unsigned long long h[4096];
  cudaMemcpy(h, d, 8 * 4096, cudaMemcpyDeviceToHost);
  const char* names[] = {"cluster barrier release/acquire", "cluster barrier relaxed", "DSMEM ld dependent",
                         "DFMA dependent", "__drcp_rn dependent", "fmax shfl64 round", "__syncthreads",
                         "LDS dependent", "STG+fence.proxy.async.global", "redux.min", "DMUL+DSUB dependent"};
  printf("3x ieee_div + lookahead per thread (256 thr): %llu cycles\n", h[13]);
  printf("decision seq (warp0, 2 DSMEM rounds) %llu / %llu cycles; barrier wait %llu\n", h[11], h[15*16+11], h[12]);
  for (int i = 0; i < 11; i++) printf("%-36s %llu cycles (CTA0) %llu (CTA15)\n", names[i], h[i], h[15 * 16 + i]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
