// lat_bench.cu — dependent-chain latency (cycles per op) of the primitives on the STATE
// warp's serial decision path: FP64 mul/add, IEEE FP64 division, uniform-datapath warp
// reduction (REDUX), double shuffle, 32-bit modulo, ballot+popc.
#include <cstdio>
#include <cstdint>
#define N 4096
__global__ void k(double* out, long long* cyc, double a0, uint32_t m0) {
  const int lane = threadIdx.x & 31;
  double a = a0 + lane * 1e-9, b = 1.0000001;
  uint32_t u = m0 + lane;
  long long t0, t1;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = __dmul_rn(a, b);
  t1 = clock64(); if (lane == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, 1e-12);
  t1 = clock64(); if (lane == 0) cyc[1] = t1 - t0;
  // division chain
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) a = __ddiv_rn(a + 1.0, 1.0000003);
  t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) * 8;
  // REDUX min chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) u = __reduce_min_sync(0xffffffffu, u + (uint32_t)lane) + 1u;
  t1 = clock64(); if (lane == 0) cyc[3] = t1 - t0;
  // double shuffle chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1e-12;
  t1 = clock64(); if (lane == 0) cyc[4] = t1 - t0;
  // 32-bit modulo chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) u = (u * 2654435761u + 7u) % (3u + (u & 7u));
  t1 = clock64(); if (lane == 0) cyc[5] = t1 - t0;
  // ballot + popc chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) u = __popc(__ballot_sync(0xffffffffu, ((u + lane) & 1u) != 0)) + u;
  t1 = clock64(); if (lane == 0) cyc[6] = t1 - t0;
  // DSETP + select chain (min of doubles)
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = (a < b) ? a + 1e-9 : b - 1e-9;
  t1 = clock64(); if (lane == 0) cyc[7] = t1 - t0;
  out[lane] = a + u;
}

// __nanosleep granularity and global-memory round trips (one warp, lane 0)
__global__ void k2(unsigned long long* g, long long* cyc) {
  if (threadIdx.x != 0) return;
  long long t0, t1;
  const int n = 256;
  for (int s = 0; s < 4; ++s) {
    const unsigned ns = 32u << (2 * s);  // 32, 128, 512, 2048
    t0 = clock64();
    for (int i = 0; i < n; ++i) __nanosleep(ns);
    t1 = clock64();
    cyc[8 + s] = (t1 - t0) / n;
  }
  // dependent L2 loads (ld.acquire.gpu), atomics, CAS
  unsigned long long v = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    unsigned int x;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(g + (v & 1)) : "memory");
    v += x + 1;
  }
  t1 = clock64(); cyc[12] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) v += atomicAdd(g + 2 + (v & 1), 1ull);
  t1 = clock64(); cyc[13] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) v += atomicCAS(g + 4, v, v + 1);
  t1 = clock64(); cyc[14] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __threadfence_system(); v += clock64() & 1; }
  t1 = clock64(); cyc[15] = (t1 - t0) / n;
  g[6] = v;
}
// fence flavours, idle, after one store to a host-mapped word (the PUBLISH pattern)
__global__ void k3(volatile unsigned int* host, long long* cyc) {
  const int n = 64;
  long long t0, t1;
  unsigned long long v = 0;
#define FENCE_CASE(idx, stmt)                                        \
  t0 = clock64();                                                    \
  for (int i = 0; i < n; ++i) { host[i & 7] = i; stmt; v += clock64() & 1; } \
  t1 = clock64(); cyc[idx] = (t1 - t0) / n;
  FENCE_CASE(0, asm volatile("fence.sc.sys;" ::: "memory"))
  FENCE_CASE(1, asm volatile("fence.acq_rel.sys;" ::: "memory"))
  FENCE_CASE(2, asm volatile("fence.sc.gpu;" ::: "memory"))
  FENCE_CASE(3, asm volatile("fence.acq_rel.gpu;" ::: "memory"))
  FENCE_CASE(4, asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(host + 8), "r"((unsigned)v) : "memory"))
  FENCE_CASE(5, (void)0)
  FENCE_CASE(6, asm volatile("fence.release.sys;" ::: "memory"))
  FENCE_CASE(7, asm volatile("fence.release.gpu;" ::: "memory"))
  host[15] = (unsigned)v;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 1.0, 3); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0, 3);
  unsigned long long* g; cudaMalloc(&g, 64); cudaMemset(g, 0, 64);
  long long* c2; cudaMalloc(&c2, 16 * 8);
  k2<<<1, 32>>>(g, c2); cudaDeviceSynchronize();
  long long h2[16]; cudaMemcpy(h2, c2, 16 * 8, cudaMemcpyDeviceToHost);
  printf("{\"nanosleep_32\": %lld, \"nanosleep_128\": %lld, \"nanosleep_512\": %lld, \"nanosleep_2048\": %lld, "
         "\"ld_acquire_gpu\": %lld, \"atomic_add\": %lld, \"atomic_cas\": %lld, \"fence_sys_idle\": %lld}\n",
         h2[8], h2[9], h2[10], h2[11], h2[12], h2[13], h2[14], h2[15]);
  {
    unsigned int* hw; cudaHostAlloc(&hw, 64, cudaHostAllocMapped);
    unsigned int* dw; cudaHostGetDevicePointer(&dw, hw, 0);
    long long* c3; cudaMalloc(&c3, 8 * 8);
    k3<<<1, 1>>>(dw, c3); cudaDeviceSynchronize();
    k3<<<1, 1>>>(dw, c3); cudaDeviceSynchronize();
    long long h3[8]; cudaMemcpy(h3, c3, 64, cudaMemcpyDeviceToHost);
    printf("{\"after_host_store\": {\"fence_sc_sys\": %lld, \"fence_acq_rel_sys\": %lld, \"fence_sc_gpu\": %lld, "
           "\"fence_acq_rel_gpu\": %lld, \"st_release_sys\": %lld, \"none\": %lld, \"fence_release_sys\": %lld, "
           "\"fence_release_gpu\": %lld}}\n",
           h3[0], h3[1], h3[2], h3[3], h3[4], h3[5], h3[6], h3[7]);
  }
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* names[8] = {"dmul", "dadd", "ddiv_rn", "redux_min", "shfl_xor_f64", "mod_u32", "ballot_popc", "dsetp_sel"};
  printf("{");
  for (int i = 0; i < 8; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", names[i], (double)h[i] / N);
  printf("}\n");
  return 0;
}
