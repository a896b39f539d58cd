// tma_copy_bench.cu — copy-worker shapes for the engine's SM rails, measured alone:
//   ldg  one warp per 64 KiB chunk, 16 x 16 B loads per lane in flight, then the stores
//        (the engine's warp_copy);
//   tma  one warp per 64 KiB chunk, lane 0 drives a bulk-copy pipeline through shared
//        memory: cp.async.bulk global->shared completing on an mbarrier, then
//        cp.async.bulk shared->global, ST stages of P bytes per warp, so (ST - 1) x P bytes
//        of loads are in flight per warp instead of 8 KiB.
// Directions: H2D (pinned host -> HBM), D2H, BOTH (half the chunks each way, interleaved
// like the KV batch), D2D. Grid = CTAs x 8 warps; chunks are taken by ticket.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_copy_bench tools/tma_copy_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

struct Job {
  const uint8_t* src[2];
  uint8_t* dst[2];
  uint64_t chunk, n_chunks;
  int both;  // chunk i goes in direction (i / 32) & 1
  unsigned long long* ticket;
};

__device__ __forceinline__ void job_ptrs(const Job& J, uint64_t i, const uint8_t*& s, uint8_t*& d) {
  const int dir = J.both ? (int)((i >> 5) & 1) : 0;
  s = J.src[dir] + i * J.chunk;
  d = J.dst[dir] + i * J.chunk;
}

struct V4 { uint32_t x, y, z, w; };
__device__ __forceinline__ V4 ldg_v4(const void* p) {
  V4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg_v4(void* p, V4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__global__ void __launch_bounds__(256) k_ldg(Job J) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(J.ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= J.n_chunks) return;
    const uint8_t* s;
    uint8_t* d;
    job_ptrs(J, t, s, d);
    constexpr int U = 16;
    for (uint64_t off = (uint64_t)lane * 16; off < J.chunk; off += 32 * 16 * U) {
      V4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t o = off + (uint64_t)u * 512;
        if (o < J.chunk) r[u] = ldg_v4(s + o);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t o = off + (uint64_t)u * 512;
        if (o < J.chunk) stg_v4(d + o, r[u]);
      }
    }
    __threadfence_system();
    __syncwarp();
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int ST>
__global__ void __launch_bounds__(256) k_tma(Job J, uint32_t P) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* buf = sm + (size_t)warp * ST * P;
  __shared__ uint64_t bars[8][ST];
  if (lane == 0)
    for (int s = 0; s < ST; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase[ST];
  for (int s = 0; s < ST; ++s) phase[s] = 0;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(J.ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= J.n_chunks) break;
    if (lane == 0) {
      const uint8_t* s;
      uint8_t* d;
      job_ptrs(J, t, s, d);
      const uint32_t np = (uint32_t)((J.chunk + P - 1) / P);
      auto issue = [&](uint32_t i) {
        const uint32_t st = i % ST;
        const uint64_t off = (uint64_t)i * P;
        const uint32_t n = (uint32_t)((J.chunk - off) < P ? (J.chunk - off) : P);
        mbar_expect(&bars[warp][st], n);
        bulk_load(buf + (size_t)st * P, s + off, n, &bars[warp][st]);
      };
      for (uint32_t i = 0; i < np && i < (uint32_t)ST; ++i) issue(i);
      for (uint32_t i = 0; i < np; ++i) {
        const uint32_t st = i % ST;
        mbar_wait(&bars[warp][st], phase[st]);
        phase[st] ^= 1u;
        const uint64_t off = (uint64_t)i * P;
        const uint32_t n = (uint32_t)((J.chunk - off) < P ? (J.chunk - off) : P);
        bulk_store(d + off, buf + (size_t)st * P, n);
        if (i + ST < np) {
          bulk_wait_read<0>();  // store i has read stage st
          issue(i + ST);
        }
      }
      bulk_wait_all();
      __threadfence_system();
    }
    __syncwarp();
  }
}

int main(int argc, char** argv) {
  const uint64_t chunk = 64 << 10, nch = 4096, bytes = chunk * nch;
  uint8_t *h0, *h1, *d0, *d1, *hd0, *hd1;
  CK(cudaHostAlloc(&h0, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocMapped));
  memset(h0, 1, bytes);
  memset(h1, 2, bytes);
  CK(cudaHostGetDevicePointer(&hd0, h0, 0));
  CK(cudaHostGetDevicePointer(&hd1, h1, 0));
  CK(cudaMalloc(&d0, bytes));
  CK(cudaMalloc(&d1, bytes));
  CK(cudaMemset(d0, 3, bytes));
  CK(cudaMemset(d1, 4, bytes));
  unsigned long long* tk;
  CK(cudaMalloc(&tk, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Dir { const char* name; Job j; int ctas; };
  Job h2d{{hd0, hd0}, {d0, d0}, chunk, nch, 0, tk};
  Job d2h{{d0, d0}, {hd1, hd1}, chunk, nch, 0, tk};
  Job both{{d0, hd0}, {hd1, d1}, chunk, nch, 1, tk};
  Job d2d{{d0, d0}, {d1, d1}, chunk, nch, 0, tk};
  Dir dirs[] = {{"h2d", h2d, 48}, {"d2h", d2h, 48}, {"both", both, 48}, {"both96", both, 96}, {"both148", both, 148},
                {"d2d", d2d, 148}};
  const uint32_t Ps[] = {4096, 8192, 16384};
  for (const Dir& D : dirs) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      CK(cudaMemset(tk, 0, 8));
      cudaEventRecord(e0);
      k_ldg<<<D.ctas, 256>>>(D.j);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it && ms < best) best = ms;
    }
    printf("{\"dir\": \"%s\", \"ctas\": %d, \"kind\": \"ldg\", \"gbs\": %.2f}\n", D.name, D.ctas, bytes / (best * 1e-3) / 1e9);
    for (uint32_t P : Ps) {
      for (int st : {2, 3, 4}) {
        const size_t smem = (size_t)8 * st * P;
        if (smem > 200 * 1024) continue;
        cudaError_t e = cudaSuccess;
        best = 1e30f;
        for (int it = 0; it < 5; ++it) {
          CK(cudaMemset(tk, 0, 8));
          cudaEventRecord(e0);
          if (st == 2) {
            cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_tma<2><<<D.ctas, 256, smem>>>(D.j, P);
          } else if (st == 3) {
            cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_tma<3><<<D.ctas, 256, smem>>>(D.j, P);
          } else {
            cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_tma<4><<<D.ctas, 256, smem>>>(D.j, P);
          }
          e = cudaGetLastError();
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (it && ms < best) best = ms;
        }
        printf("{\"dir\": \"%s\", \"ctas\": %d, \"kind\": \"tma\", \"stages\": %d, \"piece\": %u, \"gbs\": %.2f%s}\n", D.name,
               D.ctas, st, P, bytes / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : ", \"err\": 1");
      }
    }
  }
  // correctness of the tma path once: d2d with the last config
  {
    CK(cudaMemset(tk, 0, 8));
    CK(cudaMemset(d1, 0, bytes));
    cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 3 * 8192);
    k_tma<3><<<148, 256, 8 * 3 * 8192>>>(d2d, 8192);
    CK(cudaDeviceSynchronize());
    uint8_t* chk = (uint8_t*)malloc(bytes);
    CK(cudaMemcpy(chk, d1, bytes, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (uint64_t i = 0; i < bytes; ++i) bad += chk[i] != 3;
    printf("{\"check\": \"tma d2d\", \"bad\": %llu}\n", (unsigned long long)bad);
  }
  return 0;
}
