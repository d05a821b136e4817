// tcgen05.mma issue/throughput microbenchmark: one CTA per SM, thread 0 issues R MMAs (M = 128, given N,
// kind tf32 (K = 8) or f16 (K = 16), K-major operands with SWIZZLE_NONE or SWIZZLE_128B), then waits on
// a commit.  Prints cycles per MMA and the implied dense TFLOP/s over all SMs.
// usage: umma_tput <kind: tf32|f16> <N> <swz: 0|128|1 (1: A operand from TMEM)> [R]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__global__ void k(uint32_t kind, uint32_t N, uint32_t swz, uint32_t R, long long* out, uint32_t cmt) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar, cbar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&cbar[1])));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t fmt = kind == 0 ? 2u : 1u;  // tf32 : bf16
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + 64 * 1024;
    uint64_t da, db;
    if (swz == 128) {
      da = sdesc(a0, 16, 1024, 2);
      db = sdesc(b0, 16, 1024, 2);
    } else {
      da = sdesc(a0, 128 * 16, 128, 0);
      db = sdesc(b0, N * 16, 128, 0);
    }
    long long t0 = clock64();
    if (swz == 1) {
      for (uint32_t r = 0; r < R; ++r) {
        const uint32_t ta = tmem + 256 + (r & 3) * 8;  // A: 128 lanes x K columns at TMEM column 256
        const uint64_t ob = (uint64_t)((r & 3) * 2 * 128);
        if (kind == 0)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
                       :: "r"(tmem), "r"(ta), "l"(db + ob), "r"(idesc), "r"(r));
        if (cmt && r % 3 == 2) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" :: "l"((uint64_t)__cvta_generic_to_shared(&cbar[0])));
          if (cmt > 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" :: "l"((uint64_t)__cvta_generic_to_shared(&cbar[1])));
        }
        else
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                       :: "r"(tmem), "r"(ta), "l"(db + ob), "r"(idesc), "r"(r));
      }
    } else
    for (uint32_t r = 0; r < R; ++r) {
      const uint64_t o = swz ? (uint64_t)((r & 3) * 2) : (uint64_t)((r & 3) * 2 * 128);  // K advance inside the tile
      if (kind == 0)
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                     :: "r"(tmem), "l"(da + o), "l"(db + o), "r"(idesc), "r"(r));
      else
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                     :: "r"(tmem), "l"(da + o), "l"(db + o), "r"(idesc), "r"(r));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" :: "l"((uint64_t)__cvta_generic_to_shared(&mbar)));
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb));
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

int main(int argc, char** argv) {
  const uint32_t kind = strcmp(argv[1], "tf32") == 0 ? 0 : 1;
  const uint32_t N = atoi(argv[2]), swz = atoi(argv[3]), R = argc > 4 ? atoi(argv[4]) : 4095;
  const uint32_t cmt = argc > 5 ? atoi(argv[5]) : 0;
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<nsm, 128, smem>>>(kind, N, swz, R, d, cmt);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double kk = kind == 0 ? 8 : 16;
    const double flops = 2.0 * 128 * N * kk * R * nsm;
    if (rep) printf("%s N=%u swz=%u cmt=%u: %s issue %.1f cyc/mma, total %.1f cyc/mma, %.0f TFLOP/s (event %.3f ms)\n", argv[1], N, swz, cmt,
           cudaGetErrorString(e), (double)h[0] / R, (double)h[1] / R, flops / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
