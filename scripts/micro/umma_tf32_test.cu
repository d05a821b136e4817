// Standalone check of hand-built tcgen05 kind::tf32 descriptors (K-major, no swizzle):
// D[128 x N] = A[128 x K] . B[N x K]^T with fp32 containers (tf32 values), f32 accumulate.
// Core matrix = 8 rows x 16 bytes = 8 rows x 4 elements; layout [k/4][row][4];
// one MMA covers K = 8 (two core-matrix columns): LBO = rows * 16 B, SBO = 128 B.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 208, K = 104;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__global__ void k(const float* A, const float* B, float* D, uint32_t afmt) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* sA = reinterpret_cast<float*>(sm);                 // [K/4][M][4]
  float* sB = reinterpret_cast<float*>(sm + M * K * 4);     // [K/4][N][4]
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) { int r = i / K, c = i % K; sA[(c / 4) * M * 4 + r * 4 + (c % 4)] = A[i]; }
  for (int i = tid; i < N * K; i += blockDim.x) { int r = i / K, c = i % K; sB[(c / 4) * N * 4 + r * 4 + (c % 4)] = B[i]; }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar)));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  // D f32 (bit 4), A / B format (bits 7-9 / 10-12), K-major both, N >> 3 at 17, M >> 4 at 24
  const uint32_t idesc = (1u << 4) | (afmt << 7) | (afmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t da = sdesc(a0 + s * 2 * M * 16, M * 16, 128);
      const uint64_t db = sdesc(b0 + s * 2 * N * 16, N * 16, 128);
      const uint32_t acc = s > 0;
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" :: "l"((uint64_t)__cvta_generic_to_shared(&mbar)));
  }
  {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tmem));
}

static float tf32_rn(float x) {  // round to nearest even at 10 explicit mantissa bits
  uint32_t b; memcpy(&b, &x, 4);
  b = (b + 0xFFFu + ((b >> 13) & 1u)) & ~0x1FFFu;
  float r; memcpy(&r, &b, 4); return r;
}

int main(int argc, char** argv) {
  const uint32_t afmt = argc > 1 ? atoi(argv[1]) : 2;
  std::vector<float> fA(M * K), fB(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) fA[i] = tf32_rn((rand() % 2001 - 1000) / 377.0f);
  for (int i = 0; i < N * K; ++i) fB[i] = tf32_rn((rand() % 2001 - 1000) / 611.0f);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, M * K * 4); cudaMalloc(&dB, N * K * 4); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, fA.data(), M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, fB.data(), N * K * 4, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(dA, dB, dD, afmt);
  cudaError_t e = cudaDeviceSynchronize();
  printf("afmt %u kernel: %s\n", afmt, cudaGetErrorString(e));
  std::vector<float> hD(M * N);
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0; int bad = 0;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0, sa = 0;
      for (int kk = 0; kk < K; ++kk) { s += (double)fA[r * K + kk] * fB[c * K + kk]; sa += fabs((double)fA[r * K + kk] * fB[c * K + kk]); }
      double err = fabs(s - hD[r * N + c]) / sa;
      if (err > maxrel) maxrel = err;
      if (err > 1e-5 && bad++ < 5) printf("mismatch r%d c%d got %f want %f\n", r, c, hD[r * N + c], s);
    }
  printf("max err / |A||B| %g, bad %d\n", maxrel, bad);
  return 0;
}
