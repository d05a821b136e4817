// Micro-benchmark: one-thread list-scheduling chain variants (cycles per job).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ void ins(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3, uint32_t x) {
  const uint32_t w = a0 + (x << 2);
  const uint32_t n0 = min(a1, w), n1 = min(max(a1, w), a2), n2 = min(max(a2, w), a3), n3 = max(a3, w);
  a0 = n0; a1 = n1; a2 = n2; a3 = n3;
}

template <int V>
__global__ void k(const uint32_t* __restrict__ p, uint32_t n, uint8_t* out, long long* cyc, uint32_t* fails) {
  extern __shared__ uint32_t sp[];
  uint8_t* so = reinterpret_cast<uint8_t*>(sp + n);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sp[i] = p[i];
  __syncthreads();
  if (threadIdx.x) return;
  uint32_t a0 = 0, a1 = 1, a2 = 2, a3 = 3, nf = 0;
  long long t0 = clock64();
  for (uint32_t q = 0; q < n; q += 8) {
    uint32_t v[8], c[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = sp[q + t];
    if (V == 0) {
#pragma unroll
      for (int t = 0; t < 8; ++t) { c[t] = a0; ins(a0, a1, a2, a3, v[t]); }
    } else if (V == 1) {
#pragma unroll
      for (int b = 0; b < 8; b += 4) {
        const uint32_t w1 = a0 + (v[b] << 2), w2 = a1 + (v[b + 1] << 2), w3 = a2 + (v[b + 2] << 2), w4 = a3 + (v[b + 3] << 2);
        if ((w1 > a3) & (w2 > w1) & (w3 > w2) & (w4 > w3)) {
          c[b] = a0; c[b + 1] = a1; c[b + 2] = a2; c[b + 3] = a3;
          a0 = w1; a1 = w2; a2 = w3; a3 = w4;
        } else {
          ++nf;
#pragma unroll
          for (int t = 0; t < 4; ++t) { c[b + t] = a0; ins(a0, a1, a2, a3, v[b + t]); }
        }
      }
    } else if (V == 2) {
      // branch-free select between the rotation and the generic result per block of 4
#pragma unroll
      for (int b = 0; b < 8; b += 4) {
        const uint32_t w1 = a0 + (v[b] << 2), w2 = a1 + (v[b + 1] << 2), w3 = a2 + (v[b + 2] << 2), w4 = a3 + (v[b + 3] << 2);
        const bool ok = (w1 > a3) & (w2 > w1) & (w3 > w2) & (w4 > w3);
        if (__builtin_expect(ok, 1)) {
          c[b] = a0; c[b + 1] = a1; c[b + 2] = a2; c[b + 3] = a3;
          a0 = w1; a1 = w2; a2 = w3; a3 = w4;
          continue;
        }
        ++nf;
#pragma unroll
        for (int t = 0; t < 4; ++t) { c[b + t] = a0; ins(a0, a1, a2, a3, v[b + t]); }
      }
    } else {
      // block of 8 appends
      uint32_t w[8];
      w[0] = a0 + (v[0] << 2); w[1] = a1 + (v[1] << 2); w[2] = a2 + (v[2] << 2); w[3] = a3 + (v[3] << 2);
      w[4] = w[0] + (v[4] << 2); w[5] = w[1] + (v[5] << 2); w[6] = w[2] + (v[6] << 2); w[7] = w[3] + (v[7] << 2);
      bool ok = w[0] > a3;
#pragma unroll
      for (int t = 1; t < 8; ++t) ok &= w[t] > w[t - 1];
      if (ok) {
        c[0] = a0; c[1] = a1; c[2] = a2; c[3] = a3; c[4] = w[0]; c[5] = w[1]; c[6] = w[2]; c[7] = w[3];
        a0 = w[4]; a1 = w[5]; a2 = w[6]; a3 = w[7];
      } else {
        ++nf;
#pragma unroll
        for (int t = 0; t < 8; ++t) { c[t] = a0; ins(a0, a1, a2, a3, v[t]); }
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) so[q + t] = (uint8_t)(c[t] & 3u);
    const uint32_t m = a0 & ~3u;
    a0 -= m; a1 -= m; a2 -= m; a3 -= m;
  }
  long long t1 = clock64();
  *cyc = t1 - t0;
  *fails = nf;
  for (uint32_t i = 0; i < n; ++i) out[i] = so[i];
}

int main() {
  const uint32_t n = 40960;
  std::vector<uint32_t> h(n);
  FILE* fp = fopen("scripts/micro/preds.bin", "rb");
  if (!fp || fread(h.data(), 4, n, fp) != n) { printf("no preds\n"); return 1; }
  fclose(fp);
  const int smem = n * 5;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t* dp; uint8_t* dout; long long* dc; uint32_t* df;
  cudaMalloc(&dp, n * 4); cudaMalloc(&dout, n); cudaMalloc(&dc, 8); cudaMalloc(&df, 4);
  cudaMemcpy(dp, h.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<uint8_t> ref(n), o(n);
  for (int v = 0; v < 4; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      if (v == 0) k<0><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 1) k<1><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 2) k<2><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 3) k<3><<<1, 128, smem>>>(dp, n, dout, dc, df);
    }
    long long c; uint32_t f;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&f, df, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dout, n, cudaMemcpyDeviceToHost);
    if (v == 0) ref = o;
    printf("variant %d: %.2f cycles/job, fails %u, match %d\n", v, (double)c / n, f, (int)(o == ref));
  }
  return 0;
}
