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



__device__ __forceinline__ uint64_t selp64(uint32_t p, uint64_t a, uint64_t b) {  // p ? a : b
  uint64_t r;
  asm("{ .reg .pred q; setp.ne.u32 q, %3, 0; selp.b64 %0, %1, %2, q; }" : "=l"(r) : "l"(a), "l"(b), "r"(p));
  return r;
}
__device__ __forceinline__ uint64_t sel4(uint32_t i, uint64_t a0, uint64_t a1, uint64_t a2, uint64_t a3) {
  return selp64(i & 2u, selp64(i & 1u, a3, a2), selp64(i & 1u, a1, a0));
}
__device__ __forceinline__ uint64_t min64(uint64_t a, uint64_t b) { return selp64(a < b, a, b); }
__device__ __forceinline__ uint64_t max64(uint64_t a, uint64_t b) { return selp64(a < b, b, a); }
__device__ __forceinline__ uint32_t sel4u(uint32_t i, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
  const uint32_t lo = (i & 1u) ? a1 : a0, hi = (i & 1u) ? a3 : a2;
  return (i & 2u) ? hi : lo;
}
__global__ void kw(const uint32_t* __restrict__ p, uint32_t n, uint8_t* out, long long* cyc, uint32_t* fails) {
  extern __shared__ uint32_t buf32[];  // 4 + n, S4 mod 2^32
  __shared__ uint8_t so[8192];
  if (threadIdx.x == 0) {
    uint32_t r[4] = {0, 0, 0, 0};
    for (int c = 0; c < 4; ++c) buf32[c] = 0;
    for (uint32_t i = 0; i < n; ++i) { r[i & 3] += p[i] << 2; buf32[4 + i] = r[i & 3]; }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const uint32_t lane = threadIdx.x;
  uint32_t a0 = 0, a1 = 1, a2 = 2, a3 = 3;  // offsets from tb (rebased each round)
  uint64_t tb = 0;
  uint32_t rounds = 0;
  long long t0 = clock64();
  uint32_t j = 0, cnt = n;
  const uint32_t col = lane & 3u;
  while (j < cnt) {
    ++rounds;
    const uint32_t idx = j + lane;
    const bool valid = idx < cnt;
    const uint32_t base = sel4u(col, a0, a1, a2, a3);
    const uint32_t w = base + (buf32[4 + min(idx, cnt - 1)] - buf32[j + col]);
    const uint32_t wu = __shfl_up_sync(0xFFFFFFFFu, w, 1);
    const uint32_t wp = lane == 0 ? a3 : wu;
    const uint32_t fb = __ballot_sync(0xFFFFFFFFu, valid && !(w > wp));
    const uint32_t nv = min(32u, cnt - j);
    const uint32_t m = fb ? (uint32_t)__ffs(fb) : nv;
    if (lane < m) so[idx] = (uint8_t)(base & 3u);
    const int32_t i0 = fb ? (int32_t)m - 4 : (int32_t)m - 4;  // failure: u_{f-3..f-1}, w_f = u_{m-4..m-2}, w_{m-1}
    uint32_t u0, u1, u2, u3;
    if (i0 >= 0) {
      u0 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)i0);
      u1 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)i0 + 1);
      u2 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)i0 + 2);
      u3 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)i0 + 3);
    } else {
      const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)max(i0, 0));
      const uint32_t s1 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)max(i0 + 1, 0));
      const uint32_t s2 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)max(i0 + 2, 0));
      const uint32_t s3 = __shfl_sync(0xFFFFFFFFu, w, (uint32_t)max(i0 + 3, 0));
      u0 = i0 >= 0 ? s0 : sel4u((uint32_t)(i0 + 4), a0, a1, a2, a3);
      u1 = i0 + 1 >= 0 ? s1 : sel4u((uint32_t)(i0 + 5), a0, a1, a2, a3);
      u2 = i0 + 2 >= 0 ? s2 : sel4u((uint32_t)(i0 + 6), a0, a1, a2, a3);
      u3 = s3;
    }
    if (fb) {
      // u0..u2 = u_{f-3..f-1} (sorted), u3 = w_f: sorted insert
      const uint32_t x = u3;
      const uint32_t n0 = min(u0, x), n1 = min(max(u0, x), u1), n2 = min(max(u1, x), u2), n3 = max(u2, x);
      u0 = n0; u1 = n1; u2 = n2; u3 = n3;
    }
    const uint32_t m0 = u0 & ~3u;
    a0 = u0 - m0; a1 = u1 - m0; a2 = u2 - m0; a3 = u3 - m0;
    tb += m0 >> 2;
    j += m;
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *fails = rounds; }
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) out[i] = so[i];
}


__global__ void kruns(const uint32_t* __restrict__ p, uint32_t n, uint8_t* out, long long* cyc, uint32_t* fails) {
  extern __shared__ uint64_t xs[];  // n
  __shared__ uint16_t rs[8193];
  __shared__ uint32_t nr_s;
  __shared__ uint32_t dd[2048], dpat[2048];
  __shared__ uint8_t so[8192];
  if (threadIdx.x == 0) {
    uint32_t nr = 0;
    for (uint32_t i = 0; i < n; ++i) { xs[i] = p[i]; if (i == 0 || p[i] != p[i - 1]) rs[nr++] = (uint16_t)i; }
    rs[nr] = (uint16_t)n; nr_s = nr;
  }
  __syncthreads();
  if (threadIdx.x) return;
  uint64_t a0 = 0, a1 = 1, a2 = 2, a3 = 3;
  uint32_t trans = 0;
  long long t0 = clock64();
  const uint32_t nr = nr_s;
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t st = rs[k], en = rs[k + 1];
    const uint64_t X = xs[st] << 2;
    uint32_t j = st;
    while (j < en && !(a0 + X > a3)) {
      so[j] = (uint8_t)(a0 & 3u);
      const uint64_t w = a0 + X;
      const uint64_t n0 = min(a1, w), n1 = min(max(a1, w), a2), n2 = min(max(a2, w), a3), n3 = max(a3, w);
      a0 = n0; a1 = n1; a2 = n2; a3 = n3;
      ++j; ++trans;
    }
    const uint32_t r = en - j;
    const uint32_t pat = (uint32_t)(a0 & 3u) | ((uint32_t)(a1 & 3u) << 8) | ((uint32_t)(a2 & 3u) << 16) | ((uint32_t)(a3 & 3u) << 24);
    dd[k] = j | (r << 13); dpat[k] = pat;
    if (r) {
      auto rot = [&](uint32_t i) { const uint32_t c = (r + i) & 3u; return c == 0 ? a0 : c == 1 ? a1 : c == 2 ? a2 : a3; };
      const uint64_t n0 = rot(0) + X * (uint64_t)((r + 0) >> 2);
      const uint64_t n1 = rot(1) + X * (uint64_t)((r + 1) >> 2);
      const uint64_t n2 = rot(2) + X * (uint64_t)((r + 2) >> 2);
      const uint64_t n3 = rot(3) + X * (uint64_t)((r + 3) >> 2);
      a0 = n0; a1 = n1; a2 = n2; a3 = n3;
    }
  }
  long long t1 = clock64();
  *cyc = t1 - t0; *fails = trans * 65536u + nr;
  for (uint32_t k = 0; k < nr; ++k) { const uint32_t j = dd[k] & 0x1FFF, r = dd[k] >> 13; for (uint32_t t = 0; t < r; ++t) so[j + t] = (uint8_t)(dpat[k] >> (8 * (t & 3u))); }
  for (uint32_t i = 0; i < n; ++i) out[i] = so[i];
}


__global__ void kruns2(const uint32_t* __restrict__ p, uint32_t n, uint8_t* out, long long* cyc, uint32_t* fails) {
  __shared__ uint32_t rx[2048], rsl[2049], dd[2048], dpat[2048];
  __shared__ uint32_t nr_s;
  __shared__ uint8_t so[8192];
  if (threadIdx.x == 0) {
    uint32_t nr = 0;
    for (uint32_t i = 0; i < n; ++i) if (i == 0 || p[i] != p[i - 1]) { rx[nr] = p[i] << 2; rsl[nr++] = i; }
    rsl[nr] = n; nr_s = nr;
  }
  __syncthreads();
  if (threadIdx.x) return;
  uint64_t base = 0;
  uint32_t d1 = 1, d2 = 2, d3 = 3;
  uint32_t trans = 0;
  long long t0 = clock64();
  const uint32_t nr = nr_s;
  uint32_t X = rx[0], st = rsl[0], en = rsl[1];
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t Xn = rx[k + 1], enn = rsl[k + 2];  // prefetch (padding past nr is harmless)
    uint32_t j = st;
    while (j < en && !(X > d3)) {
      so[j] = (uint8_t)(base & 3u);
      const uint32_t e0 = min(d1, X), e1 = min(max(d1, X), d2), e2 = min(max(d2, X), d3), e3 = max(d3, X);
      base += e0;
      d1 = e1 - e0; d2 = e2 - e0; d3 = e3 - e0;
      ++j; ++trans;
    }
    const uint32_t r = en - j;
    dd[k] = j | (r << 13);
    dpat[k] = __byte_perm(__byte_perm((uint32_t)base, d1, 0x0040), __byte_perm(d2, d3, 0x0040), 0x5410);
    const uint32_t kk = r & 3u, q = r >> 2;
    // rotation by kk: dk = d_kk, new d_i = d_{kk+i} - dk (wrapping: + X)
    const uint32_t dk = (kk & 2u) ? ((kk & 1u) ? d3 : d2) : ((kk & 1u) ? d1 : 0u);
    const uint32_t c1 = (kk & 2u) ? ((kk & 1u) ? X : d3) : ((kk & 1u) ? d2 : d1);
    const uint32_t c2 = (kk & 2u) ? ((kk & 1u) ? X + d1 : X) : ((kk & 1u) ? d3 : d2);
    const uint32_t c3 = (kk & 2u) ? ((kk & 1u) ? X + d2 : X + d1) : ((kk & 1u) ? X : d3);
    base += (uint64_t)dk + (uint64_t)X * q;
    d1 = c1 - dk; d2 = c2 - dk; d3 = c3 - dk;
    X = Xn; st = en; en = enn;
  }
  long long t1 = clock64();
  *cyc = t1 - t0; *fails = trans * 65536u + nr;
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t j = dd[k] & 0x1FFF, r = dd[k] >> 13, pt = dpat[k];
    const uint32_t b = pt & 0xFF;
    for (uint32_t t = 0; t < r; ++t) { const uint32_t di = (t & 3u) ? ((pt >> (8 * (t & 3u))) & 0xFF) : 0u; so[j + t] = (uint8_t)((b + di) & 3u); }
  }
  for (uint32_t i = 0; i < n; ++i) out[i] = so[i];
}

int main() {
  const uint32_t n = 8192;
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
  cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (4 + n) * 4);
  cudaFuncSetAttribute(kruns, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 8);
  for (int v = 0; v < 7; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      if (v == 0) k<0><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 1) k<1><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 2) k<2><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 3) k<3><<<1, 128, smem>>>(dp, n, dout, dc, df);
      if (v == 4) kw<<<1, 64, (4 + n) * 4>>>(dp, n, dout, dc, df);
      if (v == 5) kruns<<<1, 32, n * 8>>>(dp, n, dout, dc, df);
      if (v == 6) kruns2<<<1, 32>>>(dp, n, dout, dc, df);
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
