// k_mlp.cu — K7 (NEXT-1): the lightweight MLP m_theta of Eq. 1 on the
// 5th-generation tensor cores.  Layers 6-100-200-200-100-1,
// ReLU on hidden layers, identity output clamped at 0.
//
// Persistent CTAs of 1024 threads; a tile is 128 requests (one TMEM lane and
// kQ = 8 threads per request, taking every eighth 16-column group).  Layer 1
// (6 -> 100, 600 FMA/request) and layer 5 (100 -> 1) run on the CUDA cores in
// fp32.  Layers 2-4 are tcgen05.mma (kind::f16, BF16 operands, FP32
// accumulators in TMEM, M = 128):
//   A = the tile's activations in shared memory, B = the layer's weights,
//   resident in shared memory for the whole kernel (bf16, K-major, no swizzle:
//   8-row x 16-byte core matrices, [k/8][row][8]), issued by one thread and
//   committed to an mbarrier.  The epilogue of layer l (tcgen05.ld 32x32b ->
//   bias -> ReLU -> bf16 -> st.shared) writes the A operand of layer l+1.
// Software pipeline across a CTA's tiles: layer 4 accumulates in its own TMEM
// region, so as soon as it completes the next tile's layer 1 is written and its
// layer-2 MMA issued, running under this tile's layer-4 epilogue + layer 5.
// Padding: widths 100/200 -> 112/208 (N multiple of 16 at M = 128) with zero
// weight rows and zero biases, so padded activations are exactly 0; the last
// 8-wide K chunk of every weight matrix (all-zero columns) is not stored: the
// descriptor of the last k-step reads the next region (finite bf16) there and
// multiplies it by the zero activations.  This keeps the resident weights +
// one activation tile at 224.5 KB.
#include <cuda_bf16.h>

#include "internal.cuh"

namespace rtlm {
namespace {

constexpr uint32_t kT = 128;                       // requests per tile (TMEM lanes)
#ifndef KMLP_THREADS
#define KMLP_THREADS 1024
#endif
constexpr uint32_t kThr = KMLP_THREADS;            // threads: kQ per request (column groups)
constexpr uint32_t kQ = kThr / kT;
constexpr uint32_t N1 = 112, N2 = 208, N3 = 208, N4 = 112;
constexpr uint32_t K2C = 13, K3C = 25, K4C = 25;   // stored 8-wide K chunks of W2, W3, W4
constexpr uint32_t SZ_W2 = K2C * N2 * 16, SZ_W3 = K3C * N3 * 16, SZ_W4 = K4C * N4 * 16;
constexpr uint32_t OFF_W2 = 0, OFF_W3 = OFF_W2 + SZ_W2, OFF_W4 = OFF_W3 + SZ_W3;
constexpr uint32_t OFF_A = OFF_W4 + SZ_W4, SZ_A = 26 * kT * 16;
constexpr uint32_t OFF_P = OFF_A + SZ_A;
// fp32 parameters after the bf16 region: w1[100][6] b1[112] b2[208] b3[208] b4[112] w5[112] b5[4]
constexpr uint32_t P_W1 = 0, P_B1 = 600, P_B2 = P_B1 + 112, P_B3 = P_B2 + 208, P_B4 = P_B3 + 208,
                   P_W5 = P_B4 + 112, P_B5 = P_W5 + 112, P_N = P_B5 + 4;
constexpr uint32_t kSmem = OFF_P + P_N * 4;
static_assert(kSmem <= 232448 - 64, "K7 shared memory");

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // tcgen05 shared-memory matrix descriptor: K-major, SWIZZLE_NONE, version 1
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ constexpr uint32_t idesc_bf16(uint32_t m, uint32_t n) {
  // instruction descriptor: D f32, A/B bf16, both K-major, N >> 3, M >> 4
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_layer(uint32_t tmem, uint32_t a0, uint32_t b0, uint32_t n, uint32_t ksteps,
                                          uint32_t mbar) {
  const uint32_t idesc = idesc_bf16(kT, n);
  for (uint32_t s = 0; s < ksteps; ++s) {
    const uint64_t da = sdesc(a0 + s * 2 * kT * 16, kT * 16, 128);
    const uint64_t db = sdesc(b0 + s * 2 * n * 16, n * 16, 128);
    const uint32_t acc = s > 0;
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
  }
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)mbar));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
}

// 16 consecutive accumulator columns of this thread's row (no wait)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tmem_ld16_nowait(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// ReLU + round-to-nearest bf16 + pack in one instruction (max(x, 0) then RN
// equals RN then max for every finite x)
__device__ __forceinline__ uint32_t pack_bf16_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// hidden-layer epilogue: TMEM row -> + bias -> ReLU -> bf16 -> the next A operand;
// the kQ threads of a row take every kQ-th 16-column group
__device__ __forceinline__ void store_group(const uint32_t (&r)[16], const float* bias, uint32_t c0, uint8_t* sA,
                                            uint32_t row) {
  uint32_t p[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    p[j] = pack_bf16_relu(__uint_as_float(r[2 * j]) + bias[c0 + 2 * j], __uint_as_float(r[2 * j + 1]) + bias[c0 + 2 * j + 1]);
  *reinterpret_cast<uint4*>(sA + ((c0 / 8) * kT + row) * 16) = make_uint4(p[0], p[1], p[2], p[3]);
  *reinterpret_cast<uint4*>(sA + ((c0 / 8 + 1) * kT + row) * 16) = make_uint4(p[4], p[5], p[6], p[7]);
}

__device__ __forceinline__ void epilogue_hidden(uint32_t tmem_row, const float* bias, uint32_t n, uint8_t* sA,
                                                uint32_t row, uint32_t q) {
  constexpr uint32_t S = 16 * kQ;
  uint32_t c0 = q * 16;
  for (; c0 + S < n; c0 += 2 * S) {  // two groups per wait
    uint32_t r0[16], r1[16];
    tmem_ld16_nowait(tmem_row + c0, r0);
    tmem_ld16_nowait(tmem_row + c0 + S, r1);
    tmem_wait_ld();
    store_group(r0, bias, c0, sA, row);
    store_group(r1, bias, c0 + S, sA, row);
  }
  if (c0 < n) {
    uint32_t r0[16];
    tmem_ld16_nowait(tmem_row + c0, r0);
    tmem_wait_ld();
    store_group(r0, bias, c0, sA, row);
  }
}

__device__ __forceinline__ void sync_for_mma() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// layer 1 (6 -> 100, fp32 on the CUDA cores, ReLU) of one request: this
// thread's 8-column chunks c = q, q + kQ, .. (< N1 / 8) packed to bf16 in h
constexpr uint32_t kL1C = (N1 / 8 + kQ - 1) / kQ;  // chunks per thread
__device__ __forceinline__ void layer1(const float* P, uint4 f, uint32_t q, uint4 (&h)[kL1C]) {
  float x[6];
  x[0] = (float)(f.x & 0xFFFFu); x[1] = (float)(f.x >> 16);
  x[2] = (float)(f.y & 0xFFFFu); x[3] = (float)(f.y >> 16);
  x[4] = (float)(f.z & 0xFFFFu); x[5] = (float)(f.z >> 16);
#pragma unroll
  for (uint32_t k = 0; k < kL1C; ++k) {
    const uint32_t c = q + k * kQ;
    uint32_t p[4] = {0u, 0u, 0u, 0u};
    if (c < N1 / 8) {
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        float hh[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t j = c * 8 + qq * 2 + e;
          float acc = 0.0f;
          if (j < 100) {
            acc = P[P_B1 + j];
#pragma unroll
            for (int i = 0; i < 6; ++i) acc = fmaf(P[P_W1 + j * 6 + i], x[i], acc);
            acc = fmaxf(acc, 0.0f);
          }
          hh[e] = acc;
        }
        p[qq] = pack_bf16(hh[0], hh[1]);
      }
    }
    h[k] = make_uint4(p[0], p[1], p[2], p[3]);
  }
}
__device__ __forceinline__ void store_layer1(uint8_t* sA, uint32_t row, uint32_t q, const uint4 (&h)[kL1C]) {
#pragma unroll
  for (uint32_t k = 0; k < kL1C; ++k) {
    const uint32_t c = q + k * kQ;
    if (c < N1 / 8) *reinterpret_cast<uint4*>(sA + (c * kT + row) * 16) = h[k];
  }
}

// TMEM columns: region A (D2, then D3) 0..207, region B (D4) 256..367, the
// layer-5 partial sums of a row's kQ threads at 384..384+kQ-1
constexpr uint32_t TM_D4 = 256, TM_PART = 384;

__global__ void __launch_bounds__(kThr, 1) k_mlp(const uint16_t* __restrict__ feat, uint32_t n,
                                                const uint8_t* __restrict__ wblob, float* __restrict__ u_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const uint32_t row = tid & (kT - 1), q = tid >> 7;  // warps w, w + 4, .. share TMEM lanes 32(w & 3)..
  // resident weights: bf16 blob (W2 | W3 | W4) then the fp32 parameters
  {
    const uint4* src = reinterpret_cast<const uint4*>(wblob);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = tid; i < OFF_A / 16; i += kThr) dst[i] = src[i];
    const uint32_t* ps = reinterpret_cast<const uint32_t*>(wblob + OFF_A);
    uint32_t* pd = reinterpret_cast<uint32_t*>(smem + OFF_P);
    for (uint32_t i = tid; i < P_N; i += kThr) pd[i] = ps[i];
    for (uint32_t i = tid; i < SZ_A / 16; i += kThr) reinterpret_cast<uint4*>(smem + OFF_A)[i] = make_uint4(0, 0, 0, 0);
  }
  const float* P = reinterpret_cast<const float*>(smem + OFF_P);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  sync_for_mma();
  const uint32_t tmem = tbase;
  const uint32_t tmem_row = tmem + (((warp & 3u) * 32u) << 16);  // this warp's TMEM lane quarter
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  uint8_t* sA = smem + OFF_A;
  uint32_t phase = 0;
  const uint32_t ntiles = (n + kT - 1) / kT;
  auto load_feat = [&](uint32_t t) {
    const uint32_t rq = t * kT + row;
    return (t < ntiles && rq < n) ? __ldg(reinterpret_cast<const uint4*>(feat + (size_t)rq * 8)) : make_uint4(0, 0, 0, 0);
  };
  auto wait_mma = [&]() {
    mbar_wait(mb, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };
  // Software pipeline over this CTA's tiles t, t + G, ..: layer 1 of the next
  // tile runs on the CUDA cores while layer 4's MMA runs, and the next tile's
  // layer-2 MMA runs while this tile's layer-4 epilogue + layer 5 run.
  uint32_t t = blockIdx.x;
  uint4 h1[kL1C];
  if (t < ntiles) {
    layer1(P, load_feat(t), q, h1);
    store_layer1(sA, row, q, h1);
    sync_for_mma();
    if (tid == 0) mma_layer(tmem, s0 + OFF_A, s0 + OFF_W2, N2, 7, mb);
  }
  uint4 fnext = load_feat(t + gridDim.x);
  for (; t < ntiles; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    const uint32_t req = t * kT + row;
    // ---- layer 2 done: epilogue -> A operand of layer 3: [128 x 208] . [208 x 208]
    wait_mma();
    epilogue_hidden(tmem_row, P + P_B2, N2, sA, row, q);
    sync_for_mma();
    if (tid == 0) mma_layer(tmem, s0 + OFF_A, s0 + OFF_W3, N3, 13, mb);
    wait_mma();
    epilogue_hidden(tmem_row, P + P_B3, N3, sA, row, q);
    // ---- layer 4: [128 x 208] . [208 x 112] -> region B; next tile's layer 1 meanwhile
    sync_for_mma();
    if (tid == 0) mma_layer(tmem + TM_D4, s0 + OFF_A, s0 + OFF_W4, N4, 13, mb);
    const uint4 f = fnext;
    fnext = load_feat(tn + gridDim.x);
    wait_mma();
    if (tn < ntiles) layer1(P, f, q, h1);
    // ---- the activation region is free: next tile's layer 1 -> its layer-2 MMA
    if (tn < ntiles) {
      store_layer1(sA, row, q, h1);
      sync_for_mma();
      if (tid == 0) mma_layer(tmem, s0 + OFF_A, s0 + OFF_W2, N2, 7, mb);
    }
    // ---- layer 4 epilogue + layer 5 (100 -> 1) on the CUDA cores, clamp at 0
    float y = 0.0f;
    for (uint32_t c0 = q * 16; c0 < N4; c0 += 16 * kQ) {
      float v[16];
      tmem_ld16(tmem_row + TM_D4 + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) y = fmaf(P[P_W5 + c0 + j], fmaxf(v[j] + P[P_B4 + c0 + j], 0.0f), y);
    }
    // partial sums of the row's kQ threads meet in TMEM (same lane, column TM_PART + q)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem_row + TM_PART + q),
                 "r"(__float_as_uint(y)) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (q == 0) {
      uint32_t r[kQ];
      static_assert(kQ == 8, "partial-sum load is x8");
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem_row + TM_PART));
      tmem_wait_ld();
      // fixed summation order: bias + thread 0's groups + thread 1's groups + ...
      float acc = P[P_B5] + y;
#pragma unroll
      for (uint32_t k = 1; k < kQ; ++k) acc += __uint_as_float(r[k]);
      if (req < n) u_out[req] = fmaxf(acc, 0.0f);
    }
    // region C / region B are rewritten only after later barriers
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace

size_t mlp_blob_bytes() { return OFF_A + (size_t)P_N * 4; }

// host: pack row-major fp32 weights [out][in] into the kernel's blob
void mlp_pack(const float* const w[5], const float* const b[5], uint8_t* blob) {
  memset(blob, 0, mlp_blob_bytes());
  auto put = [&](uint32_t off, uint32_t nrows, uint32_t kchunks, const float* W, uint32_t out, uint32_t in) {
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(blob + off);
    for (uint32_t r = 0; r < out; ++r)
      for (uint32_t k = 0; k < in; ++k) {
        if (k / 8 >= kchunks) continue;  // all-zero padding chunks are not stored
        d[((k / 8) * nrows + r) * 8 + (k % 8)] = __float2bfloat16_rn(W[(size_t)r * in + k]);
      }
  };
  put(OFF_W2, N2, K2C, w[1], 200, 100);
  put(OFF_W3, N3, K3C, w[2], 200, 200);
  put(OFF_W4, N4, K4C, w[3], 100, 200);
  float* p = reinterpret_cast<float*>(blob + OFF_A);
  for (uint32_t i = 0; i < 600; ++i) p[P_W1 + i] = w[0][i];
  for (uint32_t i = 0; i < 100; ++i) p[P_B1 + i] = b[0][i];
  for (uint32_t i = 0; i < 200; ++i) p[P_B2 + i] = b[1][i];
  for (uint32_t i = 0; i < 200; ++i) p[P_B3 + i] = b[2][i];
  for (uint32_t i = 0; i < 100; ++i) p[P_B4 + i] = b[3][i];
  for (uint32_t i = 0; i < 100; ++i) p[P_W5 + i] = w[4][i];
  p[P_B5] = b[4][0];
}

cudaError_t launch_mlp(const uint16_t* feat, uint32_t n, const uint8_t* blob, float* u, int num_sms, cudaStream_t s) {
  if (!n) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  if (e != cudaSuccess) return e;
  const uint32_t ntiles = (n + kT - 1) / kT;
  const uint32_t grid = ntiles < (uint32_t)num_sms ? ntiles : (uint32_t)num_sms;
  k_mlp<<<grid, kThr, kSmem, s>>>(feat, n, blob, u);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
