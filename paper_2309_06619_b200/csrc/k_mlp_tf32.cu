// k_mlp_tf32.cu — K7 (NEXT-1), RT_MLP_TF32X3 mode: the lightweight MLP
// m_theta of Eq. 1 (layers 6-100-200-200-100-1, P:620 / P:1547; ReLU on the
// hidden layers, output clamped at 0) on the tensor cores with
// fp32 accuracy from three TF32 products per multiply ("3xTF32"): every fp32
// operand x is split into hi = tf32(x) (round to nearest, 11 significant bits)
// and lo = x - hi (exact in fp32, |lo| <= 2^-11 |x|, read by the MMA to its
// leading 11 bits), and a.b is taken as hi_a.hi_b + hi_a.lo_b + lo_a.hi_b,
// accumulated in fp32 in TMEM by tcgen05.mma kind::tf32.  The residuals (lo
// truncation, the dropped lo_a.lo_b) stay below ~2^-21 |a||b| per product, a
// few fp32 unit roundoffs; the accumulation is fp32 as in the paper's model
// (an fp32 PyTorch MLP).
//
// Tile = 128 requests (TMEM lanes), persistent CTAs of 512 threads (4 per
// row; warps w, w + 4, .. read TMEM lane quarter w & 3).
// * Layers 1-4 on the tensor cores (M = 128, N = 112 / 208 / 208 / 112,
//   K = 8 / 104 / 208 / 208, K-major, no swizzle: 8-row x 16-byte core
//   matrices of 4 tf32 values, [k/4][row][4], LBO = rows * 16 B, SBO = 128 B;
//   one MMA covers K = 8).  Biases ride in the MMA: A carries a constant-1
//   column (index 6 / 100 / 200 / 200) and B the bias at that k.  The features
//   (integers < 2^16) split exactly into hi + lo.
// * The A operand (activations hi + lo) is staged in shared memory one K-half
//   of 104 columns at a time (2 x 53 KB): the epilogue of layer l writes
//   columns 0..103 of relu(D_l) split into hi / lo, the MMAs of layer l+1
//   consume them, then the epilogue writes columns 104..207 into the same
//   buffer.  D_l and D_{l+1} live in two TMEM regions (columns 0..207 and
//   256..463).
// * Layer 5 (100 -> 1) in fp32 FMA chains on the CUDA cores, straight from
//   TMEM: 4 partial sums per row, added in a fixed order.
// * Weights (hi and lo, split on the host) stream from L2 by cp.async.bulk, one
//   8-deep-K chunk (hi | lo, 64 N bytes) per k-step, through a ring of kStages
//   stages with full (complete_tx) and empty (tcgen05.commit) mbarriers; a
//   17th warp produces the chunks, thread 0 issues the MMAs.
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr uint32_t kT = 128;          // rows per tile (TMEM lanes)
constexpr uint32_t kThr = 512;        // 4 threads per row
constexpr uint32_t kQ = kThr / kT;    // column groups per row
constexpr uint32_t kHalf = 104;       // A columns staged at a time
#ifndef KTF_STAGES
#define KTF_STAGES 6
#endif
constexpr uint32_t kStages = KTF_STAGES;  // weight-chunk ring
constexpr uint32_t N1 = 112, N2 = 208, N3 = 208, N4 = 112;
constexpr uint32_t S1 = 1, S2 = 13, S3 = 26, S4 = 26;  // k-steps (K = 8, 104, 208, 208)
constexpr uint32_t kSteps = S1 + S2 + S3 + S4;          // per tile
constexpr uint32_t kChunkMax = 64 * 208;               // bytes of one k-step chunk (hi + lo) at N = 208

// weight blob (bytes): L1 | L2 | L3 | L4 chunks | w5[100] b5 (fp32)
constexpr uint32_t OFF_L1 = 0, OFF_L2 = OFF_L1 + S1 * 64 * N1, OFF_L3 = OFF_L2 + S2 * 64 * N2,
                   OFF_L4 = OFF_L3 + S3 * 64 * N3, OFF_PAR = OFF_L4 + S4 * 64 * N4;
constexpr uint32_t P_W5 = 0, P_B5 = 100, P_N = 104;

// shared memory (bytes)
constexpr uint32_t SM_AHI = 0, SM_ALO = SM_AHI + kHalf * kT * 4, SM_W = SM_ALO + kHalf * kT * 4,
                   SM_PAR = SM_W + kStages * kChunkMax, SM_RED = SM_PAR + P_N * 4, SM_N = SM_RED + kT * kQ * 4;
static_assert(SM_N <= 232448 - 1024, "K7 tf32 shared memory");

constexpr uint32_t TM_X = 0, TM_Y = 256;  // TMEM regions (columns)

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ constexpr uint32_t idesc_tf32(uint32_t m, uint32_t n) {
  // D f32, A / B tf32 (format 2), both K-major, N >> 3, M >> 4
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
               ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)mbar));
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
// 16 consecutive TMEM columns of this thread's lane (no wait: call tmem_wait before using r)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// store 4 consecutive A columns (core-matrix column cc) of this row as hi / lo
__device__ __forceinline__ void store_hl(uint8_t* smem, uint32_t cc, uint32_t row, float a, float b, float c, float d) {
  const float ha = tf32_hi(a), hb = tf32_hi(b), hc = tf32_hi(c), hd = tf32_hi(d);
  const uint32_t off = (cc * kT + row) * 16u;
  *reinterpret_cast<float4*>(smem + SM_AHI + off) = make_float4(ha, hb, hc, hd);
  *reinterpret_cast<float4*>(smem + SM_ALO + off) = make_float4(a - ha, b - hb, c - hc, d - hd);
}

// 16 A columns from D columns [c0, c0 + 16): relu for c < one, 1 at c == one (bias column), 0 beyond
__device__ __forceinline__ void put16(uint8_t* smem, const uint32_t (&r)[16], uint32_t c0, uint32_t a0, uint32_t ncol,
                                      uint32_t one, uint32_t row) {
  float x[16];
  if (c0 + 16 <= one) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fmaxf(__uint_as_float(r[j]), 0.0f);
  } else {
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j)
      x[j] = c0 + j < one ? fmaxf(__uint_as_float(r[j]), 0.0f) : (c0 + j == one ? 1.0f : 0.0f);
  }
#pragma unroll
  for (uint32_t j = 0; j < 16; j += 4)
    if (j < ncol) store_hl(smem, (a0 + j) / 4, row, x[j], x[j + 1], x[j + 2], x[j + 3]);
}

// epilogue of a hidden layer into A columns [h*104, h*104 + 104) of the next layer; the 4 threads of a row
// take 16-column groups q and q + 4 (both TMEM loads in flight before one wait)
__device__ __forceinline__ void epilogue_half(uint8_t* smem, uint32_t tmem_row, uint32_t one, uint32_t h, uint32_t row,
                                              uint32_t q) {
  uint32_t r0[16], r1[16];
  const uint32_t g1 = q + kQ;
  const bool two = g1 * 16 < kHalf;  // q <= 2 (warp-uniform)
  tmem_ld16(tmem_row + h * kHalf + q * 16, r0);
  if (two) tmem_ld16(tmem_row + h * kHalf + g1 * 16, r1);
  tmem_wait();
  put16(smem, r0, h * kHalf + q * 16, q * 16, 16, one, row);
  if (two) put16(smem, r1, h * kHalf + g1 * 16, g1 * 16, min(16u, kHalf - g1 * 16), one, row);
}

// per-tile k-step -> (chunk address, bytes)
__device__ __forceinline__ void chunk_of(const uint8_t* blob, uint32_t gs, const uint8_t*& src, uint32_t& bytes) {
  const uint32_t s = gs % kSteps;
  if (s < S1) { src = blob + OFF_L1; bytes = 64 * N1; }
  else if (s < S1 + S2) { src = blob + OFF_L2 + (s - S1) * 64 * N2; bytes = 64 * N2; }
  else if (s < S1 + S2 + S3) { src = blob + OFF_L3 + (s - S1 - S2) * 64 * N3; bytes = 64 * N3; }
  else { src = blob + OFF_L4 + (s - S1 - S2 - S3) * 64 * N4; bytes = 64 * N4; }
}

struct Ring {
  uint32_t full0, empty0;  // mbarrier addresses of stage 0 (8 bytes apart)
  uint32_t w0;             // smem address of stage 0
  uint32_t used = 0;       // k-steps consumed by MMAs (issuing thread)
};

// issuing thread: the 3xTF32 MMAs of `steps` k-steps of one layer (part) into tmem_d, then commit to done_bar
__device__ __forceinline__ void mma_steps(Ring& p, uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d, uint32_t n,
                                          uint32_t steps, bool first, uint32_t done_bar) {
  const uint32_t idesc = idesc_tf32(kT, n);
  for (uint32_t s = 0; s < steps; ++s) {
    const uint32_t st = p.used % kStages, use = p.used / kStages;
    mbar_wait(p.full0 + 8 * st, use & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t bh = p.w0 + st * kChunkMax, bl = bh + 32 * n;
    const uint64_t dah = sdesc(a_hi + s * 2 * kT * 16, kT * 16, 128), dal = sdesc(a_lo + s * 2 * kT * 16, kT * 16, 128);
    const uint64_t dbh = sdesc(bh, n * 16, 128), dbl = sdesc(bl, n * 16, 128);
    mma_tf32(tmem_d, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
    mma_tf32(tmem_d, dah, dbl, idesc, 1u);
    mma_tf32(tmem_d, dal, dbh, idesc, 1u);
    commit(p.empty0 + 8 * st);
    ++p.used;
  }
  commit(done_bar);
}

// barrier 1: the 512 compute threads (the producer warp never joins)
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThr) : "memory"); }
__device__ __forceinline__ void sync_compute_for_mma() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
  bar_compute();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// warps 0..15: TMEM epilogues and layer 5 (thread 0 also issues the MMAs); warp 16: weight-chunk producer
__global__ void __launch_bounds__(kThr + 32, 1) k_mlp_tf32(const uint16_t* __restrict__ feat, uint32_t n,
                                                          const uint8_t* __restrict__ blob, float* __restrict__ u_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[2 * kStages + 1];
  __shared__ uint32_t tbase;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const uint32_t row = tid & (kT - 1), q = tid >> 7;
  const float* gpar = reinterpret_cast<const float*>(blob + OFF_PAR);
  float* P = reinterpret_cast<float*>(smem + SM_PAR);
  for (uint32_t i = tid; i < P_N; i += kThr) P[i] = gpar[i];
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars);
  Ring ring;
  ring.full0 = b0;
  ring.empty0 = b0 + 8 * kStages;
  const uint32_t done_bar = b0 + 16 * kStages;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  ring.w0 = s0 + SM_W;
  if (tid == 0) {
    for (uint32_t i = 0; i < 2 * kStages + 1; ++i) mbar_init(b0 + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ntiles = (n + kT - 1) / kT;
  if (warp == kThr / 32) {
    // producer: every k-step chunk of this CTA's tiles, in consumption order, kStages ahead
    if ((tid & 31u) == 0) {
      const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      for (uint32_t i = 0; i < my_tiles * kSteps; ++i) {
        const uint32_t st = i % kStages, use = i / kStages;
        if (use > 0) mbar_wait(ring.empty0 + 8 * st, (use - 1) & 1u);
        const uint8_t* src;
        uint32_t bytes;
        chunk_of(blob, i, src, bytes);
        bulk_load(ring.w0 + st * kChunkMax, src, bytes, ring.full0 + 8 * st);
      }
    }
    return;
  }
  const uint32_t tmem = tbase;
  const uint32_t tmem_row = tmem + (((warp & 3u) * 32u) << 16);
  const uint32_t a_hi = s0 + SM_AHI, a_lo = s0 + SM_ALO;
  uint32_t dphase = 0;
  // one thread polls the MMA-done barrier, the others sleep in the named barrier
  auto wait_done = [&]() {
    if (tid == 0) mbar_wait(done_bar, dphase);
    dphase ^= 1u;
    bar_compute();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };
  float* red = reinterpret_cast<float*>(smem + SM_RED);
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint32_t rq = t * kT + row;
    // ---- layer 1 input: A columns 0..7 = (S, Y, M, V, O, P, 1, 0); integers < 2^16 split exactly
    if (q == 0) {
      uint4 f = make_uint4(0, 0, 0, 0);
      if (rq < n) f = __ldg(reinterpret_cast<const uint4*>(feat + (size_t)rq * 8));
      store_hl(smem, 0, row, (float)(f.x & 0xFFFFu), (float)(f.x >> 16), (float)(f.y & 0xFFFFu), (float)(f.y >> 16));
      store_hl(smem, 1, row, (float)(f.z & 0xFFFFu), (float)(f.z >> 16), 1.0f, 0.0f);
    }
    sync_compute_for_mma();
    // ---- layer 1: D1 (region Y) = [x 1] . [W1 b1]^T
    if (tid == 0) mma_steps(ring, a_hi, a_lo, tmem + TM_Y, N1, S1, true, done_bar);
    wait_done();
    epilogue_half(smem, tmem_row + TM_Y, 100, 0, row, q);
    sync_compute_for_mma();
    // ---- layer 2: D2 (region X) = [relu(D1) 1] . [W2 b2]^T
    if (tid == 0) mma_steps(ring, a_hi, a_lo, tmem + TM_X, N2, S2, true, done_bar);
    wait_done();
    // ---- layer 3: D3 (region Y), two K-halves
    for (uint32_t h = 0; h < 2; ++h) {
      epilogue_half(smem, tmem_row + TM_X, 200, h, row, q);
      sync_compute_for_mma();
      if (tid == 0) mma_steps(ring, a_hi, a_lo, tmem + TM_Y, N3, S3 / 2, h == 0, done_bar);
      wait_done();
    }
    // ---- layer 4: D4 (region X), two K-halves
    for (uint32_t h = 0; h < 2; ++h) {
      epilogue_half(smem, tmem_row + TM_Y, 200, h, row, q);
      sync_compute_for_mma();
      if (tid == 0) mma_steps(ring, a_hi, a_lo, tmem + TM_X, N4, S4 / 2, h == 0, done_bar);
      wait_done();
    }
    // ---- layer 5 (100 -> 1): w5 . relu(D4) + b5, fp32 FMA chains over columns 25q .. 25q + 24
    float y = 0.0f;
    {
      uint32_t r0[16], r1[16];
      const uint32_t c0 = q * 25 & ~7u;  // 0, 24, 48, 72: 32 loaded columns cover [25q, 25q + 25)
      tmem_ld16(tmem_row + TM_X + c0, r0);
      tmem_ld16(tmem_row + TM_X + c0 + 16, r1);
      tmem_wait();
#pragma unroll
      for (uint32_t j = 0; j < 32; ++j) {
        const uint32_t col = c0 + j;
        const float v = __uint_as_float(j < 16 ? r0[j] : r1[j - 16]);
        if (col >= q * 25 && col < q * 25 + 25) y = __fmaf_rn(P[P_W5 + col], fmaxf(v, 0.0f), y);
      }
    }
    red[q * kT + row] = y;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    bar_compute();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (q == 0 && rq < n) {
      float acc = P[P_B5];
#pragma unroll
      for (uint32_t k = 0; k < kQ; ++k) acc += red[k * kT + row];
      u_out[rq] = fmaxf(acc, 0.0f);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  bar_compute();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// host split: tf32 round-to-nearest-even of x (finite), lo = x - hi
float host_tf32(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  b = (b + 0xFFFu + ((b >> 13) & 1u)) & ~0x1FFFu;
  float r;
  memcpy(&r, &b, 4);
  return r;
}

}  // namespace

size_t mlp_tf32_blob_bytes() { return OFF_PAR + (size_t)P_N * 4; }

// host: [W_l b_l] (the bias as the weight of a constant-1 input at k = in) split into hi / lo tf32 chunks per
// k-step, each [k/4][n][4]
void mlp_tf32_pack(const float* const w[5], const float* const b[5], uint8_t* blob) {
  memset(blob, 0, mlp_tf32_blob_bytes());
  auto put = [&](uint32_t off, uint32_t steps, uint32_t N, const float* W, const float* bias, uint32_t out,
                 uint32_t in) {
    for (uint32_t s = 0; s < steps; ++s) {
      float* hi = reinterpret_cast<float*>(blob + off + (size_t)s * 64 * N);
      float* lo = hi + 8 * N;
      for (uint32_t r = 0; r < out; ++r)
        for (uint32_t kk = 0; kk < 8; ++kk) {
          const uint32_t k = s * 8 + kk;
          const float x = k < in ? W[(size_t)r * in + k] : (k == in ? bias[r] : 0.0f);
          const float h = host_tf32(x);
          const size_t idx = ((size_t)(kk / 4) * N + r) * 4 + (kk % 4);
          hi[idx] = h;
          lo[idx] = x - h;
        }
    }
  };
  put(OFF_L1, S1, N1, w[0], b[0], 100, 6);
  put(OFF_L2, S2, N2, w[1], b[1], 200, 100);
  put(OFF_L3, S3, N3, w[2], b[2], 200, 200);
  put(OFF_L4, S4, N4, w[3], b[3], 100, 200);
  float* p = reinterpret_cast<float*>(blob + OFF_PAR);
  for (uint32_t i = 0; i < 100; ++i) p[P_W5 + i] = w[4][i];
  p[P_B5] = b[4][0];
}

cudaError_t launch_mlp_tf32(const uint16_t* feat, uint32_t n, const uint8_t* blob, float* u, int num_sms,
                            cudaStream_t s) {
  if (!n) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_mlp_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_N);
  if (e != cudaSuccess) return e;
  const uint32_t ntiles = (n + kT - 1) / kT;
  const uint32_t grid = ntiles < (uint32_t)num_sms ? ntiles : (uint32_t)num_sms;
  k_mlp_tf32<<<grid, kThr + 32, SM_N, s>>>(feat, n, blob, u);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
