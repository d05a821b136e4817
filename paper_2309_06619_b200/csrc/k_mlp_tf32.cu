// k_mlp_tf32.cu — K7 (NEXT-1), RT_MLP_TF32X3 mode: the lightweight MLP
// m_theta of Eq. 1 (layers 6-100-200-200-100-1, P:620 / P:1547; ReLU on the
// hidden layers, output clamped at 0) on the tensor cores with
// fp32 accuracy from three TF32 products per multiply ("3xTF32"): every fp32
// operand x is split into hi = tf32(x) (round to nearest, 11 significant bits)
// and lo = tf32(x - hi) (|lo| <= 2^-11 |x|, |x - hi - lo| <= 2^-22 |x|), and
// a.b is taken as hi_a.hi_b + hi_a.lo_b + lo_a.hi_b, accumulated in fp32 in
// TMEM by tcgen05.mma kind::tf32.  The residuals (the split, the dropped
// lo_a.lo_b) stay below ~3 x 2^-22 |a||b| per product, a few fp32 unit
// roundoffs; the accumulation is fp32 as in the paper's model
// (an fp32 PyTorch MLP).
//
// Tile = 128 requests (TMEM lanes); persistent CTAs of 18 warps:
// * warps 0..15 (4 per row; warps w, w + 4, .. read TMEM lane quarter w & 3):
//   stage the features, run the epilogues relu(D_l) -> hi / lo A operand of
//   layer l+1, and layer 5 (100 -> 1) in fp32 FMA chains straight from TMEM;
// * warp 16, lane 0: streams the weights (hi | lo, split on the host) from L2
//   by cp.async.bulk, the 8-deep-K chunks (64 N bytes each) of one A group's
//   two k-steps per stage, through a ring of kStages stages (full:
//   complete_tx, empty: tcgen05.commit);
// * warp 17: issues the MMAs (all lanes run the loop, one elected lane
//   issues, so descriptors stay in uniform registers).
// Layers 1-4 run on the tensor cores (M = 128, N = 112 / 208 / 208 / 112,
// K = 8 / 104 / 208 / 208; K-major, no swizzle: 8-row x 16-byte core matrices
// of 4 tf32 values, [k/4][row][4], LBO = rows * 16 B, SBO = 128 B; one MMA
// covers K = 8).  Biases ride in the MMA: A carries a constant-1 column (index
// 6 / 100 / 200 / 200) and B the bias at that k.  The features (integers
// < 2^16) split exactly into hi + lo.
// The A operand flows through a ring of kA 16-column groups (hi | lo, 16 KB)
// with full (128 epilogue-thread arrivals) and empty (tcgen05.commit) barriers,
// so the MMAs of layer l+1 start on the first 16 columns of relu(D_l) while the
// epilogue produces the rest; D_l and D_{l+1} live in two TMEM regions
// (columns 0..207 and 256..463).  Per tile the groups are: the features (1),
// layer-1 output (7, 104 columns), layer-2 output (13), layer-3 output (13).
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr uint32_t kT = 128;               // rows per tile (TMEM lanes)
constexpr uint32_t kEpi = 512;             // epilogue threads: 4 per row
constexpr uint32_t kQ = kEpi / kT;         // column-group phases per row
constexpr uint32_t kThr = kEpi + 64;       // + producer warp + MMA warp
#ifndef KTF_STAGES
#define KTF_STAGES 3
#endif
#ifndef KTF_AGROUPS
#define KTF_AGROUPS 8
#endif
constexpr uint32_t kStages = KTF_STAGES;   // weight ring: one stage = the chunks of one A group (2 k-steps)
constexpr uint32_t kA = KTF_AGROUPS;       // A-group ring
constexpr uint32_t N1 = 112, N2 = 208, N3 = 208, N4 = 112;
constexpr uint32_t S1 = 1, S2 = 13, S3 = 26, S4 = 26;  // k-steps (K = 8, 104, 208, 208)
constexpr uint32_t kChunkMax = 2 * 64 * 208;           // bytes of one weight stage (2 k-steps, hi + lo) at N = 208
constexpr uint32_t G1 = 7, G2 = 13, G3 = 13;           // A groups of the layer 1 / 2 / 3 outputs
constexpr uint32_t kGroups = 1 + G1 + G2 + G3;         // per tile
constexpr uint32_t kGroupBytes = 2 * 4 * kT * 16;      // hi [4 cc][128][4] | lo

// weight blob (bytes): L1 | L2 | L3 | L4 chunks | w5[100] b5 (fp32)
constexpr uint32_t OFF_L1 = 0, OFF_L2 = OFF_L1 + S1 * 64 * N1, OFF_L3 = OFF_L2 + S2 * 64 * N2,
                   OFF_L4 = OFF_L3 + S3 * 64 * N3, OFF_PAR = OFF_L4 + S4 * 64 * N4;
constexpr uint32_t P_W5 = 0, P_B5 = 100, P_N = 104;

// shared memory (bytes)
constexpr uint32_t SM_A = 0, SM_W = SM_A + kA * kGroupBytes, SM_PAR = SM_W + kStages * kChunkMax,
                   SM_RED = SM_PAR + P_N * 4, SM_N = SM_RED + kT * kQ * 4;
static_assert(SM_N <= 232448 - 1024, "K7 tf32 shared memory");

// mbarriers (static shared): W full / empty, A full / empty, layer done x 4
constexpr uint32_t B_WF = 0, B_WE = kStages, B_AF = 2 * kStages, B_AE = 2 * kStages + kA, B_DONE = 2 * kStages + 2 * kA,
                   B_N = B_DONE + 4;

constexpr uint32_t TM_X = 0, TM_Y = 256;  // TMEM regions (columns)

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ constexpr uint32_t idesc_tf32(uint32_t m, uint32_t n) {
  // D f32, A / B tf32 (format 2), both K-major, N >> 3, M >> 4
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
// warp-collective forms for the MMA warp: every lane runs the loop with identical (uniform) operands, one
// elected lane issues
__device__ __forceinline__ void mma_tf32_w(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_w(uint32_t mbar) {
  asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0]; }" ::"r"(mbar));
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

// store 4 consecutive A columns (core-matrix column cc of a group) of this row as hi / lo
__device__ __forceinline__ void store_hl(uint8_t* grp, uint32_t cc, uint32_t row, float a, float b, float c, float d) {
  const float ha = tf32_hi(a), hb = tf32_hi(b), hc = tf32_hi(c), hd = tf32_hi(d);
  const uint32_t off = (cc * kT + row) * 16u;
  *reinterpret_cast<float4*>(grp + off) = make_float4(ha, hb, hc, hd);
  *reinterpret_cast<float4*>(grp + kGroupBytes / 2 + off) = make_float4(tf32_hi(a - ha), tf32_hi(b - hb), tf32_hi(c - hc), tf32_hi(d - hd));
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

// the A ring position of per-CTA group index G
struct Slot {
  uint32_t idx, use;
};
__device__ __forceinline__ Slot slot_of(uint32_t G) { return {G % kA, G / kA}; }

// epilogue thread: wait until ring slot of group G is free, return its smem pointer
__device__ __forceinline__ uint8_t* acquire_group(uint8_t* smem, uint32_t bars, uint32_t G) {
  const Slot sl = slot_of(G);
  if (sl.use > 0) mbar_wait(bars + 8 * (B_AE + sl.idx), (sl.use - 1) & 1u);
  return smem + SM_A + sl.idx * kGroupBytes;
}
// epilogue thread: publish this thread's stores of group G to the MMA (async proxy)
__device__ __forceinline__ void release_group(uint32_t bars, uint32_t G) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");  // this thread's TMEM reads precede the MMA
  mbar_arrive(bars + 8 * (B_AF + slot_of(G).idx));
}

// epilogue of one hidden layer: 16-column groups g = q, q + 4, .. < ng of D (TMEM columns from tsrc) become
// A groups G0 + g: relu below column `one`, 1 at `one` (the next layer's bias input), 0 above
__device__ __forceinline__ void epilogue(uint8_t* smem, uint32_t bars, uint32_t tsrc, uint32_t ng, uint32_t one,
                                         uint32_t G0, uint32_t row, uint32_t q) {
  for (uint32_t g = q; g < ng; g += kQ) {
    uint32_t r[16];
    tmem_ld16(tsrc + g * 16, r);
    tmem_wait();
    float x[16];
    const uint32_t c0 = g * 16;
    if (c0 + 16 <= one) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fmaxf(__uint_as_float(r[j]), 0.0f);
    } else {
#pragma unroll
      for (uint32_t j = 0; j < 16; ++j)
        x[j] = c0 + j < one ? fmaxf(__uint_as_float(r[j]), 0.0f) : (c0 + j == one ? 1.0f : 0.0f);
    }
    uint8_t* grp = acquire_group(smem, bars, G0 + g);
#pragma unroll
    for (uint32_t j = 0; j < 16; j += 4) store_hl(grp, j / 4, row, x[j], x[j + 1], x[j + 2], x[j + 3]);
    release_group(bars, G0 + g);
  }
}

// per-tile A group -> (weight chunks of its k-steps: address, bytes); groups: 1 (layer 1), 7 (layer 2, the last
// one k-step), 13 (layer 3), 13 (layer 4)
__device__ __forceinline__ void wgroup_of(const uint8_t* blob, uint32_t gi, const uint8_t*& src, uint32_t& bytes) {
  const uint32_t g = gi % kGroups;
  if (g < 1) { src = blob + OFF_L1; bytes = 64 * N1; }
  else if (g < 1 + G1) { src = blob + OFF_L2 + (g - 1) * 128 * N2; bytes = (g == G1 ? 64 : 128) * N2; }
  else if (g < 1 + G1 + G2) { src = blob + OFF_L3 + (g - 1 - G1) * 128 * N3; bytes = 128 * N3; }
  else { src = blob + OFF_L4 + (g - 1 - G1 - G2) * 128 * N4; bytes = 128 * N4; }
}

// MMA warp state (identical in every lane)
struct Issuer {
  uint32_t bars, w0, a0;
  uint32_t G = 0;  // A groups (and weight stages) consumed
};

// MMA warp: one layer, K = 8 * steps over A groups G, G + 1, .. (2 k-steps per group; the weight stage of a
// group holds the same k-steps) into tmem_d
__device__ __forceinline__ void mma_layer(Issuer& m, uint32_t tmem_d, uint32_t n, uint32_t steps, uint32_t done) {
  const uint32_t idesc = idesc_tf32(kT, n);
  const uint64_t da0 = sdesc(0, kT * 16, 128), db0 = sdesc(0, n * 16, 128);
  uint32_t st = m.G % kStages, wuse = m.G / kStages;
  uint32_t ai = m.G % kA, ause = m.G / kA;
  for (uint32_t s = 0; s < steps; s += 2) {
    mbar_wait(m.bars + 8 * (B_AF + ai), ause & 1u);
    mbar_wait(m.bars + 8 * (B_WF + st), wuse & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ah = m.a0 + ai * kGroupBytes, bh = m.w0 + st * kChunkMax;
    const uint64_t dah = da0 | (ah >> 4), dal = da0 | ((ah + kGroupBytes / 2) >> 4);
    const uint64_t dbh = db0 | (bh >> 4), dbl = db0 | ((bh + 32 * n) >> 4);
#ifndef KTF_NOMMA
    mma_tf32_w(tmem_d, dah, dbh, idesc, s == 0 ? 0u : 1u);
    mma_tf32_w(tmem_d, dah, dbl, idesc, 1u);
    mma_tf32_w(tmem_d, dal, dbh, idesc, 1u);
    if (s + 1 < steps) {  // second k-step: A + 2 core-matrix columns (4 KB), B + one chunk (64 n bytes)
      constexpr uint64_t a2 = (2 * kT * 16) >> 4;
      const uint64_t b2 = (64 * n) >> 4;
      mma_tf32_w(tmem_d, dah + a2, dbh + b2, idesc, 1u);
      mma_tf32_w(tmem_d, dah + a2, dbl + b2, idesc, 1u);
      mma_tf32_w(tmem_d, dal + a2, dbh + b2, idesc, 1u);
    }
#endif
    commit_w(m.bars + 8 * (B_WE + st));
    commit_w(m.bars + 8 * (B_AE + ai));
    if (++st == kStages) { st = 0; ++wuse; }
    if (++ai == kA) { ai = 0; ++ause; }
    ++m.G;
  }
  commit_w(m.bars + 8 * (B_DONE + done));
}

__global__ void __launch_bounds__(kThr, 1) k_mlp_tf32(const uint16_t* __restrict__ feat, uint32_t n,
                                                     const uint8_t* __restrict__ blob, float* __restrict__ u_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_mem[B_N];
  __shared__ uint32_t tbase;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const float* gpar = reinterpret_cast<const float*>(blob + OFF_PAR);
  float* P = reinterpret_cast<float*>(smem + SM_PAR);
  for (uint32_t i = tid; i < P_N; i += kThr) P[i] = gpar[i];
  const uint32_t bars = (uint32_t)__cvta_generic_to_shared(bar_mem);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  if (tid == 0) {
    for (uint32_t i = 0; i < B_N; ++i) mbar_init(bars + 8 * i, (i >= B_AF && i < B_AE) ? kT : 1u);
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
  const uint32_t tmem = tbase;
  const uint32_t ntiles = (n + kT - 1) / kT;
  const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == kEpi / 32) {
    // ---- producer: every weight chunk of this CTA's tiles, in consumption order
    if ((tid & 31u) == 0)
      for (uint32_t i = 0; i < my_tiles * kGroups; ++i) {
        const uint32_t st = i % kStages, use = i / kStages;
        if (use > 0) mbar_wait(bars + 8 * (B_WE + st), (use - 1) & 1u);
        const uint8_t* src;
        uint32_t bytes;
        wgroup_of(blob, i, src, bytes);
#ifdef KTF_NOCOPY
        if (use > 0) { mbar_arrive(bars + 8 * (B_WF + st)); continue; }
#endif
        bulk_load(s0 + SM_W + st * kChunkMax, src, bytes, bars + 8 * (B_WF + st));
      }
  } else if (warp == kEpi / 32 + 1) {
    // ---- MMA warp (lanes in lockstep, one elected lane issues)
    {
      Issuer m;
      m.bars = bars;
      m.w0 = s0 + SM_W;
      m.a0 = s0 + SM_A;
      for (uint32_t i = 0; i < my_tiles; ++i) {
        mma_layer(m, tmem + TM_Y, N1, S1, 0);  // D1 = [x 1] . [W1 b1]^T
        mma_layer(m, tmem + TM_X, N2, S2, 1);  // D2 = [relu(D1) 1] . [W2 b2]^T
        mma_layer(m, tmem + TM_Y, N3, S3, 2);  // D3
        mma_layer(m, tmem + TM_X, N4, S4, 3);  // D4
      }
    }
  } else {
    // ---- epilogue warps
    const uint32_t row = tid & (kT - 1), q = tid >> 7;
    const uint32_t tmem_row = tmem + (((warp & 3u) * 32u) << 16);
    float* red = reinterpret_cast<float*>(smem + SM_RED);
    auto load_feat = [&](uint32_t t) {
      uint4 f = make_uint4(0, 0, 0, 0);
      const uint32_t rq = t * kT + row;
      if (t < ntiles && rq < n) f = __ldg(reinterpret_cast<const uint4*>(feat + (size_t)rq * 8));
      return f;
    };
    // layer-1 input group: columns (S, Y, M, V, O, P, 1, 0); integers < 2^16 split exactly
    auto stage_feat = [&](uint4 f, uint32_t G) {
      uint8_t* grp = acquire_group(smem, bars, G);
      store_hl(grp, 0, row, (float)(f.x & 0xFFFFu), (float)(f.x >> 16), (float)(f.y & 0xFFFFu), (float)(f.y >> 16));
      store_hl(grp, 1, row, (float)(f.z & 0xFFFFu), (float)(f.z >> 16), 1.0f, 0.0f);
      release_group(bars, G);
    };
    if (q == 0 && my_tiles > 0) stage_feat(load_feat(blockIdx.x), 0);
    for (uint32_t i = 0; i < my_tiles; ++i) {
      const uint32_t t = blockIdx.x + i * gridDim.x;
      const uint32_t Gt = i * kGroups;
      const uint32_t ph = i & 1u;
      mbar_wait(bars + 8 * (B_DONE + 0), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue(smem, bars, tmem_row + TM_Y, G1, 100, Gt + 1, row, q);
      mbar_wait(bars + 8 * (B_DONE + 1), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue(smem, bars, tmem_row + TM_X, G2, 200, Gt + 1 + G1, row, q);
      mbar_wait(bars + 8 * (B_DONE + 2), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue(smem, bars, tmem_row + TM_Y, G3, 200, Gt + 1 + G1 + G2, row, q);
      // the next tile's layer-1 input goes ahead of this tile's layer 5 (loaded here: an outstanding global load
      // would hold up every release_group fence before it)
      if (q == 0 && i + 1 < my_tiles) stage_feat(load_feat(t + gridDim.x), Gt + kGroups);
      mbar_wait(bars + 8 * (B_DONE + 3), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
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
      asm volatile("bar.sync 1, %0;" ::"n"(kEpi) : "memory");
      const uint32_t rq = t * kT + row;
      if (q == 0 && rq < n) {
        float acc = P[P_B5];
#pragma unroll
        for (uint32_t k = 0; k < kQ; ++k) acc += red[k * kT + row];
        u_out[rq] = fmaxf(acc, 0.0f);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpi) : "memory");  // red is reused by the next tile
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
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
  k_mlp_tf32<<<grid, kThr, SM_N, s>>>(feat, n, blob, u);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
