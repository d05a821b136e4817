// k_mlp_f32.cu — K7 (NEXT-1), fp32 mode: the lightweight MLP m_theta of Eq. 1
// (layers 6-100-200-200-100-1, P:620 / P:1547; ReLU on hidden layers, output
// clamped at 0) with every multiply-add in binary32 on the CUDA
// cores, in a fixed order: out[j] = fma chain over k = 0..K-1 starting from
// b[j].  The paper's MLP is an fp32 PyTorch model; this mode is
// the default (rt_set_mlp_precision), the bf16 tensor-core kernel (k_mlp.cu)
// the opt-in fast mode.
//
// Persistent CTAs of 256 threads (two per SM), a tile is 64 requests.  The
// tile's activations stay in shared memory (one 64 x 204 fp32 buffer that each
// layer overwrites in place, row-major, rows
// padded to 204 words), weights stream from L2 in k-chunks of 32 (k-major,
// [k][208]), double-buffered with cp.async; a 4-row x 16-column register tile
// per thread (see layer()).
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr uint32_t kT = 64;        // requests per tile
constexpr uint32_t kThr = 256;
constexpr uint32_t kXS = 204;      // activation row stride (words)
constexpr uint32_t kNW = 208;      // weight chunk row (output columns, padded)
constexpr uint32_t kKC = 32;       // k per weight chunk
// fp32 blob (mlp_f32_pack): W1[100][6] b1[100] | W2t[100][208] b2[208] | W3t[200][208] b3[208] |
// W4t[200][208] b4[208] | W5[100] b5  -- Wlt = W_l transposed to [in][out], out padded to 208
constexpr uint32_t F_W1 = 0, F_B1 = 600, F_W2 = 700, F_B2 = F_W2 + 100 * kNW, F_W3 = F_B2 + kNW,
                   F_B3 = F_W3 + 200 * kNW, F_W4 = F_B3 + kNW, F_B4 = F_W4 + 200 * kNW, F_W5 = F_B4 + kNW,
                   F_B5 = F_W5 + 100, F_N = F_B5 + 4;

struct Smem {
  float X[kT][kXS];             // activations (each layer overwrites its input in place)
  float W[2][kKC][kNW];         // weight chunks (double buffer)
  float w1[600], b1[100], w5[100];
};

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// stage rows [k0, k0 + kc) of a transposed weight matrix (row = 208 floats)
__device__ __forceinline__ void stage_w(float (*dst)[kNW], const float* __restrict__ src, uint32_t k0, uint32_t kc) {
  const uint32_t nv = kc * (kNW / 4);  // 16-byte vectors
  for (uint32_t v = threadIdx.x; v < nv; v += kThr) {
    const uint32_t r = v / (kNW / 4), c4 = v % (kNW / 4);
    cp16(&dst[r][c4 * 4], src + (size_t)(k0 + r) * kNW + c4 * 4);
  }
  cp_commit();
}

// one hidden layer: Y[64][N] = relu(X[64][K] . Wt[K][N] + b), fma chain in k order.
// Thread t < 208 owns rows 4 rg .. 4 rg + 3 (rg = t / 13) and the 16 columns
// 4 cg + 52 v + e (cg = t % 13, v, e < 4; consecutive threads read consecutive
// 16-byte quads: no bank conflicts): every 4 k, four 128-bit activation loads
// and sixteen 128-bit weight loads feed 256 FMAs.
__device__ __forceinline__ void layer(Smem& S, const float* __restrict__ Wt, const float* __restrict__ b, uint32_t K,
                                      uint32_t N) {
  float (*X)[kXS] = S.X;
  const uint32_t t = threadIdx.x;
  const bool act = t < 16u * 13u;
  const uint32_t rg = act ? t / 13u : 0u, cg = act ? t % 13u : 0u;
  const uint32_t c0 = 4u * cg;
  auto colof = [&](int j) { return c0 + 52u * (uint32_t)(j >> 2) + (uint32_t)(j & 3); };
  float acc[4][16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t col = colof(j);
    const float bj = col < N ? __ldg(b + col) : 0.0f;
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r][j] = bj;
  }
  const uint32_t nch = (K + kKC - 1) / kKC;
  __syncthreads();  // previous users of S.W / X are done
  stage_w(S.W[0], Wt, 0, min(kKC, K));
  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t k0 = c * kKC, kc = min(kKC, K - k0);
    cp_wait_all();
    __syncthreads();  // chunk c visible to all; chunk c-1's buffer free
    if (c + 1 < nch) stage_w(S.W[(c + 1) & 1], Wt, k0 + kKC, min(kKC, K - k0 - kKC));
    const float (*Wc)[kNW] = S.W[c & 1];
    if (act) {
      for (uint32_t kk = 0; kk < kc; kk += 4) {  // K is a multiple of 4 (100, 200)
        float4 a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = *reinterpret_cast<const float4*>(&X[4 * rg + r][k0 + kk]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 w[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) w[v] = *reinterpret_cast<const float4*>(&Wc[kk + q][c0 + 52 * v]);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float av = q == 0 ? a[r].x : q == 1 ? a[r].y : q == 2 ? a[r].z : a[r].w;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              acc[r][4 * v + 0] = __fmaf_rn(av, w[v].x, acc[r][4 * v + 0]);
              acc[r][4 * v + 1] = __fmaf_rn(av, w[v].y, acc[r][4 * v + 1]);
              acc[r][4 * v + 2] = __fmaf_rn(av, w[v].z, acc[r][4 * v + 2]);
              acc[r][4 * v + 3] = __fmaf_rn(av, w[v].w, acc[r][4 * v + 3]);
            }
          }
        }
      }
    }
  }
  __syncthreads();  // every thread has read its inputs: overwrite X with the outputs
  if (act) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t col = colof(j);
      if (col < N)
#pragma unroll
        for (int r = 0; r < 4; ++r) X[4 * rg + r][col] = fmaxf(acc[r][j], 0.0f);
    }
  }
}

__global__ void __launch_bounds__(kThr, 2) k_mlp_f32(const uint16_t* __restrict__ feat, uint32_t n,
                                                    const float* __restrict__ P, float* __restrict__ u_out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < 600; i += kThr) S.w1[i] = P[F_W1 + i];
  for (uint32_t i = tid; i < 100; i += kThr) {
    S.b1[i] = P[F_B1 + i];
    S.w5[i] = P[F_W5 + i];
  }
  const float b5 = P[F_B5];
  __syncthreads();
  const uint32_t ntiles = (n + kT - 1) / kT;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    // ---- layer 1 (6 -> 100): X0[r][j], 64 x 100 outputs, fma chain over the 6 inputs
    __syncthreads();
    for (uint32_t o = tid; o < kT * 100; o += kThr) {
      const uint32_t r = o / 100, j = o % 100, rq = t * kT + r;
      float acc = 0.0f;
      if (rq < n) {
        const uint4 f = __ldg(reinterpret_cast<const uint4*>(feat + (size_t)rq * 8));
        const float x[6] = {(float)(f.x & 0xFFFFu), (float)(f.x >> 16), (float)(f.y & 0xFFFFu),
                            (float)(f.y >> 16), (float)(f.z & 0xFFFFu), (float)(f.z >> 16)};
        acc = S.b1[j];
#pragma unroll
        for (int i = 0; i < 6; ++i) acc = __fmaf_rn(S.w1[j * 6 + i], x[i], acc);
        acc = fmaxf(acc, 0.0f);
      }
      S.X[r][j] = acc;
    }
    // ---- layers 2-4
    layer(S, P + F_W2, P + F_B2, 100, 200);
    layer(S, P + F_W3, P + F_B3, 200, 200);
    layer(S, P + F_W4, P + F_B4, 200, 100);
    __syncthreads();
    // ---- layer 5 (100 -> 1), clamp at 0: 4 threads per row, then a fixed-order sum
    if (tid < kT) {
      const uint32_t rq = t * kT + tid;
      float acc = b5;
      for (uint32_t k = 0; k < 100; ++k) acc = __fmaf_rn(S.w5[k], S.X[tid][k], acc);
      if (rq < n) u_out[rq] = fmaxf(acc, 0.0f);
    }
  }
}

}  // namespace

size_t mlp_f32_blob_bytes() { return (size_t)F_N * 4; }

void mlp_f32_pack(const float* const w[5], const float* const b[5], float* p) {
  memset(p, 0, mlp_f32_blob_bytes());
  for (uint32_t i = 0; i < 600; ++i) p[F_W1 + i] = w[0][i];
  for (uint32_t i = 0; i < 100; ++i) p[F_B1 + i] = b[0][i];
  auto tr = [&](uint32_t off, uint32_t boff, const float* W, const float* B, uint32_t out, uint32_t in) {
    for (uint32_t o = 0; o < out; ++o) {
      for (uint32_t k = 0; k < in; ++k) p[off + (size_t)k * kNW + o] = W[(size_t)o * in + k];
      p[boff + o] = B[o];
    }
  };
  tr(F_W2, F_B2, w[1], b[1], 200, 100);
  tr(F_W3, F_B3, w[2], b[2], 200, 200);
  tr(F_W4, F_B4, w[3], b[3], 100, 200);
  for (uint32_t i = 0; i < 100; ++i) p[F_W5 + i] = w[4][i];
  p[F_B5] = b[4][0];
}

cudaError_t launch_mlp_f32(const uint16_t* feat, uint32_t n, const float* blob, float* u, int num_sms,
                           cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int smem = (int)sizeof(Smem);
  cudaError_t e = cudaFuncSetAttribute(k_mlp_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const uint32_t ntiles = (n + kT - 1) / kT;
  const uint32_t grid = ntiles < 2u * (uint32_t)num_sms ? ntiles : 2u * (uint32_t)num_sms;  // 2 CTAs per SM
  k_mlp_f32<<<grid, kThr, smem, s>>>(feat, n, blob, u);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
