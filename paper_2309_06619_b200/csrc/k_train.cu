// k_train.cu — NEXT-2 (optional part of the offline profiling, Alg. 1):
// mini-batch Adam training of the lightweight MLP m_theta on (rule scores,
// output length) pairs, minimising the MSE of P:455 (v2 P:1384) with the
// learning rate of P:620 chosen by the caller.  fp32 on the CUDA cores, every
// reduction in a fixed order (deterministic).  Host orchestration in api.cu
// (rt_train_mlp); readings R-TRAIN in DESIGN.md.
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr int kTile = 32;  // output tile (kTile x kTile), 16 x 16 threads, 2 x 2 outputs per thread

// C[m][n] = sum_k A(m, k) * B(k, n) (+ bias[n]) (ReLU if relu), k ascending.
// A(m, k) = A[m * sam + k * sak], B(k, n) = B[k * sbk + n * sbn]; C row-major [M][ldc].
__global__ void __launch_bounds__(256) k_gemm(const float* __restrict__ A, uint32_t sam, uint32_t sak,
                                              const float* __restrict__ B, uint32_t sbk, uint32_t sbn,
                                              const float* __restrict__ bias, float* __restrict__ C, uint32_t ldc,
                                              uint32_t M, uint32_t N, uint32_t K, int relu) {
  __shared__ float As[kTile][kTile + 1], Bs[kTile][kTile + 1];
  const uint32_t tx = threadIdx.x & 15u, ty = threadIdx.x >> 4;
  const uint32_t m0 = blockIdx.y * kTile, n0 = blockIdx.x * kTile;
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  for (uint32_t k0 = 0; k0 < K; k0 += kTile) {
    for (uint32_t i = threadIdx.x; i < kTile * kTile; i += 256) {
      const uint32_t r = i / kTile, c = i % kTile;
      const uint32_t am = m0 + r, ak = k0 + c, bk = k0 + r, bn = n0 + c;
      As[r][c] = (am < M && ak < K) ? A[(size_t)am * sam + (size_t)ak * sak] : 0.f;
      Bs[r][c] = (bk < K && bn < N) ? B[(size_t)bk * sbk + (size_t)bn * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (uint32_t k = 0; k < (uint32_t)kTile; ++k) {
      const float a0 = As[ty * 2][k], a1 = As[ty * 2 + 1][k];
      const float b0 = Bs[k][tx * 2], b1 = Bs[k][tx * 2 + 1];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t m = m0 + ty * 2 + i, n = n0 + tx * 2 + j;
      if (m < M && n < N) {
        float v = acc[i][j] + (bias ? bias[n] : 0.f);
        if (relu) v = fmaxf(v, 0.f);
        C[(size_t)m * ldc + n] = v;
      }
    }
}

// batch k of an epoch: rows pi(i) = (a * i + b) mod n, i in [i0, i0 + bsz)
__global__ void k_gather(const uint16_t* __restrict__ feat, const float* __restrict__ y, uint32_t n, uint64_t a,
                         uint64_t b, uint32_t i0, uint32_t bsz, float* __restrict__ x, float* __restrict__ yb) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= bsz) return;
  const uint32_t r = (uint32_t)((a * (uint64_t)(i0 + i) + b) % n);
#pragma unroll
  for (int k = 0; k < 6; ++k) x[(size_t)i * 6 + k] = (float)feat[(size_t)r * 8 + k];
  yb[i] = y[r];
}

// dz = 2 (z - y) / bsz; the batch's squared errors summed in index order (one
// warp, fixed order) into the epoch's fp64 accumulator
__global__ void __launch_bounds__(32) k_loss(const float* __restrict__ z, const float* __restrict__ yb, uint32_t bsz,
                                             float* __restrict__ dz, double* __restrict__ epoch_sq) {
  const uint32_t lane = threadIdx.x;
  double s = 0.0;
  for (uint32_t i = lane; i < bsz; i += 32) {
    const float d = z[i] - yb[i];
    dz[i] = 2.0f * d / (float)bsz;
    s += (double)d * (double)d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xFFFFFFFFu, s, o);
  if (lane == 0) *epoch_sq += s;
}

// gb[n] = sum over the batch of dZ[m][n] (m ascending)
__global__ void k_colsum(const float* __restrict__ dZ, uint32_t M, uint32_t N, float* __restrict__ gb) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float s = 0.f;
  for (uint32_t m = 0; m < M; ++m) s += dZ[(size_t)m * N + c];
  gb[c] = s;
}

// dZ_prev = dA * (A_prev > 0)   (ReLU derivative, 0 at 0)
__global__ void k_relu_back(float* __restrict__ dA, const float* __restrict__ Aprev, size_t cnt) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt && !(Aprev[i] > 0.f)) dA[i] = 0.f;
}

// Adam: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// p -= lr * (m * c1) / (sqrt(v * c2) + eps), c1 = 1/(1-b1^t), c2 = 1/(1-b2^t)
__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, uint32_t cnt, float lr, float c1, float c2) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const float gi = g[i];
  const float mi = 0.9f * m[i] + 0.1f * gi;
  const float vi = 0.999f * v[i] + 0.001f * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr * (mi * c1) / (sqrtf(vi * c2) + 1e-8f);
}

}  // namespace

cudaError_t launch_gemm(const float* A, uint32_t sam, uint32_t sak, const float* B, uint32_t sbk, uint32_t sbn,
                        const float* bias, float* C, uint32_t ldc, uint32_t M, uint32_t N, uint32_t K, int relu,
                        cudaStream_t s) {
  if (!M || !N) return cudaSuccess;
  const dim3 grid((N + kTile - 1) / kTile, (M + kTile - 1) / kTile);
  k_gemm<<<grid, 256, 0, s>>>(A, sam, sak, B, sbk, sbn, bias, C, ldc, M, N, K, relu);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_gather(const uint16_t* feat, const float* y, uint32_t n, uint64_t a, uint64_t b, uint32_t i0,
                          uint32_t bsz, float* x, float* yb, cudaStream_t s) {
  k_gather<<<(bsz + 255) / 256, 256, 0, s>>>(feat, y, n, a, b, i0, bsz, x, yb);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_loss(const float* z, const float* yb, uint32_t bsz, float* dz, double* epoch_sq, cudaStream_t s) {
  k_loss<<<1, 32, 0, s>>>(z, yb, bsz, dz, epoch_sq);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_colsum(const float* dZ, uint32_t M, uint32_t N, float* gb, cudaStream_t s) {
  k_colsum<<<(N + 127) / 128, 128, 0, s>>>(dZ, M, N, gb);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_relu_back(float* dA, const float* Aprev, size_t cnt, cudaStream_t s) {
  if (!cnt) return cudaSuccess;
  k_relu_back<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(dA, Aprev, cnt);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, uint32_t cnt, float lr, float c1, float c2,
                        cudaStream_t s) {
  k_adam<<<(cnt + 255) / 256, 256, 0, s>>>(p, g, m, v, cnt, lr, c1, c2);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
