// k_offline.cu — K8 (NEXT-2): offline-profiling primitives on the GPU
// (Alg. 1 offline part).
//
// * Weighted-rule fit: target ~ c + sum_k w_k f_k over the
//   six rule scores by the normal equations with ridge 1e-8.  X^T X holds
//   integer sums (features are u16 counts), exact in fp64 whatever the order;
//   X^T y is summed in a fixed order (fixed grid, strided threads, a fixed
//   block tree, then the block partials in index order), so results are
//   reproducible run to run.  The 7x7 system is solved by Cholesky on the
//   device.
// * Nearest-rank quantile tau = sorted(u)[ceil(k n) - 1] (Eq. 4, P:441-444;
//   S:211) and u_max = max(u): a radix sort of ord32(u) (K3) and a pick.
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr int kFitThreads = 256;
constexpr int kFitBlocks = 592;  // 4 x 148 SMs, fixed: the reduction order does not depend on the device
constexpr int kFitN = 35;        // 28 upper-triangle entries of X^T X (7x7) + 7 of X^T y

__global__ void __launch_bounds__(kFitThreads) k_fit_partial(const uint16_t* __restrict__ feat,
                                                            const float* __restrict__ y, uint32_t n,
                                                            double* __restrict__ part) {
  double acc[kFitN];
#pragma unroll
  for (int i = 0; i < kFitN; ++i) acc[i] = 0.0;
  for (uint32_t r = blockIdx.x * kFitThreads + threadIdx.x; r < n; r += kFitBlocks * kFitThreads) {
    const uint4 f = *reinterpret_cast<const uint4*>(feat + (size_t)r * 8);
    const double x[7] = {1.0, (double)(f.x & 0xFFFFu), (double)(f.x >> 16), (double)(f.y & 0xFFFFu),
                         (double)(f.y >> 16), (double)(f.z & 0xFFFFu), (double)(f.z >> 16)};
    const double yr = (double)y[r];
    int k = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i)
#pragma unroll
      for (int j = i; j < 7; ++j) acc[k++] += x[i] * x[j];
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[28 + i] += x[i] * yr;
  }
  __shared__ double s[kFitThreads];
#pragma unroll
  for (int i = 0; i < kFitN; ++i) {
    s[threadIdx.x] = acc[i];
    __syncthreads();
    for (int w = kFitThreads / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)blockIdx.x * kFitN + i] = s[0];
    __syncthreads();
  }
}

// out[0..6] = (c, w_S, w_Y, w_M, w_V, w_O, w_P); out[7] = (min/max Cholesky pivot)^2,
// a conditioning diagnostic; NaN coefficients if the damped matrix is not positive definite
__global__ void __launch_bounds__(1024) k_fit_solve(const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double tot[kFitN];
  // warp w sums entries w, w + 32 over the block partials: lane-strided, then a fixed shuffle tree
  for (int e = threadIdx.x >> 5; e < kFitN; e += 32) {
    const int lane = threadIdx.x & 31;
    double t = 0.0;
    for (int b = lane; b < kFitBlocks; b += 32) t += part[(size_t)b * kFitN + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if (lane == 0) tot[e] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double A[7][7], rhs[7], L[7][7];
  int k = 0;
  for (int i = 0; i < 7; ++i)
    for (int j = i; j < 7; ++j) { A[i][j] = tot[k]; A[j][i] = tot[k]; ++k; }
  for (int i = 0; i < 7; ++i) { A[i][i] += 1e-8; rhs[i] = tot[28 + i]; }
  double pmin = 1e300, pmax = 0.0;
  bool ok = true;
  for (int j = 0; j < 7 && ok; ++j) {
    double d = A[j][j];
    for (int q = 0; q < j; ++q) d -= L[j][q] * L[j][q];
    if (!(d > 0.0)) { ok = false; break; }
    L[j][j] = sqrt(d);
    pmin = fmin(pmin, L[j][j]);
    pmax = fmax(pmax, L[j][j]);
    for (int i = j + 1; i < 7; ++i) {
      double v = A[i][j];
      for (int q = 0; q < j; ++q) v -= L[i][q] * L[j][q];
      L[i][j] = v / L[j][j];
    }
  }
  if (!ok) {
    for (int i = 0; i < 8; ++i) out[i] = __longlong_as_double(0x7FF8000000000000ll);
    return;
  }
  double z[7], b[7];
  for (int i = 0; i < 7; ++i) {  // L z = rhs
    double v = rhs[i];
    for (int q = 0; q < i; ++q) v -= L[i][q] * z[q];
    z[i] = v / L[i][i];
  }
  for (int i = 6; i >= 0; --i) {  // L^T b = z
    double v = z[i];
    for (int q = i + 1; q < 7; ++q) v -= L[q][i] * b[q];
    b[i] = v / L[i][i];
  }
  for (int i = 0; i < 7; ++i) out[i] = b[i];
  out[7] = (pmin / pmax) * (pmin / pmax);
}

__global__ void k_u_keys(const float* __restrict__ u, uint32_t n, uint64_t* __restrict__ key) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    key[i] = ord32_bits(__float_as_uint(u[i]));
}

// perm: indices sorted by u descending (stable); ascending rank r = n - 1 - position
__global__ void k_quantile_pick(const float* __restrict__ u, const uint32_t* __restrict__ perm, uint32_t n,
                                uint32_t r, float* __restrict__ out) {
  out[0] = u[perm[n - 1 - r]];
  out[1] = u[perm[0]];
}

}  // namespace

size_t fit_workspace() { return (size_t)kFitBlocks * kFitN * sizeof(double); }

cudaError_t launch_fit(const uint16_t* feat, const float* y, uint32_t n, double* ws, double* out, cudaStream_t s) {
  k_fit_partial<<<kFitBlocks, kFitThreads, 0, s>>>(feat, y, n, ws);
  k_fit_solve<<<1, 1024, 0, s>>>(ws, out);
  note_launch(2);
  return cudaGetLastError();
}

size_t quantile_workspace(uint32_t n) {
  return (((size_t)n * 8 + 255) & ~size_t(255)) + (((size_t)n * 4 + 255) & ~size_t(255)) + radix_sort_workspace(n);
}

cudaError_t launch_quantile(const float* u, uint32_t n, uint32_t r, void* ws, float* out, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  uint64_t* key = reinterpret_cast<uint64_t*>(p);
  p += ((size_t)n * 8 + 255) & ~size_t(255);
  uint32_t* perm = reinterpret_cast<uint32_t*>(p);
  p += ((size_t)n * 4 + 255) & ~size_t(255);
  const uint32_t g = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
  k_u_keys<<<g, 256, 0, s>>>(u, n, key);
  note_launch();
  cudaError_t e = radix_sort_desc(key, 0, n, perm, 0, p, s);
  if (e != cudaSuccess) return e;
  k_quantile_pick<<<1, 1, 0, s>>>(u, perm, n, r, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
