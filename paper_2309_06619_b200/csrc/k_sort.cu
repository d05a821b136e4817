// k_sort.cu — K3: stable LSD radix sort of 64-bit priority keys in DESCENDING
// order (Alg. 1 "descending p order"; ties keep input order, R-TIE).
// Used for queues larger than one CTA (small queues and traces are sorted in
// shared memory inside their own kernels).
//
// Per 8-bit digit pass: (1) per-tile digit histograms, (2) one-CTA exclusive
// scan in digit-major order, (3) stable scatter: each tile ranks its keys
// round by round with __match_any_sync + per-warp counts, so equal digits
// keep their input order.  Keys are complemented so an ascending sort yields
// descending keys.  For binary32-valued policies only the bytes that can vary
// (0-3 and 7: value, tier, class) are passed over.
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr uint32_t kTile = kThreads * kItems;  // 4096 keys
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t* __restrict__ keys, uint32_t n, int shift,
                                                    uint32_t ntiles, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t t0 = blockIdx.x * kTile;
#pragma unroll 4
  for (int k = 0; k < kItems; ++k) {
    uint32_t i = t0 + k * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(uint32_t)(~keys[i] >> shift) & 0xFFu], 1u);
  }
  __syncthreads();
  hist[blockIdx.x * 256u + threadIdx.x] = h[threadIdx.x];  // tile-major
}

// exclusive scan of the tile-major histogram in digit-major order: thread d
// owns digit d (coalesced across threads), sums its column, a block scan over
// digits gives the digit bases, a second pass writes the running offsets.
__global__ void __launch_bounds__(256) k_scan(uint32_t* __restrict__ hist, uint32_t ntiles) {
  __shared__ uint32_t wsum[8];
  const uint32_t d = threadIdx.x, lane = d & 31u, w = d >> 5;
  uint32_t s = 0;
#pragma unroll 8
  for (uint32_t t = 0; t < ntiles; ++t) s += hist[t * 256u + d];
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t run = incl - s;
  for (uint32_t k = 0; k < w; ++k) run += wsum[k];
#pragma unroll 8
  for (uint32_t t = 0; t < ntiles; ++t) {
    const uint32_t v = hist[t * 256u + d];
    hist[t * 256u + d] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kThreads) k_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       uint32_t base_index, uint32_t n, int shift, uint32_t ntiles,
                                                       const uint32_t* __restrict__ hist, uint64_t* __restrict__ kout,
                                                       uint32_t* __restrict__ vout) {
  __shared__ uint32_t s_base[256];           // running output position per digit
  __shared__ uint16_t s_cnt[kWarps][256];    // per-warp digit counts of the current round
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  s_base[threadIdx.x] = hist[blockIdx.x * 256u + threadIdx.x];
  const uint32_t t0 = blockIdx.x * kTile;
  const uint32_t lt = (1u << lane) - 1u;
  for (int k = 0; k < kItems; ++k) {
    for (int w = 0; w < kWarps; ++w) s_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    const uint32_t i = t0 + k * kThreads + threadIdx.x;
    const bool valid = i < n;
    uint64_t key = valid ? kin[i] : 0ull;
    uint32_t val = valid ? (vin ? vin[i] : base_index + i) : 0u;
    uint32_t d = valid ? ((uint32_t)(~key >> shift) & 0xFFu) : 256u;
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) s_cnt[warp][d] = (uint16_t)__popc(peers);
    __syncthreads();
    // per digit: exclusive prefix over warps (thread = digit)
    {
      uint32_t run = 0;
      for (int w = 0; w < kWarps; ++w) {
        uint32_t c = s_cnt[w][threadIdx.x];
        s_cnt[w][threadIdx.x] = (uint16_t)run;
        run += c;
      }
      __syncthreads();
      if (valid) {
        uint32_t pos = s_base[d] + s_cnt[warp][d] + rank;
        kout[pos] = key;
        vout[pos] = val;
      }
      __syncthreads();
      s_base[threadIdx.x] += run;
    }
    __syncthreads();
  }
}

}  // namespace

size_t radix_sort_workspace(uint32_t n) {
  size_t ntiles = (n + kTile - 1) / kTile;
  size_t a = ((size_t)n * 8 + 255) & ~size_t(255);
  size_t b = ((size_t)n * 4 + 255) & ~size_t(255);
  return 2 * a + b + ((256 * ntiles * 4 + 255) & ~size_t(255));
}

// keys_in: n keys; perm_out: n global indices (base_index + i) sorted by key desc.
cudaError_t radix_sort_desc(const uint64_t* keys_in, uint32_t base_index, uint32_t n, uint32_t* perm_out, int full64,
                            void* ws, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const uint32_t ntiles = (n + kTile - 1) / kTile;
  char* p = static_cast<char*>(ws);
  size_t a = ((size_t)n * 8 + 255) & ~size_t(255);
  size_t b = ((size_t)n * 4 + 255) & ~size_t(255);
  uint64_t* k1 = reinterpret_cast<uint64_t*>(p);
  uint64_t* k2 = reinterpret_cast<uint64_t*>(p + a);
  uint32_t* v2 = reinterpret_cast<uint32_t*>(p + 2 * a);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p + 2 * a + b);
  const int shifts_f[5] = {0, 8, 16, 24, 56};
  const int nsh = full64 ? 8 : 5;
  // ping-pong: pass j reads (ksrc, vsrc) writes (kdst, vdst); last pass writes perm_out
  const uint64_t* ksrc = keys_in;
  const uint32_t* vsrc = nullptr;  // null = identity (base_index + i)
  for (int j = 0; j < nsh; ++j) {
    const int shift = full64 ? 8 * j : shifts_f[j];
    uint64_t* kdst = (j & 1) ? k2 : k1;
    // values ping-pong between perm_out and v2 so that the last pass writes perm_out
    uint32_t* vdst = ((nsh - 1 - j) & 1) ? v2 : perm_out;
    k_hist<<<ntiles, kThreads, 0, s>>>(ksrc, n, shift, ntiles, hist);
    k_scan<<<1, 256, 0, s>>>(hist, ntiles);
    k_scatter<<<ntiles, kThreads, 0, s>>>(ksrc, vsrc, base_index, n, shift, ntiles, hist, kdst, vdst);
    note_launch(3);
    ksrc = kdst;
    vsrc = vdst;
  }
  return cudaGetLastError();
}

}  // namespace rtlm
