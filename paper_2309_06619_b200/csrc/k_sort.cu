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
                                                    uint32_t ntiles, uint32_t* __restrict__ hist,
                                                    const uint32_t* __restrict__ n_dev) {
  __shared__ uint32_t h[256];
  if (n_dev) n = min(n, *n_dev);
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
                                                       uint32_t* __restrict__ vout, const uint32_t* __restrict__ n_dev) {
  if (n_dev) n = min(n, *n_dev);
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

// ---- stable split of a queue by class (bit 63): CPU class / GPU class
__global__ void __launch_bounds__(kThreads) k_split_count(const uint64_t* __restrict__ key, uint32_t n,
                                                           uint32_t* __restrict__ bsum) {
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  const bool cpu = i < n && (key[i] >> 63);
  const uint32_t c = __syncthreads_count(cpu);
  if (threadIdx.x == 0) bsum[blockIdx.x] = c;
}

__global__ void __launch_bounds__(1024) k_split_scan(uint32_t* __restrict__ bsum, uint32_t nb, uint32_t n,
                                                     uint32_t* __restrict__ counts) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, nb);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += bsum[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const uint32_t v = threadIdx.x >= (uint32_t)d ? part[threadIdx.x - d] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t v = bsum[i];
    bsum[i] = run;
    run += v;
  }
  if (threadIdx.x == 1023) {
    counts[0] = part[1023];      // CPU class
    counts[1] = n - part[1023];  // GPU class
  }
}

__global__ void __launch_bounds__(kThreads) k_split_write(const uint64_t* __restrict__ key, uint32_t n, uint32_t base,
                                                           const uint32_t* __restrict__ boff, uint64_t* __restrict__ ck,
                                                           uint32_t* __restrict__ cv, uint64_t* __restrict__ gk,
                                                           uint32_t* __restrict__ gv) {
  __shared__ uint32_t wsum[kWarps];
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint64_t k = i < n ? key[i] : 0ull;
  const bool cpu = i < n && (k >> 63);
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, cpu);
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  uint32_t c = boff[blockIdx.x];
  for (uint32_t j = 0; j < w; ++j) c += wsum[j];
  c += __popc(bal & ((1u << lane) - 1u));  // CPU-class elements before i
  if (i < n) {
    if (cpu) { ck[c] = k; cv[c] = base + i; }
    else { gk[i - c] = k; gv[i - c] = base + i; }
  }
}

}  // namespace

cudaError_t split_by_class(const uint64_t* key, uint32_t base, uint32_t n, uint32_t* bsum, uint32_t* counts,
                           uint64_t* ck, uint32_t* cv, uint64_t* gk, uint32_t* gv, cudaStream_t s) {
  const uint32_t nb = (n + kThreads - 1) / kThreads;
  k_split_count<<<nb, kThreads, 0, s>>>(key, n, bsum);
  k_split_scan<<<1, 1024, 0, s>>>(bsum, nb, n, counts);
  k_split_write<<<nb, kThreads, 0, s>>>(key, n, base, bsum, ck, cv, gk, gv);
  note_launch(3);
  return cudaGetLastError();
}

size_t radix_sort_workspace(uint32_t n) {
  size_t ntiles = (n + kTile - 1) / kTile;
  size_t a = ((size_t)n * 8 + 255) & ~size_t(255);
  size_t b = ((size_t)n * 4 + 255) & ~size_t(255);
  return 2 * a + b + ((256 * ntiles * 4 + 255) & ~size_t(255));
}

// keys_in: n keys; perm_out: n global indices (base_index + i) sorted by key desc.
cudaError_t radix_sort_desc(const uint64_t* keys_in, uint32_t base_index, uint32_t n, uint32_t* perm_out, int full64,
                            void* ws, cudaStream_t s) {
  return radix_sort_desc2(keys_in, nullptr, base_index, n, nullptr, perm_out, full64, ws, s);
}

// general form: values vals_in (NULL = base_index + i), element count n_dev read
// on the device (NULL = n); n is the host upper bound used for grid sizes
cudaError_t radix_sort_desc2(const uint64_t* keys_in, const uint32_t* vals_in, uint32_t base_index, uint32_t n,
                             const uint32_t* n_dev, uint32_t* perm_out, int full64, void* ws, cudaStream_t s) {
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
  const uint32_t* vsrc = vals_in;  // null = identity (base_index + i)
  for (int j = 0; j < nsh; ++j) {
    const int shift = full64 ? 8 * j : shifts_f[j];
    uint64_t* kdst = (j & 1) ? k2 : k1;
    // values ping-pong between perm_out and v2 so that the last pass writes perm_out
    uint32_t* vdst = ((nsh - 1 - j) & 1) ? v2 : perm_out;
    k_hist<<<ntiles, kThreads, 0, s>>>(ksrc, n, shift, ntiles, hist, n_dev);
    k_scan<<<1, 256, 0, s>>>(hist, ntiles);
    k_scatter<<<ntiles, kThreads, 0, s>>>(ksrc, vsrc, base_index, n, shift, ntiles, hist, kdst, vdst, n_dev);
    note_launch(3);
    ksrc = kdst;
    vsrc = vdst;
  }
  return cudaGetLastError();
}

}  // namespace rtlm
