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
#ifndef KSORT_ITEMS
#define KSORT_ITEMS 12
#endif
constexpr int kItems = KSORT_ITEMS;
constexpr uint32_t kTile = kThreads * kItems;  // keys per tile
constexpr int kWarps = kThreads / 32;
constexpr int kMaxPass = 8;
constexpr uint32_t kFlagA = 1u << 30;  // tile aggregate published
constexpr uint32_t kFlagP = 2u << 30;  // inclusive prefix published
constexpr uint32_t kCountMask = (1u << 30) - 1u;

struct Passes {
  int n;
  int shift[kMaxPass];
};

__device__ __forceinline__ uint32_t digit_of(uint64_t key, int shift) { return (uint32_t)(~key >> shift) & 0xFFu; }

// global digit histograms of every pass in one read of the keys
__global__ void __launch_bounds__(kThreads) k_ghist(const uint64_t* __restrict__ keys, uint32_t n,
                                                     const uint32_t* __restrict__ n_dev, Passes ps,
                                                     uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kMaxPass][256];
  if (n_dev) n = min(n, *n_dev);
  for (int p = 0; p < kMaxPass; ++p) h[p][threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int p = 0; p < kMaxPass; ++p)
      if (p < ps.n) atomicAdd(&h[p][digit_of(k, ps.shift[p])], 1u);
  }
  __syncthreads();
  for (int p = 0; p < ps.n; ++p) {
    const uint32_t c = h[p][threadIdx.x];
    if (c) atomicAdd(&ghist[p * 256 + threadIdx.x], c);
  }
}

__device__ __forceinline__ void st_relaxed(uint32_t* a, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// exclusive block scan over 256 threads (one value each)
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t* wsum) {
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t run = incl - x;
  for (uint32_t k = 0; k < w; ++k) run += wsum[k];
  return run;
}

// One stable counting pass ("onesweep"): a tile ranks its keys per warp with
// __match_any_sync, publishes its digit counts, looks back over the earlier
// tiles' published counts (decoupled look-back, tiles taken in launch order
// from an atomic counter), reorders the tile in shared memory by digit and
// writes runs of equal digits contiguously.
__global__ void __launch_bounds__(kThreads) k_onesweep(const uint64_t* __restrict__ kin,
                                                        const uint32_t* __restrict__ vin, uint32_t base_index,
                                                        uint32_t n, const uint32_t* __restrict__ n_dev, int shift,
                                                        const uint32_t* __restrict__ ghist, uint32_t* status,
                                                        uint32_t* counter, uint64_t* __restrict__ kout,
                                                        uint32_t* __restrict__ vout) {
  extern __shared__ __align__(16) uint8_t sort_smem[];
  uint64_t* s_k = reinterpret_cast<uint64_t*>(sort_smem);               // [kTile]
  uint32_t* s_v = reinterpret_cast<uint32_t*>(sort_smem + kTile * 8);   // [kTile]
  __shared__ uint32_t s_wcnt[kWarps][256];
  __shared__ uint32_t s_loc[256], s_glob[256], s_wsum[2][8];
  __shared__ uint32_t s_tile;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
#pragma unroll
  for (int k = 0; k < kWarps; ++k) s_wcnt[k][tid] = 0;
  if (n_dev) n = min(n, *n_dev);
  __syncthreads();
  const uint32_t tile = s_tile, t0 = tile * kTile;
  if (t0 >= n) return;
  uint64_t key[kItems];
  uint32_t val[kItems], dg[kItems], rk[kItems];
  const uint32_t wb = t0 + w * (kTile / kWarps);
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t i = wb + r * 32 + lane;
    const bool ok = i < n;
    key[r] = ok ? kin[i] : 0ull;
    val[r] = ok ? (vin ? vin[i] : base_index + i) : 0u;
    dg[r] = ok ? digit_of(key[r], shift) : 256u;
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t d = dg[r];
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t before = d < 256u ? s_wcnt[w][d] : 0u;
    rk[r] = before + __popc(peers & lt);
    __syncwarp();
    if (d < 256u && (peers & lt) == 0u) s_wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // thread = digit: tile count, per-warp exclusive prefix
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const uint32_t c = s_wcnt[k][tid];
    s_wcnt[k][tid] = tot;
    tot += c;
  }
  uint32_t* st = status + (size_t)tile * 256u + tid;
  if (tile == 0) st_relaxed(st, kFlagP | tot);
  else st_relaxed(st, kFlagA | tot);
  const uint32_t gbase = block_excl_scan256(ghist[tid], s_wsum[0]);
  const uint32_t lbase = block_excl_scan256(tot, s_wsum[1]);
  uint32_t excl = 0;
  if (tile > 0) {
    uint32_t p = tile - 1;
    for (;;) {
      uint32_t v;
      do { v = ld_relaxed(status + (size_t)p * 256u + tid); } while ((v & ~kCountMask) == 0u);
      excl += v & kCountMask;
      if ((v & kFlagP) || p == 0) break;
      --p;
    }
    st_relaxed(st, kFlagP | (excl + tot));
  }
  s_loc[tid] = lbase;
  s_glob[tid] = gbase + excl;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t d = dg[r];
    if (d < 256u) {
      const uint32_t lp = s_loc[d] + s_wcnt[w][d] + rk[r];
      s_k[lp] = key[r];
      s_v[lp] = val[r];
    }
  }
  __syncthreads();
  const uint32_t cnt = min(kTile, n - t0);
#pragma unroll 4
  for (uint32_t i = tid; i < cnt; i += kThreads) {
    const uint64_t k = s_k[i];
    const uint32_t d = digit_of(k, shift);
    const uint32_t pos = s_glob[d] + (i - s_loc[d]);
    kout[pos] = k;
    vout[pos] = s_v[i];
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

static size_t status_words(uint32_t n) {
  const size_t ntiles = (n + kTile - 1) / kTile;
  return (size_t)kMaxPass * 256 + kMaxPass + (size_t)kMaxPass * ntiles * 256;  // ghist, counters, status
}

size_t radix_sort_workspace(uint32_t n) {
  size_t a = ((size_t)n * 8 + 255) & ~size_t(255);
  size_t b = ((size_t)n * 4 + 255) & ~size_t(255);
  return 2 * a + b + ((status_words(n) * 4 + 255) & ~size_t(255));
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
  uint32_t* ghist = reinterpret_cast<uint32_t*>(p + 2 * a + b);
  uint32_t* counters = ghist + kMaxPass * 256;
  uint32_t* status = counters + kMaxPass;
  Passes ps;
  const int shifts_f[5] = {0, 8, 16, 24, 56};
  ps.n = full64 ? 8 : 5;
  for (int j = 0; j < kMaxPass; ++j) ps.shift[j] = j < ps.n ? (full64 ? 8 * j : shifts_f[j]) : 0;
  cudaMemsetAsync(ghist, 0, status_words(n) * 4, s);
  const uint32_t gh_blocks = ntiles < 592 ? ntiles : 592;
  k_ghist<<<gh_blocks, kThreads, 0, s>>>(keys_in, n, n_dev, ps, ghist);
  const int smem = kTile * 12;
  cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // ping-pong: pass j reads (ksrc, vsrc) writes (kdst, vdst); last pass writes perm_out
  const uint64_t* ksrc = keys_in;
  const uint32_t* vsrc = vals_in;  // null = identity (base_index + i)
  for (int j = 0; j < ps.n; ++j) {
    uint64_t* kdst = (j & 1) ? k2 : k1;
    // values ping-pong between perm_out and v2 so that the last pass writes perm_out
    uint32_t* vdst = ((ps.n - 1 - j) & 1) ? v2 : perm_out;
    k_onesweep<<<ntiles, kThreads, smem, s>>>(ksrc, vsrc, base_index, n, n_dev, ps.shift[j], ghist + j * 256,
                                              status + (size_t)j * ntiles * 256, counters + j, kdst, vdst);
    ksrc = kdst;
    vsrc = vdst;
  }
  note_launch(1 + ps.n);
  return cudaGetLastError();
}

}  // namespace rtlm
