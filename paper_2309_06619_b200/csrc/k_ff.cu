// k_ff.cu — parallel exact one-pass consolidation of ONE large queue
// (§8(a) row a6, Alg. 1 P:467-481 with R-CONS/R-CARRY/R-FLUSH), DESIGN.md §7.
//
// Reformulation (proved in DESIGN.md §7 "K4-FF"):  let S be the GPU-class
// stream in priority order, x ≺ y the window order (u, then rank), K = m - C.
// While windows are full, the carry after every cut-free round equals
// topK_≺(consumed prefix), so every element becomes *ready* exactly when it
// is evicted from a streaming top-K heap: the ready sequence Rseq (one element
// per consumed position) is computed in parallel (chunk top-K summaries, a
// scan of summaries, per-chunk heap replays).  O6 then equals the "R-process"
// on Rseq: A = L ∪ next (C - |L|) ready elements; emit the λ-prefix of sorted
// A (<= C); L = rest.  From an empty L (an "∅-point" z) the next round is the
// aligned chunk Rseq[z, z+C): if it passes the λ chain the process is at ∅
// again at z + C.  So the trajectory is ∅-runs of aligned chunks separated by
// "excursions" that start at failing chunks.  We evaluate pass(j) for every j,
// simulate the excursion from every failing position in parallel, link
// failing positions into a successor forest, find the trajectory's path by
// pointer doubling, and emit ∅-run chunks and path excursions in parallel.
// The last partial windows (stream exhausted) are finished by one warp (tail).
#include <algorithm>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace rtlm {
namespace {

constexpr uint32_t KS = 128;         // row stride of K-lists (K <= 127)
constexpr uint32_t B1 = 1024;        // heap-replay chunk
constexpr uint32_t kEnd = 0xFFFFFFFFu;
constexpr uint64_t kInf = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ float kk_u(uint64_t k) { return __uint_as_float((uint32_t)(k >> 32) & 0x7FFFFFFFu); }

struct FF {
  // inputs
  uint32_t* perm;         // queue-relative priority order output (global indices), CPU class first
  const uint32_t* gperm;  // GPU class in priority order (global indices)
  const uint32_t* ncpu_dev;
  const float* u;
  const uint64_t* key;
  uint32_t n;             // queue length
  uint32_t K, C, m;
  float lambda;
  // device scalars
  uint32_t* scal;         // [0] ncpu [1] G [2] NR [3] nfail [4] stretch elements [5] - [6] path_len [7] #descriptors
  // buffers
  uint64_t* kk;           // G
  uint64_t* rseq;         // NR
  uint64_t* summ;         // nc1 * KS
  uint64_t* heapH;        // nc1 * KS  (exclusive prefix top-K per chunk)
  uint64_t* hfinal;       // KS
  uint32_t* passbm;       // bitmap, bit j = pass(j)
  uint32_t* failpos;      // nfail (sorted)
  uint32_t* exE;          // excursion end ∅-point (kEnd = reached the stream end)
  uint32_t* exR;          // rounds inside the excursion
  uint32_t* nxt;          // levels * (nfail + 1)
  uint32_t* wr;           // levels * (nfail + 1)
  uint32_t* runz;         // per fail i (and start node nfail): ∅-point after the excursion
  uint32_t* runn;         // chunks of the ∅-run
  uint32_t* path_node;    // path nodes (unordered)
  uint32_t* path_off;     // batch offset at the node's excursion start
  uint32_t* run_z;        // sorted ∅-runs: start
  uint32_t* run_n;        // chunks
  uint32_t* run_b;        // first batch id
  uint32_t levels;
  float* vt;              // C x vstride: u(max) of Rseq[j, j+c) if that chunk passes its λ chain, else +inf
  uint32_t vstride;
  uint32_t* ds_j;         // stretch descriptors (emission): start, chunk size, rounds, first batch
  uint32_t* ds_c;
  uint32_t* ds_r;
  uint32_t* ds_b;
  uint32_t* ds_pre;       // exclusive prefix of ds_r * ds_c
  uint32_t* batch_p;      // G: batch id by stream position p (scattered to global indices at the end)
  uint8_t* slot_p;        // G
  uint32_t* batch_of;
  uint8_t* slot_of;
  uint8_t* core_of;
  uint32_t* seg_count_q;  // &seg_count[q]
};

__device__ __forceinline__ void put(const FF& f, uint64_t x, uint32_t b, uint32_t slot) {
  const uint32_t p = (uint32_t)x;
  f.batch_p[p] = b;
  f.slot_p[p] = (uint8_t)slot;
}

// ------------------------------------------------------------ 1. gather
__global__ void k_ff_gather(FF f) {
  const uint32_t ncpu = *f.ncpu_dev, G = f.n - ncpu;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < G; p += gridDim.x * blockDim.x) {
    const uint32_t g = f.gperm[p];
    f.perm[ncpu + p] = g;  // the API's priority order (GPU class after the CPU class)
    f.kk[p] = ((uint64_t)ord32_bits(__float_as_uint(f.u[g])) << 32) | p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    f.scal[0] = ncpu;
    f.scal[1] = G;
    f.scal[2] = G > f.K ? G - f.K : 0u;
  }
}

// ------------------------------------------------------------ 2. ready sequence
// 2a: top-K (descending) of every chunk of B1 positions
__global__ void __launch_bounds__(256) k_ff_topk(FF f) {
  __shared__ uint64_t s[B1];
  const uint32_t G = f.scal[1];
  const uint32_t c = blockIdx.x, p0 = c * B1;
  if (p0 >= G) return;
  for (uint32_t i = threadIdx.x; i < B1; i += 256) s[i] = p0 + i < G ? f.kk[p0 + i] : 0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= B1; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < B1; i += 256) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint64_t a = s[i], b = s[l];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) { s[i] = b; s[l] = a; }
        }
      }
      __syncthreads();
    }
  for (uint32_t i = threadIdx.x; i < KS; i += 256) f.summ[(size_t)c * KS + i] = i < f.K ? s[i] : 0ull;
}

// merge two descending K-lists (smem) into their top-K (smem out); one warp.
// Real keys are unique; zero padding may collide only with zeros.
__device__ void merge_topk(const uint64_t* A, const uint64_t* B, uint64_t* O, uint32_t K) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t i = lane; i < K; i += 32) {
    const uint64_t a = A[i];
    uint32_t lo = 0, hi = K;  // #(B > a)
    while (lo < hi) { uint32_t md = (lo + hi) >> 1; if (B[md] > a) lo = md + 1; else hi = md; }
    if (i + lo < K) O[i + lo] = a;
    const uint64_t b = B[i];
    lo = 0; hi = K;           // #(A > b)
    while (lo < hi) { uint32_t md = (lo + hi) >> 1; if (A[md] > b) lo = md + 1; else hi = md; }
    if (i + lo < K) O[i + lo] = b;
  }
  __syncwarp();
}

// 2b: exclusive prefix top-K over chunks (one CTA of 32 warps)
__global__ void __launch_bounds__(1024) k_ff_scan(FF f, uint64_t* loc) {
  extern __shared__ __align__(16) uint64_t buf_raw[];
  uint64_t (*buf)[3][KS] = reinterpret_cast<uint64_t (*)[3][KS]>(buf_raw);
  const uint32_t G = f.scal[1];
  const uint32_t nc = (G + B1 - 1) / B1;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u, K = f.K;
  const uint32_t gs = (nc + 31) / 32;
  const uint32_t c0 = w * gs, c1 = min(nc, c0 + gs);
  uint64_t* acc = buf[w][0];
  uint64_t* tmp = buf[w][1];
  uint64_t* nx = buf[w][2];
  for (uint32_t i = lane; i < KS; i += 32) acc[i] = 0ull;
  __syncwarp();
  // level 1: inclusive running top-K inside the group
  for (uint32_t c = c0; c < c1; ++c) {
    for (uint32_t i = lane; i < KS; i += 32) tmp[i] = f.summ[(size_t)c * KS + i];
    __syncwarp();
    for (uint32_t i = lane; i < KS; i += 32) nx[i] = 0ull;
    __syncwarp();
    merge_topk(acc, tmp, nx, K);
    for (uint32_t i = lane; i < KS; i += 32) { acc[i] = nx[i]; loc[(size_t)c * KS + i] = nx[i]; }
    __syncwarp();
  }
  __syncthreads();
  // level 2: warp 0 computes the exclusive prefix of group totals into buf[g][0]
  if (w == 0) {
    uint64_t* run = buf[0][1];
    uint64_t* t2 = buf[0][2];
    for (uint32_t i = lane; i < KS; i += 32) run[i] = 0ull;
    __syncwarp();
    for (uint32_t g = 0; g < 32; ++g) {
      const uint32_t gc0 = g * gs, gc1 = min(nc, gc0 + gs);
      // group g's exclusive prefix = run; stash into heapH of its first chunk (if any)
      if (gc0 < gc1)
        for (uint32_t i = lane; i < KS; i += 32) f.heapH[(size_t)gc0 * KS + i] = run[i];
      __syncwarp();
      if (gc0 < gc1) {
        // run = merge(run, loc[last of group])
        uint64_t* lastl = buf[1][0];  // scratch (warp 1 finished level 1)
        for (uint32_t i = lane; i < KS; i += 32) lastl[i] = loc[(size_t)(gc1 - 1) * KS + i];
        __syncwarp();
        for (uint32_t i = lane; i < KS; i += 32) t2[i] = 0ull;
        __syncwarp();
        merge_topk(run, lastl, t2, K);
        for (uint32_t i = lane; i < KS; i += 32) run[i] = t2[i];
        __syncwarp();
      }
    }
    // the overall top-K = final heap (elements never ready)
    for (uint32_t i = lane; i < KS; i += 32) f.hfinal[i] = run[i];
  }
  __syncthreads();
  // level 3: H[c] = merge(groupprefix, loc[c-1]) for c > c0 in the group
  if (c0 < c1) {
    uint64_t* gp = buf[w][0];
    for (uint32_t i = lane; i < KS; i += 32) gp[i] = f.heapH[(size_t)c0 * KS + i];
    __syncwarp();
    for (uint32_t c = c0 + 1; c < c1; ++c) {
      for (uint32_t i = lane; i < KS; i += 32) { tmp[i] = loc[(size_t)(c - 1) * KS + i]; nx[i] = 0ull; }
      __syncwarp();
      merge_topk(gp, tmp, nx, K);
      for (uint32_t i = lane; i < KS; i += 32) f.heapH[(size_t)c * KS + i] = nx[i];
      __syncwarp();
    }
  }
}

// ---- K <= 32: top-K lists held in a warp's registers (lane i = i-th largest,
// zero padding below every real key).
__device__ __forceinline__ uint64_t sort32_desc(uint64_t v) {  // bitonic sort across the warp
  const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
      const bool keep_max = ((lane & k) == 0) == ((lane & j) == 0);
      v = keep_max ? (v > o ? v : o) : (v < o ? v : o);
    }
  return v;
}

// top 32 of the union of two descending lists, descending
__device__ __forceinline__ uint64_t merge32_desc(uint64_t a, uint64_t b) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t br = __shfl_sync(0xFFFFFFFFu, b, 31 - lane);
  uint64_t v = a > br ? a : br;  // bitonic (decreasing, then increasing)
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
    v = (lane & j) == 0 ? (v > o ? v : o) : (v < o ? v : o);
  }
  return v;
}

// 2a (K <= 32): top-K of every chunk, one warp per chunk; a batch of 32 keys is
// merged only if one of them beats the current K-th largest
__global__ void __launch_bounds__(256) k_ff_topk32(FF f) {
  const uint32_t G = f.scal[1], K = f.K;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  const uint32_t p0 = c * B1;
  if (p0 >= G) return;
  const uint32_t p1 = min(G, p0 + B1);
  uint64_t top = 0, thr = 0;
  // eight 32-key batches loaded at once (one L2 round trip instead of eight),
  // then taken in order
  for (uint32_t pg = p0; pg < p1; pg += 8 * 32) {
    uint64_t xs[8];
#pragma unroll
    for (uint32_t t = 0; t < 8; ++t) {
      const uint32_t i = pg + t * 32 + lane;
      xs[t] = i < p1 ? __ldg(f.kk + i) : 0ull;
    }
#pragma unroll
    for (uint32_t t = 0; t < 8; ++t) {
      if (!__any_sync(0xFFFFFFFFu, xs[t] > thr)) continue;
      top = merge32_desc(top, sort32_desc(xs[t]));
      thr = __shfl_sync(0xFFFFFFFFu, top, K - 1);
    }
  }
  f.summ[(size_t)c * KS + lane] = lane < K ? top : 0ull;
}

// 2b (K <= 32): exclusive prefix top-K over chunks, one CTA of 32 warps:
// running merges inside 32 groups, a scan of the group totals, then
// H[c] = merge(group prefix, inclusive[c - 1]).
__global__ void __launch_bounds__(1024) k_ff_scan32(FF f, uint64_t* loc) {
  __shared__ uint64_t s_tot[32][32], s_pre[32][32];
  const uint32_t G = f.scal[1], K = f.K;
  const uint32_t nc = (G + B1 - 1) / B1;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t gs = (nc + 31) / 32;
  const uint32_t c0 = min(nc, w * gs), c1 = min(nc, c0 + gs);
  uint64_t acc = 0;
  uint64_t nxt = c0 < c1 ? f.summ[(size_t)c0 * KS + lane] : 0ull;
  for (uint32_t c = c0; c < c1; ++c) {
    const uint64_t t = nxt;
    if (c + 1 < c1) nxt = f.summ[(size_t)(c + 1) * KS + lane];
    acc = merge32_desc(acc, t);
    loc[(size_t)c * KS + lane] = lane < K ? acc : 0ull;
  }
  s_tot[w][lane] = lane < K ? acc : 0ull;
  __syncthreads();
  if (w == 0) {
    uint64_t run = 0;
    for (uint32_t g = 0; g < 32; ++g) {
      s_pre[g][lane] = run;
      const uint32_t gc0 = min(nc, g * gs);
      if (gc0 < min(nc, gc0 + gs)) run = merge32_desc(run, s_tot[g][lane]);
    }
    f.hfinal[lane] = lane < K ? run : 0ull;
    for (uint32_t i = 32 + lane; i < KS; i += 32) f.hfinal[i] = 0ull;
  }
  __syncthreads();
  if (c0 < c1) {
    const uint64_t gp = lane < K ? s_pre[w][lane] : 0ull;
    f.heapH[(size_t)c0 * KS + lane] = gp;
    for (uint32_t c = c0 + 1; c < c1; ++c) {
      const uint64_t h = merge32_desc(gp, loc[(size_t)(c - 1) * KS + lane]);  // whole warp
      f.heapH[(size_t)c * KS + lane] = lane < K ? h : 0ull;
    }
  }
}

// 2c: per-chunk streaming heap replay -> Rseq (evictions).  Heap slots s =
// t*32 + lane, ascending; unused slots (>= K) hold +inf.
template <int SPL>
__global__ void __launch_bounds__(128) k_ff_replay(FF f) {
  const uint32_t G = f.scal[1], K = f.K;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  const uint32_t p0 = warp * B1;
  if (p0 >= G) return;
  const uint32_t p1 = min(G, p0 + B1);
  uint64_t h[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const uint32_t s = t * 32 + lane;
    h[t] = s < K ? f.heapH[(size_t)warp * KS + (K - 1 - s)] : kInf;
  }
  uint64_t nxt = p0 + lane < p1 ? __ldg(f.kk + p0 + lane) : 0ull;  // the next batch, loaded one batch ahead
  for (uint32_t pb = p0; pb < p1; pb += 32) {
    const uint64_t mine = nxt;
    if (pb + 32 < p1) nxt = pb + 32 + lane < p1 ? __ldg(f.kk + pb + 32 + lane) : 0ull;
    const uint32_t cnt = min(32u, p1 - pb);
    // a key below the heap's minimum at the start of the batch is evicted at once
    // (the minimum only grows), so only the others go through the insertion
    const uint64_t hmin = __shfl_sync(0xFFFFFFFFu, h[0], 0);
    uint64_t outv = mine;
    uint32_t todo = __ballot_sync(0xFFFFFFFFu, lane < cnt && mine > hmin);
    while (todo) {
      const uint32_t i = __ffs(todo) - 1;
      todo &= todo - 1u;
      const uint64_t x = __shfl_sync(0xFFFFFFFFu, mine, i);
      uint32_t c = 0;
#pragma unroll
      for (int t = 0; t < SPL; ++t) c += __popc(__ballot_sync(0xFFFFFFFFu, h[t] < x));
      const uint64_t h0 = __shfl_sync(0xFFFFFFFFu, h[0], 0);
      // shift slots [1, c) down by one, x into slot c-1
      uint64_t nh[SPL];
#pragma unroll
      for (int t = 0; t < SPL; ++t) {
        uint64_t up = __shfl_down_sync(0xFFFFFFFFu, h[t], 1);
        const uint64_t wrap = (t + 1 < SPL) ? __shfl_sync(0xFFFFFFFFu, h[t + 1 < SPL ? t + 1 : t], 0) : kInf;
        if (lane == 31) up = wrap;
        const uint32_t sl = t * 32 + lane;
        nh[t] = (sl + 1 < c) ? up : ((sl + 1 == c) ? x : h[t]);
      }
#pragma unroll
      for (int t = 0; t < SPL; ++t) h[t] = nh[t];
      if (lane == i) outv = c ? h0 : x;  // evicted element of position pb + i
    }
    const uint32_t q = pb + lane;
    if (lane < cnt && q >= K) f.rseq[q - K] = outv;
  }
}

// K == 0: every element is ready at its own position
__global__ void k_ff_copy(FF f) {
  const uint32_t G = f.scal[1];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < G; p += gridDim.x * blockDim.x) f.rseq[p] = f.kk[p];
  if (blockIdx.x == 0 && threadIdx.x == 0) f.hfinal[0] = 0ull;
}

// ------------------------------------------------------------ 3. chunk tables
// For every start j and chunk size c = 1..C: vt[c-1][j] = u(max of Rseq[j, j+c))
// if the sorted chunk passes the λ chain (every adjacent ratio <= λ), else
// +inf (also +inf when j + c > NR).  Incremental insertion keeps the count of
// failing adjacent pairs.  pass(j) = vt[C-1][j] < inf.
__device__ __forceinline__ bool ratio_bad(uint64_t lo, uint64_t hi, float lam) {
  return !(kk_u(hi) <= __fmul_rn(lam, kk_u(lo)));
}

// The λ-chain of a chunk depends only on its multiset of u values: equal
// values are adjacent in the (u, rank) order and never violate u <= λ·u, so
// the violating adjacent pairs are those between consecutive DISTINCT values.
// Adding x to a chunk: no change if its u is already present, else the pairs
// (pred, x), (x, succ) replace (pred, succ), with pred / succ the nearest
// smaller / larger distinct u.  All comparisons on the u bits (u >= 0, so bit
// order = value order), stored + 1 so that 0 means "none".
__global__ void __launch_bounds__(256) k_ff_vtab(FF f) {
  __shared__ uint32_t t[256 + kMaxWindow];
  const uint32_t NR = f.scal[2], C = f.C;
  const uint32_t j0 = blockIdx.x * 256u;
  const uint32_t nwords = (NR + 31) / 32 + 1;
  if (j0 >= nwords * 32) return;  // block-uniform
  const uint32_t j = j0 + threadIdx.x;
  for (uint32_t i = threadIdx.x; i < 256 + C; i += 256)
    t[i] = j0 + i < NR ? __float_as_uint(kk_u(f.rseq[j0 + i])) + 1u : 0u;
  __syncthreads();
  const uint32_t* w = t + threadIdx.x;
  const float lam = f.lambda;
  auto bad2 = [&](uint32_t lo1, uint32_t hi1) {  // u values + 1
    return !(__uint_as_float(hi1 - 1u) <= __fmul_rn(lam, __uint_as_float(lo1 - 1u)));
  };
  int bad = 0;
  uint32_t mx = 0;
  bool passC = false;
  for (uint32_t c = 1; c <= C; ++c) {
    const bool full = j + c <= NR;
    if (full) {
      const uint32_t x = w[c - 1];
      uint32_t pred = 0u, succ = 0xFFFFFFFFu;
      bool dup = false;
      for (uint32_t b = 0; b + 1 < c; ++b) {
        const uint32_t y = w[b];
        pred = (y < x && y > pred) ? y : pred;
        succ = (y > x && y < succ) ? y : succ;
        dup |= y == x;
      }
      const bool hp = pred != 0u, hs = succ != 0xFFFFFFFFu;
      if (!dup) bad += (hp && bad2(pred, x)) + (hs && bad2(x, succ)) - (hp && hs && bad2(pred, succ));
      mx = x > mx ? x : mx;
    }
    if (j < NR) f.vt[(size_t)(c - 1) * f.vstride + j] = (full && bad == 0) ? __uint_as_float(mx - 1u) : __int_as_float(0x7f800000);
    if (c == C) passC = full && bad == 0;
  }
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, passC);
  if ((threadIdx.x & 31u) == 0 && j < nwords * 32) f.passbm[j >> 5] = bal;
}

// k_ff_vtab with the chunk size CT = C known at compile time (the profiles'
// C = 11 and 33): the chunk's u values in registers, both loops unrolled --
// the same table entry for entry
template <int CT>
__global__ void __launch_bounds__(256) k_ff_vtab_t(FF f) {
  __shared__ uint32_t t[256 + kMaxWindow];
  const uint32_t NR = f.scal[2];
  const uint32_t j0 = blockIdx.x * 256u;
  const uint32_t nwords = (NR + 31) / 32 + 1;
  if (j0 >= nwords * 32) return;  // block-uniform
  const uint32_t j = j0 + threadIdx.x;
  for (uint32_t i = threadIdx.x; i < 256 + CT; i += 256)
    t[i] = j0 + i < NR ? __float_as_uint(kk_u(f.rseq[j0 + i])) + 1u : 0u;
  __syncthreads();
  uint32_t w[CT];
#pragma unroll
  for (int b = 0; b < CT; ++b) w[b] = t[threadIdx.x + b];
  const float lam = f.lambda;
  auto bad2 = [&](uint32_t lo1, uint32_t hi1) {  // u values + 1
    return !(__uint_as_float(hi1 - 1u) <= __fmul_rn(lam, __uint_as_float(lo1 - 1u)));
  };
  int bad = 0;
  uint32_t mx = 0;
  bool passC = false;
#pragma unroll
  for (int c = 1; c <= CT; ++c) {
    const bool full = j + c <= NR;
    if (full) {
      const uint32_t x = w[c - 1];
      uint32_t pred = 0u, succ = 0xFFFFFFFFu;
      bool dup = false;
#pragma unroll
      for (int b = 0; b + 1 < c; ++b) {
        const uint32_t y = w[b];
        pred = (y < x && y > pred) ? y : pred;
        succ = (y > x && y < succ) ? y : succ;
        dup |= y == x;
      }
      const bool hp = pred != 0u, hs = succ != 0xFFFFFFFFu;
      if (!dup) bad += (hp && bad2(pred, x)) + (hs && bad2(x, succ)) - (hp && hs && bad2(pred, succ));
      mx = x > mx ? x : mx;
    }
    if (j < NR) f.vt[(size_t)(c - 1) * f.vstride + j] = (full && bad == 0) ? __uint_as_float(mx - 1u) : __int_as_float(0x7f800000);
    if (c == CT) passC = full && bad == 0;
  }
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, passC);
  if ((threadIdx.x & 31u) == 0 && j < nwords * 32) f.passbm[j >> 5] = bal;
}

__device__ __forceinline__ bool pass_at(const uint32_t* bm, uint32_t j) { return (bm[j >> 5] >> (j & 31u)) & 1u; }

// compact failing positions (j + C <= NR and !pass)
__global__ void k_ff_failcount(FF f, uint32_t* blocksum) {
  const uint32_t NR = f.scal[2], C = f.C;
  const uint32_t lim = NR >= C ? NR - C + 1 : 0u;  // positions with a full chunk
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool fl = j < lim && !pass_at(f.passbm, j);
  const uint32_t c = __syncthreads_count(fl);
  if (threadIdx.x == 0) blocksum[blockIdx.x] = c;
}

// exclusive scan of nb counters by one CTA; total -> *total
__global__ void __launch_bounds__(1024) k_ff_blockscan(uint32_t* blocksum, uint32_t nb, uint32_t* total) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, nb);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += blocksum[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    uint32_t v = threadIdx.x >= (uint32_t)d ? part[threadIdx.x - d] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (uint32_t i = lo; i < hi; ++i) {
    uint32_t v = blocksum[i];
    blocksum[i] = run;
    run += v;
  }
  if (threadIdx.x == 1023) *total = part[1023];
}

__global__ void k_ff_failwrite(FF f, const uint32_t* blockoff) {
  __shared__ uint32_t wsum[32];
  const uint32_t NR = f.scal[2], C = f.C;
  const uint32_t lim = NR >= C ? NR - C + 1 : 0u;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool fl = j < lim && !pass_at(f.passbm, j);
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, fl);
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  uint32_t base = blockoff[blockIdx.x];
  for (uint32_t i = 0; i < w; ++i) base += wsum[i];
  if (fl) f.failpos[base + __popc(bal & ((1u << lane) - 1u))] = j;
}

// ------------------------------------------------------------ 4. trajectories
// A trajectory of the R-process alternates GENERAL rounds (O6 round on
// A = L ∪ next C-|L| ready elements) and STEADY stretches: with ℓ = |L| and
// c = C - ℓ, a round at j is steady (emits exactly the chunk Rseq[j, j+c),
// leaves L unchanged) iff the chunk passes its λ chain and
// u(min L) > λ·u(max chunk) -- i.e. !(u0 <= λ·vt[c-1][j]) with u0 = u(min L)
// (+inf when L is empty).  ffwd() checks 32 consecutive rounds per warp step.
constexpr uint32_t kFfwdDepth = 4;
__device__ __forceinline__ uint32_t ffwd(const FF& f, uint32_t lc, float u0, uint32_t& j, uint32_t NR) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t c = f.C - lc;
  const float* vt = f.vt + (size_t)(c - 1) * f.vstride;
  const auto pass = [&](uint32_t jk) { return (jk + c <= NR) && !(u0 <= __fmul_rn(f.lambda, __ldg(vt + jk))); };
  uint32_t total = 0;
  {  // most stretches inside an excursion are short: one batch of 32 rounds first
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pass(j + lane * c));
    const uint32_t k = (bal == 0xFFFFFFFFu) ? 32u : (uint32_t)(__ffs(~bal) - 1);
    j += k * c;
    total += k;
    if (k < 32) return total;
  }
  // long stretch: four batches (128 rounds) in flight per step, so that one
  // L2 round trip covers 128 rounds instead of 32
  for (;;) {
    bool ok[kFfwdDepth];
#pragma unroll
    for (uint32_t u = 0; u < kFfwdDepth; ++u) ok[u] = pass(j + (u * 32u + lane) * c);
#pragma unroll
    for (uint32_t u = 0; u < kFfwdDepth; ++u) {
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, ok[u]);
      const uint32_t k = (bal == 0xFFFFFFFFu) ? 32u : (uint32_t)(__ffs(~bal) - 1);
      j += k * c;
      total += k;
      if (k < 32) return total;
    }
  }
}

// ---- general rounds, shared-memory version (any C <= 128)
struct Warp3 {
  uint64_t* L;  // capacity kMaxWindow
  uint64_t* A;
  uint64_t* S;
};

template <class Emit>
__device__ __forceinline__ uint32_t r_round(const FF& f, Warp3 w, uint32_t& lc, uint32_t& j, uint32_t na,
                                            Emit emit) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t need = na - lc;
  for (uint32_t i = lane; i < na; i += 32) w.A[i] = i < lc ? w.L[i] : f.rseq[j + (i - lc)];
  __syncwarp();
  for (uint32_t i = lane; i < na; i += 32) {
    const uint64_t x = w.A[i];
    uint32_t pos = 0;
    for (uint32_t b = 0; b < na; ++b) pos += w.A[b] < x;
    w.S[pos] = x;
  }
  __syncwarp();
  const uint32_t lim = min(f.C, na);
  uint32_t cnt = lim;
  for (uint32_t base = 1; base < lim; base += 32) {
    const uint32_t i = base + lane;
    const bool bad = i < lim && ratio_bad(w.S[i - 1], w.S[i], f.lambda);
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
    if (bal) { cnt = base + __ffs(bal) - 1; break; }
  }
  for (uint32_t i = lane; i < cnt; i += 32) emit(w.S[i], i);
  for (uint32_t i = lane; i < na - cnt; i += 32) w.L[i] = w.S[cnt + i];
  lc = na - cnt;
  j += need;
  __syncwarp();
  return cnt;
}

struct SmemTraj {
  Warp3 w;
  uint32_t lc = 0;
  __device__ void init(const FF&, uint32_t, uint32_t) { lc = 0; }
  __device__ float u0() const { return lc ? kk_u(w.L[0]) : __int_as_float(0x7f800000); }
  template <class Emit>
  __device__ uint32_t round(const FF& f, uint32_t& j, uint32_t, Emit emit) { return r_round(f, w, lc, j, f.C, emit); }
};

// ---- general rounds, register version (C <= 32): lane i holds A[i]; Rseq is
// streamed through a per-warp shared ring filled three 32-entry blocks ahead.
constexpr uint32_t kRing = 512;

__device__ __forceinline__ uint64_t ld_rseq(const FF& f, uint32_t q, uint32_t NR) { return q < NR ? f.rseq[q] : kInf; }

struct RegTraj {
  uint64_t* ring;
  uint64_t* S;
  uint32_t filled, issue;
  uint64_t pf0, pf1, pf2;
  uint64_t lv;
  uint32_t lc;
  __device__ void init(const FF& f, uint32_t j, uint32_t NR) {
    const uint32_t lane = threadIdx.x & 31u;
    filled = j;
    pf0 = ld_rseq(f, j + lane, NR);
    pf1 = ld_rseq(f, j + 32 + lane, NR);
    pf2 = ld_rseq(f, j + 64 + lane, NR);
    issue = j + 96;
    lv = kInf;
    lc = 0;
  }
  __device__ void step(const FF& f, uint32_t NR) {
    const uint32_t lane = threadIdx.x & 31u;
    ring[(filled + lane) & (kRing - 1)] = pf0;
    filled += 32;
    pf0 = pf1;
    pf1 = pf2;
    pf2 = ld_rseq(f, issue + lane, NR);
    issue += 32;
  }
  __device__ float u0() const {
    const uint64_t l0 = __shfl_sync(0xFFFFFFFFu, lv, 0);
    return lc ? kk_u(l0) : __int_as_float(0x7f800000);
  }
  template <class Emit>
  __device__ uint32_t round(const FF& f, uint32_t& j, uint32_t NR, Emit emit) {
    const uint32_t lane = threadIdx.x & 31u, C = f.C;
    if (j > filled) {  // jumped past the prefetched range: restart the pipeline at j
      const uint64_t keep = lv;
      const uint32_t klc = lc;
      init(f, j, NR);
      lv = keep;
      lc = klc;
    }
    while (filled < j + C) step(f, NR);
    if (filled < j + C + 64) step(f, NR);
    __syncwarp();
    const uint64_t x = lane < lc ? lv : (lane < C ? ring[(j + lane - lc) & (kRing - 1)] : kInf);
    uint32_t rank = 0;
    for (uint32_t k = 0; k < C; ++k) rank += __shfl_sync(0xFFFFFFFFu, x, k) < x;
    if (lane < C) S[rank] = x;
    __syncwarp();
    const uint64_t sv = lane < C ? S[lane] : kInf;
    const uint64_t pv = __shfl_up_sync(0xFFFFFFFFu, sv, 1);
    const bool bad = lane >= 1 && lane < C && ratio_bad(pv, sv, f.lambda);
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
    const uint32_t cnt = bal ? __ffs(bal) - 1 : C;
    if (lane < cnt) emit(sv, lane);
    lv = __shfl_sync(0xFFFFFFFFu, sv, min(lane + cnt, 31u));
    j += C - lc;
    lc = C - cnt;
    __syncwarp();
    return cnt;
  }
};

__device__ __forceinline__ void tr_setup(SmemTraj& t, uint64_t* base) {
  t.w = Warp3{base, base + kMaxWindow, base + 2 * kMaxWindow};
}
__device__ __forceinline__ void tr_setup(RegTraj& t, uint64_t* base) {
  t.ring = base;
  t.S = base + kRing;
}

// Run the trajectory from (∅, j) through its first general round until L is
// empty again (returns true, j = ∅-point) or no full round fits (false).
// Steady stretches are reported to `stretch(j0, c, rounds)`, general rounds
// emit through `emit`; r counts rounds.
template <class T, class Emit, class Stretch>
__device__ bool excursion(const FF& f, T& tr, uint32_t& j, uint32_t& r, uint32_t NR, Emit emit, Stretch stretch) {
  for (;;) {
    if (j + (f.C - tr.lc) > NR) return false;
    tr.round(f, j, NR, emit);
    ++r;
    if (tr.lc == 0) return true;
    const uint32_t j0 = j;
    const uint32_t k = ffwd(f, tr.lc, tr.u0(), j, NR);
    if (k) stretch(j0, f.C - tr.lc, k);
    r += k;
  }
}

// ------------------------------------------------------------ 5. excursions
template <class T>
__global__ void __launch_bounds__(128) k_ff_excursion(FF f) {
  __shared__ uint64_t sm[4][3 * kMaxWindow + kRing];
  const uint32_t wl = threadIdx.x >> 5;
  const uint32_t nfail = f.scal[3], NR = f.scal[2];
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nfail; gw += nw) {
    uint32_t j = f.failpos[gw], r = 0;
    T tr;
    tr_setup(tr, sm[wl]);
    tr.init(f, j, NR);
    const bool back = excursion(f, tr, j, r, NR, [](uint64_t, uint32_t) {}, [](uint32_t, uint32_t, uint32_t) {});
    if ((threadIdx.x & 31u) == 0) {
      f.exE[gw] = back ? j : kEnd;
      f.exR[gw] = r;
    }
    __syncwarp();
  }
}

// ∅-run from z: chunks at z + tC while pass; returns (first fail index or kEnd, #chunks)
__device__ void run_from(const FF& f, uint32_t z, uint32_t& fail_idx, uint32_t& nch) {
  const uint32_t NR = f.scal[2], C = f.C, nfail = f.scal[3];
  uint32_t jj = z;
  nch = ffwd(f, 0, __int_as_float(0x7f800000), jj, NR);
  if (jj + C <= NR) {
    uint32_t lo = 0, hi = nfail;  // jj is a failing position
    while (lo < hi) { uint32_t md = (lo + hi) >> 1; if (f.failpos[md] < jj) lo = md + 1; else hi = md; }
    fail_idx = lo;
  } else {
    fail_idx = kEnd;
  }
}

// successor of every node: node i < nfail = failing position; node nfail = start (∅ at 0)
__global__ void __launch_bounds__(128) k_ff_link(FF f) {
  const uint32_t nfail = f.scal[3];
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw <= nfail; gw += nw) {
    uint32_t z, r0;
    if (gw == nfail) { z = 0; r0 = 0; }
    else { z = f.exE[gw]; r0 = f.exR[gw]; }
    uint32_t fi = kEnd, nch = 0;
    if (z != kEnd) run_from(f, z, fi, nch);
    if ((threadIdx.x & 31u) == 0) {
      f.nxt[gw] = fi;
      f.wr[gw] = r0 + nch;
      f.runz[gw] = z;
      f.runn[gw] = nch;
    }
  }
}

// all doubling levels in one cooperative launch; stops once 2^(k-1) >= nodes
// (every path is shorter), the number of levels built goes to scal[5]
__global__ void __launch_bounds__(256) k_ff_double_all(FF f) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const uint32_t nn = f.scal[3] + 1;
  uint32_t k = 1;
  for (; k < f.levels && (1ull << (k - 1)) < nn; ++k) {
    const uint32_t* n0 = f.nxt + (size_t)(k - 1) * nn;
    const uint32_t* w0 = f.wr + (size_t)(k - 1) * nn;
    uint32_t* n1 = f.nxt + (size_t)k * nn;
    uint32_t* w1 = f.wr + (size_t)k * nn;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
      const uint32_t a = n0[i];
      if (a == kEnd) { n1[i] = kEnd; w1[i] = w0[i]; }
      else { n1[i] = n0[a]; w1[i] = w0[i] + w0[a]; }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) f.scal[5] = k;
}

// expand the path from the start node (levels high -> low), one CTA; also
// emits one stretch descriptor per path node for its ∅-run
__global__ void __launch_bounds__(1024) k_ff_expand(FF f) {
  __shared__ uint32_t cnt;
  const uint32_t nn = f.scal[3] + 1;
  if (threadIdx.x == 0) {
    cnt = 1;
    f.path_node[0] = nn - 1;
    f.path_off[0] = 0;
  }
  __syncthreads();
  for (int k = (int)min(f.levels, f.scal[5]) - 1; k >= 0; --k) {
    const uint32_t cur = cnt;
    __syncthreads();
    const uint32_t* nk = f.nxt + (size_t)k * nn;
    const uint32_t* wk = f.wr + (size_t)k * nn;
    for (uint32_t i = threadIdx.x; i < cur; i += blockDim.x) {
      const uint32_t x = f.path_node[i];
      const uint32_t y = nk[x];
      if (y != kEnd) {
        const uint32_t slot = atomicAdd(&cnt, 1u);
        f.path_node[slot] = y;
        f.path_off[slot] = f.path_off[i] + wk[x];
      }
    }
    __syncthreads();
  }
  const uint32_t np = cnt;
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
    const uint32_t x = f.path_node[i];
    if (f.runz[x] != kEnd && f.runn[x]) {
      const uint32_t d = atomicAdd(&f.scal[7], 1u);
      f.ds_j[d] = f.runz[x];
      f.ds_c[d] = f.C;
      f.ds_r[d] = f.runn[x];
      f.ds_b[d] = f.path_off[i] + (x == nn - 1 ? 0u : f.exR[x]);
    }
  }
  if (threadIdx.x == 0) f.scal[6] = np;
}

// re-run every path excursion: general rounds emit, steady stretches -> descriptors
template <class T>
__global__ void __launch_bounds__(128) k_ff_emit_exc(FF f) {
  __shared__ uint64_t sm[4][3 * kMaxWindow + kRing];
  const uint32_t wl = threadIdx.x >> 5;
  const uint32_t np = f.scal[6], nfail = f.scal[3], NR = f.scal[2];
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < np; gw += nw) {
    const uint32_t x = f.path_node[gw];
    if (x == nfail) continue;  // start node: no excursion
    uint32_t j = f.failpos[x], r = 0;
    const uint32_t b0 = f.path_off[gw];
    T tr;
    tr_setup(tr, sm[wl]);
    tr.init(f, j, NR);
    excursion(f, tr, j, r, NR, [&](uint64_t e, uint32_t slot) { put(f, e, b0 + r, slot); },
              [&](uint32_t j0, uint32_t c, uint32_t k) {
                if (lane == 0) {
                  const uint32_t d = atomicAdd(&f.scal[7], 1u);
                  f.ds_j[d] = j0; f.ds_c[d] = c; f.ds_r[d] = k; f.ds_b[d] = b0 + r;
                }
              });
    __syncwarp();
  }
}

// tail: rebuild the path end state, finish with partial windows
__global__ void __launch_bounds__(32) k_ff_tail(FF f) {
  __shared__ uint64_t L[2 * kMaxWindow], A[2 * kMaxWindow], S[2 * kMaxWindow];
  __shared__ uint32_t s_last, s_off;
  const uint32_t lane = threadIdx.x;
  const uint32_t NR = f.scal[2], nfail = f.scal[3], np = f.scal[6], G = f.scal[1];
  if (lane == 0) {
    s_last = kEnd;
    s_off = 0;
  }
  __syncwarp();
  for (uint32_t i = lane; i < np; i += 32) {
    const uint32_t x = f.path_node[i];
    if (f.nxt[x] == kEnd) { s_last = x; s_off = f.path_off[i]; }
  }
  __syncwarp();
  uint32_t lc = 0, j = 0, b = 0;
  const uint32_t x = s_last;
  if (G > f.K && x != kEnd) {
    const uint32_t ex_end = (x == nfail) ? 0u : f.exE[x];
    if (x != nfail && ex_end == kEnd) {
      // the path's last excursion reaches the stream end: replay it for (L, j)
      SmemTraj tr;
      tr.w = Warp3{L, A, S};
      j = f.failpos[x];
      tr.init(f, j, NR);
      uint32_t r = 0;
      excursion(f, tr, j, r, NR, [](uint64_t, uint32_t) {}, [](uint32_t, uint32_t, uint32_t) {});
      lc = tr.lc;
      b = s_off + r;
    } else {
      b = s_off + f.wr[x];  // excursion + ∅-run rounds (level 0)
      j = f.runz[x] + f.runn[x] * f.C;
      lc = 0;
    }
  }
  // remaining: L ∪ Rseq[j, NR) ∪ final heap
  for (uint32_t i = lane; i < NR - j; i += 32) A[lc + i] = f.rseq[j + i];
  for (uint32_t i = lane; i < lc; i += 32) A[i] = L[i];
  uint32_t na = lc + (NR - j);
  __syncwarp();
  const uint32_t nh = min(f.K, G);
  for (uint32_t i = lane; i < nh; i += 32) A[na + i] = f.hfinal[i];
  na += nh;
  __syncwarp();
  while (na) {
    for (uint32_t i = lane; i < na; i += 32) {
      const uint64_t v = A[i];
      uint32_t pos = 0;
      for (uint32_t q = 0; q < na; ++q) pos += A[q] < v;
      S[pos] = v;
    }
    __syncwarp();
    const uint32_t lim = min(f.C, na);
    uint32_t cnt = lim;
    for (uint32_t base = 1; base < lim; base += 32) {
      const uint32_t i = base + lane;
      const bool bad = i < lim && ratio_bad(S[i - 1], S[i], f.lambda);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
      if (bal) { cnt = base + __ffs(bal) - 1; break; }
    }
    for (uint32_t i = lane; i < cnt; i += 32) put(f, S[i], b, i);
    for (uint32_t i = lane; i < na - cnt; i += 32) A[i] = S[cnt + i];
    na -= cnt;
    ++b;
    __syncwarp();
  }
  if (lane == 0) *f.seg_count_q = b;
}

// exclusive prefix of descriptor element counts (one CTA); total -> scal[4]
__global__ void __launch_bounds__(1024) k_ff_dscan(FF f) {
  __shared__ uint32_t part[1024];
  const uint32_t nd = f.scal[7];
  const uint32_t per = (nd + 1023) / 1024;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, nd);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += f.ds_r[i] * f.ds_c[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    uint32_t v = threadIdx.x >= (uint32_t)d ? part[threadIdx.x - d] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (uint32_t i = lo; i < hi; ++i) {
    f.ds_pre[i] = run;
    run += f.ds_r[i] * f.ds_c[i];
  }
  if (threadIdx.x == 1023) f.scal[4] = part[1023];
}

// emit every element of every steady stretch / ∅-run (thread per element)
__global__ void k_ff_emit_stretch(FF f) {
  const uint32_t nd = f.scal[7], T = f.scal[4];
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < T; g += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nd;  // last descriptor with ds_pre <= g
    while (lo < hi) { uint32_t md = (lo + hi) >> 1; if (f.ds_pre[md] <= g) lo = md + 1; else hi = md; }
    const uint32_t d = lo - 1;
    const uint32_t c = f.ds_c[d], idx = g - f.ds_pre[d];
    const uint32_t t = idx / c, i = idx % c;
    const uint32_t s0 = f.ds_j[d] + t * c;
    const uint64_t x = f.rseq[s0 + i];
    uint32_t slot = 0;
    for (uint32_t b = 0; b < c; ++b) slot += f.rseq[s0 + b] < x;
    put(f, x, f.ds_b[d] + t, slot);
  }
}

// scatter the per-position results to global element indices
__global__ void k_ff_scatter(FF f) {
  const uint32_t G = f.scal[1];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < G; p += gridDim.x * blockDim.x) {
    const uint32_t g = f.gperm[p];
    f.batch_of[g] = f.batch_p[p];
    f.slot_of[g] = f.slot_p[p];
    f.core_of[g] = 0xFF;
  }
}

}  // namespace

// ------------------------------------------------------------ host side
size_t ff_workspace(uint32_t n, uint32_t levels, uint32_t C) {
  const size_t nc1 = (n + B1 - 1) / B1 + 1;
  size_t s = 0;
  auto add = [&](size_t bytes) { s += (bytes + 255) & ~size_t(255); };
  add(64);                       // scal
  add((size_t)n * 8);            // kk
  add((size_t)n * 8);            // rseq
  add(nc1 * KS * 8 * 3);         // summ, heapH, loc
  add(KS * 8);                   // hfinal
  add(((size_t)n / 32 + 2) * 4); // passbm
  add((size_t)n * 4 * 3);        // failpos, exE, exR
  add((size_t)(n + 1) * 4 * levels * 2);  // nxt, wr
  add((size_t)(n + 1) * 4 * 2);  // runz, runn
  add((size_t)(n + 1) * 4 * 2);  // path_node, path_off
  add((size_t)(n + 1) * 4 * 3);  // run_z, run_n, run_b
  add(((size_t)n / 256 + 2) * 4);  // fail block sums
  add((size_t)n * 5);              // batch_p, slot_p
  add((size_t)n * 4 * C);          // vt
  add((size_t)(n + 1) * 4 * 5);    // descriptors
  return s;
}

uint32_t ff_levels(uint32_t n) {
  uint32_t l = 1;
  while ((1ull << l) < (uint64_t)n + 2) ++l;
  return l + 1;
}

static cudaError_t launch_ff(const SchedLaunch& a, uint32_t q, uint32_t lo, uint32_t hi, const uint32_t* gperm,
                             const uint32_t* ncpu_dev, void* ws, cudaStream_t s) {
  const uint32_t n = hi - lo;
  const uint32_t levels = ff_levels(n);
  FF f{};
  f.perm = a.perm + lo;
  f.gperm = gperm;
  f.ncpu_dev = ncpu_dev;
  f.u = a.u;
  f.key = a.key;
  f.n = n;
  f.C = (uint32_t)a.prof.C;
  f.m = (uint32_t)a.prof.b10 * f.C / 10u;
  f.K = f.m - f.C;
  f.lambda = a.prof.lambda;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  const size_t nc1 = (n + B1 - 1) / B1 + 1;
  f.scal = reinterpret_cast<uint32_t*>(take(64));
  f.kk = reinterpret_cast<uint64_t*>(take((size_t)n * 8));
  f.rseq = reinterpret_cast<uint64_t*>(take((size_t)n * 8));
  f.summ = reinterpret_cast<uint64_t*>(take(nc1 * KS * 8 * 3));
  f.heapH = f.summ + nc1 * KS;
  uint64_t* loc = f.summ + 2 * nc1 * KS;
  f.hfinal = reinterpret_cast<uint64_t*>(take(KS * 8));
  f.passbm = reinterpret_cast<uint32_t*>(take(((size_t)n / 32 + 2) * 4));
  f.failpos = reinterpret_cast<uint32_t*>(take((size_t)n * 4 * 3));
  f.exE = f.failpos + n;
  f.exR = f.failpos + 2 * (size_t)n;
  f.nxt = reinterpret_cast<uint32_t*>(take((size_t)(n + 1) * 4 * levels * 2));
  f.wr = f.nxt + (size_t)(n + 1) * levels;
  f.runz = reinterpret_cast<uint32_t*>(take((size_t)(n + 1) * 4 * 2));
  f.runn = f.runz + (n + 1);
  f.path_node = reinterpret_cast<uint32_t*>(take((size_t)(n + 1) * 4 * 2));
  f.path_off = f.path_node + (n + 1);
  f.run_z = reinterpret_cast<uint32_t*>(take((size_t)(n + 1) * 4 * 3));
  f.run_n = f.run_z + (n + 1);
  f.run_b = f.run_z + 2 * (size_t)(n + 1);
  uint32_t* blocksum = reinterpret_cast<uint32_t*>(take(((size_t)n / 256 + 2) * 4));
  f.batch_p = reinterpret_cast<uint32_t*>(take((size_t)n * 5));
  f.slot_p = reinterpret_cast<uint8_t*>(f.batch_p + n);
  f.vt = reinterpret_cast<float*>(take((size_t)n * 4 * f.C));
  f.vstride = n;
  f.ds_j = reinterpret_cast<uint32_t*>(take((size_t)(n + 1) * 4 * 5));
  f.ds_c = f.ds_j + (n + 1);
  f.ds_r = f.ds_j + 2 * (size_t)(n + 1);
  f.ds_b = f.ds_j + 3 * (size_t)(n + 1);
  f.ds_pre = f.ds_j + 4 * (size_t)(n + 1);
  f.levels = levels;
  f.batch_of = a.batch_of;
  f.slot_of = a.slot_of;
  f.core_of = a.core_of;
  f.seg_count_q = a.seg_count + q;

  cudaMemsetAsync(f.scal, 0, 64, s);
  const uint32_t g1 = (n + 255) / 256;
  k_ff_gather<<<g1, 256, 0, s>>>(f);
  note_launch();
  if (f.K == 0) {
    k_ff_copy<<<g1, 256, 0, s>>>(f);
    note_launch();
  } else {
    const uint32_t nc = (n + B1 - 1) / B1;
    if (f.K <= 32) {
      k_ff_topk32<<<(nc * 32 + 255) / 256, 256, 0, s>>>(f);
      k_ff_scan32<<<1, 1024, 0, s>>>(f, loc);
    } else {
      k_ff_topk<<<nc, 256, 0, s>>>(f);
      const int scan_smem = 32 * 3 * KS * 8;
      cudaFuncSetAttribute(k_ff_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, scan_smem);
      k_ff_scan<<<1, 1024, scan_smem, s>>>(f, loc);
    }
    const uint32_t rg = (nc * 32 + 127) / 128;
    if (f.K <= 32) k_ff_replay<1><<<rg, 128, 0, s>>>(f);
    else if (f.K <= 64) k_ff_replay<2><<<rg, 128, 0, s>>>(f);
    else k_ff_replay<4><<<rg, 128, 0, s>>>(f);
    note_launch(3);
  }
  const uint32_t npass = ((n + 31) / 32 + 1) * 32;
  if (f.C == 11) k_ff_vtab_t<11><<<(npass + 255) / 256, 256, 0, s>>>(f);
  else if (f.C == 33) k_ff_vtab_t<33><<<(npass + 255) / 256, 256, 0, s>>>(f);
  else k_ff_vtab<<<(npass + 255) / 256, 256, 0, s>>>(f);
  const uint32_t fb = (n + 255) / 256;
  k_ff_failcount<<<fb, 256, 0, s>>>(f, blocksum);
  k_ff_blockscan<<<1, 1024, 0, s>>>(blocksum, fb, f.scal + 3);
  k_ff_failwrite<<<fb, 256, 0, s>>>(f, blocksum);
  // persistent warps (the work counts live on the device; typically a few thousand)
  const uint32_t gw = std::min<uint32_t>(((n + 1) * 32 + 127) / 128, (uint32_t)a.num_sms * 8u);
  if (f.C <= 32) k_ff_excursion<RegTraj><<<gw, 128, 0, s>>>(f);
  else k_ff_excursion<SmemTraj><<<gw, 128, 0, s>>>(f);
  k_ff_link<<<gw, 128, 0, s>>>(f);
  note_launch(6);
  {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ff_double_all, 256, 0);
    // few CTAs: a level is one pass over the nfail + 1 nodes (typically a few
    // thousand), so a full grid would hold every SM through 13 grid barriers
    const uint32_t gd = std::min<uint32_t>({(n + 256) / 256, (uint32_t)(a.num_sms * std::max(1, std::min(per_sm, 4))), 16u});
    void* args[] = {&f};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_ff_double_all, dim3(gd), dim3(256), args, 0, s);
    if (e != cudaSuccess) return e;
    note_launch();
  }
  k_ff_expand<<<1, 1024, 0, s>>>(f);
  if (f.C <= 32) k_ff_emit_exc<RegTraj><<<gw, 128, 0, s>>>(f);
  else k_ff_emit_exc<SmemTraj><<<gw, 128, 0, s>>>(f);
  k_ff_tail<<<1, 32, 0, s>>>(f);
  k_ff_dscan<<<1, 1024, 0, s>>>(f);
  k_ff_emit_stretch<<<1184, 256, 0, s>>>(f);
  k_ff_scatter<<<g1, 256, 0, s>>>(f);
  note_launch(6);
  return cudaGetLastError();
}

// ------------------------------------------------------------ one large queue
size_t big_queue_workspace(uint32_t n, uint32_t C) {
  const size_t split = (((size_t)n / 256 + 2) * 4 + 64 + (size_t)n * 12 * 2 + (size_t)n * 4 + 8 * 256);
  const size_t sortw = radix_sort_workspace(n);
  size_t ffw = ff_workspace(n, ff_levels(n), C);
  return split + std::max(sortw, cpu_big_workspace(n)) + (ffw > sortw ? ffw : sortw) + 5 * 256;
}

cudaError_t launch_big_queue(const SchedLaunch& a, uint32_t q, uint32_t lo, uint32_t hi, int full64, void* ws,
                             cudaStream_t s, cudaStream_t aux, cudaEvent_t ev_fork, cudaEvent_t ev_join) {
  const uint32_t n = hi - lo;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  uint32_t* bsum = reinterpret_cast<uint32_t*>(take(((size_t)n / 256 + 2) * 4));
  uint32_t* counts = reinterpret_cast<uint32_t*>(take(64));  // [0] CPU class, [1] GPU class
  uint64_t* ck = reinterpret_cast<uint64_t*>(take((size_t)n * 8));
  uint32_t* cv = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
  uint64_t* gk = reinterpret_cast<uint64_t*>(take((size_t)n * 8));
  uint32_t* gv = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
  uint32_t* gperm = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
  void* cpu_ws = take(std::max(radix_sort_workspace(n), cpu_big_workspace(n)));
  void* main_ws = p;  // GPU-class sort, then the consolidation pipeline
  cudaError_t e = split_by_class(a.key + lo, lo, n, bsum, counts, ck, cv, gk, gv, s);
  if (e != cudaSuccess) return e;
  // CPU class: sort + list scheduling on the forked stream
  cudaEventRecord(ev_fork, s);
  cudaStreamWaitEvent(aux, ev_fork, 0);
  e = radix_sort_desc2(ck, cv, 0, n, counts + 0, a.perm + lo, full64, cpu_ws, aux);
  if (e != cudaSuccess) return e;
  e = launch_cpu_big(a, lo, n, counts + 0, cpu_ws, aux);  // the CPU-class sort is done with cpu_ws
  if (e != cudaSuccess) return e;
  cudaEventRecord(ev_join, aux);
  // GPU class: sort + parallel consolidation on the caller's stream
  e = radix_sort_desc2(gk, gv, 0, n, counts + 1, gperm, full64, main_ws, s);
  if (e != cudaSuccess) return e;
  e = launch_ff(a, q, lo, hi, gperm, counts + 0, main_ws, s);
  if (e != cudaSuccess) return e;
  cudaStreamWaitEvent(s, ev_join, 0);
  return cudaGetLastError();
}

}  // namespace rtlm
