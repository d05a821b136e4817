// k_sched.cu — K4: one-pass schedule of priority queues (§8(a) rows a5-a6).
//
// Alg. 1 online part: pop tasks in descending priority; u > tau
// goes to the CPU batch (one task per CPU slot; core by list scheduling on
// the predicted latency, R-CORE); the rest fill a window of m = floor(b*C)
// tasks which is sorted by ascending u, cut at the first ratio > lambda or at
// C (R-CONS), emitted as one GPU batch, and the remainder carried back with
// its priority (R-CARRY); partial windows at the end are consolidated the same
// way (R-FLUSH).
//
// Small queues (<= kSmallSeg): one CTA per queue sorts the keys in shared
// memory (bitonic), then warp 0 does the CPU list scheduling while warp 1 runs
// the consolidation rounds (the two classes are independent).  Large queues:
// device radix sort (k_sort.cu), a gather of u in priority order, then the
// same two warps over global memory.
#include "internal.cuh"

namespace rtlm {
namespace {

constexpr int kSmallThreads = 128;

// -------------------------------------------------------------- CPU class
// List scheduling in key order (R-CORE): each task goes to the core with the
// smallest predicted free time (ties -> lowest index); predicted latency
// gamma * (base + ceil(eta * u)) with eta*u one binary32 product.  Run by one
// lane with the core clocks in registers.
template <int MAXC, class GetU, class GetIdx>
__device__ void cpu_list_schedule(uint32_t j0, uint32_t j1, uint32_t cores, const rt_profile& p, GetU get_u,
                                  GetIdx get_idx, uint32_t* batch_of, uint8_t* slot_of, uint8_t* core_of) {
  int64_t fr[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) fr[c] = 0;
  const float eta = __ll2float_rn(p.eta_us);
  for (uint32_t j = j0; j < j1; ++j) {
    const uint32_t i = get_idx(j);
    const float eu = __fmul_rn(eta, get_u(j));
    const int64_t pred = (int64_t)p.gamma * (p.base_us + (int64_t)ceilf(eu));
    int best = 0;
    int64_t bv = fr[0];
#pragma unroll
    for (int c = 1; c < MAXC; ++c)
      if (c < (int)cores && fr[c] < bv) { bv = fr[c]; best = c; }
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c == best) fr[c] += pred;
    core_of[i] = (uint8_t)best;
    batch_of[i] = kNoBatch;
    slot_of[i] = 0;
  }
}

template <class GetU, class GetIdx>
__device__ void cpu_class(uint32_t j0, uint32_t j1, uint32_t cores, const rt_profile& p, GetU get_u, GetIdx get_idx,
                          uint32_t* batch_of, uint8_t* slot_of, uint8_t* core_of) {
  if (cores == 0) {
    for (uint32_t j = j0; j < j1; ++j) {
      uint32_t i = get_idx(j);
      core_of[i] = 0xFF; batch_of[i] = kNoBatch; slot_of[i] = 0;
    }
  } else if (cores <= 4) {
    cpu_list_schedule<4>(j0, j1, cores, p, get_u, get_idx, batch_of, slot_of, core_of);
  } else if (cores <= 8) {
    cpu_list_schedule<8>(j0, j1, cores, p, get_u, get_idx, batch_of, slot_of, core_of);
  } else {
    cpu_list_schedule<32>(j0, j1, cores, p, get_u, get_idx, batch_of, slot_of, core_of);
  }
}

// -------------------------------------------------------------- GPU class
// One warp runs the O6 rounds over stream positions [j0, j1) (positions are
// priority ranks).  W/Wu: window (unsorted); S/Su: sorted window.  Returns the
// number of GPU batches.
template <class GetU, class GetIdx>
__device__ uint32_t consolidate_warp(uint32_t j0, uint32_t j1, uint32_t m, uint32_t C, float lambda, GetU get_u,
                                     GetIdx get_idx, uint32_t* W, float* Wu, uint32_t* S, float* Su,
                                     uint32_t* batch_of, uint8_t* slot_of, uint8_t* core_of) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t wl = 0, ptr = j0, b = 0;
  for (;;) {
    const uint32_t take = min(m - wl, j1 - ptr);
    for (uint32_t t = lane; t < take; t += 32) {
      W[wl + t] = ptr + t;
      Wu[wl + t] = get_u(ptr + t);
    }
    wl += take;
    ptr += take;
    __syncwarp();
    if (wl == 0) break;
    // sort the window by (u asc, priority rank asc) -- rank by counting
    for (uint32_t e = lane; e < wl; e += 32) {
      const float ue = Wu[e];
      const uint32_t je = W[e];
      uint32_t pos = 0;
      for (uint32_t x = 0; x < wl; ++x) {
        const float ux = Wu[x];
        pos += (ux < ue) || (ux == ue && W[x] < je);
      }
      S[pos] = je;
      Su[pos] = ue;
    }
    __syncwarp();
    // lambda chain (R-CONS): first element always accepted
    const uint32_t lim = min(C, wl);
    uint32_t cnt = lim;
    for (uint32_t base = 1; base < lim; base += 32) {
      const uint32_t i = base + lane;
      const bool bad = i < lim && !(Su[i] <= __fmul_rn(lambda, Su[i - 1]));
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
      if (bal) {
        cnt = base + __ffs(bal) - 1;
        break;
      }
    }
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t g = get_idx(S[i]);
      batch_of[g] = b;
      slot_of[g] = (uint8_t)i;
      core_of[g] = 0xFF;
    }
    const uint32_t rem = wl - cnt;
    for (uint32_t t = lane; t < rem; t += 32) {
      W[t] = S[cnt + t];
      Wu[t] = Su[cnt + t];
    }
    wl = rem;
    ++b;
    __syncwarp();
  }
  return b;
}

__device__ __forceinline__ bool before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kSmallThreads) k_sched_small(SchedLaunch a) {
  __shared__ uint64_t s_key[kSmallSeg];
  __shared__ uint16_t s_idx[kSmallSeg];
  __shared__ float s_u[kSmallSeg];
  __shared__ uint32_t W[kMaxWindow], S[kMaxWindow];
  __shared__ float Wu[kMaxWindow], Su[kMaxWindow];
  __shared__ uint32_t s_ncpu;
  const uint32_t q = blockIdx.x;
  const uint32_t lo = a.seg_off[q], hi = a.seg_off[q + 1], n = hi - lo;
  if (n > kSmallSeg) return;  // large queue: separate path
  if (n == 0) {
    if (threadIdx.x == 0) a.seg_count[q] = 0;
    return;
  }
  uint32_t npow = 1;
  while (npow < n) npow <<= 1;
  if (threadIdx.x == 0) s_ncpu = 0;
  for (uint32_t i = threadIdx.x; i < npow; i += kSmallThreads) {
    s_key[i] = i < n ? a.key[lo + i] : 0ull;
    s_idx[i] = i < n ? (uint16_t)i : (uint16_t)0xFFFF;
  }
  __syncthreads();
  // bitonic sort by (key desc, index asc)
  for (uint32_t k = 2; k <= npow; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < npow; i += kSmallThreads) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint64_t ki = s_key[i], kl = s_key[l];
          const uint32_t ii = s_idx[i], il = s_idx[l];
          const bool up = (i & k) == 0;
          const bool sw = up ? before(kl, il, ki, ii) : before(ki, ii, kl, il);
          if (sw) {
            s_key[i] = kl; s_key[l] = ki;
            s_idx[i] = (uint16_t)il; s_idx[l] = (uint16_t)ii;
          }
        }
      }
      __syncthreads();
    }
  }
  uint32_t ncpu_local = 0;
  for (uint32_t j = threadIdx.x; j < n; j += kSmallThreads) {
    const uint32_t i = s_idx[j];
    a.perm[lo + j] = lo + i;
    s_u[j] = a.u[lo + i];
    ncpu_local += (uint32_t)(s_key[j] >> 63);
  }
  if (ncpu_local) atomicAdd(&s_ncpu, ncpu_local);
  __syncthreads();
  const uint32_t ncpu = s_ncpu;
  const uint32_t warp = threadIdx.x >> 5;
  auto get_u = [&](uint32_t j) { return s_u[j]; };
  auto get_idx = [&](uint32_t j) { return lo + (uint32_t)s_idx[j]; };
  if (warp == 0) {
    if ((threadIdx.x & 31u) == 0)
      cpu_class(0, ncpu, a.cores, a.prof, get_u, get_idx, a.batch_of, a.slot_of, a.core_of);
  } else if (warp == 1) {
    const uint32_t m = (uint32_t)a.prof.b10 * (uint32_t)a.prof.C / 10u;
    uint32_t nb = consolidate_warp(ncpu, n, m, (uint32_t)a.prof.C, a.prof.lambda, get_u, get_idx, W, Wu, S, Su,
                                   a.batch_of, a.slot_of, a.core_of);
    if ((threadIdx.x & 31u) == 0) a.seg_count[q] = nb;
  }
}

// CPU class of a large queue (R-CORE), in three launches:
//  k_cpu_pred   (grid)  predicted latency of the j-th CPU task in priority
//                       order, p_j = gamma * (base + ceil(eta * u)); batch/slot
//                       outputs; per-chunk maxima of p;
//  k_cpu_chain  (1 CTA) the list-scheduling recurrence, one thread, chunks of
//                       the p stream staged in shared memory by cp.async;
//  k_cpu_scatter(grid)  core_of[perm[j]] = chosen core.
// State: the core clocks as keys (t << 5 | core) kept sorted, so the
// earliest-free core with the lowest index is key[0] and a job is an add plus
// a sorted insert of key[0] + (p << 5) (exact while t < 2^58 µs).  When the
// spread of the keys and every p of a chunk are < 2^32 (checked per chunk)
// the keys are kept as u32 offsets from a 64-bit base.
constexpr uint32_t kCpuChunk = 4096;
constexpr uint32_t kPredBlock = 1024;  // k_cpu_pred elements per CTA (max of p per CTA)

__global__ void __launch_bounds__(256) k_cpu_pred(SchedLaunch a, uint32_t lo, const uint32_t* __restrict__ ncpu_p,
                                                  uint64_t* __restrict__ pred, uint64_t* __restrict__ chunk_max) {
  __shared__ uint64_t wmax[8];
  const uint32_t ncpu = *ncpu_p;
  const uint32_t j0 = blockIdx.x * kPredBlock;
  if (j0 >= ncpu) return;
  const uint32_t* perm = a.perm + lo;
  const float eta = __ll2float_rn(a.prof.eta_us);
  uint64_t mx = 0;
#pragma unroll
  for (uint32_t k = 0; k < kPredBlock / 256; ++k) {
    const uint32_t j = j0 + k * 256 + threadIdx.x;
    if (j < ncpu) {
      const uint32_t i = perm[j];
      const float eu = __fmul_rn(eta, a.u[i]);
      const uint64_t pr = (uint64_t)((int64_t)a.prof.gamma * (a.prof.base_us + (int64_t)ceilf(eu)));
      pred[j] = pr;
      mx = max(mx, pr);
      a.batch_of[i] = kNoBatch;
      a.slot_of[i] = 0;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if ((threadIdx.x & 31u) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < 8; ++w) t = max(t, wmax[w]);
    chunk_max[blockIdx.x] = t;
  }
}

// one chunk on u32 offsets from the smallest key: d1 <= d2 <= d3 relative to
// base = key[0]; a job inserts p into (d1, d2, d3) by min/max and rebases by
// the new minimum, so every offset stays <= max(spread, max p) < 2^32.
__device__ __forceinline__ void chain4_u32(uint64_t& base, uint32_t& d1, uint32_t& d2, uint32_t& d3,
                                           const uint64_t* __restrict__ p, uint8_t* __restrict__ out, uint32_t cnt) {
  uint32_t q = 0;
  for (; q + 8 <= cnt; q += 8) {
    uint32_t v[8];
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      const uint4 w = *reinterpret_cast<const uint4*>(p + q + t);
      v[t] = w.x << 5;
      v[t + 1] = w.z << 5;
    }
    uint32_t o0 = 0, o1 = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      // low byte of the key = core index (bits 0-4) + clock bits, masked later
      const uint32_t lb = (uint32_t)base & 0xFFu;
      if (t < 4) o0 |= lb << (8 * t); else o1 |= lb << (8 * (t - 4));
      const uint32_t x = v[t];
      const uint32_t e0 = min(d1, x), e1 = min(max(d1, x), d2), e2 = min(max(d2, x), d3), e3 = max(d3, x);
      base += e0;
      d1 = e1 - e0; d2 = e2 - e0; d3 = e3 - e0;
    }
    *reinterpret_cast<uint2*>(out + q) = make_uint2(o0, o1);
  }
  for (; q < cnt; ++q) {
    out[q] = (uint8_t)base;
    const uint32_t x = (uint32_t)p[q] << 5;
    const uint32_t e0 = min(d1, x), e1 = min(max(d1, x), d2), e2 = min(max(d2, x), d3), e3 = max(d3, x);
    base += e0;
    d1 = e1 - e0; d2 = e2 - e0; d3 = e3 - e0;
  }
}

// one chunk on absolute u32 clocks a_c = (t_c - t_base) << 2 | core (4 cores):
// a job is w = a0 + (p << 2) and a sorted insert of w into (a1, a2, a3).
// Nearly every job lands on the end of the order (a job outlasts the other
// cores' remaining work), so jobs are taken 4 at a time on the assumption
// that all four append: then job k runs on the core of a_k, w_k = a_k +
// (p_k << 2) and the new state is (w1..w4) -- four independent adds checked
// by w1 > a3, w2 > w1, w3 > w2, w4 > w3.  If the check fails the 4 jobs are
// redone one by one (sorted insert by min/max).  Every 8 jobs the clocks are
// rebased by the minimum; the caller checks (spread + 9 max p) * 4 + 3 < 2^32,
// which bounds every clock between rebases.
__device__ __forceinline__ void insert4(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3, uint32_t x) {
  const uint32_t w = a0 + (x << 2);
  const uint32_t n0 = min(a1, w), n1 = min(max(a1, w), a2), n2 = min(max(a2, w), a3), n3 = max(a3, w);
  a0 = n0; a1 = n1; a2 = n2; a3 = n3;
}

__device__ __forceinline__ void block4(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3, const uint32_t* v,
                                       uint32_t* c) {
  const uint32_t w1 = a0 + (v[0] << 2), w2 = a1 + (v[1] << 2), w3 = a2 + (v[2] << 2), w4 = a3 + (v[3] << 2);
  if ((w1 > a3) & (w2 > w1) & (w3 > w2) & (w4 > w3)) {
    c[0] = a0; c[1] = a1; c[2] = a2; c[3] = a3;
    a0 = w1; a1 = w2; a2 = w3; a3 = w4;
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      c[t] = a0;
      insert4(a0, a1, a2, a3, v[t]);
    }
  }
}

__device__ __forceinline__ void chain4_abs(uint64_t& tb, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3,
                                           const uint64_t* __restrict__ p, uint8_t* __restrict__ out, uint32_t cnt) {
  uint32_t q = 0;
  for (; q + 8 <= cnt; q += 8) {
    uint32_t v[8];
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      const uint4 w = *reinterpret_cast<const uint4*>(p + q + t);
      v[t] = w.x;
      v[t + 1] = w.z;
    }
    uint32_t c[8];
    block4(a0, a1, a2, a3, v, c);
    block4(a0, a1, a2, a3, v + 4, c + 4);
    const uint32_t o0 = __byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410);
    const uint32_t o1 = __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410);
    *reinterpret_cast<uint2*>(out + q) = make_uint2(o0 & 0x03030303u, o1 & 0x03030303u);
    const uint32_t m = a0 & ~3u;
    tb += m >> 2;
    a0 -= m; a1 -= m; a2 -= m; a3 -= m;
  }
  for (; q < cnt; ++q) {
    out[q] = (uint8_t)(a0 & 3u);
    insert4(a0, a1, a2, a3, (uint32_t)p[q]);
  }
}

// one job of list scheduling on the sorted keys: remove k[0], insert k[0] + p
template <int MAXC>
__device__ __forceinline__ void list_step(uint64_t (&k)[MAXC], uint64_t p) {
  const uint64_t v = k[0] + p;
  bool lt[MAXC];
#pragma unroll
  for (int c = 1; c < MAXC; ++c) lt[c] = v < k[c];
  uint64_t nk[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const bool take_next = (c + 1 < MAXC) && !lt[c + 1 < MAXC ? c + 1 : 0];
    const bool keep = (c >= 1) && lt[c >= 1 ? c : 1];
    nk[c] = take_next ? k[c + 1 < MAXC ? c + 1 : c] : (keep ? k[c] : v);
  }
#pragma unroll
  for (int c = 0; c < MAXC; ++c) k[c] = nk[c];
}

template <int MAXC>
__device__ __forceinline__ void chain_u64(uint64_t (&k)[MAXC], const uint64_t* __restrict__ p, uint8_t* __restrict__ out,
                                          uint32_t cnt) {
  for (uint32_t q = 0; q < cnt; ++q) {
    out[q] = (uint8_t)k[0];
    list_step<MAXC>(k, p[q] << 5);
  }
}

// warps 1..3 stage chunk c+1 of p (cp.async) and write out the cores of chunk
// c-1 while lane 0 of warp 0 runs chunk c
template <int MAXC>
__global__ void __launch_bounds__(128) k_cpu_chain(uint32_t cores, const uint32_t* __restrict__ ncpu_p,
                                                   const uint64_t* __restrict__ pred,
                                                   const uint64_t* __restrict__ chunk_max, uint8_t* __restrict__ csel) {
  extern __shared__ __align__(16) uint8_t chain_smem[];
  uint64_t* s_p = reinterpret_cast<uint64_t*>(chain_smem);               // [2][kCpuChunk]
  uint8_t* s_o = chain_smem + 2 * kCpuChunk * sizeof(uint64_t);          // [2][kCpuChunk]
  __shared__ uint64_t s_pm[2];                                            // max p of the staged chunk
  const uint32_t ncpu = *ncpu_p;
  const uint32_t nchunks = (ncpu + kCpuChunk - 1) / kCpuChunk;
  auto stage = [&](uint32_t c, uint32_t t) {  // threads t = 0..95 of warps 1..3
    const uint32_t j0 = c * kCpuChunk, cnt = min(kCpuChunk, ncpu - j0);
    if (t == 0) {
      uint64_t pm = 0;
      for (uint32_t b = j0 / kPredBlock; b * kPredBlock < j0 + cnt; ++b) pm = max(pm, chunk_max[b]);
      s_pm[c & 1] = pm;
    }
    const uint32_t nv = (cnt + 1) / 2;  // 16-byte vectors (pred is padded to even length)
    uint64_t* dst = s_p + (c & 1) * kCpuChunk;
    for (uint32_t v = t; v < nv; v += 96) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + 2 * v);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(pred + j0 + 2 * v) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  };
  auto drain = [&](uint32_t c, uint32_t t, uint32_t nt) {
    const uint32_t j0 = c * kCpuChunk, cnt = min(kCpuChunk, ncpu - j0);
    const uint8_t* src = s_o + (c & 1) * kCpuChunk;
    for (uint32_t q = t; q < cnt; q += nt) csel[j0 + q] = src[q];
  };
  uint64_t k[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) k[c] = c < (int)cores ? (uint64_t)c : ~0ull;  // unused cores never chosen
  if (nchunks && threadIdx.x >= 32) stage(0, threadIdx.x - 32);
  __syncthreads();
  for (uint32_t c = 0; c < nchunks; ++c) {
    if (threadIdx.x == 0) {
      const uint32_t cnt = min(kCpuChunk, ncpu - c * kCpuChunk);
      const uint64_t* pp = s_p + (c & 1) * kCpuChunk;
      uint8_t* oo = s_o + (c & 1) * kCpuChunk;
      const uint64_t pm = s_pm[c & 1];
      const uint64_t spread_t = (k[MAXC - 1] >> 5) - (k[0] >> 5);
      if (MAXC == 4 && cores == 4 && spread_t < (1ull << 28) && pm < (1ull << 28) &&
          ((spread_t + 9 * pm) << 2) + 3 < 0xFFFFFFFFull) {
        uint64_t tb = k[0] >> 5;
        uint32_t a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = (uint32_t)(((k[i % MAXC] >> 5) - tb) << 2) | (uint32_t)(k[i % MAXC] & 3u);
        chain4_abs(tb, a[0], a[1], a[2], a[3], pp, oo, cnt);
#pragma unroll
        for (int i = 0; i < 4; ++i) k[i % MAXC] = ((tb + (a[i] >> 2)) << 5) | (a[i] & 3u);
      } else if (MAXC == 4 && cores == 4 && k[MAXC - 1] - k[0] < 0xFFFFFFFFull && pm < (1ull << 27)) {
        uint64_t base = k[0];
        uint32_t d1 = (uint32_t)(k[1 % MAXC] - base), d2 = (uint32_t)(k[2 % MAXC] - base),
                 d3 = (uint32_t)(k[3 % MAXC] - base);
        chain4_u32(base, d1, d2, d3, pp, oo, cnt);
        k[0] = base;
        k[1 % MAXC] = base + d1;
        k[2 % MAXC] = base + d2;
        k[3 % MAXC] = base + d3;
      } else {
        chain_u64<MAXC>(k, pp, oo, cnt);
      }
    } else if (threadIdx.x >= 32) {
      if (c + 1 < nchunks) stage(c + 1, threadIdx.x - 32);
      if (c >= 1) drain(c - 1, threadIdx.x - 32, 96);
    }
    __syncthreads();
  }
  if (nchunks) drain(nchunks - 1, threadIdx.x, 128);
}

__global__ void k_cpu_scatter(SchedLaunch a, uint32_t lo, const uint32_t* __restrict__ ncpu_p,
                              const uint8_t* __restrict__ csel) {
  const uint32_t ncpu = *ncpu_p;
  const uint32_t* perm = a.perm + lo;
  const bool any = a.cores != 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < ncpu; j += gridDim.x * blockDim.x)
    a.core_of[perm[j]] = any ? (uint8_t)(csel[j] & 31u) : (uint8_t)0xFF;
}

// seg_batch_off = exclusive scan of seg_count (one CTA)
__global__ void __launch_bounds__(1024) k_seg_scan(const uint32_t* __restrict__ cnt, uint32_t nq,
                                                    uint32_t* __restrict__ off) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (nq + 1023) / 1024;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, nq);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += cnt[i];
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
    off[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == 1023) off[nq] = part[1023];
}

// add each queue's first batch id to its local batch ids
__global__ void k_batch_fix(uint32_t* __restrict__ batch_of, const uint32_t* __restrict__ seg_off, uint32_t nq,
                            const uint32_t* __restrict__ seg_batch_off) {
  const uint32_t n = seg_off[nq];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t b = batch_of[i];
    if (b == kNoBatch) continue;
    uint32_t lo = 0, hi = nq;  // find q with seg_off[q] <= i < seg_off[q+1]
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (seg_off[mid] <= i) lo = mid; else hi = mid;
    }
    batch_of[i] = b + seg_batch_off[lo];
  }
}

}  // namespace

cudaError_t launch_sched_small(const SchedLaunch& a, cudaStream_t s) {
  if (!a.nq) return cudaSuccess;
  k_sched_small<<<a.nq, kSmallThreads, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

size_t cpu_big_workspace(uint32_t n) {
  const size_t nch = (size_t)n / kPredBlock + 2;
  return (((size_t)n + 2) * 8 + 255 & ~size_t(255)) + (nch * 8 + 255 & ~size_t(255)) + ((size_t)n + 255 & ~size_t(255));
}

cudaError_t launch_cpu_big(const SchedLaunch& a, uint32_t lo, uint32_t n, const uint32_t* ncpu, void* ws,
                           cudaStream_t s) {
  if (!n) return cudaSuccess;
  char* w = static_cast<char*>(ws);
  uint64_t* pred = reinterpret_cast<uint64_t*>(w);
  w += ((size_t)n + 2) * 8 + 255 & ~size_t(255);
  uint64_t* chunk_max = reinterpret_cast<uint64_t*>(w);
  w += ((size_t)n / kPredBlock + 2) * 8 + 255 & ~size_t(255);
  uint8_t* csel = reinterpret_cast<uint8_t*>(w);
  const uint32_t nch = (n + kPredBlock - 1) / kPredBlock;
  k_cpu_pred<<<nch, 256, 0, s>>>(a, lo, ncpu, pred, chunk_max);
  // the serial chain is latency-bound: ask for (nearly) a whole SM's shared memory so
  // that no other kernel's CTA is co-scheduled on its SM
  const int smem = 200 * 1024;
  if (a.cores <= 4) {
    cudaFuncSetAttribute(k_cpu_chain<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_chain<4><<<1, 128, smem, s>>>(a.cores, ncpu, pred, chunk_max, csel);
  } else if (a.cores <= 8) {
    cudaFuncSetAttribute(k_cpu_chain<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_chain<8><<<1, 128, smem, s>>>(a.cores, ncpu, pred, chunk_max, csel);
  } else {
    cudaFuncSetAttribute(k_cpu_chain<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_chain<32><<<1, 128, smem, s>>>(a.cores, ncpu, pred, chunk_max, csel);
  }
  k_cpu_scatter<<<(n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184, 256, 0, s>>>(a, lo, ncpu, csel);
  note_launch(3);
  return cudaGetLastError();
}

cudaError_t launch_sched_finish(const SchedLaunch& a, cudaStream_t s) {
  k_seg_scan<<<1, 1024, 0, s>>>(a.seg_count, a.nq, a.seg_batch_off);
  note_launch();
  if (a.nq > 1) {
    k_batch_fix<<<1184, 256, 0, s>>>(a.batch_of, a.seg_off, a.nq, a.seg_batch_off);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace rtlm
