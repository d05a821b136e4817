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

// gather u in priority order; count the CPU class (keys are sorted, so the CPU
// class is a prefix)
__global__ void k_gather(const uint32_t* __restrict__ perm, const float* __restrict__ u,
                         const uint64_t* __restrict__ key, uint32_t lo, uint32_t n, float* __restrict__ u_sorted,
                         uint32_t* __restrict__ ncpu) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t i = perm[lo + j];
  u_sorted[j] = u[i];
  const bool cpu = (key[i] >> 63) != 0;
  const bool next_gpu = (j + 1 == n) || ((key[perm[lo + j + 1]] >> 63) == 0);
  if (cpu && next_gpu) *ncpu = j + 1;
}

__global__ void __launch_bounds__(64) k_sched_big(SchedLaunch a, uint32_t q, uint32_t lo, uint32_t n,
                                                   const float* __restrict__ u_sorted,
                                                   const uint32_t* __restrict__ ncpu_p) {
  __shared__ uint32_t W[kMaxWindow], S[kMaxWindow];
  __shared__ float Wu[kMaxWindow], Su[kMaxWindow];
  const uint32_t ncpu = *ncpu_p;
  const uint32_t* perm = a.perm + lo;
  auto get_u = [&](uint32_t j) { return u_sorted[j]; };
  auto get_idx = [&](uint32_t j) { return perm[j]; };
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) {
    if ((threadIdx.x & 31u) == 0)
      cpu_class(0, ncpu, a.cores, a.prof, get_u, get_idx, a.batch_of, a.slot_of, a.core_of);
  } else {
    const uint32_t m = (uint32_t)a.prof.b10 * (uint32_t)a.prof.C / 10u;
    uint32_t nb = consolidate_warp(ncpu, n, m, (uint32_t)a.prof.C, a.prof.lambda, get_u, get_idx, W, Wu, S, Su,
                                   a.batch_of, a.slot_of, a.core_of);
    if ((threadIdx.x & 31u) == 0) a.seg_count[q] = nb;
  }
}

// CPU class of a large queue: predicted latencies computed in parallel into
// shared memory, the list-scheduling recurrence (R-CORE) run by one thread on
// a sorted state, outputs written in parallel.  State: the core clocks as
// keys (t << 5 | core) kept sorted, so the earliest-free core with the lowest
// index is key[0] and a job is an add plus a sorted insert of key[0] + (p << 5)
// (exact while t < 2^58 µs).
constexpr uint32_t kCpuChunk = 4096;

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
__device__ __forceinline__ void cpu_chunk_serial(uint64_t (&k)[MAXC], const int64_t* pred, uint8_t* core,
                                                 uint32_t cnt, bool small) {
  if (small) {
    // keys relative to the smallest one: d_c = k_c - k_0 (u32), base = k_0.
    // A job: insert p into (d1, d2, d3) by min/max, rebase by the new minimum.
    uint64_t base = k[0];
    uint32_t d1 = (uint32_t)(k[1] - base), d2 = (uint32_t)(k[MAXC > 2 ? 2 : 1] - base),
             d3 = (uint32_t)(k[MAXC > 3 ? 3 : 1] - base);
    uint32_t q = 0;
    for (; q + 8 <= cnt; q += 8) {
      uint32_t pp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) pp[t] = (uint32_t)pred[q + t];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        core[q + t] = (uint8_t)(base & 31u);
        const uint32_t v = pp[t];
        const uint32_t e0 = min(d1, v), e1 = min(max(d1, v), d2), e2 = min(max(d2, v), d3), e3 = max(d3, v);
        base += e0;
        d1 = e1 - e0; d2 = e2 - e0; d3 = e3 - e0;
      }
    }
    for (; q < cnt; ++q) {
      core[q] = (uint8_t)(base & 31u);
      const uint32_t v = (uint32_t)pred[q];
      const uint32_t e0 = min(d1, v), e1 = min(max(d1, v), d2), e2 = min(max(d2, v), d3), e3 = max(d3, v);
      base += e0;
      d1 = e1 - e0; d2 = e2 - e0; d3 = e3 - e0;
    }
    k[0] = base;
    k[1] = base + d1;
    if (MAXC > 2) k[MAXC > 2 ? 2 : 1] = base + d2;
    if (MAXC > 3) k[MAXC > 3 ? 3 : 1] = base + d3;
  } else {
    uint32_t q = 0;
    for (; q + 8 <= cnt; q += 8) {
      uint64_t pp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) pp[t] = (uint64_t)pred[q + t];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        core[q + t] = (uint8_t)(k[0] & 31u);
        list_step<MAXC>(k, pp[t]);
      }
    }
    for (; q < cnt; ++q) {
      core[q] = (uint8_t)(k[0] & 31u);
      list_step<MAXC>(k, (uint64_t)pred[q]);
    }
  }
}

// CPU class of a large queue.  Warp 0 (one lane) runs the list-scheduling
// recurrence on chunk c while warps 1..7 compute the predicted latencies of
// chunk c+1 and write the assignments of chunk c-1 (double-buffered).
template <int MAXC>
__global__ void __launch_bounds__(256) k_cpu_big(SchedLaunch a, uint32_t lo, const uint32_t* __restrict__ ncpu_p) {
  extern __shared__ __align__(16) uint8_t cpu_smem[];
  int64_t* s_pred = reinterpret_cast<int64_t*>(cpu_smem);                 // [2][kCpuChunk]
  uint8_t* s_core = cpu_smem + 2 * kCpuChunk * sizeof(int64_t);           // [2][kCpuChunk]
  __shared__ int s_small[2];
  const uint32_t ncpu = *ncpu_p;
  const uint32_t* perm = a.perm + lo;
  const float eta = __ll2float_rn(a.prof.eta_us);
  const uint32_t cores = a.cores;
  const uint32_t nchunks = (ncpu + kCpuChunk - 1) / kCpuChunk;
  auto fill = [&](uint32_t c, uint32_t t0, uint32_t nt) {  // predictions of chunk c by threads t0..t0+nt-1
    const uint32_t j0 = c * kCpuChunk, cnt = min(kCpuChunk, ncpu - j0);
    int64_t* pb = s_pred + (c & 1) * kCpuChunk;
    bool big = false;
    for (uint32_t q = threadIdx.x - t0; q < cnt; q += nt) {
      const float eu = __fmul_rn(eta, a.u[perm[j0 + q]]);
      const int64_t pr = ((int64_t)a.prof.gamma * (a.prof.base_us + (int64_t)ceilf(eu))) << 5;
      pb[q] = pr;
      big |= (uint64_t)pr >= 0xFFFFFFFFull;
    }
    if (big) s_small[c & 1] = 0;
  };
  auto drain = [&](uint32_t c, uint32_t t0, uint32_t nt) {  // write assignments of chunk c
    const uint32_t j0 = c * kCpuChunk, cnt = min(kCpuChunk, ncpu - j0);
    const uint8_t* cb = s_core + (c & 1) * kCpuChunk;
    for (uint32_t q = threadIdx.x - t0; q < cnt; q += nt) {
      const uint32_t i = perm[j0 + q];
      a.core_of[i] = cores ? cb[q] : (uint8_t)0xFF;
      a.batch_of[i] = kNoBatch;
      a.slot_of[i] = 0;
    }
  };
  uint64_t k[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) k[c] = c < (int)cores ? (uint64_t)c : ~0ull;  // unused cores never chosen
  if (threadIdx.x < 2) s_small[threadIdx.x] = (MAXC == 4 && cores == 4) ? 1 : 0;
  __syncthreads();
  if (nchunks) fill(0, 0, 256);
  __syncthreads();
  for (uint32_t c = 0; c < nchunks; ++c) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0 && cores)
        cpu_chunk_serial<MAXC>(k, s_pred + (c & 1) * kCpuChunk, s_core + (c & 1) * kCpuChunk,
                               min(kCpuChunk, ncpu - c * kCpuChunk), s_small[c & 1] != 0);
    } else {
      if (threadIdx.x == 32) s_small[(c + 1) & 1] = (MAXC == 4 && cores == 4) ? 1 : 0;
      asm volatile("bar.sync 1, 224;");
      if (c + 1 < nchunks) fill(c + 1, 32, 224);
      if (c >= 1) drain(c - 1, 32, 224);
    }
    __syncthreads();
  }
  if (nchunks) drain(nchunks - 1, 0, 256);
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

cudaError_t launch_sched_big(const SchedLaunch& a, uint32_t q, uint32_t lo, uint32_t hi, float* ws,
                             cudaStream_t s) {
  const uint32_t n = hi - lo;
  float* u_sorted = ws;
  uint32_t* ncpu = reinterpret_cast<uint32_t*>(ws + ((n + 63) & ~63u));
  cudaMemsetAsync(ncpu, 0, sizeof(uint32_t), s);
  k_gather<<<(n + 255) / 256, 256, 0, s>>>(a.perm, a.u, a.key, lo, n, u_sorted, ncpu);
  k_sched_big<<<1, 64, 0, s>>>(a, q, lo, n, u_sorted, ncpu);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_cpu_big(const SchedLaunch& a, uint32_t lo, uint32_t n, const uint32_t* ncpu, cudaStream_t s) {
  (void)n;
  const int smem = 2 * kCpuChunk * (sizeof(int64_t) + 1);
  if (a.cores <= 4) {
    cudaFuncSetAttribute(k_cpu_big<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_big<4><<<1, 256, smem, s>>>(a, lo, ncpu);
  } else if (a.cores <= 8) {
    cudaFuncSetAttribute(k_cpu_big<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_big<8><<<1, 256, smem, s>>>(a, lo, ncpu);
  } else {
    cudaFuncSetAttribute(k_cpu_big<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_cpu_big<32><<<1, 256, smem, s>>>(a, lo, ncpu);
  }
  note_launch();
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
