// k_replay.cu — K5: discrete-event replay of independent arrival traces
// (§8(a) row a7) and K6: integer statistics reduction (row a8).
//
// One warp (one CTA) per trace of <= 1024 tasks (R-REPLAY; §V-A).
// Priorities are static per task (Eq. 3 depends on d - r, not on the clock,
// P:377), so the trace's keys are sorted once (k_trace_rank, a CTA per trace)
// and every
// "ready" set is a 1024-bit bitmap over key rank, one 32-bit word per lane:
// the top-m ready tasks are the first m set bits (popc + warp scan), the
// highest-key CPU task is the first set bit, and a second bitmap over arrival
// index gives the oldest waiting task for the xi flush (R-XI).  Batches are
// consolidated with the same O6 round as rt_schedule (R-CONS) and timed with
// the latency model R-LAT in int64 microseconds (R-TIME).
#include "internal.cuh"

namespace rtlm {
namespace {

// Arrival times are read from global memory (L1 / L2): 5.7 KB of shared memory
// per trace, so 32 one-warp CTAs (the per-SM maximum) fit on an SM and a
// config-3 launch (4096 traces) runs in one wave on 148 SMs.
struct ReplaySmem {
  uint16_t sidx[kMaxTrace];  // rank -> arrival index
  uint16_t rank[kMaxTrace];  // arrival index -> rank
  uint32_t ready_gpu[32], ready_cpu[32], wait_arr[32];
  int64_t core_free[kMaxCores];
  uint32_t W[kMaxWindow];
  float Su[kMaxWindow];
};  // 5.7 KB: arrival times, u, D and lengths are read from global memory (L1 / L2)

__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Priority order of every trace: stable sort of (key desc, arrival index asc)
// by a bitonic network in shared memory, one CTA per trace; writes the
// arrival index of each rank (u16, kMaxTrace per trace) for k_replay.
// Thread p holds the element at position p (key, arrival index); partners at
// distance j < 32 are exchanged by shuffles, larger distances through shared
// memory (double-buffered, one barrier per step).
constexpr uint32_t kRankThr = kMaxTrace;
__global__ void __launch_bounds__(kRankThr) k_trace_rank(const uint64_t* __restrict__ key,
                                                         const uint32_t* __restrict__ trace_off,
                                                         uint16_t* __restrict__ sidx_out) {
  __shared__ uint64_t sk[2][kMaxTrace];
  __shared__ uint16_t si[2][kMaxTrace];
  const uint32_t t = blockIdx.x, p = threadIdx.x;
  const uint32_t lo = trace_off[t], n = trace_off[t + 1] - lo;
  if (n == 0 || n > kMaxTrace) return;  // long traces: radix sort + k_replay_long
  uint32_t npow = 2;
  while (npow < n) npow <<= 1;
  // padding (positions >= n) sorts last: key 0, index 0xFFFF; threads >= npow
  // only ever pair among themselves
  uint64_t k0 = p < n ? key[lo + p] : 0ull;
  uint32_t i0 = p < n ? p : 0xFFFFu;
  uint32_t buf = 0;
  for (uint32_t k = 2; k <= npow; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      uint64_t k1;
      uint32_t i1;
      if (j >= 32u) {
        sk[buf][p] = k0;
        si[buf][p] = (uint16_t)i0;
        __syncthreads();
        k1 = sk[buf][p ^ j];
        i1 = si[buf][p ^ j];
        buf ^= 1u;
      } else {
        k1 = __shfl_xor_sync(0xFFFFFFFFu, k0, j);
        i1 = __shfl_xor_sync(0xFFFFFFFFu, i0, j);
      }
      // order: key descending, arrival index ascending; the lower position of
      // a pair takes the first element when ((lower & k) == 0), else the later
      const bool mine_first = k0 > k1 || (k0 == k1 && i0 < i1);
      const bool lower = (p & j) == 0;
      const bool want_first = lower == ((p & k) == 0);
      if (mine_first != want_first) {
        k0 = k1;
        i0 = i1;
      }
    }
  }
  if (p < n) sidx_out[(size_t)t * kMaxTrace + p] = (uint16_t)i0;
}

// KCH = 32-element chunks of the largest window of the launch's profiles
// (ceil(max(b10 * C / 10, C) / 32)): the window's per-lane arrays and loops
// are sized for it at compile time
template <uint32_t KCH>
__global__ void __launch_bounds__(32) k_replay(ReplayLaunch a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  ReplaySmem& sm = *reinterpret_cast<ReplaySmem*>(smem_raw);
  const uint32_t lane = threadIdx.x;
  const uint32_t t = blockIdx.x;
  const uint32_t lo = a.trace_off[t], n = a.trace_off[t + 1] - lo;
  if (n > kMaxTrace) return;  // k_replay_long's
  const rt_profile p = a.profiles[a.trace_prof ? a.trace_prof[t] : 0];
  if (n == 0) {
    if (lane == 0) a.stats[t] = rt_trace_stats{0, 0u, 0u};
    return;
  }
  // ---- key rank (sorted by k_trace_rank): rank -> arrival index and back;
  // the CPU class is the ranks [0, ncpu) (class bit on top of the key)
  uint32_t ncpu_l = 0;
  const uint16_t* g_sidx = a.sidx + (size_t)t * kMaxTrace;
  for (uint32_t j = lane; j < n; j += 32) {
    const uint32_t i = g_sidx[j];
    sm.sidx[j] = (uint16_t)i;
    sm.rank[i] = (uint16_t)j;
    ncpu_l += (uint32_t)(a.key[lo + j] >> 63);
  }
  const uint32_t ncpu = __reduce_add_sync(0xFFFFFFFFu, ncpu_l);
  const int64_t* __restrict__ g_r = a.arrival + lo;
  const uint16_t* g_len = a.len + lo;
  const float* g_u = a.u + lo;
  const uint32_t* g_D = a.D + lo;
  sm.ready_gpu[lane] = 0; sm.ready_cpu[lane] = 0; sm.wait_arr[lane] = 0;
  sm.core_free[lane] = 0;
  __syncwarp();

  const uint32_t C = (uint32_t)p.C, m = (uint32_t)p.b10 * C / 10u, cores = (uint32_t)p.cores;
  const int64_t gpu_fixed = p.setup_us + p.base_us;
  int64_t now = __ldg(g_r + (0)), gpu_free = 0;
  uint32_t next = 0, done = 0;
  uint32_t cpu_ready = 0, gpu_ready = 0;  // ready-set sizes (warp-uniform)
  bool have_oldest = false;                // oldest_r = arrival of the oldest waiting GPU-class task
  int64_t cpu_min_free = INT64_MAX;        // min core clock while CPU tasks wait (see below)
  bool cpu_min_valid = false;
  int64_t oldest_r = 0;
  int64_t resp = 0;     // per-lane partial sums
  uint32_t misses = 0;
  const uint32_t lt = (1u << lane) - 1u;
  // the next 32 arrival times, one per lane (index next + lane), reloaded only
  // when `next` advances: events that admit nothing read no arrival times
  int64_t rw = lane < n ? __ldg(g_r + (lane)) : INT64_MAX;
  int64_t next_arr = __shfl_sync(0xFFFFFFFFu, rw, 0);  // arrival time of task `next` (warp-uniform)

  for (;;) {
    // ---- admit arrivals <= now (arrival order is non-decreasing)
    while (next < n) {
      const uint32_t i = next + lane;
      const bool arr = rw <= now;  // rw = INT64_MAX past the end
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, arr);
      if (!bal) break;  // no arrival due (most events)
      const uint32_t cnt = __popc(bal);  // a prefix of ones
      const uint32_t rk = arr ? (uint32_t)sm.rank[i] : 0xFFFFFFFFu;
      const uint32_t cb = __ballot_sync(0xFFFFFFFFu, rk < ncpu);
      const uint32_t nc = __popc(cb);
      if (gpu_ready == 0 && (bal & ~cb)) {  // the first waiting GPU-class task is the oldest
        oldest_r = __shfl_sync(0xFFFFFFFFu, rw, __ffs(bal & ~cb) - 1);
        have_oldest = true;
      }
      cpu_ready += nc;
      gpu_ready += cnt - nc;
      if (arr) {
        if (rk < ncpu) {
          atomicOr(&sm.ready_cpu[rk >> 5], 1u << (rk & 31));
        } else {
          atomicOr(&sm.ready_gpu[rk >> 5], 1u << (rk & 31));
          atomicOr(&sm.wait_arr[i >> 5], 1u << (i & 31));
        }
      }
      if (cnt) {
        next += cnt;
        rw = next + lane < n ? __ldg(g_r + (next + lane)) : INT64_MAX;
        next_arr = __shfl_sync(0xFFFFFFFFu, rw, 0);
      }
      if (cnt < 32) break;
    }
    __syncwarp();
    // ---- CPU cores: highest-key ready CPU task -> lowest-index free core
    bool cpu_started = false;
    while (cpu_ready) {  // the ready bitmap is non-empty: find a free core first
      const uint32_t fm = __ballot_sync(0xFFFFFFFFu, lane < cores && sm.core_free[lane] <= now);
      if (!fm) break;
      const uint32_t wcpu = sm.ready_cpu[lane];
      const uint32_t any = __ballot_sync(0xFFFFFFFFu, wcpu != 0);
      const uint32_t c = __ffs(fm) - 1, wl = __ffs(any) - 1;
      const uint32_t word = __shfl_sync(0xFFFFFFFFu, wcpu, wl);
      const uint32_t rk = wl * 32 + (__ffs(word) - 1);
      const uint32_t i = sm.sidx[rk];
      const int64_t end = now + (int64_t)p.gamma * (p.base_us + p.eta_us * (int64_t)g_len[i]);
      __syncwarp();  // every lane's reads of ready_cpu / core_free before lane 0 updates them
      if (lane == 0) {
        sm.core_free[c] = end;
        sm.ready_cpu[wl] = word & (word - 1u);
        resp += end - __ldg(g_r + (i));
        misses += end > __ldg(g_r + (i)) + (int64_t)g_D[i];
        if (a.end_us) a.end_us[lo + i] = end;
      }
      ++done;
      --cpu_ready;
      cpu_started = true;
      __syncwarp();
    }
    if (cpu_started) cpu_min_valid = false;  // a core clock changed
    // ---- GPU dispatch
    bool waiting = false;
    if (gpu_free <= now) {
      const uint32_t total = gpu_ready;
      if (total) {
        if (!have_oldest) {  // after a dispatch: lowest set bit of the arrival-index bitmap
          const uint32_t aw = sm.wait_arr[lane];
          const uint32_t anyw = __ballot_sync(0xFFFFFFFFu, aw != 0);
          const uint32_t owl = __ffs(anyw) - 1;
          const uint32_t oword = __shfl_sync(0xFFFFFFFFu, aw, owl);
          oldest_r = __ldg(g_r + (owl * 32 + (__ffs(oword) - 1)));
          have_oldest = true;
        }
        const bool flush = (oldest_r <= now - p.xi_us) || next == n;
        const uint32_t full = p.consolidate ? m : C;
        const uint32_t take = total >= full ? full : (flush ? total : 0u);
        if (!take) {
          waiting = true;
        } else {
          // first `take` set bits in rank order -> W
          uint32_t gw = sm.ready_gpu[lane];
          const uint32_t cl = __popc(gw);
          uint32_t excl = cl;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            uint32_t v = __shfl_up_sync(0xFFFFFFFFu, excl, o);
            if (lane >= (uint32_t)o) excl += v;
          }
          excl -= cl;
          if (excl < take) {
            uint32_t k = min(cl, take - excl);
            for (uint32_t e = 0; e < k; ++e) {
              const uint32_t b = __ffs(gw) - 1;
              gw &= gw - 1u;
              sm.W[excl + e] = lane * 32 + b;
            }
          }
          __syncwarp();
          // the window's elements stay on the lanes that loaded them (lane e % 32,
          // slot e / 32): rank, arrival index, u, length, deadline and arrival,
          // all loads issued together; each element learns its position in the
          // (u, rank) order, and the batch is the positions below cnt
          constexpr uint32_t kCh = KCH;
          const uint32_t nch = (take + 31u) >> 5;
          uint32_t re[kCh], pos[kCh], len_e[kCh], D_e[kCh];
          float ue[kCh];
          int64_t r_e[kCh];
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k) {
            const uint32_t e = k * 32u + lane;
            re[k] = 0xFFFFFFFFu; ue[k] = 0.0f; len_e[k] = 0u; D_e[k] = 0u; r_e[k] = 0; pos[k] = 0xFFFFFFFFu;
            if (k < nch && e < take) {
              re[k] = sm.W[e];
              const uint32_t i = sm.sidx[re[k]];
              ue[k] = g_u[i];
              len_e[k] = g_len[i];
              D_e[k] = g_D[i];
              r_e[k] = __ldg(g_r + (i));
              pos[k] = e;
              re[k] |= i << 16;  // rank (low 16 bits) | arrival index (high)
            }
          }
          uint32_t cnt;
          if (p.consolidate) {
            // position in the (u asc, rank asc) order, by shuffles over all elements
#pragma unroll
            for (uint32_t k = 0; k < kCh; ++k) pos[k] = 0u;
            if (kCh == 1 || nch == 1) {  // windows of <= 32 (m = 19 at C = 11)
              const uint32_t r0 = re[0] & 0xFFFFu;
              for (uint32_t x = 0; x < take; ++x) {
                const float ux = __shfl_sync(0xFFFFFFFFu, ue[0], x);
                const uint32_t rx = __shfl_sync(0xFFFFFFFFu, re[0], x) & 0xFFFFu;
                pos[0] += (ux < ue[0]) || (ux == ue[0] && rx < r0);
              }
            } else {
#pragma unroll
              for (uint32_t xk = 0; xk < kCh; ++xk) {
                if (xk < nch) {
                  const uint32_t lim = min(32u, take - xk * 32u);
                  for (uint32_t x = 0; x < lim; ++x) {
                    const float ux = __shfl_sync(0xFFFFFFFFu, ue[xk], x);
                    const uint32_t rx = __shfl_sync(0xFFFFFFFFu, re[xk], x) & 0xFFFFu;
#pragma unroll
                    for (uint32_t k = 0; k < kCh; ++k)
                      pos[k] += (ux < ue[k]) || (ux == ue[k] && rx < (re[k] & 0xFFFFu));
                  }
                }
              }
            }
#pragma unroll
            for (uint32_t k = 0; k < kCh; ++k) {
              const uint32_t e = k * 32u + lane;
              if (k < nch && e < take) sm.Su[pos[k]] = ue[k];
              else pos[k] = 0xFFFFFFFFu;
            }
            __syncwarp();
            const uint32_t lim = min(C, take);
            cnt = lim;
            for (uint32_t base = 1; base < lim; base += 32) {
              const uint32_t ii = base + lane;
              const bool bad = ii < lim && !(sm.Su[ii] <= __fmul_rn(p.lambda, sm.Su[ii - 1]));
              const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
              if (bal) {
                cnt = base + __ffs(bal) - 1;
                break;
              }
            }
          } else {
            cnt = take;
          }
          uint32_t ml = 0;
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k)
            if (pos[k] < cnt) ml = max(ml, len_e[k]);
          ml = __reduce_max_sync(0xFFFFFFFFu, ml);
          const int64_t end = now + gpu_fixed + p.eta_us * (int64_t)ml;
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k) {
            if (pos[k] < cnt) {
              const uint32_t rk = re[k] & 0xFFFFu, i = re[k] >> 16;
              atomicAnd(&sm.ready_gpu[rk >> 5], ~(1u << (rk & 31)));
              atomicAnd(&sm.wait_arr[i >> 5], ~(1u << (i & 31)));
              resp += end - r_e[k];
              misses += end > r_e[k] + (int64_t)D_e[k];
              if (a.end_us) a.end_us[lo + i] = end;
            }
          }
          done += cnt;
          gpu_ready -= cnt;
          have_oldest = false;
          gpu_free = end;
          __syncwarp();
        }
      }
    }
    if (done >= n) break;
    // ---- next event time
    int64_t nxt = INT64_MAX;
    if (next < n) nxt = next_arr;
    if (gpu_free > now) nxt = min(nxt, gpu_free);
    const bool cpu_waiting = cpu_ready != 0;
    if (cpu_waiting) {
      // earliest core clock, recomputed only after a core was given a task: while
      // CPU tasks stay ready every core is busy, so this is the next CPU event
      if (!cpu_min_valid) {
        cpu_min_free = warp_min64(lane < cores ? sm.core_free[lane] : INT64_MAX);
        cpu_min_valid = true;
      }
      nxt = min(nxt, cpu_min_free);
    }
    if (waiting) nxt = min(nxt, oldest_r + p.xi_us);
    if (nxt == INT64_MAX) break;  // unreachable with valid inputs (cores >= 1)
    now = nxt;
    (void)lt;
  }
  const int64_t sr = warp_sum64(resp);
  const uint32_t ms = __reduce_add_sync(0xFFFFFFFFu, misses);
  if (lane == 0) a.stats[t] = rt_trace_stats{sr, n, ms};
}

// ---- K5 for long traces (kMaxTrace < n <= kMaxLongTrace tasks, e.g. the paper's
// full beta = 10..150 ramp, ~11 280 arrivals): the same event loop
// (R-REPLAY) as k_replay, with the ready sets as multi-word bitmaps in shared
// memory plus a summary bitmap of their non-zero words (first set bit = two
// ballots; the top-m ready tasks = a scan over the set summary bits), the rank
// order from a radix sort of the trace's keys (launched per long trace by the
// host, stable: key desc, arrival index asc, R-TIE) and the arrival times, ranks
// and task data read from global memory (L2).  One warp per trace.
constexpr uint32_t kLW = kMaxLongTrace / 32;  // bitmap words
constexpr uint32_t kLS = kLW / 32;            // summary words
enum : uint32_t { BM_GPU = 0, BM_CPU = 1, BM_WAIT = 2 };

struct LongSmem {
  uint32_t bits[3][kLW];  // ready GPU-class (by rank), ready CPU-class (by rank), waiting GPU-class (by arrival)
  uint32_t sums[3][kLS];  // bit (w & 31) of sums[b][w >> 5]: bits[b][w] != 0
  int64_t core_free[kMaxCores];
  uint32_t W[kMaxWindow];
  float Su[kMaxWindow];
};

__device__ __forceinline__ void lbit_set(LongSmem& sm, uint32_t b, uint32_t x) {
  atomicOr(&sm.bits[b][x >> 5], 1u << (x & 31u));
  atomicOr(&sm.sums[b][x >> 10], 1u << ((x >> 5) & 31u));
}
__device__ __forceinline__ void lbit_clear(LongSmem& sm, uint32_t b, uint32_t x) {
  const uint32_t m = 1u << (x & 31u);
  const uint32_t old = atomicAnd(&sm.bits[b][x >> 5], ~m);
  if ((old & ~m) == 0u) atomicAnd(&sm.sums[b][x >> 10], ~(1u << ((x >> 5) & 31u)));
}
// lowest set bit of a non-empty bitmap (warp-uniform)
__device__ __forceinline__ uint32_t lbit_first(const LongSmem& sm, uint32_t b, uint32_t lane) {
  static_assert(kLS == 64, "two summary words per lane");
  const uint32_t s0 = sm.sums[b][lane], s1 = sm.sums[b][lane + 32];
  const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, s0 != 0u), b1 = __ballot_sync(0xFFFFFFFFu, s1 != 0u);
  const uint32_t src = b0 ? __ffs(b0) - 1u : __ffs(b1) - 1u;
  const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, s0, src), w1 = __shfl_sync(0xFFFFFFFFu, s1, src);
  const uint32_t sw = b0 ? src : 32u + src, sword = b0 ? w0 : w1;
  const uint32_t w = sw * 32u + __ffs(sword) - 1u;
  return w * 32u + __ffs(sm.bits[b][w]) - 1u;
}
// the first `take` set bits of the GPU-class ready bitmap (rank order) -> sm.W
__device__ __forceinline__ void lbit_take(LongSmem& sm, uint32_t take, uint32_t lane) {
  uint32_t got = 0;
  for (uint32_t sw = 0; sw < kLS && got < take; ++sw) {
    const uint32_t sbits = sm.sums[BM_GPU][sw];
    if (!sbits) continue;
    uint32_t w = 0, word = 0;
    if (lane < (uint32_t)__popc(sbits)) {
      w = sw * 32u + __fns(sbits, 0, (int)lane + 1);
      word = sm.bits[BM_GPU][w];
    }
    const uint32_t c = __popc(word);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += v;
    }
    const uint32_t excl = incl - c, tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (got + excl < take) {
      const uint32_t k = min(c, take - got - excl);
      for (uint32_t e = 0; e < k; ++e) {
        sm.W[got + excl + e] = w * 32u + (__ffs(word) - 1u);
        word &= word - 1u;
      }
    }
    got += tot;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32) k_replay_long(ReplayLaunch a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  LongSmem& sm = *reinterpret_cast<LongSmem*>(smem_raw);
  const uint32_t lane = threadIdx.x;
  const uint32_t t = blockIdx.x;
  const uint32_t lo = a.trace_off[t], n = a.trace_off[t + 1] - lo;
  if (n <= kMaxTrace) return;  // k_replay's
  const rt_profile p = a.profiles[a.trace_prof ? a.trace_prof[t] : 0];
  const uint32_t* perm = a.long_perm + lo;  // rank -> global index (radix sort)
  uint32_t* rank = a.long_rank + lo;        // arrival index -> rank
  uint32_t ncpu_l = 0;
  for (uint32_t j = lane; j < n; j += 32) {
    rank[perm[j] - lo] = j;
    ncpu_l += (uint32_t)(a.key[lo + j] >> 63);
  }
  const uint32_t ncpu = __reduce_add_sync(0xFFFFFFFFu, ncpu_l);
  const uint32_t nw = (n + 31) / 32;
  for (uint32_t w = lane; w < nw; w += 32) {
    sm.bits[0][w] = 0; sm.bits[1][w] = 0; sm.bits[2][w] = 0;
  }
  for (uint32_t w = lane; w < kLS; w += 32) {
    sm.sums[0][w] = 0; sm.sums[1][w] = 0; sm.sums[2][w] = 0;
  }
  sm.core_free[lane] = 0;
  const int64_t* g_r = a.arrival + lo;
  const uint16_t* g_len = a.len + lo;
  const float* g_u = a.u + lo;
  const uint32_t* g_D = a.D + lo;
  __syncwarp();

  const uint32_t C = (uint32_t)p.C, m = (uint32_t)p.b10 * C / 10u, cores = (uint32_t)p.cores;
  const int64_t gpu_fixed = p.setup_us + p.base_us;
  int64_t now = g_r[0], gpu_free = 0;
  uint32_t next = 0, done = 0;
  uint32_t cpu_ready = 0, gpu_ready = 0;
  bool have_oldest = false;
  int64_t cpu_min_free = INT64_MAX;
  bool cpu_min_valid = false;
  int64_t oldest_r = 0;
  int64_t resp = 0;
  uint32_t misses = 0;
  int64_t rw = lane < n ? g_r[lane] : INT64_MAX;

  for (;;) {
    // ---- admit arrivals <= now
    while (next < n) {
      const uint32_t i = next + lane;
      const bool arr = rw <= now;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, arr);
      if (!bal) break;
      const uint32_t cnt = __popc(bal);
      const uint32_t rk = arr ? rank[i] : 0xFFFFFFFFu;
      const uint32_t cb = __ballot_sync(0xFFFFFFFFu, rk < ncpu);
      const uint32_t nc = __popc(cb);
      if (gpu_ready == 0 && (bal & ~cb)) {
        oldest_r = __shfl_sync(0xFFFFFFFFu, rw, __ffs(bal & ~cb) - 1);
        have_oldest = true;
      }
      cpu_ready += nc;
      gpu_ready += cnt - nc;
      if (arr) {
        if (rk < ncpu) {
          lbit_set(sm, BM_CPU, rk);
        } else {
          lbit_set(sm, BM_GPU, rk);
          lbit_set(sm, BM_WAIT, i);
        }
      }
      next += cnt;
      rw = next + lane < n ? g_r[next + lane] : INT64_MAX;
      if (cnt < 32) break;
    }
    __syncwarp();
    // ---- CPU cores: highest-key ready CPU task -> lowest-index free core
    bool cpu_started = false;
    while (cpu_ready) {
      const uint32_t fm = __ballot_sync(0xFFFFFFFFu, lane < cores && sm.core_free[lane] <= now);
      if (!fm) break;
      const uint32_t c = __ffs(fm) - 1;
      const uint32_t rk = lbit_first(sm, BM_CPU, lane);
      const uint32_t i = perm[rk] - lo;
      const int64_t end = now + (int64_t)p.gamma * (p.base_us + p.eta_us * (int64_t)g_len[i]);
      __syncwarp();
      if (lane == 0) {
        sm.core_free[c] = end;
        lbit_clear(sm, BM_CPU, rk);
        const int64_t ri = g_r[i];
        resp += end - ri;
        misses += end > ri + (int64_t)g_D[i];
        if (a.end_us) a.end_us[lo + i] = end;
      }
      ++done;
      --cpu_ready;
      cpu_started = true;
      __syncwarp();
    }
    if (cpu_started) cpu_min_valid = false;
    // ---- GPU dispatch
    bool waiting = false;
    if (gpu_free <= now) {
      const uint32_t total = gpu_ready;
      if (total) {
        if (!have_oldest) {
          oldest_r = g_r[lbit_first(sm, BM_WAIT, lane)];
          have_oldest = true;
        }
        const bool flush = (oldest_r <= now - p.xi_us) || next == n;
        const uint32_t full = p.consolidate ? m : C;
        const uint32_t take = total >= full ? full : (flush ? total : 0u);
        if (!take) {
          waiting = true;
        } else {
          lbit_take(sm, take, lane);
          constexpr uint32_t kCh = kMaxWindow / 32;
          const uint32_t nch = (take + 31u) >> 5;
          uint32_t re[kCh], ix[kCh], pos[kCh], len_e[kCh], D_e[kCh];
          float ue[kCh];
          int64_t r_e[kCh];
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k) {
            const uint32_t e = k * 32u + lane;
            re[k] = 0xFFFFFFFFu; ix[k] = 0; ue[k] = 0.0f; len_e[k] = 0u; D_e[k] = 0u; r_e[k] = 0;
            pos[k] = 0xFFFFFFFFu;
            if (k < nch && e < take) {
              re[k] = sm.W[e];
              const uint32_t i = perm[re[k]] - lo;
              ix[k] = i;
              ue[k] = g_u[i];
              len_e[k] = g_len[i];
              D_e[k] = g_D[i];
              r_e[k] = g_r[i];
              pos[k] = e;
            }
          }
          uint32_t cnt;
          if (p.consolidate) {
            // position in the (u asc, rank asc) order (R-TIE), by shuffles
#pragma unroll
            for (uint32_t k = 0; k < kCh; ++k) pos[k] = 0u;
#pragma unroll
            for (uint32_t xk = 0; xk < kCh; ++xk) {
              if (xk < nch) {
                const uint32_t lim = min(32u, take - xk * 32u);
                for (uint32_t x = 0; x < lim; ++x) {
                  const float ux = __shfl_sync(0xFFFFFFFFu, ue[xk], x);
                  const uint32_t rx = __shfl_sync(0xFFFFFFFFu, re[xk], x);
#pragma unroll
                  for (uint32_t k = 0; k < kCh; ++k) pos[k] += (ux < ue[k]) || (ux == ue[k] && rx < re[k]);
                }
              }
            }
#pragma unroll
            for (uint32_t k = 0; k < kCh; ++k) {
              const uint32_t e = k * 32u + lane;
              if (k < nch && e < take) sm.Su[pos[k]] = ue[k];
              else pos[k] = 0xFFFFFFFFu;
            }
            __syncwarp();
            const uint32_t lim = min(C, take);
            cnt = lim;
            for (uint32_t base = 1; base < lim; base += 32) {
              const uint32_t ii = base + lane;
              const bool bad = ii < lim && !(sm.Su[ii] <= __fmul_rn(p.lambda, sm.Su[ii - 1]));
              const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bad);
              if (bal) {
                cnt = base + __ffs(bal) - 1;
                break;
              }
            }
          } else {
            cnt = take;
          }
          uint32_t ml = 0;
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k)
            if (pos[k] < cnt) ml = max(ml, len_e[k]);
          ml = __reduce_max_sync(0xFFFFFFFFu, ml);
          const int64_t end = now + gpu_fixed + p.eta_us * (int64_t)ml;
#pragma unroll
          for (uint32_t k = 0; k < kCh; ++k) {
            if (pos[k] < cnt) {
              lbit_clear(sm, BM_GPU, re[k]);
              lbit_clear(sm, BM_WAIT, ix[k]);
              resp += end - r_e[k];
              misses += end > r_e[k] + (int64_t)D_e[k];
              if (a.end_us) a.end_us[lo + ix[k]] = end;
            }
          }
          done += cnt;
          gpu_ready -= cnt;
          have_oldest = false;
          gpu_free = end;
          __syncwarp();
        }
      }
    }
    if (done >= n) break;
    // ---- next event time
    int64_t nxt = INT64_MAX;
    if (next < n) nxt = __shfl_sync(0xFFFFFFFFu, rw, 0);
    if (gpu_free > now) nxt = min(nxt, gpu_free);
    if (cpu_ready != 0) {
      if (!cpu_min_valid) {
        cpu_min_free = warp_min64(lane < cores ? sm.core_free[lane] : INT64_MAX);
        cpu_min_valid = true;
      }
      nxt = min(nxt, cpu_min_free);
    }
    if (waiting) nxt = min(nxt, oldest_r + p.xi_us);
    if (nxt == INT64_MAX) break;
    now = nxt;
  }
  const int64_t sr = warp_sum64(resp);
  const uint32_t ms = __reduce_add_sync(0xFFFFFFFFu, misses);
  if (lane == 0) a.stats[t] = rt_trace_stats{sr, n, ms};
}

__global__ void k_reduce_stats(const rt_trace_stats* __restrict__ st, uint32_t nt, const uint16_t* __restrict__ grp,
                               uint32_t ngroups, int64_t* __restrict__ sums) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const uint32_t g = grp ? grp[t] : 0u;
    if (g >= ngroups) continue;
    unsigned long long* s = reinterpret_cast<unsigned long long*>(sums + (size_t)g * 3);
    atomicAdd(s + 0, (unsigned long long)st[t].sum_resp_us);
    atomicAdd(s + 1, (unsigned long long)st[t].n);
    atomicAdd(s + 2, (unsigned long long)st[t].misses);
  }
}

// NEXT-4: per-trace response statistics from the replay's end times (one warp
// per trace, n <= 1024): max and nearest-rank p95 of end - r,
// makespan = last end - first arrival, completions.
__global__ void __launch_bounds__(32) k_trace_report(const int64_t* __restrict__ arrival,
                                                     const int64_t* __restrict__ end_us,
                                                     const uint32_t* __restrict__ trace_off,
                                                     rt_trace_summary* __restrict__ out) {
  __shared__ int64_t resp[kMaxTrace];
  const uint32_t t = blockIdx.x, lane = threadIdx.x;
  const uint32_t lo = trace_off[t], n = trace_off[t + 1] - lo;
  if (n > kMaxTrace) return;  // long traces: launch_trace_report_long
  if (n == 0) {
    if (lane == 0) out[t] = rt_trace_summary{0, 0, 0, 0u, 0u};
    return;
  }
  uint32_t npow = 32;
  while (npow < n) npow <<= 1;
  int64_t mx_end = INT64_MIN, mn_r = INT64_MAX;
  for (uint32_t i = lane; i < npow; i += 32) {
    if (i < n) {
      const int64_t r = arrival[lo + i], e = end_us[lo + i];
      resp[i] = e - r;
      mx_end = max(mx_end, e);
      mn_r = min(mn_r, r);
    } else {
      resp[i] = INT64_MAX;  // sorts last
    }
  }
  __syncwarp();
  for (uint32_t k = 2; k <= npow; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < npow; i += 32) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const int64_t a = resp[i], b = resp[l];
          if (((i & k) == 0) == (a > b)) { resp[i] = b; resp[l] = a; }
        }
      }
      __syncwarp();
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx_end = max(mx_end, __shfl_xor_sync(0xFFFFFFFFu, mx_end, o));
    mn_r = min(mn_r, __shfl_xor_sync(0xFFFFFFFFu, mn_r, o));
  }
  if (lane == 0) {
    const uint32_t p = (95u * n + 99u) / 100u;  // ceil(0.95 n), nearest rank
    out[t] = rt_trace_summary{resp[n - 1], resp[p - 1], mx_end - mn_r, n, 0u};
  }
}

// NEXT-4 executor utilization from the replay's end
// times, one warp per trace: a CPU task ran gamma*(base + eta*len);
// the GPU-class tasks that share one end time form one batch (the GPU runs one
// batch at a time and every batch of positive duration ends strictly after the
// previous one), whose duration is setup + base + eta*max len.  The
// GPU tasks are sorted by (end, len) so each batch's last element carries its
// max len.
__global__ void __launch_bounds__(32) k_trace_util(const uint16_t* __restrict__ len,
                                                   const uint64_t* __restrict__ key,
                                                   const int64_t* __restrict__ end_us,
                                                   const uint32_t* __restrict__ trace_off,
                                                   const rt_profile* __restrict__ profiles,
                                                   const uint16_t* __restrict__ trace_prof,
                                                   rt_trace_util* __restrict__ out) {
  __shared__ int64_t se[kMaxTrace];
  __shared__ uint16_t sl[kMaxTrace];
  const uint32_t t = blockIdx.x, lane = threadIdx.x;
  const uint32_t lo = trace_off[t], n = trace_off[t + 1] - lo;
  if (n > kMaxTrace) return;  // long traces: launch_trace_util_long
  const rt_profile& p = profiles[trace_prof ? trace_prof[t] : 0];
  uint32_t npow = 32;
  while (npow < n) npow <<= 1;
  int64_t cbusy = 0;
  uint32_t ccnt = 0;
  for (uint32_t i = lane; i < npow; i += 32) {
    int64_t e = INT64_MAX;  // CPU tasks and padding sort last
    uint16_t l = 0;
    if (i < n) {
      const uint16_t li = len[lo + i];
      if (key[lo + i] >> 63) {
        cbusy += (int64_t)p.gamma * (p.base_us + p.eta_us * (int64_t)li);
        ++ccnt;
      } else {
        e = end_us[lo + i];
        l = li;
      }
    }
    se[i] = e;
    sl[i] = l;
  }
  __syncwarp();
  for (uint32_t k = 2; k <= npow; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < npow; i += 32) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const int64_t ea = se[i], eb = se[l];
          const uint16_t la = sl[i], lb = sl[l];
          const bool gt = ea > eb || (ea == eb && la > lb);
          if (((i & k) == 0) == gt) { se[i] = eb; se[l] = ea; sl[i] = lb; sl[l] = la; }
        }
      }
      __syncwarp();
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cbusy += __shfl_xor_sync(0xFFFFFFFFu, cbusy, o);
    ccnt += __shfl_xor_sync(0xFFFFFFFFu, ccnt, o);
  }
  const uint32_t ngpu = n - ccnt;
  int64_t gbusy = 0;
  uint32_t gcnt = 0;
  for (uint32_t i = lane; i < ngpu; i += 32)
    if (i + 1 == ngpu || se[i + 1] != se[i]) {
      gbusy += p.setup_us + p.base_us + p.eta_us * (int64_t)sl[i];
      ++gcnt;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gbusy += __shfl_xor_sync(0xFFFFFFFFu, gbusy, o);
    gcnt += __shfl_xor_sync(0xFFFFFFFFu, gcnt, o);
  }
  if (lane == 0) out[t] = rt_trace_util{gbusy, cbusy, gcnt, ccnt};
}


// ---- NEXT-4 for long traces (> kMaxTrace tasks): sort keys built per trace,
// ordered by one radix sort (K3, descending), then a one-CTA pass.
// report: key = response end - r (>= 0); util: GPU-class key = end << 16 | len
// (the first element of each equal-end group in descending order carries the
// batch's max len), CPU-class tasks key 0 (sort last).
__global__ void k_long_keys(const int64_t* __restrict__ arrival, const int64_t* __restrict__ end_us,
                            const uint16_t* __restrict__ len, const uint64_t* __restrict__ key, uint32_t n,
                            int util, uint64_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (!util) out[i] = (uint64_t)(end_us[i] - arrival[i]);
    else out[i] = (key[i] >> 63) ? 0ull : (((uint64_t)end_us[i] << 16) | len[i]);
  }
}

__device__ __forceinline__ int64_t block_sum64(int64_t v, int64_t* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31u) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t t = 0;
  for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += sh[w];
  __syncthreads();
  return t;
}

// one CTA (1024 threads): max / p95 response from the sorted order, makespan
__global__ void __launch_bounds__(1024) k_long_report(const int64_t* __restrict__ arrival,
                                                      const int64_t* __restrict__ end_us, uint32_t lo, uint32_t n,
                                                      const uint32_t* __restrict__ perm, const uint64_t* __restrict__ k,
                                                      rt_trace_summary* __restrict__ out) {
  int64_t mx_end = INT64_MIN, mn_r = INT64_MAX;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    mx_end = max(mx_end, end_us[lo + i]);
    mn_r = min(mn_r, arrival[lo + i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx_end = max(mx_end, __shfl_xor_sync(0xFFFFFFFFu, mx_end, o));
    mn_r = min(mn_r, __shfl_xor_sync(0xFFFFFFFFu, mn_r, o));
  }
  __shared__ int64_t smx[32], smn[32];
  if ((threadIdx.x & 31u) == 0) { smx[threadIdx.x >> 5] = mx_end; smn[threadIdx.x >> 5] = mn_r; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w) { mx_end = max(mx_end, smx[w]); mn_r = min(mn_r, smn[w]); }
    const uint32_t p = (95u * n + 99u) / 100u;  // ceil(0.95 n), nearest rank (ascending)
    const int64_t rmax = (int64_t)k[perm[0] - lo], rp95 = (int64_t)k[perm[n - p] - lo];
    *out = rt_trace_summary{rmax, rp95, mx_end - mn_r, n, 0u};
  }
}

// one CTA: GPU busy = sum over equal-end groups (batches) of setup + base + eta * max len;
// CPU busy = sum over CPU-class tasks of gamma * (base + eta * len)
__global__ void __launch_bounds__(1024) k_long_util(const uint16_t* __restrict__ len, const uint64_t* __restrict__ key,
                                                    uint32_t lo, uint32_t n, const rt_profile* __restrict__ profiles,
                                                    const uint16_t* __restrict__ trace_prof, uint32_t t,
                                                    const uint32_t* __restrict__ perm,
                                                    const uint64_t* __restrict__ k, rt_trace_util* __restrict__ out) {
  __shared__ int64_t sh[32];
  const rt_profile& p = profiles[trace_prof ? trace_prof[t] : 0];
  int64_t cb = 0, gb = 0, cc = 0, gc = 0;
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
    const uint32_t i = perm[j] - lo;  // j-th in descending (end, len); CPU-class keys 0 at the end
    const uint64_t kj = k[i];
    if (key[lo + i] >> 63) {
      cb += (int64_t)p.gamma * (p.base_us + p.eta_us * (int64_t)len[lo + i]);
      ++cc;
    } else if (j == 0 || (k[perm[j - 1] - lo] >> 16) != (kj >> 16)) {  // first (max len) of its end group
      gb += p.setup_us + p.base_us + p.eta_us * (int64_t)(kj & 0xFFFFu);
      ++gc;
    }
  }
  cb = block_sum64(cb, sh);
  gb = block_sum64(gb, sh);
  cc = block_sum64(cc, sh);
  gc = block_sum64(gc, sh);
  if (threadIdx.x == 0) *out = rt_trace_util{gb, cb, (uint32_t)gc, (uint32_t)cc};
}

}  // namespace

cudaError_t launch_trace_util(const uint16_t* len, const uint64_t* key, const int64_t* end_us,
                              const uint32_t* d_trace_off, uint32_t nt, const rt_profile* d_prof,
                              const uint16_t* d_trace_prof, rt_trace_util* out, cudaStream_t s) {
  if (!nt) return cudaSuccess;
  k_trace_util<<<nt, 32, 0, s>>>(len, key, end_us, d_trace_off, d_prof, d_trace_prof, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_trace_report(const int64_t* arrival, const int64_t* end_us, const uint32_t* d_trace_off,
                                uint32_t nt, rt_trace_summary* out, cudaStream_t s) {
  if (!nt) return cudaSuccess;
  k_trace_report<<<nt, 32, 0, s>>>(arrival, end_us, d_trace_off, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_trace_long(const int64_t* arrival, const int64_t* end_us, const uint16_t* len,
                              const uint64_t* key, uint32_t lo, uint32_t n, const rt_profile* d_prof,
                              const uint16_t* d_trace_prof, uint32_t t, rt_trace_summary* rep, rt_trace_util* util,
                              void* ws, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  uint64_t* k = reinterpret_cast<uint64_t*>(p);
  uint32_t* perm = reinterpret_cast<uint32_t*>(p + (((size_t)n * 8 + 255) & ~size_t(255)));
  void* rws = p + (((size_t)n * 8 + 255) & ~size_t(255)) + (((size_t)n * 4 + 255) & ~size_t(255));
  k_long_keys<<<(n + 255) / 256, 256, 0, s>>>(arrival + lo, end_us + lo, len ? len + lo : nullptr,
                                               key ? key + lo : nullptr, n, util ? 1 : 0, k);
  note_launch();
  cudaError_t e = radix_sort_desc(k, lo, n, perm, 1, rws, s);
  if (e != cudaSuccess) return e;
  if (util) k_long_util<<<1, 1024, 0, s>>>(len, key, lo, n, d_prof, d_trace_prof, t, perm, k, util);
  else k_long_report<<<1, 1024, 0, s>>>(arrival, end_us, lo, n, perm, k, rep);
  note_launch();
  return cudaGetLastError();
}

size_t trace_long_workspace(uint32_t n) {
  return (((size_t)n * 8 + 255) & ~size_t(255)) + (((size_t)n * 4 + 255) & ~size_t(255)) + radix_sort_workspace(n);
}

cudaError_t launch_replay(const ReplayLaunch& a, uint32_t max_window, cudaStream_t s) {
  if (!a.nt) return cudaSuccess;
  const size_t smem = sizeof(ReplaySmem);
  const uint32_t kch = (max_window + 31u) / 32u;
  void (*kern)(ReplayLaunch) = kch <= 1 ? k_replay<1> : (kch <= 2 ? k_replay<2> : k_replay<4>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_trace_rank<<<a.nt, kRankThr, 0, s>>>(a.key, a.trace_off, a.sidx);
  note_launch();
  kern<<<a.nt, 32, smem, s>>>(a);
  note_launch();
  if (a.long_perm) {  // some trace is longer than kMaxTrace (its rank order is already in long_perm)
    e = cudaFuncSetAttribute(k_replay_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LongSmem));
    if (e != cudaSuccess) return e;
    k_replay_long<<<a.nt, 32, sizeof(LongSmem), s>>>(a);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_reduce_stats(const rt_trace_stats* st, uint32_t nt, const uint16_t* grp, uint32_t ngroups,
                                int64_t* sums, cudaStream_t s) {
  if (!nt) return cudaSuccess;
  uint32_t blocks = (nt + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_reduce_stats<<<blocks, 256, 0, s>>>(st, nt, grp, ngroups, sums);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
