// k_score.cu — K1 (RuleGen: tokenize, lemmatize, lexicon probe, six rule
// scorers) fused with K2 (weighted-rule regression, deadline, priority key,
// offload class).  §8(a) rows a1-a4.
//
// Design (DESIGN.md §7 K1): persistent CTAs of 256 threads; each tile is 256
// consecutive requests whose packed bytes are staged HBM -> shared memory with
// coalesced 128-bit non-allocating loads; then one lane runs one request's
// finite-state machine over shared memory; the epilogue computes u and the
// key in registers and writes 4 B + 8 B (+ optional 16 B feature row).
// The lexicon (<= 1024 lemmas) lives in shared memory as an open-addressing
// table.  All arithmetic that decides an integer is binary32 with explicit
// round-to-nearest intrinsics (R-FP).
#include "internal.cuh"

namespace rtlm {

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kStage = 32768;  // staged text bytes per tile

// ------------------------------------------------------------ epilogue math
__device__ __forceinline__ float regress(const uint32_t f[7], const rt_regressor& r) {
  // O3 / R-FP: acc = c; acc = fma(w_k, (float)f_k, acc), k = 0..6; clamp at 0
  float acc = r.c;
#pragma unroll
  for (int k = 0; k < 7; ++k) acc = __fmaf_rn(r.w[k], __uint2float_rn(f[k]), acc);
  return acc > 0.0f ? acc : 0.0f;
}

__device__ __forceinline__ uint32_t deadline_us(uint32_t ntok, const rt_profile& p) {
  // R-D: D = min(tightness * mu * ntok, 2^32 - 1)
  unsigned long long d = (unsigned long long)(long long)p.tightness * (unsigned long long)p.mu_us *
                         (unsigned long long)ntok;
  return d > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d;
}

__device__ __forceinline__ uint64_t priority_key(float u, uint32_t D_us, int64_t r, const rt_profile& p) {
  // R-KEY / O4: key = cls<<63 | tier<<62 | ord(v)
  uint64_t tier = 0, val;
  if (p.policy == RT_UP || p.policy == RT_SLACK) {
    float D = __uint2float_rn(D_us);
    float num = 1.0f;
    if (p.policy == RT_UP) {  // Eq. 3 numerator with R-NUM
      float un = p.raw_numerator ? u : fminf(1.0f, __fdiv_rn(u, p.u_max));
      num = __fsub_rn(1.0f, __fmul_rn(p.alpha, un));
    }
    float slk = __fsub_rn(D, __fmul_rn(__ll2float_rn(p.eta_us), u));  // d - r - eta*u
    float v;
    if (slk <= 1.0f) {  // R-OVERDUE
      tier = 1;
      v = -slk;
    } else {
      v = __fdiv_rn(num, slk);
    }
    val = ord32_bits(__float_as_uint(v));
  } else if (p.policy == RT_FIFO) {
    val = (uint64_t)(-r + (1ll << 61));
  } else if (p.policy == RT_EDF) {
    val = (uint64_t)(-(r + (int64_t)D_us) + (1ll << 61));
  } else if (p.policy == RT_LUF) {
    val = ord32_bits(__float_as_uint(-u));
  } else {
    val = ord32_bits(__float_as_uint(u));
  }
  uint64_t cls = (p.offload && u > p.tau) ? 1ull : 0ull;  // strict
  return (cls << 63) | (tier << 62) | val;
}

// ------------------------------------------------------------ lexicon probe
struct Lex {
  const LexEntry* e;
  const uint16_t* slots;
  uint32_t bits;
};

__device__ __forceinline__ uint32_t probe(const Lex& L, uint64_t k0, uint64_t k1, uint32_t len) {
  const uint32_t mask = (1u << L.bits) - 1u;
  uint32_t h = lex_hash(k0, k1, len, L.bits);
  for (;;) {
    uint32_t s = L.slots[h];
    if (!s) return 0;
    const LexEntry& e = L.e[s - 1];
    if (e.k0 == k0 && e.k1 == k1 && e.len == len) return e.attr;
    h = (h + 1u) & mask;
  }
}

__device__ __forceinline__ uint64_t mask_bytes(uint32_t nbytes) {  // nbytes in 0..8
  return nbytes >= 8 ? ~0ull : ((1ull << (8 * nbytes)) - 1ull);
}

// Lemma attributes of a word token of length L whose first bytes (lowercased,
// little-endian) are k0/k1 (valid up to min(L,16)) and whose last three bytes
// are s3 = b[L-3]<<16 | b[L-2]<<8 | b[L-1].  R-LEMMA.
__device__ __forceinline__ uint32_t word_attr(const Lex& L, uint32_t len, uint64_t k0, uint64_t k1, uint32_t s3) {
  const uint32_t b1 = s3 & 0xFFu, b2 = (s3 >> 8) & 0xFFu, b3 = (s3 >> 16) & 0xFFu;
  if (len == 3 && s3 == (('n' << 16) | ('\'' << 8) | 't'))  // n't -> not
    return probe(L, (uint64_t)'n' | ((uint64_t)'o' << 8) | ((uint64_t)'t' << 16), 0ull, 3);
  uint32_t strip = 0;
  if (len >= 5 && b3 == 'i' && b2 == 'n' && b1 == 'g') strip = 3;
  else if (len >= 4 && b2 == 'e' && b1 == 'd') strip = 2;
  else if (len >= 4 && b2 == 'e' && b1 == 's') strip = 2;
  else if (len >= 3 && b1 == 's' && b2 != 's') strip = 1;
  const uint32_t ll = len - strip;
  if (ll == 0 || ll > 16) return 0;
  uint64_t m0 = k0 & mask_bytes(ll < 8 ? ll : 8);
  uint64_t m1 = ll > 8 ? (k1 & mask_bytes(ll - 8)) : 0ull;
  return probe(L, m0, m1, ll);
}

// ------------------------------------------------------------ rule FSM
enum : uint32_t { T_NONE = 0, T_WORD = 1, T_COMMA = 2, T_OTHER = 3 };
enum : uint32_t { F_NOUN_TWO = 1, F_SENT_WORD = 2, F_LAST_BROAD = 4, F_COORD_PEND = 8 };
constexpr uint32_t kNoNoun = 0xFFFFFFFFu;

struct Rules {
  uint32_t S, Y, M, V, O, P, ntok, nd, nq;
  uint32_t noun_first, fl, what_cd, chain, wsc, prev, prev2;
  // current word run
  uint32_t wlen;
  uint64_t k0, k1, tail;

  __device__ __forceinline__ void init() {
    S = Y = M = V = O = P = ntok = nd = nq = 0;
    noun_first = kNoNoun;
    fl = 0; what_cd = 0; chain = 0; wsc = 0; prev = T_NONE; prev2 = T_NONE;
    wlen = 0; k0 = k1 = tail = 0;
  }

  // R-RULES, one word token with lexicon attributes `a`
  __device__ __forceinline__ void on_word(uint32_t a) {
    ++ntok;
    V += a & A_VAGUE;
    Y += (a >> 8) & 1u;
    M = min(M + ((a >> A_SEM_SHIFT) & A_SEM_MASK), 0xFFFFFFu);
    if ((a & A_PREP) && (fl & F_NOUN_TWO)) ++S;                 // structural: PREP first
    if (a & A_NOUN) {
      uint32_t id = a >> A_ID_SHIFT;
      if (noun_first == kNoNoun) noun_first = id;
      else if (id != noun_first) fl |= F_NOUN_TWO;
    }
    if (!(fl & F_SENT_WORD)) {                                   // first word of the sentence
      fl |= F_SENT_WORD;
      if (a & A_OPENER) ++O;
      what_cd = (a & A_WHAT) ? 3u : 0u;
    } else if (what_cd) {
      if (a & A_CAUSE) { ++O; what_cd = 0; } else --what_cd;
    }
    fl = (a & A_BROAD) ? (fl | F_LAST_BROAD) : (fl & ~F_LAST_BROAD);
    if (fl & F_COORD_PEND) ++P;                                  // coordinator followed by a word
    bool pend = (a & A_COORD) && (prev == T_WORD || (prev == T_COMMA && prev2 == T_WORD));
    fl = pend ? (fl | F_COORD_PEND) : (fl & ~F_COORD_PEND);
    ++wsc;
    prev2 = prev;
    prev = T_WORD;
  }

  __device__ __forceinline__ void on_punct(uint32_t c) {
    ++ntok;
    fl &= ~F_COORD_PEND;
    if (what_cd) --what_cd;
    if (c == ',') {
      if (chain && wsc) {
        if (++chain == 2) ++P;                                   // comma list of >= 3 items
      } else {
        chain = 1;
      }
      wsc = 0;
      prev2 = prev;
      prev = T_COMMA;
      return;
    }
    chain = 0;
    if (c == '.' || c == '?' || c == '!') {
      if (c == '?') {
        ++nq;
        if ((fl & F_SENT_WORD) && (fl & F_LAST_BROAD)) ++O;      // broad-scope interrogative
      }
      noun_first = kNoNoun;
      fl &= F_COORD_PEND;  // (already cleared) reset sentence state
      what_cd = 0;
    }
    prev2 = prev;
    prev = T_OTHER;
  }

  // end of a W run: one clitic split (R-CLITIC), then word tokens
  __device__ __forceinline__ void end_run(const Lex& L) {
    const uint32_t n = wlen;
    const uint32_t t3 = (uint32_t)(tail & 0xFFFFFFu), t2 = (uint32_t)(tail & 0xFFFFu);
    uint32_t cut = 0;
    if (n > 3 && t3 == (('n' << 16) | ('\'' << 8) | 't')) cut = 3;
    else if (n > 2 && (t2 == (('\'' << 8) | 's') || t2 == (('\'' << 8) | 'm') || t2 == (('\'' << 8) | 'd'))) cut = 2;
    else if (n > 3 && (t3 == (('\'' << 16) | ('r' << 8) | 'e') || t3 == (('\'' << 16) | ('v' << 8) | 'e') ||
                       t3 == (('\'' << 16) | ('l' << 8) | 'l')))
      cut = 3;
    if (!cut) {
      on_word(word_attr(L, n, k0, k1, t3));
    } else {
      const uint32_t ns = n - cut;
      on_word(word_attr(L, ns, k0, k1, (uint32_t)((tail >> (8 * cut)) & 0xFFFFFFu)));
      // clitic bytes b[n-cut..n-1] -> little-endian key
      uint32_t ck = cut == 3 ? __byte_perm(t3, 0, 0x4012) : __byte_perm(t2, 0, 0x4401);
      on_word(word_attr(L, cut, (uint64_t)ck, 0ull, t3 & (cut == 3 ? 0xFFFFFFu : 0xFFFFu)));
    }
    wlen = 0;
  }

  __device__ __forceinline__ void byte(uint32_t c, const Lex& L) {
    const uint32_t lc = c | 0x20u;
    const bool isW = (lc - 'a' < 26u) || (c - '0' < 10u) || c == '\'';
    if (isW) {
      if (wlen == 0) { k0 = 0; k1 = 0; tail = 0; }
      if (wlen < 8) k0 |= (uint64_t)lc << (8 * wlen);
      else if (wlen < 16) k1 |= (uint64_t)lc << (8 * (wlen - 8));
      tail = (tail << 8) | lc;
      ++wlen;
      return;
    }
    if (wlen) end_run(L);
    if (c == ' ' || (c - 9u) < 5u) return;        // S
    if (c - 0x21u < 0x5Eu) on_punct(c);           // P
    else ++nd;                                    // X: dropped, counted
  }

  __device__ __forceinline__ void finish(const Lex& L, uint32_t f[8], bool& sat) {
    if (wlen) end_run(L);
    unsigned long long Pt = (unsigned long long)P + (nq > 1 ? nq - 1 : 0);
    uint64_t raw[8] = {S, Y, M, V, O, Pt, ntok, nd};
    sat = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sat |= raw[k] > 65535ull;
      f[k] = raw[k] > 65535ull ? 65535u : (uint32_t)raw[k];
    }
  }
};

__device__ __forceinline__ uint4 ld_nc_v4(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(kThreads) k_score(ScoreLaunch a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // ---- lexicon -> shared memory
  LexEntry* s_ent = reinterpret_cast<LexEntry*>(smem);
  const uint32_t ent_bytes = a.lex.n_entries * (uint32_t)sizeof(LexEntry);
  uint16_t* s_slots = reinterpret_cast<uint16_t*>(smem + ((ent_bytes + 15u) & ~15u));
  const uint32_t nslots = 1u << a.lex.bits;
  uint8_t* stage = reinterpret_cast<uint8_t*>(s_slots) + ((nslots * 2u + 15u) & ~15u);
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.lex.entries);
    uint32_t* dst = reinterpret_cast<uint32_t*>(s_ent);
    for (uint32_t i = threadIdx.x; i < ent_bytes / 4; i += kThreads) dst[i] = src[i];
    for (uint32_t i = threadIdx.x; i < nslots; i += kThreads) s_slots[i] = a.lex.slots[i];
  }
  const Lex L{s_ent, s_slots, a.lex.bits};
  const uint32_t total = a.n ? a.offsets[a.n] : 0u;
  const uint32_t ntiles = (a.n + kThreads - 1) / kThreads;

  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t r0 = tile * kThreads;
    const uint32_t r1 = min(r0 + kThreads, a.n);
    const uint32_t b0 = a.offsets[r0];
    uint32_t b1 = a.offsets[r1];
    if (b1 < b0) b1 = b0;
    const uint32_t base = b0 & ~15u;
    const uint32_t span = min(b1 - base, kStage);
    __syncthreads();  // previous tile done with `stage` (and lexicon copied)
    for (uint32_t off = threadIdx.x * 16u; off < span; off += kThreads * 16u) {
      const uint32_t g = base + off;
      if (g + 16u <= total) {
        *reinterpret_cast<uint4*>(stage + off) = ld_nc_v4(a.bytes + g);
      } else {
#pragma unroll 1
        for (uint32_t j = 0; j < 16u && g + j < total; ++j) stage[off + j] = a.bytes[g + j];
      }
    }
    __syncthreads();

    const uint32_t r = r0 + threadIdx.x;
    if (r < r1) {
      uint32_t s = a.offsets[r], e = a.offsets[r + 1];
      if (e < s) {
        atomicOr(a.flags, RT_FLAG_BAD_OFFSETS);
        e = s;
      }
      Rules R;
      R.init();
      if (s >= base && e <= base + span) {
        const uint8_t* q = stage + (s - base);
        const uint32_t len = e - s;
#pragma unroll 4
        for (uint32_t i = 0; i < len; ++i) R.byte(q[i], L);
      } else {
        for (uint32_t i = s; i < e; ++i) R.byte(__ldg(a.bytes + i), L);
      }
      uint32_t f[8];
      bool sat;
      R.finish(L, f, sat);
      if (sat) atomicOr(a.flags, RT_FLAG_SATURATED);
      if (!a.fused || a.feat) {
        uint4 pk = make_uint4(f[0] | (f[1] << 16), f[2] | (f[3] << 16), f[4] | (f[5] << 16), f[6] | (f[7] << 16));
        *reinterpret_cast<uint4*>(a.feat + (size_t)r * 8) = pk;
      }
      if (a.fused) {
        const float u = regress(f, a.reg);
        const uint32_t D = a.D_in ? a.D_in[r] : deadline_us(f[6], a.prof);
        const int64_t arr = a.arrival ? a.arrival[r] : 0;
        a.u[r] = u;
        a.key[r] = priority_key(u, D, arr, a.prof);
        if (a.D_out) a.D_out[r] = D;
      }
    }
  }
}

__global__ void k_predict(const uint16_t* __restrict__ feat, uint32_t n, rt_regressor reg, float* __restrict__ u) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint4 pk = *reinterpret_cast<const uint4*>(feat + (size_t)i * 8);
  uint32_t f[7] = {pk.x & 0xFFFFu, pk.x >> 16, pk.y & 0xFFFFu, pk.y >> 16, pk.z & 0xFFFFu, pk.z >> 16, pk.w & 0xFFFFu};
  u[i] = regress(f, reg);
}

__global__ void k_key(const float* __restrict__ u, const uint16_t* __restrict__ feat, const int64_t* __restrict__ arr,
                      const uint32_t* __restrict__ D_in, uint32_t n, rt_profile p, uint64_t* __restrict__ key,
                      uint32_t* __restrict__ D_out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t D = D_in ? D_in[i] : deadline_us(feat[(size_t)i * 8 + 6], p);
  key[i] = priority_key(u[i], D, arr ? arr[i] : 0, p);
  if (D_out) D_out[i] = D;
}

}  // namespace

size_t score_smem_bytes(const DevLexicon& lex) {
  return ((lex.n_entries * sizeof(LexEntry) + 15) & ~size_t(15)) + (((size_t(1) << lex.bits) * 2 + 15) & ~size_t(15)) +
         kStage;
}

cudaError_t launch_score(const ScoreLaunch& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const size_t smem = score_smem_bytes(a.lex);
  cudaError_t e = cudaFuncSetAttribute(k_score, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const uint32_t ntiles = (a.n + kThreads - 1) / kThreads;
  uint32_t grid = (uint32_t)(a.num_sms * per_sm);
  if (grid > ntiles) grid = ntiles;
  k_score<<<grid, kThreads, smem, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_predict(const uint16_t* feat, uint32_t n, const rt_regressor& reg, float* u, cudaStream_t s) {
  if (!n) return cudaSuccess;
  k_predict<<<(n + 255) / 256, 256, 0, s>>>(feat, n, reg, u);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_key(const float* u, const uint16_t* feat, const int64_t* arr, const uint32_t* D_in, uint32_t n,
                       const rt_profile& p, uint64_t* key, uint32_t* D_out, cudaStream_t s) {
  if (!n) return cudaSuccess;
  k_key<<<(n + 255) / 256, 256, 0, s>>>(u, feat, arr, D_in, n, p, key, D_out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtlm
