// k_score.cu — K1 (RuleGen: tokenize, lemmatize, lexicon probe, six rule
// scorers) fused with K2 (weighted-rule regression, deadline, priority key,
// offload class).  §8(a) rows a1-a4.
//
// Design (DESIGN.md §7 K1): persistent CTAs of 32 warps; every warp streams
// the bytes of 32 consecutive requests (a task from a global work counter) in
// 512-byte chunks: byte classes and word-run starts as bit masks, one lane per
// token event (run -> clitic split, lemma, lexicon probe), and the six rules
// as per-token predicates evaluated one token per lane with ballots (see the
// K1 v4 block).  The epilogue computes u and the key in registers and writes
// 4 B + 8 B (+ optional 16 B feature row) per request.  The lexicon (<= 1024
// lemmas) lives in shared memory as an open-addressing table.  All arithmetic
// that decides an integer is binary32 with explicit round-to-nearest
// intrinsics (R-FP).  Warps whose offsets decrease use the per-lane byte FSM
// (Rules::byte), which implements the same rules sequentially.
#include "internal.cuh"

namespace rtlm {

namespace {

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

// entry index + 1 of a lemma (0 = not in the lexicon)
__device__ __forceinline__ uint32_t probe_idx(const Lex& L, uint64_t k0, uint64_t k1, uint32_t len) {
  const uint32_t mask = (1u << L.bits) - 1u;
  uint32_t h = lex_hash(k0, k1, len, L.bits);
  for (;;) {
    const uint32_t s = L.slots[h];
    if (!s) return 0;
    const LexEntry& e = L.e[s - 1];
    if (e.k0 == k0 && e.k1 == k1 && e.len == len) return s;
    h = (h + 1u) & mask;
  }
}

// 12-bit prefilter index of a lemma from its first two bytes (b1 = 0 if the lemma has one byte)
__host__ __device__ __forceinline__ uint32_t pref_idx(uint32_t b0, uint32_t b1) { return ((b0 << 5) ^ b1) & 0xFFFu; }

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

// Entry index + 1 of a word token (R-LEMMA), with the 2-byte prefilter.
__device__ __forceinline__ uint32_t word_idx(const Lex& L, const uint32_t* pref, uint32_t len, uint64_t k0,
                                             uint64_t k1, uint32_t s3) {
  const uint32_t b1 = s3 & 0xFFu, b2 = (s3 >> 8) & 0xFFu, b3 = (s3 >> 16) & 0xFFu;
  if (len == 3 && s3 == (('n' << 16) | ('\'' << 8) | 't')) {  // n't -> not
    const uint32_t pi = pref_idx('n', 'o');
    if (!((pref[pi >> 5] >> (pi & 31u)) & 1u)) return 0;
    return probe_idx(L, (uint64_t)'n' | ((uint64_t)'o' << 8) | ((uint64_t)'t' << 16), 0ull, 3);
  }
  uint32_t strip = 0;
  if (len >= 5 && b3 == 'i' && b2 == 'n' && b1 == 'g') strip = 3;
  else if (len >= 4 && b2 == 'e' && b1 == 'd') strip = 2;
  else if (len >= 4 && b2 == 'e' && b1 == 's') strip = 2;
  else if (len >= 3 && b1 == 's' && b2 != 's') strip = 1;
  const uint32_t ll = len - strip;
  if (ll == 0 || ll > 16) return 0;
  const uint32_t pi = pref_idx((uint32_t)(k0 & 0xFFu), ll >= 2 ? (uint32_t)((k0 >> 8) & 0xFFu) : 0u);
  if (!((pref[pi >> 5] >> (pi & 31u)) & 1u)) return 0;
  const uint64_t m0 = k0 & mask_bytes(ll < 8 ? ll : 8);
  const uint64_t m1 = ll > 8 ? (k1 & mask_bytes(ll - 8)) : 0ull;
  return probe_idx(L, m0, m1, ll);
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

  // add this thread's partial counters of one request into the tile accumulators
  __device__ __forceinline__ void flush(uint32_t* acc9) {
    const uint32_t v[9] = {S, Y, M, V, O, P, ntok, nd, nq};
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if (v[i]) atomicAdd(&acc9[i], v[i]);
  }

  // token record of the two-phase path: kind in bits 0..2, entry+1 in bits 3..15
  __device__ __forceinline__ void on_record(uint32_t rec, const Lex& L) {
    const uint32_t kind = rec & 7u;
    if (kind == 1u) {
      const uint32_t e = rec >> 3;
      on_word(e ? L.e[e - 1].attr : 0u);
    } else if (kind == 7u) {
      ++nd;
    } else if (kind != 0u) {
      const uint32_t c = kind == 2u ? ',' : kind == 3u ? '.' : kind == 4u ? '?' : kind == 5u ? '!' : '#';
      on_punct(c);
    }
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

  static __device__ __forceinline__ void finish_acc(const uint32_t* a9, uint32_t f[8], bool& sat) {
    unsigned long long Pt = (unsigned long long)a9[5] + (a9[8] > 1 ? a9[8] - 1 : 0);
    uint64_t raw[8] = {a9[0], a9[1], a9[2], a9[3], a9[4], Pt, a9[6], a9[7]};
    sat = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sat |= raw[k] > 65535ull;
      f[k] = raw[k] > 65535ull ? 65535u : (uint32_t)raw[k];
    }
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

// ============================================================ helpers of the scorer
__device__ __forceinline__ uint32_t class_bits(uint32_t b) {
  const uint32_t lc = b | 0x20u;
  const bool w = (lc - 'a' < 26u) || (b - '0' < 10u) || b == '\'';
  const bool sp = b == ' ' || (b - 9u) < 5u;
  const bool p = !w && (b - 0x21u < 0x5Eu);
  return w ? 0x1u : (p ? 0x100u : (sp ? 0u : 0x10000u));
}

__device__ __forceinline__ void epilogue(const ScoreLaunch& a, uint32_t r, const uint32_t f[8]) {
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

// ============================================================ K1 v4 (warp streams)
// One warp owns 32 consecutive requests (taken from a global work counter) and
// streams their bytes in 512-byte chunks; no CTA-wide barriers.
//  (1) classify: each lane classifies its 16 staged bytes through a per-lane
//      replicated class table -> word / punctuation / dropped bit masks;
//  (2) events: word-run starts (a run never crosses a request start) and
//      punctuation bytes, compacted in byte order; a run reaching the chunk end
//      is carried into the next chunk;
//  (3) tokens: lane per event -- punctuation kind, or the run's clitic split
//      (R-CLITIC), lemma (R-LEMMA) and lexicon probe -> 1 or 2 tokens written
//      in order into a small ring;
//  (4) rules (R-RULES, in the oracle's sentence formulation O2): lane per
//      token.  Every rule is a predicate on the token, its three predecessors
//      and "last earlier token with property X" positions (request start,
//      sentence end, word, first word, noun, first noun, second distinct
//      noun, punctuation) obtained with ballots, so the counters become
//      per-token contributions summed per request (segmented warp scan).
// Warps whose offsets are not non-decreasing use the per-lane byte FSM.
constexpr uint32_t kT4 = 1024;                // threads per CTA (32 warps)
constexpr uint32_t kW4 = kT4 / 32;
constexpr uint32_t kChunk = 512;              // bytes per warp chunk (16 per lane)
constexpr uint32_t kRing = 128;               // token ring per warp

enum : uint32_t { K_W = 1, K_COMMA = 2, K_END = 3, K_Q = 4, K_OTH = 5 };

struct Carry {
  int32_t rs, end, word, fw, noun, fn, d, punct;
  uint32_t fn_id, word_broad, punct_comma, punct_link;
  uint32_t prev_req;  // request of the last token (0xFFFFFFFF: none)
};

struct __align__(16) WarpBuf {
  uint32_t stage[4 + 2 * kChunk / 4 + 8];  // 16 B pad | previous chunk | chunk | 32 B pad
  uint32_t wm[kChunk / 32 + 1], mk[kChunk / 32 + 1];
  uint16_t ev[kChunk + 1];
  uint8_t evq[kChunk + 1];             // request of each event
  uint32_t rs[32];                     // request starts (absolute byte offsets)
  uint32_t t_attr[kRing];
  uint8_t t_meta[kRing];               // kind | req << 3
  uint32_t acc[32][9];                 // S Y M V O P ntok nd nq
  Carry cy;                            // rule-scan carries between token batches (kept out of registers)
};

struct Smem4 {
  uint32_t lut[256 * 32];              // class bits per byte, replicated per lane: W 0x1, P 0x100, X 0x10000
  uint32_t pref[128];
  WarpBuf w[kW4];
};

__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t lanemask_le() { uint32_t m; asm("mov.u32 %0, %%lanemask_le;" : "=r"(m)); return m; }

// last position (global token index) among lanes whose bit is set in m, else carry
__device__ __forceinline__ int32_t last_pos(uint32_t m, int32_t tb, int32_t carry) {
  return m ? tb + 31 - (int32_t)__clz(m) : carry;
}

// request index of absolute byte position pos: last i < cnt with rs[i] <= pos
__device__ __forceinline__ uint32_t req_of(const uint32_t* rs, uint32_t cnt, uint32_t pos) {
  uint32_t lo = 0;
#pragma unroll
  for (uint32_t st = 16; st; st >>= 1)
    if (lo + st < cnt && rs[lo + st] <= pos) lo += st;
  return lo;
}

// Word token(s) of a run of n bytes whose first 16 bytes (lowercased) are k0/k1
// and whose last bytes (newest low) are `tail`; returns the token count.
__device__ __forceinline__ uint32_t run_tokens(const Lex& L, const uint32_t* pref, uint32_t n, uint64_t k0,
                                               uint64_t k1, uint64_t tail, uint32_t& attr0, uint32_t& attr1) {
  tail = (tail | 0x2020202020202020ull) & mask_bytes(n < 6 ? n : 6);
  const uint32_t t3 = (uint32_t)(tail & 0xFFFFFFu), t2 = (uint32_t)(tail & 0xFFFFu);
  uint32_t cut = 0;
  if (n > 3 && t3 == (('n' << 16) | ('\'' << 8) | 't')) cut = 3;
  else if (n > 2 && (t2 == (('\'' << 8) | 's') || t2 == (('\'' << 8) | 'm') || t2 == (('\'' << 8) | 'd')))
    cut = 2;
  else if (n > 3 && (t3 == (('\'' << 16) | ('r' << 8) | 'e') || t3 == (('\'' << 16) | ('v' << 8) | 'e') ||
                     t3 == (('\'' << 16) | ('l' << 8) | 'l')))
    cut = 3;
  // the stem (or the whole run) on every lane, the clitic only where there is one:
  // a warp runs at most two lexicon lookups per run, whatever its lanes' mix
  const uint32_t e0 = word_idx(L, pref, n - cut, k0, k1, cut ? (uint32_t)((tail >> (8 * cut)) & 0xFFFFFFu) : t3);
  attr0 = e0 ? L.e[e0 - 1].attr : 0u;
  if (!cut) return 1;
  const uint32_t ck = cut == 3 ? __byte_perm(t3, 0, 0x4012) : __byte_perm(t2, 0, 0x4401);
  const uint32_t e1 = word_idx(L, pref, cut, (uint64_t)ck, 0ull, t3 & (cut == 3 ? 0xFFFFFFu : 0xFFFFu));
  attr1 = e1 ? L.e[e1 - 1].attr : 0u;
  return 2;
}

// word token(s) of the run of n bytes at stage byte x
__device__ __forceinline__ uint32_t stage_run(const WarpBuf& B, uint32_t x, uint32_t n, const Lex& L,
                                              const uint32_t* pref, uint32_t& at0, uint32_t& at1) {
  const uint32_t a0 = x >> 2, sh = (x & 3u) * 8u;
  const uint32_t w0 = B.stage[a0], w1 = B.stage[a0 + 1], w2 = B.stage[a0 + 2], w3 = B.stage[a0 + 3],
                 w4 = B.stage[a0 + 4];
  const uint32_t o0 = __funnelshift_r(w0, w1, sh) | 0x20202020u, o1 = __funnelshift_r(w1, w2, sh) | 0x20202020u;
  const uint32_t o2 = __funnelshift_r(w2, w3, sh) | 0x20202020u, o3 = __funnelshift_r(w3, w4, sh) | 0x20202020u;
  const uint64_t k0 = (uint64_t)o0 | ((uint64_t)o1 << 32);
  const uint64_t k1 = (uint64_t)o2 | ((uint64_t)o3 << 32);
  const uint32_t tb8 = x + n - 8;  // >= 8
  const uint32_t ta = tb8 >> 2, tsh = (tb8 & 3u) * 8u;
  const uint32_t v0 = B.stage[ta], v1 = B.stage[ta + 1], v2 = B.stage[ta + 2];
  const uint32_t lo8 = __funnelshift_r(v0, v1, tsh), hi8 = __funnelshift_r(v1, v2, tsh);
  const uint64_t tl = ((uint64_t)__byte_perm(hi8, 0, 0x0123) | ((uint64_t)__byte_perm(lo8, 0, 0x0123) << 32));
  return run_tokens(L, pref, n, k0, k1, tl, at0, at1);
}

// one request by the per-lane byte FSM (fallback path; kept out of line)
__device__ __noinline__ void fsm_request(const ScoreLaunch& a, const Lex& L, uint32_t r, uint32_t s, uint32_t e) {
  Rules R;
  R.init();
  for (uint32_t i = s; i < e; ++i) R.byte(__ldg(a.bytes + i), L);
  uint32_t f[8];
  bool sat;
  R.finish(L, f, sat);
  if (sat) atomicOr(a.flags, RT_FLAG_SATURATED);
  epilogue(a, r, f);
}


// rules over tokens [tb, tend) of the ring (tend - tb <= 32)
__device__ __forceinline__ void rules_batch(WarpBuf& B, int32_t tb, int32_t tend, uint32_t lane) {
  Carry cy = B.cy;
  const int32_t T = tb + (int32_t)lane;
  const bool valid = T < tend;
  uint32_t meta = 0, attr = 0;
  if (valid) { meta = B.t_meta[T & (kRing - 1)]; attr = B.t_attr[T & (kRing - 1)]; }
  const uint32_t kind = meta & 7u, req = meta >> 3;
  // three predecessors (same request only): shuffles within the batch, and a
  // halo of the three tokens before it (lanes 0-2 load it once; 0xFF = none)
  const int32_t hT = tb - 3 + (int32_t)lane;
  uint32_t hm = 0xFFu, ha = 0;
  if (lane < 3 && hT >= 0) { hm = B.t_meta[hT & (kRing - 1)]; ha = B.t_attr[hT & (kRing - 1)]; }
  uint32_t pk[4], pa[4];
#pragma unroll
  for (int k = 1; k <= 3; ++k) {
    const uint32_t mu = __shfl_up_sync(0xFFFFFFFFu, meta, k), au = __shfl_up_sync(0xFFFFFFFFu, attr, k);
    const uint32_t src = (lane + 3u - (uint32_t)k) & 31u;  // halo lane for lanes < k
    const uint32_t mh = __shfl_sync(0xFFFFFFFFu, hm, src), ah = __shfl_sync(0xFFFFFFFFu, ha, src);
    const bool in_batch = lane >= (uint32_t)k;
    const uint32_t m = in_batch ? mu : mh, at = in_batch ? au : ah;
    const bool same = valid && (m >> 3) == req && m != 0xFFu;
    pk[k] = same ? (m & 7u) : 0u;
    pa[k] = same ? at : 0u;
  }
  const bool isW = valid && kind == K_W, isComma = valid && kind == K_COMMA;
  const bool isQ = valid && kind == K_Q, isEnd = valid && (kind == K_END || kind == K_Q);
  const bool isP = valid && kind >= K_COMMA;
  const uint32_t prev_req_lane = __shfl_up_sync(0xFFFFFFFFu, req, 1);
  const bool isRS = valid && (lane == 0 ? req != cy.prev_req : req != prev_req_lane);
  const uint32_t lt = lanemask_lt(), le = lanemask_le();
  const int32_t rstart = last_pos(__ballot_sync(0xFFFFFFFFu, isRS) & le, tb, cy.rs);
  const uint32_t b_end = __ballot_sync(0xFFFFFFFFu, isEnd);
  const int32_t lend = last_pos(b_end & lt, tb, cy.end);
  const int32_t sst = max(lend + 1, rstart);  // sentence start
  const uint32_t b_w = __ballot_sync(0xFFFFFFFFu, isW);
  const int32_t lword = last_pos(b_w & lt, tb, cy.word);
  const bool firstW = isW && lword < sst;
  const uint32_t b_fw = __ballot_sync(0xFFFFFFFFu, firstW);
  const int32_t f = last_pos(b_fw & le, tb, cy.fw);
  const bool isN = isW && (attr & A_NOUN);
  const uint32_t nid = attr >> A_ID_SHIFT;
  const uint32_t b_n = __ballot_sync(0xFFFFFFFFu, isN);
  const int32_t lnoun = last_pos(b_n & lt, tb, cy.noun);
  const bool firstN = isN && lnoun < sst;
  const uint32_t b_fn = __ballot_sync(0xFFFFFFFFu, firstN);
  const int32_t fn = last_pos(b_fn & le, tb, cy.fn);
  const uint32_t fn_id_l = __shfl_sync(0xFFFFFFFFu, nid, (uint32_t)max(fn - tb, 0) & 31u);
  const uint32_t fn_id = fn >= tb ? fn_id_l : cy.fn_id;
  const bool isD = isN && fn >= sst && nid != fn_id;
  const uint32_t b_d = __ballot_sync(0xFFFFFFFFu, isD);
  const int32_t ld = last_pos(b_d & lt, tb, cy.d);
  // structural: PREP after a second distinct noun of the sentence
  const uint32_t cS = (isW && (attr & A_PREP) && ld >= sst) ? 1u : 0u;
  // open-endedness
  uint32_t cO = (firstW && (attr & A_OPENER)) ? 1u : 0u;
  if (isW && !firstW && f >= sst && (attr & A_CAUSE)) {
    const int32_t dd = T - f;
    if (dd >= 1 && dd <= 3) {
      const uint32_t af = pa[dd == 1 ? 1 : dd == 2 ? 2 : 3];
      bool earlier = false;  // a CAUSE word between f and T
      if (dd >= 2 && pk[1] == K_W && (pa[1] & A_CAUSE)) earlier = true;
      if (dd >= 3 && pk[2] == K_W && (pa[2] & A_CAUSE)) earlier = true;
      if ((af & A_WHAT) && !earlier) cO = 1u;
    }
  }
  const uint32_t broad_l = __shfl_sync(0xFFFFFFFFu, (attr & A_BROAD) ? 1u : 0u, (uint32_t)max(lword - tb, 0) & 31u);
  const uint32_t lw_broad = lword >= tb ? broad_l : cy.word_broad;
  if (isQ && lword >= sst && lw_broad) cO += 1u;
  // content spans: coordinator between words (counted at the word after it)
  uint32_t cP = 0;
  // (non-short-circuit: no branches)
  cP = (uint32_t)(isW & (pk[1] == K_W) & ((pa[1] & A_COORD) != 0u) & ((pk[2] == K_W) | ((pk[2] == K_COMMA) & (pk[3] == K_W))));
  // comma chains: link = previous punctuation is a comma with >= 1 word between
  const uint32_t b_p = __ballot_sync(0xFFFFFFFFu, isP);
  const int32_t lp = last_pos(b_p & lt, tb, cy.punct);
  const uint32_t lpl = (uint32_t)max(lp - tb, 0) & 31u;
  const uint32_t lp_comma_l = __shfl_sync(0xFFFFFFFFu, isComma ? 1u : 0u, lpl);
  const uint32_t lp_comma = lp >= tb ? lp_comma_l : cy.punct_comma;
  const bool link = isComma && lp >= rstart && lp_comma && lp <= T - 2;
  const uint32_t lp_link_l = __shfl_sync(0xFFFFFFFFu, link ? 1u : 0u, lpl);
  const uint32_t lp_link = lp >= tb ? lp_link_l : cy.punct_link;
  if (link && !lp_link) cP += 1u;
  // per-request sums (requests are contiguous, increasing runs of lanes): the
  // 0/1 counters by popcounts of ballots over the run, the senses count M by a
  // segmented scan; the run's last lane adds them to the request's accumulators
  const uint32_t b_V = __ballot_sync(0xFFFFFFFFu, isW && (attr & A_VAGUE));
  const uint32_t b_Y = __ballot_sync(0xFFFFFFFFu, isW && ((attr >> 8) & 1u));
  const uint32_t b_S = __ballot_sync(0xFFFFFFFFu, cS != 0u), b_O = __ballot_sync(0xFFFFFFFFu, cO != 0u);
  const uint32_t b_P = __ballot_sync(0xFFFFFFFFu, cP != 0u), b_Q = __ballot_sync(0xFFFFFFFFu, isQ);
  const uint32_t b_head = __ballot_sync(0xFFFFFFFFu, valid && (lane == 0 || req != prev_req_lane));
  const int32_t head = 31 - (int32_t)__clz(b_head & le);
  uint32_t msum = isW ? (attr >> A_SEM_SHIFT) & A_SEM_MASK : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, msum, o);
    if ((int32_t)lane - o >= head) msum += up;
  }
  const uint32_t next_req = __shfl_down_sync(0xFFFFFFFFu, req, 1);
  const bool next_valid = __shfl_down_sync(0xFFFFFFFFu, valid ? 1u : 0u, 1) != 0u;
  if (valid && (lane == 31 || !next_valid || next_req != req)) {
    const uint32_t seg = le & ~((1u << head) - 1u);  // lanes head..lane
    uint32_t* a = B.acc[req];
    a[6] += __popc(seg);
    a[3] += __popc(b_V & seg);
    a[1] += __popc(b_Y & seg);
    a[0] += __popc(b_S & seg);
    a[4] += __popc(b_O & seg);
    a[5] += __popc(b_P & seg);
    a[8] += __popc(b_Q & seg);
    a[2] = min(a[2] + msum, 0xFFFFFFu);
  }
  // carries for the next batch
  const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
  if (vm) {
    const int32_t lastT = tb + 31 - (int32_t)__clz(vm);
    cy.prev_req = __shfl_sync(0xFFFFFFFFu, req, (uint32_t)(lastT - tb));
    cy.rs = last_pos(__ballot_sync(0xFFFFFFFFu, isRS), tb, cy.rs);
    cy.end = last_pos(b_end, tb, cy.end);
    if (b_w) cy.word_broad = __shfl_sync(0xFFFFFFFFu, (attr & A_BROAD) ? 1u : 0u, 31 - __clz(b_w));
    cy.word = last_pos(b_w, tb, cy.word);
    cy.fw = last_pos(b_fw, tb, cy.fw);
    cy.noun = last_pos(b_n, tb, cy.noun);
    if (b_fn) cy.fn_id = __shfl_sync(0xFFFFFFFFu, nid, 31 - __clz(b_fn));
    cy.fn = last_pos(b_fn, tb, cy.fn);
    cy.d = last_pos(b_d, tb, cy.d);
    if (b_p) {
      const uint32_t L = 31 - __clz(b_p);
      cy.punct_comma = __shfl_sync(0xFFFFFFFFu, isComma ? 1u : 0u, L);
      cy.punct_link = __shfl_sync(0xFFFFFFFFu, link ? 1u : 0u, L);
    }
    cy.punct = last_pos(b_p, tb, cy.punct);
  }
  if (lane == 0) B.cy = cy;
  __syncwarp();
}

__global__ void __launch_bounds__(kT4, 1) k_score4(ScoreLaunch a, uint32_t* work) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem4& S = *reinterpret_cast<Smem4*>(smem_raw);
  uint8_t* tail_mem = smem_raw + ((sizeof(Smem4) + 15) & ~size_t(15));
  LexEntry* s_ent = reinterpret_cast<LexEntry*>(tail_mem);
  const uint32_t ent_bytes = a.lex.n_entries * (uint32_t)sizeof(LexEntry);
  uint16_t* s_slots = reinterpret_cast<uint16_t*>(tail_mem + ((ent_bytes + 15u) & ~15u));
  const uint32_t nslots = 1u << a.lex.bits;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.lex.entries);
    uint32_t* dst = reinterpret_cast<uint32_t*>(s_ent);
    for (uint32_t i = tid; i < ent_bytes / 4; i += kT4) dst[i] = src[i];
    for (uint32_t i = tid; i < nslots; i += kT4) s_slots[i] = a.lex.slots[i];
    for (uint32_t i = tid; i < 128; i += kT4) S.pref[i] = 0;
    for (uint32_t i = tid; i < 256 * 32; i += kT4) S.lut[i] = class_bits(i >> 5);
  }
  __syncthreads();
  for (uint32_t i = tid; i < a.lex.n_entries; i += kT4) {
    const LexEntry e = a.lex.entries[i];
    const uint32_t pi = pref_idx((uint32_t)(e.k0 & 0xFFu), e.len >= 2 ? (uint32_t)((e.k0 >> 8) & 0xFFu) : 0u);
    atomicOr(&S.pref[pi >> 5], 1u << (pi & 31u));
  }
  __syncthreads();
  const Lex L{s_ent, s_slots, a.lex.bits};
  WarpBuf& B = S.w[wid];
  const uint32_t total_bytes = a.n ? a.offsets[a.n] : 0u;
  const uint32_t ntasks = (a.n + 31) / 32;
  const uint8_t* st8 = reinterpret_cast<const uint8_t*>(B.stage);
  if (lane < 4) B.stage[lane] = 0;

  for (;;) {
    uint32_t task = 0;
    if (lane == 0) task = atomicAdd(work, 1u);
    task = __shfl_sync(0xFFFFFFFFu, task, 0);
    if (task >= ntasks) break;
    const uint32_t r0 = task * 32, rcnt = min(32u, a.n - r0);
    const uint32_t r = r0 + lane;
    const bool rv = lane < rcnt;
    const uint32_t s_r = rv ? a.offsets[r] : 0u;
    const uint32_t e_r = rv ? a.offsets[r + 1] : 0u;
    const bool bad = rv && e_r < s_r;
    if (__any_sync(0xFFFFFFFFu, bad)) {
      // offsets not non-decreasing: per-lane byte FSM (requests with e < s are empty)
      if (bad) atomicOr(a.flags, RT_FLAG_BAD_OFFSETS);
      if (rv) fsm_request(a, L, r, s_r, bad ? s_r : e_r);
      continue;
    }
    // request of a byte = (# request starts at or before it) - 1; a popcount of the
    // start marks when no two requests start at the same byte (no empty request
    // in the middle), else a search of the starts
    const uint32_t s_prev = __shfl_up_sync(0xFFFFFFFFu, s_r, 1);
    const bool uniq_starts = !__any_sync(0xFFFFFFFFu, rv && lane > 0 && s_r == s_prev);
    const uint32_t B0 = __shfl_sync(0xFFFFFFFFu, s_r, 0);
    const uint32_t B1 = __shfl_sync(0xFFFFFFFFu, e_r, rcnt - 1);
    B.rs[lane] = s_r;
#pragma unroll
    for (int k = 0; k < 9; ++k) B.acc[lane][k] = 0;
    if (lane == 0) B.cy = Carry{-1, -1, -1, -1, -1, -1, -1, -1, 0u, 0u, 0u, 0u, 0xFFFFFFFFu};
    int32_t tokbase = 0;
    uint32_t prevW = 0;                 // W bit of the byte before the chunk
    int32_t pend_start = -1;            // absolute start of a run carried from earlier chunks
    const uint32_t base = B0 & ~15u;
    uint4 qprev = make_uint4(0, 0, 0, 0);
    int32_t tokdone = 0;                // tokens already through the rules
    __syncwarp();
    for (uint32_t cb = base; cb < B1; cb += kChunk) {
      // ---- (1) stage + classify 16 bytes per lane
      const uint32_t g = cb + lane * 16u;
      uint4 q;
      if (g + 16u <= total_bytes) q = ld_nc_v4(a.bytes + g);
      else {
        uint32_t w4[4] = {0, 0, 0, 0};
        for (uint32_t j = 0; j < 16u; ++j)
          if (g + j < total_bytes) w4[j >> 2] |= (uint32_t)a.bytes[g + j] << (8 * (j & 3u));
        q = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
      *reinterpret_cast<uint4*>(&B.stage[4 + lane * 4]) = qprev;
      *reinterpret_cast<uint4*>(&B.stage[4 + kChunk / 4 + lane * 4]) = q;
      qprev = q;
      if (lane < kChunk / 32 + 1) B.mk[lane] = 0;
      __syncwarp();
      if (rv && s_r >= cb && s_r < cb + kChunk && s_r < B1)
        atomicOr(&B.mk[(s_r - cb) >> 5], 1u << ((s_r - cb) & 31u));
      uint32_t accA = 0, accB = 0;
      {
        const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t byte = (wv[j * 2 + (i >> 2)] >> (8 * (i & 3))) & 0xFFu;
            const uint32_t c = S.lut[byte * 32u + lane] << i;
            if (j == 0) accA += c; else accB += c;
          }
      }
      // in-range bytes of this lane: [B0, B1)
      uint32_t vmask = 0xFFFFu;
      if (g < B0) vmask &= B0 - g >= 16u ? 0u : (0xFFFFu << (B0 - g)) & 0xFFFFu;
      if (g + 16u > B1) vmask &= B1 <= g ? 0u : (0xFFFFu >> (g + 16u - B1));
      const uint32_t W16 = ((accA & 0xFFu) | ((accB & 0xFFu) << 8)) & vmask;
      const uint32_t P16 = (((accA >> 8) & 0xFFu) | (((accB >> 8) & 0xFFu) << 8)) & vmask;
      const uint32_t X16 = (((accA >> 16) & 0xFFu) | (((accB >> 16) & 0xFFu) << 8)) & vmask;
      const uint32_t Wn = __shfl_down_sync(0xFFFFFFFFu, W16, 1);
      if (!(lane & 1u)) B.wm[lane >> 1] = W16 | (Wn << 16);
      if (lane == 0) B.wm[kChunk / 32] = 0;
      __syncwarp();
      // ---- (2) events
      const uint32_t mk16 = (B.mk[lane >> 1] >> (16u * (lane & 1u))) & 0xFFFFu;
      const uint32_t Wp = __shfl_up_sync(0xFFFFFFFFu, W16, 1);
      const uint32_t pw = lane ? (Wp >> 15) & 1u : prevW;
      uint32_t R16 = (W16 & ~((W16 << 1) | pw)) | (W16 & mk16);
      // a run reaching the chunk end continues in the next chunk
      const bool last_chunk = cb + kChunk >= B1;
      const bool defer = !last_chunk && ((__shfl_sync(0xFFFFFFFFu, W16, 31) >> 15) & 1u);
      const uint32_t b_r = __ballot_sync(0xFFFFFFFFu, R16 != 0u);
      bool pend_here = false;  // the carried run ends in this chunk
      int32_t new_pend = -1;
      if (defer) {
        if (b_r) {
          const uint32_t L2 = 31 - __clz(b_r);
          const uint32_t top = __shfl_sync(0xFFFFFFFFu, R16, L2);
          const uint32_t bit = 31 - __clz(top);
          new_pend = (int32_t)(cb + L2 * 16u + bit);
          if (lane == L2) R16 &= ~(1u << bit);
          pend_here = pend_start >= 0;
        }  // else: the carried run spans the whole chunk
      } else {
        pend_here = pend_start >= 0;
      }
      const uint32_t E16 = R16 | P16;
      const uint32_t cnt = __popc(E16);
      // one scan for the event count (low half) and the request-start count (high half)
      const uint32_t cm = cnt | ((uint32_t)__popc(mk16) << 16);
      uint32_t incl = cm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      const uint32_t ph = pend_here ? 1u : 0u;
      const uint32_t nev = (__shfl_sync(0xFFFFFFFFu, incl, 31) & 0xFFFFu) + ph;
      const uint32_t base_rq = __popc(__ballot_sync(0xFFFFFFFFu, rv && s_r < cb));  // requests started earlier
      if (E16) {
        uint32_t k = ((incl - cm) & 0xFFFFu) + ph;
        uint32_t e = E16;
        if (uniq_starts) {
          const uint32_t rq0 = base_rq + ((incl - cm) >> 16) - 1u;  // + starts in this lane up to the byte
          while (e) {
            const uint32_t bit = __ffs(e) - 1;
            e &= e - 1u;
            B.ev[k] = (uint16_t)(lane * 16u + bit);
            B.evq[k++] = (uint8_t)(rq0 + __popc(mk16 & ((2u << bit) - 1u)));
          }
        } else {
          uint32_t rq = req_of(B.rs, rcnt, g);  // request at this lane's first byte, advanced per event
          while (e) {
            const uint32_t bit = __ffs(e) - 1;
            e &= e - 1u;
            while (rq + 1 < rcnt && B.rs[rq + 1] <= g + bit) ++rq;
            B.ev[k] = (uint16_t)(lane * 16u + bit);
            B.evq[k++] = (uint8_t)rq;
          }
        }
      }
      if (lane == 0 && ph) B.ev[0] = 0xFFFFu;
      __syncwarp();
      // ---- (3) tokens, 32 events at a time, then (4) rules
      // (at least one pass, so that the last chunk always flushes the rules)
      for (uint32_t e0 = 0; e0 < max(nev, 1u); e0 += 32) {
        const uint32_t k = e0 + lane;
        uint32_t ntk = 0, at0 = 0, at1 = 0, kind = K_W, rq = 0;
        if (k < nev) {
          const uint32_t p = B.ev[k];
          uint32_t x = 0, n = 0;
          bool isrun = false;
          if (p == 0xFFFFu) {
            // carried run: [pend_start, stop) with stop the first non-word byte or request start here
            const uint32_t ps = (uint32_t)pend_start;
            uint32_t stop = 0;
            for (uint32_t w = 0;; ++w) {
              const uint32_t sm = ~B.wm[w] | B.mk[w];
              if (sm) { stop = w * 32 + __ffs(sm) - 1; break; }
            }
            n = cb + stop - ps;
            rq = req_of(B.rs, rcnt, ps);
            isrun = true;
            if (ps + kChunk >= cb) {
              x = 16 + kChunk + ps - cb;
            } else {
              // longer than a chunk (> 512 bytes): its tokens depend only on its last
              // 6 bytes (any stem is > 16 bytes, no lemma) -> stage them as a 24-byte run
              const uint32_t pad = 16 + 2 * kChunk + 8;  // in the stage's tail padding
              uint8_t* st = reinterpret_cast<uint8_t*>(B.stage);
              for (uint32_t j = 0; j < 8u; ++j) st[pad + j] = __ldg(a.bytes + ps + n - 8 + j);
              x = pad + 8 - 24;
              n = 24;
            }
          } else {
            const uint32_t c = st8[16 + kChunk + p];
            rq = B.evq[k];
            if ((B.wm[p >> 5] >> (p & 31u)) & 1u) {
              // run length: up to the first non-word byte or request start
              uint32_t qq = p + 1;
              n = 1;
              for (;;) {
                const uint32_t qw = qq >> 5, qb = qq & 31u;
                const uint32_t stop = (~B.wm[qw] | B.mk[qw]) >> qb;
                if (stop) { n += __ffs(stop) - 1; break; }
                n += 32 - qb;
                qq += 32 - qb;
              }
              x = 16 + kChunk + p;
              isrun = true;
            } else {
              ntk = 1;
              kind = c == ',' ? K_COMMA : (c == '.' || c == '!') ? K_END : c == '?' ? K_Q : K_OTH;
            }
          }
          if (isrun) ntk = stage_run(B, x, n, L, S.pref, at0, at1);
        }
        uint32_t ti = ntk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, ti, o);
          if (lane >= (uint32_t)o) ti += t;
        }
        const uint32_t nt = __shfl_sync(0xFFFFFFFFu, ti, 31);
        if (ntk) {
          const uint32_t t0 = (uint32_t)tokbase + ti - ntk;
          B.t_meta[t0 & (kRing - 1)] = (uint8_t)(kind | (rq << 3));
          B.t_attr[t0 & (kRing - 1)] = at0;
          if (ntk == 2) {
            B.t_meta[(t0 + 1) & (kRing - 1)] = (uint8_t)(K_W | (rq << 3));
            B.t_attr[(t0 + 1) & (kRing - 1)] = at1;
          }
        }
        __syncwarp();
        tokbase += (int32_t)nt;
        // full 32-token batches; everything after the last event of the task
        const int32_t lim = (last_chunk && e0 + 32 >= nev) ? tokbase : tokbase - 31;
        for (; tokdone < lim; tokdone += 32) rules_batch(B, tokdone, min(tokdone + 32, tokbase), lane);
        __syncwarp();
      }
      // dropped bytes (rare): count per request
      if (__any_sync(0xFFFFFFFFu, X16 != 0u)) {
        uint32_t xm = X16;
        while (xm) {
          const uint32_t bit = __ffs(xm) - 1;
          xm &= xm - 1u;
          atomicAdd(&B.acc[req_of(B.rs, rcnt, g + bit)][7], 1u);
        }
      }
      if (pend_here) pend_start = -1;
      if (defer && b_r) pend_start = new_pend;
      prevW = (__shfl_sync(0xFFFFFFFFu, W16, 31) >> 15) & 1u;
      __syncwarp();
    }
    // ---- epilogue: lane = request
    if (rv) {
      const uint32_t* ac = B.acc[lane];
      uint32_t a9[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) a9[k] = ac[k];
      uint32_t f[8];
      bool sat;
      Rules::finish_acc(a9, f, sat);
      if (sat) atomicOr(a.flags, RT_FLAG_SATURATED);
      epilogue(a, r, f);
    }
    __syncwarp();
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


cudaError_t launch_score(const ScoreLaunch& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const size_t smem = ((sizeof(Smem4) + 15) & ~size_t(15)) + ((a.lex.n_entries * sizeof(LexEntry) + 15) & ~size_t(15)) +
                      (((size_t(1) << a.lex.bits) * 2 + 15) & ~size_t(15));
  cudaError_t e = cudaFuncSetAttribute(k_score4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.work, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const uint32_t ntasks = (a.n + 31) / 32;
  uint32_t grid = (uint32_t)a.num_sms;
  if (grid * kW4 > ntasks) grid = (ntasks + kW4 - 1) / kW4;
  k_score4<<<grid, kT4, smem, s>>>(a, a.work);
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
