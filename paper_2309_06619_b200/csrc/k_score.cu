// k_score.cu — K1 (RuleGen: tokenize, lemmatize, lexicon probe, six rule
// scorers) fused with K2 (weighted-rule regression, deadline, priority key,
// offload class).  §8(a) rows a1-a4.
//
// Design (DESIGN.md §7 K1, kernel k_score6): persistent CTAs of 32 warps.  A
// warp takes warp tasks of 32 consecutive requests from a global work counter
// and tokenizes up to 16 of them into a per-warp token buffer (a pool): 512-byte
// chunks staged in shared memory, byte classes and word-run starts as bit
// masks, one lane per token event (run -> clitic split, lemma, two-choice
// lexicon probe).  Then every lane runs the sequential rule machine over a
// contiguous range of whole requests of the pool, and the epilogue computes u
// and the key per request and writes 4 B + 8 B (+ optional 16 B feature row).
// The lexicon (<= 1024 lemmas) lives in shared memory as a fingerprinted
// two-choice table.  All arithmetic that decides an integer is binary32 with
// explicit round-to-nearest intrinsics (R-FP).  Tasks with decreasing offsets
// or more bytes than a pool buffer use the per-lane byte FSM (Rules::byte),
// which implements the same rules sequentially.
#include "internal.cuh"

// RTLM_CHECK builds (scripts/build_variant.sh with EXTRA_NVCC=-DRTLM_CHECK): bounds
// of every computed shared / scratch index in k_score6 are checked, a violation
// traps (the call then fails with a CUDA error)
#ifdef RTLM_CHECK
#define KS_CHECK(c) do { if (!(c)) __trap(); } while (0)
#else
#define KS_CHECK(c) do { } while (0)
#endif

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
// Two-choice hashing (DevLexicon): a lemma is at one of its two slots; keys
// are zero-padded 16-byte words (lemma bytes are never 0, so the padding
// encodes the length), keys[0] = 0 so an empty slot never matches a lemma.
struct Lex {
  const uint4* keys;        // shared memory
  const uint32_t* slots;    // shared memory
  const LexEntry* e;        // global (attributes, byte-FSM path only)
  uint32_t bits, seed;
};

// token code (entry index + 1, 0 = not in the lexicon) of a zero-padded lemma:
// the slot whose fingerprint matches names the one key compared (a second
// compare only when both fingerprints match and the first key differs)
__device__ __forceinline__ uint32_t lookup(const Lex& L, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  const uint32_t x = lex_mix(w0, w1, w2, w3, L.seed), fp = lex_fp(x);
  const uint32_t v1 = L.slots[lex_slot1(x, L.bits)], v2 = L.slots[lex_slot2(x, L.bits)];
  const bool f1 = (v1 >> 11) == fp, f2 = (v2 >> 11) == fp;
  const uint32_t c = f1 ? (v1 & 0x7FFu) : (f2 ? (v2 & 0x7FFu) : 0u);
  KS_CHECK(c <= 1024u);
  const uint4 k = L.keys[c];
  const bool m = ((k.x ^ w0) | (k.y ^ w1) | (k.z ^ w2) | (k.w ^ w3)) == 0u;
  uint32_t code = m ? c : 0u;
  if (__builtin_expect(f1 && f2 && !m, 0)) {
    const uint32_t c2 = v2 & 0x7FFu;
    const uint4 k2 = L.keys[c2];
    code = ((k2.x ^ w0) | (k2.y ^ w1) | (k2.z ^ w2) | (k2.w ^ w3)) == 0u ? c2 : 0u;
  }
  return code;
}

__device__ __forceinline__ uint32_t probe(const Lex& L, uint64_t k0, uint64_t k1, uint32_t len) {
  (void)len;  // zero padding encodes the length
  const uint32_t c = lookup(L, (uint32_t)k0, (uint32_t)(k0 >> 32), (uint32_t)k1, (uint32_t)(k1 >> 32));
  return c ? L.e[c - 1].attr : 0u;
}

__device__ __forceinline__ uint64_t mask_bytes(uint32_t nbytes) {  // nbytes in 0..8
  return nbytes >= 8 ? ~0ull : ((1ull << (8 * nbytes)) - 1ull);
}

// Lemma attributes of a word token of length L whose first bytes (lowercased,
// little-endian) are k0/k1 (valid up to min(L,16)) and whose last three bytes
// are s3 = b[L-3]<<16 | b[L-2]<<8 | b[L-1].  R-LEMMA.  (byte-FSM path)
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

// Token code of a word token (R-LEMMA): len bytes, first 16 (lowercased) in
// o0..o3, last three s3 = b[len-3]<<16 | b[len-2]<<8 | b[len-1]; branch-free.
__device__ __forceinline__ uint32_t word_code(const Lex& L, uint32_t len, uint32_t o0, uint32_t o1, uint32_t o2,
                                              uint32_t o3, uint32_t s3) {
  constexpr uint32_t NT = ('n' << 16) | ('\'' << 8) | 't';
  const uint32_t b1 = s3 & 0xFFu, b2 = (s3 >> 8) & 0xFFu, b3 = s3 >> 16;
  uint32_t strip = 0;
  if (len >= 3 && b1 == 's' && b2 != 's') strip = 1;
  if (len >= 4 && b2 == 'e' && (b1 == 'd' || b1 == 's')) strip = 2;
  if (len >= 5 && b3 == 'i' && b2 == 'n' && b1 == 'g') strip = 3;
  const bool nt = len == 3 && s3 == NT;  // n't -> not
  const uint32_t ll = nt ? 3u : len - strip;
  if (nt) o0 = 'n' | ('o' << 8) | ('t' << 16);
  const int32_t sh = ll > 16u ? 0 : 8 * (int32_t)ll;  // lemma bytes kept (0: no lemma -> code 0)
  o0 &= __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(sh, 0));
  o1 &= __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(sh - 32, 0));
  o2 &= __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(sh - 64, 0));
  o3 &= __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(sh - 96, 0));
  return lookup(L, o0, o1, o2, o3);
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

// ============================================================ helpers of the scorer
__device__ __forceinline__ uint32_t class_bits(uint32_t b) {
  const uint32_t lc = b | 0x20u;
  const bool w = (lc - 'a' < 26u) || (b - '0' < 10u) || b == '\'';
  const bool sp = b == ' ' || (b - 9u) < 5u;
  const bool p = !w && (b - 0x21u < 0x5Eu);
  return w ? 0x1u : (p ? 0x100u : (sp ? 0u : 0x10000u));
}

// token kind of a punctuation byte (K_* below; 0 for other bytes).  The class
// table carries it in bits 24..26: classify's shifted sums of 8 bytes only
// spill upwards from there, so the W / P / X fields stay exact
__device__ __forceinline__ uint32_t punct_kind(uint32_t b) {
  if (!(class_bits(b) & 0x100u)) return 0u;
  return b == ',' ? 2u : (b == '.' || b == '!') ? 3u : b == '?' ? 4u : 5u;
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

// ============================================================ K1 (shared pieces)
constexpr uint32_t kT4 = 1024;                // threads per CTA (32 warps)
constexpr uint32_t kW4 = kT4 / 32;
constexpr uint32_t kChunk = 1024;             // bytes per warp chunk (32 per lane)
constexpr uint32_t kCB = 64;                  // stage byte of the chunk's first byte (32 B pad, previous chunk's last 32 B)

// Token codes (u16 in the per-warp token buffer): 0 a word outside the
// lexicon, 1..1024 a word with lexicon entry code-1, kPunct + PK_* a
// punctuation token.
enum : uint32_t { PK_COMMA = 1, PK_END = 2, PK_Q = 3, PK_OTH = 4 };
constexpr uint32_t kPunct = 1024;

// request index of absolute byte position pos: last i < cnt with rs[i] <= pos
__device__ __forceinline__ uint32_t req_of(const uint32_t* rs, uint32_t cnt, uint32_t pos) {
  uint32_t lo = 0;
#pragma unroll
  for (uint32_t st = 16; st; st >>= 1)
    if (lo + st < cnt && rs[lo + st] <= pos) lo += st;
  return lo;
}

// The seven clitics of R-CLITIC in a fixed order: n't 're 've 'll 's 'm 'd.
// A clitic token's lemma (R-LEMMA: n't -> not; the others are too short or
// end in no suffix) and so its lexicon code depend only on which clitic it is:
// the codes are looked up once per CTA (Smem6::clit, Smem6::cl3 / cl2).
__host__ __device__ __forceinline__ uint32_t clitic_bytes(uint32_t kind) {
  switch (kind) {
    case 0: return 'n' | ('\'' << 8) | ('t' << 16);
    case 1: return '\'' | ('r' << 8) | ('e' << 16);
    case 2: return '\'' | ('v' << 8) | ('e' << 16);
    case 3: return '\'' | ('l' << 8) | ('l' << 16);
    case 4: return '\'' | ('s' << 8);
    case 5: return '\'' | ('m' << 8);
    default: return '\'' | ('d' << 8);
  }
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


// ---- R-RULES as a finite-state machine (O2 in the sequential form of
// Rules::on_word / on_punct).  The machine's context equals the fresh one at
// every request start, and the counts are sums per request.  Three
// independent parts (each rule reads only its own part's context):
//  * O-part (open-endedness): context SWORD (a word seen in the sentence),
//    BROAD (last word BROAD), wcd (what-countdown 0..3) -> 16 states; token
//    class: word with flags {OPENER, WHAT, CAUSE, BROAD} (0..15), '?' (16),
//    '.' '!' (17), other punctuation (18); o_step = next state | O increment << 4.
//  * P-part (multi-part): context PW, PC, P2W (previous two token kinds),
//    CPEND (coordinator after a word), WSC (word since the last comma), chain
//    (0..2) -> 7 bits; token class: word (0), COORD word (1), comma (2), other
//    punctuation (3); p_step = next | P increment << 7.
//  * S-part (structural): first noun id of the sentence and NOUN2 (a second
//    distinct noun seen), in registers.
enum : uint32_t { OC_Q = 16, OC_END = 17, OC_PUNCT = 18 };
enum : uint32_t { PC_WORD = 0, PC_COORD = 1, PC_COMMA = 2, PC_PUNCT = 3 };

// O-part transition (Rules::on_word / on_punct restricted to SENT_WORD, LAST_BROAD, what_cd)
__host__ __device__ __forceinline__ uint32_t o_step(uint32_t st, uint32_t cls) {
  const uint32_t sword = st & 1u, broad = (st >> 1) & 1u, wcd = st >> 2;
  if (cls < 16u) {  // word
    const bool first = !sword, cause = sword && wcd && (cls & 4u);
    const uint32_t inc = ((first && (cls & 1u)) || cause) ? 1u : 0u;
    const uint32_t w2 = first ? ((cls & 2u) ? 3u : 0u) : ((cause || !wcd) ? 0u : wcd - 1u);
    return 1u | (((cls >> 3) & 1u) << 1) | (w2 << 2) | (inc << 4);
  }
  if (cls == OC_Q) return ((sword && broad) ? 1u : 0u) << 4;  // broad-scope interrogative; sentence ends
  if (cls == OC_END) return 0u;
  return sword | (broad << 1) | ((wcd ? wcd - 1u : 0u) << 2);
}

// P-part transition: bits 0 PW, 1 PC, 2 P2W, 3 CPEND, 4 WSC, 5..6 chain
__host__ __device__ __forceinline__ uint32_t p_step(uint32_t st, uint32_t cls) {
  const uint32_t pw = st & 1u, pc = (st >> 1) & 1u, p2w = (st >> 2) & 1u, cp = (st >> 3) & 1u, wsc = (st >> 4) & 1u,
                 ch = (st >> 5) & 3u;
  if (cls == PC_WORD || cls == PC_COORD) {
    const uint32_t cp2 = (cls == PC_COORD && (pw || (pc && p2w))) ? 1u : 0u;
    return 1u | (pw << 2) | (cp2 << 3) | (1u << 4) | (ch << 5) | (cp << 7);
  }
  if (cls == PC_COMMA) {
    const uint32_t inc = (ch == 1u && wsc) ? 1u : 0u;
    const uint32_t ch2 = (ch && wsc) ? 2u : 1u;
    return (1u << 1) | (pw << 2) | (ch2 << 5) | (inc << 7);
  }
  return (pw << 2) | (wsc << 4);
}

// ============================================================ K1 v6 (round 2): pools of tasks
// Two phases per warp, both with (almost) every lane busy:
//  (A) tokenize: up to kPoolTasks warp tasks (32 requests each) are streamed
//      (classify, events, one lane per event); a token's code goes to a
//      per-warp token buffer in global memory (u16, kTokCap tokens; the pool's
//      tokens are contiguous there) and each request's first token index is
//      recorded.  The event path is branch-free: the clitic split (R-CLITIC)
//      by perfect hashes of the run's last three / two bytes, the lemma
//      (R-LEMMA) from the stem's last four bytes and its length, masks from a
//      table, then the fingerprinted two-choice probe; punctuation lanes run
//      the same instructions and keep their punctuation code.
//  (B) rules: the pool's requests with tokens are cut into 32 contiguous
//      ranges of about equal token count (request granularity, so no request
//      is shared by two lanes); every lane runs the sequential R-RULES
//      machine over its tokens, one token per step, reading them from the
//      global buffer (L1/L2-resident: written microseconds earlier by the same
//      warp).  A request's counts live in registers until its last token
//      (16-bit fields: a pool holds <= kTokCap < 2^16 tokens) and then go to
//      its 16-byte record in the warp's scratch; the epilogue (u, key) runs
//      lane-parallel per pool.
// Tasks whose bytes exceed kTokCap (tokens <= bytes) and tasks with decreasing
// offsets use the per-lane byte FSM.
constexpr uint32_t kPoolTasks = 8;
constexpr uint32_t kPoolReq = kPoolTasks * 32;
constexpr uint32_t kTokCap = 16384;   // tokens per warp buffer
constexpr uint32_t kTokPad = 64;      // read-ahead slack
// per-warp global scratch: kTokCap + kTokPad tokens, then kPoolReq count records (16 B)
constexpr size_t kWarpScratch = (kTokCap + kTokPad) * 2 + kPoolReq * 16;

// Token attributes for the v6 machine (Smem6::fa by token code), two words
// so that every field is one or two instructions away:
//   x = O-class * 4 | (senses - 1) << 8 | noun id << 16 (0xFFFF: not a noun)
//   y = VAGUE | P-class * 4 | '?' << 8 | END << 12 | MULTIPOS << 16 | PREP << 24
//       (y & 0x10001 is added to the V | Y counter; (y >> 8) masked by 0x1 or
//       0x10001 -- "a second distinct noun seen" -- to the q | S counter)
__host__ __device__ __forceinline__ uint2 fsm_attr6(uint32_t code, uint32_t at) {
  constexpr uint32_t NONE = 0xFFFFu;
  if (code > kPunct) {
    const uint32_t pk = code - kPunct;
    if (pk == PK_COMMA) return make_uint2((OC_PUNCT * 4) | (NONE << 16), PC_COMMA * 4);
    if (pk == PK_END) return make_uint2((OC_END * 4) | (NONE << 16), (PC_PUNCT * 4) | (1u << 12));
    if (pk == PK_Q) return make_uint2((OC_Q * 4) | (NONE << 16), (PC_PUNCT * 4) | (1u << 12) | (1u << 8));
    return make_uint2((OC_PUNCT * 4) | (NONE << 16), PC_PUNCT * 4);
  }
  if (code == 0u) return make_uint2(NONE << 16, PC_WORD * 4);
  const uint32_t oc = ((at & A_OPENER) ? 1u : 0u) | ((at & A_WHAT) ? 2u : 0u) | ((at & A_CAUSE) ? 4u : 0u) |
                      ((at & A_BROAD) ? 8u : 0u);
  const uint32_t nid = (at & A_NOUN) ? ((at >> A_ID_SHIFT) & 0x3FFu) : NONE;
  return make_uint2((oc * 4) | (((at >> A_SEM_SHIFT) & A_SEM_MASK) << 8) | (nid << 16),
                    ((at & A_VAGUE) ? 1u : 0u) | (((at & A_COORD) ? PC_COORD : PC_WORD) * 4) |
                        ((at & A_MULTIPOS) ? 0x10000u : 0u) | ((at & A_PREP) ? 0x1000000u : 0u));
}

struct __align__(16) WarpBuf6 {
  union {
    struct {
      uint32_t stage[(kCB + kChunk + 32) / 4 + 4];  // 32 B pad | previous chunk's last 32 B | chunk | pad
      uint32_t mk[kChunk / 32 + 1];
      uint32_t sp[kChunk / 32 + 2];
      uint32_t rs[32];
      uint16_t ev[kChunk + 2];
    } t;                                     // phase A
    struct {
      uint16_t ids[kPoolReq + 1];            // requests with tokens, in order
      uint16_t ends[kPoolReq + 1];           // their end token index
    } q;                                     // phase B
  };
  uint16_t nd[kPoolReq];                     // dropped bytes per request (<= task bytes <= kTokCap)
  uint16_t tbeg[kPoolReq + 2];               // first token of each request in the pool buffer
  uint32_t task[kPoolTasks];
};

struct Smem6 {
  uint32_t lut[256];
  uint32_t clit[8];
  uint2 cl3[8], cl2[8];                // clitic patterns (last 3 / 2 bytes) -> token code, see clitic_hash3/2
  uint4 lmask[18];                     // lemma byte masks for lengths 0..16 (17: none)
  uint2 fa[kPunct + 8];                // rule-machine attributes by token code (fsm_attr6)
  uint32_t tO[16 * 32], tP[128 * 4];   // transitions: next row byte offset | increment << 16
  WarpBuf6 w[kW4];
};

// Perfect hashes of the R-CLITIC patterns (lowercased little-endian bytes):
// n't 're 've 'll -> slots 5 6 1 4 of 8; 's 'm 'd -> slots 0 5 6 of 8.
__host__ __device__ __forceinline__ uint32_t clitic_hash3(uint32_t h) { return (h * 0x165667B1u) >> 29; }
__host__ __device__ __forceinline__ uint32_t clitic_hash2(uint32_t h) { return (h * 0x9E3779B1u) >> 29; }

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

// Tokenize one warp task (requests r0 .. r0+rcnt-1, bytes [B0, B1)) into the
// pool: tokens appended at gt[tok ..]; request lr0 + i's first token index in
// tbeg.  A request's first token index is counted at the chunk holding its
// first byte: the tokens before the chunk + the events of the chunk before
// that byte (+ one per clitic split among them); requests without tokens get
// the index of the next token.
__device__ __forceinline__ void tokenize_task(const ScoreLaunch& a, const Smem6& S, WarpBuf6& B, const Lex& L,
                                              uint16_t* gt, uint32_t& tok, uint32_t lr0, uint32_t rcnt,
                                              uint32_t s_r, uint32_t e_r, bool rv, uint32_t lane,
                                              uint32_t total_bytes) {
  auto& T = B.t;
  const uint8_t* st8 = reinterpret_cast<const uint8_t*>(T.stage);
  const uint32_t B0 = __shfl_sync(0xFFFFFFFFu, s_r, 0);
  const uint32_t B1 = __shfl_sync(0xFFFFFFFFu, e_r, rcnt - 1);
  T.rs[lane] = s_r;
  B.nd[lr0 + lane] = 0;
  uint32_t tb = 0xFFFFFFFFu;          // this lane's request: first token index (pool)
  uint32_t prevW = 0;
  int32_t pend_start = -1;
  const uint32_t base = B0 & ~15u;
  uint4 qa = make_uint4(0, 0, 0, 0), qb = qa;  // this lane's 32 bytes of the current chunk
  if (lane < 8) T.stage[lane] = 0;
  __syncwarp();
  for (uint32_t cb = base; cb < B1; cb += kChunk) {
    // ---- (1) stage + classify 32 bytes per lane (the previous chunk keeps its
    // last 32 bytes at stage bytes 32..63, where a carried run's bytes are)
    if (lane == 31) {
      *reinterpret_cast<uint4*>(&T.stage[8]) = qa;
      *reinterpret_cast<uint4*>(&T.stage[12]) = qb;
    }
    const uint32_t g = cb + lane * 32u;
    if (g + 32u <= total_bytes) {
      qa = ld_nc_v4(a.bytes + g);
      qb = ld_nc_v4(a.bytes + g + 16u);
    } else {
      uint32_t w8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (uint32_t j = 0; j < 32u; ++j)
        if (g + j < total_bytes) w8[j >> 2] |= (uint32_t)a.bytes[g + j] << (8 * (j & 3u));
      qa = make_uint4(w8[0], w8[1], w8[2], w8[3]);
      qb = make_uint4(w8[4], w8[5], w8[6], w8[7]);
    }
    __syncwarp();
    *reinterpret_cast<uint4*>(&T.stage[kCB / 4 + lane * 8]) = qa;
    *reinterpret_cast<uint4*>(&T.stage[kCB / 4 + lane * 8 + 4]) = qb;
    T.mk[lane] = 0;
    if (lane == 0) T.mk[32] = 0;
    __syncwarp();
    const bool here = rv && s_r >= cb && s_r < cb + kChunk;  // this lane's request starts in the chunk
    if (here && s_r < B1) atomicOr(&T.mk[(s_r - cb) >> 5], 1u << ((s_r - cb) & 31u));
    uint32_t acc[4] = {0, 0, 0, 0};
    {
      const uint32_t wv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[j] += S.lut[(wv[j * 2 + (i >> 2)] >> (8 * (i & 3))) & 0xFFu] << i;
    }
    uint32_t vmask = 0xFFFFFFFFu;
    if (g < B0) vmask &= B0 - g >= 32u ? 0u : (0xFFFFFFFFu << (B0 - g));
    if (g + 32u > B1) vmask &= B1 <= g ? 0u : (0xFFFFFFFFu >> (g + 32u - B1));
    const uint32_t W32 = ((acc[0] & 0xFFu) | ((acc[1] & 0xFFu) << 8) | ((acc[2] & 0xFFu) << 16) | (acc[3] << 24)) & vmask;
    const uint32_t P32 = (((acc[0] >> 8) & 0xFFu) | (acc[1] & 0xFF00u) | ((acc[2] & 0xFF00u) << 8) |
                          ((acc[3] & 0xFF00u) << 16)) & vmask;
    const uint32_t X32 = (((acc[0] >> 16) & 0xFFu) | ((acc[1] >> 8) & 0xFF00u) | (acc[2] & 0xFF0000u) |
                          ((acc[3] & 0xFF0000u) << 8)) & vmask;
    __syncwarp();
    // ---- (2) events: run starts and punctuation bytes, in byte order
    const uint32_t mk32 = T.mk[lane];
    T.sp[lane] = ~W32 | mk32;  // run stops: a non-word byte or a request start
    if (lane < 2) T.sp[32 + lane] = 0xFFFFFFFFu;
    const uint32_t Wp = __shfl_up_sync(0xFFFFFFFFu, W32, 1);
    const uint32_t pw = lane ? (Wp >> 31) : prevW;
    uint32_t R32 = (W32 & ~((W32 << 1) | pw)) | (W32 & mk32);
    const bool last_chunk = cb + kChunk >= B1;
    const bool defer = !last_chunk && (__shfl_sync(0xFFFFFFFFu, W32, 31) >> 31);
    const uint32_t b_r = __ballot_sync(0xFFFFFFFFu, R32 != 0u);
    const bool pend_here = pend_start >= 0 && (!defer || b_r);  // the carried run ends in this chunk
    int32_t new_pend = -1;
    if (defer && b_r) {  // the last run start of the chunk is carried into the next chunk
      const uint32_t L2 = 31 - __clz(b_r);
      const uint32_t top = __shfl_sync(0xFFFFFFFFu, R32, L2);
      const uint32_t bit = 31 - __clz(top);
      new_pend = (int32_t)(cb + L2 * 32u + bit);
      if (lane == L2) R32 &= ~(1u << bit);
    }
    const uint32_t E32 = R32 | P32;
    uint32_t incl = __popc(E32);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    const uint32_t ph = pend_here ? 1u : 0u;
    const uint32_t nev = __shfl_sync(0xFFFFFFFFu, incl, 31) + ph;
    const uint32_t excl = incl - __popc(E32) + ph;  // events before this lane's bytes
    {
      uint32_t k = excl, e = E32;
      while (e) {
        const uint32_t bit = __ffs(e) - 1;
        e &= e - 1u;
        KS_CHECK(k < kChunk + 2u);
        T.ev[k++] = (uint16_t)(lane * 32u + bit);
      }
    }
    if (lane == 0 && ph) T.ev[0] = 0xFFFFu;
    // first event index of this lane's request (starting in the chunk)
    uint32_t fe = 0xFFFFFFFFu;
    {
      const uint32_t off = s_r - cb, Lr = (off >> 5) & 31u;
      const uint32_t exL = __shfl_sync(0xFFFFFFFFu, excl, Lr), EL = __shfl_sync(0xFFFFFFFFu, E32, Lr);
      if (here) {
        fe = exL + __popc(EL & ((1u << (off & 31u)) - 1u));
        tb = tok + fe;
      }
    }
    __syncwarp();
    // the carried run: [pend_start, first stop of the chunk)
    uint32_t cx = 0, cn = 0;
    if (pend_here) {
      const uint32_t ps = (uint32_t)pend_start;
      uint32_t stop = 0;
      for (uint32_t w = 0;; ++w) {
        KS_CHECK(w < kChunk / 32 + 2u);
        const uint32_t sm = T.sp[w];
        if (sm) { stop = w * 32 + __ffs(sm) - 1; break; }
      }
      cn = cb + stop - ps;
      if (ps + 32u >= cb) {
        cx = kCB + ps - cb;  // starts in the previous chunk's last 32 bytes
      } else {
        // longer than 32 bytes: its tokens depend only on its last 6 bytes (any
        // stem is > 16 bytes, no lemma) -> the 24-byte run that ends where it ends
        cx = kCB + stop - 24u;
        cn = 24u;
      }
    }
    // ---- (3) tokens, 32 events at a time (branch-free; punctuation lanes
    // compute a discarded word path)
    for (uint32_t e0 = 0; e0 < nev; e0 += 32) {
      const uint32_t k = e0 + lane;
      const bool valid = k < nev;
      KS_CHECK(!valid || k < kChunk + 2u);
      const uint32_t pe = valid ? T.ev[k] : 0u;
      const bool carried = pe == 0xFFFFu;
      const uint32_t p = pe & 1023u;
      const uint32_t lc = S.lut[st8[kCB + p]];
      const bool isw = carried || (lc & 1u);
      const uint32_t qq = p + 1, qw = qq >> 5, qb = qq & 31u;
      KS_CHECK(qw + 1u < kChunk / 32 + 2u);
      const uint32_t st = __funnelshift_r(T.sp[qw], T.sp[qw + 1], qb);  // stops after p (sp[16], sp[17]: all ones)
      uint32_t n = __ffs(st);
      if (__any_sync(0xFFFFFFFFu, st == 0u && valid && isw && !carried)) {  // run of > 32 bytes (rare)
        if (st == 0u) {  // st held bits qq .. qq+31: the rest of word qw+1, then whole words
          const uint32_t hi = T.sp[qw + 1] >> qb;
          if (hi) {
            n = 32u + __ffs(hi);
          } else {
            n = 65u - qb;
            for (uint32_t w = qw + 2;; ++w) {
              KS_CHECK(w < kChunk / 32 + 2u);
              const uint32_t stop = T.sp[w];
              if (stop) { n += __ffs(stop) - 1; break; }
              n += 32u;
            }
          }
        }
      }
      const uint32_t x = carried ? cx : kCB + p;
      n = carried ? cn : n;
      // last eight bytes of the run (lowercased): Th = b[n-4] | .. | b[n-1] << 24, Tlo = b[n-8] .. b[n-5]
      const uint32_t te = x + n - 8u, ta = te >> 2, tsh = (te & 3u) * 8u;
      KS_CHECK(ta + 2u < sizeof(T.stage) / 4);
      const uint32_t v0 = T.stage[ta], v1 = T.stage[ta + 1], v2 = T.stage[ta + 2];
      const uint32_t Tlo = __funnelshift_r(v0, v1, tsh) | 0x20202020u, Th = __funnelshift_r(v1, v2, tsh) | 0x20202020u;
      // R-CLITIC: the run's last three / two bytes against the seven clitics
      // (perfect hashes, branch-free); the stem keeps n - cut bytes
      constexpr uint32_t NT = 'n' | ('\'' << 8) | ('t' << 16);
      const uint32_t h3 = Th >> 8, h2 = Th >> 16;
      const uint2 e3 = S.cl3[clitic_hash3(h3)], e2 = S.cl2[clitic_hash2(h2)];
      const bool m3 = isw && n > 3u && e3.x == h3, m2 = isw && n > 2u && e2.x == h2;
      const uint32_t cut = m3 ? 3u : (m2 ? 2u : 0u);
      const uint32_t c1 = m3 ? e3.y : e2.y;
      const uint32_t ns = n - cut;
      const uint32_t Tl = __funnelshift_rc(Tlo, Th, 8u * (4u - cut));  // the stem's last four bytes
      const bool nt3 = ns == 3u && (Tl >> 8) == NT;  // the word n't: lemma "not" (R-LEMMA)
      // R-LEMMA of the (stem) word: first rule wins (ing > ed / es > s)
      const uint32_t a0 = x >> 2, sh = (x & 3u) * 8u;
      KS_CHECK(a0 + 4u < sizeof(T.stage) / 4);
      const uint32_t w0 = T.stage[a0], w1 = T.stage[a0 + 1], w2 = T.stage[a0 + 2], w3 = T.stage[a0 + 3],
                     w4 = T.stage[a0 + 4];
      const uint32_t t2 = Tl >> 16, t3 = Tl >> 8, b1 = Tl >> 24;
      uint32_t strip = (ns >= 3u && b1 == 's' && (t2 & 0xFFu) != 's') ? 1u : 0u;
      strip = (ns >= 4u && (t2 == ('e' | ('d' << 8)) || t2 == ('e' | ('s' << 8)))) ? 2u : strip;
      strip = (ns >= 5u && t3 == ('i' | ('n' << 8) | ('g' << 16))) ? 3u : strip;
      const uint4 mk = S.lmask[min(ns - strip, 17u)];  // lemma bytes kept (none above 16)
      const uint32_t o0 = nt3 ? ('n' | ('o' << 8) | ('t' << 16)) : ((__funnelshift_r(w0, w1, sh) | 0x20202020u) & mk.x);
      const uint32_t o1 = (__funnelshift_r(w1, w2, sh) | 0x20202020u) & mk.y;
      const uint32_t o2 = (__funnelshift_r(w2, w3, sh) | 0x20202020u) & mk.z;
      const uint32_t o3 = (__funnelshift_r(w3, w4, sh) | 0x20202020u) & mk.w;
      const uint32_t cw = lookup(L, o0, o1, o2, o3);
      const uint32_t c0 = isw ? cw : kPunct + (lc >> 24) - 1u;
      // token positions: one token per event, two for a clitic split
      const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, valid && cut != 0u);
      if (valid) {
        const uint32_t t0 = tok + lane + __popc(b2 & ((1u << lane) - 1u));
        KS_CHECK(t0 + 1u < kTokCap + kTokPad);
        gt[t0] = (uint16_t)c0;
        if (cut) gt[t0 + 1] = (uint16_t)c1;
      }
      if (b2) {  // requests whose first event follows a split start one token later
        uint32_t m = b2;
        while (m) {
          const uint32_t c = __ffs(m) - 1;
          m &= m - 1u;
          if (fe != 0xFFFFFFFFu && fe > e0 + c) ++tb;
        }
      }
      tok += min(32u, nev - e0) + __popc(b2);
    }
    if (__any_sync(0xFFFFFFFFu, X32 != 0u)) {  // dropped bytes (rare): count per request
      uint32_t xm = X32;
      while (xm) {
        const uint32_t bit = __ffs(xm) - 1;
        xm &= xm - 1u;
        atomicAdd(reinterpret_cast<uint32_t*>(&B.nd[(lr0 + req_of(T.rs, rcnt, g + bit)) & ~1u]),
                  1u << (16u * ((lr0 + req_of(T.rs, rcnt, g + bit)) & 1u)));
      }
    }
    if (pend_here) pend_start = -1;
    if (new_pend >= 0) pend_start = new_pend;
    prevW = __shfl_sync(0xFFFFFFFFu, W32, 31) >> 31;
    __syncwarp();
  }
  KS_CHECK(lr0 + lane < kPoolReq && tok <= kTokCap && (tb == 0xFFFFFFFFu || tb <= tok));
  B.tbeg[lr0 + lane] = (uint16_t)(tb == 0xFFFFFFFFu ? tok : tb);
  __syncwarp();
}

// R-RULES over the pool's tokens: lane = a contiguous range of whole requests
// of about T/32 tokens; the R-RULES machine (O-part / P-part tables,
// S-part in registers), restarted at every request start.  Requests without
// tokens are compacted away first; a request's counts go to its 16-byte record
// in the warp's global scratch when its last token has been read.  Branch-free
// per token: lanes past their range run the machine on ignored tokens.
__device__ __forceinline__ void rules_pool(const Smem6& S, WarpBuf6& B, const uint16_t* gt, uint4* gcnt, uint32_t R,
                                           uint32_t T, uint32_t lane) {
  if (lane == 0) B.tbeg[R] = (uint16_t)T;
  __syncwarp();
  auto& Q = B.q;
  uint32_t nne = 0;
  for (uint32_t b = 0; b < R; b += 32) {
    const uint32_t r = b + lane;
    const uint32_t e = B.tbeg[r + 1];
    const bool ne = e > B.tbeg[r];
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, ne);
    if (ne) {
      const uint32_t pos = nne + __popc(m & ((1u << lane) - 1u));
      Q.ids[pos] = (uint16_t)r;
      Q.ends[pos] = (uint16_t)e;
    }
    nne += __popc(m);
  }
  KS_CHECK(nne <= kPoolReq && R <= kPoolReq);
  if (lane == 0) { Q.ids[nne] = 0; Q.ends[nne] = (uint16_t)T; }
  __syncwarp();
  // this lane's entries [ja, jend): from the first entry starting at or after lane * T / 32
  uint32_t ja = 0;
  if (lane) {
    const uint32_t target = (uint32_t)(((uint64_t)T * lane + 31u) >> 5);
    uint32_t lo = 0, hi = nne;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (Q.ends[mid] < target) lo = mid + 1; else hi = mid;
    }
    ja = min(lo + 1, nne);
  }
  uint32_t jend = __shfl_down_sync(0xFFFFFFFFu, ja, 1);
  if (lane == 31) jend = nne;
  uint32_t idx = ja ? Q.ends[ja - 1] : 0u;
  const uint32_t stop = jend ? Q.ends[jend - 1] : 0u;
  uint32_t j = ja;
  uint32_t r = Q.ids[j], nxt = Q.ends[j];
  const uint16_t* tp = gt + idx;
  KS_CHECK(idx <= stop && stop <= T && ja <= jend && jend <= nne);
  uint32_t tk0 = tp[0], tk1 = tp[1];
  const uint32_t fa_s = (uint32_t)__cvta_generic_to_shared(S.fa);
  const uint32_t tO_s = (uint32_t)__cvta_generic_to_shared(S.tO), tP_s = (uint32_t)__cvta_generic_to_shared(S.tP);
  uint32_t c1 = 0, cq = 0, co = 0, cp = 0, M = 0;   // V | Y<<16, q | S<<16, O, P, M of request r
  uint32_t ro = 0, rp = 0;                          // O-part / P-part state (row byte offsets)
  uint32_t nf = 0xFFFFu, n2m = 1u;                 // first noun id of the sentence; 0x10001 once a second one is seen
  while (__any_sync(0xFFFFFFFFu, idx < stop)) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const bool act = idx < stop;
      const uint32_t t = tk0;
      tk0 = tk1;
      tk1 = tp[2];
      tp += act ? 1 : 0;
      const uint2 a = lds64(fa_s + t * 8u);
      c1 += a.y & 0x10001u;
      cq += (a.y >> 8) & n2m;  // '?', and PREP after a second distinct noun of the sentence (tested first)
      M += (a.x >> 8) & 0xFFu;
      const uint32_t vo = lds32(tO_s + ro + (a.x & 0xFFu));
      const uint32_t vp = lds32(tP_s + rp + (a.y & 0xCu));
      ro = vo & 0xFFFFu;
      rp = vp & 0xFFFFu;
      co += vo >> 16;
      cp += vp >> 16;
      const uint32_t nid = a.x >> 16;
      n2m = (nid != 0xFFFFu && nf != 0xFFFFu && nid != nf) ? 0x10001u : n2m;
      nf = nf == 0xFFFFu ? nid : nf;
      const bool end = (a.y & 0x1000u) != 0u;  // sentence end: fresh S-part
      nf = end ? 0xFFFFu : nf;
      n2m = end ? 1u : n2m;
      idx += act ? 1u : 0u;
      const bool fin = act && idx == nxt;  // last token of request r: store, fresh context
      if (fin) gcnt[r] = make_uint4(c1, cq, co | (cp << 16), M);
      const uint32_t keep = fin ? 0u : 1u;
      c1 *= keep; cq *= keep; co *= keep; cp *= keep; M *= keep;
      ro *= keep; rp *= keep;
      nf = fin ? 0xFFFFu : nf;
      n2m = fin ? 1u : n2m;
      j += fin ? 1u : 0u;
      KS_CHECK(j <= nne && idx <= T + 1u);
      if (fin) { r = Q.ids[j]; nxt = Q.ends[j]; }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kT4, 1) k_score6(ScoreLaunch a, uint32_t* work, uint16_t* tokbuf) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem6& S = *reinterpret_cast<Smem6*>(smem_raw);
  uint8_t* tail_mem = smem_raw + ((sizeof(Smem6) + 15) & ~size_t(15));
  uint4* s_keys = reinterpret_cast<uint4*>(tail_mem);
  const uint32_t key_bytes = (a.lex.n_entries + 1u) * 16u;
  uint32_t* s_slots = reinterpret_cast<uint32_t*>(tail_mem + key_bytes);
  const uint32_t nslots = 1u << a.lex.bits;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  {
    for (uint32_t i = tid; i <= a.lex.n_entries; i += kT4) s_keys[i] = a.lex.keys[i];
    for (uint32_t i = tid; i < nslots; i += kT4) s_slots[i] = a.lex.slots[i];
    for (uint32_t i = tid; i < 256; i += kT4) S.lut[i] = class_bits(i) | (punct_kind(i) << 24);
    for (uint32_t i = tid; i < kPunct + 8; i += kT4)
      S.fa[i] = fsm_attr6(i, (i >= 1u && i <= a.lex.n_entries) ? a.lex.entries[i - 1].attr : 0u);
    for (uint32_t i = tid; i < 16 * 32; i += kT4) {
      const uint32_t v = o_step(i >> 5, i & 31u);
      S.tO[i] = (v & 15u) * 128u | ((v >> 4) << 16);
    }
    for (uint32_t i = tid; i < 128 * 4; i += kT4) {
      const uint32_t v = p_step(i >> 2, i & 3u);
      S.tP[i] = (v & 127u) * 16u | ((v >> 7) << 16);
    }
    for (uint32_t i = tid; i < 18; i += kT4) {
      const uint32_t sh = i > 16u ? 0u : 8u * i;
      S.lmask[i] = make_uint4(__funnelshift_lc(0xFFFFFFFFu, 0u, sh), __funnelshift_lc(0xFFFFFFFFu, 0u, sh > 32u ? sh - 32u : 0u),
                              __funnelshift_lc(0xFFFFFFFFu, 0u, sh > 64u ? sh - 64u : 0u),
                              __funnelshift_lc(0xFFFFFFFFu, 0u, sh > 96u ? sh - 96u : 0u));
    }
    for (uint32_t i = tid; i < 8; i += kT4) {
      S.cl3[i] = make_uint2(0xFFFFFFFFu, 0u);
      S.cl2[i] = make_uint2(0xFFFFFFFFu, 0u);
    }
  }
  __syncthreads();
  const Lex L{s_keys, s_slots, a.lex.entries, a.lex.bits, a.lex.seed};
  if (tid < 7) {
    const uint32_t cb = clitic_bytes(tid), len = tid < 4 ? 3u : 2u;
    const uint32_t s3 = len == 3 ? (((cb & 0xFFu) << 16) | (cb & 0xFF00u) | ((cb >> 16) & 0xFFu))
                                 : (((cb & 0xFFu) << 8) | ((cb >> 8) & 0xFFu));
    const uint32_t code = word_code(L, len, cb, 0u, 0u, 0u, s3);
    S.clit[tid] = code;
    if (len == 3) S.cl3[clitic_hash3(cb)] = make_uint2(cb, code);
    else S.cl2[clitic_hash2(cb)] = make_uint2(cb, code);
  }
  __syncthreads();
  WarpBuf6& B = S.w[wid];
  uint8_t* wscr = reinterpret_cast<uint8_t*>(tokbuf) + (size_t)(blockIdx.x * kW4 + wid) * kWarpScratch;
  uint16_t* gt = reinterpret_cast<uint16_t*>(wscr);
  uint4* gcnt = reinterpret_cast<uint4*>(wscr + (kTokCap + kTokPad) * 2);
  const uint32_t total_bytes = a.n ? a.offsets[a.n] : 0u;
  const uint32_t ntasks = (a.n + 31) / 32;
  uint32_t pending = 0xFFFFFFFFu;
  bool done = false;
  while (!done) {
    // ---- (A) fill a pool
    uint32_t np = 0, tok = 0;
    for (;;) {
      uint32_t task;
      if (pending != 0xFFFFFFFFu) {
        task = pending;
        pending = 0xFFFFFFFFu;
      } else {
        task = 0;
        if (lane == 0) task = atomicAdd(work, 1u);
        task = __shfl_sync(0xFFFFFFFFu, task, 0);
        if (task >= ntasks) { done = true; break; }
      }
      const uint32_t r0 = task * 32, rcnt = min(32u, a.n - r0);
      const uint32_t r = r0 + lane;
      const bool rv = lane < rcnt;
      const uint32_t s_r = rv ? a.offsets[r] : 0u;
      const uint32_t e_r = rv ? a.offsets[r + 1] : 0u;
      const bool bad = rv && e_r < s_r;
      const uint32_t B0 = __shfl_sync(0xFFFFFFFFu, s_r, 0);
      const uint32_t B1 = __shfl_sync(0xFFFFFFFFu, e_r, rcnt - 1);
      if (__any_sync(0xFFFFFFFFu, bad) || B1 - B0 > kTokCap) {
        // decreasing offsets, or more bytes than a pool buffer holds: per-lane byte FSM
        if (bad) atomicOr(a.flags, RT_FLAG_BAD_OFFSETS);
        // (offsets that are not non-decreasing: reads stay inside [0, offsets[n]))
        if (rv) fsm_request(a, L, r, min(s_r, total_bytes), bad ? min(s_r, total_bytes) : min(e_r, total_bytes));
        continue;
      }
      if (tok + (B1 - B0) > kTokCap) { pending = task; break; }  // tokens <= bytes
      if (lane == 0) B.task[np] = task;
      tokenize_task(a, S, B, L, gt, tok, np * 32, rcnt, s_r, e_r, rv, lane, total_bytes);
      if (++np == kPoolTasks) break;
    }
    if (np == 0) continue;
    // ---- (B) rules, (C) epilogue
    const uint32_t R = np * 32;
    rules_pool(S, B, gt, gcnt, R, tok, lane);
    for (uint32_t lr = lane; lr < R; lr += 32) {
      const uint32_t gr = B.task[lr >> 5] * 32 + (lr & 31u);
      if (gr >= a.n) continue;
      const uint32_t ntk = (uint32_t)B.tbeg[lr + 1] - (uint32_t)B.tbeg[lr];
      const uint4 c = ntk ? gcnt[lr] : make_uint4(0, 0, 0, 0);
      const uint32_t q = c.y & 0xFFFFu;
      const uint32_t Pt = (c.z >> 16) + (q > 1u ? q - 1u : 0u);
      const uint32_t raw[8] = {c.y >> 16, c.x >> 16, c.w, c.x & 0xFFFFu, c.z & 0xFFFFu, Pt,
                               ntk, B.nd[lr]};
      uint32_t f[8];
      bool sat = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        sat |= raw[k] > 65535u;
        f[k] = min(raw[k], 65535u);
      }
      if (sat) atomicOr(a.flags, RT_FLAG_SATURATED);
      epilogue(a, gr, f);
    }
    __syncwarp();
  }
  // the last CTA to finish resets the work counter (work[0]) and the CTA
  // counter (work[1]) for the next launch, which stream order starts after this
  // one has completed; a faulting launch leaves the context unusable anyway
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(work + 1, 1u) == gridDim.x - 1u) {
      work[0] = 0u;
      work[1] = 0u;
      __threadfence();
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


size_t score_scratch_bytes(int ctas) { return (size_t)ctas * kW4 * kWarpScratch; }

cudaError_t launch_score(const ScoreLaunch& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;  // a.work[0..1] are zero here: reset by the previous launch's last CTA
  const uint32_t ntasks = (a.n + 31) / 32;
  uint32_t grid = (uint32_t)a.num_sms;
  if (grid * kW4 > ntasks) grid = (ntasks + kW4 - 1) / kW4;
  const size_t lex_bytes = (size_t(a.lex.n_entries) + 1) * 16 + (size_t(1) << a.lex.bits) * 4;
  if (!a.tokbuf) return cudaErrorInvalidValue;
  const size_t smem = ((sizeof(Smem6) + 15) & ~size_t(15)) + lex_bytes;
  e = cudaFuncSetAttribute(k_score6, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_score6<<<grid, kT4, smem, s>>>(a, a.work, a.tokbuf);
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
