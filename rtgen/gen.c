/*
 * rtgen — seeded synthetic workload generator (TEST/BENCH INPUT ONLY).
 *
 * This module is shared by the oracle side and the CUDA side as their common
 * INPUT source, so it deliberately holds none of the method's arithmetic: no
 * tokenizer, no lemmatizer, no rule scorer, no regression, no priority key.
 * It only draws random words from fixed word lists and records what it
 * planted ("latent counts"), draws ground-truth output lengths from those
 * latent counts, and draws Poisson arrival times.
 *
 * Every request is generated from a counter-based SplitMix64 stream keyed by
 * (seed, stream id, global request id), so any shard [gid0, gid0+n) is
 * byte-identical to the same range of a larger run (SURVEY.md §8(d) "Seeds").
 *
 * Recipe:
 *  - words per request ~ round(lognormal(mu=2.385, sigma=0.6)) clipped to
 *    [1, 200]  (mean ~13 words, the paper's sample query is 15 words / 73
 *    chars);
 *  - 1..3 sentences, ~50% ending in '?' (S:500 templated sentences per
 *    Table 1 type, plus neutral ones);
 *  - per sentence a Table-1 "type" boosts one word category;
 *  - rare clitics ("don't", "it's"), digits and non-ASCII UTF-8 words.
 * True output length for LM f:
 *    max(1, round(s_f * (c + sum_k w_k * latent_k) + N(0, 0.25 * s_f * c)))
 * Arrivals: per minute j rate beta_j = min(b0 + step*j, bmax)
 * per minute, exponential gaps, quantised to microseconds.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>

#define ST_TEXT    0x74657874ULL  /* "text" */
#define ST_LEN     0x6c656e00ULL  /* "len"  */
#define ST_ARRIVAL 0x61727276ULL  /* "arrv" */
#define ST_SHUFFLE 0x73687566ULL  /* "shuf" */

typedef struct { uint64_t s; } rng_t;

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t next64(rng_t* r) {
  r->s += 0x9E3779B97F4A7C15ULL;
  return mix64(r->s);
}
static inline rng_t rng_for(uint64_t seed, uint64_t stream, uint64_t id) {
  rng_t r;
  r.s = mix64(seed ^ mix64(stream * 0xD1B54A32D192ED03ULL) ^ mix64(id + 0x632BE59BD9B4E019ULL));
  return r;
}
/* uniform in [0,1) with 53 bits */
static inline double unif(rng_t* r) { return (double)(next64(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint32_t below(rng_t* r, uint32_t n) { return (uint32_t)(((next64(r) >> 32) * (uint64_t)n) >> 32); }
static inline double gauss(rng_t* r) {
  double u1 = unif(r), u2 = unif(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* ---- word lists (generator data; categories mirror data/lexicon_v1.txt) ---- */
static const char* NOUNS[] = {"boy","girl","man","woman","park","telescope","rice","sand","cat","dog","poverty",
  "city","house","car","movie","garden","river","school","teacher","doctor","student","table","window","phone",
  "computer","road","bridge","forest","mountain","village","market","kitchen","bottle","letter","picture","friend",
  "family","child","ocean","island","airport","museum","library","hospital","office","store","restaurant","camera",
  "shirt","chair","door","bird","horse","tree","flower","apple","bread","coffee","lake","beach","castle","farmer",
  "pilot","engine","wall","floor","street","cats","dogs","books"};
static const char* PROPN[] = {"John","Mary","Paris","London","Peter","Anna","Tokyo","Berlin"};
static const char* PREPS[] = {"in","with","of","about","to","on","at","for","from","by","into","near","under","over",
  "through","between","without","across","behind","during"};
static const char* VAGUE[] = {"history","stuff","things","thing","something","anything","everything","topic","topics",
  "aspects","matters","issues","general","overall","various","kind","sort","basically","somewhat","whatever","lots",
  "bunch","generally","broadly","concepts","ideas","details","info"};
static const char* POLY[] = {"bat","bats","bank","trunk","monitor","spring","bark","crane","bass","seal","match","light",
  "pitch","date","bow","fan","jam","mole","nail","palm","ring","rose","scale","star","tie","wave","bolt","club","cell",
  "current","degree","key","mouse","net","plant","port","present","row","sink","spirit","strike","suit","tank","tip","yard"};
static const unsigned char POLY_EXTRA[] = {1,1,2,2,1,2,1,1,1,1,2,2, 2,1,1,1,1,2,1,1,1,1,2,1,1,1,1,1,2, 1,1,2,1,1,1,1,1,1,1,1,2,1,1,2,1};
static const char* MULTI[] = {"saw","flies","like","watch","run","play","fly","duck","check","cook","dance","dream","drink",
  "drive","jump","kiss","laugh","mark","move","paint","plan","rain","ride","sail","show","smile","swim","train","trust",
  "turn","visit","vote","walk","wish","answer","guide","judge","shop","fast","back","down","round"};
static const char* OPENERS[] = {"Why","How","Tell","Explain","Describe","Discuss","Compare","Analyze","Elaborate","Summarize"};
static const char* CAUSES[] = {"causes","consequences","effects","reasons","impacts","implications","benefits","risks","factors","origins"};
static const char* BROAD[] = {"art","countries","world","society","life","culture","science","economy","politics","humanity",
  "nature","technology","religion","philosophy","education"};
static const char* COORDS[] = {"and","or"};
static const char* FILLERS[] = {"the","a","an","is","was","it","this","that","we","they","he","she","very","quite","some",
  "new","old","good","great","small","big","red","blue","green","happy","quickly","often","always","never","today",
  "yesterday","just","also","then","there","here","my","your","our","their","his","her","every","each","many","few",
  "more","most","other","same","different","important","possible","simple","strong","young","long","short","high",
  "low","early","late","first","last","next","want","need","know","think","see","get","make","go","come","take","give",
  "find","say","feel","try","ask","seem","keep","begin","write","read","hear","bring","hold","meet","sit","stand",
  "lose","pay","learn","grow","build","buy","send","spend","fall","cut","reach","raise","pass","sell","decide","pull",
  "carry","break","hang","wear","seek","would","could","should","will","might","must","been","being","am","were","has",
  "had","does","did","who","when","where","which","if","because","while","so","too","not","no","yes","maybe","please",
  "thanks","sorry","okay","well","very","really","actually","probably","usually","sometimes","again","still","already"};
static const char* CLITICS[] = {"don't","it's","I'm","they're","we'll","can't","isn't","what's","you've","she'd","won't","that's"};
static const char* NONASCII[] = {"caf\xc3\xa9","na\xc3\xafve","r\xc3\xa9sum\xc3\xa9","\xe2\x80\x9cquote\xe2\x80\x9d","stra\xc3\x9f" "e"};
static const char* DIGITS[] = {"2023","42","7","100","3","1999","12"};

#define NELEM(a) (sizeof(a) / sizeof((a)[0]))
_Static_assert(NELEM(POLY) == NELEM(POLY_EXTRA), "POLY_EXTRA must parallel POLY");

/* latent slots: 0 S(structural) 1 Y(syntactic) 2 M(semantic) 3 V(vague) 4 O(open) 5 P(multi-part) 6 ntok */
enum { CAT_FILLER, CAT_NOUN, CAT_PREP, CAT_MULTI, CAT_POLY, CAT_VAGUE, CAT_COORD, CAT_CAUSE, CAT_BROAD, NCAT };
/* base per-slot probabilities (x1000), boosted per sentence type */
static const int BASE_P[NCAT] = {600, 150, 70, 45, 35, 30, 40, 10, 20};

typedef struct {
  uint8_t* out; uint64_t cap; uint64_t len;  /* out may be NULL (length pass) */
} sink_t;

static inline void put(sink_t* s, const char* w) {
  size_t n = strlen(w);
  if (s->out && s->len + n <= s->cap) memcpy(s->out + s->len, w, n);
  s->len += n;
}
static inline void putc_(sink_t* s, char c) {
  if (s->out && s->len + 1 <= s->cap) s->out[s->len] = (uint8_t)c;
  s->len += 1;
}
static void put_cap(sink_t* s, const char* w, int capitalize) {
  if (!capitalize || w[0] < 'a' || w[0] > 'z') { put(s, w); return; }
  putc_(s, (char)(w[0] - 32));
  put(s, w + 1);
}

/* one request; returns bytes written; latent[7] accumulates */
static uint64_t gen_request(uint64_t seed, uint64_t gid, sink_t* s, int32_t* lat) {
  rng_t r = rng_for(seed, ST_TEXT, gid);
  uint64_t start = s->len;
  double ln = 2.385 + 0.6 * gauss(&r);
  int nwords = (int)lround(exp(ln));
  if (nwords < 1) nwords = 1;
  if (nwords > 200) nwords = 200;
  int nsent = 1 + (int)below(&r, 3);
  if (nsent > nwords) nsent = nwords;
  int remaining = nwords;
  int nq = 0;
  for (int k = 0; k < 7; ++k) lat[k] = 0;
  int nonascii = (below(&r, 100) == 0);
  for (int si = 0; si < nsent; ++si) {
    int w_s = (si == nsent - 1) ? remaining : 1 + (int)below(&r, (uint32_t)(remaining - (nsent - 1 - si)));
    if (w_s < 1) w_s = 1;
    remaining -= w_s;
    if (si > 0) putc_(s, ' ');
    /* sentence type (Table 1 rows + neutral) */
    uint32_t tp = below(&r, 1000);
    int type = tp < 300 ? 0 : tp < 420 ? 1 : tp < 520 ? 2 : tp < 620 ? 3 : tp < 740 ? 4 : tp < 870 ? 5 : 6;
    int p[NCAT];
    for (int c = 0; c < NCAT; ++c) p[c] = BASE_P[c];
    switch (type) {
      case 1: p[CAT_NOUN] *= 2; p[CAT_PREP] *= 2; break;   /* structural */
      case 2: p[CAT_MULTI] *= 4; break;                     /* syntactic */
      case 3: p[CAT_POLY] *= 4; break;                      /* semantic */
      case 4: p[CAT_VAGUE] *= 5; break;                     /* vague */
      case 5: p[CAT_CAUSE] *= 3; p[CAT_BROAD] *= 3; break;  /* open-ended */
      case 6: p[CAT_COORD] *= 3; p[CAT_NOUN] *= 2; break;   /* multi-part */
      default: break;
    }
    int ptot = 0;
    for (int c = 0; c < NCAT; ++c) ptot += p[c];
    /* terminator */
    uint32_t tr = below(&r, 100);
    char term = tr < 50 ? '?' : tr < 95 ? '.' : '!';
    int nouns_in_sent = 0, commas_run = 0, lists = 0, wi = 0, force_broad = 0;
    /* sentence-initial opener / what-question */
    if (type == 5 || below(&r, 10) == 0) {
      uint32_t o = below(&r, 100);
      if (o < 45) {
        put(s, OPENERS[below(&r, NELEM(OPENERS))]); lat[4]++; lat[6]++; wi++;
      } else if (o < 80 && w_s >= 4) {
        put(s, "What are the "); put(s, CAUSES[below(&r, NELEM(CAUSES))]); lat[4]++; lat[6] += 4; wi += 4;
      } else if (term == '?' && w_s >= 2) {
        force_broad = 1;  /* broad-scope interrogative: planted at the end */
      }
    }
    int broad_end = (term == '?' && (force_broad || below(&r, 4) == 0));
    while (wi < w_s) {
      int last = (wi == w_s - 1);
      if (wi > 0) putc_(s, ' ');
      int cap = (wi == 0);
      if (last && broad_end) {
        put_cap(s, BROAD[below(&r, NELEM(BROAD))], cap); lat[4]++; lat[6]++; wi++; break;
      }
      if (nonascii && below(&r, 8) == 0) { put(s, NONASCII[below(&r, NELEM(NONASCII))]); nonascii = 0; lat[6]++; wi++; continue; }
      if (below(&r, 40) == 0) { put_cap(s, CLITICS[below(&r, NELEM(CLITICS))], cap); lat[6] += 2; wi++; continue; }
      if (below(&r, 60) == 0) { put(s, DIGITS[below(&r, NELEM(DIGITS))]); lat[6]++; wi++; continue; }
      int x = (int)below(&r, (uint32_t)ptot), c = 0;
      while (x >= p[c]) { x -= p[c]; ++c; }
      if (cap && (c == CAT_COORD || c == CAT_PREP)) c = CAT_FILLER;
      switch (c) {
        case CAT_NOUN:
          if (below(&r, 8) == 0) put(s, PROPN[below(&r, NELEM(PROPN))]);
          else put_cap(s, NOUNS[below(&r, NELEM(NOUNS))], cap);
          nouns_in_sent++;
          break;
        case CAT_PREP: put(s, PREPS[below(&r, NELEM(PREPS))]); if (nouns_in_sent >= 1) lat[0]++; break;
        case CAT_MULTI: put_cap(s, MULTI[below(&r, NELEM(MULTI))], cap); lat[1]++; break;
        case CAT_POLY: { uint32_t k = below(&r, NELEM(POLY)); put_cap(s, POLY[k], cap); lat[2] += POLY_EXTRA[k]; break; }
        case CAT_VAGUE: put_cap(s, VAGUE[below(&r, NELEM(VAGUE))], cap); lat[3]++; break;
        case CAT_COORD: put(s, COORDS[below(&r, NELEM(COORDS))]); lat[5]++; break;
        case CAT_CAUSE: put_cap(s, CAUSES[below(&r, NELEM(CAUSES))], cap); break;
        case CAT_BROAD: put_cap(s, BROAD[below(&r, NELEM(BROAD))], cap); break;
        default: put_cap(s, FILLERS[below(&r, NELEM(FILLERS))], cap); break;
      }
      lat[6]++;
      wi++;
      /* list commas after nouns (multi-part lists) */
      if (!last && c == CAT_NOUN && below(&r, (type == 6) ? 3 : 8) == 0) {
        putc_(s, ','); lat[6]++;
        if (++commas_run == 2) lists++;
      } else if (c != CAT_NOUN && c != CAT_FILLER) {
        commas_run = 0;
      }
    }
    putc_(s, term); lat[6]++;
    if (term == '?') nq++;
    lat[5] += lists;
    /* occasional double space / tab between sentences */
    if (si + 1 < nsent && below(&r, 20) == 0) putc_(s, below(&r, 2) ? '\t' : ' ');
  }
  if (nq > 1) lat[5] += nq - 1;
  return s->len - start;
}

/* Generates n requests with global ids gid0..gid0+n-1.
 * offsets: n+1 entries (byte offsets, offsets[0] = 0).  out may be NULL to
 * only compute offsets; otherwise cap must be >= offsets[n].  latent (n*7
 * int32) may be NULL.  Returns total bytes. */
uint64_t rtgen_text(uint64_t seed, uint64_t gid0, uint32_t n, uint8_t* out, uint64_t cap,
                    uint64_t* offsets, int32_t* latent) {
  sink_t s = {out, cap, 0};
  int32_t lat[7];
  offsets[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    gen_request(seed, gid0 + i, &s, lat);
    offsets[i + 1] = s.len;
    if (latent) memcpy(latent + (size_t)i * 7, lat, sizeof(lat));
  }
  return s.len;
}

/* Ground-truth output lengths from latent counts (generator model, not the
 * method): len = max(1, round(scale*(c + sum w_k lat_k) + N(0, sigma))).
 * w has 7 entries (6 categories + ntok).  'lm' selects an independent noise
 * stream per LM.  Results clipped to 65535. */
void rtgen_true_len(uint64_t seed, uint64_t gid0, uint32_t n, const int32_t* latent, double scale, double c,
                    const double* w, double sigma, uint32_t lm, uint16_t* out) {
  for (uint32_t i = 0; i < n; ++i) {
    rng_t r = rng_for(seed ^ ((uint64_t)lm << 56), ST_LEN, gid0 + i);
    double m = c;
    for (int k = 0; k < 7; ++k) m += w[k] * (double)latent[(size_t)i * 7 + k];
    double v = scale * m + sigma * gauss(&r);
    long q = lround(v);
    if (q < 1) q = 1;
    if (q > 65535) q = 65535;
    out[i] = (uint16_t)q;
  }
}

/* Poisson arrivals for one trace: minute j has rate
 * min(beta0 + step*j, beta_max) arrivals per minute; exponential gaps drawn at
 * the rate of the minute the previous arrival fell in; microsecond quantised. */
void rtgen_arrivals(uint64_t seed, uint64_t trace_id, uint32_t n, double beta0, double step, double beta_max,
                    int64_t* out_us) {
  rng_t r = rng_for(seed, ST_ARRIVAL, trace_id);
  double t = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    double minute = floor(t / 60.0);
    double beta = beta0 + step * minute;
    if (beta > beta_max) beta = beta_max;
    double u = unif(&r);
    t += -log1p(-u) * 60.0 / beta;
    out_us[i] = (int64_t)llround(t * 1e6);
  }
}

/* Seeded Fisher-Yates permutation of 0..n-1 ("we shuffle the test dataset and
 * map them to the created arrival patterns"). */
void rtgen_shuffle(uint64_t seed, uint64_t id, uint32_t n, uint32_t* perm) {
  rng_t r = rng_for(seed, ST_SHUFFLE, id);
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) {
    uint32_t j = below(&r, i);
    uint32_t t = perm[i - 1]; perm[i - 1] = perm[j]; perm[j] = t;
  }
}
