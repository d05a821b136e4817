// rtlm_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU implementation of the RT-LM hot path
// (arXiv 2309.06619) written from the paper and DESIGN.md's readings, used
// ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` leg.  The product path (paper_2309_06619_b200/) never
// links, imports or calls it, and this file shares no source, header, table
// or constant generator with csrc/.
//
// Citations: P:a-b = /root/reference/PAPER.md lines, S:a-b = SPEC.md lines.
// Step names O1..O8 follow DESIGN.md §3 (= SURVEY.md §8(c)).
//
// Precision: the method's decisions (priority key, offload, λ-cut) are taken in
// IEEE binary32 with every operation written out separately (DESIGN.md R-FP):
// this file is compiled with -ffp-contract=off and uses std::fmaf only where
// the definition says fma.  Times are int64 microseconds.
//
// Parity status: every function below is pinned by tests/test_oracle_*.py
// (see DESIGN.md §4 "Pins"); none is "parity unpinned".

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace {

// ---------------------------------------------------------------- O1 tokens
// Byte classes (DESIGN R-TOK): W = [A-Za-z0-9'], S = space and
// 0x09-0x0D, P = other printable ASCII 0x21-0x7E, X = everything else
// (dropped, counted, acts as a separator).
enum ByteClass { BC_W, BC_S, BC_P, BC_X };

ByteClass byte_class(uint8_t b) {
  if ((b >= 'A' && b <= 'Z') || (b >= 'a' && b <= 'z') || (b >= '0' && b <= '9') || b == '\'') return BC_W;
  if (b == 0x20 || (b >= 0x09 && b <= 0x0D)) return BC_S;
  if (b >= 0x21 && b <= 0x7E) return BC_P;
  return BC_X;
}

struct Token {
  bool word;            // word token (from a W run) vs punctuation token
  std::string surface;  // original bytes
};

std::string lower(const std::string& s) {
  std::string r = s;
  for (auto& c : r)
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
  return r;
}

bool ends_with(const std::string& s, const char* suf) {
  size_t k = std::strlen(suf);
  return s.size() >= k && s.compare(s.size() - k, k, suf) == 0;
}

// One clitic split of a W run, case-insensitive (DESIGN R-CLITIC; S:63
// "don't stop" -> ["do","n't","stop"]):  n't (run length > 3) splits 3;
// else 's 'm 'd (length > 2) split 2; else 're 've 'll (length > 3) split 3.
void push_run(const std::string& run, std::vector<Token>& out) {
  const std::string lo = lower(run);
  const size_t n = run.size();
  size_t cut = 0;
  if (n > 3 && ends_with(lo, "n't")) cut = 3;
  else if (n > 2 && (ends_with(lo, "'s") || ends_with(lo, "'m") || ends_with(lo, "'d"))) cut = 2;
  else if (n > 3 && (ends_with(lo, "'re") || ends_with(lo, "'ve") || ends_with(lo, "'ll"))) cut = 3;
  if (cut) {
    out.push_back({true, run.substr(0, n - cut)});
    out.push_back({true, run.substr(n - cut)});
  } else {
    out.push_back({true, run});
  }
}

// Tokenize one request: maximal W runs are word tokens (after the clitic
// split); every P byte is its own token; S and X bytes separate; X counted.
std::vector<Token> tokenize(const uint8_t* p, size_t n, uint32_t* ndropped) {
  std::vector<Token> toks;
  std::string run;
  uint32_t dropped = 0;
  for (size_t i = 0; i < n; ++i) {
    ByteClass c = byte_class(p[i]);
    if (c == BC_W) {
      run.push_back(char(p[i]));
      continue;
    }
    if (!run.empty()) {
      push_run(run, toks);
      run.clear();
    }
    if (c == BC_P) toks.push_back({false, std::string(1, char(p[i]))});
    if (c == BC_X) ++dropped;
  }
  if (!run.empty()) push_run(run, toks);
  if (ndropped) *ndropped = dropped;
  return toks;
}

// Lemma (DESIGN R-LEMMA; "lowercase + fixed suffix-strip table (s/es/
// ed/ing with minimal-stem guard)"; Listing 1 P:190 lemmatizes each token):
// lowercase; "n't" -> "not"; first matching rule wins:
//   len>=5 & "ing" -> strip 3;  len>=4 & "ed" -> strip 2;
//   len>=4 & "es"  -> strip 2;  len>=3 & "s" & not "ss" -> strip 1.
std::string lemma_of(const std::string& surface) {
  std::string s = lower(surface);
  if (s == "n't") return "not";
  const size_t L = s.size();
  if (L >= 5 && ends_with(s, "ing")) return s.substr(0, L - 3);
  if (L >= 4 && ends_with(s, "ed")) return s.substr(0, L - 2);
  if (L >= 4 && ends_with(s, "es")) return s.substr(0, L - 2);
  if (L >= 3 && ends_with(s, "s") && !ends_with(s, "ss")) return s.substr(0, L - 1);
  return s;
}

// ---------------------------------------------------------------- lexicon
// SPEC S:147 format + the `wh` flag extension (DESIGN R-LEX).  Entries are
// surface forms, lemmatized on load like Listing 1's lemmatize(phrase)
// (P:193); duplicates merge (union of flags/tags, max of sense counts).
const char* kPosTags[] = {"NOUN", "PROPN", "VERB", "ADJ", "ADV", "ADP", "PRON", "DET",
                          "CCONJ", "SCONJ", "NUM", "PART", "INTJ", "AUX", "X", "SYM", "PUNCT"};

struct Entry {
  uint32_t id = 0;       // order of first appearance; doubles as the noun id
  bool vague = false, prep = false, coord = false;
  bool opener = false, what = false, cause = false, broad = false;
  uint32_t tags = 0;     // PoS tag bitmask
  uint32_t senses = 0;   // 0 = not listed as polysemous
  bool noun() const { return (tags & 3u) != 0; }  // NOUN or PROPN
  int npos() const { return __builtin_popcount(tags); }
};

struct Lexicon {
  std::map<std::string, Entry> map;
  const Entry* find(const std::string& lemma) const {
    auto it = map.find(lemma);
    return it == map.end() ? nullptr : &it->second;
  }
};

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
  return s.substr(a, b - a);
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> r;
  size_t a = 0;
  for (;;) {
    size_t b = s.find(sep, a);
    r.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  return r;
}

bool parse_lexicon(const std::string& text, Lexicon& lex, std::string& err) {
  std::string section;
  uint32_t next_id = 0;
  int lineno = 0;
  for (const std::string& raw : split(text, '\n')) {
    ++lineno;
    std::string line = raw;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::string t = trim(line);
    if (t.empty() || t[0] == '#') continue;
    if (t.back() == ':' && t.find('\t') == std::string::npos) {
      section = t.substr(0, t.size() - 1);
      if (section != "vague" && section != "polysemy" && section != "pos" && section != "wh" &&
          section != "coord" && section != "prep") {
        err = "line " + std::to_string(lineno) + ": unknown section '" + section + "'";
        return false;
      }
      continue;
    }
    if (section.empty()) {
      err = "line " + std::to_string(lineno) + ": entry before any section header";
      return false;
    }
    size_t tab = line.find('\t');
    std::string word = trim(tab == std::string::npos ? line : line.substr(0, tab));
    std::string value = tab == std::string::npos ? "" : trim(line.substr(tab + 1));
    // the entry must be exactly one word token
    std::vector<Token> tk = tokenize(reinterpret_cast<const uint8_t*>(word.data()), word.size(), nullptr);
    if (tk.size() != 1 || !tk[0].word || tk[0].surface != word) {
      err = "line " + std::to_string(lineno) + ": entry '" + word + "' is not a single word token";
      return false;
    }
    std::string lem = lemma_of(word);
    if (lem.empty() || lem.size() > 16) {
      err = "line " + std::to_string(lineno) + ": lemma of '" + word + "' longer than 16 bytes";
      return false;
    }
    auto it = lex.map.find(lem);
    if (it == lex.map.end()) {
      it = lex.map.emplace(lem, Entry{}).first;
      it->second.id = next_id++;
    }
    Entry& e = it->second;
    if (section == "vague" || section == "coord" || section == "prep") {
      if (!value.empty()) {
        err = "line " + std::to_string(lineno) + ": unexpected value in section " + section;
        return false;
      }
      if (section == "vague") e.vague = true;
      if (section == "coord") e.coord = true;
      if (section == "prep") e.prep = true;
    } else if (section == "polysemy") {
      char* end = nullptr;
      long v = std::strtol(value.c_str(), &end, 10);
      if (value.empty() || *end != '\0' || v < 2 || v > 255) {
        err = "line " + std::to_string(lineno) + ": polysemy count must be an integer in [2,255]";
        return false;
      }
      e.senses = std::max<uint32_t>(e.senses, uint32_t(v));
    } else if (section == "pos") {
      if (value.empty()) {
        err = "line " + std::to_string(lineno) + ": pos entry without tags";
        return false;
      }
      for (const std::string& tag0 : split(value, ',')) {
        std::string tag = trim(tag0);
        int k = -1;
        for (int j = 0; j < int(sizeof(kPosTags) / sizeof(kPosTags[0])); ++j)
          if (tag == kPosTags[j]) k = j;
        if (k < 0) {
          err = "line " + std::to_string(lineno) + ": unknown PoS tag '" + tag + "'";
          return false;
        }
        e.tags |= 1u << k;
      }
    } else {  // wh
      if (value.empty()) {
        err = "line " + std::to_string(lineno) + ": wh entry without flags";
        return false;
      }
      for (const std::string& f0 : split(value, '|')) {
        std::string f = trim(f0);
        if (f == "OPENER") e.opener = true;
        else if (f == "WHAT") e.what = true;
        else if (f == "CAUSE") e.cause = true;
        else if (f == "BROAD") e.broad = true;
        else {
          err = "line " + std::to_string(lineno) + ": unknown wh flag '" + f + "'";
          return false;
        }
      }
    }
  }
  return true;
}

// ---------------------------------------------------------------- O2 scorers
// Six rule scores of Table 1 as realized by SPEC S:64-113 and
// made exact in DESIGN R-RULES, plus ntok and ndropped.  Weight 1.
struct Feat {
  uint64_t S = 0, Y = 0, M = 0, V = 0, O = 0, P = 0, ntok = 0, ndropped = 0;
};

bool is_punct(const Token& t, char c) { return !t.word && t.surface[0] == c; }
bool is_terminator(const Token& t) { return is_punct(t, '.') || is_punct(t, '?') || is_punct(t, '!'); }

Feat rule_gen(const Lexicon& lex, const uint8_t* p, size_t n) {
  Feat f;
  uint32_t dropped = 0;
  std::vector<Token> toks = tokenize(p, n, &dropped);
  f.ntok = toks.size();
  f.ndropped = dropped;
  std::vector<const Entry*> ent(toks.size(), nullptr);
  for (size_t i = 0; i < toks.size(); ++i)
    if (toks[i].word) ent[i] = lex.find(lemma_of(toks[i].surface));

  // sentences: a sentence ends after a '.', '?' or '!' token
  size_t a = 0;
  while (a < toks.size()) {
    size_t b = a;
    while (b < toks.size() && !is_terminator(toks[b])) ++b;
    size_t end = (b < toks.size()) ? b + 1 : b;  // [a, end) is the sentence

    std::set<uint32_t> nouns;
    long first_word = -1, last_word = -1;
    for (size_t i = a; i < end; ++i) {
      if (!toks[i].word) continue;
      if (first_word < 0) first_word = long(i);
      last_word = long(i);
      const Entry* e = ent[i];
      if (!e) continue;
      if (e->vague) ++f.V;                                  // vague (Listing 1)
      if (e->npos() >= 2) ++f.Y;                            // syntactic
      if (e->senses >= 2) f.M += e->senses - 1;             // semantic
      if (e->prep && nouns.size() >= 2) ++f.S;              // structural, PREP tested first
      if (e->noun()) nouns.insert(e->id);
    }
    // open-endedness, per sentence
    if (first_word >= 0 && ent[first_word]) {
      const Entry* e0 = ent[first_word];
      if (e0->opener) ++f.O;
      if (e0->what) {
        for (size_t j = size_t(first_word) + 1; j < end && j <= size_t(first_word) + 3; ++j)
          if (toks[j].word && ent[j] && ent[j]->cause) {
            ++f.O;
            break;
          }
      }
    }
    if (end > a && is_punct(toks[end - 1], '?') && last_word >= 0 && ent[last_word] && ent[last_word]->broad) ++f.O;
    // comma chains: consecutive commas linked when >= 1 token lies between
    // them and every such token is a word; count chains of >= 2 commas
    long prev_comma = -1;
    int chain = 0;
    for (size_t i = a; i < end; ++i) {
      if (!is_punct(toks[i], ',')) continue;
      bool linked = false;
      if (prev_comma >= 0 && long(i) - prev_comma >= 2) {
        linked = true;
        for (size_t j = size_t(prev_comma) + 1; j < i; ++j)
          if (!toks[j].word) linked = false;
      }
      chain = linked ? chain + 1 : 1;
      if (chain == 2) ++f.P;
      prev_comma = long(i);
    }
    a = end;
  }
  // coordinators joining content spans: next token a word; previous
  // token a word, or ',' preceded by a word
  for (size_t i = 0; i < toks.size(); ++i) {
    if (!toks[i].word || !ent[i] || !ent[i]->coord) continue;
    bool next_ok = i + 1 < toks.size() && toks[i + 1].word;
    bool prev_ok = i >= 1 && (toks[i - 1].word || (is_punct(toks[i - 1], ',') && i >= 2 && toks[i - 2].word));
    if (next_ok && prev_ok) ++f.P;
  }
  uint64_t nq = 0;
  for (const Token& t : toks)
    if (is_punct(t, '?')) ++nq;
  if (nq > 1) f.P += nq - 1;
  return f;
}

uint16_t sat16(uint64_t v) { return v > 65535 ? uint16_t(65535) : uint16_t(v); }

// ---------------------------------------------------------------- O4 key
uint32_t ord32(float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  if (b == 0x80000000u) b = 0;  // -0 -> +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

}  // namespace

// ============================================================== C interface
extern "C" {

// The oracle's own profile record (NOT shared with include/rtlm.h).
struct orc_profile {
  int64_t eta_us, mu_us, base_us, setup_us, xi_us;
  float lambda, alpha, tau, u_max;
  int32_t C, b10, tightness, gamma, cores, policy, consolidate, offload, raw_numerator, pad;
};
struct orc_stats {
  int64_t sum_resp_us;
  uint32_t n, misses;
};

void* orc_lex_load(const char* text, uint64_t len, char* err, uint64_t errcap) {
  Lexicon* lex = new Lexicon();
  std::string e;
  if (!parse_lexicon(std::string(text, len), *lex, e)) {
    if (err && errcap) {
      std::strncpy(err, e.c_str(), errcap - 1);
      err[errcap - 1] = 0;
    }
    delete lex;
    return nullptr;
  }
  return lex;
}

void orc_lex_free(void* h) { delete static_cast<Lexicon*>(h); }

uint32_t orc_lex_size(void* h) { return uint32_t(static_cast<Lexicon*>(h)->map.size()); }

// Looks a SURFACE word up (lemmatized first).  flags bit0 vague, 1 prep,
// 2 coord, 3 noun, 4 opener, 5 what, 6 cause, 7 broad.  Returns 1 if found.
int orc_lex_lookup(void* h, const char* word, uint32_t* flags, uint32_t* id, uint32_t* senses, uint32_t* npos) {
  const Entry* e = static_cast<Lexicon*>(h)->find(lemma_of(word));
  if (!e) return 0;
  *flags = (e->vague ? 1u : 0u) | (e->prep ? 2u : 0u) | (e->coord ? 4u : 0u) | (e->noun() ? 8u : 0u) |
           (e->opener ? 16u : 0u) | (e->what ? 32u : 0u) | (e->cause ? 64u : 0u) | (e->broad ? 128u : 0u);
  *id = e->id;
  *senses = e->senses;
  *npos = uint32_t(e->npos());
  return 1;
}

int orc_lemma(const char* surface, char* out, uint64_t cap) {
  std::string l = lemma_of(surface);
  if (l.size() + 1 > cap) return -1;
  std::memcpy(out, l.c_str(), l.size() + 1);
  return int(l.size());
}

// Tokens joined by '\n' (word tokens prefixed 'W', punctuation 'P').
int orc_tokenize(const uint8_t* bytes, uint64_t len, char* out, uint64_t cap, uint32_t* ndropped) {
  std::vector<Token> toks = tokenize(bytes, len, ndropped);
  std::string s;
  for (size_t i = 0; i < toks.size(); ++i) {
    if (i) s.push_back('\n');
    s.push_back(toks[i].word ? 'W' : 'P');
    s += toks[i].surface;
  }
  if (s.size() + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return int(toks.size());
}

// O1+O2: feat[i*8 + k] = {S, Y, M, V, O, P, ntok, ndropped}, saturating u16.
void orc_rule_gen(void* h, const uint8_t* bytes, const uint32_t* offsets, uint32_t n, uint16_t* feat) {
  const Lexicon& lex = *static_cast<Lexicon*>(h);
  for (uint32_t i = 0; i < n; ++i) {
    Feat f = rule_gen(lex, bytes + offsets[i], offsets[i + 1] - offsets[i]);
    uint16_t* o = feat + size_t(i) * 8;
    o[0] = sat16(f.S); o[1] = sat16(f.Y); o[2] = sat16(f.M); o[3] = sat16(f.V);
    o[4] = sat16(f.O); o[5] = sat16(f.P); o[6] = sat16(f.ntok); o[7] = sat16(f.ndropped);
  }
}

// O3 (weighted rule; Eq. 1): u = max(0, fma chain over
// f0..f6 in index order starting from c).  reg = {c, w0..w6}.
void orc_predict(const uint16_t* feat, uint32_t n, const float* reg, float* u) {
  for (uint32_t i = 0; i < n; ++i) {
    float acc = reg[0];
    for (int k = 0; k < 7; ++k) acc = std::fmaf(reg[1 + k], float(feat[size_t(i) * 8 + k]), acc);
    u[i] = acc > 0.0f ? acc : 0.0f;
  }
}

// O4 (Eq. 2, Eq. 3, d = μ|J| P:357 / φ|J| P:1288,
// offload Alg. 1): D_us = min(tightness*mu_us*ntok, 2^32-1) unless
// D_in is given; key = cls<<63 | tier<<62 | ord(v).
// r_us (arrival) may be NULL (= all zero); D_in may be NULL; D_out may be NULL.
void orc_key(const float* u, const uint16_t* feat, const int64_t* r_us, const uint32_t* D_in, uint32_t n,
             const orc_profile* p, uint64_t* key, uint32_t* D_out) {
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t D_us;
    if (D_in) {
      D_us = D_in[i];
    } else {
      int64_t d = int64_t(p->tightness) * p->mu_us * int64_t(feat[size_t(i) * 8 + 6]);
      D_us = d > int64_t(0xFFFFFFFFu) ? 0xFFFFFFFFu : uint32_t(d);
    }
    if (D_out) D_out[i] = D_us;
    const float ui = u[i];
    const int64_t r = r_us ? r_us[i] : 0;
    uint64_t tier = 0, val = 0;
    if (p->policy == 4 || p->policy == 5) {  // SLACK (Eq. 2) / UP (Eq. 3)
      float D = float(D_us);
      float num = 1.0f;
      if (p->policy == 5) {
        float un = p->raw_numerator ? ui : std::fmin(1.0f, ui / p->u_max);
        float t = p->alpha * un;
        num = 1.0f - t;
      }
      float etau = float(p->eta_us) * ui;
      float slk = D - etau;
      float v;
      if (slk <= 1.0f) {  // overdue tier, most-negative slack first (DESIGN R-OVERDUE)
        tier = 1;
        v = -slk;
      } else {
        v = num / slk;
      }
      val = ord32(v);
    } else if (p->policy == 0) {  // FIFO: p = -r
      val = uint64_t(-r + (int64_t(1) << 61));
    } else if (p->policy == 1) {  // EDF / HPF: p = -(r + D)
      val = uint64_t(-(r + int64_t(D_us)) + (int64_t(1) << 61));
    } else if (p->policy == 2) {  // LUF: p = -u
      val = ord32(-ui);
    } else {  // MUF: p = +u
      val = ord32(ui);
    }
    uint64_t cls = (p->offload && ui > p->tau) ? 1 : 0;  // strict
    key[i] = (cls << 63) | (tier << 62) | val;
  }
}

// O5: per segment, stable sort by key descending (input order breaks ties,
// S:345).  perm receives global indices.
void orc_order(const uint64_t* key, const uint32_t* seg_off, uint32_t nseg, uint32_t* perm) {
  for (uint32_t s = 0; s < nseg; ++s) {
    std::vector<uint32_t> idx;
    for (uint32_t i = seg_off[s]; i < seg_off[s + 1]; ++i) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return key[a] > key[b]; });
    std::copy(idx.begin(), idx.end(), perm + seg_off[s]);
  }
}

// O6 one-pass schedule (Alg. 1 online part P:467-481; §IV-C bullets
// P:410-419; flush P:490-492).  Returns the total number of GPU batches.
// batch_of: global GPU batch id (UINT32_MAX for CPU tasks); slot_of: position
// in the batch; core_of: CPU core (0xFF for GPU tasks); seg_batch_off[nseg+1].
uint32_t orc_schedule(const uint64_t* key, const float* u, const uint32_t* seg_off, uint32_t nseg,
                      const orc_profile* p, uint32_t cores, uint32_t* perm, uint32_t* batch_of, uint8_t* slot_of,
                      uint8_t* core_of, uint32_t* seg_batch_off) {
  orc_order(key, seg_off, nseg, perm);
  const uint32_t C = uint32_t(p->C);
  const uint32_t m = uint32_t(p->b10) * C / 10;  // ⌊b·C⌋ with b in tenths (DESIGN R-B)
  uint32_t nb = 0;
  seg_batch_off[0] = 0;
  for (uint32_t s = 0; s < nseg; ++s) {
    const uint32_t lo = seg_off[s], hi = seg_off[s + 1];
    // CPU class: key order, one task per CPU batch, list scheduling on the
    // predicted latency γ·(base + ceil(η·u)) (DESIGN R-CORE)
    std::vector<int64_t> free_at(cores, 0);
    std::vector<uint32_t> gpu;  // GPU-class stream in priority order
    std::vector<uint32_t> rank(hi - lo);
    for (uint32_t j = lo; j < hi; ++j) {
      const uint32_t i = perm[j];
      rank[i - lo] = j - lo;
      if (key[i] >> 63) {
        uint32_t best = 0;
        for (uint32_t c = 1; c < cores; ++c)
          if (free_at[c] < free_at[best]) best = c;
        float eu = float(p->eta_us) * u[i];
        int64_t pred = int64_t(p->gamma) * (p->base_us + int64_t(std::ceil(eu)));
        if (cores) free_at[best] += pred;
        core_of[i] = cores ? uint8_t(best) : 0xFF;
        batch_of[i] = 0xFFFFFFFFu;
        slot_of[i] = 0;
      } else {
        gpu.push_back(i);
        core_of[i] = 0xFF;
      }
    }
    // GPU class: windows of m, ascending-u sort, λ/C cut, carry back
    std::vector<uint32_t> W;
    size_t ptr = 0;
    uint32_t b = 0;
    for (;;) {
      while (W.size() < m && ptr < gpu.size()) W.push_back(gpu[ptr++]);
      if (W.empty()) break;
      std::sort(W.begin(), W.end(), [&](uint32_t x, uint32_t y) {
        if (u[x] != u[y]) return u[x] < u[y];
        return rank[x - lo] < rank[y - lo];
      });
      size_t lim = std::min<size_t>(C, W.size());
      size_t cnt = 1;
      while (cnt < lim) {
        float bound = p->lambda * u[W[cnt - 1]];
        if (!(u[W[cnt]] <= bound)) break;
        ++cnt;
      }
      for (size_t k = 0; k < cnt; ++k) {
        batch_of[W[k]] = nb + b;
        slot_of[W[k]] = uint8_t(k);
      }
      W.erase(W.begin(), W.begin() + long(cnt));
      ++b;
    }
    nb += b;
    seg_batch_off[s + 1] = nb;
  }
  return nb;
}

// O7 replay (§V-A workload P:1580-1589; response P:634-635 / P:1596; miss
// P:673-676; DESIGN R-REPLAY).  Tasks of trace t are [trace_off[t],
// trace_off[t+1]) in arrival order.  end_us may be NULL.
// util (nullable, NEXT-4 / SPEC S:374): per trace, the executors' busy
// time accumulated as the loop dispatches -- each GPU batch adds its duration
// setup + base + eta*max len, each CPU task gamma*(base + eta*len)
// -- and the counts of GPU batches and CPU tasks.
struct orc_util {
  int64_t gpu_busy_us, cpu_busy_us;
  uint32_t gpu_batches, cpu_tasks;
};

void orc_simulate_util(const int64_t* r, const uint16_t* len, const float* u, const uint64_t* key, const uint32_t* D,
                       const uint32_t* trace_off, uint32_t nt, const orc_profile* profs, const uint16_t* trace_prof,
                       orc_stats* stats, int64_t* end_us, orc_util* util) {
  for (uint32_t t = 0; t < nt; ++t) {
    const orc_profile& p = profs[trace_prof ? trace_prof[t] : 0];
    const uint32_t lo = trace_off[t], n = trace_off[t + 1] - lo;
    const uint32_t C = uint32_t(p.C), m = uint32_t(p.b10) * C / 10, cores = uint32_t(p.cores);
    // key rank within the trace (stable, descending key)
    std::vector<uint32_t> order(n), rank(n);
    for (uint32_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key[lo + a] > key[lo + b]; });
    for (uint32_t j = 0; j < n; ++j) rank[order[j]] = j;

    std::vector<int64_t> end(n, -1), core_free(cores, 0);
    std::set<std::pair<uint32_t, uint32_t>> ready_gpu, ready_cpu;  // (rank, i)
    std::set<uint32_t> gpu_by_arrival;                              // arrival index
    int64_t gpu_free = 0;
    orc_util ut{0, 0, 0u, 0u};
    uint32_t next = 0, done = 0;
    int64_t now = n ? r[lo] : 0;
    while (done < n) {
      // admit arrivals <= now, by class
      while (next < n && r[lo + next] <= now) {
        if (key[lo + next] >> 63) ready_cpu.insert({rank[next], next});
        else {
          ready_gpu.insert({rank[next], next});
          gpu_by_arrival.insert(next);
        }
        ++next;
      }
      // CPU cores: highest key on the lowest-index free core
      for (uint32_t c = 0; c < cores && !ready_cpu.empty(); ++c) {
        if (core_free[c] > now) continue;
        uint32_t i = ready_cpu.begin()->second;
        ready_cpu.erase(ready_cpu.begin());
        int64_t e = now + int64_t(p.gamma) * (p.base_us + p.eta_us * int64_t(len[lo + i]));
        end[i] = e;
        core_free[c] = e;
        ut.cpu_busy_us += e - now;
        ++ut.cpu_tasks;
        ++done;
      }
      // GPU dispatch
      bool waiting = false;
      if (gpu_free <= now && !ready_gpu.empty()) {
        uint32_t oldest = *gpu_by_arrival.begin();
        bool flush = (r[lo + oldest] <= now - p.xi_us) || next == n;
        std::vector<uint32_t> batch;
        if (p.consolidate) {
          if (ready_gpu.size() >= m || flush) {
            std::vector<uint32_t> Wd;
            for (auto it = ready_gpu.begin(); it != ready_gpu.end() && Wd.size() < m; ++it) Wd.push_back(it->second);
            std::sort(Wd.begin(), Wd.end(), [&](uint32_t x, uint32_t y) {
              if (u[lo + x] != u[lo + y]) return u[lo + x] < u[lo + y];
              return rank[x] < rank[y];
            });
            size_t lim = std::min<size_t>(C, Wd.size()), cnt = 1;
            while (cnt < lim) {
              float bound = p.lambda * u[lo + Wd[cnt - 1]];
              if (!(u[lo + Wd[cnt]] <= bound)) break;
              ++cnt;
            }
            batch.assign(Wd.begin(), Wd.begin() + long(cnt));
          }
        } else if (ready_gpu.size() >= C || flush) {
          for (auto it = ready_gpu.begin(); it != ready_gpu.end() && batch.size() < C; ++it) batch.push_back(it->second);
        }
        if (batch.empty()) {
          waiting = true;
        } else {
          int64_t mx = 0;
          for (uint32_t i : batch) mx = std::max<int64_t>(mx, len[lo + i]);
          int64_t e = now + p.setup_us + p.base_us + p.eta_us * mx;
          for (uint32_t i : batch) {
            end[i] = e;
            ready_gpu.erase({rank[i], i});
            gpu_by_arrival.erase(i);
            ++done;
          }
          gpu_free = e;
          ut.gpu_busy_us += e - now;
          ++ut.gpu_batches;
        }
      }
      if (done == n) break;
      // next event time
      int64_t nxt = INT64_MAX;
      if (next < n) nxt = std::min(nxt, r[lo + next]);
      if (gpu_free > now) nxt = std::min(nxt, gpu_free);
      if (!ready_cpu.empty())
        for (uint32_t c = 0; c < cores; ++c)
          if (core_free[c] > now) nxt = std::min(nxt, core_free[c]);
      if (waiting) nxt = std::min(nxt, r[lo + *gpu_by_arrival.begin()] + p.xi_us);
      now = nxt;
    }
    orc_stats st{0, n, 0};
    for (uint32_t i = 0; i < n; ++i) {
      st.sum_resp_us += end[i] - r[lo + i];
      if (end[i] > r[lo + i] + int64_t(D[lo + i])) ++st.misses;
      if (end_us) end_us[lo + i] = end[i];
    }
    stats[t] = st;
    if (util) util[t] = ut;
  }
}

void orc_simulate(const int64_t* r, const uint16_t* len, const float* u, const uint64_t* key, const uint32_t* D,
                  const uint32_t* trace_off, uint32_t nt, const orc_profile* profs, const uint16_t* trace_prof,
                  orc_stats* stats, int64_t* end_us) {
  orc_simulate_util(r, len, u, key, D, trace_off, nt, profs, trace_prof, stats, end_us, nullptr);
}

}  // extern "C"
