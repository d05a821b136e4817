// api.cu — the C ABI of include/rtlm.h: context, lexicon upload, argument
// validation, workspace, launches.  No compute happens on the host.
#include <atomic>
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

struct rt_ctx {
  int device = 0;
  int num_sms = 148;
  uint32_t sm_limit = 0;  // rt_set_sm_limit (0: one CTA per SM)
  rtlm::LexEntry* d_entries = nullptr;
  uint4* d_keys = nullptr;
  uint32_t* d_slots = nullptr;
  uint32_t n_entries = 0, bits = 0, seed = 0;
  uint32_t* d_flags = nullptr;
  uint16_t* d_tok = nullptr;  // scoring token buffers (one per persistent warp)
  void* ws = nullptr;
  size_t ws_size = 0;
  uint32_t* d_off = nullptr;  // device copy of segment / trace offsets
  size_t off_cap = 0;
  rt_profile* d_prof = nullptr;
  size_t prof_cap = 0;
  cudaStream_t aux = nullptr;  // internal fork stream (CPU-class list scheduling)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint8_t* d_mlp = nullptr;  // packed MLP weights (rt_set_mlp): bf16 tensor-core blob
  float* d_mlp32 = nullptr;  // fp32 blob (k_mlp_f32)
  uint8_t* d_mlptf = nullptr;  // hi / lo tf32 blob (k_mlp_tf32)
  int mlp_precision = RT_MLP_FP32;
  std::vector<float> mlp_host;  // the current weights, fp32, flat: W0 b0 W1 b1 .. W4 b4 (rt_set_mlp / rt_train_mlp)
  void* io = nullptr;        // device buffers of rt_score_schedule_host
  size_t io_size = 0;
  uint64_t* kbuf = nullptr;  // keys of rt_schedule_deadlines
  size_t kbuf_n = 0;
  // pinned staging of small host arguments (segment / trace offsets, profiles): a
  // copy from pageable memory would synchronise the stream before it starts
  struct HostStage {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
  } st_off, st_prof;
  // pinned blocks staged while a stream was being captured into a CUDA graph:
  // the graph's copy nodes read them at every replay, so they are never reused
  // (freed with the context)
  std::vector<void*> captured_stage;
  // device buffers replaced after a capture: a graph may still address them
  bool captured = false;
  std::vector<void*> retired;
  std::string err;
};

namespace rtlm {
static std::atomic<unsigned long long> g_launches{0};
void note_launch(unsigned k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace rtlm

namespace {

using rtlm::LexEntry;

constexpr uint32_t kMlpDims[6] = {6, 100, 200, 200, 100, 1};  // m_theta

thread_local std::string t_err;  // the calling thread's last error (rt_last_error(NULL))

rt_status fail(rt_ctx* c, rt_status st, const std::string& msg) {
  t_err = msg;
  if (c) c->err = msg;
  return st;
}
rt_status cuda_fail(rt_ctx* c, cudaError_t e, const char* where) {
  return fail(c, RT_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define RT_CUDA(ctx, call)                                  \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------ lexicon (host)
bool is_w(unsigned char b) {
  return (b >= 'a' && b <= 'z') || (b >= 'A' && b <= 'Z') || (b >= '0' && b <= '9') || b == '\'';
}

// R-LEMMA on a lowercased word (host side of the product; the device has its
// own register-level implementation in k_score.cu).
std::string lemma_host(const std::string& lw) {
  const size_t n = lw.size();
  if (lw == "n't") return "not";
  auto tail = [&](const char* s) {
    size_t k = std::strlen(s);
    return n >= k && std::memcmp(lw.data() + n - k, s, k) == 0;
  };
  size_t strip = 0;
  if (n >= 5 && tail("ing")) strip = 3;
  else if (n >= 4 && tail("ed")) strip = 2;
  else if (n >= 4 && tail("es")) strip = 2;
  else if (n >= 3 && tail("s") && !tail("ss")) strip = 1;
  return lw.substr(0, n - strip);
}

// true when R-CLITIC would split this W run (so it is not a single token)
bool clitic_splits(const std::string& lw) {
  const size_t n = lw.size();
  auto tail = [&](const char* s) {
    size_t k = std::strlen(s);
    return n >= k && std::memcmp(lw.data() + n - k, s, k) == 0;
  };
  if (n > 3 && tail("n't")) return true;
  if (n > 2 && (tail("'s") || tail("'m") || tail("'d"))) return true;
  if (n > 3 && (tail("'re") || tail("'ve") || tail("'ll"))) return true;
  return false;
}

struct HostLemma {
  uint32_t flags = 0;
  uint32_t tags = 0;
  uint32_t senses = 0;
  uint32_t id = 0;
};

const char* kTags[] = {"NOUN", "PROPN", "VERB", "ADJ", "ADV", "ADP", "PRON", "DET", "CCONJ",
                       "SCONJ", "NUM", "PART", "INTJ", "AUX", "X", "SYM", "PUNCT"};

std::string strip_ws(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
  return s.substr(a, b - a);
}

bool parse_lexicon(const char* text, size_t len, std::vector<std::string>& lemmas, std::vector<HostLemma>& attrs,
                   std::string& err) {
  enum Sec { NONE, VAGUE, POLY, POS, WH, COORD, PREP } sec = NONE;
  size_t pos = 0;
  int line_no = 0;
  while (pos <= len) {
    size_t eol = pos;
    while (eol < len && text[eol] != '\n') ++eol;
    std::string line(text + pos, eol - pos);
    pos = eol + 1;
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const std::string t = strip_ws(line);
    auto bad = [&](const std::string& m) {
      err = "lexicon line " + std::to_string(line_no) + ": " + m;
      return false;
    };
    if (t.empty() || t[0] == '#') {
      if (eol >= len) break;
      continue;
    }
    if (t.back() == ':' && t.find('\t') == std::string::npos) {
      const std::string name = t.substr(0, t.size() - 1);
      if (name == "vague") sec = VAGUE;
      else if (name == "polysemy") sec = POLY;
      else if (name == "pos") sec = POS;
      else if (name == "wh") sec = WH;
      else if (name == "coord") sec = COORD;
      else if (name == "prep") sec = PREP;
      else return bad("unknown section '" + name + "'");
      if (eol >= len) break;
      continue;
    }
    if (sec == NONE) return bad("entry before any section header");
    const size_t tab = line.find('\t');
    const std::string word = strip_ws(tab == std::string::npos ? line : line.substr(0, tab));
    const std::string value = tab == std::string::npos ? std::string() : strip_ws(line.substr(tab + 1));
    std::string lw;
    for (unsigned char ch : word) {
      if (!is_w(ch)) return bad("entry '" + word + "' is not a single word token");
      lw.push_back((char)(ch | 0x20));
    }
    if (lw.empty() || clitic_splits(lw)) return bad("entry '" + word + "' is not a single word token");
    const std::string lem = lemma_host(lw);
    if (lem.empty() || lem.size() > 16) return bad("lemma of '" + word + "' longer than 16 bytes");
    size_t k = 0;
    while (k < lemmas.size() && lemmas[k] != lem) ++k;
    if (k == lemmas.size()) {
      if (lemmas.size() >= rtlm::kMaxLexEntries) return bad("more than 1024 distinct lemmas");
      lemmas.push_back(lem);
      HostLemma h;
      h.id = (uint32_t)k;
      attrs.push_back(h);
    }
    HostLemma& h = attrs[k];
    switch (sec) {
      case VAGUE:
      case COORD:
      case PREP:
        if (!value.empty()) return bad("unexpected value");
        h.flags |= sec == VAGUE ? rtlm::A_VAGUE : sec == COORD ? rtlm::A_COORD : rtlm::A_PREP;
        break;
      case POLY: {
        char* end = nullptr;
        long v = std::strtol(value.c_str(), &end, 10);
        if (value.empty() || *end || v < 2 || v > 255) return bad("polysemy count must be an integer in [2,255]");
        if ((uint32_t)v > h.senses) h.senses = (uint32_t)v;
        break;
      }
      case POS: {
        if (value.empty()) return bad("pos entry without tags");
        size_t a = 0;
        while (a <= value.size()) {
          size_t b = value.find(',', a);
          if (b == std::string::npos) b = value.size();
          const std::string tag = strip_ws(value.substr(a, b - a));
          int idx = -1;
          for (int q = 0; q < (int)(sizeof(kTags) / sizeof(kTags[0])); ++q)
            if (tag == kTags[q]) idx = q;
          if (idx < 0) return bad("unknown PoS tag '" + tag + "'");
          h.tags |= 1u << idx;
          a = b + 1;
        }
        break;
      }
      case WH: {
        if (value.empty()) return bad("wh entry without flags");
        size_t a = 0;
        while (a <= value.size()) {
          size_t b = value.find('|', a);
          if (b == std::string::npos) b = value.size();
          const std::string f = strip_ws(value.substr(a, b - a));
          if (f == "OPENER") h.flags |= rtlm::A_OPENER;
          else if (f == "WHAT") h.flags |= rtlm::A_WHAT;
          else if (f == "CAUSE") h.flags |= rtlm::A_CAUSE;
          else if (f == "BROAD") h.flags |= rtlm::A_BROAD;
          else return bad("unknown wh flag '" + f + "'");
          a = b + 1;
        }
        break;
      }
      default:
        break;
    }
    if (eol >= len) break;
  }
  return true;
}

rt_status upload_lexicon(rt_ctx* c, const char* text, size_t len) {
  std::vector<std::string> lemmas;
  std::vector<HostLemma> attrs;
  std::string err;
  if (!parse_lexicon(text, len, lemmas, attrs, err)) return fail(c, RT_ELEXICON, err);
  const uint32_t n = (uint32_t)lemmas.size();
  uint32_t bits = 6;
  while ((1u << bits) < 4 * n) ++bits;  // load factor <= 1/4
  std::vector<LexEntry> ent(n);
  std::vector<uint4> keys(n + 1, uint4{0, 0, 0, 0});
  for (uint32_t k = 0; k < n; ++k) {
    LexEntry e{};
    uint32_t w[4] = {0, 0, 0, 0};
    for (size_t b = 0; b < lemmas[k].size(); ++b) {
      uint64_t byte = (unsigned char)lemmas[k][b];
      if (b < 8) e.k0 |= byte << (8 * b);
      else e.k1 |= byte << (8 * (b - 8));
      w[b >> 2] |= (uint32_t)byte << (8 * (b & 3));
    }
    e.len = (uint32_t)lemmas[k].size();
    const HostLemma& h = attrs[k];
    uint32_t a = h.flags;
    if (h.tags & 3u) a |= rtlm::A_NOUN;                   // NOUN or PROPN
    if (__builtin_popcount(h.tags) >= 2) a |= rtlm::A_MULTIPOS;
    if (h.senses >= 2) a |= (h.senses - 1) << rtlm::A_SEM_SHIFT;
    a |= h.id << rtlm::A_ID_SHIFT;
    e.attr = a;
    ent[k] = e;
    keys[k + 1] = uint4{w[0], w[1], w[2], w[3]};
  }
  // cuckoo placement (two slots per key); a new seed if an insertion cycles
  std::vector<uint32_t> slots;
  uint32_t seed = 0;
  for (;; ++seed) {
    slots.assign(1u << bits, 0);
    bool ok = true;
    for (uint32_t k = 0; k < n && ok; ++k) {
      uint32_t cur = k + 1;
      bool placed = false;
      for (int kick = 0; kick < 512 && !placed; ++kick) {
        const uint4& q = keys[cur];
        const uint32_t x = rtlm::lex_mix(q.x, q.y, q.z, q.w, seed);
        const uint32_t s1 = rtlm::lex_slot1(x, bits), s2 = rtlm::lex_slot2(x, bits);
        if (!slots[s1]) { slots[s1] = cur; placed = true; }
        else if (!slots[s2]) { slots[s2] = cur; placed = true; }
        else {  // evict the occupant of the slot that is not where we came from
          const uint32_t s = (kick & 1) ? s2 : s1;
          const uint32_t ev = slots[s];
          slots[s] = cur;
          cur = ev;
        }
      }
      ok = placed;
    }
    if (ok) break;
    if (seed > 1000) return fail(c, RT_ELEXICON, "lexicon hash table could not be built");
  }
  // each occupied slot also carries the top 21 bits of its key's hash (the
  // device compares one key: the one whose fingerprint matches)
  for (uint32_t& v : slots) {
    if (!v) continue;
    const uint4& q = keys[v];
    v |= (rtlm::lex_mix(q.x, q.y, q.z, q.w, seed) >> 11) << 11;
  }
  c->n_entries = n;
  c->bits = bits;
  c->seed = seed;
  RT_CUDA(c, cudaMalloc(&c->d_entries, std::max<size_t>(1, n) * sizeof(LexEntry)));
  RT_CUDA(c, cudaMalloc(&c->d_keys, keys.size() * sizeof(uint4)));
  RT_CUDA(c, cudaMalloc(&c->d_slots, slots.size() * sizeof(uint32_t)));
  if (n) RT_CUDA(c, cudaMemcpy(c->d_entries, ent.data(), n * sizeof(LexEntry), cudaMemcpyHostToDevice));
  RT_CUDA(c, cudaMemcpy(c->d_keys, keys.data(), keys.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  RT_CUDA(c, cudaMemcpy(c->d_slots, slots.data(), slots.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  return RT_OK;
}

rtlm::DevLexicon dev_lex(const rt_ctx* c) {
  return rtlm::DevLexicon{c->d_entries, c->d_keys, c->d_slots, c->n_entries, c->bits, c->seed};
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive;
}

// a device buffer being replaced: freed, unless a graph captured on this
// context may still address it (then kept until rt_destroy)
void retire(rt_ctx* c, void* p) {
  if (!p) return;
  if (c->captured) c->retired.push_back(p);
  else cudaFree(p);
}

// device buffers only grow outside graph capture (a free would synchronise)
rt_status no_growth_in_capture(rt_ctx* c, cudaStream_t s) {
  if (capturing(s))
    return fail(c, RT_EINVAL, "buffer growth during CUDA graph capture: run the call once before capturing it");
  return RT_OK;
}

rt_status ensure_ws(rt_ctx* c, size_t bytes, cudaStream_t s) {
  if (bytes <= c->ws_size) return RT_OK;
  if (no_growth_in_capture(c, s) != RT_OK) return RT_EINVAL;
  retire(c, c->ws);  // cudaFree: implicit device sync, no in-flight user
  c->ws = nullptr;
  c->ws_size = 0;
  cudaError_t e = cudaMalloc(&c->ws, bytes);
  if (e != cudaSuccess) return fail(c, RT_ENOMEM, std::string("workspace: ") + cudaGetErrorString(e));
  c->ws_size = bytes;
  return RT_OK;
}

// host -> device copy through a pinned staging buffer (waits only for the
// previous copy out of the same buffer)
rt_status stage_copy(rt_ctx* c, rt_ctx::HostStage& st, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (capturing(s)) {  // a block of its own for the graph (see rt_ctx::captured_stage)
    c->captured = true;
    void* p = nullptr;
    RT_CUDA(c, cudaMallocHost(&p, bytes));
    c->captured_stage.push_back(p);
    std::memcpy(p, src, bytes);
    RT_CUDA(c, cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
    return RT_OK;
  }
  if (!st.ev) RT_CUDA(c, cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming));
  else RT_CUDA(c, cudaEventSynchronize(st.ev));
  if (bytes > st.cap) {
    if (st.p) cudaFreeHost(st.p);
    st.p = nullptr;
    st.cap = 0;
    RT_CUDA(c, cudaMallocHost(&st.p, bytes));
    st.cap = bytes;
  }
  std::memcpy(st.p, src, bytes);
  RT_CUDA(c, cudaMemcpyAsync(dst, st.p, bytes, cudaMemcpyHostToDevice, s));
  RT_CUDA(c, cudaEventRecord(st.ev, s));
  return RT_OK;
}

rt_status upload_offsets(rt_ctx* c, const uint32_t* h, uint32_t count, cudaStream_t s) {
  if (count > c->off_cap) {
    if (no_growth_in_capture(c, s) != RT_OK) return RT_EINVAL;
    retire(c, c->d_off);
    c->d_off = nullptr;
    c->off_cap = 0;
    if (cudaMalloc(&c->d_off, (size_t)count * 4) != cudaSuccess) return fail(c, RT_ENOMEM, "offsets buffer");
    c->off_cap = count;
  }
  return stage_copy(c, c->st_off, c->d_off, h, (size_t)count * 4, s);
}

rt_status check_profile(rt_ctx* c, const rt_profile* p, bool need_cores) {
  if (!p) return fail(c, RT_EINVAL, "profile is NULL");
  if (p->policy < RT_FIFO || p->policy > RT_UP) return fail(c, RT_EINVAL, "policy out of range");
  if (p->C < 1 || p->C > (int)rtlm::kMaxWindow) return fail(c, RT_EINVAL, "C must be in [1,128]");
  if (p->b10 < 10) return fail(c, RT_EINVAL, "b must be >= 1 (b10 >= 10, S:264)");
  if ((int64_t)p->b10 * p->C / 10 > (int64_t)rtlm::kMaxWindow) return fail(c, RT_EINVAL, "window b*C must be <= 128");
  if (!(p->lambda >= 1.0f)) return fail(c, RT_EINVAL, "lambda must be >= 1 (S:264)");
  if (!(p->u_max > 0.0f) && !p->raw_numerator && p->policy == RT_UP) return fail(c, RT_EINVAL, "u_max must be > 0");
  if (p->cores < 0 || p->cores > (int)rtlm::kMaxCores) return fail(c, RT_EINVAL, "cores must be in [0,32]");
  if (need_cores && p->cores < 1) return fail(c, RT_EINVAL, "replay needs cores >= 1");
  if (p->eta_us < 0 || p->mu_us < 0 || p->base_us < 0 || p->setup_us < 0 || p->xi_us < 0 || p->gamma < 0 ||
      p->tightness < 0)
    return fail(c, RT_EINVAL, "negative time coefficient");
  if (p->reserved != 0) return fail(c, RT_EINVAL, "reserved must be 0");
  return RT_OK;
}

cudaStream_t cs(rt_stream s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int rt_abi_version(void) { return RTLM_ABI_VERSION; }

uint64_t rt_launch_count(void) { return rtlm::g_launches.load(); }

rt_status rt_create(int device, const char* lexicon_text, size_t len, rt_ctx** out) {
  if (!out) return RT_EINVAL;
  *out = nullptr;
  rt_ctx* c = new rt_ctx();
  *out = c;
  c->device = device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(c, RT_EINVAL, "no such CUDA device");
  DeviceGuard g(device);
  RT_CUDA(c, cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  RT_CUDA(c, cudaMalloc(&c->d_flags, 4 * sizeof(uint32_t)));  // [0] flags, [2] scoring work counter, [3] its CTA counter
  RT_CUDA(c, cudaMemset(c->d_flags, 0, 4 * sizeof(uint32_t)));
  RT_CUDA(c, cudaMalloc(&c->d_tok, rtlm::score_scratch_bytes(c->num_sms)));
  RT_CUDA(c, cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  RT_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  RT_CUDA(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  if (!lexicon_text && len) return fail(c, RT_EINVAL, "lexicon_text is NULL");
  return upload_lexicon(c, lexicon_text ? lexicon_text : "", len);
}

rt_status rt_destroy(rt_ctx* c) {
  if (!c) return RT_OK;
  {
    DeviceGuard g(c->device);
    cudaFree(c->d_entries);
    cudaFree(c->d_keys);
    cudaFree(c->d_slots);
    cudaFree(c->d_flags);
    cudaFree(c->d_tok);
    cudaFree(c->ws);
    cudaFree(c->d_off);
    cudaFree(c->d_prof);
    cudaFree(c->d_mlp);
    cudaFree(c->d_mlp32);
    cudaFree(c->d_mlptf);
    cudaFree(c->io);
    cudaFree(c->kbuf);
    for (void* p : c->captured_stage) cudaFreeHost(p);
    for (void* p : c->retired) cudaFree(p);
    for (rt_ctx::HostStage* st : {&c->st_off, &c->st_prof}) {
      if (st->p) cudaFreeHost(st->p);
      if (st->ev) cudaEventDestroy(st->ev);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->aux) cudaStreamDestroy(c->aux);
  }
  delete c;
  return RT_OK;
}

const char* rt_last_error(const rt_ctx* c) { return c ? c->err.c_str() : t_err.c_str(); }

uint32_t rt_lexicon_size(const rt_ctx* c) { return c ? c->n_entries : 0; }

rt_status rt_set_sm_limit(rt_ctx* c, uint32_t max_ctas) {
  if (!c) return RT_EINVAL;
  c->sm_limit = max_ctas;
  return RT_OK;
}

static int persistent_ctas(const rt_ctx* c) {
  return (c->sm_limit && (int)c->sm_limit < c->num_sms) ? (int)c->sm_limit : c->num_sms;
}

rt_status rt_get_flags(rt_ctx* c, uint32_t* flags) {
  if (!c || !flags) return fail(c, RT_EINVAL, "null argument");
  DeviceGuard g(c->device);
  RT_CUDA(c, cudaDeviceSynchronize());
  RT_CUDA(c, cudaMemcpy(flags, c->d_flags, 4, cudaMemcpyDeviceToHost));
  RT_CUDA(c, cudaMemset(c->d_flags, 0, 4));
  return RT_OK;
}

static rt_status score_common(rt_ctx* c, const uint8_t* d_bytes, const uint32_t* d_offsets, uint32_t n, int fused,
                              const rt_regressor* reg, const rt_profile* prof, const int64_t* d_arr,
                              const uint32_t* d_D_in, uint16_t* d_feat, float* d_u, uint64_t* d_key,
                              uint32_t* d_D_out, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (n == 0) return RT_OK;
  if (!d_offsets || !d_bytes) return fail(c, RT_EINVAL, "bytes/offsets are NULL");
  if (reinterpret_cast<uintptr_t>(d_bytes) & 15u) return fail(c, RT_EINVAL, "d_bytes must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(d_feat) & 15u) return fail(c, RT_EINVAL, "d_feat must be 16-byte aligned");
  if (n > 0xFFFFFFFEu) return fail(c, RT_EOVERFLOW, "n too large");
  if (fused) {
    if (!reg || !d_u || !d_key) return fail(c, RT_EINVAL, "regressor / u / key are required");
    rt_status st = check_profile(c, prof, false);
    if (st != RT_OK) return st;
  } else if (!d_feat) {
    return fail(c, RT_EINVAL, "d_feat is NULL");
  }
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  rtlm::ScoreLaunch a{};
  a.bytes = d_bytes;
  a.offsets = d_offsets;
  a.n = n;
  a.lex = dev_lex(c);
  a.fused = fused;
  if (reg) a.reg = *reg;
  if (prof) a.prof = *prof;
  a.arrival = d_arr;
  a.D_in = d_D_in;
  a.feat = d_feat;
  a.u = d_u;
  a.key = d_key;
  a.D_out = d_D_out;
  a.flags = c->d_flags;
  a.work = c->d_flags + 2;
  a.tokbuf = c->d_tok;
  a.num_sms = persistent_ctas(c);
  cudaError_t e = rtlm::launch_score(a, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_score");
  return RT_OK;
}

rt_status rt_score(rt_ctx* c, const uint8_t* d_bytes, const uint32_t* d_offsets, uint32_t n, uint16_t* d_feat,
                   rt_stream stream) {
  return score_common(c, d_bytes, d_offsets, n, 0, nullptr, nullptr, nullptr, nullptr, d_feat, nullptr, nullptr,
                      nullptr, stream);
}

rt_status rt_score_key(rt_ctx* c, const uint8_t* d_bytes, const uint32_t* d_offsets, uint32_t n,
                       const rt_regressor* reg, const rt_profile* prof, const int64_t* d_arr, const uint32_t* d_D_in,
                       uint16_t* d_feat, float* d_u, uint64_t* d_key, uint32_t* d_D_out, rt_stream stream) {
  return score_common(c, d_bytes, d_offsets, n, 1, reg, prof, d_arr, d_D_in, d_feat, d_u, d_key, d_D_out, stream);
}

rt_status rt_predict(rt_ctx* c, const uint16_t* d_feat, uint32_t n, const rt_regressor* reg, float* d_u,
                     rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!n) return RT_OK;
  if (!d_feat || !reg || !d_u) return fail(c, RT_EINVAL, "null argument");
  if (reinterpret_cast<uintptr_t>(d_feat) & 15u) return fail(c, RT_EINVAL, "d_feat must be 16-byte aligned");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaError_t e = rtlm::launch_predict(d_feat, n, *reg, d_u, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_predict");
  return RT_OK;
}

rt_status rt_set_mlp(rt_ctx* c, const rt_mlp* mlp) {
  if (!c) return RT_EINVAL;
  if (!mlp) return fail(c, RT_EINVAL, "mlp is NULL");
  for (int l = 0; l < 5; ++l)
    if (!mlp->w[l] || !mlp->b[l]) return fail(c, RT_EINVAL, "null MLP weight or bias");
  DeviceGuard g(c->device);
  {  // host copy of the weights (the starting point of rt_train_mlp, rt_get_mlp)
    std::vector<float> flat;
    for (int l = 0; l < 5; ++l) {
      const size_t nw = (size_t)kMlpDims[l + 1] * kMlpDims[l];
      flat.insert(flat.end(), mlp->w[l], mlp->w[l] + nw);
      flat.insert(flat.end(), mlp->b[l], mlp->b[l] + kMlpDims[l + 1]);
    }
    c->mlp_host.swap(flat);
  }
  std::vector<uint8_t> blob(rtlm::mlp_blob_bytes());
  rtlm::mlp_pack(mlp->w, mlp->b, blob.data());
  if (!c->d_mlp) {
    cudaError_t e = cudaMalloc(&c->d_mlp, blob.size());
    if (e != cudaSuccess) return fail(c, RT_ENOMEM, std::string("mlp weights: ") + cudaGetErrorString(e));
  }
  RT_CUDA(c, cudaMemcpy(c->d_mlp, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  std::vector<float> blob32(rtlm::mlp_f32_blob_bytes() / 4);
  rtlm::mlp_f32_pack(mlp->w, mlp->b, blob32.data());
  if (!c->d_mlp32) {
    cudaError_t e = cudaMalloc(&c->d_mlp32, rtlm::mlp_f32_blob_bytes());
    if (e != cudaSuccess) return fail(c, RT_ENOMEM, std::string("mlp weights: ") + cudaGetErrorString(e));
  }
  RT_CUDA(c, cudaMemcpy(c->d_mlp32, blob32.data(), rtlm::mlp_f32_blob_bytes(), cudaMemcpyHostToDevice));
  std::vector<uint8_t> blobtf(rtlm::mlp_tf32_blob_bytes());
  rtlm::mlp_tf32_pack(mlp->w, mlp->b, blobtf.data());
  if (!c->d_mlptf) {
    cudaError_t e = cudaMalloc(&c->d_mlptf, blobtf.size());
    if (e != cudaSuccess) return fail(c, RT_ENOMEM, std::string("mlp weights: ") + cudaGetErrorString(e));
  }
  RT_CUDA(c, cudaMemcpy(c->d_mlptf, blobtf.data(), blobtf.size(), cudaMemcpyHostToDevice));
  return RT_OK;
}

rt_status rt_set_mlp_precision(rt_ctx* c, int precision) {
  if (!c) return RT_EINVAL;
  if (precision != RT_MLP_FP32 && precision != RT_MLP_BF16 && precision != RT_MLP_TF32X3)
    return fail(c, RT_EINVAL, "unknown MLP precision");
  c->mlp_precision = precision;
  return RT_OK;
}

rt_status rt_predict_mlp(rt_ctx* c, const uint16_t* d_feat, uint32_t n, float* d_u, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!c->d_mlp) return fail(c, RT_EINVAL, "no MLP model (rt_set_mlp)");
  if (!n) return RT_OK;
  if (!d_feat || !d_u) return fail(c, RT_EINVAL, "null argument");
  if (reinterpret_cast<uintptr_t>(d_feat) & 15u) return fail(c, RT_EINVAL, "d_feat must be 16-byte aligned");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaError_t e;
  const char* what;
  if (c->mlp_precision == RT_MLP_BF16) {
    e = rtlm::launch_mlp(d_feat, n, c->d_mlp, d_u, persistent_ctas(c), cs(stream));
    what = "k_mlp";
  } else if (c->mlp_precision == RT_MLP_TF32X3) {
    e = rtlm::launch_mlp_tf32(d_feat, n, c->d_mlptf, d_u, persistent_ctas(c), cs(stream));
    what = "k_mlp_tf32";
  } else {
    e = rtlm::launch_mlp_f32(d_feat, n, c->d_mlp32, d_u, persistent_ctas(c), cs(stream));
    what = "k_mlp_f32";
  }
  if (e != cudaSuccess) return cuda_fail(c, e, what);
  return RT_OK;
}

rt_status rt_fit_rule(rt_ctx* c, const uint16_t* d_feat, const float* d_target, uint32_t n, double* d_out,
                      rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (n < 7) return fail(c, RT_EINVAL, "fit needs >= 7 records (S:183)");
  if (!d_feat || !d_target || !d_out) return fail(c, RT_EINVAL, "null argument");
  if (reinterpret_cast<uintptr_t>(d_feat) & 15u) return fail(c, RT_EINVAL, "d_feat must be 16-byte aligned");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  rt_status st = ensure_ws(c, rtlm::fit_workspace(), cs(stream));
  if (st != RT_OK) return st;
  cudaError_t e = rtlm::launch_fit(d_feat, d_target, n, static_cast<double*>(c->ws), d_out, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_fit");
  return RT_OK;
}

rt_status rt_quantile(rt_ctx* c, const float* d_u, uint32_t n, double k, float* d_out, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!n) return fail(c, RT_EINVAL, "EmptyScores (S:212)");
  if (!(k > 0.0 && k <= 1.0)) return fail(c, RT_EINVAL, "k must be in (0, 1]");
  if (!d_u || !d_out) return fail(c, RT_EINVAL, "null argument");
  // nearest rank ceil(k n) - 1, with k n computed in fp64 as the oracle does
  double kn = std::ceil(k * (double)n);
  uint32_t r = kn < 1.0 ? 0u : (uint32_t)kn - 1u;
  if (r >= n) r = n - 1;
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  rt_status st = ensure_ws(c, rtlm::quantile_workspace(n), cs(stream));
  if (st != RT_OK) return st;
  cudaError_t e = rtlm::launch_quantile(d_u, n, r, c->ws, d_out, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_quantile");
  return RT_OK;
}

rt_status rt_key(rt_ctx* c, const float* d_u, const uint16_t* d_feat, const int64_t* d_arr, const uint32_t* d_D_in,
                 uint32_t n, const rt_profile* prof, uint64_t* d_key, uint32_t* d_D_out, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!n) return RT_OK;
  if (!d_u || !d_key) return fail(c, RT_EINVAL, "u / key are NULL");
  if (!d_feat && !d_D_in) return fail(c, RT_EINVAL, "need d_feat (ntok) or d_D_in");
  rt_status st = check_profile(c, prof, false);
  if (st != RT_OK) return st;
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaError_t e = rtlm::launch_key(d_u, d_feat, d_arr, d_D_in, n, *prof, d_key, d_D_out, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_key");
  return RT_OK;
}

// Argument checks of a one-pass schedule (rt_schedule and the calls built on it),
// run before anything is enqueued (rtlm.h: argument checks launch nothing).
static rt_status check_schedule_args(rt_ctx* c, const uint32_t* h_seg_off, uint32_t nq, const rt_profile* prof,
                                     uint32_t cores) {
  if (!h_seg_off) return fail(c, RT_EINVAL, "h_seg_off is NULL");
  rt_status st = check_profile(c, prof, false);
  if (st != RT_OK) return st;
  if (cores > rtlm::kMaxCores) return fail(c, RT_EINVAL, "cores must be <= 32");
  if (prof->offload && cores == 0) return fail(c, RT_EINVAL, "offload needs cores >= 1 (CPU-class tasks need a core)");
  if (h_seg_off[0] != 0) return fail(c, RT_EINVAL, "h_seg_off[0] must be 0");
  for (uint32_t q = 0; q < nq; ++q)
    if (h_seg_off[q + 1] < h_seg_off[q]) return fail(c, RT_EINVAL, "h_seg_off must be non-decreasing");
  return RT_OK;
}

rt_status rt_schedule(rt_ctx* c, const uint64_t* d_key, const float* d_u, const uint32_t* h_seg_off, uint32_t nq,
                      const rt_profile* prof, uint32_t cores, uint32_t* d_perm, uint32_t* d_batch_of,
                      uint8_t* d_slot_of, uint8_t* d_core_of, uint32_t* d_seg_batch_off, rt_stream stream) {
  if (!c) return RT_EINVAL;
  rt_status st = check_schedule_args(c, h_seg_off, nq, prof, cores);
  if (st != RT_OK) return st;
  const uint32_t n = h_seg_off[nq];
  if (!d_seg_batch_off) return fail(c, RT_EINVAL, "d_seg_batch_off is NULL");
  if (n && (!d_key || !d_u || !d_perm || !d_batch_of || !d_slot_of || !d_core_of))
    return fail(c, RT_EINVAL, "null device buffer");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaStream_t s = cs(stream);
  // workspace: seg counts | big-queue sort + gather
  size_t big_ws = 0;
  for (uint32_t q = 0; q < nq; ++q) {
    const uint32_t m = h_seg_off[q + 1] - h_seg_off[q];
    if (m > rtlm::kSmallSeg) {
      size_t need = rtlm::big_queue_workspace(m, (uint32_t)prof->C);
      if (need > big_ws) big_ws = need;
    }
  }
  const size_t cnt_bytes = (((size_t)nq + 1) * 4 + 255) & ~size_t(255);
  st = ensure_ws(c, cnt_bytes + big_ws, s);
  if (st != RT_OK) return st;
  st = upload_offsets(c, h_seg_off, nq + 1, s);
  if (st != RT_OK) return st;
  rtlm::SchedLaunch a{};
  a.key = d_key;
  a.u = d_u;
  a.seg_off = c->d_off;
  a.nq = nq;
  a.prof = *prof;
  a.cores = cores;
  a.perm = d_perm;
  a.batch_of = d_batch_of;
  a.slot_of = d_slot_of;
  a.core_of = d_core_of;
  a.seg_count = static_cast<uint32_t*>(c->ws);
  a.seg_batch_off = d_seg_batch_off;
  a.num_sms = c->num_sms;
  char* big = static_cast<char*>(c->ws) + cnt_bytes;
  cudaError_t e = rtlm::launch_sched_small(a, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "k_sched_small");
  const int full64 = (prof->policy == RT_FIFO || prof->policy == RT_EDF) ? 1 : 0;
  for (uint32_t q = 0; q < nq; ++q) {
    const uint32_t lo = h_seg_off[q], hi = h_seg_off[q + 1];
    if (hi - lo <= rtlm::kSmallSeg) continue;
    e = rtlm::launch_big_queue(a, q, lo, hi, full64, big, s, c->aux, c->ev_fork, c->ev_join);
    if (e != cudaSuccess) return cuda_fail(c, e, "big queue schedule");
  }
  e = rtlm::launch_sched_finish(a, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "k_sched_finish");
  return RT_OK;
}

static rt_status upload_profiles(rt_ctx* c, const rt_profile* h_profiles, uint32_t np, cudaStream_t s) {
  if (np > c->prof_cap) {
    if (no_growth_in_capture(c, s) != RT_OK) return RT_EINVAL;
    retire(c, c->d_prof);
    c->d_prof = nullptr;
    c->prof_cap = 0;
    if (cudaMalloc(&c->d_prof, np * sizeof(rt_profile)) != cudaSuccess) return fail(c, RT_ENOMEM, "profiles");
    c->prof_cap = np;
  }
  return stage_copy(c, c->st_prof, c->d_prof, h_profiles, np * sizeof(rt_profile), s);
}

static rt_status check_trace_off(rt_ctx* c, const uint32_t* h_trace_off, uint32_t nt, uint32_t* longest) {
  if (h_trace_off[0] != 0) return fail(c, RT_EINVAL, "h_trace_off[0] must be 0");
  uint32_t lg = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    if (h_trace_off[t + 1] < h_trace_off[t]) return fail(c, RT_EINVAL, "h_trace_off must be non-decreasing");
    lg = std::max(lg, h_trace_off[t + 1] - h_trace_off[t]);
  }
  if (lg > rtlm::kMaxLongTrace) return fail(c, RT_EINVAL, "trace longer than 65536");
  *longest = lg;
  return RT_OK;
}

rt_status rt_simulate(rt_ctx* c, const int64_t* d_arr, const uint16_t* d_len, const float* d_u,
                      const uint64_t* d_key, const uint32_t* d_D, const uint32_t* h_trace_off, uint32_t nt,
                      const rt_profile* h_profiles, uint32_t np, const uint16_t* d_trace_prof,
                      rt_trace_stats* d_stats, int64_t* d_end_us, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!nt) return RT_OK;
  if (!h_trace_off || !h_profiles || !np || !d_stats) return fail(c, RT_EINVAL, "null argument");
  if (!d_trace_prof && np < 1) return fail(c, RT_EINVAL, "no profile");
  for (uint32_t k = 0; k < np; ++k) {
    rt_status st = check_profile(c, &h_profiles[k], true);
    if (st != RT_OK) return st;
  }
  if (h_trace_off[0] != 0) return fail(c, RT_EINVAL, "h_trace_off[0] must be 0");
  uint32_t longest = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    if (h_trace_off[t + 1] < h_trace_off[t]) return fail(c, RT_EINVAL, "h_trace_off must be non-decreasing");
    longest = std::max(longest, h_trace_off[t + 1] - h_trace_off[t]);
  }
  if (longest > rtlm::kMaxLongTrace) return fail(c, RT_EINVAL, "trace longer than 65536");
  if (h_trace_off[nt] && (!d_arr || !d_len || !d_u || !d_key || !d_D)) return fail(c, RT_EINVAL, "null task array");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaStream_t s = cs(stream);
  rt_status st = upload_offsets(c, h_trace_off, nt + 1, s);
  if (st != RT_OK) return st;
  st = upload_profiles(c, h_profiles, np, s);
  if (st != RT_OK) return st;
  rtlm::ReplayLaunch a{};
  a.arrival = d_arr;
  a.len = d_len;
  a.u = d_u;
  a.key = d_key;
  a.D = d_D;
  a.trace_off = c->d_off;
  a.nt = nt;
  a.profiles = c->d_prof;
  a.trace_prof = d_trace_prof;
  a.stats = d_stats;
  a.end_us = d_end_us;
  // workspace: per-trace rank order of short traces (u16) | long traces: rank order
  // and its inverse over all tasks (u32) and the radix sort's buffers
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t total = h_trace_off[nt];
  const size_t sidx_bytes = up((size_t)nt * rtlm::kMaxTrace * sizeof(uint16_t));
  size_t long_bytes = 0;
  if (longest > rtlm::kMaxTrace) long_bytes = 2 * up(total * 4) + rtlm::radix_sort_workspace(longest);
  st = ensure_ws(c, sidx_bytes + long_bytes, s);
  if (st != RT_OK) return st;
  a.sidx = static_cast<uint16_t*>(c->ws);
  cudaError_t e = cudaSuccess;
  if (long_bytes) {
    char* lp = static_cast<char*>(c->ws) + sidx_bytes;
    uint32_t* perm = reinterpret_cast<uint32_t*>(lp);
    a.long_perm = perm;
    a.long_rank = reinterpret_cast<uint32_t*>(lp + up(total * 4));
    void* rws = lp + 2 * up(total * 4);
    for (uint32_t t = 0; t < nt; ++t) {  // stable sort by key desc of each long trace (R-TIE)
      const uint32_t lo = h_trace_off[t], m = h_trace_off[t + 1] - lo;
      if (m <= rtlm::kMaxTrace) continue;
      e = rtlm::radix_sort_desc(d_key + lo, lo, m, perm + lo, 1, rws, s);
      if (e != cudaSuccess) return cuda_fail(c, e, "long-trace rank sort");
    }
  }
  uint32_t max_window = 1;
  for (uint32_t k = 0; k < np; ++k) {
    const uint32_t C = (uint32_t)h_profiles[k].C, m = (uint32_t)h_profiles[k].b10 * C / 10u;
    max_window = std::max(max_window, h_profiles[k].consolidate ? std::max(m, C) : C);
  }
  e = rtlm::launch_replay(a, max_window, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "k_replay");
  return RT_OK;
}

rt_status rt_schedule_deadlines(rt_ctx* c, const float* d_u, const uint32_t* d_D_us, const int64_t* d_arrival_us,
                                const uint32_t* h_seg_off, uint32_t nq, const rt_profile* prof, uint32_t cores,
                                uint32_t* d_perm, uint32_t* d_batch_of, uint8_t* d_slot_of, uint8_t* d_core_of,
                                uint32_t* d_seg_batch_off, rt_stream stream) {
  if (!c) return RT_EINVAL;
  rt_status st0 = check_schedule_args(c, h_seg_off, nq, prof, cores);
  if (st0 != RT_OK) return st0;
  const uint32_t n = h_seg_off[nq];
  if (n && (!d_u || !d_D_us)) return fail(c, RT_EINVAL, "u / deadlines are NULL");
  if (n && (!d_perm || !d_batch_of || !d_slot_of || !d_core_of)) return fail(c, RT_EINVAL, "null device buffer");
  if (!d_seg_batch_off) return fail(c, RT_EINVAL, "d_seg_batch_off is NULL");
  if (n > c->kbuf_n) {
    if (no_growth_in_capture(c, cs(stream)) != RT_OK) return RT_EINVAL;
    DeviceGuard g(c->device);
    retire(c, c->kbuf);
    c->kbuf = nullptr;
    c->kbuf_n = 0;
    if (cudaMalloc(&c->kbuf, (size_t)n * sizeof(uint64_t)) != cudaSuccess) return fail(c, RT_ENOMEM, "key buffer");
    c->kbuf_n = n;
  }
  rt_status st = rt_key(c, d_u, nullptr, d_arrival_us, d_D_us, n, prof, c->kbuf, nullptr, stream);
  if (st != RT_OK) return st;
  return rt_schedule(c, c->kbuf, d_u, h_seg_off, nq, prof, cores, d_perm, d_batch_of, d_slot_of, d_core_of,
                     d_seg_batch_off, stream);
}

rt_status rt_score_schedule_host(rt_ctx* c, const uint8_t* h_bytes, const uint32_t* h_offsets, uint32_t n,
                                 const rt_regressor* reg, const rt_profile* prof, uint32_t cores,
                                 uint32_t* h_batch_of, uint8_t* h_slot_of, uint8_t* h_core_of, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!n) return RT_OK;
  if (!h_bytes || !h_offsets || !reg || !prof || !h_batch_of || !h_slot_of || !h_core_of)
    return fail(c, RT_EINVAL, "null argument");
  {
    const uint32_t seg0[2] = {0u, n};
    rt_status st0 = check_schedule_args(c, seg0, 1, prof, cores);
    if (st0 != RT_OK) return st0;
  }
  if ((uint64_t)h_offsets[n] >= (1ull << 32) - 1) return fail(c, RT_EOVERFLOW, "text too large");
  const size_t nbytes = h_offsets[n];
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t need = up(nbytes) + up(4 * ((size_t)n + 1)) + up(4 * (size_t)n) + up(8 * (size_t)n) +
                      3 * up(4 * (size_t)n) + 2 * up(n) + up(8);
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  if (need > c->io_size) {
    if (no_growth_in_capture(c, cs(stream)) != RT_OK) return RT_EINVAL;
    retire(c, c->io);  // cudaFree: implicit device sync, no in-flight user
    c->io = nullptr;
    c->io_size = 0;
    cudaError_t e = cudaMalloc(&c->io, need);
    if (e != cudaSuccess) return fail(c, RT_ENOMEM, std::string("io buffers: ") + cudaGetErrorString(e));
    c->io_size = need;
  }
  char* p = static_cast<char*>(c->io);
  auto take = [&](size_t b) { char* r = p; p += up(b); return r; };
  uint8_t* d_bytes = reinterpret_cast<uint8_t*>(take(nbytes));
  uint32_t* d_off = reinterpret_cast<uint32_t*>(take(4 * ((size_t)n + 1)));
  float* d_u = reinterpret_cast<float*>(take(4 * (size_t)n));
  uint64_t* d_key = reinterpret_cast<uint64_t*>(take(8 * (size_t)n));
  uint32_t* d_perm = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
  uint32_t* d_batch = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
  uint32_t* d_sbo = reinterpret_cast<uint32_t*>(take(8));
  uint8_t* d_slot = reinterpret_cast<uint8_t*>(take(n));
  uint8_t* d_core = reinterpret_cast<uint8_t*>(take(n));
  cudaStream_t s = cs(stream);
  RT_CUDA(c, cudaMemcpyAsync(d_bytes, h_bytes, nbytes, cudaMemcpyHostToDevice, s));
  RT_CUDA(c, cudaMemcpyAsync(d_off, h_offsets, 4 * ((size_t)n + 1), cudaMemcpyHostToDevice, s));
  rt_status st = rt_score_key(c, d_bytes, d_off, n, reg, prof, nullptr, nullptr, nullptr, d_u, d_key, nullptr, stream);
  if (st != RT_OK) return st;
  const uint32_t seg[2] = {0u, n};
  st = rt_schedule(c, d_key, d_u, seg, 1, prof, cores, d_perm, d_batch, d_slot, d_core, d_sbo, stream);
  if (st != RT_OK) return st;
  RT_CUDA(c, cudaMemcpyAsync(h_batch_of, d_batch, 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
  RT_CUDA(c, cudaMemcpyAsync(h_slot_of, d_slot, n, cudaMemcpyDeviceToHost, s));
  RT_CUDA(c, cudaMemcpyAsync(h_core_of, d_core, n, cudaMemcpyDeviceToHost, s));
  return RT_OK;
}

rt_status rt_reduce_stats(rt_ctx* c, const rt_trace_stats* d_stats, uint32_t nt, const uint16_t* d_group_of,
                          uint32_t ngroups, int64_t* d_sums, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!nt) return RT_OK;
  if (!d_stats || !d_sums || !ngroups) return fail(c, RT_EINVAL, "null argument");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaError_t e = rtlm::launch_reduce_stats(d_stats, nt, d_group_of, ngroups, d_sums, cs(stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "k_reduce_stats");
  return RT_OK;
}

rt_status rt_trace_report(rt_ctx* c, const int64_t* d_arrival_us, const int64_t* d_end_us,
                          const uint32_t* h_trace_off, uint32_t nt, rt_trace_summary* d_report, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!nt) return RT_OK;
  if (!d_arrival_us || !d_end_us || !h_trace_off || !d_report) return fail(c, RT_EINVAL, "null argument");
  uint32_t longest = 0;
  rt_status st = check_trace_off(c, h_trace_off, nt, &longest);
  if (st != RT_OK) return st;
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaStream_t s = cs(stream);
  st = upload_offsets(c, h_trace_off, nt + 1, s);
  if (st != RT_OK) return st;
  cudaError_t e = rtlm::launch_trace_report(d_arrival_us, d_end_us, c->d_off, nt, d_report, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "k_trace_report");
  if (longest > rtlm::kMaxTrace) {  // long traces: key sort + one-CTA pick each
    st = ensure_ws(c, rtlm::trace_long_workspace(longest), s);
    if (st != RT_OK) return st;
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t lo = h_trace_off[t], m = h_trace_off[t + 1] - lo;
      if (m <= rtlm::kMaxTrace) continue;
      e = rtlm::launch_trace_long(d_arrival_us, d_end_us, nullptr, nullptr, lo, m, nullptr, nullptr, t,
                                  d_report + t, nullptr, c->ws, s);
      if (e != cudaSuccess) return cuda_fail(c, e, "long-trace report");
    }
  }
  return RT_OK;
}

rt_status rt_trace_utilization(rt_ctx* c, const uint16_t* d_len, const uint64_t* d_key, const int64_t* d_end_us,
                               const uint32_t* h_trace_off, uint32_t nt, const rt_profile* h_profiles, uint32_t np,
                               const uint16_t* d_trace_prof, rt_trace_util* d_util, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (!nt) return RT_OK;
  if (!h_trace_off || !h_profiles || !np || !d_util) return fail(c, RT_EINVAL, "null argument");
  for (uint32_t k = 0; k < np; ++k) {
    rt_status st = check_profile(c, &h_profiles[k], true);
    if (st != RT_OK) return st;
  }
  uint32_t longest = 0;
  rt_status st = check_trace_off(c, h_trace_off, nt, &longest);
  if (st != RT_OK) return st;
  if (h_trace_off[nt] && (!d_len || !d_key || !d_end_us)) return fail(c, RT_EINVAL, "null task array");
  DeviceGuard g(c->device);
  if (capturing(cs(stream))) c->captured = true;  // see retire()
  cudaStream_t s = cs(stream);
  st = upload_offsets(c, h_trace_off, nt + 1, s);
  if (st != RT_OK) return st;
  st = upload_profiles(c, h_profiles, np, s);
  if (st != RT_OK) return st;
  cudaError_t e = rtlm::launch_trace_util(d_len, d_key, d_end_us, c->d_off, nt, c->d_prof, d_trace_prof, d_util, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "k_trace_util");
  if (longest > rtlm::kMaxTrace) {
    st = ensure_ws(c, rtlm::trace_long_workspace(longest), s);
    if (st != RT_OK) return st;
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t lo = h_trace_off[t], m = h_trace_off[t + 1] - lo;
      if (m <= rtlm::kMaxTrace) continue;
      // arrival is not needed for the utilization keys: pass end_us in its place
      e = rtlm::launch_trace_long(d_end_us, d_end_us, d_len, d_key, lo, m, c->d_prof, d_trace_prof, t, nullptr,
                                  d_util + t, c->ws, s);
      if (e != cudaSuccess) return cuda_fail(c, e, "long-trace utilization");
    }
  }
  return RT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- NEXT-2: training (k_train.cu)
namespace {
uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// R-TRAIN: epoch e visits the requests in the order i -> (a * i + b) mod n
void epoch_perm(uint32_t n, uint64_t seed, uint32_t e, uint64_t& a, uint64_t& b) {
  const uint64_t h = splitmix64(seed + e);
  a = 1 + h % n;
  auto gcd = [](uint64_t x, uint64_t y) { while (y) { const uint64_t t = x % y; x = y; y = t; } return x; };
  while (gcd(a, n) != 1) ++a;
  a %= n;
  b = (h >> 32) % n;
}
}  // namespace

rt_status rt_get_mlp(rt_ctx* c, float* const w[5], float* const b[5]) {
  if (!c) return RT_EINVAL;
  if (c->mlp_host.empty()) return fail(c, RT_EINVAL, "no MLP model (rt_set_mlp)");
  size_t off = 0;
  for (int l = 0; l < 5; ++l) {
    const size_t nw = (size_t)kMlpDims[l + 1] * kMlpDims[l];
    if (!w[l] || !b[l]) return fail(c, RT_EINVAL, "null MLP weight or bias");
    std::memcpy(w[l], c->mlp_host.data() + off, nw * sizeof(float));
    off += nw;
    std::memcpy(b[l], c->mlp_host.data() + off, kMlpDims[l + 1] * sizeof(float));
    off += kMlpDims[l + 1];
  }
  return RT_OK;
}

rt_status rt_train_mlp(rt_ctx* c, const uint16_t* d_feat, const float* d_y, uint32_t n, uint32_t epochs,
                       uint32_t batch, float lr, uint64_t seed, double* h_losses, rt_stream stream) {
  if (!c) return RT_EINVAL;
  if (c->mlp_host.empty()) return fail(c, RT_EINVAL, "no MLP model to start from (rt_set_mlp)");
  if (!epochs) return RT_OK;
  if (!n || !d_feat || !d_y || !h_losses) return fail(c, RT_EINVAL, "null argument or n == 0");
  if (batch == 0 || batch > 65536) return fail(c, RT_EINVAL, "batch must be in [1, 65536]");
  if (!(lr > 0.0f) || !std::isfinite(lr)) return fail(c, RT_EINVAL, "lr must be positive and finite");
  DeviceGuard g(c->device);
  cudaStream_t s = cs(stream);
  if (capturing(s)) return fail(c, RT_EINVAL, "rt_train_mlp cannot be captured into a CUDA graph");
  const uint32_t bmax = std::min(batch, n);
  const size_t np = c->mlp_host.size();
  size_t lofs[5], off = 0;  // offset of W_l in the flat parameter array (b_l follows)
  for (int l = 0; l < 5; ++l) {
    lofs[l] = off;
    off += (size_t)kMlpDims[l + 1] * kMlpDims[l] + kMlpDims[l + 1];
  }
  size_t act_ofs[6], acts = 0;  // activations of one batch: x, h1..h4, z
  for (int l = 0; l < 6; ++l) {
    act_ofs[l] = acts;
    acts += (size_t)bmax * kMlpDims[l];
  }
  const size_t nbytes = (4 * np + acts + 2 * (size_t)bmax * 200 + bmax) * sizeof(float) + epochs * sizeof(double);
  void* mem = nullptr;
  if (cudaMalloc(&mem, nbytes) != cudaSuccess) return fail(c, RT_ENOMEM, "training buffers");
  struct Free { void* p; ~Free() { cudaFree(p); } } fr{mem};
  float* P = reinterpret_cast<float*>(mem);
  float* G = P + np;
  float* Mo = G + np;
  float* Vo = Mo + np;
  float* act = Vo + np;
  float* D0 = act + acts;
  float* D1 = D0 + (size_t)bmax * 200;
  float* yb = D1 + (size_t)bmax * 200;
  double* esq = reinterpret_cast<double*>(yb + bmax);
  RT_CUDA(c, cudaMemcpyAsync(P, c->mlp_host.data(), np * sizeof(float), cudaMemcpyHostToDevice, s));
  RT_CUDA(c, cudaMemsetAsync(Mo, 0, 2 * np * sizeof(float), s));
  RT_CUDA(c, cudaMemsetAsync(esq, 0, epochs * sizeof(double), s));
  uint64_t t = 0;
  for (uint32_t e = 0; e < epochs; ++e) {
    uint64_t pa, pb;
    epoch_perm(n, seed, e, pa, pb);
    for (uint32_t i0 = 0; i0 < n; i0 += bmax) {
      const uint32_t B = std::min(bmax, n - i0);
      RT_CUDA(c, rtlm::launch_gather(d_feat, d_y, n, pa, pb, i0, B, act + act_ofs[0], yb, s));
      // forward: h_{l+1} = relu(h_l W_l^T + b_l), raw output z (no clamp: R-TRAIN)
      for (int l = 0; l < 5; ++l) {
        const uint32_t in = kMlpDims[l], out = kMlpDims[l + 1];
        const float* W = P + lofs[l];
        RT_CUDA(c, rtlm::launch_gemm(act + act_ofs[l], in, 1, W, 1, in, W + (size_t)out * in, act + act_ofs[l + 1],
                                     out, B, out, in, l < 4 ? 1 : 0, s));
      }
      float* dZ = D0;
      RT_CUDA(c, rtlm::launch_loss(act + act_ofs[5], yb, B, dZ, esq + e, s));
      for (int l = 4; l >= 0; --l) {
        const uint32_t in = kMlpDims[l], out = kMlpDims[l + 1];
        float* gW = G + lofs[l];
        // gW[o][i] = sum_m dZ[m][o] h_l[m][i];  gb[o] = sum_m dZ[m][o]
        RT_CUDA(c, rtlm::launch_gemm(dZ, 1, out, act + act_ofs[l], in, 1, nullptr, gW, in, out, in, B, 0, s));
        RT_CUDA(c, rtlm::launch_colsum(dZ, B, out, gW + (size_t)out * in, s));
        if (l > 0) {  // dh_l[m][i] = sum_o dZ[m][o] W_l[o][i], then the ReLU derivative of h_l
          float* dA = dZ == D0 ? D1 : D0;
          RT_CUDA(c, rtlm::launch_gemm(dZ, out, 1, P + lofs[l], in, 1, nullptr, dA, in, B, in, out, 0, s));
          RT_CUDA(c, rtlm::launch_relu_back(dA, act + act_ofs[l], (size_t)B * in, s));
          dZ = dA;
        }
      }
      ++t;
      const float c1 = (float)(1.0 / (1.0 - std::pow(0.9, (double)t)));
      const float c2 = (float)(1.0 / (1.0 - std::pow(0.999, (double)t)));
      RT_CUDA(c, rtlm::launch_adam(P, G, Mo, Vo, (uint32_t)np, lr, c1, c2, s));
    }
  }
  std::vector<float> trained(np);
  std::vector<double> sq(epochs);
  RT_CUDA(c, cudaMemcpyAsync(trained.data(), P, np * sizeof(float), cudaMemcpyDeviceToHost, s));
  RT_CUDA(c, cudaMemcpyAsync(sq.data(), esq, epochs * sizeof(double), cudaMemcpyDeviceToHost, s));
  RT_CUDA(c, cudaStreamSynchronize(s));
  for (uint32_t e = 0; e < epochs; ++e) h_losses[e] = sq[e] / n;
  rt_mlp m{};
  for (int l = 0; l < 5; ++l) {
    m.w[l] = trained.data() + lofs[l];
    m.b[l] = trained.data() + lofs[l] + (size_t)kMlpDims[l + 1] * kMlpDims[l];
  }
  return rt_set_mlp(c, &m);  // the packed inference blobs and the host copy follow the trained weights
}
