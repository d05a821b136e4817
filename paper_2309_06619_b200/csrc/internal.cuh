// internal.cuh — shared definitions of librtlm.so (product code only; the
// oracle in oracle/ shares nothing with this file).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rtlm.h"

namespace rtlm {

// ---------------------------------------------------------------- lexicon
// Device lexicon: open-addressing table of lemma keys (<= 16 bytes, zero
// padded, little-endian in two u64) -> packed attributes.
enum : uint32_t {
  A_VAGUE = 1u << 0,
  A_PREP = 1u << 1,
  A_COORD = 1u << 2,
  A_NOUN = 1u << 3,
  A_OPENER = 1u << 4,
  A_WHAT = 1u << 5,
  A_CAUSE = 1u << 6,
  A_BROAD = 1u << 7,
  A_MULTIPOS = 1u << 8,
};
constexpr int A_SEM_SHIFT = 9;    // bits 9..16: senses - 1 (0..254)
constexpr uint32_t A_SEM_MASK = 0xFFu;
constexpr int A_ID_SHIFT = 17;    // bits 17..31: entry id (noun id)
constexpr uint32_t kMaxLexEntries = 1024;

struct LexEntry {
  uint64_t k0, k1;
  uint32_t attr, len;
};

struct DevLexicon {
  const LexEntry* entries;  // n_entries (global; attributes)
  const uint4* keys;        // n_entries + 1: keys[0] = 0, keys[i] = zero-padded lemma of entry i - 1
  const uint32_t* slots;    // 1 << bits; 0 = empty, else entry index + 1 | fingerprint << 11 (lex_fp of the key);
                            // a key sits at one of its two slots
  uint32_t n_entries;
  uint32_t bits;
  uint32_t seed;
};

// Two-choice (cuckoo) hashing of a zero-padded <= 16-byte lemma (four
// little-endian words): a lemma sits at slot lex_slot1 or lex_slot2 (bits >= 6).
__host__ __device__ __forceinline__ uint32_t lex_mix(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                                     uint32_t seed) {
  uint32_t x = (w0 * 0x9E3779B1u) ^ (w1 * 0x85EBCA77u) ^ (w2 * 0xC2B2AE3Du) ^ (w3 * 0x27D4EB2Fu) ^ seed;
  return x ^ (x >> 15);
}
__host__ __device__ __forceinline__ uint32_t lex_fp(uint32_t x) { return x >> 11; }
__host__ __device__ __forceinline__ uint32_t lex_slot1(uint32_t x, uint32_t bits) { return (x * 0x2C1B3C6Du) >> (32 - bits); }
__host__ __device__ __forceinline__ uint32_t lex_slot2(uint32_t x, uint32_t bits) { return (x * 0x297A2D39u) >> (32 - bits); }

// ---------------------------------------------------------------- keys
__host__ __device__ __forceinline__ uint32_t ord32_bits(uint32_t b) {
  if (b == 0x80000000u) b = 0;  // -0 -> +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

constexpr uint32_t kNoBatch = 0xFFFFFFFFu;
constexpr uint32_t kSmallSeg = 2048;     // queues up to this size are scheduled inside one CTA
constexpr uint32_t kMaxWindow = 128;     // m = b10*C/10 <= 128
constexpr uint32_t kMaxTrace = 1024;     // tasks per trace on the short replay path (and in rt_trace_report / _utilization)
constexpr uint32_t kMaxLongTrace = 65536; // tasks per replayed trace (rt_simulate)
constexpr uint32_t kMaxCores = 32;

// ---------------------------------------------------------------- launchers
// Every kernel launch of the library is counted (rt_launch_count).
void note_launch(unsigned k = 1);
struct ScoreLaunch {
  const uint8_t* bytes;
  const uint32_t* offsets;
  uint32_t n;
  DevLexicon lex;
  int fused;  // 0: feat only; 1: + u, key (and D, feat if non-null)
  rt_regressor reg;
  rt_profile prof;
  const int64_t* arrival;
  const uint32_t* D_in;
  uint16_t* feat;
  float* u;
  uint64_t* key;
  uint32_t* D_out;
  uint32_t* flags;
  uint32_t* work;  // device counter (scoring work queue), zeroed by the launcher
  uint16_t* tokbuf;  // per-warp token buffers (score_scratch_bytes(num_sms))
  int num_sms;
};
size_t score_scratch_bytes(int ctas);
cudaError_t launch_score(const ScoreLaunch& a, cudaStream_t s);
cudaError_t launch_predict(const uint16_t* feat, uint32_t n, const rt_regressor& reg, float* u, cudaStream_t s);
cudaError_t launch_key(const float* u, const uint16_t* feat, const int64_t* arrival, const uint32_t* D_in,
                       uint32_t n, const rt_profile& p, uint64_t* key, uint32_t* D_out, cudaStream_t s);

// Radix sort (stable, descending 64-bit keys) of one range; values = global
// element indices.  Workspace sized by radix_sort_workspace(n).
size_t radix_sort_workspace(uint32_t n);
cudaError_t radix_sort_desc(const uint64_t* keys_in, uint32_t base_index, uint32_t n, uint32_t* perm_out,
                            int full64, void* workspace, cudaStream_t s);
cudaError_t radix_sort_desc2(const uint64_t* keys_in, const uint32_t* vals_in, uint32_t base_index, uint32_t n,
                             const uint32_t* n_dev, uint32_t* perm_out, int full64, void* workspace, cudaStream_t s);
// stable split by class bit: CPU-class keys/indices (ck, cv), GPU-class (gk, gv); counts[0..1] on device
cudaError_t split_by_class(const uint64_t* key, uint32_t base, uint32_t n, uint32_t* bsum, uint32_t* counts,
                           uint64_t* ck, uint32_t* cv, uint64_t* gk, uint32_t* gv, cudaStream_t s);

struct SchedLaunch {
  const uint64_t* key;
  const float* u;
  const uint32_t* seg_off;   // device copy, nq + 1
  uint32_t nq;
  rt_profile prof;
  uint32_t cores;
  uint32_t* perm;
  uint32_t* batch_of;
  uint8_t* slot_of;
  uint8_t* core_of;
  uint32_t* seg_count;       // device, nq (local batch counts)
  uint32_t* seg_batch_off;   // device, nq + 1
  int num_sms;
};
// small queues (all segments with n <= kSmallSeg; others skipped)
cudaError_t launch_sched_small(const SchedLaunch& a, cudaStream_t s);
cudaError_t launch_sched_finish(const SchedLaunch& a, cudaStream_t s);
// CPU class of a large queue [lo, lo+n) (ncpu read from device memory)
size_t cpu_big_workspace(uint32_t n);
cudaError_t launch_cpu_big(const SchedLaunch& a, uint32_t lo, uint32_t n, const uint32_t* ncpu_dev, void* ws,
                           cudaStream_t s);
// GPU class of a large queue: parallel exact consolidation (k_ff.cu)
size_t ff_workspace(uint32_t n, uint32_t levels, uint32_t C);
uint32_t ff_levels(uint32_t n);
// one large queue: class split, CPU-class sort + list scheduling on `aux`,
// GPU-class sort + consolidation on `s` (joined before return)
size_t big_queue_workspace(uint32_t n, uint32_t C);
cudaError_t launch_big_queue(const SchedLaunch& a, uint32_t q, uint32_t lo, uint32_t hi, int full64, void* ws,
                             cudaStream_t s, cudaStream_t aux, cudaEvent_t ev_fork, cudaEvent_t ev_join);

struct ReplayLaunch {
  const int64_t* arrival;
  const uint16_t* len;
  const float* u;
  const uint64_t* key;
  const uint32_t* D;
  const uint32_t* trace_off;  // device, nt + 1
  uint32_t nt;
  const rt_profile* profiles; // device
  const uint16_t* trace_prof;
  rt_trace_stats* stats;
  int64_t* end_us;
  uint16_t* sidx;             // workspace: nt x kMaxTrace (rank -> arrival index)
  const uint32_t* long_perm;  // traces > kMaxTrace: rank -> global index at [lo, lo + n) (NULL: none)
  uint32_t* long_rank;        //                      arrival index -> rank (workspace)
};
cudaError_t launch_replay(const ReplayLaunch& a, uint32_t max_window, cudaStream_t s);  // max_window: max(m, C) over the profiles
cudaError_t launch_trace_util(const uint16_t* len, const uint64_t* key, const int64_t* end_us,
                              const uint32_t* d_trace_off, uint32_t nt, const rt_profile* d_prof,
                              const uint16_t* d_trace_prof, rt_trace_util* out, cudaStream_t s);
// traces longer than kMaxTrace (one call per trace, after the short-trace launch):
// exactly one of rep / util non-null
size_t trace_long_workspace(uint32_t n);
cudaError_t launch_trace_long(const int64_t* arrival, const int64_t* end_us, const uint16_t* len,
                              const uint64_t* key, uint32_t lo, uint32_t n, const rt_profile* d_prof,
                              const uint16_t* d_trace_prof, uint32_t t, rt_trace_summary* rep, rt_trace_util* util,
                              void* ws, cudaStream_t s);
cudaError_t launch_trace_report(const int64_t* arrival, const int64_t* end_us, const uint32_t* d_trace_off,
                                uint32_t nt, rt_trace_summary* out, cudaStream_t s);
// K8 (NEXT-2): offline profiling (k_offline.cu)
size_t fit_workspace();
cudaError_t launch_fit(const uint16_t* feat, const float* y, uint32_t n, double* ws, double* out, cudaStream_t s);
size_t quantile_workspace(uint32_t n);
cudaError_t launch_quantile(const float* u, uint32_t n, uint32_t r, void* ws, float* out, cudaStream_t s);
// K7 (NEXT-1): lightweight MLP on tcgen05 (k_mlp.cu)
size_t mlp_blob_bytes();
void mlp_pack(const float* const w[5], const float* const b[5], uint8_t* blob);
cudaError_t launch_mlp(const uint16_t* feat, uint32_t n, const uint8_t* blob, float* u, int num_sms, cudaStream_t s);
// K7 fp32 mode (k_mlp_f32.cu): CUDA-core binary32 FMA chains
size_t mlp_f32_blob_bytes();
void mlp_f32_pack(const float* const w[5], const float* const b[5], float* blob);
cudaError_t launch_mlp_f32(const uint16_t* feat, uint32_t n, const float* blob, float* u, int num_sms,
                           cudaStream_t s);
// K7 3xTF32 mode (k_mlp_tf32.cu): layers 2-4 as hi.hi + hi.lo + lo.hi tcgen05 kind::tf32 products
size_t mlp_tf32_blob_bytes();
void mlp_tf32_pack(const float* const w[5], const float* const b[5], uint8_t* blob);
cudaError_t launch_mlp_tf32(const uint16_t* feat, uint32_t n, const uint8_t* blob, float* u, int num_sms,
                            cudaStream_t s);
// NEXT-2 training (k_train.cu)
cudaError_t launch_gemm(const float* A, uint32_t sam, uint32_t sak, const float* B, uint32_t sbk, uint32_t sbn,
                        const float* bias, float* C, uint32_t ldc, uint32_t M, uint32_t N, uint32_t K, int relu,
                        cudaStream_t s);
cudaError_t launch_gather(const uint16_t* feat, const float* y, uint32_t n, uint64_t a, uint64_t b, uint32_t i0,
                          uint32_t bsz, float* x, float* yb, cudaStream_t s);
cudaError_t launch_loss(const float* z, const float* yb, uint32_t bsz, float* dz, double* epoch_sq, cudaStream_t s);
cudaError_t launch_colsum(const float* dZ, uint32_t M, uint32_t N, float* gb, cudaStream_t s);
cudaError_t launch_relu_back(float* dA, const float* Aprev, size_t cnt, cudaStream_t s);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, uint32_t cnt, float lr, float c1, float c2,
                        cudaStream_t s);
cudaError_t launch_reduce_stats(const rt_trace_stats* st, uint32_t nt, const uint16_t* group_of, uint32_t ngroups,
                                int64_t* sums, cudaStream_t s);

}  // namespace rtlm
