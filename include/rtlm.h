/*
 * rtlm.h — C ABI of the B200-native RT-LM hot path (arXiv 2309.06619).
 *
 * Every compute step runs in CUDA kernels for sm_100a inside librtlm.so; the
 * host side only validates arguments and launches.  There is no CPU fallback.
 *
 * Conventions (all calls):
 *  - d_* pointers are CALLER-OWNED device memory on the context's device; the
 *    caller keeps them alive until `stream` has executed the call.  h_* are
 *    host pointers read synchronously during the call.  Structs passed by
 *    pointer are copied by value at call time.
 *  - Every call is asynchronous on `stream` (NULL = legacy default stream)
 *    unless stated otherwise.  Argument checks are synchronous and launch
 *    nothing on error.
 *  - Return codes: RT_OK; RT_EINVAL (bad argument, message via rt_last_error);
 *    RT_ELEXICON (lexicon parse error); RT_ENOMEM (workspace allocation);
 *    RT_ECUDA (CUDA launch/runtime error, message carries the CUDA string);
 *    RT_EOVERFLOW (a size exceeds a 32-bit index).
 *  - Data conditions that are NOT errors: non-ASCII bytes are dropped and
 *    counted in feat[7]; counts saturate at 65535 (sticky flag
 *    RT_FLAG_SATURATED, read with rt_get_flags).
 *  - One context per device, used by one host thread at a time.  A context's
 *    workspace, work counter and fork stream are reused by every call, so calls
 *    on one context must be ordered (one stream, or events between streams);
 *    overlap independent batches with one context per stream.  Small host
 *    arguments (offsets, profiles) go through a pinned staging buffer, so a
 *    call returns without waiting for the stream (it waits only for the
 *    previous call's staging copy on the same context).  Kernels are
 *    pure functions of their inputs: same inputs -> same bits.
 *  - CUDA graphs: every call may be captured (relaxed capture mode) once the
 *    same call has run outside capture (so no context buffer has to grow
 *    during capture; growth under capture fails with RT_EINVAL).  Host
 *    arguments staged under capture get a pinned block of their own that the
 *    graph's copy node reads at every replay; buffers a graph may address are
 *    kept until rt_destroy even if a later call replaces them.  Replays of a
 *    context's graphs and its other calls must be ordered like ordinary calls.
 *
 * Citations: P:a-b = PAPER.md lines (v1 P:1-912, v2 P:913-1887); S:a-b =
 * SPEC.md lines; R-* = readings in DESIGN.md §2.
 */
#ifndef RTLM_H
#define RTLM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTLM_ABI_VERSION 1

typedef struct rt_ctx rt_ctx;
typedef struct CUstream_st* rt_stream; /* == cudaStream_t */

typedef enum {
  RT_OK = 0,
  RT_EINVAL = 1,
  RT_ELEXICON = 2,
  RT_ENOMEM = 3,
  RT_ECUDA = 4,
  RT_EOVERFLOW = 5
} rt_status;

/* Sticky context flags (rt_get_flags). */
#define RT_FLAG_SATURATED 0x1u   /* some feature count saturated at 65535 */
#define RT_FLAG_BAD_OFFSETS 0x2u /* offsets were not non-decreasing; affected requests scored as empty */

/* Policies (A12-A14): priority key of Eq. 3 (UP/EUDF), Eq. 2
 * (slack) and the baselines FIFO / EDF=HPF / LUF / MUF
 * (S:301). */
enum { RT_FIFO = 0, RT_EDF = 1, RT_LUF = 2, RT_MUF = 3, RT_SLACK = 4, RT_UP = 5 };

/* Weighted-rule regression m_theta (Eq. 1):
 * u = max(0, fma(w6,f6, ... fma(w0,f0, c))) over f = {S,Y,M,V,O,P,ntok}
 * in binary32, index order (R-FP). */
typedef struct {
  float c;
  float w[7];
} rt_regressor;

/* One LM profile (paper constants P:619-625). */
typedef struct {
  int64_t eta_us;   /* eta_f: latency per output token, µs */
  int64_t mu_us;    /* mu_f / phi_f: deadline per input token, µs */
  int64_t base_us;  /* GPU base latency per batch (R-LAT) */
  int64_t setup_us; /* GPU batch setup (R-LAT) */
  int64_t xi_us;    /* wait interval xi (R-XI) */
  float lambda;     /* max uncertainty ratio inside a batch, >= 1 */
  float alpha;      /* uncertainty weight of Eq. 3 */
  float tau;        /* offload threshold: CPU iff u > tau (Alg. 1; Eq. 4) */
  float u_max;      /* normaliser of alpha*u (R-NUM), > 0 */
  int32_t C;        /* batch size C_f, 1..128 */
  int32_t b10;      /* b in tenths (R-B): window m = b10*C/10, 10..; m <= 128 */
  int32_t tightness;/* 1 tight, 2 loose */
  int32_t gamma;    /* CPU slowdown (R-LAT) */
  int32_t cores;    /* CPU cores, 0..32 (>= 1 when offload is on) */
  int32_t policy;   /* RT_FIFO .. RT_UP */
  int32_t consolidate; /* 1: dynamic consolidation (§IV-C); 0: fixed batch size C */
  int32_t offload;  /* 1: strategic offloading (§IV-D) */
  int32_t raw_numerator; /* 1: alpha*u uses raw u (R-NUM) */
  int32_t reserved; /* must be 0 */
} rt_profile;

typedef struct {
  int64_t max_resp_us; /* max over tasks of end - arrival */
  int64_t p95_resp_us; /* nearest-rank 95th percentile of end - arrival */
  int64_t makespan_us; /* last end - first arrival */
  uint32_t n;          /* completed tasks (all of the trace: no horizon) */
  uint32_t reserved;
} rt_trace_summary;

typedef struct {
  int64_t gpu_busy_us;  /* sum over GPU batches of setup + base + eta*max len */
  int64_t cpu_busy_us;  /* sum over CPU tasks of gamma*(base + eta*len), all cores */
  uint32_t gpu_batches; /* GPU batches dispatched */
  uint32_t cpu_tasks;   /* tasks run on the CPU cores */
} rt_trace_util;

typedef struct {
  int64_t sum_resp_us; /* sum over tasks of end - arrival */
  uint32_t n;          /* tasks in the trace */
  uint32_t misses;     /* tasks with end > arrival + D */
} rt_trace_stats;

/* ---------------------------------------------------------------- context */

/* Creates a context on `device` and uploads the lexicon (SPEC S:147 format,
 * R-LEX: sections vague/polysemy/pos/wh/coord/prep; entries are single word
 * tokens lemmatized at load; <= 1024 distinct lemmas of <= 16 bytes).
 * Returns RT_ELEXICON on a parse error (message via rt_last_error(*out) --
 * *out is still created so the message can be read; destroy it).
 * Device memory owned by the context: the lexicon tables, and the scoring
 * scratch of rt_score / rt_score_key (one token buffer of 16 448 u16 tokens +
 * 256 count records of 16 B per persistent warp: 32 warps x SM count x 37 KB,
 * ~175 MB on 148 SMs), allocated here so that scoring never allocates. */
rt_status rt_create(int device, const char* lexicon_text, size_t len, rt_ctx** out);
rt_status rt_destroy(rt_ctx* ctx);
/* Message of the last non-OK status on this context, or, with ctx == NULL,
 * of the calling thread's last non-OK status on any context (thread-local;
 * e.g. after rt_create failed before a context existed).  Never NULL. */
const char* rt_last_error(const rt_ctx* ctx);
/* Reads and clears the sticky flags (synchronises the device). */
rt_status rt_get_flags(rt_ctx* ctx, uint32_t* flags);
int rt_abi_version(void);
/* Total CUDA kernel launches issued by this library in this process (all contexts). */
uint64_t rt_launch_count(void);
/* Number of distinct lexicon lemmas. */
uint32_t rt_lexicon_size(const rt_ctx* ctx);
/* Caps the CTAs of this context's persistent kernels (scoring, MLP) at
 * max_ctas (0 = one per SM, the default).  Use it when several contexts run
 * concurrently: rt_schedule forks a one-CTA list-scheduling kernel that holds
 * an SM for ~1 ms per 2^20-request queue, and a persistent kernel with one CTA
 * per SM would wait for that SM before it can complete.  No effect on
 * results.  RT_EINVAL if ctx is NULL.
 * Pipelining batches over many streams (each context's rt_schedule also forks
 * onto one internal stream per context): CUDA maps streams onto
 * CUDA_DEVICE_MAX_CONNECTIONS hardware queues (default 8), and kernels of
 * streams that share a queue wait for each other in submission order; set it
 * to >= 2 x contexts + 1 (max 32) in the environment before the process
 * creates its CUDA context (bench.py uses 32: DESIGN.md section 9). */
rt_status rt_set_sm_limit(rt_ctx* ctx, uint32_t max_ctas);

/* ---------------------------------------------------------------- (1) score */

/* RuleGen(J) (Eq. 1; Table 1; Listing 1; R-TOK,
 * R-CLITIC, R-LEMMA, R-RULES).  Request i is bytes d_bytes[d_offsets[i] ..
 * d_offsets[i+1]).  d_offsets: n+1 non-decreasing u32; d_bytes holds
 * d_offsets[n] bytes (with offsets that decrease somewhere, RT_FLAG_BAD_OFFSETS
 * is set, requests with end < start score as empty and the others of their
 * 32-request group are clamped to [0, d_offsets[n])).  Output feat[i][0..7] =
 * {S, Y, M, V, O, P, ntok, ndropped} (u16, saturating; row = 16 bytes).
 * n == 0 is a no-op. */
rt_status rt_score(rt_ctx* ctx, const uint8_t* d_bytes, const uint32_t* d_offsets, uint32_t n, uint16_t* d_feat,
                   rt_stream stream);

/* ---------------------------------------------------------------- (2) predict */

/* u[i] = m_theta(feat[i]) (R-REG, R-FP).  d_feat as produced by rt_score. */
rt_status rt_predict(rt_ctx* ctx, const uint16_t* d_feat, uint32_t n, const rt_regressor* reg, float* d_u,
                     rt_stream stream);

/* ---------------------------------------------------------------- (2b) MLP (NEXT-1) */

/* The lightweight MLP m_theta of Eq. 1 (hidden sizes P:620 / P:1547;
 * SPEC S:160-165): layers 6-100-200-200-100-1, ReLU on hidden
 * layers, identity output, u = max(0, output).  Inputs are the six rule scores
 * feat[i][0..5] = {S, Y, M, V, O, P}.  Weights are HOST fp32, row-major
 * [out][in]: w[0] 100x6, w[1] 200x100, w[2] 200x200, w[3] 100x200, w[4] 1x100;
 * b[l] has `out` entries.  Three precisions (rt_set_mlp_precision):
 *   RT_MLP_FP32 (default): every multiply-add in binary32 on the CUDA cores,
 *     out[j] = fma chain over k in index order from b[j] (the paper's model is
 *     fp32); error vs the fp64 oracle within fp32 rounding;
 *   RT_MLP_BF16 (opt-in fast mode): layers 2-4 on the tensor cores (tcgen05,
 *     BF16 operands, FP32 accumulation), layers 1 and 5 in fp32;
 *     |u - u_fp64| <= 2^-5 x the oracle's |W|,|b|,|x| pass (DESIGN.md §7 K7);
 *   RT_MLP_TF32X3: layers 2-4 on the tensor cores with fp32 accuracy — every
 *     operand split x = hi + lo (two TF32 numbers, |x - hi - lo| <= 2^-22 |x|),
 *     products hi.hi + hi.lo + lo.hi accumulated in fp32 in TMEM; same error
 *     bound as RT_MLP_FP32 (1024 x 2^-24 x the |.| pass), not the same bits. */
typedef struct {
  const float* w[5];
  const float* b[5];
} rt_mlp;

/* Packs and uploads the weights into the context (synchronous; copies the
 * host arrays).  Replaces any previous model. */
rt_status rt_set_mlp(rt_ctx* ctx, const rt_mlp* mlp);
/* u[i] = m_theta(feat[i]) for i < n (d_feat as produced by rt_score).
 * RT_EINVAL if no model was set. n == 0 is a no-op. */
rt_status rt_predict_mlp(rt_ctx* ctx, const uint16_t* d_feat, uint32_t n, float* d_u, rt_stream stream);

/* NEXT-2, optional part of the offline profiling (Alg. 1: "Minimize
 * L_MSE <- ||m_theta(r_J) - l_J||^2"; "train the model with a learning
 * rate of 1e-4"; "for 100 epochs"): trains this
 * context's MLP from the weights of the last rt_set_mlp (or rt_train_mlp) by
 * mini-batch Adam (beta1 0.9, beta2 0.999, eps 1e-8) on mean((z - y)^2), z the
 * raw network output for the six rule scores of d_feat rows (u16 [n][8], as
 * rt_score writes them), y = d_y[n] (fp32 output lengths).  R-TRAIN: epoch e
 * visits rows (a_e * i + b_e) mod n, i = 0 .. n-1, in batches of `batch`
 * (the last one partial), with (a_e, b_e) from SplitMix64(seed + e) (a_e made
 * coprime with n), one Adam step per batch.  h_losses[e] (host, `epochs`
 * doubles) = the epoch's squared errors (forward passes before each step)
 * summed / n.  fp32 on the CUDA cores, every sum in a fixed order
 * (deterministic).  On return the context's MLP (all precisions) holds the
 * trained weights.  Allocates its buffers (not graph-capturable) and
 * synchronizes `stream`.  RT_EINVAL: no model set, n == 0, NULL pointers,
 * batch outside [1, 65536], lr not positive; epochs == 0 is a no-op. */
rt_status rt_train_mlp(rt_ctx* ctx, const uint16_t* d_feat, const float* d_y, uint32_t n, uint32_t epochs,
                       uint32_t batch, float lr, uint64_t seed, double* h_losses, rt_stream stream);
/* Copies the context's current MLP weights (fp32, layout of rt_mlp) into the
 * caller's arrays w[l] ([out][in]) and b[l] ([out]). */
rt_status rt_get_mlp(rt_ctx* ctx, float* const w[5], float* const b[5]);
#define RT_MLP_FP32 0
#define RT_MLP_BF16 1
#define RT_MLP_TF32X3 2
/* Selects the arithmetic of rt_predict_mlp for this context (RT_MLP_FP32,
 * RT_MLP_BF16 or RT_MLP_TF32X3; RT_EINVAL otherwise).  Takes effect for later calls. */
rt_status rt_set_mlp_precision(rt_ctx* ctx, int precision);

/* ---------------------------------------------------------------- (2c) offline profiling (NEXT-2) */

/* Weighted-rule fit ("learning a linear regression"):
 * target ~ c + sum_k w_k f_k over the six rule scores f = d_feat[i][0..5]
 * (u16 [n][8], 16-byte aligned) and fp32 targets d_target[n], by the normal
 * equations with ridge 1e-8 on the diagonal, fp64, solved by Cholesky.
 * d_out[8] (device fp64): (c, w_S, w_Y, w_M, w_V, w_O, w_P, cond) where cond =
 * (min/max Cholesky pivot)^2 (S:185 calls the fit degenerate below ~1e-12);
 * all NaN if the damped matrix is not positive definite.  Reproducible: fixed
 * reduction order.  RT_EINVAL if n < 7. */
rt_status rt_fit_rule(rt_ctx* ctx, const uint16_t* d_feat, const float* d_target, uint32_t n, double* d_out,
                      rt_stream stream);
/* Nearest-rank quantile (Eq. 4 tau = quantile_k) and
 * maximum (u_max) of d_u[n]: d_out[0] = sorted(u)[ceil(k n) - 1],
 * d_out[1] = max(u) (device fp32).  0 < k <= 1; RT_EINVAL if n == 0. */
rt_status rt_quantile(rt_ctx* ctx, const float* d_u, uint32_t n, double k, float* d_out, rt_stream stream);

/* ---------------------------------------------------------------- (3) key */

/* Deadline + priority key + class (R-D, R-NUM, R-OVERDUE, R-KEY; Eq. 2/3):
 *   D_us = d_D_in ? d_D_in[i] : min(tightness*mu_us*ntok_i, 2^32-1), ntok from d_feat[i][6];
 *   key  = cls<<63 | tier<<62 | ord(v),  cls = offload && u > tau.
 * d_arrival_us (int64 µs, may be NULL = 0) is used by FIFO/EDF only.
 * d_feat may be NULL iff d_D_in is given.  d_D_out may be NULL. */
rt_status rt_key(rt_ctx* ctx, const float* d_u, const uint16_t* d_feat, const int64_t* d_arrival_us,
                 const uint32_t* d_D_in, uint32_t n, const rt_profile* prof, uint64_t* d_key, uint32_t* d_D_out,
                 rt_stream stream);

/* Fused hot path (1)+(2)+(3) in one pass over the text: writes u and key,
 * D_us iff d_D_out != NULL, feat iff d_feat != NULL. */
rt_status rt_score_key(rt_ctx* ctx, const uint8_t* d_bytes, const uint32_t* d_offsets, uint32_t n,
                       const rt_regressor* reg, const rt_profile* prof, const int64_t* d_arrival_us,
                       const uint32_t* d_D_in, uint16_t* d_feat, float* d_u, uint64_t* d_key, uint32_t* d_D_out,
                       rt_stream stream);

/* ---------------------------------------------------------------- (4) schedule */

/* One-pass schedule (Alg. 1 online part P:467-481; §IV-C; flush
 * P:490-492; R-CONS, R-CARRY, R-FLUSH, R-CORE) of nq queues; queue q is
 * elements [h_seg_off[q], h_seg_off[q+1]) (HOST array, nq+1 entries).
 * Inputs: d_key (priority keys, e.g. from rt_score_key) and d_u.
 * `cores` overrides prof->cores for the CPU class (0..32; RT_EINVAL if 0 while
 * prof->offload is set: the CPU class would have no core).  Every argument
 * check runs before anything is enqueued.
 * Outputs (device, n = h_seg_off[nq]):
 *   d_perm[n]      priority order per queue (global indices), stable descending key;
 *   d_batch_of[n]  global GPU batch id (queues' batches are numbered
 *                  consecutively in queue order), UINT32_MAX for CPU tasks;
 *   d_slot_of[n]   position inside the batch (ascending u), 0 for CPU tasks;
 *   d_core_of[n]   CPU core for CPU tasks, 0xFF for GPU tasks;
 *   d_seg_batch_off[nq+1] first batch id of each queue (last = total). */
rt_status rt_schedule(rt_ctx* ctx, const uint64_t* d_key, const float* d_u, const uint32_t* h_seg_off, uint32_t nq,
                      const rt_profile* prof, uint32_t cores, uint32_t* d_perm, uint32_t* d_batch_of,
                      uint8_t* d_slot_of, uint8_t* d_core_of, uint32_t* d_seg_batch_off, rt_stream stream);

/* The north-star form rt_schedule(queue, deadlines, cores): the priority keys
 * are computed in-call from d_u and the caller's relative deadlines d_D_us
 * (the user deadline t_J of P:1286; as rt_key with d_D_in = d_D_us, Eq. 3
 * P:376-378 / Eq. 2 P:363-365 / baselines P:637-646; d_arrival_us, nullable,
 * for FIFO/EDF) into a buffer owned by the context, then the queues are
 * scheduled exactly as by rt_schedule (Alg. 1).  Same outputs and
 * errors as rt_schedule. */
rt_status rt_schedule_deadlines(rt_ctx* ctx, const float* d_u, const uint32_t* d_D_us, const int64_t* d_arrival_us,
                                const uint32_t* h_seg_off, uint32_t nq, const rt_profile* prof, uint32_t cores,
                                uint32_t* d_perm, uint32_t* d_batch_of, uint8_t* d_slot_of, uint8_t* d_core_of,
                                uint32_t* d_seg_batch_off, rt_stream stream);

/* ---------------------------------------------------------------- (5) simulate */

/* Discrete-event replay of nt traces (§V-A; R-REPLAY, R-LAT,
 * R-XI).  Trace t = tasks [h_trace_off[t], h_trace_off[t+1]) (HOST array),
 * at most 65536 tasks (RT_EINVAL beyond), in arrival order (d_arrival_us
 * non-decreasing within the trace).  Traces of <= 1024 tasks are replayed by
 * one warp each with register-word ready bitmaps; longer ones (e.g. the
 * paper's full 141-minute beta = 10..150 ramp, ~11 280 tasks)
 * are rank-sorted by a radix sort per trace and replayed by one warp each with
 * multi-word bitmaps (same events, same results).  Per task: arrival (int64 µs), true output length, u, key, D_us.
 * h_profiles[np] (host), d_trace_prof[nt] (u16 profile index; NULL = 0).
 * Output d_stats[nt]; d_end_us[n] (nullable) receives each task's end time. */
rt_status rt_simulate(rt_ctx* ctx, const int64_t* d_arrival_us, const uint16_t* d_true_len, const float* d_u,
                      const uint64_t* d_key, const uint32_t* d_D_us, const uint32_t* h_trace_off, uint32_t nt,
                      const rt_profile* h_profiles, uint32_t np, const uint16_t* d_trace_prof,
                      rt_trace_stats* d_stats, int64_t* d_end_us, rt_stream stream);

/* Richer replay statistics (NEXT-4; tables; SPEC
 * S:523-546) from per-task end times (rt_simulate's d_end_us): per trace t in
 * [0, nt) (tasks h_trace_off[t] .. h_trace_off[t+1], HOST offsets, <= 65536 per
 * trace; traces over 1024 tasks are sorted by a radix sort each), d_report[t] = {max response, nearest-rank p95 response, makespan,
 * n} (rt_trace_summary).  Throughput = n / makespan (completions per unit time). */
rt_status rt_trace_report(rt_ctx* ctx, const int64_t* d_arrival_us, const int64_t* d_end_us,
                          const uint32_t* h_trace_off, uint32_t nt, rt_trace_summary* d_report, rt_stream stream);

/* Executor utilization (NEXT-4, the simulated analogue
 * of the paper's "CPU / GPU util." table) from rt_simulate's per-task end
 * times: d_util[t] = {GPU busy µs, CPU busy µs (summed over cores), GPU
 * batches, CPU tasks} for trace t (same h_trace_off / h_profiles[np] /
 * d_trace_prof conventions as rt_simulate; the class is d_key >> 63).  GPU
 * batches are recovered as the GPU-class tasks sharing one end time, exact for
 * rt_simulate's serial GPU.  Fractions: gpu_busy / makespan and cpu_busy /
 * (cores * makespan), makespan from rt_trace_report.  RT_EINVAL on null
 * arguments, bad offsets or traces longer than 1024. */
rt_status rt_trace_utilization(rt_ctx* ctx, const uint16_t* d_true_len, const uint64_t* d_key,
                               const int64_t* d_end_us, const uint32_t* h_trace_off, uint32_t nt,
                               const rt_profile* h_profiles, uint32_t np, const uint16_t* d_trace_prof,
                               rt_trace_util* d_util, rt_stream stream);

/* ---------------------------------------------------------------- (4b) end to end from host */

/* The whole requests path of one queue from HOST buffers (the bench's e2e
 * leg; RuleGen + Eq. 1 + Eq. 3 + Alg. 1's online part, P:211-233, P:346-378,
 * P:467-481): copies h_bytes[0 .. h_offsets[n]) and h_offsets[n+1] to device buffers
 * owned by the context, runs rt_score_key (1)-(3) and rt_schedule (4) on the
 * queue [0, n), and copies the assignment back: h_batch_of[n] (global GPU
 * batch id, UINT32_MAX for CPU tasks), h_slot_of[n], h_core_of[n] (as in
 * rt_schedule).  All copies and kernels are asynchronous on `stream`: the
 * host inputs must stay unchanged and the outputs are valid only after the
 * stream has executed the call (page-locked host memory makes the copies
 * asynchronous; pageable memory makes them synchronous).  h_offsets[n] is read
 * by the host at call time (the byte count).  Same errors as rt_score_key /
 * rt_schedule; RT_ENOMEM if the context's buffers cannot grow (growing frees
 * the previous buffers, an implicit device synchronisation). */
rt_status rt_score_schedule_host(rt_ctx* ctx, const uint8_t* h_bytes, const uint32_t* h_offsets, uint32_t n,
                                 const rt_regressor* reg, const rt_profile* prof, uint32_t cores,
                                 uint32_t* h_batch_of, uint8_t* h_slot_of, uint8_t* h_core_of, rt_stream stream);

/* ---------------------------------------------------------------- (6) aggregate */

/* Integer sums per group (O8): d_sums[g*3 + {0,1,2}] += {sum_resp_us, n,
 * misses} over traces with d_group_of[t] == g (NULL = group 0).  d_sums is
 * ACCUMULATED into (zero it first); exact and order-independent, so the
 * per-rank results can be all-reduced with SUM. */
rt_status rt_reduce_stats(rt_ctx* ctx, const rt_trace_stats* d_stats, uint32_t nt, const uint16_t* d_group_of,
                          uint32_t ngroups, int64_t* d_sums, rt_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* RTLM_H */
