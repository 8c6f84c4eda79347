/*
 * sae.h — C ABI v1 of the SAECache hot path on B200 (sm_100a).
 *
 * The operation is the batched trace replay of the SAECache prefix-cache
 * eviction policy (arxiv 2605.18825, /root/reference/PAPER.md, cited "P:<line>"):
 *   (a) chained block hashing + strict prefix lookup
 *   (b) per-round scoring of every resident block, Eq.(1)-(3)
 *   (c) victim selection: Alg.1 Evict (EF first by num_tokens, then the global
 *       argmin of Eq.(3)), segmented per queue/class with a total-order tie-break
 *       on (P, last, id)
 *   (d) the online learners driven by eviction feedback
 * Readings of silent / conflicting passages: DESIGN.md "Readings".
 *
 * Conventions
 *  - Every call returns sae_status (0 = SAE_OK, < 0 = error).  Host-detectable
 *    errors (NULL pointers, ABI mismatch, capacity 0, bad sizes) return
 *    immediately.  Errors found on the device (arrival time going backwards,
 *    empty prompt, output overflow, replica not grouped) set a STICKY flag that
 *    the next synchronising call (sae_stats, sae_sync) returns, as CUDA does for
 *    asynchronous errors; sae_last_error() gives the text.
 *  - A ctx is single-threaded; one ctx per device per process.  It owns ALL
 *    device state (block SoA, hash tables, ghost rings, counters, parameters,
 *    scratch); it is allocated in sae_create.  Per-batch scratch grows with
 *    stream-ordered allocation when a larger batch arrives.
 *  - sae_batch / sae_admit_out pointers are DEVICE pointers owned by the caller;
 *    they must stay valid until the stream passes the call.  Calls are
 *    stream-ordered and asynchronous except sae_create, sae_destroy,
 *    sae_batch_blocks, sae_stats, sae_sync and the sae_get_* readers.
 *  - Numerics: fp64, every + - * / sqrt a single IEEE round-to-nearest op
 *    (no FMA contraction), our own ln/exp/erfc (fdlibm 5.3 algorithms); integer
 *    counters u64 with the 0.99 decay done as floor(99 x / 100).  Results are
 *    bit-identical to the CPU oracle (oracle/, test infrastructure only).
 */
#ifndef SAE_H_
#define SAE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAE_ABI_VERSION 3u

typedef struct sae_ctx sae_ctx;
typedef int sae_status;
typedef struct CUstream_st* sae_stream;  /* == cudaStream_t; NULL = legacy default stream */

enum {
  SAE_OK = 0,
  SAE_E_INVAL = -1,          /* bad argument / empty prompt (O1: L >= 1)            */
  SAE_E_CAPACITY_ZERO = -2,  /* capacity_blocks == 0                        */
  SAE_E_EMPTY = -3,          /* sae_evict ran out of evictable blocks       */
  SAE_E_NOT_RESIDENT = -4,   /* reserved                                           */
  SAE_E_TIME = -5,           /* arrival earlier than the replica's current time     */
  SAE_E_OVERFLOW = -6,       /* victim buffer too small / 2^32 block ids exhausted  */
  SAE_E_OOM = -7,
  SAE_E_CUDA = -8,
  SAE_E_ABI = -9,
  SAE_E_INTERNAL = -10       /* an exactness check still failed after a full rescan
                                (select); never expected -- raised, not hidden */
};

/* queues and token types */
enum { SAE_Q_EF = 0, SAE_Q_CHAT = 1, SAE_Q_AGENT = 2, SAE_Q_STRUCT = 3 };
enum { SAE_T_SYS = 0, SAE_T_USER = 1, SAE_T_TOOL = 2, SAE_T_RESP = 3, SAE_T_COT = 4, SAE_T_DECODE = 5 };

/* learner flags: which learners run at each firing (a disabled learner is skipped
 * entirely: no update, no counter decay, no reset) and which rule variant. */
enum {
  SAE_L_TOKENS = 1,          /* TokenWeights */
  SAE_L_QUEUES = 2,          /* QueueWeights */
  SAE_L_LOGNORMAL = 4,       /* LognormalParams */
  SAE_L_DECAY = 8,           /* decay power */
  SAE_L_TOKEN_MULT = 16,     /* multiplicative token rule (Alg. P:725) instead of P:703-707 */
  SAE_L_QUEUE_RELATIVE = 32, /* relative queue rule P:814-817 instead of Alg. P:583-593 */
  SAE_L_ADAPTIVE_BETA = 64   /* LognormalParams' EMA factor adapts (A28):
                                rho = mean (x - mu)^2 / sigma^2 over the ln-intervals x;
                                beta_ln doubled (at most 1) if rho > 1, else halved */
};

/* Eviction policy of a replica (sae_params.mode).  SAE_MODE_SAE is the paper's method; the
 * others are its baselines and its ablation variant, replayed by the
 * same kernels for side-by-side sweeps.  In the baselines every block sits in one queue
 * (CHAT) -- no EF stage, no structural queue -- and the victim is the argmin of:
 *   SAE_MODE_LRU  (last, id)                       least recently used
 *   SAE_MODE_LFU  (accesses, last, id)             least frequently used
 *   SAE_MODE_TWO  (w_tau / dt, last, id)           Token-Weight-Only: the learned token-type
 *                                                  weights without the multi-queue
 *                                                  architecture (decode blocks weigh as CoT)
 * Counters and learners run as configured.  Fixed-Param MQ and the learner ladder
 * are SAE_MODE_SAE with learn_flags / (mu, sigma) settings. */
enum { SAE_MODE_SAE = 0, SAE_MODE_LRU = 1, SAE_MODE_LFU = 2, SAE_MODE_TWO = 3 };

/* Learned values and meta-parameters, fp64.  Index order: w[sys,user,tool,resp,cot],
 * alpha[chat,agent,struct], mu/sigma[chat,agent].  beta_* weight the NEW value. */
typedef struct {
  double w[5], alpha[3], mu[2], sigma[2], gamma;
  double eta, a_miss, b_reuse, T, beta_q, beta_ln, beta_gamma;
  uint32_t learn_flags;
  uint32_t mode;              /* SAE_MODE_* */
} sae_params;

typedef struct {
  uint32_t abi_version;       /* must be SAE_ABI_VERSION */
  uint32_t block_tokens;      /* 16; 1..16 supported */
  uint32_t capacity_blocks;   /* C, per replica */
  uint32_t n_replicas;        /* R independent caches in this ctx */
  uint32_t ghost_capacity;    /* G, recently_evicted FIFO length (A30) */
  uint32_t K;                 /* learners fire when evictions reach a multiple of K (A14) */
  uint32_t interval_ring;     /* R_max ring of ln(dt) samples (A25), <= 4096 */
  uint32_t interval_keep;     /* 200 */
  uint32_t interval_min;      /* 20: update when > interval_min samples */
  uint32_t n_pos_bins;        /* 10 positional bins (A27), <= 16 */
  uint32_t ctas_per_replica;  /* 0 = auto (1 for small pools, the whole GPU for one huge pool) */
  uint32_t traj_capacity;     /* learner-trajectory snapshots kept per replica (0 = none) */
  uint64_t hash_seed;         /* H_{-1} of every chain (A1) */
  double dt_eps;              /* dt floor, 1e-3 s (A7) */
  double z_cut;               /* survival := 0 when z > z_cut (A36) */
  sae_params init;            /* initial parameters of every replica */
  int32_t device;
  uint32_t _pad;
} sae_config;

/* One batch of requests.  DEVICE pointers, caller-owned, read-only.
 * Requests of one replica must be contiguous and in arrival order; replicas may
 * appear in any order.  Request i's prompt tokens are tokens[prompt_off[i] ..
 * + prompt_len[i]) with per-token types types[...] (0 sys,1 user,2 tool,3 resp,
 * 4 cot); its decode span is tokens[decode_off[i] .. + decode_len[i]) (blocks of
 * type decode, chained after the last prompt block, A34).  flags: b0
 * is_multi_turn (predicted for turn 0), b1 is_agentic, b2 has conversation id.
 * shared_prefix_blocks[i] = number of leading template blocks (is_shared_prefix). */
typedef struct {
  uint32_t n;
  uint32_t _pad;
  uint64_t total_blocks;      /* sum_i ceil(prompt_len/B) + ceil(decode_len/B); see sae_batch_blocks */
  const uint32_t* replica;
  const double* arrival;
  const uint64_t* prompt_off;
  const uint32_t* prompt_len;
  const uint64_t* decode_off;
  const uint32_t* decode_len;
  const uint32_t* tokens;
  const uint8_t* types;
  const uint8_t* flags;
  const uint32_t* shared_prefix_blocks;
} sae_batch;

/* Outputs of sae_admit_batch.  DEVICE pointers, caller-allocated, written by the
 * library.  Per request i: hit_blocks = length h of the resident chained prefix,
 * miss_blocks = n_i - h, matched_tokens = tokens in prompt blocks j < h (A41),
 * n_victims = blocks evicted to admit it; its victim ids (admission counters, in
 * eviction order) are victim_ids[victim_off[i] .. + n_victims[i]).  victim_off[i]
 * is the request's first block index (so victim_cap >= total_blocks suffices).
 * block_hash / block_tau (optional, may be NULL) receive every block's chained
 * hash and type tau at block_off[i] + j (block_off = victim_off). */
typedef struct {
  uint32_t* hit_blocks;
  uint32_t* miss_blocks;
  uint32_t* matched_tokens;
  uint32_t* n_victims;
  uint64_t* victim_off;       /* [n+1] */
  uint32_t* victim_ids;
  uint64_t victim_cap;
  uint64_t* block_hash;       /* optional [total_blocks] */
  uint8_t* block_tau;         /* optional [total_blocks] */
} sae_admit_out;

typedef struct {
  uint64_t requests, blocks_looked_up, hit_blocks, hit_tokens, prompt_tokens;
  uint64_t evictions, evict_by_queue[4], evict_by_type[6], mae_by_type[6];
  uint64_t learner_firings, eviction_rounds, blocks_scored, blocks_scored_struct;
  uint64_t resident, resident_by_queue[4];
  uint64_t E, next_id, gseq;
  double now;
  uint64_t ts_ev[5], ts_mae[5], ts_hit[5], ts_acc[5];  /* token_stats */
  uint64_t qh[3], qe[3];                             /* queue_hits / queue_evictions */
  uint64_t pb_hit[16], pb_acc[16];                   /* positional bins */
  uint64_t iv_len[2];                                /* reuse_intervals sizes */
  uint64_t traj_count;
  /* select diagnostics: scan passes actually run (>= chunks; extra passes are threshold
   * fallbacks), candidates sorted, passes with > 512 candidates, fallbacks per segment */
  uint64_t select_passes, select_cands, select_big, select_fail_seg[10];
  /* device time (ns, globaltimer) spent by the replica leader per phase: probe+touch,
   * scan passes, narrowing, sort+check, apply, learn, insert+outputs, table rebuild, and for
   * multi-CTA groups: command post, leader's own partition, wait for the workers, worker 1's
   * scan time; [12] threshold carry (trim / grow) after the select; [13] candidate gather from
   * the group buffer (groups) or victim rank placement (private pools); [14] the select's radix
   * passes; [15] victim staging + ordering */
  uint64_t phase_ns[16];
  uint64_t select_narrow, select_raw;   /* narrowings (candidate sets > 4096) and raw candidates */
  sae_params params;
  uint64_t stage2_chunks;   /* victim chunks that reached Alg.1 Stage 2: EF could not cover them */
} sae_replica_stats;

/* Whole-ctx totals of the additive counters (every replica summed), u64, for the multi-GPU
 * int64 all-reduce of hit / eviction / miss-after-evict statistics. */
typedef struct {
  uint64_t requests, blocks_looked_up, hit_blocks, hit_tokens, prompt_tokens, evictions;
  uint64_t evict_by_queue[4], evict_by_type[6], mae_by_type[6];
  uint64_t learner_firings, eviction_rounds, blocks_scored, blocks_scored_struct;
} sae_counters;

/* Trajectory snapshot taken at each learner firing. */
typedef struct {
  uint64_t E, request;
  double w[5], alpha[3], mu[2], sigma[2], gamma;
} sae_traj;

/* Allocate a ctx with all device state on cfg->device: n_replicas independent caches of
 * capacity_blocks blocks each (the paper's block pool, "cache of capacity C";
 * S:19-30 CacheStore), with the learners' state initialised from cfg->init (P:910-912,
 * DESIGN.md A29).  cfg is a HOST pointer, read once.  *out receives the ctx (owned by the
 * caller until sae_destroy).  Errors: SAE_E_ABI on version mismatch, SAE_E_CAPACITY_ZERO if
 * capacity_blocks == 0, SAE_E_INVAL on other bad sizes or sigma <= 0, SAE_E_OOM /
 * SAE_E_CUDA on allocation failure.  On any error nothing is leaked, *out is untouched and
 * sae_last_error(NULL) gives the text. */
sae_status sae_create(const sae_config* cfg, sae_ctx** out);
/* Free every device allocation of the ctx (synchronises the device first). */
sae_status sae_destroy(sae_ctx* ctx);

/* Replace one replica's learned values and meta-parameters (Appendix C parameter sweep,
 * P:842-853; C5).  p is a HOST pointer, copied before the call returns (synchronous on s).
 * Every score reads the parameters from the replica state, so nothing cached needs a
 * refresh.  SAE_E_INVAL if replica >= n_replicas or a sigma <= 0. */
sae_status sae_set_params(sae_ctx* ctx, uint32_t replica, const sae_params* p, sae_stream s);
/* Copy every replica's parameters into dev_out[n_replicas] (device), stream-ordered, for
 * the multi-GPU all-gather of the learned token-type weights. */
sae_status sae_params_gather(sae_ctx* ctx, sae_params* dev_out, sae_stream s);
/* Replace every replica's parameters from dev_in[n_replicas] (device), stream-ordered. */
sae_status sae_params_scatter(sae_ctx* ctx, const sae_params* dev_in, sae_stream s);
/* mean_w sync over the ALL-GATHERED parameters of n_total replicas laid out
 * replica = point + n_points * seed: out[r] = all[r] with w replaced by the mean of w over
 * the replicas of r's point, summed in seed order (identical at any GPU count).  Device
 * pointers; n_total must be a multiple of n_points. */
sae_status sae_params_point_mean(const sae_params* all_dev, uint32_t n_total, uint32_t n_points,
                                 sae_params* out_dev, sae_stream s);

/* Synchronously compute batch->total_blocks = sum_i ceil(prompt_len/B) + ceil(decode_len/B)
 * (P:319 16-token blocks; A34 decode blocks) from the DEVICE length arrays of batch. */
sae_status sae_batch_blocks(sae_ctx* ctx, const sae_batch* batch, uint64_t* total_blocks, sae_stream s);

/* Replay a batch: for every request, steps a1..a7 -- chained hashing,
 * strict-prefix lookup + touch, Classify, Eq.(1)-(3)
 * scores, Alg.1 Evict, the learners every K evictions (P:540-545,
 * P:689-823) -- replicas in parallel, the requests of a replica in array order (S:56-64
 * insert_request).  batch and out hold DEVICE pointers (caller-owned, valid until the
 * stream passes the call).  batch->total_blocks must equal sum_i ceil(prompt_len/B) +
 * ceil(decode_len/B) (sae_batch_blocks): the device recomputes it and raises the sticky
 * SAE_E_INVAL (nothing written) if it is smaller.  A replica whose requests are not
 * contiguous raises SAE_E_INVAL and is skipped (its state is untouched).  Device errors
 * (SAE_E_TIME, SAE_E_INVAL for an empty prompt, SAE_E_OVERFLOW) stop that replica at the
 * failing request and are reported by the next sae_stats / sae_sync. */
sae_status sae_admit_batch(sae_ctx* ctx, const sae_batch* batch, sae_admit_out* out, sae_stream s);

/* sae_admit_batch with HOST buffers (the end-to-end call): every array of host_batch is a
 * HOST pointer (pinned for asynchronous copies); the request arrays are copied into
 * ctx-owned device staging, and the token/type arena range [tok_lo, tok_hi) of
 * host_batch->tokens / ->types into the caller's DEVICE arena tokens_dev / types_dev at the
 * same offsets (prompt_off / decode_off index that arena).  host_out holds HOST pointers:
 * per-request outputs [n], victim_off [n+1] and victim_ids [victim_cap >= total_blocks] are
 * copied back device->host on s (read them after synchronising s); block_hash / block_tau
 * may be NULL.  *h2d_bytes / *d2h_bytes (optional, host) receive the bytes copied each way.
 * Pipelining: the inputs are staged in one of two ctx-owned slots, alternately, and copied
 * on a ctx-owned copy stream, so a call's host->device copies overlap the replay of the
 * previous call (the replay on s waits for them; the device->host copies stay on s).  A call
 * blocks until the call two before it is complete: host buffers (inputs and outputs) passed
 * to a call must stay valid until the second-next call returns or s is synchronised, and the
 * arena range [tok_lo, tok_hi) must not be rewritten by the next call while this one may
 * still read it.  Errors as sae_admit_batch. */
sae_status sae_admit_batch_host(sae_ctx* ctx, const sae_batch* host_batch, uint64_t tok_lo,
                                uint64_t tok_hi, uint32_t* tokens_dev, uint8_t* types_dev,
                                sae_admit_out* host_out, uint64_t* h2d_bytes, uint64_t* d2h_bytes,
                                sae_stream s);

/* Read-only probe (S:56-64 prefix match without the insert; P:158 strict prefix):
 * hit_blocks[i] (device u32 [n]) = resident chained-prefix length of request i against the
 * CURRENT state of its replica.  No touch, no counters, no hint update.  batch as in
 * sae_admit_batch (device pointers; total_blocks checked on the device). */
sae_status sae_lookup(sae_ctx* ctx, const sae_batch* batch, uint32_t* hit_blocks, sae_stream s);

/* Alg.1 Evict() x k on one replica at time `now` (>= the replica's time;
 * advances it) with an empty pin set and full accounting: ghost push, ts.ev / qe /
 * E (A35) and the learners at every multiple of K (A14).
 * victim_ids (device, >= k) receive the ids, *n_out (device u32) the count.  If
 * fewer than k blocks are resident the sticky error SAE_E_EMPTY is raised. */
sae_status sae_evict(sae_ctx* ctx, uint32_t replica, uint32_t k, double now,
                     uint32_t* victim_ids, uint32_t* n_out, sae_stream s);

/* The fused score/select pass alone (K3): Alg.1 Evict's choice of the next m <= 96 victims of
 * one replica at time `now` (>= the replica's time) -- EF by (num_tokens, id), then the
 * smallest Eq.(3) priorities by (P, last, id) -- with an empty pin set,
 * computed `passes` >= 1 times back to back in one launch (a measurement of the pass).
 * READ-ONLY: nothing is evicted, no counter, parameter or clock changes; only the carried
 * per-segment candidacy thresholds (a performance hint) and the diagnostics
 * of sae_replica_stats (phase_ns, select_passes / cands / raw / narrow / big) are kept.  victim_ids
 * (device, >= m) receive the ids in eviction order -- exactly those sae_evict(m, now) would
 * remove if no learner fires in between -- and *n_out (device u32, may be NULL) their count
 * (min(m, resident)).  SAE_E_INVAL for a bad replica, m > 96 or passes == 0; SAE_E_TIME
 * (sticky) if now is earlier than the replica's time. */
sae_status sae_select(sae_ctx* ctx, uint32_t replica, uint32_t m, double now, uint32_t passes,
                      uint32_t* victim_ids, uint32_t* n_out, sae_stream s);

/* Run the learners now -- TokenWeights, QueueWeights, LognormalParams, DecayPower
 * with the replica's learn_flags -- on one replica or on all
 * (UINT32_MAX); E is unchanged; one trajectory snapshot is appended.  Stream-ordered. */
sae_status sae_update(sae_ctx* ctx, uint32_t replica, sae_stream s);

/* Synchronous: copy one replica's counters (token_stats P:720-730, queue counters P:581-593,
 * positional bins P:793, hit/eviction totals), parameters and diagnostics to host_out (HOST
 * pointer); returns and clears the sticky device error if one was raised. */
sae_status sae_stats(sae_ctx* ctx, uint32_t replica, sae_replica_stats* host_out, sae_stream s);
/* Stream-ordered: dev_out (DEVICE pointer to one sae_counters) = the sum over every replica
 * of this ctx of its additive counters (hit accounting A41, evictions by queue / type A35,
 * miss-after-evict by type P:535-538).  Exact (integer) in any order, so the per-GPU totals
 * can be all-reduced with NCCL (int64 SUM) into the job's totals. */
sae_status sae_counters_device(sae_ctx* ctx, sae_counters* dev_out, sae_stream s);
/* Synchronous: copy up to cap trajectory snapshots (one per learner firing: E, request,
 * w, alpha, mu, sigma, gamma) of a replica, oldest first, to host_out (HOST);
 * host_out == NULL only returns the count in *n_out. */
sae_status sae_get_traj(sae_ctx* ctx, uint32_t replica, sae_traj* host_out, uint64_t cap,
                        uint64_t* n_out, sae_stream s);
/* Synchronize the stream and return (and clear) the sticky device error. */
sae_status sae_sync(sae_ctx* ctx, sae_stream s);
/* Text of the last error of ctx; of the last failed sae_create when ctx is NULL. */
const char* sae_last_error(const sae_ctx* ctx);

/* Eq.(1)-(3) evaluated on the device with the same arithmetic, operation order
 * and fdlibm-algorithm ln/exp/erfc as the replay's select uses for a candidate:
 * out[i] = ((alpha[q-1] * w[tau]) * p) / dt with dt = max(dt_in[i], dt_eps) (A7), p = Eq.(1)
 * survival for q in {1 chat, 2 agent} (0 when z > z_cut, A36) or Eq.(2) for q = 3 struct from
 * (ob[i], omax[i]).  q = 0 (EF, not scored) gives NaN.  params: HOST pointer; q, tau, dt_in,
 * ob, omax, out: DEVICE arrays of n.  For property tests (class monotonicity) and parity of
 * the score function itself. */
sae_status sae_priority(const sae_params* params, double dt_eps, double z_cut, uint64_t n,
                        const uint8_t* q, const uint8_t* tau, const double* dt_in, const uint32_t* ob,
                        const uint32_t* omax, double* out, sae_stream s);

/* Characterisation pass (A42): an unbounded cache (C = infinity,
 * nothing evicted) over one trace in arrival order.  A block is reused if its chained hash
 * occurred in an earlier request, intra-session if an earlier occurrence was in the
 * same session, else inter-session.  Counters by token type tau (0..5):
 *   blocks / reused                      every block            (Table 1 "combined")
 *   later_blocks / later_intra           blocks of turn > 0     (Table 1 "intra-conv.")
 *   first_blocks / first_inter           blocks of turn 0       (Table 1 "inter-conv.")
 * pos_blocks / pos_reused by bin min(9, 10 j / np) over the prompt blocks of single-turn
 * sessions (positional reuse), and reuses_intra / reuses_inter (session locality). */
typedef struct {
  uint64_t blocks[6], reused[6];
  uint64_t later_blocks[6], later_intra[6];
  uint64_t first_blocks[6], first_inter[6];
  uint64_t pos_blocks[10], pos_reused[10];
  uint64_t reuses_intra, reuses_inter;
} sae_char_stats;

/* Run the characterisation pass on the device (K1 hashing + two insert-or-find tables) and
 * copy the counters to host_out (HOST).  batch: DEVICE arrays as for sae_admit_batch (the
 * replica array is not read); session, turn (u32 [n]) and single_turn (u8 [n], 1 = the
 * request's session has one turn) are DEVICE arrays.  The (hash, session) key is a 64-bit
 * mix of both (a collision is possible with probability ~ blocks^2 / 2^64).  Synchronous;
 * the ctx supplies block_tokens, hash_seed and scratch only -- its cache state is untouched. */
sae_status sae_characterize(sae_ctx* ctx, const sae_batch* batch, const uint32_t* session,
                            const uint32_t* turn, const uint8_t* single_turn,
                            sae_char_stats* host_out, sae_stream s);

/* Synthetic-trace token materialisation (input generator, not the method):
 * tokens[dst[p] + i] = SM(SM(seed ^ SM(stream[p])) ^ (start[p] + i)) mod 2^17 and
 * types[dst[p] + i] = type[p] for every piece p, i < len[p]. Device pointers. */
sae_status sae_gen_tokens(uint64_t seed, uint64_t n_pieces, const uint64_t* stream,
                          const uint64_t* start, const uint32_t* len, const uint64_t* dst,
                          const uint8_t* type, uint32_t* tokens, uint8_t* types, sae_stream s);

/* Counts of device kernels launched by this ctx so far (for bench accounting). */
uint64_t sae_launch_count(const sae_ctx* ctx);

/* How sae_create laid the replay out on the device (for reports and tests; no device work).
 * threads: per replay CTA (128 / 256 / 512); ctas_per_replica: group size GP; ctas_per_sm:
 * co-resident replay CTAs per SM (occupancy); coresident: ctas_per_sm x SMs; chunks: > 1 when
 * single-CTA replicas outnumber the co-resident CTAs and each replica's run is replayed as
 * that many consecutive tasks by a persistent grid (wave balancing); cand_global: 1 when the
 * candidate buffer lives in global memory instead of shared memory.  host_out: HOST. */
typedef struct {
  uint32_t threads, ctas_per_replica, ctas_per_sm, chunks, cand_global, coresident;
} sae_layout_info;
sae_status sae_layout(const sae_ctx* ctx, sae_layout_info* host_out);

/* Profiling (bench roofline): when enabled, every replay-kernel launch is bracketed
 * by CUDA events on its stream; sae_profile_read synchronizes, returns the summed
 * elapsed milliseconds and the number of launches since the last read, and resets. */
sae_status sae_profile(sae_ctx* ctx, int enable);
sae_status sae_profile_read(sae_ctx* ctx, double* ms_total, uint64_t* n_launches);
/* Same for the K1 hashing kernel (chained XXH64 + tau of every block of a batch, P:158-159,
 * P:318-320) launched by sae_admit_batch / sae_lookup while profiling is enabled. */
sae_status sae_profile_read_hash(sae_ctx* ctx, double* ms_total, uint64_t* n_launches);

/* ---------------------------------------------------------------------------------------
 * Multi-turn session predictor (Eq.(4)).  For a history-free
 * request the final-layer hidden state h (d wide) of its last prompt token goes through a
 * three-layer MLP with hidden widths 256 and 64:
 *     y = W3 relu(W2 relu(W1 h + b1) + b2) + b3,    is_multi_turn = (y > 0)
 * DESIGN.md readings A43-A45: h, W1, W2 are bf16 (the serving model's activations; tensor-core
 * operands), b1, b2, W3, b3 fp32; products accumulate in fp32; relu(W1 h + b1) is rounded to
 * bf16 as GEMM2's operand.  Runs on tcgen05 tensor cores (TMA + TMEM), one persistent CTA per
 * SM over 256-row tiles.  Errors: SAE_E_INVAL (null pointer, d not a positive multiple of 32,
 * h not 16-byte aligned), SAE_E_ABI, SAE_E_OOM, SAE_E_CUDA; sae_predictor_last_error() text.
 * --------------------------------------------------------------------------------------- */
typedef struct sae_predictor sae_predictor;
typedef struct {
  uint32_t abi_version;       /* SAE_ABI_VERSION */
  uint32_t d;                 /* hidden size of h (multiple of 32); 4096 in DESIGN.md A43 */
  int32_t device;
  uint32_t _pad;
} sae_predictor_config;

/* Create a predictor on cfg->device.  Weights are HOST pointers, copied to the device before
 * the call returns: w1 bf16 bits [256 x d] row-major (W1[i][j]: output i, input j), b1 f32
 * [256], w2 bf16 bits [64 x 256], b2 f32 [64], w3 f32 [64], b3.  *out owned by the caller
 * until sae_predictor_destroy; nothing is leaked on error. */
sae_status sae_predictor_create(const sae_predictor_config* cfg, const uint16_t* w1, const float* b1,
                                const uint16_t* w2, const float* b2, const float* w3, float b3,
                                sae_predictor** out);
sae_status sae_predictor_destroy(sae_predictor* p);
/* Predict n requests, stream-ordered and asynchronous.  h: DEVICE bf16 bits [n x d]
 * row-major (16-byte aligned), read-only.  Outputs (DEVICE, either may be NULL but not both):
 * logit[o] = y (f32) and flags[o] = (flags[o] & ~1) | (y > 0) -- bit 0 of sae_batch.flags,
 * is_multi_turn -- with o = rows[i] when rows (DEVICE u32 [n], distinct) is given, else i. */
sae_status sae_predict(sae_predictor* p, const uint16_t* h, uint32_t n, const uint32_t* rows, float* logit,
                       uint8_t* flags, sae_stream s);
uint64_t sae_predictor_launch_count(const sae_predictor* p);
/* Text of the last error of p; of the last failed sae_predictor_create when p is NULL. */
const char* sae_predictor_last_error(const sae_predictor* p);

#ifdef __cplusplus
}
#endif
#endif /* SAE_H_ */
