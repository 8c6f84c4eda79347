// sae.cu — SAECache hot path on B200 (sm_100a): kernels + C ABI (include/sae.h).
//
// Paper: arxiv 2605.18825, /root/reference/PAPER.md ("P:<line>").  Readings of
// silent/conflicting passages: DESIGN.md "Readings".
//
// Device layout: per replica r a struct-of-
// arrays block table of C slots (hash u64, last f64, key u64 = the scan key, id u32,
// meta u32 = q|tau|ntok|live|pin|candidacy-table entry, ob u32, omax u32, acc u32,
// table position u32), an open-addressing resident table (u64 key -> slot,
// tombstones + rebuild), a free-slot stack, the ghost ring (recently_evicted,
// P:535) with its own hash index, the ln(dt) interval rings, and a scalar
// state record (counters, learned parameters, E, ids).
//
// Kernels:
//   k_nblocks / k_scan*   block offsets of the batch
//   k_runs                per-replica request runs
//   k_hash      (K1)      chained XXH64 + tau (median token) per block, one thread per request
//   k_replay    (K2-K5)   persistent: one CTA owns one replica and replays its requests in
//                         order: probe+touch+stats -> fused score/select -> apply -> learn
//   k_lookup              read-only probes, one warp per request
//   k_gen_tokens (K7)     synthetic token materialisation (input generator)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sae.h"
#include "dmath.cuh"
#include "xxh64.cuh"

namespace sae {

constexpr uint64_t KEY_EMPTY = ~0ull;
constexpr uint64_t KEY_TOMB = ~0ull - 1;
constexpr uint32_t SLACK = 32;     // extra candidates kept per segment across chunks (min)
constexpr int NSEG = 13;           // EF, 8 multi-turn classes (queue, tau), 4 STRUCT classes (tau)
constexpr uint32_t MSUB = 96;      // victims selected per scan pass (keys are frozen within a chunk)
constexpr uint32_t VCAP = 256;      // victim staging buffer (m smallest + key ties); power of two >= 2*MSUB
constexpr int RMAX = 4096;         // max interval ring
constexpr uint32_t SLOT_MASK = 0x0FFFFFFFu;
constexpr double INV_SQRT2 = 0.70710678118654757;  // 0x3FE6A09E667F3BCD

enum { Q_EF = 0, Q_CHAT = 1, Q_AGENT = 2, Q_STRUCT = 3 };
enum { M_LIVE = 1u << 10, M_PIN = 1u << 11 };
// meta bits 12..23: tix, the block's entry in the per-pass candidacy table: its segment
// (0 EF, 1..8 multi-turn classes) or, for STRUCT, 16 + (tau & 3) * 256 + q8 with
// q8 = floor(-ln(o_b/o_max) * 32) (255 for o_b = 0): -q8/32 is an upper bound of ln(o_b/o_max).
constexpr uint32_t M_TIX_SHIFT = 12;

__host__ __device__ inline uint32_t meta_pack(uint32_t q, uint32_t tau, uint32_t ntok) {
  return q | (tau << 2) | (ntok << 5) | M_LIVE;
}
__device__ inline uint32_t meta_q(uint32_t m) { return m & 3u; }
__device__ inline uint32_t meta_tau(uint32_t m) { return (m >> 2) & 7u; }
__device__ inline uint32_t meta_ntok(uint32_t m) { return (m >> 5) & 31u; }

// Replica scalar state (counters, learned params, bookkeeping).  Lives in global
// memory between launches and in the owning CTA's shared memory during a replay.
struct RState {
  double now;
  uint32_t has_now, err;
  uint64_t E, next_id, gseq, round;
  uint32_t live, free_top, tbl_used, gtbl_used;
  uint32_t iv_head[2], iv_len[2];
  uint64_t ts_ev[5], ts_mae[5], ts_hit[5], ts_acc[5];
  uint64_t qh[3], qe[3];
  uint64_t pb_hit[16], pb_acc[16];
  uint64_t traj_n;
  // statistics
  uint64_t requests, blocks_looked_up, hit_blocks, hit_tokens, prompt_tokens, evictions;
  uint64_t evict_by_queue[4], evict_by_type[6], mae_by_type[6];
  uint64_t learner_firings, eviction_rounds, blocks_scored, blocks_scored_struct;
  uint64_t select_passes, select_cands, select_big, select_fail_seg[10];
  uint64_t select_narrow, select_raw;
  uint64_t stage2_chunks;  // chunks whose victims reach Alg.1 Stage 2 (EF cannot cover them)
  uint64_t tph[16];         // leader phase timers (ns): probe, scan, narrow, select, apply, learn, insert, rebuild,
                            // + issue(): start barrier, own partition, end barrier, (spare)
  uint32_t segcnt[16];     // live blocks per segment (maintained at insert / touch / evict)
  uint64_t thr[16];        // per-segment candidate thresholds on k0 (heuristic; exactness never depends on them)
  uint8_t trim_skip[16];   // passes left before a segment may be trimmed again (a trim that did not
                           // lower its threshold backs off: STRUCT candidates are a superset of
                           // the blocks under the threshold, which trimming cannot shrink)
  sae_params par;
};

struct alignas(16) Cand {  // one candidate victim: sort key (tier, k0, k1, k2) + slot + segment
  uint64_t k0, k1;
  uint32_t k2, ss;      // ss = slot | tier << 28
  uint32_t seg, pad;
};

// Control block of a multi-CTA replica group (global memory, one per replica).  The
// leader CTA publishes a command + its parameters; all CTAs of the group execute their
// partition of it between two group barriers.
enum { CMD_SCAN = 1, CMD_HIST, CMD_COMPACT, CMD_CLEAR_T, CMD_FILL_T, CMD_CLEAR_G,
       CMD_FILL_G, CMD_COUNTQ, CMD_EXIT };
struct GroupCtl {          // hot words on separate 128-byte lines (polled / atomically updated)
  alignas(128) unsigned long long cmdw;   // posted command word (epoch:24 | seq:32 | cmd:8)
  alignas(128) unsigned long long done;   // cumulative worker completions this launch
  alignas(128) unsigned ncand;
  alignas(128) unsigned nsel;
  alignas(128) unsigned tblcnt;
  alignas(128) unsigned gtblcnt;
  alignas(128) unsigned segtot[16];
  alignas(128) unsigned cnt[16];
  alignas(128) unsigned selcnt[16];
  alignas(128) unsigned cntq[4];
  unsigned long long wscan_ns;        // worker 1's accumulated scan time (diagnostic)
  unsigned long long wdbg[4];         // SAE_WORKER_TIMERS debug build: per-pass worker maxima
  alignas(128) unsigned cmd, stamp, shift, active;   // read-only while a command runs
  unsigned long long thr[16], pfx[16], pmask[16];
  double now, gamma, dt_eps, z_cut;
  double cw[3][5], mu[2], sigma[2], w[5];
  unsigned mode;
  alignas(128) unsigned hist[NSEG * 256];
};

struct Dev {
  uint32_t R, C, tmask, G, gmask, K, iv_ring, iv_keep, iv_min, nbins, B, traj_cap;
  uint32_t GP;          // CTAs per replica (group size)
  uint32_t epoch;       // launch counter of the ctx (group command words are tagged with it)
  uint32_t cand_smem;   // 1: candidates live in the leader's smem (C <= CAND_MAX, GP == 1)
  uint32_t bulk_ok;     // 1: replica bases are 16-byte aligned (C % 4 == 0): bulk-copy scan
  uint32_t slack;              // minimum reserve of candidates per segment (env SAE_SLACK; default 32)
  uint32_t trim_at, trim_to;   // threshold trimming: a segment holding > trim_at x its want is
                               // cut to trim_to x want (env SAE_TRIM="at,to"; default 8,4)
  uint32_t scan_l2;     // L2 policy of the streamed scan columns: 1 evict_last (they fit in L2
                        // next to the random-access state), 2 evict_first (they do not)
  uint32_t nchunk;      // > 1: task-split replay (single-CTA replicas, more replicas than
                        // co-resident CTAs): each replica's run is cut into nchunk consecutive
                        // chunks, a persistent grid takes (chunk, replica) tasks in order from
                        // *taskctr, and chunk k of replica r waits for rflag[r] = (epoch, k)
  uint32_t early_q;     // the select's radix stops once the chosen prefix set holds at most
                        // early_q/4 of the staging limit (env SAE_EARLY = 1..8; default 4)
  uint32_t* taskctr;    // [1] next task of the current launch (zeroed before each launch)
  uint32_t* rflag;      // [R] (epoch << 8) | chunks of the replica's run done this launch
  Cand* gcand;          // [R*C] global candidate buffer (large pools)
  Cand* gsel;           // [R*CAND_MAX] compacted candidates after narrowing
  Cand* cpriv;          // [R*CAND_MAX] private candidate buffers of the v256g variant
  GroupCtl* ctl;        // [R]
  uint64_t hash_seed;
  double dt_eps, z_cut;
  RState* st;
  uint64_t* bhash;
  double* blast;
  uint32_t* bid;
  uint32_t* bmeta;
  uint32_t* bob;
  uint32_t* bomax;
  uint64_t* bkey;       // scan key: EF ? (ntok << 32 | id) : obits(last)
  uint32_t* bacc;
  uint32_t* btpos;       // the block's position in the resident table (set at insert / rebuild)
  uint32_t* freestk;
  uint64_t* tkey;
  uint32_t* tval;
  uint64_t* ghash;
  uint8_t* gtau;
  uint8_t* glive;
  uint32_t* gtslot;
  uint64_t* gkey;
  uint32_t* gval;
  double* iv;
  sae_traj* traj;
  uint32_t* err;      // sticky first error (as -status), global
};

struct BatchDev {
  uint32_t n;
  const uint32_t* replica;
  const double* arrival;
  const uint64_t* poff;
  const uint32_t* plen;
  const uint64_t* doff;
  const uint32_t* dlen;
  const uint32_t* tokens;
  const uint8_t* types;
  const uint8_t* flags;
  const uint32_t* spb;
  uint64_t* boff;         // [n+1]
  uint64_t tb;            // the caller's total_blocks (workspace size); checked against boff[n]
  uint64_t* h;            // [TB]
  uint8_t* tau;
  uint8_t* ntok;
  int32_t* slot;
  uint8_t* q;
  int32_t* nrank;
  uint32_t* run_start;    // [R]
  uint32_t* run_end;
  // outputs
  uint32_t* o_hit;
  uint32_t* o_miss;
  uint32_t* o_matched;
  uint32_t* o_nvict;
  uint64_t* o_voff;
  uint32_t* o_vids;
  uint64_t vcap;
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ inline void raise_err(const Dev& d, int status) {
  atomicCAS(d.err, 0u, (uint32_t)(-status));
}

// ordered-bits transform: u64 order == double order (non-NaN)
__device__ __forceinline__ uint64_t obits(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ double from_obits(uint64_t o) {
  uint64_t b = (o >> 63) ? (o & ~(1ull << 63)) : ~o;
  return __longlong_as_double((long long)b);
}

// ---------------------------------------------------------------------------
// Policy arithmetic (fixed op order, explicit RN intrinsics; SURVEY c.4)
// ---------------------------------------------------------------------------
// Eq.(1): p = 1 - F_LN(dt) = 0.5*erfc(z/sqrt2), z = (ln dt - mu)/sigma (A36)
// (Keeping the large multiply-called device functions out of line cut the replay kernel's SASS
//  by a third but measured much slower: C5 2.4 vs 2.95 M req/s, k_select 77.8 vs 60.3 us.)
__device__ double survival(double dt, double mu, double sg, double z_cut) {
  double z = __ddiv_rn(__dsub_rn(dm::ln(dt), mu), sg);
  if (z > z_cut) return 0.0;
  return __dmul_rn(0.5, dm::erfc(__dmul_rn(z, INV_SQRT2)));
}
// Eq.(2): p = 1 - (o/o_max)^gamma with pow(x,y) = exp(y ln x)
__device__ double p_struct(uint32_t ob, uint32_t omax, double gam) {
  if (ob == 0) return 1.0;
  double r = __ddiv_rn((double)ob, (double)omax);
  return __dsub_rn(1.0, dm::ex(__dmul_rn(gam, dm::ln(r))));
}
// gamma-independent per-block input of the STRUCT prefilter (meta tix): q8 with
// -q8/32 >= ln(o_b/o_max), so the bound below stays a lower bound of p; 255 encodes o_b = 0.
__device__ __forceinline__ uint32_t q8_of(uint32_t ob, uint32_t omax) {
  if (ob == 0) return 255u;
  const double x = -dm::ln(__ddiv_rn((double)ob, (double)omax)) * 32.0;
  const double f = floor(x * (1.0 - 0x1p-40));     // never rounds past the true value
  return (uint32_t)fmin(fmax(f, 0.0), 254.0);
}
__device__ __forceinline__ uint32_t tix_of(uint32_t q, uint32_t tau, uint32_t ob, uint32_t omax) {
  if (q == Q_EF) return 0u;
  if (q != Q_STRUCT) return 1u + (q - 1u) * 4u + (tau & 3u);
  return 16u + ((tau & 3u) << 8) + q8_of(ob, omax);
}
__device__ __forceinline__ uint32_t meta_tix(uint32_t m) { return (m >> M_TIX_SHIFT) & 0xFFFu; }
// segment of a table index: EF 0, multi-turn classes 1..8, STRUCT classes 9..12
__device__ __forceinline__ uint32_t seg_of_tix(uint32_t tix) { return tix < 16u ? tix : 9u + ((tix - 16u) >> 8); }
// A guaranteed lower bound of Eq.(2)'s p = 1 - exp(gamma * ln(o/o_max)) (gamma > 0) from
// q8: fp32 exp (relative error < 1e-5 over the argument range) inflated by 2^-10.  Used
// only to decide which STRUCT blocks need their exact score; never to order them.
__device__ __forceinline__ double p_struct_lo8(uint32_t q8, float gam) {
  if (q8 == 255u) return 1.0 - 0x1p-10;
  const double e = (double)__expf(-gam * ((float)q8 * (1.0f / 32.0f)));
  return 1.0 - fmin(1.0, e * (1.0 + 0x1p-10));
}
// scan key of a block (see Dev::bkey)
__device__ __forceinline__ uint64_t scan_key(uint32_t q, uint32_t ntok, uint32_t id, double last) {
  return q == Q_EF ? (((uint64_t)ntok << 32) | id) : obits(last);
}

// Alg.1 Classify
__device__ __forceinline__ uint32_t classify(uint32_t tau, bool mt, bool ag, bool cid, bool is_struct,
                                             bool untempl) {
  if (tau == 4 || tau == 5 || untempl) return Q_EF;
  if (mt && ag) return Q_AGENT;
  if (mt || cid) return Q_CHAT;
  if (is_struct || tau == 0) return Q_STRUCT;
  return Q_EF;
}

// ---------------------------------------------------------------------------
// Open-addressing tables (linear probing; EMPTY / TOMB sentinels)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t home(uint64_t h, uint32_t mask) {
  return (uint32_t)(h ^ (h >> 29)) & mask;
}
__device__ int32_t tbl_find(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                            uint32_t mask, uint64_t h) {
  uint32_t i = home(h, mask);
  while (true) {
    uint64_t k = keys[i];
    if (k == h) return (int32_t)vals[i];
    if (k == KEY_EMPTY) return -1;
    i = (i + 1) & mask;
  }
}
__device__ int32_t tbl_find_pos(const uint64_t* __restrict__ keys, uint32_t mask, uint64_t h) {
  uint32_t i = home(h, mask);
  while (true) {
    uint64_t k = keys[i];
    if (k == h) return (int32_t)i;
    if (k == KEY_EMPTY) return -1;
    i = (i + 1) & mask;
  }
}
// Insert a key known to be absent.  Concurrent inserts of distinct keys are safe;
// no lookups run concurrently.  Returns the position; *fresh = consumed an EMPTY.
__device__ uint32_t tbl_insert(uint64_t* keys, uint32_t* vals, uint32_t mask, uint64_t h, uint32_t v,
                               uint32_t* used) {
  uint32_t i = home(h, mask);
  while (true) {
    uint64_t k = keys[i];
    if (k == KEY_EMPTY || k == KEY_TOMB) {
      unsigned long long prev = atomicCAS((unsigned long long*)&keys[i], (unsigned long long)k,
                                          (unsigned long long)h);
      if (prev == k) {
        vals[i] = v;
        if (k == KEY_EMPTY) atomicAdd(used, 1u);
        return i;
      }
      continue;  // lost the race: re-examine slot i
    }
    i = (i + 1) & mask;
  }
}

// ---------------------------------------------------------------------------
// Batch preparation kernels
// ---------------------------------------------------------------------------
__global__ void k_nblocks(BatchDev b, uint32_t B, uint64_t* cnt) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b.n) cnt[i] = (uint64_t)((b.plen[i] + B - 1) / B) + (uint64_t)((b.dlen[i] + B - 1) / B);
}

// exclusive scan of n u64 values (in place into out[0..n], out[n] = total); 3 phases
constexpr int SCAN_TILE = 4096;
__global__ void k_scan_reduce(const uint64_t* in, uint64_t n, uint64_t* part) {
  __shared__ uint64_t s[32];
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  uint64_t acc = 0;
  for (uint64_t i = base + threadIdx.x; i < base + SCAN_TILE && i < n; i += blockDim.x) acc += in[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_scan_parts(uint64_t* part, uint32_t np) {
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (uint32_t i = 0; i < np; ++i) { uint64_t v = part[i]; part[i] = run; run += v; }
    part[np] = run;
  }
}
__global__ void k_scan_apply(const uint64_t* in, uint64_t n, const uint64_t* part, uint64_t* out,
                             uint32_t np) {
  // one CTA per tile, 1024 threads x 4 items, sequential within thread then block scan
  __shared__ uint64_t s[1024];
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  uint64_t v[4], loc = 0;
  for (int k = 0; k < 4; ++k) {
    uint64_t i = base + threadIdx.x * 4 + k;
    v[k] = i < n ? in[i] : 0;
    loc += v[k];
  }
  s[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint64_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  uint64_t run = part[blockIdx.x] + s[threadIdx.x] - loc;
  for (int k = 0; k < 4; ++k) {
    uint64_t i = base + threadIdx.x * 4 + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (blockIdx.x == np - 1 && threadIdx.x == 0) out[n] = part[np];
}

constexpr uint32_t RUN_INVALID = 0xFFFFFFFEu;   // run_start of a replica whose requests are split

// The caller's total_blocks sizes the per-batch workspace: a batch whose real block count
// (boff[n], computed on the device) exceeds it would write past the workspace.  Every kernel
// that indexes by block offset checks this first and does nothing on a mismatch.
__device__ __forceinline__ bool batch_size_ok(const BatchDev& b) { return b.boff[b.n] <= b.tb; }

__global__ void k_runs(BatchDev b, Dev d) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  uint32_t r = b.replica[i];
  if (r >= d.R) { raise_err(d, SAE_E_INVAL); return; }
  if (i == 0 || b.replica[i - 1] != r) {
    // a second run of the same replica: its requests are not contiguous.  Mark the replica
    // invalid (k_replay skips it, its state stays untouched) and raise the sticky error.
    if (atomicCAS(&b.run_start[r], 0xFFFFFFFFu, i) != 0xFFFFFFFFu) {
      atomicExch(&b.run_start[r], RUN_INVALID);
      raise_err(d, SAE_E_INVAL);
    }
  }
  if (i == b.n - 1 || b.replica[i + 1] != r) b.run_end[r] = i + 1;
}

// K1: chained hashing + tau (A1-A4, A34). One thread per request.
__global__ void __launch_bounds__(128) k_hash(BatchDev b, Dev d) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  if (!batch_size_ok(b)) {
    if (i == 0) raise_err(d, SAE_E_INVAL);
    return;
  }
  const uint32_t B = d.B;
  uint32_t L = b.plen[i], O = b.dlen[i];
  uint32_t np = (L + B - 1) / B, nd = (O + B - 1) / B;
  uint64_t bo = b.boff[i];
  const uint32_t* pt = b.tokens + b.poff[i];
  const uint8_t* py = b.types + b.poff[i];
  uint64_t prev = d.hash_seed;
  for (uint32_t j = 0; j < np; ++j) {
    uint32_t s = j * B, nj = min(B, L - s);
    prev = xx::block(prev, pt + s, (int)nj);
    b.h[bo + j] = prev;
    b.tau[bo + j] = py[s + nj / 2];
    b.ntok[bo + j] = (uint8_t)nj;
  }
  const uint32_t* dt = b.tokens + b.doff[i];
  for (uint32_t j = 0; j < nd; ++j) {
    uint32_t s = j * B, nj = min(B, O - s);
    prev = xx::block(prev, dt + s, (int)nj);
    b.h[bo + np + j] = prev;
    b.tau[bo + np + j] = 5;
    b.ntok[bo + np + j] = (uint8_t)nj;
  }
}

// The replay kernels in three compiled variants (NT threads, candidate buffer of CAND_MAX
// records in shared memory or -- CAND_GLOBAL -- in the replica's L1-resident global region,
// MINB CTAs per SM):
//   v512  groups / few replicas / large pools: lowest latency per replica
//   v256  many small replicas, two CTAs per SM
//   v256g many small replicas, three CTAs per SM (candidates in global memory)
namespace v512 {
constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int CAND_MAX = 4096;   // (6144, a ring of four 48 KB tiles, measured no faster: k_select 62.1 vs 61.2 us)
constexpr bool CAND_GLOBAL = false;
constexpr int MINB = 1;
#include "replay_impl.cuh"
}  // namespace v512
namespace v256 {
constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int CAND_MAX = 2560;
constexpr bool CAND_GLOBAL = false;
constexpr int MINB = 2;
#include "replay_impl.cuh"
}  // namespace v256
namespace v256g {
constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int CAND_MAX = 2560;
constexpr bool CAND_GLOBAL = true;
constexpr int MINB = 3;
#include "replay_impl.cuh"
}  // namespace v256g
#ifndef SAE_V128_MINB
#define SAE_V128_MINB 7
#endif
namespace v128g {
constexpr int NT = 128;
constexpr int NW = NT / 32;
constexpr int CAND_MAX = 2560;
constexpr bool CAND_GLOBAL = true;
constexpr int MINB = SAE_V128_MINB;
#include "replay_impl.cuh"
}  // namespace v128g

// read-only probe, one warp per request
__global__ void k_lookup(Dev d, BatchDev b, uint32_t* out) {
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= b.n || !batch_size_ok(b)) return;
  const uint32_t r = b.replica[wid];
  if (r >= d.R) return;
  const uint32_t B = d.B;
  const uint32_t n = (b.plen[wid] + B - 1) / B + (b.dlen[wid] + B - 1) / B;
  const uint64_t bo = b.boff[wid], tb = (uint64_t)d.tmask + 1;
  const uint64_t* tkey = d.tkey + (uint64_t)r * tb;
  const uint32_t* tval = d.tval + (uint64_t)r * tb;
  uint32_t h = n;
  for (uint32_t j0 = 0; j0 < n; j0 += 32) {
    const uint32_t j = j0 + lane;
    bool miss = j < n && tbl_find(tkey, tval, d.tmask, b.h[bo + j]) < 0;
    uint32_t bal = __ballot_sync(~0u, miss);
    if (bal) { h = j0 + __ffs(bal) - 1; break; }
  }
  if (lane == 0) out[wid] = h;
}

__global__ void k_init(Dev d) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t RC = (uint64_t)d.R * d.C;
  for (uint64_t i = tid; i < RC; i += stride) {
    d.bmeta[i] = 0;
    d.btpos[i] = 0;
    d.freestk[i] = d.C - 1 - (uint32_t)(i % d.C);
  }
  const uint64_t TBn = (uint64_t)d.R * (d.tmask + 1ull);
  for (uint64_t i = tid; i < TBn; i += stride) d.tkey[i] = KEY_EMPTY;
  const uint64_t GTn = (uint64_t)d.R * (d.gmask + 1ull);
  for (uint64_t i = tid; i < GTn; i += stride) d.gkey[i] = KEY_EMPTY;
  const uint64_t RG = (uint64_t)d.R * d.G;
  for (uint64_t i = tid; i < RG; i += stride) d.glive[i] = 0;
}

// params gather / scatter (all replicas) for multi-GPU parameter sync (NCCL all-gather)
__global__ void k_params_gather(Dev d, sae_params* out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < d.R; r += gridDim.x * blockDim.x)
    out[r] = d.st[r].par;
}
// replace parameters (they feed the kernels only through RState: no cached
// parameter-dependent block state to refresh)
__global__ void k_params_commit(Dev d, const sae_params* in, uint32_t r0, uint32_t nr) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x)
    if (r0 + i < d.R) d.st[r0 + i].par = in[i];
}

// mean_w sync: for parameter point p, w_mean[tau] = (sum over i = 0..S-1 in
// index order of w[p + P*i][tau]) / S; every replica of point p gets w_mean.  Fixed
// order => identical results at any GPU count (no fp64 all-reduce).
__global__ void k_point_mean(const sae_params* all, uint32_t n_total, uint32_t n_points, sae_params* out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_total) return;
  const uint32_t p = r % n_points, S = n_total / n_points;
  sae_params o = all[r];
  for (int t = 0; t < 5; ++t) {
    double acc = 0.0;
    for (uint32_t i = 0; i < S; ++i) acc = __dadd_rn(acc, all[p + n_points * i].w[t]);
    o.w[t] = __ddiv_rn(acc, (double)S);
  }
  out[r] = o;
}

// sae_counters_device: thread f sums additive counter f over the replicas (fixed layout of
// sae_counters = the leading fields of RState's statistics block, in the same order)
static_assert(offsetof(RState, blocks_scored_struct) - offsetof(RState, requests) + 8 == sizeof(sae_counters),
              "sae_counters mirrors the leading statistics of RState");
__global__ void k_counters(Dev d, sae_counters* out) {
  constexpr int NF = (int)(sizeof(sae_counters) / 8);
  const int f = threadIdx.x;
  if (f >= NF) return;
  unsigned long long acc = 0;
  for (uint32_t r = 0; r < d.R; ++r) {
    const RState& st = d.st[r];
    const uint64_t* base = &st.requests;    // requests .. blocks_scored_struct are contiguous
    acc += base[f];
  }
  reinterpret_cast<uint64_t*>(out)[f] = acc;
}

__global__ void k_count_queues(Dev d, uint32_t r, unsigned long long* out5) {
  const uint64_t base = (uint64_t)r * d.C;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < d.C; s += gridDim.x * blockDim.x) {
    uint32_t m = d.bmeta[base + s];
    if (m & M_LIVE) { atomicAdd(&out5[meta_q(m)], 1ull); atomicAdd(&out5[4], 1ull); }
  }
}

// sae_priority: Eq.(1)-(3) exactly as finalize_key scores a candidate (cw = alpha * w first)
__global__ void k_priority(sae_params p, double dt_eps, double z_cut, uint64_t n, const uint8_t* q,
                           const uint8_t* tau, const double* dt_in, const uint32_t* ob,
                           const uint32_t* omax, double* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t qq = q[i], t = tau[i] & 3u;
  if (qq == 0 || qq > 3) { out[i] = __longlong_as_double(0x7ff8000000000000ll); return; }
  double dt = dt_in[i];
  if (dt < dt_eps) dt = dt_eps;
  const double cw = __dmul_rn(p.alpha[qq - 1], p.w[t]);
  const double pp = qq == 3 ? p_struct(ob[i], omax[i], p.gamma)
                            : survival(dt, p.mu[qq - 1], p.sigma[qq - 1], z_cut);
  out[i] = __ddiv_rn(__dmul_rn(cw, pp), dt);
}

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// Characterisation pass (A42): unbounded cache over a trace.
// Two insert-or-find tables keyed by the block hash and by (hash, session) hold the first
// global block index of each key (atomicMin); a block at index g is reused iff its hash's
// first index < g, intra-session iff its (hash, session)'s first index < g.
// ---------------------------------------------------------------------------
struct CharDev {
  uint64_t* k1; unsigned long long* v1;   // hash -> first global block index
  uint64_t* k2; unsigned long long* v2;   // (hash, session) -> first global block index
  uint32_t mask;
  const uint32_t* session; const uint32_t* turn; const uint8_t* single;
  unsigned long long* out;                // sae_char_stats as u64[58]
};
__device__ __forceinline__ uint64_t char_key2(uint64_t h, uint32_t sess) {
  return sm64(h ^ sm64((uint64_t)sess + 0x632BE59BD9B4E019ull));
}
__device__ __forceinline__ uint32_t ctab_slot(uint64_t* keys, uint32_t mask, uint64_t k) {
  uint32_t i = home(k, mask);
  while (true) {
    const uint64_t cur = keys[i];
    if (cur == k) return i;
    if (cur == KEY_EMPTY) {
      const unsigned long long prev = atomicCAS((unsigned long long*)&keys[i], KEY_EMPTY, k);
      if (prev == KEY_EMPTY || prev == k) return i;
    }
    i = (i + 1) & mask;
  }
}
__device__ __forceinline__ uint32_t ctab_find(const uint64_t* keys, uint32_t mask, uint64_t k) {
  uint32_t i = home(k, mask);
  while (keys[i] != k) i = (i + 1) & mask;   // every looked-up key was inserted
  return i;
}
__global__ void k_char_insert(BatchDev b, CharDev c) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= b.n || !batch_size_ok(b)) return;
  const uint64_t b0 = b.boff[w], b1 = b.boff[w + 1];
  for (uint64_t g = b0 + lane; g < b1; g += 32) {
    const uint64_t H = b.h[g];
    atomicMin(&c.v1[ctab_slot(c.k1, c.mask, H)], (unsigned long long)g);
    atomicMin(&c.v2[ctab_slot(c.k2, c.mask, char_key2(H, c.session[w]))], (unsigned long long)g);
  }
}
// counter layout (sae_char_stats): blocks[6] reused[6] later_blocks[6] later_intra[6]
// first_blocks[6] first_inter[6] pos_blocks[10] pos_reused[10] reuses_intra reuses_inter
__global__ void k_char_count(BatchDev b, CharDev c, uint32_t B) {
  __shared__ unsigned int acc[58];
  for (int i = threadIdx.x; i < 58; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w < b.n && batch_size_ok(b)) {
    const uint64_t b0 = b.boff[w], b1 = b.boff[w + 1];
    const uint32_t np = (b.plen[w] + B - 1) / B, sess = c.session[w];
    const bool later = c.turn[w] > 0, single = c.single[w] != 0;
    for (uint64_t g = b0 + lane; g < b1; g += 32) {
      const uint64_t H = b.h[g];
      const uint32_t t = b.tau[g], j = (uint32_t)(g - b0);
      const bool reused = c.v1[ctab_find(c.k1, c.mask, H)] < g;
      const bool intra = c.v2[ctab_find(c.k2, c.mask, char_key2(H, sess))] < g;
      atomicAdd(&acc[t], 1u);
      if (reused) atomicAdd(&acc[6 + t], 1u);
      if (later) {
        atomicAdd(&acc[12 + t], 1u);
        if (intra) atomicAdd(&acc[18 + t], 1u);
      } else {
        atomicAdd(&acc[24 + t], 1u);
        if (reused) atomicAdd(&acc[30 + t], 1u);
      }
      if (reused) atomicAdd(&acc[intra ? 56 : 57], 1u);
      if (single && j < np) {
        const uint32_t bin = min(9u, (10u * j) / np);
        atomicAdd(&acc[36 + bin], 1u);
        if (reused) atomicAdd(&acc[46 + bin], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 58; i += blockDim.x)
    if (acc[i]) atomicAdd(&c.out[i], (unsigned long long)acc[i]);
}
// K7: synthetic token materialisation, one CTA per piece (input generator)
__global__ void k_gen_tokens(uint64_t seed, uint64_t np, const uint64_t* stream, const uint64_t* start,
                             const uint32_t* len, const uint64_t* dst, const uint8_t* type,
                             uint32_t* tokens, uint8_t* types) {
  for (uint64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const uint64_t key = sm64(seed ^ sm64(stream[p]));
    const uint64_t s0 = start[p], d0 = dst[p];
    const uint32_t n = len[p];
    const uint8_t ty = type[p];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      tokens[d0 + i] = (uint32_t)(sm64(key ^ (s0 + i)) & 0x1FFFFull);
      types[d0 + i] = ty;
    }
  }
}

}  // namespace sae

// ===========================================================================
// Host side: C ABI
// ===========================================================================
using namespace sae;

// The two compiled replay variants (replay_impl.cuh).
struct Variant {
  const void* replay;
  const void* evict;
  const void* update;
  const void* select;
  int nt;
  size_t smem;
  uint32_t cand_max;
};
static Variant variant(int nt) {
  if (nt == 129)   // v128g
    return {(const void*)v128g::k_replay, (const void*)v128g::k_evict, (const void*)v128g::k_update,
            (const void*)v128g::k_select, 128,
            v128g::smem_bytes(), (uint32_t)v128g::CAND_MAX};
  if (nt == 257)   // v256g
    return {(const void*)v256g::k_replay, (const void*)v256g::k_evict, (const void*)v256g::k_update,
            (const void*)v256g::k_select, 256,
            v256g::smem_bytes(), (uint32_t)v256g::CAND_MAX};
  if (nt == 256)
    return {(const void*)v256::k_replay, (const void*)v256::k_evict, (const void*)v256::k_update,
            (const void*)v256::k_select, 256,
            v256::smem_bytes(), (uint32_t)v256::CAND_MAX};
  return {(const void*)v512::k_replay, (const void*)v512::k_evict, (const void*)v512::k_update,
            (const void*)v512::k_select, 512,
          v512::smem_bytes(), (uint32_t)v512::CAND_MAX};
}

static cudaError_t launch_group(const Variant& v, const void* fn, uint32_t grid, bool coop, cudaStream_t s,
                                Dev& d, BatchDev* x) {
  d.epoch++;
  void* args[] = {(void*)&d, (void*)x};
  if (coop) return cudaLaunchCooperativeKernel(fn, grid, v.nt, args, v.smem, s);
  return cudaLaunchKernel(fn, grid, v.nt, args, v.smem, s);
}

struct sae_ctx {
  sae_config cfg;
  Dev d;
  int device;
  std::string last_error;
  uint64_t launches = 0;
  // per-batch workspace (stream-ordered allocations)
  void* ws = nullptr;
  size_t ws_cap = 0;
  // device staging of sae_admit_batch_host (request arrays + outputs): two slots used
  // alternately, filled on a ctx-owned copy stream so that a call's host->device copies
  // overlap the replay of the previous call; ev_in[k]: slot k's inputs landed, ev_out[k]:
  // slot k's replay + device->host copies done (the slot may be overwritten)
  void* stage[2] = {nullptr, nullptr};
  size_t stage_cap[2] = {0, 0};
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  int slot = 0;
  std::vector<void*> allocs;
  // optional profiling: CUDA events around every k_replay launch (bench roofline)
  uint64_t coresident = 0;
  Variant var;
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_hash;   // K1 (k_hash) launches
};

static uint32_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return (uint32_t)p;
}

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      if (ctx) ctx->last_error = std::string(#call ": ") + cudaGetErrorString(e_); \
      return e_ == cudaErrorMemoryAllocation ? SAE_E_OOM : SAE_E_CUDA;  \
    }                                                                   \
  } while (0)

template <class T>
static cudaError_t dalloc(sae_ctx* ctx, T** p, uint64_t n) {
  cudaError_t e = cudaMalloc((void**)p, (n ? n : 1) * sizeof(T));
  if (e == cudaSuccess) ctx->allocs.push_back((void*)*p);
  return e;
}

extern "C" {

static sae_status create_impl(const sae_config* cfg, sae_ctx* ctx) {
  ctx->cfg = *cfg;
  ctx->device = cfg->device;
  CK(cudaSetDevice(cfg->device));
  {
    // the per-batch workspace comes from the device's default stream-ordered pool: keep freed
    // blocks in the pool (the default threshold 0 hands them back to the driver at every
    // synchronisation, and re-mapping them inside a later step stalled it by 100+ ms)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  Dev& d = ctx->d;
  std::memset(&d, 0, sizeof d);
  d.R = cfg->n_replicas;
  d.C = cfg->capacity_blocks;
  d.G = cfg->ghost_capacity;
  d.K = cfg->K;
  d.iv_ring = cfg->interval_ring;
  d.iv_keep = cfg->interval_keep;
  d.iv_min = cfg->interval_min;
  d.nbins = cfg->n_pos_bins;
  d.B = cfg->block_tokens;
  d.traj_cap = cfg->traj_capacity;
  d.hash_seed = cfg->hash_seed;
  d.dt_eps = cfg->dt_eps;
  d.z_cut = cfg->z_cut;
  // open-addressing tables of 2^ceil(log2 2C) slots (measured on C5: 5C/3-sized tables, half
  // the working set, were slower -- 3.25 vs 3.50 M req/s: longer probe chains, more rebuilds)
  const uint64_t TB = pow2_at_least(2ull * d.C), GT = pow2_at_least(2ull * d.G);
  d.tmask = (uint32_t)(TB - 1);
  d.gmask = (uint32_t)(GT - 1);
  const uint64_t R = d.R, RC = R * d.C;
  CK(dalloc(ctx, &d.st, R));
  CK(dalloc(ctx, &d.bhash, RC));
  CK(dalloc(ctx, &d.blast, RC + 4));   // +4: bulk-copy tail padding
  CK(dalloc(ctx, &d.bid, RC + 4));   // +4: bulk-copy tail padding
  CK(dalloc(ctx, &d.bmeta, RC + 4));   // +4: bulk-copy tail padding
  CK(dalloc(ctx, &d.bob, RC));
  CK(dalloc(ctx, &d.bomax, RC));
  CK(dalloc(ctx, &d.bkey, RC + 4));   // +4: bulk-copy tail padding
  CK(dalloc(ctx, &d.bacc, RC));
  CK(dalloc(ctx, &d.btpos, RC));
  CK(dalloc(ctx, &d.freestk, RC));
  CK(dalloc(ctx, &d.tkey, R * TB));
  CK(dalloc(ctx, &d.tval, R * TB));
  CK(dalloc(ctx, &d.ghash, R * d.G));
  CK(dalloc(ctx, &d.gtau, R * d.G));
  CK(dalloc(ctx, &d.glive, R * d.G));
  CK(dalloc(ctx, &d.gtslot, R * d.G));
  CK(dalloc(ctx, &d.gkey, R * GT));
  CK(dalloc(ctx, &d.gval, R * GT));
  CK(dalloc(ctx, &d.iv, R * 2 * RMAX));
  CK(dalloc(ctx, &d.traj, R * (uint64_t)(d.traj_cap ? d.traj_cap : 1)));
  CK(dalloc(ctx, &d.err, 1));
  // group size: one CTA per replica while the pool fits the leader's candidate buffer;
  // otherwise a co-resident group (cooperative launch) that splits every scan pass
  int nsm = 0, occ = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device));
  for (int vnt : {129, 256, 257, 512}) {
    const Variant v = variant(vnt);
    for (const void* f : {v.replay, v.evict, v.update, v.select})
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem));
  }
  // many small single-CTA replicas (more than SMs) take the 256-thread variant with the
  // candidate buffer in global memory: three per SM hide each other's per-round latency; few
  // replicas, groups and larger pools the 512-thread one (lower latency per replica)
  const bool small = d.C <= variant(256).cand_max && cfg->ctas_per_replica <= 1 && R > (uint64_t)nsm;
  // SAE_VARIANT=256|257|512 forces a variant (measurements); 257 = v256g
  int vsel = small ? 257 : 512;   // v256g: three CTAs per SM (measured 3.05 M vs 2.94 M req/s on C5)
  if (const char* e = getenv("SAE_VARIANT")) {
    const int v = atoi(e);
    if (v == 129 || v == 256 || v == 257 || v == 512) vsel = v;
    if (vsel != 512 && d.C > variant(vsel).cand_max) vsel = 512;
  }
  ctx->var = variant(vsel);
  if (vsel == 257 || vsel == 129) CK(dalloc(ctx, &d.cpriv, R * (uint64_t)ctx->var.cand_max));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->var.replay, ctx->var.nt, ctx->var.smem));
  const uint64_t coresident = (uint64_t)nsm * (uint64_t)(occ > 0 ? occ : 1);
  uint64_t gp = cfg->ctas_per_replica;
  if (gp == 0) {
    if (d.C <= ctx->var.cand_max) gp = 1;
    else gp = std::min<uint64_t>(std::max<uint64_t>(1, d.C / 8192), coresident / R);
  }
  if (gp == 0 || (gp > 1 && gp * R > coresident)) {
    ctx->last_error = "ctas_per_replica x n_replicas exceeds the co-resident CTA capacity";
    return SAE_E_INVAL;
  }
  d.GP = (uint32_t)gp;
  d.cand_smem = (d.C <= ctx->var.cand_max && d.GP == 1) ? 1u : 0u;
  if (cfg->init.mode > SAE_MODE_TWO || (cfg->init.mode != SAE_MODE_SAE && !d.cand_smem)) {
    ctx->last_error = "baseline modes need a pool that fits one CTA's candidate buffer";
    return SAE_E_INVAL;
  }
  d.bulk_ok = (d.C % 4 == 0) ? 1u : 0u;
  d.trim_at = 8;
  d.trim_to = 4;
  d.slack = d.cand_smem ? SLACK / 2 : SLACK;   // private pools: rescans are cheap, keep fewer
  if (const char* e = getenv("SAE_SLACK")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 1024) d.slack = (uint32_t)v;
  }
  if (const char* e = getenv("SAE_TRIM")) {
    unsigned a = 0, b = 0;
    if (sscanf(e, "%u,%u", &a, &b) == 2 && a >= 2 && b >= 1 && b < a) { d.trim_at = a; d.trim_to = b; }
  }
  {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, cfg->device);
    const uint64_t scan_bytes = (uint64_t)d.R * d.C * 12ull;
    d.scan_l2 = scan_bytes * 2 <= (uint64_t)l2 ? 1u : 2u;
  }
  ctx->coresident = coresident;
  // task-split replay when single-CTA replicas outnumber the co-resident CTAs: about 32
  // tasks per CTA, so the dynamic task order evens out both the wave quantisation and the
  // replicas' unequal costs (C5 on one B200, 1024 replicas on 444 CTAs: whole replicas
  // 3.07 M req/s; 3 / 6 / 10 / 25 chunks 3.39 / 3.58 / 3.61 / 3.64 M)
  d.nchunk = 1;
  if (d.GP == 1 && R > coresident)
    d.nchunk = (uint32_t)std::min<uint64_t>(32, (32 * coresident + R - 1) / R);
  if (const char* e = getenv("SAE_CHUNKS")) {   // measurements: force (1 = whole replicas)
    const int v = atoi(e);
    if (v >= 1 && v <= 255 && d.GP == 1) d.nchunk = (uint32_t)v;
  }
  d.early_q = 4;    // measured on C5 (select phase per step): 1: 14.9 ms, 2: 13.5-13.9, 3: 13.2, 4: 12.8
  if (const char* e = getenv("SAE_EARLY")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 8) d.early_q = (uint32_t)v;   // up to 8: twice the limit = the whole staging buffer
  }
  CK(dalloc(ctx, &d.taskctr, 1));
  CK(dalloc(ctx, &d.rflag, R));
  CK(cudaMemset(d.rflag, 0, R * 4));
  CK(dalloc(ctx, &d.ctl, R));
  CK(cudaMemset(d.ctl, 0, R * sizeof(GroupCtl)));
  if (!d.cand_smem) {
    CK(dalloc(ctx, &d.gcand, RC));
    CK(dalloc(ctx, &d.gsel, R * (uint64_t)ctx->var.cand_max));
  }
  // initial scalar state
  std::vector<RState> st(R);
  for (uint64_t r = 0; r < R; ++r) {
    RState s;
    std::memset(&s, 0, sizeof s);
    s.free_top = d.C;
    for (int g = 0; g < 16; ++g) s.thr[g] = ~0ull;
    s.par = cfg->init;
    st[r] = s;
  }
  CK(cudaMemcpy(d.st, st.data(), R * sizeof(RState), cudaMemcpyHostToDevice));
  CK(cudaMemset(d.err, 0, sizeof(uint32_t)));
  k_init<<<1024, 256>>>(d);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return SAE_OK;
}

// text of the last failed sae_create (sae_last_error(NULL))
static thread_local std::string g_create_error;

sae_status sae_create(const sae_config* cfg, sae_ctx** out) {
  g_create_error.clear();
  if (!cfg || !out) { g_create_error = "null argument"; return SAE_E_INVAL; }
  if (cfg->abi_version != SAE_ABI_VERSION) { g_create_error = "ABI version mismatch"; return SAE_E_ABI; }
  if (cfg->capacity_blocks == 0) { g_create_error = "capacity_blocks == 0"; return SAE_E_CAPACITY_ZERO; }
  if (cfg->n_replicas == 0 || cfg->block_tokens == 0 || cfg->block_tokens > 16 || cfg->K == 0 ||
      cfg->ghost_capacity == 0 || cfg->interval_ring == 0 || cfg->interval_ring > RMAX ||
      cfg->n_pos_bins == 0 || cfg->n_pos_bins > 16 || cfg->capacity_blocks > SLOT_MASK ||
      !(cfg->init.sigma[0] > 0.0) || !(cfg->init.sigma[1] > 0.0)) {
    g_create_error = "invalid configuration";
    return SAE_E_INVAL;
  }
  sae_ctx* ctx = new sae_ctx();
  const sae_status rc = create_impl(cfg, ctx);
  if (rc != SAE_OK) {               // free everything allocated so far; keep the message
    g_create_error = ctx->last_error.empty() ? "sae_create failed" : ctx->last_error;
    cudaDeviceSynchronize();
    for (void* p : ctx->allocs) cudaFree(p);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return SAE_OK;
}

sae_status sae_destroy(sae_ctx* ctx) {
  if (!ctx) return SAE_E_INVAL;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->ws) cudaFree(ctx->ws);
  for (int k = 0; k < 2; ++k) {
    if (ctx->stage[k]) cudaFree(ctx->stage[k]);
    if (ctx->ev_in[k]) cudaEventDestroy(ctx->ev_in[k]);
    if (ctx->ev_out[k]) cudaEventDestroy(ctx->ev_out[k]);
  }
  if (ctx->cs) cudaStreamDestroy(ctx->cs);
  delete ctx;
  return SAE_OK;
}

static sae_status scatter_params(sae_ctx* ctx, const sae_params* dev_in, uint32_t r0, uint32_t nr,
                                 cudaStream_t s) {
  k_params_commit<<<(nr + 255) / 256, 256, 0, s>>>(ctx->d, dev_in, r0, nr);
  ctx->launches += 1;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_set_params(sae_ctx* ctx, uint32_t replica, const sae_params* p, sae_stream st) {
  if (!ctx || !p || replica >= ctx->d.R) return SAE_E_INVAL;
  if (!(p->sigma[0] > 0.0) || !(p->sigma[1] > 0.0)) return SAE_E_INVAL;
  if (p->mode > SAE_MODE_TWO || (p->mode != SAE_MODE_SAE && !ctx->d.cand_smem)) {
    ctx->last_error = "baseline modes need a pool that fits one CTA's candidate buffer";
    return SAE_E_INVAL;
  }
  cudaStream_t s = (cudaStream_t)st;
  sae_params* tmp;
  CK(cudaMallocAsync(&tmp, sizeof(sae_params), s));
  CK(cudaMemcpyAsync(tmp, p, sizeof(sae_params), cudaMemcpyHostToDevice, s));
  sae_status rc = scatter_params(ctx, tmp, replica, 1, s);
  CK(cudaFreeAsync(tmp, s));
  if (rc == SAE_OK) CK(cudaStreamSynchronize(s));  // p is a host pointer
  return rc;
}

sae_status sae_params_gather(sae_ctx* ctx, sae_params* dev_out, sae_stream st) {
  if (!ctx || !dev_out) return SAE_E_INVAL;
  k_params_gather<<<(ctx->d.R + 255) / 256, 256, 0, (cudaStream_t)st>>>(ctx->d, dev_out);
  ctx->launches++;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_params_scatter(sae_ctx* ctx, const sae_params* dev_in, sae_stream st) {
  if (!ctx || !dev_in) return SAE_E_INVAL;
  return scatter_params(ctx, dev_in, 0, ctx->d.R, (cudaStream_t)st);
}

static BatchDev batch_dev(const sae_batch* b) {
  BatchDev x;
  std::memset(&x, 0, sizeof x);
  x.n = b->n;
  x.replica = b->replica;
  x.arrival = b->arrival;
  x.poff = b->prompt_off;
  x.plen = b->prompt_len;
  x.doff = b->decode_off;
  x.dlen = b->decode_len;
  x.tokens = b->tokens;
  x.types = b->types;
  x.flags = b->flags;
  x.spb = b->shared_prefix_blocks;
  return x;
}

// carve the per-batch workspace
static sae_status prepare(sae_ctx* ctx, const sae_batch* b, BatchDev& x, cudaStream_t s,
                          uint64_t total_blocks, bool runs = true) {
  const uint64_t n = b->n, R = ctx->d.R;
  const uint32_t ntile = (uint32_t)((n + SCAN_TILE - 1) / SCAN_TILE);
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  size_t need = al((n + 1) * 8) * 2 + al(ntile + 1) * 8 + al(total_blocks * 8) + al(total_blocks) * 3 +
                al(total_blocks * 4) * 2 + al(R * 4) * 2;
  if (need > ctx->ws_cap) {
    if (ctx->ws) CK(cudaFreeAsync(ctx->ws, s));
    ctx->ws = nullptr;
    size_t cap = need + need / 2;
    CK(cudaMallocAsync(&ctx->ws, cap, s));
    ctx->ws_cap = cap;
  }
  char* p = (char*)ctx->ws;
  auto take = [&](size_t bytes) { char* q = p; p += al(bytes); return (void*)q; };
  x.tb = total_blocks;
  uint64_t* cnt = (uint64_t*)take((n + 1) * 8);
  x.boff = (uint64_t*)take((n + 1) * 8);
  uint64_t* part = (uint64_t*)take((ntile + 1) * 8);
  x.h = (uint64_t*)take(total_blocks * 8);
  x.tau = (uint8_t*)take(total_blocks);
  x.ntok = (uint8_t*)take(total_blocks);
  x.q = (uint8_t*)take(total_blocks);
  x.slot = (int32_t*)take(total_blocks * 4);
  x.nrank = (int32_t*)take(total_blocks * 4);
  x.run_start = (uint32_t*)take(R * 4);
  x.run_end = (uint32_t*)take(R * 4);
  if (n == 0) return SAE_OK;
  k_nblocks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, ctx->d.B, cnt);
  k_scan_reduce<<<ntile, 1024, 0, s>>>(cnt, n, part);
  k_scan_parts<<<1, 32, 0, s>>>(part, ntile);
  k_scan_apply<<<ntile, 1024, 0, s>>>(cnt, n, part, x.boff, ntile);
  CK(cudaMemsetAsync(x.run_start, 0xFF, R * 4, s));
  CK(cudaMemsetAsync(x.run_end, 0, R * 4, s));
  if (runs) k_runs<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, ctx->d);
  cudaEvent_t h0 = nullptr, h1 = nullptr;
  if (ctx->prof) {
    CK(cudaEventCreate(&h0));
    CK(cudaEventCreate(&h1));
    CK(cudaEventRecord(h0, s));
  }
  k_hash<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(x, ctx->d);
  if (ctx->prof) {
    CK(cudaEventRecord(h1, s));
    ctx->prof_hash.push_back({h0, h1});
  }
  ctx->launches += 6;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_batch_blocks(sae_ctx* ctx, const sae_batch* b, uint64_t* total, sae_stream st) {
  if (!ctx || !b || !total) return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  const uint64_t n = b->n;
  if (n == 0) { *total = 0; return SAE_OK; }
  const uint32_t ntile = (uint32_t)((n + SCAN_TILE - 1) / SCAN_TILE);
  uint64_t *cnt, *part;
  CK(cudaMallocAsync(&cnt, (n + 1) * 8, s));
  CK(cudaMallocAsync(&part, (ntile + 1) * 8, s));
  BatchDev x = batch_dev(b);
  k_nblocks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, ctx->d.B, cnt);
  k_scan_reduce<<<ntile, 1024, 0, s>>>(cnt, n, part);
  k_scan_parts<<<1, 32, 0, s>>>(part, ntile);
  ctx->launches += 3;
  CK(cudaMemcpyAsync(total, part + ntile, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(cnt, s));
  CK(cudaFreeAsync(part, s));
  CK(cudaStreamSynchronize(s));
  return SAE_OK;
}

sae_status sae_admit_batch(sae_ctx* ctx, const sae_batch* b, sae_admit_out* o, sae_stream st) {
  if (!ctx || !b || !o) return SAE_E_INVAL;
  if (b->n && (!b->replica || !b->arrival || !b->prompt_off || !b->prompt_len || !b->decode_off ||
               !b->decode_len || !b->tokens || !b->types || !b->flags || !b->shared_prefix_blocks))
    return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  CK(cudaSetDevice(ctx->device));
  BatchDev x = batch_dev(b);
  sae_status rc = prepare(ctx, b, x, s, b->total_blocks);
  if (rc) return rc;
  if (b->n == 0) return SAE_OK;
  x.o_hit = o->hit_blocks;
  x.o_miss = o->miss_blocks;
  x.o_matched = o->matched_tokens;
  x.o_nvict = o->n_victims;
  x.o_voff = o->victim_off;
  x.o_vids = o->victim_ids;
  x.vcap = o->victim_ids ? o->victim_cap : ~0ull;
  if (o->victim_off) CK(cudaMemcpyAsync(o->victim_off, x.boff, (b->n + 1) * 8, cudaMemcpyDeviceToDevice, s));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->prof) {
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
  }
  uint32_t grid = ctx->d.R * ctx->d.GP;
  if (ctx->d.nchunk > 1) {            // task-split replay: a persistent grid, tasks from a counter
    CK(cudaMemsetAsync(ctx->d.taskctr, 0, 4, s));
    grid = (uint32_t)std::min<uint64_t>(ctx->coresident, (uint64_t)ctx->d.R * ctx->d.nchunk);
  }
  CK(launch_group(ctx->var, ctx->var.replay, grid, ctx->d.GP > 1, s, ctx->d, &x));
  ctx->launches++;
  if (ctx->prof) {
    CK(cudaEventRecord(e1, s));
    ctx->prof_ev.push_back({e0, e1});
  }
  CK(cudaGetLastError());
  if (o->block_hash) CK(cudaMemcpyAsync(o->block_hash, x.h, b->total_blocks * 8, cudaMemcpyDeviceToDevice, s));
  if (o->block_tau) CK(cudaMemcpyAsync(o->block_tau, x.tau, b->total_blocks, cudaMemcpyDeviceToDevice, s));
  return SAE_OK;
}

// End-to-end call with HOST buffers: H2D of the request arrays and of the token arena range,
// the replay, D2H of the outputs -- all stream-ordered on s (include/sae.h).
sae_status sae_admit_batch_host(sae_ctx* ctx, const sae_batch* hb, uint64_t tok_lo, uint64_t tok_hi,
                                uint32_t* tokens_dev, uint8_t* types_dev, sae_admit_out* ho,
                                uint64_t* h2d_bytes, uint64_t* d2h_bytes, sae_stream st) {
  if (!ctx || !hb || !ho || tok_hi < tok_lo) return SAE_E_INVAL;
  const uint64_t n = hb->n, tb = hb->total_blocks;
  if (n && (!tokens_dev || !types_dev || !hb->replica || !hb->arrival || !hb->prompt_off ||
            !hb->prompt_len || !hb->decode_off || !hb->decode_len || !hb->tokens || !hb->types ||
            !hb->flags || !hb->shared_prefix_blocks))
    return SAE_E_INVAL;
  if (n && ho->victim_ids && ho->victim_cap < tb) return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  CK(cudaSetDevice(ctx->device));
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  const uint64_t tbx = tb ? tb : 1;
  size_t need = al(n * 4) * 4 + al(n * 8) * 3 + al(n) + al(n * 4) * 4 + al((n + 1) * 8) + al(tbx * 4) +
                (ho->block_hash ? al(tbx * 8) : 0) + (ho->block_tau ? al(tbx) : 0) + 256;
  if (!ctx->cs) {
    CK(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&ctx->ev_in[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out[k], cudaEventDisableTiming));
      CK(cudaEventRecord(ctx->ev_out[k], s));
    }
  }
  const int k = ctx->slot;
  ctx->slot ^= 1;
  // at most two calls in flight: slot k's previous call (two calls ago) must be done -- its
  // host buffers are then free for the caller and its outputs final
  CK(cudaEventSynchronize(ctx->ev_out[k]));
  if (need > ctx->stage_cap[k]) {             // grow slot k (its last use is done)
    if (ctx->stage[k]) CK(cudaFree(ctx->stage[k]));
    ctx->stage[k] = nullptr;
    ctx->stage_cap[k] = 0;
    const size_t cap = need + need / 4;
    CK(cudaMalloc(&ctx->stage[k], cap));
    ctx->stage_cap[k] = cap;
  }
  // inputs on the copy stream once slot k is free: they overlap the previous call's replay
  CK(cudaStreamWaitEvent(ctx->cs, ctx->ev_out[k], 0));
  char* p = (char*)ctx->stage[k];
  auto take = [&](size_t bytes) { char* q = p; p += al(bytes); return (void*)q; };
  uint64_t hin = 0, hout = 0;
  auto h2d = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    hin += bytes;
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->cs) : cudaSuccess;
  };
  sae_batch db = *hb;
  db.replica = (const uint32_t*)take(n * 4);
  db.arrival = (const double*)take(n * 8);
  db.prompt_off = (const uint64_t*)take(n * 8);
  db.prompt_len = (const uint32_t*)take(n * 4);
  db.decode_off = (const uint64_t*)take(n * 8);
  db.decode_len = (const uint32_t*)take(n * 4);
  db.flags = (const uint8_t*)take(n);
  db.shared_prefix_blocks = (const uint32_t*)take(n * 4);
  CK(h2d((void*)db.replica, hb->replica, n * 4));
  CK(h2d((void*)db.arrival, hb->arrival, n * 8));
  CK(h2d((void*)db.prompt_off, hb->prompt_off, n * 8));
  CK(h2d((void*)db.prompt_len, hb->prompt_len, n * 4));
  CK(h2d((void*)db.decode_off, hb->decode_off, n * 8));
  CK(h2d((void*)db.decode_len, hb->decode_len, n * 4));
  CK(h2d((void*)db.flags, hb->flags, n));
  CK(h2d((void*)db.shared_prefix_blocks, hb->shared_prefix_blocks, n * 4));
  CK(h2d(tokens_dev + tok_lo, hb->tokens + tok_lo, (tok_hi - tok_lo) * 4));
  CK(h2d(types_dev + tok_lo, hb->types + tok_lo, tok_hi - tok_lo));
  db.tokens = tokens_dev;
  db.types = types_dev;
  CK(cudaEventRecord(ctx->ev_in[k], ctx->cs));
  CK(cudaStreamWaitEvent(s, ctx->ev_in[k], 0));     // the replay on s waits for its inputs
  sae_admit_out dout;
  std::memset(&dout, 0, sizeof dout);
  dout.hit_blocks = (uint32_t*)take(n * 4);
  dout.miss_blocks = (uint32_t*)take(n * 4);
  dout.matched_tokens = (uint32_t*)take(n * 4);
  dout.n_victims = (uint32_t*)take(n * 4);
  dout.victim_off = (uint64_t*)take((n + 1) * 8);
  dout.victim_ids = (uint32_t*)take(tbx * 4);
  dout.victim_cap = tbx;
  dout.block_hash = ho->block_hash ? (uint64_t*)take(tbx * 8) : nullptr;
  dout.block_tau = ho->block_tau ? (uint8_t*)take(tbx) : nullptr;
  sae_status rc = sae_admit_batch(ctx, &db, &dout, st);
  if (rc != SAE_OK) return rc;
  auto d2h = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst || !bytes) return cudaSuccess;
    hout += bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  };
  CK(d2h(ho->hit_blocks, dout.hit_blocks, n * 4));
  CK(d2h(ho->miss_blocks, dout.miss_blocks, n * 4));
  CK(d2h(ho->matched_tokens, dout.matched_tokens, n * 4));
  CK(d2h(ho->n_victims, dout.n_victims, n * 4));
  CK(d2h(ho->victim_off, dout.victim_off, n ? (n + 1) * 8 : 0));
  CK(d2h(ho->victim_ids, dout.victim_ids, tb * 4));
  CK(d2h(ho->block_hash, dout.block_hash, tb * 8));
  CK(d2h(ho->block_tau, dout.block_tau, tb));
  if (h2d_bytes) *h2d_bytes = hin;
  if (d2h_bytes) *d2h_bytes = hout;
  return SAE_OK;
}

sae_status sae_lookup(sae_ctx* ctx, const sae_batch* b, uint32_t* hit, sae_stream st) {
  if (!ctx || !b || !hit) return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  BatchDev x = batch_dev(b);
  sae_status rc = prepare(ctx, b, x, s, b->total_blocks);
  if (rc) return rc;
  if (b->n == 0) return SAE_OK;
  k_lookup<<<(unsigned)((b->n * 32ull + 255) / 256), 256, 0, s>>>(ctx->d, x, hit);
  ctx->launches++;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_evict(sae_ctx* ctx, uint32_t replica, uint32_t k, double now, uint32_t* vids,
                     uint32_t* n_out, sae_stream st) {
  if (!ctx || replica >= ctx->d.R || (k > 0 && !vids)) return SAE_E_INVAL;
  ctx->d.epoch++;
  void* args[] = {(void*)&ctx->d, (void*)&replica, (void*)&k, (void*)&now, (void*)&vids, (void*)&n_out};
  if (ctx->d.GP > 1)
    CK(cudaLaunchCooperativeKernel(ctx->var.evict, ctx->d.GP, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
  else
    CK(cudaLaunchKernel(ctx->var.evict, 1, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
  ctx->launches++;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_select(sae_ctx* ctx, uint32_t replica, uint32_t m, double now, uint32_t passes,
                      uint32_t* vids, uint32_t* n_out, sae_stream st) {
  if (!ctx || replica >= ctx->d.R || m > MSUB || passes == 0 || (m > 0 && !vids)) {
    if (ctx) ctx->last_error = "sae_select: bad replica, m > 96, passes == 0 or null victim buffer";
    return SAE_E_INVAL;
  }
  ctx->d.epoch++;
  void* args[] = {(void*)&ctx->d, (void*)&replica, (void*)&m, (void*)&now, (void*)&passes, (void*)&vids,
                  (void*)&n_out};
  if (ctx->d.GP > 1)
    CK(cudaLaunchCooperativeKernel(ctx->var.select, ctx->d.GP, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
  else
    CK(cudaLaunchKernel(ctx->var.select, 1, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
  ctx->launches++;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_update(sae_ctx* ctx, uint32_t replica, sae_stream st) {
  if (!ctx) return SAE_E_INVAL;
  uint32_t r0 = replica, r1 = replica + 1;
  if (replica == 0xFFFFFFFFu) { r0 = 0; r1 = ctx->d.R; }
  else if (replica >= ctx->d.R) return SAE_E_INVAL;
  // groups must be co-resident: update at most coresident/GP replicas per launch
  const uint32_t per = ctx->d.GP > 1 ? (uint32_t)std::max<uint64_t>(1, ctx->coresident / ctx->d.GP) : (r1 - r0);
  for (uint32_t a = r0; a < r1; a += per) {
    uint32_t b = std::min(r1, a + per);
    ctx->d.epoch++;
    void* args[] = {(void*)&ctx->d, (void*)&a, (void*)&b};
    if (ctx->d.GP > 1)
      CK(cudaLaunchCooperativeKernel(ctx->var.update, (b - a) * ctx->d.GP, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
    else
      CK(cudaLaunchKernel(ctx->var.update, b - a, ctx->var.nt, args, ctx->var.smem, (cudaStream_t)st));
    ctx->launches++;
  }
  CK(cudaGetLastError());
  return SAE_OK;
}

static sae_status take_sticky(sae_ctx* ctx, cudaStream_t s) {
  uint32_t e = 0;
  CK(cudaMemcpyAsync(&e, ctx->d.err, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (e) {
    CK(cudaMemsetAsync(ctx->d.err, 0, 4, s));
    CK(cudaStreamSynchronize(s));
    ctx->last_error = "device error " + std::to_string(-(int)e);
    return -(int)e;
  }
  return SAE_OK;
}

sae_status sae_sync(sae_ctx* ctx, sae_stream st) {
  if (!ctx) return SAE_E_INVAL;
  return take_sticky(ctx, (cudaStream_t)st);
}

sae_status sae_stats(sae_ctx* ctx, uint32_t replica, sae_replica_stats* out, sae_stream st) {
  if (!ctx || !out || replica >= ctx->d.R) return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  RState rs;
  unsigned long long* q5;
  CK(cudaMallocAsync(&q5, 5 * 8, s));
  CK(cudaMemsetAsync(q5, 0, 5 * 8, s));
  k_count_queues<<<64, 256, 0, s>>>(ctx->d, replica, q5);
  ctx->launches++;
  unsigned long long hq[5];
  CK(cudaMemcpyAsync(hq, q5, 5 * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&rs, ctx->d.st + replica, sizeof rs, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(q5, s));
  CK(cudaStreamSynchronize(s));
  std::memset(out, 0, sizeof *out);
  out->requests = rs.requests;
  out->blocks_looked_up = rs.blocks_looked_up;
  out->hit_blocks = rs.hit_blocks;
  out->hit_tokens = rs.hit_tokens;
  out->prompt_tokens = rs.prompt_tokens;
  out->evictions = rs.evictions;
  for (int i = 0; i < 4; ++i) out->evict_by_queue[i] = rs.evict_by_queue[i];
  for (int i = 0; i < 6; ++i) { out->evict_by_type[i] = rs.evict_by_type[i]; out->mae_by_type[i] = rs.mae_by_type[i]; }
  out->learner_firings = rs.learner_firings;
  out->eviction_rounds = rs.eviction_rounds;
  out->blocks_scored = rs.blocks_scored;
  out->blocks_scored_struct = rs.blocks_scored_struct;
  out->select_passes = rs.select_passes;
  out->select_cands = rs.select_cands;
  out->select_big = rs.select_big;
  for (int g = 0; g < 10; ++g) out->select_fail_seg[g] = rs.select_fail_seg[g];
  for (int g = 0; g < 16; ++g) out->phase_ns[g] = rs.tph[g];
  out->select_narrow = rs.select_narrow;
  out->select_raw = rs.select_raw;
  out->stage2_chunks = rs.stage2_chunks;
  {
    unsigned long long w = 0;
    CK(cudaMemcpy(&w, &ctx->d.ctl[replica].wscan_ns, 8, cudaMemcpyDeviceToHost));
    out->phase_ns[11] = w;
  }
  out->resident = hq[4];
  for (int i = 0; i < 4; ++i) out->resident_by_queue[i] = hq[i];
  out->E = rs.E;
  out->next_id = rs.next_id;
  out->gseq = rs.gseq;
  out->now = rs.now;
  for (int t = 0; t < 5; ++t) {
    out->ts_ev[t] = rs.ts_ev[t]; out->ts_mae[t] = rs.ts_mae[t];
    out->ts_hit[t] = rs.ts_hit[t]; out->ts_acc[t] = rs.ts_acc[t];
  }
  for (int q = 0; q < 3; ++q) { out->qh[q] = rs.qh[q]; out->qe[q] = rs.qe[q]; }
  for (int i = 0; i < 16; ++i) { out->pb_hit[i] = rs.pb_hit[i]; out->pb_acc[i] = rs.pb_acc[i]; }
  out->iv_len[0] = rs.iv_len[0];
  out->iv_len[1] = rs.iv_len[1];
  out->traj_count = rs.traj_n;
  out->params = rs.par;
  return take_sticky(ctx, s);
}

sae_status sae_counters_device(sae_ctx* ctx, sae_counters* dev_out, sae_stream st) {
  if (!ctx || !dev_out) return SAE_E_INVAL;
  k_counters<<<1, 32, 0, (cudaStream_t)st>>>(ctx->d, dev_out);
  ctx->launches++;
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_get_traj(sae_ctx* ctx, uint32_t replica, sae_traj* out, uint64_t cap, uint64_t* n_out,
                        sae_stream st) {
  if (!ctx || replica >= ctx->d.R) return SAE_E_INVAL;
  cudaStream_t s = (cudaStream_t)st;
  RState rs;
  CK(cudaMemcpyAsync(&rs, ctx->d.st + replica, sizeof rs, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t tc = ctx->d.traj_cap;
  uint64_t n = rs.traj_n < tc ? rs.traj_n : tc;
  if (!out) {  // query the number available
    if (n_out) *n_out = n;
    return SAE_OK;
  }
  if (n > cap) n = cap;
  if (n_out) *n_out = n;
  if (n == 0) return SAE_OK;
  std::vector<sae_traj> all(tc);
  CK(cudaMemcpyAsync(all.data(), ctx->d.traj + (uint64_t)replica * tc, tc * sizeof(sae_traj),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  uint64_t first = rs.traj_n > tc ? rs.traj_n - tc : 0;
  for (uint64_t i = 0; i < n; ++i) out[i] = all[(first + i) % tc];
  return SAE_OK;
}

const char* sae_last_error(const sae_ctx* ctx) { return ctx ? ctx->last_error.c_str() : g_create_error.c_str(); }

sae_status sae_gen_tokens(uint64_t seed, uint64_t n_pieces, const uint64_t* stream, const uint64_t* start,
                          const uint32_t* len, const uint64_t* dst, const uint8_t* type, uint32_t* tokens,
                          uint8_t* types, sae_stream st) {
  sae_ctx* ctx = nullptr;
  if (n_pieces == 0) return SAE_OK;
  unsigned grid = (unsigned)(n_pieces < 65535ull * 8 ? n_pieces : 65535ull * 8);
  k_gen_tokens<<<grid, 128, 0, (cudaStream_t)st>>>(seed, n_pieces, stream, start, len, dst, type, tokens, types);
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_priority(const sae_params* params, double dt_eps, double z_cut, uint64_t n,
                        const uint8_t* q, const uint8_t* tau, const double* dt_in, const uint32_t* ob,
                        const uint32_t* omax, double* out, sae_stream st) {
  sae_ctx* ctx = nullptr;
  if (!params || (n && (!q || !tau || !dt_in || !ob || !omax || !out))) return SAE_E_INVAL;
  if (n == 0) return SAE_OK;
  k_priority<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)st>>>(*params, dt_eps, z_cut, n, q, tau,
                                                                        dt_in, ob, omax, out);
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_characterize(sae_ctx* ctx, const sae_batch* b, const uint32_t* session, const uint32_t* turn,
                            const uint8_t* single_turn, sae_char_stats* host_out, sae_stream st) {
  if (!ctx || !b || !host_out) return SAE_E_INVAL;
  if (b->n && (!b->arrival || !b->prompt_off || !b->prompt_len || !b->decode_off || !b->decode_len ||
               !b->tokens || !b->types || !session || !turn || !single_turn))
    return SAE_E_INVAL;
  std::memset(host_out, 0, sizeof *host_out);
  if (b->n == 0) return SAE_OK;
  cudaStream_t s = (cudaStream_t)st;
  CK(cudaSetDevice(ctx->device));
  BatchDev x = batch_dev(b);
  sae_status rc = prepare(ctx, b, x, s, b->total_blocks, false);   // K1 hashes + tau
  if (rc) return rc;
  uint64_t slots = 1;
  while (slots < 2ull * (b->total_blocks ? b->total_blocks : 1)) slots <<= 1;
  if (slots > (1ull << 31)) return SAE_E_INVAL;
  CharDev c;
  CK(cudaMallocAsync(&c.k1, slots * 8, s));
  CK(cudaMallocAsync(&c.v1, slots * 8, s));
  CK(cudaMallocAsync(&c.k2, slots * 8, s));
  CK(cudaMallocAsync(&c.v2, slots * 8, s));
  CK(cudaMallocAsync(&c.out, 58 * 8, s));
  CK(cudaMemsetAsync(c.k1, 0xFF, slots * 8, s));
  CK(cudaMemsetAsync(c.v1, 0xFF, slots * 8, s));
  CK(cudaMemsetAsync(c.k2, 0xFF, slots * 8, s));
  CK(cudaMemsetAsync(c.v2, 0xFF, slots * 8, s));
  CK(cudaMemsetAsync(c.out, 0, 58 * 8, s));
  c.mask = (uint32_t)(slots - 1);
  c.session = session; c.turn = turn; c.single = single_turn;
  const unsigned grid = (unsigned)((b->n * 32ull + 255) / 256);
  k_char_insert<<<grid, 256, 0, s>>>(x, c);
  k_char_count<<<grid, 256, 0, s>>>(x, c, ctx->d.B);
  ctx->launches += 2;
  CK(cudaGetLastError());
  static_assert(sizeof(sae_char_stats) == 58 * 8, "sae_char_stats layout");
  CK(cudaMemcpyAsync(host_out, c.out, 58 * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(c.k1, s));
  CK(cudaFreeAsync(c.v1, s));
  CK(cudaFreeAsync(c.k2, s));
  CK(cudaFreeAsync(c.v2, s));
  CK(cudaFreeAsync(c.out, s));
  CK(cudaStreamSynchronize(s));
  return take_sticky(ctx, s);
}

uint64_t sae_launch_count(const sae_ctx* ctx) { return ctx ? ctx->launches : 0; }

sae_status sae_layout(const sae_ctx* ctx, sae_layout_info* o) {
  if (!ctx || !o) return SAE_E_INVAL;
  int nsm = 1;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  o->threads = ctx->var.nt;
  o->ctas_per_replica = ctx->d.GP;
  o->coresident = (uint32_t)ctx->coresident;
  o->ctas_per_sm = (uint32_t)(ctx->coresident / (uint64_t)(nsm > 0 ? nsm : 1));
  o->chunks = ctx->d.nchunk;
  o->cand_global = ctx->d.cpriv != nullptr ? 1u : 0u;
  return SAE_OK;
}

sae_status sae_params_point_mean(const sae_params* all_dev, uint32_t n_total, uint32_t n_points,
                                 sae_params* out_dev, sae_stream st) {
  sae_ctx* ctx = nullptr;
  if (!all_dev || !out_dev || n_points == 0 || n_total % n_points != 0) return SAE_E_INVAL;
  k_point_mean<<<(n_total + 255) / 256, 256, 0, (cudaStream_t)st>>>(all_dev, n_total, n_points, out_dev);
  CK(cudaGetLastError());
  return SAE_OK;
}

sae_status sae_profile(sae_ctx* ctx, int enable) {
  if (!ctx) return SAE_E_INVAL;
  ctx->prof = enable != 0;
  return SAE_OK;
}

static sae_status read_events(sae_ctx* ctx, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& ev,
                              double* ms_total, uint64_t* n_launches) {
  double tot = 0.0;
  uint64_t n = 0;
  for (auto& pr : ev) {
    CK(cudaEventSynchronize(pr.second));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
    ++n;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  ev.clear();
  if (ms_total) *ms_total = tot;
  if (n_launches) *n_launches = n;
  return SAE_OK;
}

sae_status sae_profile_read_hash(sae_ctx* ctx, double* ms_total, uint64_t* n_launches) {
  if (!ctx) return SAE_E_INVAL;
  return read_events(ctx, ctx->prof_hash, ms_total, n_launches);
}

sae_status sae_profile_read(sae_ctx* ctx, double* ms_total, uint64_t* n_launches) {
  if (!ctx) return SAE_E_INVAL;
  double tot = 0.0;
  uint64_t n = 0;
  for (auto& pr : ctx->prof_ev) {
    CK(cudaEventSynchronize(pr.second));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
    ++n;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  ctx->prof_ev.clear();
  if (ms_total) *ms_total = tot;
  if (n_launches) *n_launches = n;
  return SAE_OK;
}

}  // extern "C"
