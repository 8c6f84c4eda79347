// replay_impl.cuh -- the replay kernels (K2-K5) and their CTA-level building blocks,
// compiled twice by sae.cu inside namespaces sae::v512 (NT = 512 threads, 4096-entry
// candidate buffer: multi-CTA groups and pools up to 4096 blocks) and sae::v256 (NT = 256,
// 2560-entry buffer: two single-CTA replicas fit one SM, e.g. C5's 2304-block replicas).
// The including namespace defines NT, NW and CAND_MAX; everything else comes from sae::.
// (No include guard: included once per variant.)

// ---------------------------------------------------------------------------
// Block-wide helpers (NT threads)
// ---------------------------------------------------------------------------
// CTA barrier in its non-aligned form (barrier.sync): every thread arrives individually.
// bar.sync / __syncthreads() is the .aligned form, which presumes that a warp reaches it
// converged; the replay loops diverge lanes (hash probes, fdlibm calls) right before
// block-wide steps, and with the aligned form a lane that reconverged late was observed to
// drift one barrier generation behind its block ("CTA barriers").
__device__ __forceinline__ void cta_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }
// exclusive scan of up to 3 flags per thread; returns ranks; totals in tot[3]
__device__ __forceinline__ void block_scan3(uint32_t a, uint32_t b, uint32_t c, uint32_t& ra,
                                            uint32_t& rb, uint32_t& rc, uint32_t* tot,
                                            uint32_t* wsum /* [3*NW] smem */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t ba = __ballot_sync(~0u, a), bb = __ballot_sync(~0u, b), bc = __ballot_sync(~0u, c);
  uint32_t lm = (1u << lane) - 1u;
  ra = __popc(ba & lm); rb = __popc(bb & lm); rc = __popc(bc & lm);
  if (lane == 0) { wsum[w] = __popc(ba); wsum[NW + w] = __popc(bb); wsum[2 * NW + w] = __popc(bc); }
  cta_sync();
  uint32_t oa = 0, ob = 0, oc = 0, ta = 0, tb = 0, tc = 0;
  for (int i = 0; i < NW; ++i) {
    uint32_t x = wsum[i], y = wsum[NW + i], z = wsum[2 * NW + i];
    if (i < w) { oa += x; ob += y; oc += z; }
    ta += x; tb += y; tc += z;
  }
  ra += oa; rb += ob; rc += oc;
  tot[0] = ta; tot[1] = tb; tot[2] = tc;
  cta_sync();
}

__device__ __forceinline__ bool cand_less(const Cand& a, const Cand& b) {
  uint32_t sa = a.ss >> 28, sb = b.ss >> 28;
  if (sa != sb) return sa < sb;
  if (a.k0 != b.k0) return a.k0 < b.k0;
  if (a.k1 != b.k1) return a.k1 < b.k1;
  return a.k2 < b.k2;
}

// bitonic sort of cand[0..N), N a power of two, ascending by (seg, k0, k1, k2)
__device__ void block_sort(Cand* cand, int N) {
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          Cand x = cand[i], y = cand[ixj];
          bool up = (i & k) == 0;
          if (cand_less(y, x) == up) { cand[i] = y; cand[ixj] = x; }
        }
      }
      cta_sync();
    }
  }
}

__device__ __forceinline__ Cand shfl_cand(const Cand& x, int j) {
  Cand y;
  y.k0 = __shfl_xor_sync(~0u, x.k0, j);
  y.k1 = __shfl_xor_sync(~0u, x.k1, j);
  y.k2 = __shfl_xor_sync(~0u, x.k2, j);
  y.ss = __shfl_xor_sync(~0u, x.ss, j);
  y.seg = __shfl_xor_sync(~0u, x.seg, j);
  return y;
}

// Bitonic sort of a[0..N) (N a power of two, 32 <= N <= E*NT) with E elements per
// thread held in registers: element e of thread t is index e*NT + t.  Strides >= NT
// stay inside a thread, strides < 32 use warp shuffles, the rest go through smem.
template <int E>
__device__ void sort_reg(Cand* a, int N) {
  const int t = threadIdx.x;
  Cand x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * NT + t;
    if (i < N) {
      x[e] = a[i];
    } else {
      x[e].k0 = ~0ull; x[e].k1 = ~0ull; x[e].k2 = ~0u; x[e].ss = ~0u; x[e].seg = 15;
    }
  }
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= NT) {
        const int pe = j / NT;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & pe) == 0 && (e | pe) < E) {
            const int i = e * NT + t;
            const bool up = (i & k) == 0;
            Cand& lo = x[e];
            Cand& hi = x[e | pe];
            if (cand_less(hi, lo) == up) { Cand tmp = lo; lo = hi; hi = tmp; }
          }
        }
        continue;
      }
      Cand y[E];
      if (j >= 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) if (e * NT + t < N) a[e * NT + t] = x[e];
        cta_sync();
#pragma unroll
        for (int e = 0; e < E; ++e) y[e] = (e * NT + t < N) ? a[(e * NT + t) ^ j] : x[e];
        cta_sync();
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) y[e] = shfl_cand(x[e], j);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = e * NT + t;
        const bool up = (i & k) == 0, lower = (i & j) == 0;
        const bool take_y = (lower == up) ? cand_less(y[e], x[e]) : cand_less(x[e], y[e]);
        if (take_y && i < N) x[e] = y[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) if (e * NT + t < N) a[e * NT + t] = x[e];
  cta_sync();
}

__device__ void sort_cands(Cand* a, int N) {
  if (N <= NT) sort_reg<1>(a, N);
  else if (N <= 2 * NT) sort_reg<2>(a, N);
  else if (N <= 4 * NT) sort_reg<4>(a, N);
  else block_sort(a, N);
}

// ---------------------------------------------------------------------------
// Replay CTA: shared state
// ---------------------------------------------------------------------------
struct Smem {
  RState st;
  double cw[3][5];         // alpha_q * w_tau per scored queue (CHAT, AGENT, STRUCT)
  uint32_t wsum[16 * NW];
  uint32_t tot[3];
  uint32_t cnt[16], start[16], segtot[16], used[16];
  uint32_t fail, ncand;
  int32_t h;
  uint32_t npin, matched;
  uint64_t k, admit;
  uint64_t pfx[16], pmask[16];
  uint32_t below[16], target[16], binc[16];
  unsigned long long kmin[16];
  unsigned long long drefs[16], dors[16];  // radix_select: AND / OR of each class's keys
  uint32_t nv, nw;          // nw: this CTA's candidates awaiting finalize_key (global mode)
  uint32_t cseq, wcmd;      // leader: commands posted this launch; worker: command to run
  uint32_t gbase;           // worker: this CTA's reservation in the group candidate buffer
  uint32_t fin;             // 1: the scored candidates carry their exact keys (finalize_key ran)
  uint32_t pincnt[16];      // leader: this round's pinned blocks per segment
  unsigned long long thr64[16];   // candidacy table of the current scan: keys (EF, multi-turn)
  uint32_t thrS[1024];            // STRUCT: upper 32 bits of a bound on obits(last), per (tau, q8)
  __align__(16) uint32_t rhist[NSEG * 256];   // radix-select histograms (one 256-bin digit per
                                // segment); worker scan: its finished candidate records
  __align__(8) uint64_t mbar[24];  // bulk-copy stage barriers (worker scan pipeline): full[12], empty[12]
  uint64_t wt_pick, wt_end;        // worker: command pickup / stream end times (SAE_WORKER_TIMERS)
  uint64_t wthr[16], wpfx[16], wpmask[16];   // worker copies of the leader's command parameters
  double wcw[15], wmu[2], wsg[2], ww[5];
  double wnow, wgam;        // worker copies of the scan's time and gamma
  uint32_t wmode, wstamp;
};

struct Ctx {               // per-CTA view of one replica (group)
  const Dev* d;
  Smem* s;
  Cand* cand;
  Cand* vbuf;              // [VCAP] victims staging
  GroupCtl* ctl;
  uint32_t r, rank, GP;
  uint64_t base;           // r * C
  const uint64_t* pf_h;    // leader of a group: the next request's block hashes (prefetched
  uint32_t pf_n;           // into L2 while the workers scan), count
};

__device__ void recompute_cw(Smem& s) {
  if (threadIdx.x < 15) {
    int q = threadIdx.x / 5, t = threadIdx.x % 5;
    s.cw[q][t] = __dmul_rn(s.st.par.alpha[q], s.st.par.w[t]);
  }
}

__device__ __forceinline__ uint32_t seg_of(uint32_t q, uint32_t tau) {
  return q == Q_EF ? 0u : (q == Q_STRUCT ? 9u + (tau & 3u) : 1u + (q - 1u) * 4u + (tau & 3u));
}
// the key a segment's threshold applies to: (last) for multi-turn classes, k0 otherwise
__device__ __forceinline__ uint64_t seg_key(const Cand& x) {
  return (x.seg >= 1 && x.seg <= 8) ? x.k1 : x.k0;
}
__device__ __forceinline__ void part_range(uint64_t n, uint32_t rank, uint32_t GP, uint64_t& lo,
                                           uint64_t& hi) {
  lo = n * rank / GP;
  hi = n * (rank + 1) / GP;
}

// ---------------------------------------------------------------------------
// Group command channel (GP CTAs of one replica, co-resident by cooperative launch).
// The leader publishes command number seq of this launch as one 64-bit word
// (epoch:24 | seq:32 | cmd:8) with a release store after its parameters; workers poll it
// with acquire loads, run their partition and count themselves done on a cumulative
// counter the leader waits on.  One hop each way (no all-to-all barrier).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long cmd_tag(uint32_t epoch, uint32_t seq) {
  return ((unsigned long long)(epoch & 0xFFFFFFu) << 32) | seq;
}

// Parameters of a scan, from the leader's smem (leader) or the control block (workers).
struct ScanP {
  double now, dt_eps, z_cut, gamma;
  uint32_t stamp;
  uint32_t mode;           // SAE_MODE_* (baselines key every block differently, see sae.h)
  const double* w;         // [5] token-type weights (Token-Weight-Only)
  const unsigned long long* thr;
  const double* cw;        // [3][5]
  const double* mu;
  const double* sg;
};

// One pass over slots [lo, hi) of the replica's SoA: segment + key of every resident,
// unpinned block (a4); those at or below the segment's threshold become candidates.
// Each thread handles 4 consecutive slots per step with 128-bit cache-global loads
// (meta, id, last; p_struct only for STRUCT blocks); per-segment counts accumulate in
// registers (16-bit fields) and are reduced once per pass.  Counts go to smem
// (segtot, cnt); candidates to smem (cand_smem) or the group's global buffer.

// Candidacy table of one scan pass (a4), built by every scanning CTA from the pass
// parameters: a block is a candidate iff its key is at or below its table entry.
//  * EF / multi-turn class: entry = the segment's carried threshold (key (ntok, id) / obits(last)).
//  * STRUCT class tau, bound q8: P = c * p / dt with p >= p_lo(q8), so P <= T implies
//    dt >= A = c * p_lo / T, i.e. last <= now - A (or any block if A <= eps).  The entry is
//    the upper 32 bits of obits(now - A * (1 - 2^-20)) rounded up: a superset of the
//    blocks with P <= T (a non-candidate has P > T * (1 + 2^-20), far beyond rounding).
// Exact Eq.(1)-(3) scores of the (few) candidates are computed afterwards by finalize_key.
__device__ void build_thr_table(Smem& s, const ScanP& P) {
  const int tid = threadIdx.x;
  if (tid < 16) s.thr64[tid] = tid < NSEG ? P.thr[tid] : 0ull;
  const float gamf = (float)P.gamma;
  for (int e = tid; e < 1024; e += NT) {
    const int tau = e >> 8;
    const uint32_t q8 = (uint32_t)(e & 255);
    const uint64_t T = P.thr[9 + tau];
    uint32_t ent = 0xFFFFFFFFu;
    if (T != ~0ull) {
      const double Tp = from_obits(T);
      const double pl = p_struct_lo8(q8, gamf);
      const double num = __dmul_rn(P.cw[10 + tau], pl);
      if (num > 0.0) {
        const double A = __dmul_rn(__ddiv_rn(num, Tp), 1.0 - 0x1p-20);   // Tp = 0: A = inf
        if (A > P.dt_eps) {
          const double L = __dsub_rn(P.now, A);
          const double Lu = __dadd_rn(__dadd_rn(L, fabs(L) * 0x1p-30), 0x1p-30);
          ent = (uint32_t)(obits(Lu) >> 32);
        }
      }
    }
    s.thrS[e] = ent;
  }
}
__device__ __forceinline__ bool cand_test(const Smem& s, uint32_t meta, uint64_t key) {
  const uint32_t tix = meta_tix(meta);
  return tix < 16u ? key <= s.thr64[tix] : (uint32_t)(key >> 32) <= s.thrS[tix - 16u];
}
// The candidate record of a block (exact keys of scored ones are set by finalize_key).
__device__ __forceinline__ Cand make_cand(uint32_t meta, uint64_t key, uint32_t sl) {
  const uint32_t q = meta_q(meta);
  Cand x;
  x.ss = sl | ((q == Q_EF ? 0u : 1u) << 28);
  x.seg = seg_of_tix(meta_tix(meta));
  x.k0 = q == Q_EF ? key : ~0ull;    // scored: set by finalize_key (until then after every EF key)
  x.k1 = q == Q_EF ? 0ull : key;
  x.k2 = 0;
  x.pad = 0;
  return x;
}

// Exact score of a scored candidate: Eq.(1) survival (multi-turn) or Eq.(2) (STRUCT),
// then Eq.(3) P = ((alpha_q * w_tau) * p) / dt, fixed op order (SURVEY c.4).
__device__ __forceinline__ void finalize_key(const Dev& d, uint64_t base, const ScanP& P, Cand& x) {
  if (x.seg == 0 || x.seg >= 16) return;
  x.k2 = __ldcg(d.bid + base + (x.ss & SLOT_MASK));
  const double last = from_obits(x.k1);
  double dt = __dsub_rn(P.now, last);
  if (dt < P.dt_eps) dt = P.dt_eps;
  if (P.mode != SAE_MODE_SAE) {        // baselines (sae.h): (key, last, id) with key =
    if (P.mode == SAE_MODE_LRU) {      //   last                       (LRU)
      x.k0 = x.k1;
    } else if (P.mode == SAE_MODE_LFU) {   // accesses               (LFU)
      x.k0 = (uint64_t)__ldcg(d.bacc + base + (x.ss & SLOT_MASK));
    } else {                           //   w_tau / dt, decode as CoT  (Token-Weight-Only)
      const uint32_t tau = meta_tau(__ldcg(d.bmeta + base + (x.ss & SLOT_MASK)));
      x.k0 = obits(__ddiv_rn(P.w[tau < 4 ? tau : 4], dt));
    }
    return;
  }
  if (x.seg <= 8) {
    const uint32_t q = 1 + (x.seg - 1) / 4, tau = (x.seg - 1) & 3;
    const double p = survival(dt, P.mu[q - 1], P.sg[q - 1], P.z_cut);
    x.k0 = obits(__ddiv_rn(__dmul_rn(P.cw[(q - 1) * 5 + tau], p), dt));
  } else {
    const uint32_t tau = x.seg - 9;
    const uint64_t gi = base + (x.ss & SLOT_MASK);
    const double ps = p_struct(__ldcg(d.bob + gi), __ldcg(d.bomax + gi), P.gamma);
    x.k0 = obits(__ddiv_rn(__dmul_rn(P.cw[10 + tau], ps), dt));
  }
}

// The scanning CTA keeps the positions of its scored candidates in smem (reusing the
// radix histogram area) and scores them exactly after streaming (no transcendental inside
// the streaming loop); overflow is scored in place.
constexpr uint32_t WCAP = NSEG * 256;
constexpr uint32_t WCAPC = (uint32_t)(NSEG * 256 * 4 / sizeof(Cand));   // records in the same area
constexpr uint32_t WCAP4 = WCAP / 4;   // bulk scan: (slot, meta, key lo, key hi) records
__device__ __forceinline__ void note_cand(Ctx& c, const ScanP& P, Cand* gdst, uint32_t pos) {
  const uint32_t w = atomicAdd(&c.s->nw, 1u);
  if (w < WCAP) {
    c.s->rhist[w] = pos;
  } else {
    Cand x = gdst[pos];
    finalize_key(*c.d, c.base, P, x);
    gdst[pos].k0 = x.k0;
    gdst[pos].k2 = x.k2;
  }
}
__device__ void finalize_noted(Ctx& c, const ScanP& P, Cand* gdst) {
  const uint32_t n = min(c.s->nw, WCAP);
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    const uint32_t pos = c.s->rhist[i];
    Cand x = gdst[pos];
    finalize_key(*c.d, c.base, P, x);
    gdst[pos].k0 = x.k0;
    gdst[pos].k2 = x.k2;
  }
}

// One pass over slots [lo, hi) of the replica's SoA with 128-bit loads, 4 consecutive slots
// per thread per step (software-pipelined one step ahead): candidacy by the table; the
// candidates go to smem (cand_smem) or the group's global buffer, counted per segment in
// s.cnt.  Exact scores after the stream.
__device__ void scan_range(Ctx& c, uint64_t lo, uint64_t hi, const ScanP& P) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool gm = !d.cand_smem;
  Cand* gdst = gm ? d.gcand + c.base : nullptr;
  const bool vec = ((c.base + lo) & 3u) == 0;
  uint32_t mt[4];
  uint64_t kt[4];
  auto load = [&](uint64_t s0, uint32_t (&m)[4], uint64_t (&k)[4]) {
    if (vec && s0 + 3 < hi && !gm) {   // single-CTA replica: the SoA is private -> L1-cached loads
      const uint4 m4 = *reinterpret_cast<const uint4*>(d.bmeta + c.base + s0);
      const ulonglong2 k0 = *reinterpret_cast<const ulonglong2*>(d.bkey + c.base + s0);
      const ulonglong2 k1 = *reinterpret_cast<const ulonglong2*>(d.bkey + c.base + s0 + 2);
      m[0] = m4.x; m[1] = m4.y; m[2] = m4.z; m[3] = m4.w;
      k[0] = k0.x; k[1] = k0.y; k[2] = k1.x; k[3] = k1.y;
    } else if (vec && s0 + 3 < hi) {
      const uint4 m4 = __ldcg(reinterpret_cast<const uint4*>(d.bmeta + c.base + s0));
      const ulonglong2 k0 = __ldcg(reinterpret_cast<const ulonglong2*>(d.bkey + c.base + s0));
      const ulonglong2 k1 = __ldcg(reinterpret_cast<const ulonglong2*>(d.bkey + c.base + s0 + 2));
      m[0] = m4.x; m[1] = m4.y; m[2] = m4.z; m[3] = m4.w;
      k[0] = k0.x; k[1] = k0.y; k[2] = k1.x; k[3] = k1.y;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = s0 + u < hi;
        m[u] = ok ? __ldcg(d.bmeta + c.base + s0 + u) : 0u;
        k[u] = ok ? __ldcg(d.bkey + c.base + s0 + u) : 0ull;
      }
    }
  };
  uint64_t s0 = lo + 4ull * tid;
  if (s0 < hi) load(s0, mt, kt);
  else { mt[0] = mt[1] = mt[2] = mt[3] = 0; }
  for (uint64_t i0 = lo; i0 < hi; i0 += 4 * NT) {
    const uint64_t sn = s0 + 4ull * NT;
    uint32_t mn[4] = {0, 0, 0, 0};
    uint64_t kn[4] = {0, 0, 0, 0};
    if (sn < hi) load(sn, mn, kn);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t meta = s0 < hi ? mt[u] : 0u;
      const bool take = (meta & (M_LIVE | M_PIN)) == M_LIVE && cand_test(s, meta, kt[u]);
      if (gm) {
        const uint32_t bal = __ballot_sync(~0u, take);
        if (bal) {
          uint32_t basep = 0;
          if (lane == 0) basep = atomicAdd(&c.ctl->ncand, (unsigned)__popc(bal));
          basep = __shfl_sync(~0u, basep, 0);
          if (take) {
            const uint32_t pos = basep + __popc(bal & ((1u << lane) - 1u));
            const Cand x = make_cand(meta, kt[u], (uint32_t)(s0 + u));
            atomicAdd(&s.cnt[x.seg], 1u);
            gdst[pos] = x;
            if (x.seg != 0) note_cand(c, P, gdst, pos);
          }
        }
      } else {
        const uint32_t bal = __ballot_sync(~0u, take);
        if (bal) {
          uint32_t basep = 0;
          if (lane == 0) basep = atomicAdd(&s.ncand, (unsigned)__popc(bal));
          basep = __shfl_sync(~0u, basep, 0);
          if (take) {
            const Cand x = make_cand(meta, kt[u], (uint32_t)(s0 + u));
            atomicAdd(&s.cnt[x.seg], 1u);
            c.cand[basep + __popc(bal & ((1u << lane) - 1u))] = x;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { mt[u] = mn[u]; kt[u] = kn[u]; }
    s0 = sn;
  }
  cta_sync();
  if (gm) {
    finalize_noted(c, P, gdst);
  } else {
    // private pool: exact scores are computed lazily by select_chunk, only when the EF
    // candidates cannot cover the chunk (Stage 2 needed)
    if (tid == 0) s.fin = 0;
  }
}

// ---- bulk asynchronous copies (cp.async.bulk, completion on an mbarrier) -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// same, with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_pol(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(uint32_t which) {
  uint64_t p;
  if (which == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// (Static equal slices per worker.  Tiles handed out dynamically from one group counter were
//  measured slower: k_select pass 74.1 vs 66 us on C4x, worker stream 42 vs 37 us.)
// Worker scan over [lo, hi) (lo a multiple of 4, replica base 16-byte aligned): the two
// scan columns (meta u32, key u64: 12 B per slot) are streamed tile by tile into shared
// memory by bulk asynchronous copies, BSTAGES tiles in flight, and scored from shared
// memory.  Stage reuse is tracked per stage by a "full" mbarrier (transaction bytes) and an
// "empty" mbarrier (one arrival per warp), so warps never wait for each other: only the
// producer thread (thread 0) waits for a stage to drain before refilling it.  Same outputs
// as scan_range.
#ifndef SAE_BTILE
#define SAE_BTILE 4096   // measured per c4x pass: 1024 x 10 stages 63.5 us, 2048 x 5 45.2, 3072 x 3 40.4, 4096 x 2 38.1
#endif
// (a variant whose buffer cannot hold two tiles of SAE_BTILE falls back to 2048-slot tiles)
constexpr int BTILE = (SAE_BTILE * 12 * 2 <= CAND_MAX * (int)sizeof(Cand)) ? SAE_BTILE : 2048;
constexpr uint32_t BTILE_BYTES = BTILE * (4 + 8);
constexpr int BSTAGES = (int)((CAND_MAX * sizeof(Cand)) / BTILE_BYTES) < 12
                            ? (int)((CAND_MAX * sizeof(Cand)) / BTILE_BYTES) : 12;
static_assert(BSTAGES >= 2, "bulk scan needs two stages");
__device__ void scan_bulk_begin(Ctx& c, uint64_t lo, uint64_t hi) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  if (threadIdx.x != 0) return;
  unsigned char* buf = reinterpret_cast<unsigned char*>(c.cand);
  const uint64_t ntiles = (hi - lo + BTILE - 1) / BTILE;
  uint64_t* full = &s.mbar[0];
  uint64_t* empty = &s.mbar[12];
  for (int st = 0; st < BSTAGES; ++st) { mbar_init(&full[st], 1); mbar_init(&empty[st], NW); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint64_t pol = d.scan_l2 ? l2_policy(d.scan_l2) : 0ull;
  for (uint64_t t = 0; t < ntiles && t < (uint64_t)BSTAGES; ++t) {
    const uint64_t t0 = lo + t * BTILE;
    const uint32_t n4 = ((uint32_t)min((uint64_t)BTILE, hi - t0) + 3) & ~3u;
    unsigned char* b = buf + (size_t)t * BTILE_BYTES;
    mbar_expect_tx(&full[t], n4 * 12u);
    if (d.scan_l2) {
      bulk_g2s_pol(b, d.bmeta + c.base + t0, n4 * 4u, &full[t], pol);
      bulk_g2s_pol(b + BTILE * 4, d.bkey + c.base + t0, n4 * 8u, &full[t], pol);
    } else {
      bulk_g2s(b, d.bmeta + c.base + t0, n4 * 4u, &full[t]);
      bulk_g2s(b + BTILE * 4, d.bkey + c.base + t0, n4 * 8u, &full[t]);
    }
  }
}
__device__ void scan_range_bulk(Ctx& c, uint64_t lo, uint64_t hi, const ScanP& P) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  const int tid = threadIdx.x, lane = tid & 31;
  Cand* gdst = d.gcand + c.base;
  unsigned char* buf = reinterpret_cast<unsigned char*>(c.cand);
  const uint64_t ntiles = (hi - lo + BTILE - 1) / BTILE;
  uint64_t* full = &s.mbar[0];
  uint64_t* empty = &s.mbar[12];
  auto issue_tile = [&](uint64_t t) {
    const int st = (int)(t % BSTAGES);
    const uint64_t t0 = lo + t * BTILE;
    const uint32_t n = (uint32_t)min((uint64_t)BTILE, hi - t0);
    const uint32_t n4 = (n + 3) & ~3u;                 // 16-byte multiple (SoA is padded)
    unsigned char* b = buf + (size_t)st * BTILE_BYTES;
    mbar_expect_tx(&full[st], n4 * 12u);
    if (d.scan_l2) {
      const uint64_t pol = l2_policy(d.scan_l2);
      bulk_g2s_pol(b, d.bmeta + c.base + t0, n4 * 4u, &full[st], pol);
      bulk_g2s_pol(b + BTILE * 4, d.bkey + c.base + t0, n4 * 8u, &full[st], pol);
    } else {
      bulk_g2s(b, d.bmeta + c.base + t0, n4 * 4u, &full[st]);
      bulk_g2s(b + BTILE * 4, d.bkey + c.base + t0, n4 * 8u, &full[st]);
    }
  };
  // (prologue -- barrier init and the first BSTAGES tiles -- issued by scan_bulk_begin
  //  before the pass parameters and the candidacy table are staged, so they overlap)
  for (uint64_t t = 0; t < ntiles; ++t) {
    const int st = (int)(t % BSTAGES);
    const uint32_t par = (uint32_t)((t / BSTAGES) & 1);
    mbar_wait(&full[st], par);
    const unsigned char* b = buf + (size_t)st * BTILE_BYTES;
    const uint32_t* m = reinterpret_cast<const uint32_t*>(b);
    const uint64_t* kk = reinterpret_cast<const uint64_t*>(b + BTILE * 4);
    const uint64_t t0 = lo + t * BTILE;
    const uint32_t n = (uint32_t)min((uint64_t)BTILE, hi - t0);
    uint32_t mv[BTILE / NT];
    uint64_t kv[BTILE / NT];
#pragma unroll
    for (int u = 0; u < BTILE / NT; ++u) {
      const uint32_t k = (uint32_t)(u * NT + tid);
      mv[u] = k < n ? m[k] : 0u;
      kv[u] = kk[k];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);   // this warp is done reading stage st
#pragma unroll
    for (int u = 0; u < BTILE / NT; ++u) {
      const bool take = (mv[u] & (M_LIVE | M_PIN)) == M_LIVE && cand_test(s, mv[u], kv[u]);
      const uint32_t bal = __ballot_sync(~0u, take);
      if (bal) {                          // CTA-local list of candidate slots (smem)
        uint32_t basep = 0;
        if (lane == 0) basep = atomicAdd(&s.nw, (unsigned)__popc(bal));
        basep = __shfl_sync(~0u, basep, 0);
        if (take) {
          // only the slot now: the exact score (a dependent fp64 chain) is computed after the
          // stream -- stalling a warp on it here delays its stage release (measured slower)
          const uint32_t sl = (uint32_t)(t0 + u * NT + tid);
          const uint32_t w = basep + __popc(bal & ((1u << lane) - 1u));
          if (w < WCAP4) {                // (slot, meta, key): publishing re-reads nothing
            *reinterpret_cast<uint4*>(&s.rhist[4 * w]) =
                make_uint4(sl, mv[u], (uint32_t)kv[u], (uint32_t)(kv[u] >> 32));
          } else {                        // list full (rare): append to the group buffer directly
            Cand x = make_cand(mv[u], kv[u], sl);
            finalize_key(d, c.base, P, x);
            atomicAdd(&s.cnt[x.seg], 1u);
            gdst[atomicAdd(&c.ctl->ncand, 1u)] = x;
          }
        }
      }
    }
    if (tid == 0 && t + BSTAGES < ntiles) {     // refill stage st once every warp drained it
      mbar_wait(&empty[st], par);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads -> async writes
      issue_tile(t + BSTAGES);
    }
  }
  cta_sync();
  if (tid == 0) {       // drain the empty barriers' last phases before the next scan re-inits them
    for (uint64_t t = ntiles > (uint64_t)BSTAGES ? ntiles - BSTAGES : 0; t < ntiles; ++t)
      mbar_wait(&empty[t % BSTAGES], (uint32_t)((t / BSTAGES) & 1));
    for (int st = 0; st < BSTAGES; ++st) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st])) : "memory");
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
  }
#ifdef SAE_WORKER_TIMERS
  if (tid == 0) s.wt_end = gtimer();
#endif
  // publish the CTA's candidates: one reservation in the group buffer, then the records
  // (meta/key from the smem list; exact Eq.(1)-(3) scores, ids) written contiguously
  const uint32_t nl = min(s.nw, WCAP4);
  if (tid == 0) s.gbase = atomicAdd(&c.ctl->ncand, nl);
  cta_sync();
  const uint32_t gb0 = s.gbase;
  for (uint32_t i = tid; i < nl; i += NT) {
    const uint4 rec = *reinterpret_cast<const uint4*>(&s.rhist[4 * i]);
    Cand x = make_cand(rec.y, ((uint64_t)rec.w << 32) | rec.z, rec.x);
    finalize_key(d, c.base, P, x);
    atomicAdd(&s.cnt[x.seg], 1u);
    gdst[gb0 + i] = x;
  }
}

// stride-halving tree sum over y[0..P) in smem (SURVEY c.3 TREE)
__device__ double tree_sum(double* y, int P);

// Execute this CTA's share of a group command (all CTAs of the group, or the only CTA).
__device__ void run_cmd(Ctx& c, unsigned cmd, bool leader) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  GroupCtl* g = c.ctl;
  const int tid = threadIdx.x;
  uint64_t lo, hi;
  switch (cmd) {
    case CMD_SCAN: {
      uint64_t wlo = 0, whi = 0;
      const bool bulk = c.GP > 1 && !leader && d.bulk_ok;
      if (c.GP > 1 && !leader) {
        const uint64_t nw = c.GP - 1, w = c.rank - 1;
        wlo = ((uint64_t)d.C * w / nw) & ~3ull;
        whi = w + 1 == nw ? d.C : (((uint64_t)d.C * (w + 1) / nw) & ~3ull);
        if (bulk) scan_bulk_begin(c, wlo, whi);   // first tiles in flight while staging
      }
      if (tid < 16) s.cnt[tid] = 0;
      if (tid == 0) { s.ncand = 0; s.nw = 0; }
      cta_sync();
      ScanP P;
      if (leader) {   // the leader scans with its own smem copies
        P.now = s.st.now;
        P.thr = (const unsigned long long*)s.st.thr; P.cw = &s.cw[0][0];
        P.mu = s.st.par.mu; P.sg = s.st.par.sigma;
        P.mode = s.st.par.mode; P.w = s.st.par.w;
      } else {        // published by the leader before the command: stage into smem, every
                      // value by its own thread (one L2 round trip, one barrier)
        if (tid < 16) s.wthr[tid] = __ldcg(&g->thr[tid]);
        else if (tid < 31) s.wcw[tid - 16] = __ldcg(&g->cw[0][0] + (tid - 16));
        else if (tid < 36) s.ww[tid - 31] = __ldcg(&g->w[tid - 31]);
        else if (tid < 38) s.wmu[tid - 36] = __ldcg(&g->mu[tid - 36]);
        else if (tid < 40) s.wsg[tid - 38] = __ldcg(&g->sigma[tid - 38]);
        else if (tid == 40) s.wnow = __ldcg(&g->now);
        else if (tid == 41) s.wgam = __ldcg(&g->gamma);
        else if (tid == 42) s.wmode = __ldcg(&g->mode);
        else if (tid == 43) s.wstamp = __ldcg(&g->stamp);
        cta_sync();
        P.now = s.wnow;
        P.thr = (const unsigned long long*)s.wthr; P.cw = s.wcw; P.mu = s.wmu; P.sg = s.wsg;
        P.mode = s.wmode; P.w = s.ww;
      }
      P.stamp = leader ? __ldcg(&g->stamp) : s.wstamp;
      P.gamma = leader ? s.st.par.gamma : s.wgam;
      P.dt_eps = d.dt_eps;
      P.z_cut = d.z_cut;
      if (c.GP == 1 || !leader) {
        build_thr_table(s, P);
        cta_sync();
      }
      if (c.GP > 1) {
        // the leader's smem holds the candidates: workers 1..GP-1 split the pool in
        // 4-slot-aligned slices and stream it through shared memory
        if (!leader) {
          const uint64_t tw0 = gtimer();
          if (bulk) scan_range_bulk(c, wlo, whi, P);
          else scan_range(c, wlo, whi, P);
          if (c.rank == 1 && tid == 0) g->wscan_ns += gtimer() - tw0;
#ifdef SAE_WORKER_TIMERS   // debug build: per-pass max pre-stream / max + min stream / max publish
          if (tid == 0) {
            const uint64_t tp = gtimer();
            atomicMax(&g->wdbg[0], (unsigned long long)(tw0 - s.wt_pick));
            atomicMax(&g->wdbg[1], (unsigned long long)(s.wt_end - tw0));
            atomicMin(&g->wdbg[2], (unsigned long long)(s.wt_end - tw0));
            atomicMax(&g->wdbg[3], (unsigned long long)(tp - s.wt_end));
          }
#endif
        }
      } else {
        part_range(d.C, c.rank, c.GP, lo, hi);
        scan_range(c, lo, hi, P);
      }
      cta_sync();
      if (!d.cand_smem && tid < NSEG && s.cnt[tid]) atomicAdd(&g->cnt[tid], s.cnt[tid]);
      break;
    }
    case CMD_HIST: {   // radix histograms of the active segments' keys (global candidates)
      unsigned* h = reinterpret_cast<unsigned*>(c.cand);
      for (int i = tid; i < NSEG * 256; i += NT) h[i] = 0;
      cta_sync();
      if (tid < 16) { s.wpfx[tid] = __ldcg(&g->pfx[tid]); s.wpmask[tid] = __ldcg(&g->pmask[tid]); }
      cta_sync();
      const unsigned shift = __ldcg(&g->shift), active = __ldcg(&g->active);
      part_range(__ldcg(&g->ncand), c.rank, c.GP, lo, hi);
      const Cand* src = d.gcand + c.base;
      for (uint64_t i = lo + tid; i < hi; i += NT) {
        const uint32_t seg = __ldcg(&src[i].seg);
        if (!((active >> seg) & 1u)) continue;
        const uint64_t key = seg >= 1 && seg <= 8 ? __ldcg(&src[i].k1) : __ldcg(&src[i].k0);
        if ((key & s.wpmask[seg]) != s.wpfx[seg]) continue;
        atomicAdd(&h[seg * 256 + ((key >> shift) & 255u)], 1u);
      }
      cta_sync();
      for (int i = tid; i < NSEG * 256; i += NT)
        if (h[i]) atomicAdd(&g->hist[i], h[i]);
      cta_sync();
      break;
    }
    case CMD_COMPACT: {  // keep candidates at or below the (new) thresholds
      if (tid < 16) s.wthr[tid] = __ldcg(&g->thr[tid]);
      cta_sync();
      part_range(__ldcg(&g->ncand), c.rank, c.GP, lo, hi);
      const Cand* src = d.gcand + c.base;
      Cand* dst = d.gsel + (uint64_t)c.r * CAND_MAX;
      const int lane = tid & 31;
      for (uint64_t i0 = lo; i0 < hi; i0 += NT) {
        const uint64_t i = i0 + tid;
        bool take = false;
        Cand x;
        if (i < hi) {
          x.k0 = __ldcg(&src[i].k0); x.k1 = __ldcg(&src[i].k1);
          x.k2 = __ldcg(&src[i].k2); x.ss = __ldcg(&src[i].ss); x.seg = __ldcg(&src[i].seg);
          take = seg_key(x) <= s.wthr[x.seg];
        }
        const uint32_t bal = __ballot_sync(~0u, take);
        if (bal) {
          uint32_t basep = 0;
          if (lane == 0) basep = atomicAdd(&g->nsel, (unsigned)__popc(bal));
          basep = __shfl_sync(~0u, basep, 0);
          const uint32_t pos = basep + __popc(bal & ((1u << lane) - 1u));
          if (take) {
            atomicAdd(&g->selcnt[x.seg], 1u);
            if (pos < (uint32_t)CAND_MAX) dst[pos] = x;
          }
        }
      }
      break;
    }
    case CMD_CLEAR_T: {
      const uint64_t tb = (uint64_t)d.tmask + 1;
      part_range(tb, c.rank, c.GP, lo, hi);
      uint64_t* keys = d.tkey + (uint64_t)c.r * tb;
      for (uint64_t i = lo + tid; i < hi; i += NT) keys[i] = KEY_EMPTY;
      break;
    }
    case CMD_FILL_T: {
      const uint64_t tb = (uint64_t)d.tmask + 1;
      part_range(d.C, c.rank, c.GP, lo, hi);
      uint64_t* keys = d.tkey + (uint64_t)c.r * tb;
      uint32_t* vals = d.tval + (uint64_t)c.r * tb;
      for (uint64_t sl = lo + tid; sl < hi; sl += NT) {
        const uint64_t gi = c.base + sl;
        if (__ldcg(d.bmeta + gi) & M_LIVE)
          d.btpos[gi] = tbl_insert(keys, vals, d.tmask, __ldcg(d.bhash + gi), (uint32_t)sl, &g->tblcnt);
      }
      break;
    }
    case CMD_CLEAR_G: {
      const uint64_t gt = (uint64_t)d.gmask + 1;
      part_range(gt, c.rank, c.GP, lo, hi);
      uint64_t* keys = d.gkey + (uint64_t)c.r * gt;
      for (uint64_t i = lo + tid; i < hi; i += NT) keys[i] = KEY_EMPTY;
      break;
    }
    case CMD_FILL_G: {
      const uint64_t gt = (uint64_t)d.gmask + 1, gb = (uint64_t)c.r * d.G;
      part_range(d.G, c.rank, c.GP, lo, hi);
      uint64_t* keys = d.gkey + (uint64_t)c.r * gt;
      uint32_t* vals = d.gval + (uint64_t)c.r * gt;
      for (uint64_t p = lo + tid; p < hi; p += NT)
        if (__ldcg(d.glive + gb + p))
          d.gtslot[gb + p] = tbl_insert(keys, vals, d.gmask, __ldcg(d.ghash + gb + p),
                                        (uint32_t)p | ((uint32_t)__ldcg(d.gtau + gb + p) << 28), &g->gtblcnt);
      break;
    }
    case CMD_COUNTQ: {
      if (tid < 4) s.cnt[tid] = 0;
      cta_sync();
      part_range(d.C, c.rank, c.GP, lo, hi);
      for (uint64_t sl = lo + tid; sl < hi; sl += NT) {
        const uint32_t m = __ldcg(d.bmeta + c.base + sl);
        if (m & M_LIVE) atomicAdd(&s.cnt[meta_q(m)], 1u);
      }
      cta_sync();
      if (tid < 4 && s.cnt[tid]) atomicAdd(&g->cntq[tid], s.cnt[tid]);
      break;
    }
    default:
      break;
  }
  cta_sync();
}

// Leader: run a command on the whole group (GP == 1: just run it over everything).
__device__ void issue(Ctx& c, unsigned cmd) {
  if (c.GP == 1) {
    run_cmd(c, cmd, true);
    return;
  }
  const uint64_t t0 = gtimer();
  cta_sync();                   // every leader thread's parameter writes precede the post
  if (threadIdx.x == 0) {
    const uint32_t seq = ++c.s->cseq;
    __threadfence();
    st_release_u64(&c.ctl->cmdw, (cmd_tag(c.d->epoch, seq) << 8) | cmd);
  }
  if (cmd == CMD_EXIT) return;
  const uint64_t t1 = gtimer();
  run_cmd(c, cmd, true);
  if (cmd == CMD_SCAN && c.pf_n) {
    // idle while the workers stream: pull the next request's resident-table and ghost-table
    // home lines into L2 (its probes then start from L2; state is not read here)
    const Dev& d = *c.d;
    const uint64_t tb = (uint64_t)d.tmask + 1, gt = (uint64_t)d.gmask + 1;
    for (uint32_t j = threadIdx.x; j < c.pf_n; j += NT) {
      const uint64_t H = c.pf_h[j];
      const uint64_t* tk = d.tkey + (uint64_t)c.r * tb + home(H, d.tmask);
      const uint32_t* tv = d.tval + (uint64_t)c.r * tb + home(H, d.tmask);
      const uint64_t* gk = d.gkey + (uint64_t)c.r * gt + home(H, d.gmask);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(tk));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(tv));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(gk));
    }
  }
  const uint64_t t2 = gtimer();
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)(c.GP - 1) * c.s->cseq;
    while (ld_acquire_u64(&c.ctl->done) < target) __nanosleep(20);
    const uint64_t t3 = gtimer();
    c.s->st.tph[8] += t1 - t0;
    c.s->st.tph[9] += t2 - t1;
    c.s->st.tph[10] += t3 - t2;
#ifdef SAE_WORKER_TIMERS
    if (cmd == CMD_SCAN) {
      for (int k = 0; k < 4; ++k) { c.s->st.tph[4 + k] += __ldcg(&c.ctl->wdbg[k]); c.ctl->wdbg[k] = k == 2 ? ~0ull : 0ull; }
    }
#endif
  }
  cta_sync();
}

// Leader, before its first command of a launch: reset the done counter.
__device__ void group_open(Ctx& c) {
  if (threadIdx.x == 0) {
    c.s->cseq = 0;
    if (c.GP > 1) { c.ctl->done = 0; __threadfence(); }
  }
  cta_sync();
}

__device__ void worker_loop(Ctx& c) {
  for (uint32_t seq = 1;; ++seq) {
    if (threadIdx.x == 0) {
      const unsigned long long want = cmd_tag(c.d->epoch, seq);
      unsigned long long w;
      while (((w = ld_acquire_u64(&c.ctl->cmdw)) >> 8) != want) __nanosleep(128);
      c.s->wcmd = (unsigned)(w & 0xFFu);
#ifdef SAE_WORKER_TIMERS
      c.s->wt_pick = gtimer();
#endif
    }
    cta_sync();
    const unsigned cmd = c.s->wcmd;
    if (cmd == CMD_EXIT) return;
    run_cmd(c, cmd, false);     // ends with a CTA barrier
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&c.ctl->done, 1ull);
    }
  }
}

// Rebuild the resident table (tombstone cleanup) from the live SoA.
__device__ void rebuild_table(Ctx& c) {
  if (threadIdx.x == 0) c.ctl->tblcnt = 0;
  cta_sync();
  issue(c, CMD_CLEAR_T);
  issue(c, CMD_FILL_T);
  if (threadIdx.x == 0) c.s->st.tbl_used = __ldcg(&c.ctl->tblcnt);
  cta_sync();
}
__device__ void rebuild_ghost(Ctx& c) {
  if (threadIdx.x == 0) c.ctl->gtblcnt = 0;
  cta_sync();
  issue(c, CMD_CLEAR_G);
  issue(c, CMD_FILL_G);
  if (threadIdx.x == 0) c.s->st.gtbl_used = __ldcg(&c.ctl->gtblcnt);
  cta_sync();
}

// stride-halving tree sum over y[0..P) in smem (SURVEY c.3 TREE)
__device__ double tree_sum(double* y, int P) {
  int h = P >> 1;
  for (; h >= 32; h >>= 1) {
    for (int i = threadIdx.x; i < h; i += NT) y[i] = __dadd_rn(y[i], y[i + h]);
    cta_sync();
  }
  // the last levels (h <= 16) inside warp 0 by shuffles: lane i holds y[i]; the same
  // operands and order as y[i] = y[i] + y[i + h]
  if (threadIdx.x < 32) {
    double v = (int)threadIdx.x < P ? y[threadIdx.x] : 0.0;
    for (; h >= 1; h >>= 1) {
      const double o = __shfl_down_sync(~0u, v, h);
      if ((int)threadIdx.x < h) v = __dadd_rn(v, o);
    }
    if (threadIdx.x == 0) y[0] = v;
  }
  cta_sync();
  double r = y[0];
  cta_sync();
  return r;
}

__device__ __forceinline__ double clampd(double x, double lo, double hi) {
  return x < lo ? lo : (x > hi ? hi : x);
}

// LEARN (SURVEY c.3): TokenWeights -> QueueWeights -> LognormalParams -> DecayPower.
__device__ void learn(Ctx& c) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  RState& st = s.st;
  sae_params& p = st.par;
  const uint32_t f = p.learn_flags;
  const double gamma_old = p.gamma;
  // L1 TokenWeights (A16, A17)
  // (each type is independent: one thread per type, the same arithmetic)
  if ((f & SAE_L_TOKENS) && threadIdx.x < 5) {
    {
      const int t = threadIdx.x;
      if (st.ts_ev[t] > 10) {
        double rm = __ddiv_rn((double)st.ts_mae[t], (double)st.ts_ev[t]);
        double rr = st.ts_acc[t] > 0 ? __ddiv_rn((double)st.ts_hit[t], (double)st.ts_acc[t]) : 0.0;
        if (f & SAE_L_TOKEN_MULT) {
          p.w[t] = __dmul_rn(p.w[t], __dadd_rn(1.0, __dmul_rn(p.eta, rm)));
        } else {
          double tgt = __dadd_rn(__dadd_rn(1.0, __dmul_rn(rm, p.a_miss)), __dmul_rn(rr, p.b_reuse));
          p.w[t] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, p.eta), p.w[t]), __dmul_rn(p.eta, tgt));
        }
        p.w[t] = clampd(p.w[t], 0.1, 5.0);
      }
    }
    {
      const int t = threadIdx.x;
      st.ts_ev[t] = (99ull * st.ts_ev[t]) / 100ull;
      st.ts_mae[t] = (99ull * st.ts_mae[t]) / 100ull;
      st.ts_hit[t] = (99ull * st.ts_hit[t]) / 100ull;
      st.ts_acc[t] = (99ull * st.ts_acc[t]) / 100ull;
    }
  }
  // L2 QueueWeights (Alg. P:575-597 or relative rule P:814-817)
  if (f & SAE_L_QUEUES) {
    if (f & SAE_L_QUEUE_RELATIVE) {
      if (threadIdx.x < 4) c.ctl->cntq[threadIdx.x] = 0;
      cta_sync();
      issue(c, CMD_COUNTQ);
      if (threadIdx.x < 3) s.cnt[threadIdx.x] = __ldcg(&c.ctl->cntq[threadIdx.x + 1]);
      cta_sync();
      if (threadIdx.x == 0) {
        double Eq[3];
        bool def[3];
        double sum = 0.0;
        int nd = 0;
        for (int q = 0; q < 3; ++q) {
          double frac = __ddiv_rn((double)s.cnt[q], (double)d.C);
          def[q] = frac > 0.0;
          if (def[q]) { Eq[q] = __ddiv_rn((double)st.qh[q], frac); sum = __dadd_rn(sum, Eq[q]); nd++; }
        }
        if (nd > 0) {
          double Ebar = __ddiv_rn(sum, (double)nd);
          if (Ebar > 0.0) {
            for (int q = 0; q < 3; ++q) {
              if (!def[q]) continue;
              double x = __ddiv_rn(Eq[q], Ebar);
              double pw = (x == 0.0) ? 0.0 : dm::ex(__ddiv_rn(dm::ln(x), p.T));
              p.alpha[q] = __dadd_rn(p.alpha[q], __dmul_rn(p.beta_q, __dsub_rn(pw, p.alpha[q])));
              p.alpha[q] = clampd(p.alpha[q], 0.1, 3.0);
            }
          }
        }
        for (int q = 0; q < 3; ++q) { st.qh[q] = 0; st.qe[q] = 0; }
      }
    } else if (threadIdx.x < 3) {   // queues are independent: one thread per queue
      {
        const int q = threadIdx.x;
        if (st.qe[q] > 5) {
          double eff = __ddiv_rn((double)st.qh[q], (double)st.qe[q]);
          double tgt = __dadd_rn(1.0, __ddiv_rn(eff, p.T));
          p.alpha[q] = __dadd_rn(p.alpha[q], __dmul_rn(p.beta_q, __dsub_rn(tgt, p.alpha[q])));
          p.alpha[q] = clampd(p.alpha[q], 0.1, 3.0);
        }
        st.qh[q] = 0;
        st.qe[q] = 0;
      }
    }
  }
  cta_sync();
  // L3 LognormalParams (Alg. P:762-784; A23, A24, A25)
  if (f & SAE_L_LOGNORMAL) {
    double* y = reinterpret_cast<double*>(c.cand);
    for (int sidx = 0; sidx < 2; ++sidx) {
      uint32_t n = st.iv_len[sidx];
      if (n > d.iv_min) {
        int P = 1;
        while ((uint32_t)P < n) P <<= 1;
        const double* ring = d.iv + ((uint64_t)c.r * 2 + sidx) * RMAX;
        uint32_t first = (st.iv_head[sidx] + RMAX - n) % RMAX;
        for (int i = threadIdx.x; i < P; i += NT) y[i] = (uint32_t)i < n ? ring[(first + i) % RMAX] : 0.0;
        cta_sync();
        double sum = tree_sum(y, P);
        double m = __ddiv_rn(sum, (double)n);
        for (int i = threadIdx.x; i < P; i += NT) {
          double x = (uint32_t)i < n ? ring[(first + i) % RMAX] : 0.0;
          double dd = __dsub_rn(x, m);
          y[i] = (uint32_t)i < n ? __dmul_rn(dd, dd) : 0.0;
        }
        cta_sync();
        double v = __ddiv_rn(tree_sum(y, P), (double)n);
        double b = p.beta_ln;
        if (f & SAE_L_ADAPTIVE_BETA) {   // P:758-760 (A28): observation variance around the model
          const double mu0 = p.mu[sidx];
          for (int i = threadIdx.x; i < P; i += NT) {
            double x = (uint32_t)i < n ? ring[(first + i) % RMAX] : 0.0;
            double dd = __dsub_rn(x, mu0);
            y[i] = (uint32_t)i < n ? __dmul_rn(dd, dd) : 0.0;
          }
          cta_sync();
          const double vobs = __ddiv_rn(tree_sum(y, P), (double)n);
          const double rho = __ddiv_rn(vobs, __dmul_rn(p.sigma[sidx], p.sigma[sidx]));
          b = rho > 1.0 ? fmin(__dmul_rn(2.0, p.beta_ln), 1.0) : __dmul_rn(0.5, p.beta_ln);
        }
        if (threadIdx.x == 0) {
          double sd = __dsqrt_rn(v);
          p.mu[sidx] = __dadd_rn(p.mu[sidx], __dmul_rn(b, __dsub_rn(m, p.mu[sidx])));
          p.sigma[sidx] = __dadd_rn(p.sigma[sidx], __dmul_rn(b, __dsub_rn(sd, p.sigma[sidx])));
          if (p.sigma[sidx] < 0.1) p.sigma[sidx] = 0.1;
          if (n > d.iv_keep) st.iv_len[sidx] = d.iv_keep;
        }
        cta_sync();
      }
    }
  }
  // L4 DecayPower (A27)
  if (f & SAE_L_DECAY) {
    // per-bin hit rates in parallel (scratch: the candidate buffer), sums in bin order
    double* rt = reinterpret_cast<double*>(c.cand);
    const uint32_t NB = d.nbins;
    if (threadIdx.x < NB) {
      const uint32_t i = threadIdx.x;
      rt[i] = st.pb_acc[i] == 0 ? -1.0 : __ddiv_rn((double)st.pb_hit[i], (double)st.pb_acc[i]);
    }
    cta_sync();
  }
  if ((f & SAE_L_DECAY) && threadIdx.x == 0) {
    const double* rt = reinterpret_cast<const double*>(c.cand);
    uint32_t NB = d.nbins, half = NB / 2;
    double fs = 0.0, bs = 0.0;
    int fc = 0, bc = 0;
    for (uint32_t i = 0; i < NB; ++i) {
      if (st.pb_acc[i] == 0) continue;
      const double rate = rt[i];
      if (i < half) { fs = __dadd_rn(fs, rate); fc++; } else { bs = __dadd_rn(bs, rate); bc++; }
    }
    if (fc > 0 && bc > 0) {
      double fa = __ddiv_rn(fs, (double)fc), ba = __ddiv_rn(bs, (double)bc);
      if (fa > 0.0) {
        double ratio = __ddiv_rn(ba, fa);
        double est = __ddiv_rn(1.0, __dadd_rn(ratio, 0.1));
        p.gamma = __dadd_rn(p.gamma, __dmul_rn(p.beta_gamma, __dsub_rn(est, p.gamma)));
        p.gamma = clampd(p.gamma, 0.3, 3.0);
      }
    }
  }
  cta_sync();
  if ((f & SAE_L_DECAY) && threadIdx.x < d.nbins) {
    const uint32_t i = threadIdx.x;
    st.pb_hit[i] = (99ull * st.pb_hit[i]) / 100ull;
    st.pb_acc[i] = (99ull * st.pb_acc[i]) / 100ull;
  }
  cta_sync();
  double cw_old[4];
  for (int t = 0; t < 4; ++t) cw_old[t] = s.cw[2][t];
  cta_sync();
  recompute_cw(s);
  cta_sync();
  // STRUCT-class thresholds follow the parameter change (heuristic only; the exactness
  // check in select_chunk never depends on them): P scales with alpha*w, and for a gamma
  // decrease p(gamma')/p(gamma) lies in [gamma'/gamma, 1], so T' = T * gamma'/gamma keeps
  // the new candidate set inside the old one (no candidate explosion after a firing).
  if (threadIdx.x < 4 && st.thr[9 + threadIdx.x] != ~0ull && cw_old[threadIdx.x] > 0.0) {
    double f = s.cw[2][threadIdx.x] / cw_old[threadIdx.x];
    if (p.gamma < gamma_old) f *= p.gamma / gamma_old;
    if (f != 1.0) {
      const double T = from_obits(st.thr[9 + threadIdx.x]);
      st.thr[9 + threadIdx.x] = obits(T * f);
    }
  }
  if (threadIdx.x == 0) {
    st.learner_firings++;
    if (d.traj_cap > 0) {
      sae_traj t;
      t.E = st.E;
      t.request = st.requests;
      for (int i = 0; i < 5; ++i) t.w[i] = p.w[i];
      for (int i = 0; i < 3; ++i) t.alpha[i] = p.alpha[i];
      for (int i = 0; i < 2; ++i) { t.mu[i] = p.mu[i]; t.sigma[i] = p.sigma[i]; }
      t.gamma = p.gamma;
      d.traj[(uint64_t)c.r * d.traj_cap + (st.traj_n % d.traj_cap)] = t;
      st.traj_n++;
    }
  }
  cta_sync();
}

// ---------------------------------------------------------------------------
// Fused score + select (a4 + a5) for one chunk of m <= MSUB victims (no learner firing
// inside).  Exact: key = (tier, primary, last, id) per SURVEY c.2 O11.  One pass over
// the SoA (split over the group's CTAs) computes every resident, unpinned block's
// segment (EF / 8 multi-turn classes (queue, tau) / 4 STRUCT classes (tau)) and key:
// EF (ntok, id); multi-turn (last, id) -- P is strictly decreasing in dt within a class
// (§8(a) a4), so only class heads need Eq.(1); STRUCT (P, last, id) with the cached
// p_struct.  Blocks at or below their segment's carried threshold are candidates; the
// candidates are sorted by (tier, key), an exactness check proves no excluded block can
// be a victim (else the segment is rescanned), thresholds are re-carried.
// Output: the victims' slots in eviction order in cand[0..m).
// ---------------------------------------------------------------------------
__device__ void narrow(Ctx& c, uint32_t e, uint32_t mp);

// Block-wide MSB radix select over a[0..n): for every class g in `active` find the key of
// rank s.target[g] (1-based) -> s.pfx[g], and the number of smaller keys -> s.below[g].
// Global mode: one class (0), key k0.  Per-segment mode: class = segment, key = seg_key.
__device__ void radix_select(const Cand* a, uint32_t n, bool per_seg, uint32_t active, Smem& s,
                             int tie = 0, uint64_t K0 = 0, uint64_t K1 = 0, int digits = 8,
                             uint32_t early = 0, int tier = -1) {
  // tier >= 0 (global mode): only candidates of that tier (0 EF, 1 scored) take part
  // early > 0 (global mode): stop as soon as the chosen bin and everything below it hold at
  // most `early` keys (below[0] + binc[0]); the caller then sorts that prefix set
  // digits < 8: stop after that many 8-bit digits (the rank-target key then lies in
  // [pfx, pfx | ~pmask]; used for threshold trimming, where any bound is exact)
  // tie = 1: key k1 over the candidates with k0 == K0; tie = 2: key k2 over k0 == K0 && k1 == K1
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 16) { s.pfx[tid] = 0; s.pmask[tid] = 0; s.below[tid] = 0; }
  // The digits above the highest bit in which two keys of one class differ are common to
  // the whole class: start below them.  Differing bits = OR(keys) ^ AND(keys) per class
  // (one pass: lanes of one class reduce together, one smem atomic per group).
  if (tid < 16) { s.drefs[tid] = ~0ull; s.dors[tid] = 0ull; }   // drefs: AND, dors: OR
  cta_sync();
  for (uint32_t i0 = 0; i0 < n; i0 += NT) {
    const uint32_t i = i0 + tid;
    uint32_t g = 0xFFFFFFFFu;
    uint64_t key = 0;
    if (i < n) {
      const Cand x = a[i];
      const uint32_t gg = per_seg ? x.seg : 0u;
      if (gg < 16 && ((active >> gg) & 1u) && (tie == 0 || (x.k0 == K0 && (tie == 1 || x.k1 == K1))) &&
          (tier < 0 || (int)(x.ss >> 28) == tier)) {
        key = per_seg ? seg_key(x) : (tie == 0 ? x.k0 : tie == 1 ? x.k1 : (uint64_t)x.k2);
        g = gg;
      }
    }
    const uint32_t peers = __match_any_sync(~0u, g);
    if (g != 0xFFFFFFFFu) {
      const uint32_t ohi = __reduce_or_sync(peers, (uint32_t)(key >> 32));
      const uint32_t olo = __reduce_or_sync(peers, (uint32_t)key);
      const uint32_t ahi = __reduce_and_sync(peers, (uint32_t)(key >> 32));
      const uint32_t alo = __reduce_and_sync(peers, (uint32_t)key);
      if (lane == __ffs(peers) - 1) {
        atomicOr(&s.dors[g], ((unsigned long long)ohi << 32) | olo);
        atomicAnd(&s.drefs[g], ((unsigned long long)ahi << 32) | alo);
      }
    }
  }
  cta_sync();
  if (tid < 16)                                   // differing bits (0 for an empty class)
    s.dors[tid] = (s.dors[tid] == 0ull && s.drefs[tid] == ~0ull) ? 0ull : (s.dors[tid] ^ s.drefs[tid]);
  cta_sync();
  int top = 0;
  for (int g = 0; g < 16; ++g)
    if ((active >> g) & 1u) {
      const uint64_t dif = s.dors[g];
      if (dif) top = max(top, (63 - __clzll((long long)dif)) & ~7);
    }
  if (tid < 16 && ((active >> tid) & 1u) && top < 56 && s.drefs[tid] != ~0ull) {
    s.pmask[tid] = ~0ull << (top + 8);
    s.pfx[tid] = s.drefs[tid] & s.pmask[tid];
  }
  cta_sync();
  const uint32_t nact = __popc(active);
  for (int shift = top; shift >= 0 && shift > top - 8 * digits; shift -= 8) {
    for (uint32_t i = tid; i < nact * 256; i += NT) {      // clear the active classes' bins only
      uint32_t a = active;
      for (uint32_t j = i >> 8; j > 0; --j) a &= a - 1;
      s.rhist[(__ffs(a) - 1) * 256 + (i & 255u)] = 0;
    }
    cta_sync();
    for (uint32_t i0 = 0; i0 < n; i0 += NT) {
      const uint32_t i = i0 + tid;
      uint32_t bin = 0xFFFFFFFFu;
      if (i < n) {
        const Cand x = a[i];
        const uint32_t g = per_seg ? x.seg : 0u;
        const bool in_tie = (tie == 0 || (x.k0 == K0 && (tie == 1 || x.k1 == K1))) &&
                            (tier < 0 || (int)(x.ss >> 28) == tier);
        if (g < 16 && ((active >> g) & 1u) && in_tie) {
          const uint64_t key = per_seg ? seg_key(x) : (tie == 0 ? x.k0 : tie == 1 ? x.k1 : (uint64_t)x.k2);
          if ((key & s.pmask[g]) == s.pfx[g]) bin = g * 256u + (uint32_t)((key >> shift) & 255u);
        }
      }
      const uint32_t peers = __match_any_sync(~0u, bin);
      if (bin != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&s.rhist[bin], (uint32_t)__popc(peers));
    }
    cta_sync();
    for (int g = wid; g < NSEG; g += NW) {
      if (!((active >> g) & 1u)) continue;
      uint32_t v[8], loc = 0;
      for (int j = 0; j < 8; ++j) { v[j] = s.rhist[g * 256 + lane * 8 + j]; loc += v[j]; }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t need = s.target[g] - s.below[g];
      const uint32_t excl = inc - loc;
      const uint32_t bal = __ballot_sync(~0u, excl < need && inc >= need);
      __syncwarp();
      if (lane == __ffs(bal) - 1) {
        uint32_t run = excl;
        int bsel = 0;
        for (int j = 0; j < 8; ++j) {
          if (run + v[j] >= need) { bsel = lane * 8 + j; break; }
          run += v[j];
        }
        s.below[g] += run;
        s.binc[g] = v[bsel & 7];
        s.pfx[g] |= (uint64_t)bsel << shift;
        s.pmask[g] |= 0xFFull << shift;
      }
    }
    cta_sync();
    if (early && s.below[0] + s.binc[0] <= early) break;
  }
}

// Stage the candidates with k0 <= Ub (at most VCAP) into vbuf and sort them by (k0, k1, k2);
// also the per-segment minimum keys (kmin) over all candidates, for threshold growth.
__device__ void stage_victims(Ctx& c, uint32_t nc, uint64_t Ub) {
  Smem& s = *c.s;
  RState& st = s.st;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s.nv = 0;
  cta_sync();
  for (uint32_t i0 = 0; i0 < nc; i0 += NT) {
    const uint32_t i = i0 + tid;
    bool take = false;
    if (i < nc) take = c.cand[i].k0 <= Ub;
    const uint32_t bal = __ballot_sync(~0u, take);
    uint32_t basep = 0;
    if (lane == 0 && bal) basep = atomicAdd(&s.nv, (uint32_t)__popc(bal));
    basep = __shfl_sync(~0u, basep, 0);
    const uint32_t pos = basep + __popc(bal & ((1u << lane) - 1u));
    if (take && pos < VCAP) c.vbuf[pos] = c.cand[i];
  }
  cta_sync();
  const uint64_t tO = gtimer();
  const uint32_t nv = min(s.nv, (uint32_t)VCAP);
  if (nv <= (uint32_t)NT) {
    // rank placement: (k0, k1, k2) is a total order without ties (ids are unique), so each
    // staged record's rank is the number of smaller ones -- no barriers inside the count
    // T consecutive lanes share one record and split the count (T = NT / nv rounded down
    // to a power of two, at most 32), then combine with shuffles
    uint32_t T = 1;
    while (T < 32u && T * 2u * max(nv, 1u) <= (uint32_t)NT) T <<= 1;
    const uint32_t e = (uint32_t)tid / T, r = (uint32_t)tid & (T - 1u);
    Cand x;
    uint32_t rank = 0;
    if (e < nv) {
      x = c.vbuf[e];
      for (uint32_t j = r; j < nv; j += T) rank += cand_less(c.vbuf[j], x) ? 1u : 0u;
    }
    for (uint32_t o = 1; o < T; o <<= 1) rank += __shfl_xor_sync(~0u, rank, o);
    cta_sync();
    if (e < nv && r == 0) c.vbuf[rank] = x;
    cta_sync();
    if (tid == 0 && c.d->cand_smem) st.tph[13] += gtimer() - tO;   // (groups: [13] is the gather)
    return;
  }
  int N = 32;
  while ((uint32_t)N < nv) N <<= 1;
  for (uint32_t i = nv + tid; i < (uint32_t)N; i += NT) {
    c.vbuf[i].k0 = ~0ull; c.vbuf[i].k1 = ~0ull; c.vbuf[i].k2 = ~0u; c.vbuf[i].ss = 15u << 28;
    c.vbuf[i].seg = 15;
  }
  cta_sync();
  sort_cands(c.vbuf, N);
}

__device__ void select_chunk(Ctx& c, uint32_t m, uint32_t stamp, bool count_pass) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  RState& st = s.st;
  GroupCtl* g = c.ctl;
  const double now = st.now;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool gm = !d.cand_smem;
  uint32_t e = 0, mp = 0, c0 = 0;
  bool staged = false;
  // live, unpinned blocks per segment (maintained counts minus this round's pins)
  if (tid < 16) s.segtot[tid] = tid < NSEG ? st.segcnt[tid] - s.pincnt[tid] : 0u;
  bool proved = false;
  // The baselines (sae.h SAE_MODE_*) key every block by a value without the class
  // monotonicity the thresholds rely on: each of their passes takes every unpinned block as a
  // candidate (Alg.1's full rescan), so their selection is exact by construction.
  const bool baseline = st.par.mode != SAE_MODE_SAE;
  for (int attempt = 0; attempt < 3; ++attempt) {
    if (tid < 16) { s.used[tid] = 0; }
    if (tid == 0) {
      s.fail = 0;
      g->stamp = stamp;
      if (gm) {
        g->ncand = 0;
        g->now = now;
        for (int i = 0; i < 16; ++i) { g->cnt[i] = 0; g->thr[i] = st.thr[i]; }
        for (int q = 0; q < 3; ++q) for (int t = 0; t < 5; ++t) g->cw[q][t] = s.cw[q][t];
        for (int i = 0; i < 2; ++i) { g->mu[i] = st.par.mu[i]; g->sigma[i] = st.par.sigma[i]; }
        for (int i = 0; i < 5; ++i) g->w[i] = st.par.w[i];
        g->gamma = st.par.gamma;
        g->mode = st.par.mode;
      }
    }
    if (baseline && tid < 16) st.thr[tid] = ~0ull;   // baselines: every block is a candidate
    cta_sync();
    if (gm && baseline && tid < 16) g->thr[tid] = ~0ull;
    cta_sync();
    uint64_t t0 = gtimer();
    issue(c, CMD_SCAN);
    if (tid == 0) { const uint64_t t1 = gtimer(); st.tph[1] += t1 - t0; t0 = t1; }
    if (gm) {            // gather the group's counts; bring the candidates into smem
      if (tid < 16) s.cnt[tid] = __ldcg(&g->cnt[tid]);
      if (tid == 0) { s.ncand = __ldcg(&g->ncand); s.fin = 1; }
      cta_sync();
      const uint32_t e0 = min(m, s.segtot[0]);
      const bool narrowed = s.ncand > (uint32_t)CAND_MAX;
      if (tid == 0) { st.select_raw += s.ncand; st.select_narrow += narrowed ? 1 : 0; }
      if (narrowed) narrow(c, e0, m - e0);
      if (tid == 0 && narrowed) { const uint64_t t1 = gtimer(); st.tph[2] += t1 - t0; t0 = t1; }
      const uint64_t tL = gtimer();
      const Cand* src = narrowed ? d.gsel + (uint64_t)c.r * CAND_MAX : d.gcand + c.base;
      for (uint32_t i = tid; i < s.ncand; i += NT) {
        const uint4* sp = reinterpret_cast<const uint4*>(src + i);   // 2 x 16 B per record
        uint4* dp = reinterpret_cast<uint4*>(c.cand + i);
        const uint4 a0 = __ldcg(sp), a1 = __ldcg(sp + 1);
        dp[0] = a0;
        dp[1] = a1;
      }
      cta_sync();
      if (tid == 0) st.tph[13] += gtimer() - tL;
    }
    const uint32_t nc = s.ncand;
    if (tid == 0) {
      st.select_passes++;
      st.select_cands += nc;
      if (nc > (uint32_t)NT) st.select_big++;
      if (attempt == 0 && count_pass) {   // one required pass per chunk (extra passes are overhead)
        uint32_t tot = 0;
        for (int k = 0; k < NSEG; ++k) tot += s.segtot[k];
        st.blocks_scored += tot;
        for (int k = 9; k < NSEG; ++k) st.blocks_scored_struct += s.segtot[k];
      }
    }
    cta_sync();
    if (!gm && s.cnt[0] < m) {       // Stage 2 needed: exact scores of the scored candidates
      ScanP P;
      P.now = now; P.thr = (const unsigned long long*)st.thr; P.cw = &s.cw[0][0];
      P.mu = st.par.mu; P.sg = st.par.sigma; P.gamma = st.par.gamma;
      P.dt_eps = d.dt_eps; P.z_cut = d.z_cut; P.stamp = 0;
      P.mode = st.par.mode; P.w = st.par.w;
      for (uint32_t i = tid; i < nc; i += NT) finalize_key(d, c.base, P, c.cand[i]);
      if (tid == 0) s.fin = 1;
      cta_sync();
    }
    // The victims are the m smallest candidates by (k0, k1, k2): EF keys (ntok, id) are
    // < 2^63 <= obits(P), so Stage 1 precedes Stage 2 by construction.
    c0 = s.cnt[0];
    e = min(m, s.segtot[0]);
    mp = m - e;
    if (tid == 0 && attempt == 0 && count_pass && mp > 0) st.stage2_chunks++;
    uint64_t Kth = ~0ull, Kth1 = ~0ull;   // the m-th victim's (P, last) when staged
    staged = false;
    const uint64_t tR = gtimer();
    if (nc >= m) {
      // Stage 1 / Stage 2: if the EF candidates cover all m victims, select
      // among them only; otherwise every EF candidate is a victim and the rest come from the
      // scored candidates -- each radix then runs over one tier (narrow key ranges)
      const uint32_t ef = s.cnt[0];
      const bool in_ef = ef >= m;
      if (tid == 0) s.target[0] = in_ef ? m : m - ef;
      cta_sync();
      const uint32_t lim = in_ef ? VCAP / 2 : (ef + 16 < VCAP / 2 ? VCAP / 2 - ef : 16u);
      radix_select(c.cand, nc, false, 1u, s, 0, 0, 0, 8, lim * d.early_q / 4, in_ef ? 0 : 1);
      staged = (in_ef ? 0u : ef) + s.below[0] + s.binc[0] <= VCAP;
      if (!staged) {               // rare: fall back to the exact global rank m
        if (tid == 0) s.target[0] = m;
        cta_sync();
        radix_select(c.cand, nc, false, 1u, s);
        // the m-th victim's last (for the exactness check's tie rule): rank m - nless by k1
        // inside the k0 tie group (a large tie group is one request's blocks in one class)
        const uint64_t K0 = s.pfx[0];
        const uint32_t nless = s.below[0];
        cta_sync();
        if (tid == 0) s.target[0] = m - nless;
        cta_sync();
        radix_select(c.cand, nc, false, 1u, s, 1, K0);
        Kth1 = s.pfx[0];
        cta_sync();
        if (tid == 0) { s.pfx[0] = K0; s.below[0] = nless; }   // restore for the unstaged path
        cta_sync();
      }
      Kth = s.pfx[0];
    } else {
      staged = true;                     // nc < m <= MSUB < VCAP
    }
    const uint64_t tV = gtimer();
    if (tid == 0) st.tph[14] += tV - tR;
    if (staged) {
      // stage every candidate whose k0 is at most the chosen bin's upper bound (a superset
      // of the m smallest by (k0, k1, k2)), plus the per-segment minimum keys for threshold
      // growth, then sort the staged set: its first m are the victims, in order
      const uint64_t Ub = nc >= m ? (s.pfx[0] | ~s.pmask[0]) : ~0ull;
      stage_victims(c, nc, Ub);
      if (nc >= m) { Kth = c.vbuf[m - 1].k0; Kth1 = c.vbuf[m - 1].k1; }
      if (tid == 0) st.tph[15] += gtimer() - tV;
    }
    // ---- exactness check: every block a threshold left out must lose to the mp-th
    //      scored candidate.  EF: enough heads.  Class c: a non-candidate has last > T_c,
    //      so dt < now - T_c and, P being non-increasing in dt within a class (tests/
    //      test_prop_monotone.py), P >= P_c(now - T_c) =: PT; it loses to the m-th victim
    //      (Pth, last_m, id_m) if Pth < PT, or if Pth == PT and last_m <= T_c (the tie on P is
    //      broken by last: every non-candidate is younger) -- the case of a tie group of equal
    //      last (one request's blocks) straddling the threshold.  STRUCT: a non-candidate has
    //      P > T_S.
    if (tid == 0 && c0 < e) atomicOr(&s.fail, 1u);
    if (mp > 0 && tid >= 1 && tid < NSEG && s.segtot[tid] > s.cnt[tid]) {
      const uint32_t gsg = tid;
      const double Pth = nc >= m ? from_obits(Kth) : __longlong_as_double(0x7ff0000000000000ll);
      bool ok;
      if (gsg >= 9) {
        ok = Pth <= from_obits(st.thr[gsg]);
      } else {
        const uint32_t q = 1 + (gsg - 1) / 4, tau = (gsg - 1) & 3;
        double dt = __dsub_rn(now, from_obits(st.thr[gsg]));
        if (dt < d.dt_eps) dt = d.dt_eps;
        const double p = survival(dt, st.par.mu[q - 1], st.par.sigma[q - 1], d.z_cut);
        // a relative margin of 2^-30 covers any ulp-level non-monotonicity of the evaluated
        // P(dt) (fdlibm ln/erfc: a few ulp, amplified by at most |z| <= z_cut in the erfc
        // tail); a segment that misses the margin is only rescanned, never decided wrongly
        const double PT = __ddiv_rn(__dmul_rn(s.cw[q - 1][tau], p), dt);
        ok = Pth < PT - PT * 0x1p-30 || (Pth <= PT && Kth1 <= st.thr[gsg]);
      }
      if (!ok) atomicOr(&s.fail, 1u << gsg);
    }
    cta_sync();
    const uint32_t fail = s.fail;
    if (tid == 0) st.tph[3] += gtimer() - t0;
    if (fail == 0) { proved = true; break; }
#ifdef SAE_DEBUG_SELECT
    if (tid == 0)
      printf("select fail r=%u req=%llu attempt=%d m=%u e=%u mp=%u nc=%u c0=%u staged=%d Kth=%.17g Kth1=%.17g fail=%x\n",
             c.r, (unsigned long long)st.requests, attempt, m, e, mp, nc, c0, (int)staged, from_obits(Kth),
             from_obits(Kth1), fail);
    if (tid < NSEG && ((fail >> tid) & 1u))
      printf("   seg %d segtot=%u cnt=%u thr=%.17g (raw %llx)\n", tid, s.segtot[tid], s.cnt[tid],
             from_obits(st.thr[tid]), (unsigned long long)st.thr[tid]);
#endif
    if (tid < 10 && ((fail >> tid) & 1u)) st.select_fail_seg[tid]++;
    if (tid < NSEG && (((fail >> tid) & 1u) || attempt >= 1)) st.thr[tid] = ~0ull;
    cta_sync();
  }
  if (!proved && tid == 0) {   // every threshold was lifted and the check still failed: a bug
    st.err = (uint32_t)(-SAE_E_INTERNAL);
    raise_err(d, SAE_E_INTERNAL);
  }
  const uint64_t tS = gtimer();
  const uint32_t nc = s.ncand;
  uint64_t Kth = nc >= m ? s.pfx[0] : ~0ull;
  if (!staged) {           // rare: a k0 tie group larger than the staging buffer
  // ---- stage exactly the m smallest by (k0, k1, k2): k0 < Kth, then inside the k0 tie
  //      group (k1, k2) < the tie-break rank found by two more radix selects (ids unique)
  uint64_t K1th = ~0ull, K2th = ~0ull;
  if (nc >= m) {
    const uint32_t nless = s.below[0];
    if (tid == 0) s.nv = 0;
    cta_sync();
    for (uint32_t i = tid; i < nc; i += NT)          // size of the k0 tie group
      if (c.cand[i].k0 == Kth) atomicAdd(&s.nv, 1u);
    cta_sync();
    const bool straddle = nless + s.nv > m;          // block-uniform decision...
    cta_sync();                                 // ...taken before s.nv is reused
    if (straddle) {                                  // the tie group straddles rank m
      if (tid == 0) s.target[0] = m - nless;
      cta_sync();
      radix_select(c.cand, nc, false, 1u, s, 1, Kth);
      K1th = s.pfx[0];
      const uint32_t nless1 = s.below[0];
      if (tid == 0) s.target[0] = m - nless - nless1;
      cta_sync();
      radix_select(c.cand, nc, false, 1u, s, 2, Kth, K1th);
      K2th = s.pfx[0];
    }
  }
  if (tid == 0) s.nv = 0;
  cta_sync();
  for (uint32_t i0 = 0; i0 < nc; i0 += NT) {
    const uint32_t i = i0 + tid;
    bool take = false;
    if (i < nc) {
      const Cand x = c.cand[i];
      take = x.k0 < Kth || (x.k0 == Kth && (x.k1 < K1th || (x.k1 == K1th && (uint64_t)x.k2 <= K2th)));
    }
    const uint32_t bal = __ballot_sync(~0u, take);
    uint32_t basep = 0;
    if (lane == 0 && bal) basep = atomicAdd(&s.nv, (uint32_t)__popc(bal));
    basep = __shfl_sync(~0u, basep, 0);
    const uint32_t pos = basep + __popc(bal & ((1u << lane) - 1u));
    if (take && pos < VCAP) c.vbuf[pos] = c.cand[i];
  }
  cta_sync();
  const uint32_t nv = min(s.nv, (uint32_t)VCAP);
  {
    int N = 32;
    while ((uint32_t)N < nv) N <<= 1;
    for (uint32_t i = nv + tid; i < (uint32_t)N; i += NT) {
      c.vbuf[i].k0 = ~0ull; c.vbuf[i].k1 = ~0ull; c.vbuf[i].k2 = ~0u; c.vbuf[i].ss = 15u << 28;
      c.vbuf[i].seg = 15;
    }
    cta_sync();
    sort_cands(c.vbuf, N);       // small: the m victims in (k0, last, id) order
  }
  }                        // !staged
  if (baseline) {                    // no thresholds to carry: copy the victims out
    for (uint32_t v = tid; v < m; v += NT) c.cand[v] = c.vbuf[v];
    if (tid == 0) st.tph[12] += gtimer() - tS;
    cta_sync();
    return;
  }
  // ---- carry thresholds: trim segments holding far more candidates than they use
#ifdef SAE_CARRY_TIMERS   // debug build: sub-phases of the carry in the apply/learn/insert/rebuild slots
  uint64_t tC = gtimer();
#define CARRY_T(k) do { if (tid == 0) { const uint64_t t_ = gtimer(); st.tph[k] += t_ - tC; tC = t_; } } while (0)
#else
#define CARRY_T(k) do { } while (0)
#endif
  for (uint32_t v = tid; v < m; v += NT) atomicAdd(&s.used[c.vbuf[v].seg], 1u);
  cta_sync();
  CARRY_T(4);
  // small private pools (rescans are cheap) trim hard; large pools trim lazily
  const uint32_t trim_at = d.trim_at, trim_to = d.trim_to;
  uint32_t shrink = 0;
  for (int g = 0; g < NSEG; ++g) {
    const uint32_t want = 3 * s.used[g] + d.slack;
    if (s.cnt[g] > trim_at * want && (s.fin || g < 9) && st.trim_skip[g] == 0)   // STRUCT keys need scores
      shrink |= 1u << g;
  }
  cta_sync();                                    // (every thread read trim_skip before it changes)
  if (tid < NSEG && st.trim_skip[tid]) st.trim_skip[tid]--;
  if (shrink) {
    if (tid < NSEG) s.target[tid] = trim_to * (3 * s.used[tid] + d.slack);
    cta_sync();
    // one segment at a time, so each radix starts below ITS OWN common key prefix (a shared
    // start -- the highest differing bit over all segments -- left the two digits of a
    // segment with narrowly spread keys inside its common prefix: no cut, and the same
    // useless trim every pass, 5.7 us per C4x pass)
    for (uint32_t rest = shrink; rest; rest &= rest - 1) {
      const int g = __ffs(rest) - 1;
      radix_select(c.cand, nc, true, 1u << g, s, 0, 0, 0, 2);   // two digits: a bound, not a rank
      if (tid == g) {
        const uint64_t cut = s.pfx[g] | ~s.pmask[g];
        if (cut < st.thr[g]) st.thr[g] = cut;
        else st.trim_skip[g] = 16;               // no cut: back off for 16 passes
      }
      cta_sync();
    }
  }
  CARRY_T(5);
  // ---- grow a segment's threshold before its reserve runs dry (avoids refills): double
  //      the key distance from the smallest candidate (keys: EF (ntok,id); class last;
  //      STRUCT P).  Heuristic only -- exactness is re-proved every pass.
  //      (the per-segment minimum keys are computed only for the segments that grow)
  if (tid == 0) s.nv = 0;                      // reused: mask of growing segments
  if (tid < 16) s.kmin[tid] = ~0ull;
  cta_sync();
  if (tid < NSEG && !((shrink >> tid) & 1u) && (s.fin || tid < 9)) {
    const uint32_t left = s.cnt[tid] - min(s.cnt[tid], s.used[tid]);
    if (st.thr[tid] != ~0ull && s.segtot[tid] > s.cnt[tid] && left < 2 * s.used[tid] + d.slack)
      atomicOr(&s.nv, 1u << tid);
  }
  cta_sync();
  const uint32_t growm = s.nv;
  if (growm) {
    for (uint32_t i0 = 0; i0 < nc; i0 += NT) {
      const uint32_t i = i0 + tid;
      uint32_t g = 0xFFFFFFFFu;
      uint64_t key = ~0ull;
      if (i < nc) {
        const Cand x = c.cand[i];
        // EF grows within its threshold's num_tokens band: min over that band only
        if (((growm >> x.seg) & 1u) && (x.seg != 0 || (x.k0 >> 32) == (st.thr[0] >> 32))) {
          g = x.seg;
          key = seg_key(x);
        }
      }
      const uint32_t peers = __match_any_sync(~0u, g);
      if (g != 0xFFFFFFFFu) {
        const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
        const uint32_t mhi = __reduce_min_sync(peers, hi);
        const uint32_t p2 = peers & __ballot_sync(peers, hi == mhi);
        if (hi == mhi) {
          const uint32_t mlo = __reduce_min_sync(p2, lo);
          if (lane == __ffs(p2) - 1) atomicMin(&s.kmin[g], ((unsigned long long)mhi << 32) | mlo);
        }
      }
    }
    cta_sync();
  }
  CARRY_T(6);
  if (tid < NSEG && ((growm >> tid) & 1u)) {
    const uint32_t g = tid;
    const uint64_t T = st.thr[g];
    {
      const uint64_t km = s.kmin[g] == ~0ull ? T : (uint64_t)s.kmin[g];
      uint64_t Tn;
      if (g == 0) {                 // id part only, saturating inside the ntok band
        const uint64_t band = T & ~0xFFFFFFFFull, idT = T & 0xFFFFFFFFull;
        const uint64_t idm = (km & ~0xFFFFFFFFull) == band ? (km & 0xFFFFFFFFull) : idT;
        const uint64_t dlt = max(idT - min(idm, idT), (uint64_t)4096);
        Tn = band | min(idT + dlt, (uint64_t)0xFFFFFFFFull);
      } else if (g <= 8) {
        const double Tl = from_obits(T), kl = from_obits(km);
        Tn = obits(Tl + fmax(Tl - kl, 1.0));
      } else {
        const double Tp = from_obits(T), kp = from_obits(km);
        Tn = obits(fmax(2.0 * Tp - kp, 1.5 * Tp));
      }
      st.thr[g] = Tn;
    }
  }
  cta_sync();
  for (uint32_t v = tid; v < m; v += NT) c.cand[v] = c.vbuf[v];
  CARRY_T(7);
#undef CARRY_T
  if (tid == 0) st.tph[12] += gtimer() - tS;
  cta_sync();
}

// Too many candidates for the leader's smem: choose, per over-full segment, the exact key
// of rank target_s by a group-parallel MSB radix select over the candidate buffer, then
// compact the candidates at or below the new thresholds.  The new thresholds are exact
// bounds (every dropped candidate has a larger key), so the exactness check still holds.
__device__ void narrow(Ctx& c, uint32_t e, uint32_t mp) {
  Smem& s = *c.s;
  RState& st = s.st;
  GroupCtl* g = c.ctl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < NSEG) {
    const uint32_t need = tid == 0 ? e : mp;
    s.target[tid] = 3 * (need + SLACK);   // refill a reserve for several chunks
    s.pfx[tid] = 0;
    s.pmask[tid] = 0;
    s.below[tid] = 0;
  }
  cta_sync();
  uint32_t active = 0;
  for (int k = 0; k < NSEG; ++k) if (s.cnt[k] > s.target[k]) active |= 1u << k;
  for (int shift = 56; shift >= 0 && active; shift -= 8) {
    if (tid == 0) {
      g->shift = (unsigned)shift;
      g->active = active;
      for (int k = 0; k < NSEG; ++k) { g->pfx[k] = s.pfx[k]; g->pmask[k] = s.pmask[k]; }
    }
    for (int i = tid; i < NSEG * 256; i += NT) g->hist[i] = 0;
    cta_sync();
    issue(c, CMD_HIST);
    // one warp per active segment: find the digit holding rank target
    for (int k = wid; k < NSEG; k += NW) {
      if (!((active >> k) & 1u)) continue;
      uint32_t v[8], loc = 0;
      for (int j = 0; j < 8; ++j) { v[j] = __ldcg(&g->hist[k * 256 + lane * 8 + j]); loc += v[j]; }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t need = s.target[k] - s.below[k];     // >= 1
      const uint32_t excl = inc - loc;
      const bool mine = excl < need && inc >= need;
      const uint32_t bal = __ballot_sync(~0u, mine);
      __syncwarp();
      const int src = __ffs(bal) - 1;
      if (lane == src) {
        uint32_t run = excl;
        int b = 0;
        for (int j = 0; j < 8; ++j) {
          if (run + v[j] >= need) { b = lane * 8 + j; break; }
          run += v[j];
        }
        s.below[k] += run;
        s.pfx[k] |= (uint64_t)b << shift;
        s.pmask[k] |= 0xFFull << shift;
      }
    }
    cta_sync();
  }
  if (tid == 0) {
    for (int k = 0; k < NSEG; ++k) if ((active >> k) & 1u) st.thr[k] = s.pfx[k];
    for (int k = 0; k < 16; ++k) { g->thr[k] = st.thr[k]; g->selcnt[k] = 0; }
    g->nsel = 0;
  }
  cta_sync();
  issue(c, CMD_COMPACT);
  if (tid < 16) s.cnt[tid] = __ldcg(&g->selcnt[tid]);
  if (tid == 0) {
    s.ncand = __ldcg(&g->nsel);
    if (s.ncand > (uint32_t)CAND_MAX) {     // pathological key ties: cannot hold them all
      st.err = (uint32_t)(-SAE_E_OVERFLOW);
      raise_err(*c.d, SAE_E_OVERFLOW);
      s.ncand = CAND_MAX;
    }
  }
  cta_sync();
}

// Apply a chunk of m victims (cand[0..m) in eviction order): SURVEY c.2 O11 steps 1-4.
__device__ void apply_chunk(Ctx& c, uint32_t m, uint32_t* vids_out) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  RState& st = s.st;
  const uint64_t tb = (uint64_t)d.tmask + 1, gt = (uint64_t)d.gmask + 1;
  uint64_t* tkey = d.tkey + (uint64_t)c.r * tb;
  uint64_t* gkey = d.gkey + (uint64_t)c.r * gt;
  uint32_t* gval = d.gval + (uint64_t)c.r * gt;
  const uint64_t gb = (uint64_t)c.r * d.G;
  for (uint32_t v0 = 0; v0 < m; v0 += d.G) {
    const uint32_t mb = min(m - v0, d.G);
    // phase 1: remove from the resident table (position kept in the SoA: no probe), count,
    // expire the ghost slots; all loads of a victim are independent (one round trip)
    for (uint32_t vb = 0; vb < mb; vb += NT) {
      const uint32_t v = vb + threadIdx.x;
      uint64_t H = 0;
      uint32_t p = 0, sl = 0, tau = 0;
      if (v < mb) {
        sl = c.cand[v0 + v].ss & SLOT_MASK;
        const uint64_t gi = c.base + sl;
        p = (uint32_t)((st.gseq + v0 + v) % d.G);
        H = d.bhash[gi];
        const uint32_t meta = d.bmeta[gi];
        const uint32_t tp = d.btpos[gi];
        const uint8_t glv = d.glive[gb + p];
        const uint32_t gts = d.gtslot[gb + p];
        const uint32_t q = meta_q(meta);
        tau = meta_tau(meta);
        if (vids_out) vids_out[v0 + v] = d.bid[gi];
        tkey[tp] = KEY_TOMB;
        d.bmeta[gi] = 0;
        atomicSub(&st.segcnt[seg_of_tix(meta_tix(meta))], 1u);
        if (tau < 5) atomicAdd((unsigned long long*)&st.ts_ev[tau], 1ull);
        if (q != Q_EF) atomicAdd((unsigned long long*)&st.qe[q - 1], 1ull);
        atomicAdd((unsigned long long*)&st.evict_by_queue[q], 1ull);
        atomicAdd((unsigned long long*)&st.evict_by_type[tau], 1ull);
        if (glv) gkey[gts] = KEY_TOMB;   // FIFO expiry of the oldest ghost (A30)
        d.ghash[gb + p] = H;
        d.gtau[gb + p] = (uint8_t)tau;
      }
      cta_sync();
      // phase 2: ghost push (recently_evicted[hash] = tau), free the slot
      if (v < mb) {
        d.glive[gb + p] = 1;
        d.gtslot[gb + p] = tbl_insert(gkey, gval, d.gmask, H, p | (tau << 28), &st.gtbl_used);
        d.freestk[c.base + st.free_top + v0 + v] = sl;
      }
      cta_sync();
    }
    if (threadIdx.x == 0) {
      st.free_top += mb;
      st.live -= mb;
      st.gseq += mb;
      st.E += mb;
      st.evictions += mb;
    }
    cta_sync();
  }
}

// Evict k victims with pin stamp (k <= unpinned residents), chunked at K crossings (A14)
// and in passes of at most MSUB victims (keys are frozen between firings).
__device__ void evict_k(Ctx& c, uint64_t k, uint32_t stamp, uint32_t* vids_out) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  uint64_t done = 0, chunk_end = 0;
  while (done < k) {
    const uint64_t to_cross = d.K - (s.st.E % d.K);
    const bool first = done >= chunk_end;          // first sub-pass of a chunk between firings
    if (first) chunk_end = done + min(k - done, to_cross);
    const uint32_t m = (uint32_t)min(min(k - done, to_cross), (uint64_t)MSUB);
    select_chunk(c, m, stamp, first);
    uint64_t t0 = gtimer();
    apply_chunk(c, m, vids_out ? vids_out + done : nullptr);
    if (threadIdx.x == 0) { const uint64_t t1 = gtimer(); s.st.tph[4] += t1 - t0; t0 = t1; }
    done += m;
    if (s.st.E % d.K == 0) {
      learn(c);
      if (threadIdx.x == 0) s.st.tph[5] += gtimer() - t0;
    }
  }
  if (s.st.gtbl_used > ((d.gmask + 1) / 4) * 3) rebuild_ghost(c);
}

__device__ void load_state(Ctx& c) {
  const Dev& d = *c.d;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(d.st + c.r);
  uint32_t* dst = reinterpret_cast<uint32_t*>(&c.s->st);
  for (int i = threadIdx.x; i < (int)(sizeof(RState) / 4); i += NT) dst[i] = __ldcg(src + i);
  if (threadIdx.x < 16) c.s->pincnt[threadIdx.x] = 0;
  cta_sync();
  recompute_cw(*c.s);
  cta_sync();
}
__device__ void store_state(Ctx& c) {
  cta_sync();
  const Dev& d = *c.d;
  uint32_t* dst = reinterpret_cast<uint32_t*>(d.st + c.r);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(&c.s->st);
  for (int i = threadIdx.x; i < (int)(sizeof(RState) / 4); i += NT) dst[i] = src[i];
}

// One request round (SURVEY c.2 O1-O13).  Returns false on a sticky error.
__device__ bool admit_one(Ctx& c, const BatchDev& b, uint32_t i) {
  const Dev& d = *c.d;
  Smem& s = *c.s;
  RState& st = s.st;
  const uint64_t tb = (uint64_t)d.tmask + 1, gt = (uint64_t)d.gmask + 1;
  uint64_t* tkey = d.tkey + (uint64_t)c.r * tb;
  uint32_t* tval = d.tval + (uint64_t)c.r * tb;
  uint64_t* gkey = d.gkey + (uint64_t)c.r * gt;
  uint32_t* gval = d.gval + (uint64_t)c.r * gt;
  const uint64_t gb = (uint64_t)c.r * d.G;
  const double now = b.arrival[i];
  const uint32_t L = b.plen[i], O = b.dlen[i];
  // O1 / time check
  if (L < 1 || (st.has_now && now < st.now)) {
    if (threadIdx.x == 0) {
      st.err = L < 1 ? (uint32_t)(-SAE_E_INVAL) : (uint32_t)(-SAE_E_TIME);
      raise_err(d, L < 1 ? SAE_E_INVAL : SAE_E_TIME);
    }
    cta_sync();
    return false;
  }
  const uint32_t B = d.B;
  const uint32_t np = (L + B - 1) / B, n = np + (O + B - 1) / B;
  const uint64_t bo = b.boff[i];
  const uint32_t fl = b.flags[i], spb = b.spb[i];
  const bool mt = fl & 1, ag = fl & 2, cid = fl & 4;
  const bool untempl = !mt && spb == 0;             // A31
  const uint32_t omax = np > 1 ? np - 1 : 1;         // A8
  cta_sync();
  if (threadIdx.x == 0) {
    st.now = now;
    st.has_now = 1;
    st.round++;
    s.h = (int32_t)n;
    s.npin = 0;
    s.matched = 0;
  }
  if (threadIdx.x < 16) s.pincnt[threadIdx.x] = 0;
  cta_sync();
  const uint32_t stamp = (uint32_t)st.round;
  uint64_t tA = gtimer();
  // ---- O4/O5 classify + probe (Alg.1 Classify P:550-564; strict prefix P:158)
  // (the first NT blocks' values stay in registers for the next loop: same thread, same j)
  uint64_t rH = 0;
  int32_t rsl = -1;
  uint32_t rq = 0, rtau = 0;
  for (uint32_t j = threadIdx.x; j < n; j += NT) {
    const uint64_t H = b.h[bo + j];
    const uint32_t tau = b.tau[bo + j];
    const int32_t sl = tbl_find(tkey, tval, d.tmask, H);
    const uint32_t q = st.par.mode == SAE_MODE_SAE ? classify(tau, mt, ag, cid, j < spb, untempl)
                                                   : (uint32_t)Q_CHAT;   // baselines: one queue
    b.slot[bo + j] = sl;
    b.q[bo + j] = (uint8_t)q;
    if (j < (uint32_t)NT) { rH = H; rsl = sl; rq = q; rtau = tau; }
    if (sl < 0) atomicMin(&s.h, (int32_t)j);
    else atomicAdd(&s.npin, 1u);
  }
  cta_sync();
  const uint32_t h = (uint32_t)s.h;
  // ---- O6-O9 stats, touch, orphans, miss-after-evict; ordered ranks by block scans
  uint32_t new_base = 0;
  for (uint32_t j0 = 0; j0 < n; j0 += NT) {
    const uint32_t j = j0 + threadIdx.x;
    const bool valid = j < n;
    uint32_t fc = 0, fa = 0, fn = 0;
    double lnv = 0.0;
    if (valid) {
      const bool inreg = j0 == 0;
      const int32_t sl = inreg ? rsl : b.slot[bo + j];
      const uint32_t q = inreg ? rq : b.q[bo + j], tau = inreg ? rtau : b.tau[bo + j];
      const uint32_t bin = min(d.nbins - 1, (d.nbins * j) / omax);
      if (tau < 5) atomicAdd((unsigned long long*)&st.ts_acc[tau], 1ull);
      if (q == Q_STRUCT) atomicAdd((unsigned long long*)&st.pb_acc[bin], 1ull);
      if (sl >= 0) {
        const uint64_t gi = c.base + (uint32_t)sl;
        const uint32_t meta = d.bmeta[gi];
        const double lastv = d.blast[gi];
        const uint32_t idv = d.bid[gi];
        if (j < h) {  // O7 hit (A9: credited to the old queue before re-routing)
          double dt = __dsub_rn(now, lastv);
          if (dt < d.dt_eps) dt = d.dt_eps;
          const uint32_t qo = meta_q(meta);
          if (qo == Q_CHAT || qo == Q_AGENT) {
            atomicAdd((unsigned long long*)&st.qh[qo - 1], 1ull);
            lnv = dm::ln(dt);
            if (qo == Q_CHAT) fc = 1; else fa = 1;
          } else if (qo == Q_STRUCT) {
            atomicAdd((unsigned long long*)&st.qh[2], 1ull);
          }
          if (tau < 5) atomicAdd((unsigned long long*)&st.ts_hit[tau], 1ull);
          if (q == Q_STRUCT) atomicAdd((unsigned long long*)&st.pb_hit[bin], 1ull);
          if (j < np) atomicAdd(&s.matched, (uint32_t)b.ntok[bo + j]);
          d.bacc[gi] += 1;
        }
        // O7/O8 touch: last = now, hint overwritten (A9, A10)
        d.blast[gi] = now;
        d.bkey[gi] = scan_key(q, meta_ntok(meta), idv, now);
        const uint32_t tix = tix_of(q, tau, j, omax);
        d.bmeta[gi] = meta_pack(q, tau, meta_ntok(meta)) | M_PIN |       // pinned for this round (A11)
                      (tix << M_TIX_SHIFT);
        const uint32_t so = seg_of_tix(meta_tix(meta)), sn = seg_of_tix(tix);
        if (so != sn) { atomicSub(&st.segcnt[so], 1u); atomicAdd(&st.segcnt[sn], 1u); }
        atomicAdd(&s.pincnt[sn], 1u);
        d.bob[gi] = j;
        d.bomax[gi] = omax;
      } else if (j >= h) {  // O9 miss-after-evict, consumed (A30)
        const uint64_t H = inreg ? rH : b.h[bo + j];
        const int32_t gp = tbl_find_pos(gkey, d.gmask, H);
        if (gp >= 0) {
          const uint32_t gv = gval[gp];            // ring position | tau << 28
          const uint32_t rp = gv & SLOT_MASK, gtau = gv >> 28;
          if (gtau < 5) atomicAdd((unsigned long long*)&st.ts_mae[gtau], 1ull);
          atomicAdd((unsigned long long*)&st.mae_by_type[gtau], 1ull);
          gkey[gp] = KEY_TOMB;
          d.glive[gb + rp] = 0;
        }
        fn = 1;
      }
    }
    uint32_t rc, ra, rn;
    block_scan3(fc, fa, fn, rc, ra, rn, s.tot, s.wsum);
    if (fc) d.iv[((uint64_t)c.r * 2 + 0) * RMAX + (st.iv_head[0] + rc) % RMAX] = lnv;
    if (fa) d.iv[((uint64_t)c.r * 2 + 1) * RMAX + (st.iv_head[1] + ra) % RMAX] = lnv;
    if (valid) b.nrank[bo + j] = fn ? (int32_t)(new_base + rn) : -1;
    new_base += s.tot[2];
    cta_sync();
    if (threadIdx.x == 0) {
      for (int q = 0; q < 2; ++q) {
        st.iv_head[q] = (st.iv_head[q] + s.tot[q]) % RMAX;
        st.iv_len[q] = min(d.iv_ring, st.iv_len[q] + s.tot[q]);
      }
    }
    cta_sync();
  }
  // ---- O10 admission size (A11)
  if (threadIdx.x == 0) {
    const uint64_t f = d.C - st.live;
    const uint64_t U = st.live - s.npin;
    uint64_t k = new_base > f ? new_base - f : 0;
    uint64_t admit = new_base;
    if (k > U) { k = U; admit = f + U; }
    s.k = k;
    s.admit = admit;
    if (k > 0) st.eviction_rounds++;
    if (b.boff[i] + k > b.vcap) { st.err = (uint32_t)(-SAE_E_OVERFLOW); raise_err(d, SAE_E_OVERFLOW); }
  }
  cta_sync();
  if (st.err) return false;
  const uint64_t k = s.k, admit = s.admit;
  if (threadIdx.x == 0) st.tph[0] += gtimer() - tA;
  // ---- O11 evictions (Alg.1 Evict x k, chunked at K crossings)
  if (c.GP > 1 && i + 1 < b.n) {     // next request of this replica's run (prefetch hint)
    c.pf_h = b.h + b.boff[i + 1];
    c.pf_n = (uint32_t)min(b.boff[i + 2] - b.boff[i + 1], (uint64_t)512);
  } else {
    c.pf_n = 0;
  }
  if (k > 0) evict_k(c, k, stamp, b.o_vids ? b.o_vids + b.boff[i] : nullptr);
  tA = gtimer();
  // ---- unpin this request's resident blocks
  for (uint32_t j = threadIdx.x; j < n; j += NT) {
    const int32_t sl = b.slot[bo + j];
    if (sl >= 0) d.bmeta[c.base + (uint32_t)sl] &= ~M_PIN;
  }
  // ---- O12 insert New (Alg.1 Add: q.insert(b))
  if (threadIdx.x == 0 && st.next_id + admit > 0xFFFFFFFFull) {
    st.err = (uint32_t)(-SAE_E_OVERFLOW);
    raise_err(d, SAE_E_OVERFLOW);
  }
  cta_sync();
  if (st.err) return false;
  for (uint32_t j = threadIdx.x; j < n; j += NT) {
    const int32_t rk = b.nrank[bo + j];
    if (rk < 0 || (uint64_t)rk >= admit) continue;
    const uint32_t sl = d.freestk[c.base + st.free_top - 1 - rk];
    const uint64_t gi = c.base + sl;
    const uint64_t H = b.h[bo + j];
    const uint32_t q = b.q[bo + j], tau = b.tau[bo + j];
    d.bhash[gi] = H;
    d.blast[gi] = now;
    d.bid[gi] = (uint32_t)(st.next_id + rk);
    d.bacc[gi] = 1;
    d.bkey[gi] = scan_key(q, b.ntok[bo + j], (uint32_t)(st.next_id + rk), now);
    const uint32_t tix = tix_of(q, tau, j, omax);
    d.bmeta[gi] = meta_pack(q, tau, b.ntok[bo + j]) | (tix << M_TIX_SHIFT);
    atomicAdd(&st.segcnt[seg_of_tix(tix)], 1u);
    d.bob[gi] = j;
    d.bomax[gi] = omax;
    d.btpos[gi] = tbl_insert(tkey, tval, d.tmask, H, sl, &st.tbl_used);
  }
  cta_sync();
  if (threadIdx.x == 0) {
    st.free_top -= (uint32_t)admit;
    st.live += (uint32_t)admit;
    st.next_id += admit;
    // ---- O13 outputs
    if (b.o_hit) b.o_hit[i] = h;
    if (b.o_miss) b.o_miss[i] = n - h;
    if (b.o_matched) b.o_matched[i] = s.matched;
    if (b.o_nvict) b.o_nvict[i] = (uint32_t)k;
    st.requests++;
    st.blocks_looked_up += n;
    st.hit_blocks += h;
    st.hit_tokens += s.matched;
    st.prompt_tokens += L;
  }
  cta_sync();
  if (threadIdx.x == 0) { const uint64_t t1 = gtimer(); st.tph[6] += t1 - tA; tA = t1; }
  if (st.tbl_used > (d.tmask + 1) / 4 * 3) {
    rebuild_table(c);
    if (threadIdx.x == 0) st.tph[7] += gtimer() - tA;
  }
  return true;
}

extern __shared__ __align__(16) unsigned char g_smem[];

__device__ Ctx make_ctx(const Dev& d, uint32_t r, uint32_t rank) {
  Ctx c;
  c.d = &d;
  c.s = reinterpret_cast<Smem*>(g_smem);
  if (CAND_GLOBAL) {
    // candidate buffer in the replica's own region of global memory (L1-resident: only this
    // CTA touches it), shared memory keeps the state and the victim staging: a smaller CTA
    // footprint, so more replicas are resident per SM
    c.cand = d.cpriv + (uint64_t)r * CAND_MAX;
    c.vbuf = reinterpret_cast<Cand*>(g_smem + ((sizeof(Smem) + 15) / 16) * 16);
  } else {
    c.cand = reinterpret_cast<Cand*>(g_smem + ((sizeof(Smem) + 15) / 16) * 16);
    c.vbuf = c.cand + CAND_MAX;
  }
  c.ctl = d.ctl + r;
  c.r = r;
  c.rank = rank;
  c.GP = d.GP;
  c.base = (uint64_t)r * d.C;
  c.pf_h = nullptr;
  c.pf_n = 0;
  return c;
}

// Persistent replay: the group of GP CTAs (blockIdx / GP) owns replica r; its leader
// (rank 0) replays the replica's run of the batch in order, the others execute the
// leader's group commands (scan / histogram / compact / refresh / rebuild).
// Task-split replay (d.nchunk > 1; single-CTA replicas only): a persistent grid of at most
// the co-resident CTAs takes tasks t = chunk * R + r in increasing order from one counter;
// task (k, r) replays the k-th of nchunk consecutive pieces of replica r's run.  Chunk k > 0
// first waits (acquire) for rflag[r] = (epoch, k), which the CTA that ran chunk k - 1 stored
// (release) after its state: the replica's requests stay in order, and its state may move
// between SMs (the acquire orders every later load of this CTA after the other CTA's
// stores).  Every waited-for task was taken earlier by a running CTA whose own waits are on
// still earlier tasks, so the chain ends at a chunk 0 (no deadlock, no co-residency needed).
// Balances the waves: R x nchunk tasks over G CTAs instead of ceil(R / G) whole replicas.
__device__ void replay_tasks(const Dev& d, const BatchDev& b) {
  Smem& s = *reinterpret_cast<Smem*>(g_smem);
  const uint32_t R = d.R, nch = d.nchunk;
  const uint64_t ntask = (uint64_t)R * nch;
  for (;;) {
    if (threadIdx.x == 0) s.wcmd = atomicAdd(d.taskctr, 1u);
    cta_sync();
    const uint32_t t = s.wcmd;
    cta_sync();                                   // (s.wcmd is rewritten by the next task)
    if ((uint64_t)t >= ntask) return;
    const uint32_t k = t / R, r = t % R;
    Ctx c = make_ctx(d, r, 0);
    const uint32_t lo = b.run_start[r];
    if (k > 0 && threadIdx.x == 0) {
      const uint32_t want = (d.epoch << 8) | k;
      while (ld_acquire_u32(&d.rflag[r]) != want) __nanosleep(64);
    }
    cta_sync();
    if (lo < RUN_INVALID && batch_size_ok(b)) {
      const uint32_t n = b.run_end[r] - lo;
      const uint32_t clo = lo + (uint32_t)((uint64_t)n * k / nch);
      const uint32_t chi = lo + (uint32_t)((uint64_t)n * (k + 1) / nch);
      if (clo < chi) {
        load_state(c);
        if (c.s->st.err == 0) {
          for (uint32_t i = clo; i < chi; ++i)
            if (!admit_one(c, b, i)) break;
        }
        store_state(c);
      }
    }
    cta_sync();                                   // every thread's stores precede the release
    if (threadIdx.x == 0 && k + 1 < nch) {
      __threadfence();
      st_release_u32(&d.rflag[r], (d.epoch << 8) | (k + 1));
    }
  }
}

__global__ void __launch_bounds__(NT, MINB) k_replay(Dev d, BatchDev b) {
  if (d.nchunk > 1) {
    replay_tasks(d, b);
    return;
  }
  const uint32_t r = blockIdx.x / d.GP, rank = blockIdx.x % d.GP;
  if (r >= d.R) return;
  Ctx c = make_ctx(d, r, rank);
  if (rank != 0) {
    worker_loop(c);
    return;
  }
  group_open(c);
  const uint32_t lo = b.run_start[r];
  // (no requests for this replica, a replica split into several runs, or a batch larger
  //  than its declared workspace: k_runs / k_hash raised the sticky error; skip)
  if (lo < RUN_INVALID && batch_size_ok(b)) {
    const uint32_t hi = b.run_end[r];
    load_state(c);
    if (c.s->st.err == 0) {
      for (uint32_t i = lo; i < hi; ++i)
        if (!admit_one(c, b, i)) break;
    }
    store_state(c);
  }
  if (c.GP > 1) issue(c, CMD_EXIT);
}

// sae_evict: Alg.1 Evict x k with an empty pin set.
__global__ void __launch_bounds__(NT, MINB) k_evict(Dev d, uint32_t r, uint32_t k, double now,
                                                 uint32_t* vids, uint32_t* n_out) {
  Ctx c = make_ctx(d, r, blockIdx.x);
  if (blockIdx.x != 0) {
    worker_loop(c);
    return;
  }
  group_open(c);
  load_state(c);
  RState& st = c.s->st;
  if (st.err == 0) {
    if (st.has_now && now < st.now) {
      if (threadIdx.x == 0) { st.err = (uint32_t)(-SAE_E_TIME); raise_err(d, SAE_E_TIME); }
    } else {
      cta_sync();
      if (threadIdx.x == 0) { st.now = now; st.has_now = 1; st.round++; }
      cta_sync();
      const uint32_t kk = min(k, st.live);
      if (kk > 0) {
        if (threadIdx.x == 0) st.eviction_rounds++;
        evict_k(c, kk, 0xFFFFFFFFu /* no block carries this stamp */, vids);
      }
      if (threadIdx.x == 0) {
        if (n_out) *n_out = kk;
        if (kk < k) raise_err(d, SAE_E_EMPTY);
      }
    }
  }
  store_state(c);
  if (c.GP > 1) issue(c, CMD_EXIT);
}

// sae_select: the fused score/select pass alone (K3, Alg.1 Evict's choice of m victims,
// P:504-525), `passes` times back to back, read-only: no block is removed and no counter,
// parameter or clock of the replica changes.  Only the carried per-segment thresholds are
// written back -- a performance hint that exactness never depends on (§6) -- and the
// diagnostics (phase timers, pass and candidate counts).
__global__ void __launch_bounds__(NT, MINB) k_select(Dev d, uint32_t r, uint32_t m, double now,
                                                  uint32_t passes, uint32_t* vids, uint32_t* n_out) {
  Ctx c = make_ctx(d, r, blockIdx.x);
  if (blockIdx.x != 0) {
    worker_loop(c);
    return;
  }
  group_open(c);
  load_state(c);
  RState& st = c.s->st;
  bool ok = st.err == 0;
  if (ok && st.has_now && now < st.now) {
    if (threadIdx.x == 0) raise_err(d, SAE_E_TIME);
    ok = false;
  }
  const uint32_t mm = min(m, st.live);
  if (ok && mm > 0) {
    cta_sync();
    if (threadIdx.x == 0) st.now = now;
    cta_sync();
    for (uint32_t p = 0; p < passes; ++p) select_chunk(c, mm, 0xFFFFFFFFu, false);
    for (uint32_t v = threadIdx.x; v < mm; v += NT)
      vids[v] = __ldcg(d.bid + c.base + (c.cand[v].ss & SLOT_MASK));
    cta_sync();
    // carry the thresholds only (exactness never depends on them), plus the diagnostics
    // (phase timers, pass / candidate counts: no replica semantics)
    if (threadIdx.x < 16) {
      d.st[c.r].thr[threadIdx.x] = st.thr[threadIdx.x];
      d.st[c.r].tph[threadIdx.x] = st.tph[threadIdx.x];
    }
    if (threadIdx.x == 0) {
      d.st[c.r].select_passes = st.select_passes;
      d.st[c.r].select_cands = st.select_cands;
      d.st[c.r].select_raw = st.select_raw;
      d.st[c.r].select_narrow = st.select_narrow;
      d.st[c.r].select_big = st.select_big;
    }
  }
  if (threadIdx.x == 0 && n_out) *n_out = ok ? mm : 0u;
  cta_sync();
  if (c.GP > 1) issue(c, CMD_EXIT);
}

__global__ void __launch_bounds__(NT, MINB) k_update(Dev d, uint32_t r0, uint32_t r1) {
  const uint32_t r = r0 + blockIdx.x / d.GP, rank = blockIdx.x % d.GP;
  if (r >= r1) return;
  Ctx c = make_ctx(d, r, rank);
  if (rank != 0) {
    worker_loop(c);
    return;
  }
  group_open(c);
  load_state(c);
  learn(c);
  store_state(c);
  if (c.GP > 1) issue(c, CMD_EXIT);
}


// dynamic shared memory of one replay CTA of this variant
inline size_t smem_bytes() {
  return ((sizeof(Smem) + 15) / 16) * 16 + sizeof(Cand) * ((CAND_GLOBAL ? 0 : CAND_MAX) + VCAP);
}
