// SAECache CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct replay of the SAECache eviction policy
// (arxiv 2605.18825, /root/reference/PAPER.md = "P:<line>") written directly
// from the paper, in the paper's order, in IEEE binary64 with no FMA
// contraction (build with -O2 -ffp-contract=off -fno-fast-math).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load this library.  It shares no code, header, table or constant
// generator with the CUDA path (paper_2605_18825_b200/csrc); the two are
// written independently and compared element by element.
//
// Readings of silent / conflicting passages follow SURVEY.md §8(c) and are
// listed in DESIGN.md ("Readings").  Every function cites the passage it
// implements.  Parity-pinned by tests/test_oracle_*.py;
// functions without an independent pin say "parity unpinned" below.

#include <cstdint>
#include <cstring>
#include <cmath>      // sqrt only (IEEE correctly rounded); no libm transcendentals
#include <vector>
#include <deque>
#include <unordered_map>
#include <unordered_set>
#include <set>
#include <algorithm>
#include <tuple>
#include <thread>
#include <cstdlib>

namespace orc {

// ---------------------------------------------------------------------------
// 0. bit helpers
// ---------------------------------------------------------------------------
static inline uint64_t bits_of(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
static inline double dbl_of(uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; }
static inline int32_t hi_word(double x) { return (int32_t)(bits_of(x) >> 32); }
static inline uint32_t lo_word(double x) { return (uint32_t)bits_of(x); }
static inline double with_hi(double x, int32_t hi) {
  return dbl_of(((uint64_t)(uint32_t)hi << 32) | (uint64_t)lo_word(x));
}
static inline double with_lo(double x, uint32_t lo) {
  return dbl_of((bits_of(x) & 0xFFFFFFFF00000000ull) | (uint64_t)lo);
}

// ---------------------------------------------------------------------------
// 1. Transcendentals: our own implementations of the fdlibm 5.3 algorithms
//    (e_log.c, e_exp.c, s_erf.c:erfc).  SURVEY §8(c) c.4: never call libm on
//    a path that feeds P or a learned parameter.  Pinned against mpmath
//    (tests/test_oracle_math.py).
// ---------------------------------------------------------------------------
static const double ln2_hi = 6.93147180369123816490e-01;  // 3fe62e42 fee00000
static const double ln2_lo = 1.90821492927058770002e-10;  // 3dea39ef 35793c76
static const double two54 = 1.80143985094819840000e+16;   // 43500000 00000000
static const double Lg1 = 6.666666666666735130e-01;  // 3FE55555 55555593
static const double Lg2 = 3.999999999940941908e-01;  // 3FD99999 9997FA04
static const double Lg3 = 2.857142874366239149e-01;  // 3FD24924 94229359
static const double Lg4 = 2.222219843214978396e-01;  // 3FCC71C5 1D8E78AF
static const double Lg5 = 1.818357216161805012e-01;  // 3FC74664 96CB03DE
static const double Lg6 = 1.531383769920937332e-01;  // 3FC39A09 D078C69F
static const double Lg7 = 1.479819860511658591e-01;  // 3FC2F112 DF3E5244

double ln(double x) {
  double hfsq, f, s, z, R, w, t1, t2, dk;
  int32_t k, hx, i, j;
  uint32_t lx;
  hx = hi_word(x);
  lx = lo_word(x);
  k = 0;
  if (hx < 0x00100000) {                       // x < 2**-1022
    if (((hx & 0x7fffffff) | lx) == 0) return -two54 / 0.0;  // log(+-0) = -inf
    if (hx < 0) return (x - x) / 0.0;          // log(-#) = NaN
    k -= 54;
    x *= two54;                                // subnormal: scale up
    hx = hi_word(x);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  i = (hx + 0x95f64) & 0x100000;
  x = with_hi(x, hx | (i ^ 0x3ff00000));       // normalize x or x/2
  k += (i >> 20);
  f = x - 1.0;
  if ((0x000fffff & (2 + hx)) < 3) {           // |f| < 2**-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      dk = (double)k;
      return dk * ln2_hi + dk * ln2_lo;
    }
    R = f * f * (0.5 - 0.33333333333333333 * f);
    if (k == 0) return f - R;
    dk = (double)k;
    return dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  s = f / (2.0 + f);
  dk = (double)k;
  z = s * s;
  i = hx - 0x6147a;
  w = z * z;
  j = 0x6b851 - hx;
  t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  R = t2 + t1;
  if (i > 0) {
    hfsq = 0.5 * f * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

static const double halF[2] = {0.5, -0.5};
static const double huge_v = 1.0e+300;
static const double twom1000 = 9.33263618503218878990e-302;     // 2**-1000
static const double o_threshold = 7.09782712893383973096e+02;   // 40862E42 FEFA39EF
static const double u_threshold = -7.45133219101941108420e+02;  // c0874910 D52D3051
static const double ln2HI[2] = {6.93147180369123816490e-01, -6.93147180369123816490e-01};
static const double ln2LO[2] = {1.90821492927058770002e-10, -1.90821492927058770002e-10};
static const double invln2 = 1.44269504088896338700e+00;        // 3ff71547 652b82fe
static const double P1 = 1.66666666666666019037e-01;   // 3FC55555 5555553E
static const double P2 = -2.77777777770155933842e-03;  // BF66C16C 16BEBD93
static const double P3 = 6.61375632143793436117e-05;   // 3F11566A AF25DE2C
static const double P4 = -1.65339022054652515390e-06;  // BEBBBD41 C5D26BF1
static const double P5 = 4.13813679705723846039e-08;   // 3E663769 72BEA4D0

double exp_(double x) {
  double y, hi = 0.0, lo = 0.0, c, t;
  int32_t k = 0, xsb;
  uint32_t hx;
  hx = (uint32_t)hi_word(x);
  xsb = (int32_t)((hx >> 31) & 1);
  hx &= 0x7fffffff;
  if (hx >= 0x40862E42) {                       // |x| >= 709.78...
    if (hx >= 0x7ff00000) {
      if (((hx & 0xfffff) | lo_word(x)) != 0) return x + x;  // NaN
      return (xsb == 0) ? x : 0.0;                           // exp(+-inf)
    }
    if (x > o_threshold) return huge_v * huge_v;
    if (x < u_threshold) return twom1000 * twom1000;
  }
  if (hx > 0x3fd62e42) {                        // |x| > 0.5 ln2
    if (hx < 0x3FF0A2B2) {                      // and |x| < 1.5 ln2
      hi = x - ln2HI[xsb];
      lo = ln2LO[xsb];
      k = 1 - xsb - xsb;
    } else {
      k = (int32_t)(invln2 * x + halF[xsb]);
      t = (double)k;
      hi = x - t * ln2HI[0];
      lo = t * ln2LO[0];
    }
    x = hi - lo;
  } else if (hx < 0x3e300000) {                 // |x| < 2**-28
    if (huge_v + x > 1.0) return 1.0 + x;
  } else {
    k = 0;
  }
  t = x * x;
  c = x - t * (P1 + t * (P2 + t * (P3 + t * (P4 + t * P5))));
  if (k == 0) return 1.0 - ((x * c) / (c - 2.0) - x);
  y = 1.0 - ((lo - (x * c) / (2.0 - c)) - hi);
  if (k >= -1021) {
    return with_hi(y, (int32_t)((uint32_t)hi_word(y) + ((uint32_t)k << 20)));
  }
  y = with_hi(y, (int32_t)((uint32_t)hi_word(y) + ((uint32_t)(k + 1000) << 20)));
  return y * twom1000;
}

// s_erf.c coefficients
static const double tiny = 1e-300;
static const double erx = 8.45062911510467529297e-01;   // 3FEB0AC1 60000000
static const double pp0 = 1.28379167095512558561e-01;   // 3FC06EBA 8214DB68
static const double pp1 = -3.25042107247001499370e-01;  // BFD4CD7D 691CB913
static const double pp2 = -2.84817495755985104766e-02;  // BF9D2A51 DBD7194F
static const double pp3 = -5.77027029648944159157e-03;  // BF77A291 236668E4
static const double pp4 = -2.37630166566501626084e-05;  // BEF8EAD6 120016AC
static const double qq1 = 3.97917223959155352819e-01;   // 3FD97779 CDDADC09
static const double qq2 = 6.50222499887672944485e-02;   // 3FB0A54C 5536CEBA
static const double qq3 = 5.08130628187576562776e-03;   // 3F74D022 C4D36B0F
static const double qq4 = 1.32494738004321644526e-04;   // 3F215DC9 221C1A10
static const double qq5 = -3.96022827877536812320e-06;  // BED09C43 42A26120
static const double pa0 = -2.36211856075265944077e-03;  // BF6359B8 BEF77538
static const double pa1 = 4.14856118683748331666e-01;   // 3FDA8D00 AD92B34D
static const double pa2 = -3.72207876035701323847e-01;  // BFD7D240 FBB8C3F1
static const double pa3 = 3.18346619901161753674e-01;   // 3FD45FCA 805120E4
static const double pa4 = -1.10894694282396677476e-01;  // BFBC6398 3D3E28EC
static const double pa5 = 3.54783043256182359371e-02;   // 3FA22A36 599795EB
static const double pa6 = -2.16637559486879084300e-03;  // BF61BF38 0A96073F
static const double qa1 = 1.06420880400844228286e-01;   // 3FBB3E66 18EEE323
static const double qa2 = 5.40397917702171048937e-01;   // 3FE14AF0 92EB6F33
static const double qa3 = 7.18286544141962662868e-02;   // 3FB2635C D99FE9A7
static const double qa4 = 1.26171219808761642112e-01;   // 3FC02660 E763351F
static const double qa5 = 1.36370839120290507362e-02;   // 3F8BEDC2 6B51DD1C
static const double qa6 = 1.19844998467991074170e-02;   // 3F888B54 5735151D
static const double ra0 = -9.86494403484714822705e-03;  // BF843412 600D6435
static const double ra1 = -6.93858572707181764372e-01;  // BFE63416 E4BA7360
static const double ra2 = -1.05586262253232909814e+01;  // C0251E04 41B0E726
static const double ra3 = -6.23753324503260060396e+01;  // C04F300A E4CBA38D
static const double ra4 = -1.62396669462573470355e+02;  // C0644CB1 84282266
static const double ra5 = -1.84605092906711035994e+02;  // C067135C EBCCABB2
static const double ra6 = -8.12874355063065934246e+01;  // C0545265 57E4D2F2
static const double ra7 = -9.81432934416914548592e+00;  // C023A0EF C69AC25C
static const double sa1 = 1.96512716674392571292e+01;   // 4033A6B9 BD707687
static const double sa2 = 1.37657754143519042600e+02;   // 4061350C 526AE721
static const double sa3 = 4.34565877475229228821e+02;   // 407B290D D58A1A71
static const double sa4 = 6.45387271733267880336e+02;   // 40842B19 21EC2868
static const double sa5 = 4.29008140027567833386e+02;   // 407AD021 57700314
static const double sa6 = 1.08635005541779435134e+02;   // 405B28A3 EE48AE2C
static const double sa7 = 6.57024977031928170135e+00;   // 401A47EF 8E484A93
static const double sa8 = -6.04244152148580987438e-02;  // BFAEEFF2 EE749A62
static const double rb0 = -9.86494292470009928597e-03;  // BF843412 39E86F4A
static const double rb1 = -7.99283237680523006574e-01;  // BFE993BA 70C285DE
static const double rb2 = -1.77579549177547519889e+01;  // C031C209 555F995A
static const double rb3 = -1.60636384855821916062e+02;  // C064145D 43C5ED98
static const double rb4 = -6.37566443368389627722e+02;  // C083EC88 1375F228
static const double rb5 = -1.02509513161107724954e+03;  // C0900461 6A2E5992
static const double rb6 = -4.83519191608651397019e+02;  // C07E384E 9BDC383F
static const double sb1 = 3.03380607434824582924e+01;   // 403E568B 261D5190
static const double sb2 = 3.25792512996573918826e+02;   // 40745CAE 221B9F0A
static const double sb3 = 1.53672958608443695994e+03;   // 409802EB 189D5118
static const double sb4 = 3.19985821950859553908e+03;   // 40A8FFB7 688C246A
static const double sb5 = 2.55305040643316442583e+03;   // 40A3F219 CEDF3BE6
static const double sb6 = 4.74528541206955367215e+02;   // 407DA874 E79FE763
static const double sb7 = -2.24409524465858183362e+01;  // C03670E2 42712D62

double erfc_(double x) {
  int32_t hx, ix;
  double R, S, P, Q, s, y, z, r;
  hx = hi_word(x);
  ix = hx & 0x7fffffff;
  if (ix >= 0x7ff00000) return (double)(((uint32_t)hx >> 31) << 1) + 1.0 / x;
  if (ix < 0x3feb0000) {                       // |x| < 0.84375
    if (ix < 0x3c700000) return 1.0 - x;       // |x| < 2**-56
    z = x * x;
    r = pp0 + z * (pp1 + z * (pp2 + z * (pp3 + z * pp4)));
    s = 1.0 + z * (qq1 + z * (qq2 + z * (qq3 + z * (qq4 + z * qq5))));
    y = r / s;
    if (hx < 0x3fd00000) return 1.0 - (x + x * y);   // x < 1/4
    r = x * y;
    r += (x - 0.5);
    return 0.5 - r;
  }
  if (ix < 0x3ff40000) {                       // 0.84375 <= |x| < 1.25
    s = std::fabs(x) - 1.0;
    P = pa0 + s * (pa1 + s * (pa2 + s * (pa3 + s * (pa4 + s * (pa5 + s * pa6)))));
    Q = 1.0 + s * (qa1 + s * (qa2 + s * (qa3 + s * (qa4 + s * (qa5 + s * qa6)))));
    if (hx >= 0) {
      z = 1.0 - erx;
      return z - P / Q;
    }
    z = erx + P / Q;
    return 1.0 + z;
  }
  if (ix < 0x403c0000) {                       // |x| < 28
    x = std::fabs(x);
    s = 1.0 / (x * x);
    if (ix < 0x4006DB6D) {                     // |x| < 1/.35
      R = ra0 + s * (ra1 + s * (ra2 + s * (ra3 + s * (ra4 + s * (ra5 + s * (ra6 + s * ra7))))));
      S = 1.0 + s * (sa1 + s * (sa2 + s * (sa3 + s * (sa4 + s * (sa5 + s * (sa6 + s * (sa7 + s * sa8)))))));
    } else {                                   // |x| >= 1/.35
      if (hx < 0 && ix >= 0x40180000) return 2.0 - tiny;  // x < -6
      R = rb0 + s * (rb1 + s * (rb2 + s * (rb3 + s * (rb4 + s * (rb5 + s * rb6)))));
      S = 1.0 + s * (sb1 + s * (sb2 + s * (sb3 + s * (sb4 + s * (sb5 + s * (sb6 + s * sb7))))));
    }
    z = with_lo(x, 0);
    r = exp_(-z * z - 0.5625) * exp_((z - x) * (z + x) + R / S);
    if (hx > 0) return r / x;
    return 2.0 - r / x;
  }
  if (hx > 0) return tiny * tiny;
  return 2.0 - tiny;
}

// ---------------------------------------------------------------------------
// 2. Chained block hashing (P:158-159 strict prefix matching, P:319 16-token
//    blocks; reading A1: XXH64 with seed 0 over le64(prev) || le32(tokens)).
//    XXH64 pinned against the python `xxhash` package.
// ---------------------------------------------------------------------------
static const uint64_t XP1 = 0x9E3779B185EBCA87ull;
static const uint64_t XP2 = 0xC2B2AE3D27D4EB4Full;
static const uint64_t XP3 = 0x165667B19E3779F9ull;
static const uint64_t XP4 = 0x85EBCA77C2B2AE63ull;
static const uint64_t XP5 = 0x27D4EB2F165667C5ull;
static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static inline uint64_t rd64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
static inline uint32_t rd32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static inline uint64_t xround(uint64_t acc, uint64_t in) {
  acc += in * XP2;
  acc = rotl64(acc, 31);
  return acc * XP1;
}
static inline uint64_t xmerge(uint64_t acc, uint64_t v) {
  acc ^= xround(0, v);
  return acc * XP1 + XP4;
}

uint64_t xxh64(const uint8_t* p, size_t len, uint64_t seed) {
  const uint8_t* end = p + len;
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = seed + XP1 + XP2, v2 = seed + XP2, v3 = seed, v4 = seed - XP1;
    const uint8_t* limit = end - 32;
    do {
      v1 = xround(v1, rd64(p)); p += 8;
      v2 = xround(v2, rd64(p)); p += 8;
      v3 = xround(v3, rd64(p)); p += 8;
      v4 = xround(v4, rd64(p)); p += 8;
    } while (p <= limit);
    h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
    h = xmerge(h, v1); h = xmerge(h, v2); h = xmerge(h, v3); h = xmerge(h, v4);
  } else {
    h = seed + XP5;
  }
  h += (uint64_t)len;
  while (p + 8 <= end) {
    h ^= xround(0, rd64(p));
    h = rotl64(h, 27) * XP1 + XP4;
    p += 8;
  }
  if (p + 4 <= end) {
    h ^= (uint64_t)rd32(p) * XP1;
    h = rotl64(h, 23) * XP2 + XP3;
    p += 4;
  }
  while (p < end) {
    h ^= (uint64_t)(*p) * XP5;
    h = rotl64(h, 11) * XP1;
    ++p;
  }
  h ^= h >> 33; h *= XP2;
  h ^= h >> 29; h *= XP3;
  h ^= h >> 32;
  return h;
}

// H_j = XXH64(le64(H_{j-1}) || le32(tok_j[0..n_j-1]), seed 0)  (SURVEY c.2 O2)
uint64_t block_hash(uint64_t prev, const uint32_t* tok, uint32_t n) {
  std::vector<uint8_t> buf(8 + 4 * (size_t)n);
  for (int i = 0; i < 8; ++i) buf[i] = (uint8_t)(prev >> (8 * i));
  for (uint32_t t = 0; t < n; ++t)
    for (int i = 0; i < 4; ++i) buf[8 + 4 * t + i] = (uint8_t)(tok[t] >> (8 * i));
  return xxh64(buf.data(), buf.size(), 0);
}

// ---------------------------------------------------------------------------
// 3. Policy constants and state
// ---------------------------------------------------------------------------
enum { Q_EF = 0, Q_CHAT = 1, Q_AGENT = 2, Q_STRUCT = 3 };
enum { T_SYS = 0, T_USER = 1, T_TOOL = 2, T_RESP = 3, T_COT = 4, T_DECODE = 5 };
enum { L_TOKENS = 1, L_QUEUES = 2, L_LOGNORMAL = 4, L_DECAY = 8, L_TOKEN_MULT = 16, L_QUEUE_RELATIVE = 32,
       L_ADAPTIVE_BETA = 64 };
// Baselines of the paper's comparison and ablation, on the same replay:
//  MODE_LRU   victim = least recently used: argmin (last, id)
//  MODE_LFU   victim = least frequently used: argmin (accesses, last, id)
//  MODE_TWO   Token-Weight-Only: the token-type weights without the multi-queue
//             architecture: argmin (w_tau / dt, last, id); decode blocks weigh as CoT
// In the baselines every block sits in one queue (CHAT); counters and learners run as usual.
enum { MODE_SAE = 0, MODE_LRU = 1, MODE_LFU = 2, MODE_TWO = 3 };
static const double INV_SQRT2 = 0.70710678118654757;  // 0x3FE6A09E667F3BCD

}  // namespace orc

extern "C" {

// Parameters (learned values + meta-parameters), SURVEY §8(c) c.5.
typedef struct {
  double w[5], alpha[3], mu[2], sigma[2], gamma;
  double eta, a_miss, b_reuse, T, beta_q, beta_ln, beta_gamma;
  uint32_t learn_flags;
  uint32_t mode;        // eviction policy: 0 SAECache, 1 LRU, 2 LFU, 3 Token-Weight-Only
} orc_params;

typedef struct {
  uint32_t block_tokens, capacity, ghost_capacity, K, interval_ring, interval_keep,
      interval_min, n_bins;
  uint64_t hash_seed;
  double dt_eps, z_cut;
  orc_params init;
} orc_config;

// One trajectory snapshot per learner firing (SURVEY c.3 "Trajectory output").
typedef struct {
  uint64_t E, request;
  double w[5], alpha[3], mu[2], sigma[2], gamma;
} orc_traj;

typedef struct {
  uint64_t requests, blocks_looked_up, hit_blocks, hit_tokens, prompt_tokens;
  uint64_t evictions, evict_by_queue[4], evict_by_type[6], mae_by_type[6];
  uint64_t learner_firings, eviction_rounds, blocks_scored, resident, resident_by_queue[4];
  uint64_t E, next_id, gseq;
  double now;
  uint64_t ts_ev[5], ts_mae[5], ts_hit[5], ts_acc[5];
  uint64_t qh[3], qe[3], pb_hit[16], pb_acc[16];
  uint64_t iv_len[2];
} orc_stats;

}  // extern "C"

namespace orc {

struct Block {
  uint32_t id;
  double last;
  uint64_t acc;
  uint8_t ntok, q, tau;
  uint32_t ob, omax;
};

struct Replica {
  orc_config cfg;
  orc_params par;
  std::unordered_map<uint64_t, Block> res;        // resident block table (D11)
  uint64_t next_id = 0;
  // recently_evicted: ghost FIFO ring + map hash -> (tau, seq) (A30)
  std::vector<std::pair<uint64_t, uint64_t>> gh;  // (hash, seq)
  std::vector<uint8_t> gh_used;
  std::unordered_map<uint64_t, std::pair<uint8_t, uint64_t>> gmap;
  uint64_t gseq = 0;
  uint64_t ts_ev[5] = {0}, ts_mae[5] = {0}, ts_hit[5] = {0}, ts_acc[5] = {0};  // D5
  uint64_t qh[3] = {0}, qe[3] = {0};                                          // D6
  std::deque<double> iv[2];                                                   // D7 ln(dt)
  std::vector<uint64_t> pb_hit, pb_acc;                                       // D8
  uint64_t E = 0;
  double now = -INFINITY;
  bool have_now = false;
  uint64_t req_index = 0;
  orc_stats st;
  std::vector<orc_traj> traj;
};

// Eq. (1): p = 1 - F_LN(dt; mu, sigma) = 0.5*erfc(z/sqrt2), z=(ln dt - mu)/sigma
// (reading A36: 0.5*erfc with z > z_cut -> 0).
double survival(double dt, double mu, double sg, double z_cut) {
  double z = (ln(dt) - mu) / sg;
  if (z > z_cut) return 0.0;
  return 0.5 * erfc_(z * INV_SQRT2);
}

// Eq. (2): p = 1 - (o_b/o_max)^gamma, pow(x,y) = exp(y*ln x) (c.4)
double p_struct(uint32_t ob, uint32_t omax, double gam) {
  if (ob == 0) return 1.0;
  double r = (double)ob / (double)omax;
  return 1.0 - exp_(gam * ln(r));
}

// Eq. (3), P:322-325 (Alg.1 line P:516): P = alpha_q * w_tau * p_q / dt, left to right.
double score(const Replica& R, const Block& b, double now) {
  double dt = now - b.last;
  if (dt < R.cfg.dt_eps) dt = R.cfg.dt_eps;  // A7
  double p;
  int qi = b.q - 1;
  if (b.q == Q_CHAT || b.q == Q_AGENT) {
    p = survival(dt, R.par.mu[qi], R.par.sigma[qi], R.cfg.z_cut);
  } else {
    p = p_struct(b.ob, b.omax, R.par.gamma);
  }
  return ((R.par.alpha[qi] * R.par.w[b.tau]) * p) / dt;
}

// Alg.1 Classify, P:550-564 (SURVEY c.2 O4).
int classify(int tau, bool mt, bool ag, bool cid, bool is_struct, bool untempl) {
  if (tau == T_COT || tau == T_DECODE || untempl) return Q_EF;
  if (mt && ag) return Q_AGENT;
  if (mt || cid) return Q_CHAT;
  if (is_struct || tau == T_SYS) return Q_STRUCT;
  return Q_EF;
}

// Stride-halving tree sum (SURVEY c.3 TREE): pad to a power of two P >= n with
// +0.0, then y[i] += y[i+h] for h = P/2 .. 1.
double tree_sum(std::vector<double> y) {
  size_t n = y.size();
  if (n == 0) return 0.0;
  size_t P = 1;
  while (P < n) P <<= 1;
  y.resize(P, 0.0);
  for (size_t h = P / 2; h >= 1; h >>= 1) {
    for (size_t i = 0; i < h; ++i) y[i] = y[i] + y[i + h];
    if (h == 1) break;
  }
  return y[0];
}

static inline double clampd(double x, double lo, double hi) {
  return x < lo ? lo : (x > hi ? hi : x);
}

// --- Learners (Appendix B), order of Alg.1 P:542-544 + DecayPower ---

// TokenWeights: prose target P:703-707 (default, A16) or Alg. P:714-734 (TOKEN_MULT);
// threshold, clamp and floor-decay from Alg. P:722-730 (A17: lambda = 99/100).
void learn_tokens(Replica& R) {
  orc_params& p = R.par;
  for (int t = 0; t < 5; ++t) {
    if (R.ts_ev[t] > 10) {
      double rm = (double)R.ts_mae[t] / (double)R.ts_ev[t];
      double rr = R.ts_acc[t] > 0 ? (double)R.ts_hit[t] / (double)R.ts_acc[t] : 0.0;
      if (p.learn_flags & L_TOKEN_MULT) {
        p.w[t] = p.w[t] * (1.0 + p.eta * rm);
      } else {
        double tgt = (1.0 + rm * p.a_miss) + rr * p.b_reuse;
        p.w[t] = (1.0 - p.eta) * p.w[t] + p.eta * tgt;
      }
      p.w[t] = clampd(p.w[t], 0.1, 5.0);
    }
  }
  for (int t = 0; t < 5; ++t) {
    R.ts_ev[t] = (99 * R.ts_ev[t]) / 100;
    R.ts_mae[t] = (99 * R.ts_mae[t]) / 100;
    R.ts_hit[t] = (99 * R.ts_hit[t]) / 100;
    R.ts_acc[t] = (99 * R.ts_acc[t]) / 100;
  }
}

// QueueWeights: Alg. P:575-597 (default, A19) or relative rule P:814-817.
void learn_queues(Replica& R) {
  orc_params& p = R.par;
  if (p.learn_flags & L_QUEUE_RELATIVE) {
    uint64_t cnt[3] = {0, 0, 0};
    for (auto& kv : R.res)
      if (kv.second.q != Q_EF) cnt[kv.second.q - 1]++;
    double Eq[3];
    bool def[3];
    double sum = 0.0;
    int nd = 0;
    for (int q = 0; q < 3; ++q) {
      double frac = (double)cnt[q] / (double)R.cfg.capacity;
      def[q] = frac > 0.0;
      if (def[q]) {
        Eq[q] = (double)R.qh[q] / frac;
        sum = sum + Eq[q];
        nd++;
      }
    }
    if (nd > 0) {
      double Ebar = sum / (double)nd;
      if (Ebar > 0.0) {
        for (int q = 0; q < 3; ++q) {
          if (!def[q]) continue;
          double x = Eq[q] / Ebar;
          double pw = (x == 0.0) ? 0.0 : exp_(ln(x) / p.T);
          p.alpha[q] = p.alpha[q] + p.beta_q * (pw - p.alpha[q]);
          p.alpha[q] = clampd(p.alpha[q], 0.1, 3.0);
        }
      }
    }
  } else {
    for (int q = 0; q < 3; ++q) {
      if (R.qe[q] > 5) {
        double eff = (double)R.qh[q] / (double)R.qe[q];
        double tgt = 1.0 + eff / p.T;
        p.alpha[q] = p.alpha[q] + p.beta_q * (tgt - p.alpha[q]);
        p.alpha[q] = clampd(p.alpha[q], 0.1, 3.0);
      }
    }
  }
  for (int q = 0; q < 3; ++q) { R.qh[q] = 0; R.qe[q] = 0; }
}

// LognormalParams: Alg. P:762-784 (threshold > 20 per A23; population std A24); with
// L_ADAPTIVE_BETA the EMA factor adapts to the observation variance (A28).
void learn_lognormal(Replica& R) {
  orc_params& p = R.par;
  for (int s = 0; s < 2; ++s) {
    std::deque<double>& iv = R.iv[s];
    size_t n = iv.size();
    if (n > R.cfg.interval_min) {
      std::vector<double> x(iv.begin(), iv.end());
      double m = tree_sum(x) / (double)n;
      std::vector<double> d(n);
      for (size_t i = 0; i < n; ++i) d[i] = (x[i] - m) * (x[i] - m);
      double v = tree_sum(d) / (double)n;
      double sd = std::sqrt(v);
      double b = p.beta_ln;
      if (p.learn_flags & L_ADAPTIVE_BETA) {
        // adaptive EMA factor (reading A28): the observations' variance around the
        // CURRENT model, v_obs = mean (x - mu)^2, against the model's sigma^2: high (rho > 1)
        // -> track faster (beta doubled, at most 1), low -> steadier (beta halved)
        for (size_t i = 0; i < n; ++i) d[i] = (x[i] - p.mu[s]) * (x[i] - p.mu[s]);
        double vobs = tree_sum(d) / (double)n;
        double rho = vobs / (p.sigma[s] * p.sigma[s]);
        b = rho > 1.0 ? std::min(2.0 * p.beta_ln, 1.0) : 0.5 * p.beta_ln;
      }
      p.mu[s] = p.mu[s] + b * (m - p.mu[s]);
      p.sigma[s] = p.sigma[s] + b * (sd - p.sigma[s]);
      if (p.sigma[s] < 0.1) p.sigma[s] = 0.1;
      while (iv.size() > R.cfg.interval_keep) iv.pop_front();
    }
  }
}

// DecayPower: P:786-803 (A27).
void learn_decay(Replica& R) {
  orc_params& p = R.par;
  uint32_t NB = R.cfg.n_bins, half = NB / 2;
  double fs = 0.0, bs = 0.0;
  int fc = 0, bc = 0;
  for (uint32_t i = 0; i < NB; ++i) {
    if (R.pb_acc[i] == 0) continue;
    double rate = (double)R.pb_hit[i] / (double)R.pb_acc[i];
    if (i < half) { fs = fs + rate; fc++; }
    else { bs = bs + rate; bc++; }
  }
  if (fc > 0 && bc > 0) {
    double fa = fs / (double)fc;
    double ba = bs / (double)bc;
    if (fa > 0.0) {
      double ratio = ba / fa;
      double est = 1.0 / (ratio + 0.1);
      p.gamma = p.gamma + p.beta_gamma * (est - p.gamma);
      p.gamma = clampd(p.gamma, 0.3, 3.0);
    }
  }
  for (uint32_t i = 0; i < NB; ++i) {
    R.pb_hit[i] = (99 * R.pb_hit[i]) / 100;
    R.pb_acc[i] = (99 * R.pb_acc[i]) / 100;
  }
}

void learn(Replica& R) {
  uint32_t f = R.par.learn_flags;
  if (f & L_TOKENS) learn_tokens(R);
  if (f & L_QUEUES) learn_queues(R);
  if (f & L_LOGNORMAL) learn_lognormal(R);
  if (f & L_DECAY) learn_decay(R);
  R.st.learner_firings++;
  orc_traj t;
  t.E = R.E;
  t.request = R.req_index;
  std::memcpy(t.w, R.par.w, sizeof t.w);
  std::memcpy(t.alpha, R.par.alpha, sizeof t.alpha);
  std::memcpy(t.mu, R.par.mu, sizeof t.mu);
  std::memcpy(t.sigma, R.par.sigma, sizeof t.sigma);
  t.gamma = R.par.gamma;
  R.traj.push_back(t);
}

// Ghost push, SURVEY c.2 O11 step 3 (A30: FIFO of G entries, consumed on match).
void ghost_push(Replica& R, uint64_t hash, uint8_t tau) {
  uint64_t s = R.gseq++;
  size_t slot = (size_t)(s % R.cfg.ghost_capacity);
  if (R.gh_used[slot]) {
    uint64_t oh = R.gh[slot].first, os = R.gh[slot].second;
    auto it = R.gmap.find(oh);
    if (it != R.gmap.end() && it->second.second == os) R.gmap.erase(it);
  }
  R.gh[slot] = {hash, s};
  R.gh_used[slot] = 1;
  R.gmap[hash] = {tau, s};
}

// Threads for the key computation of large pools: ORACLE_THREADS, else every host core.
static size_t oracle_threads() {
  if (const char* e = std::getenv("ORACLE_THREADS")) {
    const long v = std::atol(e);
    if (v >= 1) return (size_t)v;
  }
  const unsigned h = std::thread::hardware_concurrency();
  return h ? h : 1;
}

// Remove one victim (SURVEY c.2 O11 steps 1-4), with Alg.1 K trigger (A14).
void evict_one(Replica& R, uint64_t hash, std::vector<uint32_t>& out) {
  auto it = R.res.find(hash);
  Block b = it->second;
  R.res.erase(it);
  out.push_back(b.id);
  if (b.tau < 5) R.ts_ev[b.tau]++;
  if (b.q != Q_EF) R.qe[b.q - 1]++;
  R.st.evictions++;
  R.st.evict_by_queue[b.q]++;
  R.st.evict_by_type[b.tau]++;
  ghost_push(R, hash, b.tau);
  R.E++;
  if (R.E % R.cfg.K == 0) learn(R);
}

// Alg.1 Evict() x k with a pin set (SURVEY c.2 O11).  Stage 1: EF by
// (num_tokens, id) (A13); Stage 2: global argmin of Eq.3 over the
// scored queues, ties by (last, id) (A13).  Keys are frozen
// between learner firings, so each chunk computes every key once and takes
// them in order (identical to k sequential argmin scans).
void evict_k(Replica& R, uint64_t k, const std::unordered_map<uint64_t, int>* pin,
             std::vector<uint32_t>& out) {
  uint64_t remaining = k;
  while (remaining > 0) {
    uint64_t to_cross = R.cfg.K - (R.E % R.cfg.K);
    uint64_t m = std::min(remaining, to_cross);
    // key = (tier, primary, last, id); tier 0 = EF (ntok, id), tier 1 = scored.
    struct Key {
      int tier;
      double p;      // EF: ntok; scored: P
      double last;
      uint32_t id;
      uint64_t hash;
    };
    // every unpinned resident block's key (Alg.1 scans every block)
    auto pinned = [&](const std::pair<const uint64_t, Block>* kv) { return pin && pin->count(kv->first); };
    auto key_of = [&](const std::pair<const uint64_t, Block>& kv) {
      const Block& b = kv.second;
      Key key;
      key.hash = kv.first;
      key.id = b.id;
      key.last = b.last;
      if (R.par.mode == MODE_LRU) {
        key.tier = 1;
        key.p = b.last;
      } else if (R.par.mode == MODE_LFU) {
        key.tier = 1;
        key.p = (double)b.acc;
      } else if (R.par.mode == MODE_TWO) {
        double dt = R.now - b.last;
        if (dt < R.cfg.dt_eps) dt = R.cfg.dt_eps;
        key.tier = 1;
        key.p = R.par.w[b.tau < 4 ? b.tau : 4] / dt;
      } else if (b.q == Q_EF) {
        key.tier = 0;
        key.p = (double)b.ntok;
        key.last = 0.0;  // EF ordered by (ntok, id) only
      } else {
        key.tier = 1;
        key.p = score(R, b, R.now);
      }
      return key;
    };
    auto less = [](const Key& a, const Key& b) {
      return std::tie(a.tier, a.p, a.last, a.id) < std::tie(b.tier, b.p, b.last, b.id);
    };
    const size_t NB = R.res.size();
    std::vector<Key> keys;
    // Large pools: the same keys computed by T threads over contiguous
    // slices, each keeping its slice's m smallest; the union is then ordered.  The m smallest
    // under a total order do not depend on the partition, so this equals the serial rescan.
    const size_t T = NB >= 16384 ? oracle_threads() : 1;
    size_t N = 0;         // unpinned blocks scored
    if (T <= 1) {
      keys.reserve(NB);
      for (auto& kv : R.res)
        if (!pinned(&kv)) keys.push_back(key_of(kv));
      N = keys.size();
      if (m > N) m = N;
    } else {
      std::vector<size_t> cnt(T, 0);
      std::vector<std::vector<Key>> part(T);
      std::vector<std::thread> th;
      for (size_t t = 0; t < T; ++t)
        th.emplace_back([&, t]() {
          // thread t walks its share of the hash map's buckets (read-only)
          const size_t nb = R.res.bucket_count();
          const size_t lo = nb * t / T, hi = nb * (t + 1) / T;
          std::vector<Key>& v = part[t];
          v.reserve(NB / T + 16);
          for (size_t bk = lo; bk < hi; ++bk)
            for (auto it = R.res.begin(bk); it != R.res.end(bk); ++it)
              if (!pinned(&*it)) v.push_back(key_of(*it));
          cnt[t] = v.size();
          const size_t mm = std::min<size_t>(m, v.size());
          std::partial_sort(v.begin(), v.begin() + (ptrdiff_t)mm, v.end(), less);
          v.resize(mm);
        });
      for (auto& x : th) x.join();
      for (size_t t = 0; t < T; ++t) N += cnt[t];
      for (auto& v : part) keys.insert(keys.end(), v.begin(), v.end());
      if (m > N) m = N;
    }
    R.st.blocks_scored += N;
    std::partial_sort(keys.begin(), keys.begin() + (ptrdiff_t)m, keys.end(), less);
    for (uint64_t i = 0; i < m; ++i) evict_one(R, keys[i].hash, out);
    remaining -= m;
    if (N == 0) break;
  }
}

}  // namespace orc

using namespace orc;

extern "C" {

enum { ORC_OK = 0, ORC_E_INVAL = -1, ORC_E_CAPACITY_ZERO = -2, ORC_E_EMPTY = -3,
       ORC_E_TIME = -5, ORC_E_OVERFLOW = -6 };

// --- pure functions exposed for pins -------------------------------------------------
double orc_ln(double x) { return ln(x); }
double orc_exp(double x) { return exp_(x); }
double orc_erfc(double x) { return erfc_(x); }
uint64_t orc_xxh64(const uint8_t* p, uint64_t len, uint64_t seed) { return xxh64(p, (size_t)len, seed); }
uint64_t orc_block_hash(uint64_t prev, const uint32_t* tok, uint32_t n) { return block_hash(prev, tok, n); }
double orc_survival(double dt, double mu, double sg, double z_cut) { return survival(dt, mu, sg, z_cut); }
double orc_p_struct(uint32_t ob, uint32_t omax, double gam) { return p_struct(ob, omax, gam); }
int orc_classify(int tau, int mt, int ag, int cid, int is_struct, int untempl) {
  return classify(tau, mt != 0, ag != 0, cid != 0, is_struct != 0, untempl != 0);
}
double orc_tree_sum(const double* y, uint64_t n) { return tree_sum(std::vector<double>(y, y + n)); }
double orc_score(double alpha, double w, double p, double dt) { return ((alpha * w) * p) / dt; }

// Eq.(1)-(3) of one block at elapsed time dt through score() itself (a throwaway replica
// holding only the parameters; last = 0, now = dt): for property tests of the priority.
double orc_priority(const orc_params* p, double dt_eps, double z_cut, int q, int tau, double dt,
                    uint32_t ob, uint32_t omax) {
  Replica R;
  R.cfg.dt_eps = dt_eps;
  R.cfg.z_cut = z_cut;
  R.par = *p;
  Block b;
  b.id = 0; b.last = 0.0; b.acc = 1; b.ntok = 16;
  b.q = (uint8_t)q; b.tau = (uint8_t)tau; b.ob = ob; b.omax = omax;
  return score(R, b, dt);
}

// --- replica handle -----------------------------------------------------------------
void* orc_create(const orc_config* cfg) {
  if (!cfg || cfg->capacity == 0 || cfg->ghost_capacity == 0 || cfg->K == 0 ||
      cfg->n_bins == 0 || cfg->n_bins > 16 || cfg->block_tokens == 0)
    return nullptr;
  Replica* R = new Replica();
  R->cfg = *cfg;
  R->par = cfg->init;
  R->gh.assign(cfg->ghost_capacity, {0, 0});
  R->gh_used.assign(cfg->ghost_capacity, 0);
  R->pb_hit.assign(cfg->n_bins, 0);
  R->pb_acc.assign(cfg->n_bins, 0);
  std::memset(&R->st, 0, sizeof R->st);
  return R;
}
void orc_destroy(void* h) { delete (Replica*)h; }
void orc_set_params(void* h, const orc_params* p) { ((Replica*)h)->par = *p; }
void orc_get_params(void* h, orc_params* p) { *p = ((Replica*)h)->par; }

// Hash every block of one request (SURVEY c.2 O1-O3).  Outputs n blocks.
static void hash_request(const orc_config& cfg, const uint32_t* ptok, const uint8_t* ptyp,
                         uint32_t L, const uint32_t* dtok, uint32_t O,
                         std::vector<uint64_t>& H, std::vector<uint8_t>& tau,
                         std::vector<uint8_t>& ntok) {
  uint32_t B = cfg.block_tokens;
  uint32_t np = (L + B - 1) / B, nd = (O + B - 1) / B;
  H.resize(np + nd); tau.resize(np + nd); ntok.resize(np + nd);
  uint64_t prev = cfg.hash_seed;
  for (uint32_t j = 0; j < np; ++j) {
    uint32_t s = j * B, n = std::min(B, L - s);
    prev = block_hash(prev, ptok + s, n);
    H[j] = prev;
    tau[j] = ptyp[s + n / 2];          // A3: median token = index floor(n/2)
    ntok[j] = (uint8_t)n;
  }
  for (uint32_t d = 0; d < nd; ++d) {  // A34: decode span starts a new block chain
    uint32_t s = d * B, n = std::min(B, O - s);
    prev = block_hash(prev, dtok + s, n);
    H[np + d] = prev;
    tau[np + d] = T_DECODE;
    ntok[np + d] = (uint8_t)n;
  }
}

// Replay one request (SURVEY c.2 O1-O13).  Outputs: res4 = {hit_blocks,
// miss_blocks, matched_tokens, n_victims}; victims appended to *vout (cap
// vcap, *vn in/out); block hashes/types optionally written.
int orc_admit(void* h, double now, const uint32_t* ptok, const uint8_t* ptyp, uint32_t L,
              const uint32_t* dtok, uint32_t O, uint32_t flags, uint32_t spb,
              uint32_t* res4, uint32_t* vout, uint64_t vcap, uint64_t* vn,
              uint64_t* hash_out, uint8_t* tau_out) {
  Replica& R = *(Replica*)h;
  const orc_config& cfg = R.cfg;
  if (L < 1) return ORC_E_INVAL;
  if (R.have_now && now < R.now) return ORC_E_TIME;
  R.now = now;
  R.have_now = true;
  std::vector<uint64_t> H;
  std::vector<uint8_t> tau, ntok;
  hash_request(cfg, ptok, ptyp, L, dtok, O, H, tau, ntok);
  uint32_t B = cfg.block_tokens;
  uint32_t np = (L + B - 1) / B;
  uint32_t n = (uint32_t)H.size();
  if (hash_out) for (uint32_t j = 0; j < n; ++j) hash_out[j] = H[j];
  if (tau_out) for (uint32_t j = 0; j < n; ++j) tau_out[j] = tau[j];

  // O4 hint + Classify (A31 untemplated, A32 cid, A8 o_b/o_max)
  bool mt = flags & 1, ag = flags & 2, cid = flags & 4;
  bool untempl = !mt && spb == 0;
  uint32_t omax = std::max<uint32_t>(np - 1, 1);
  std::vector<uint8_t> q(n);
  for (uint32_t j = 0; j < n; ++j)
    q[j] = R.par.mode == MODE_SAE ? (uint8_t)classify(tau[j], mt, ag, cid, j < spb, untempl)
                                  : (uint8_t)Q_CHAT;   // baselines: one queue
  auto bin = [&](uint32_t j) { return std::min<uint32_t>(cfg.n_bins - 1, (cfg.n_bins * j) / omax); };

  // O5 lookup: h = first miss (strict prefix); Pin = resident blocks of the request
  uint32_t hh = n;
  for (uint32_t j = 0; j < n; ++j)
    if (!R.res.count(H[j])) { hh = j; break; }
  std::unordered_map<uint64_t, int> pin;
  for (uint32_t j = 0; j < n; ++j)
    if (R.res.count(H[j])) pin[H[j]] = 1;

  // O6 access statistics (r_reuse denominator A18; positional bins P:793)
  for (uint32_t j = 0; j < n; ++j) {
    if (tau[j] < 5) R.ts_acc[tau[j]]++;
    if (q[j] == Q_STRUCT) R.pb_acc[bin(j)]++;
  }
  // O7 hits (touch; interval recording P:752; hit credited before re-route A9)
  for (uint32_t j = 0; j < hh; ++j) {
    Block& b = R.res[H[j]];
    double dt = now - b.last;
    if (dt < cfg.dt_eps) dt = cfg.dt_eps;  // A26
    if (b.q == Q_CHAT || b.q == Q_AGENT) {
      R.qh[b.q - 1]++;
      std::deque<double>& iv = R.iv[b.q - 1];
      iv.push_back(ln(dt));
      while (iv.size() > cfg.interval_ring) iv.pop_front();  // A25
    } else if (b.q == Q_STRUCT) {
      R.qh[2]++;
    }
    if (tau[j] < 5) R.ts_hit[tau[j]]++;
    if (q[j] == Q_STRUCT) R.pb_hit[bin(j)]++;
    b.last = now;
    b.acc++;
    b.q = q[j]; b.tau = tau[j]; b.ob = j; b.omax = omax;
  }
  // O8 orphans (A10): refreshed in place, counted as misses
  for (uint32_t j = hh; j < n; ++j) {
    auto it = R.res.find(H[j]);
    if (it == R.res.end()) continue;
    Block& b = it->second;
    b.last = now;
    b.q = q[j]; b.tau = tau[j]; b.ob = j; b.omax = omax;
  }
  // O9 miss-after-evict (Alg.1 Add P:535-538), consumed on match (A30)
  std::vector<uint32_t> New;
  for (uint32_t j = hh; j < n; ++j) {
    if (R.res.count(H[j])) continue;
    auto g = R.gmap.find(H[j]);
    if (g != R.gmap.end()) {
      if (g->second.first < 5) R.ts_mae[g->second.first]++;
      R.st.mae_by_type[g->second.first]++;
      R.gmap.erase(g);
    }
    New.push_back(j);
  }
  // O10 admission size (A11)
  uint64_t f = cfg.capacity - R.res.size();
  uint64_t U = R.res.size() - pin.size();
  uint64_t k = New.size() > f ? New.size() - f : 0;
  if (k > U) {
    k = U;
    New.resize(f + U);
  }
  // O11 evictions
  std::vector<uint32_t> victims;
  if (k > 0) {
    R.st.eviction_rounds++;
    evict_k(R, k, &pin, victims);
  }
  // O12 insert (Alg.1 Add: q.insert(b))
  for (uint32_t j : New) {
    if (R.next_id >= 0xFFFFFFFFull) return ORC_E_OVERFLOW;
    Block b;
    b.id = (uint32_t)R.next_id++;
    b.last = now;
    b.acc = 1;
    b.ntok = ntok[j]; b.q = q[j]; b.tau = tau[j]; b.ob = j; b.omax = omax;
    R.res[H[j]] = b;
  }
  // O13 outputs (A41 token-level hit accounting)
  uint32_t matched = 0;
  for (uint32_t j = 0; j < std::min(hh, np); ++j) matched += ntok[j];
  res4[0] = hh;
  res4[1] = n - hh;
  res4[2] = matched;
  res4[3] = (uint32_t)victims.size();
  for (uint32_t v : victims) {
    if (*vn >= vcap) return ORC_E_OVERFLOW;
    vout[(*vn)++] = v;
  }
  R.st.requests++;
  R.st.blocks_looked_up += n;
  R.st.hit_blocks += hh;
  R.st.hit_tokens += matched;
  R.st.prompt_tokens += L;
  R.req_index++;
  return ORC_OK;
}

// Read-only probe (sae_lookup): hit prefix h of a request against current state.
int orc_lookup(void* h, const uint32_t* ptok, const uint8_t* ptyp, uint32_t L,
               const uint32_t* dtok, uint32_t O, uint32_t* hit_out) {
  Replica& R = *(Replica*)h;
  if (L < 1) return ORC_E_INVAL;
  std::vector<uint64_t> H;
  std::vector<uint8_t> tau, ntok;
  hash_request(R.cfg, ptok, ptyp, L, dtok, O, H, tau, ntok);
  uint32_t hh = (uint32_t)H.size();
  for (uint32_t j = 0; j < H.size(); ++j)
    if (!R.res.count(H[j])) { hh = j; break; }
  *hit_out = hh;
  return ORC_OK;
}

// sae_evict: k victims with an empty pin set at time `now`.
int orc_evict(void* h, uint64_t k, double now, uint32_t* vout, uint64_t* n_out) {
  Replica& R = *(Replica*)h;
  if (R.have_now && now < R.now) return ORC_E_TIME;
  R.now = now;
  R.have_now = true;
  std::vector<uint32_t> victims;
  uint64_t kk = std::min<uint64_t>(k, R.res.size());
  if (kk > 0) {
    R.st.eviction_rounds++;
    evict_k(R, kk, nullptr, victims);
  }
  for (size_t i = 0; i < victims.size(); ++i) vout[i] = victims[i];
  *n_out = victims.size();
  return kk < k ? ORC_E_EMPTY : ORC_OK;
}

// sae_update: run L1-L4 now (E unchanged).
void orc_update(void* h) { learn(*(Replica*)h); }

void orc_get_stats(void* h, orc_stats* out) {
  Replica& R = *(Replica*)h;
  orc_stats s = R.st;
  s.resident = R.res.size();
  for (int q = 0; q < 4; ++q) s.resident_by_queue[q] = 0;
  for (auto& kv : R.res) s.resident_by_queue[kv.second.q]++;
  s.E = R.E; s.next_id = R.next_id; s.gseq = R.gseq; s.now = R.now;
  for (int t = 0; t < 5; ++t) {
    s.ts_ev[t] = R.ts_ev[t]; s.ts_mae[t] = R.ts_mae[t];
    s.ts_hit[t] = R.ts_hit[t]; s.ts_acc[t] = R.ts_acc[t];
  }
  for (int q = 0; q < 3; ++q) { s.qh[q] = R.qh[q]; s.qe[q] = R.qe[q]; }
  for (uint32_t i = 0; i < 16; ++i) {
    s.pb_hit[i] = i < R.cfg.n_bins ? R.pb_hit[i] : 0;
    s.pb_acc[i] = i < R.cfg.n_bins ? R.pb_acc[i] : 0;
  }
  s.iv_len[0] = R.iv[0].size();
  s.iv_len[1] = R.iv[1].size();
  *out = s;
}

uint64_t orc_traj_count(void* h) { return ((Replica*)h)->traj.size(); }
uint64_t orc_size(void* h) { return ((Replica*)h)->res.size(); }
void orc_traj_get(void* h, orc_traj* out) {
  Replica& R = *(Replica*)h;
  for (size_t i = 0; i < R.traj.size(); ++i) out[i] = R.traj[i];
}
// Interval deque contents (oldest first), for learner pins.
uint64_t orc_intervals(void* h, int s, double* out, uint64_t cap) {
  Replica& R = *(Replica*)h;
  uint64_t i = 0;
  for (double x : R.iv[s]) { if (i < cap) out[i] = x; ++i; }
  return i;
}
// Resident set dump: (hash, id, last, q, tau, ntok, ob, omax), any order.
uint64_t orc_resident(void* h, uint64_t* hash, uint32_t* id, double* last, uint8_t* q,
                      uint8_t* tau, uint8_t* ntok, uint32_t* ob, uint32_t* omax, uint64_t cap) {
  Replica& R = *(Replica*)h;
  uint64_t i = 0;
  for (auto& kv : R.res) {
    if (i < cap) {
      hash[i] = kv.first; id[i] = kv.second.id; last[i] = kv.second.last;
      q[i] = kv.second.q; tau[i] = kv.second.tau; ntok[i] = kv.second.ntok;
      ob[i] = kv.second.ob; omax[i] = kv.second.omax;
    }
    ++i;
  }
  return i;
}
// Test hooks to drive the learners from hand-set counters.
void orc_set_counters(void* h, const uint64_t* ts4x5, const uint64_t* qh3, const uint64_t* qe3,
                      const uint64_t* pbh, const uint64_t* pba) {
  Replica& R = *(Replica*)h;
  if (ts4x5) for (int t = 0; t < 5; ++t) {
    R.ts_ev[t] = ts4x5[t]; R.ts_mae[t] = ts4x5[5 + t];
    R.ts_hit[t] = ts4x5[10 + t]; R.ts_acc[t] = ts4x5[15 + t];
  }
  if (qh3) for (int q = 0; q < 3; ++q) R.qh[q] = qh3[q];
  if (qe3) for (int q = 0; q < 3; ++q) R.qe[q] = qe3[q];
  if (pbh) for (uint32_t i = 0; i < R.cfg.n_bins; ++i) R.pb_hit[i] = pbh[i];
  if (pba) for (uint32_t i = 0; i < R.cfg.n_bins; ++i) R.pb_acc[i] = pba[i];
}
void orc_push_interval(void* h, int s, double ln_dt) {
  Replica& R = *(Replica*)h;
  R.iv[s].push_back(ln_dt);
  while (R.iv[s].size() > R.cfg.interval_ring) R.iv[s].pop_front();
}

// Characterisation pass (reading A42): an unbounded cache (C = infinity,
// nothing evicted) over a trace in arrival order.  A block is REUSED if its chained hash
// occurred in an earlier request (P:158 strict prefix); the reuse is INTRA-session if an
// earlier occurrence was in the same session, else INTER-session (Fig. 2a/d).
// Table 1 columns by token type: intra-conv. = reused-intra share of the blocks of
// later turns (turn > 0, which can reuse their own history); inter-conv. = reused share of
// the blocks of first turns (turn 0: only other sessions precede them); combined = reused
// share of all blocks.  Positional reuse (Fig. 2c): prompt blocks of single-turn
// sessions by bin min(9, 10 j / np).
typedef struct {
  uint64_t blocks[6], reused[6];
  uint64_t later_blocks[6], later_intra[6];
  uint64_t first_blocks[6], first_inter[6];
  uint64_t pos_blocks[10], pos_reused[10];
  uint64_t reuses_intra, reuses_inter;
} orc_char_stats;

int orc_characterize(const orc_config* cfg, uint64_t n, const uint64_t* poff, const uint32_t* plen,
                     const uint64_t* doff, const uint32_t* dlen, const uint32_t* tokens,
                     const uint8_t* types, const uint32_t* session, const uint32_t* turn,
                     const uint8_t* single_turn, orc_char_stats* out) {
  std::memset(out, 0, sizeof *out);
  std::unordered_set<uint64_t> seen;
  std::set<std::pair<uint64_t, uint32_t>> seen_sess;
  const uint32_t B = cfg->block_tokens;
  for (uint64_t i = 0; i < n; ++i) {
    if (plen[i] < 1) return ORC_E_INVAL;
    std::vector<uint64_t> H;
    std::vector<uint8_t> tau, ntok;
    hash_request(*cfg, tokens + poff[i], types + poff[i], plen[i], tokens + doff[i], dlen[i], H, tau, ntok);
    const uint32_t np = (plen[i] + B - 1) / B;
    for (uint32_t j = 0; j < H.size(); ++j) {
      const int t = tau[j];
      const bool reused = seen.count(H[j]) > 0;
      const bool intra = seen_sess.count({H[j], session[i]}) > 0;
      out->blocks[t]++;
      if (reused) out->reused[t]++;
      if (turn[i] > 0) {
        out->later_blocks[t]++;
        if (intra) out->later_intra[t]++;
      } else {
        out->first_blocks[t]++;
        if (reused) out->first_inter[t]++;
      }
      if (reused) {
        if (intra) out->reuses_intra++;
        else out->reuses_inter++;
      }
      if (single_turn[i] && j < np) {
        const uint32_t bin = std::min<uint32_t>(9, (10 * j) / np);
        out->pos_blocks[bin]++;
        if (reused) out->pos_reused[bin]++;
      }
    }
    for (uint64_t h : H) {
      seen.insert(h);
      seen_sess.insert({h, session[i]});
    }
  }
  return ORC_OK;
}

// Whole-trace replay of one replica's requests (array order), for parity and
// the cpu_baseline.  Request i's prompt tokens are tokens[poff[i] .. +plen[i]],
// decode tokens tokens[doff[i] .. +dlen[i]].  out4 is [n][4].
int orc_replay(void* h, uint64_t n, const double* arrival, const uint64_t* poff,
               const uint32_t* plen, const uint64_t* doff, const uint32_t* dlen,
               const uint32_t* tokens, const uint8_t* types, const uint8_t* flags,
               const uint32_t* spb, uint32_t* out4, uint32_t* vout, uint64_t vcap,
               uint64_t* voff /* [n+1] */, uint64_t* hash_out, uint8_t* tau_out,
               uint64_t* boff /* [n+1] block offsets, optional */) {
  uint64_t vn = 0, bo = 0;
  uint32_t B = ((Replica*)h)->cfg.block_tokens;
  for (uint64_t i = 0; i < n; ++i) {
    if (voff) voff[i] = vn;
    if (boff) boff[i] = bo;
    uint32_t nb = (plen[i] + B - 1) / B + (dlen[i] + B - 1) / B;
    int rc = orc_admit(h, arrival[i], tokens + poff[i], types + poff[i], plen[i],
                       tokens + doff[i], dlen[i], flags[i], spb[i], out4 + 4 * i, vout, vcap,
                       &vn, hash_out ? hash_out + bo : nullptr, tau_out ? tau_out + bo : nullptr);
    if (rc != ORC_OK) return rc;
    bo += nb;
  }
  if (voff) voff[n] = vn;
  if (boff) boff[n] = bo;
  return ORC_OK;
}

}  // extern "C"
