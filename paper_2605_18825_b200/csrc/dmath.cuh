// dmath.cuh — fp64 transcendentals for the SAECache score on sm_100a.
//
// ln / exp / erfc implement the fdlibm 5.3 algorithms (e_log.c, e_exp.c,
// s_erf.c:erfc) so the GPU and the independently written CPU oracle round
// identically (CUDA libdevice and glibc differ in the last
// bits, and a one-ulp difference can flip a near-tie victim).  Every +,-,*,/ is
// an explicit round-to-nearest intrinsic, so no FMA contraction can happen
// whatever the compile flags.  Coefficients are written as IEEE bit patterns.
#pragma once
#include <cstdint>

namespace sae {
namespace dm {

__device__ __forceinline__ double A(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double S(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double M(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double D(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double H(uint64_t bits) { return __longlong_as_double((long long)bits); }
__device__ __forceinline__ int hiw(double x) { return __double2hiint(x); }
__device__ __forceinline__ unsigned low(double x) { return (unsigned)__double2loint(x); }
__device__ __forceinline__ double mk(int hi, unsigned lo) { return __hiloint2double(hi, (int)lo); }

// ---- natural log (e_log.c) --------------------------------------------------
__device__ __noinline__ double ln(double x) {
  const double ln2_hi = H(0x3fe62e42fee00000ull), ln2_lo = H(0x3dea39ef35793c76ull);
  const double two54 = H(0x4350000000000000ull);
  const double Lg1 = H(0x3FE5555555555593ull), Lg2 = H(0x3FD999999997FA04ull),
               Lg3 = H(0x3FD2492494229359ull), Lg4 = H(0x3FCC71C51D8E78AFull),
               Lg5 = H(0x3FC7466496CB03DEull), Lg6 = H(0x3FC39A09D078C69Full),
               Lg7 = H(0x3FC2F112DF3E5244ull);
  int hx = hiw(x);
  unsigned lx = low(x);
  int k = 0;
  if (hx < 0x00100000) {
    if (((hx & 0x7fffffff) | lx) == 0) return D(-two54, 0.0);
    if (hx < 0) return D(S(x, x), 0.0);
    k -= 54;
    x = M(x, two54);
    hx = hiw(x);
  }
  if (hx >= 0x7ff00000) return A(x, x);
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int i = (hx + 0x95f64) & 0x100000;
  x = mk(hx | (i ^ 0x3ff00000), low(x));
  k += (i >> 20);
  double f = S(x, 1.0);
  double dk;
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      dk = (double)k;
      return A(M(dk, ln2_hi), M(dk, ln2_lo));
    }
    double R = M(M(f, f), S(0.5, M(0.33333333333333333, f)));
    if (k == 0) return S(f, R);
    dk = (double)k;
    return S(M(dk, ln2_hi), S(S(R, M(dk, ln2_lo)), f));
  }
  double s = D(f, A(2.0, f));
  dk = (double)k;
  double z = M(s, s);
  i = hx - 0x6147a;
  double w = M(z, z);
  int j = 0x6b851 - hx;
  double t1 = M(w, A(Lg2, M(w, A(Lg4, M(w, Lg6)))));
  double t2 = M(z, A(Lg1, M(w, A(Lg3, M(w, A(Lg5, M(w, Lg7)))))));
  i |= j;
  double R = A(t2, t1);
  if (i > 0) {
    double hfsq = M(M(0.5, f), f);
    if (k == 0) return S(f, S(hfsq, M(s, A(hfsq, R))));
    return S(M(dk, ln2_hi), S(S(hfsq, A(M(s, A(hfsq, R)), M(dk, ln2_lo))), f));
  }
  if (k == 0) return S(f, M(s, S(f, R)));
  return S(M(dk, ln2_hi), S(S(M(s, S(f, R)), M(dk, ln2_lo)), f));
}

// ---- exp (e_exp.c) ----------------------------------------------------------
__device__ __noinline__ double ex(double x) {
  const double o_thr = H(0x40862E42FEFA39EFull), u_thr = H(0xc0874910D52D3051ull);
  const double ln2HI = H(0x3fe62e42fee00000ull), ln2LO = H(0x3dea39ef35793c76ull);
  const double invln2 = H(0x3ff71547652b82feull);
  const double twom1000 = H(0x0170000000000000ull);
  const double P1 = H(0x3FC555555555553Eull), P2 = H(0xBF66C16C16BEBD93ull),
               P3 = H(0x3F11566AAF25DE2Cull), P4 = H(0xBEBBBD41C5D26BF1ull),
               P5 = H(0x3E66376972BEA4D0ull);
  unsigned hx = (unsigned)hiw(x);
  int xsb = (int)((hx >> 31) & 1);
  hx &= 0x7fffffff;
  if (hx >= 0x40862E42u) {
    if (hx >= 0x7ff00000u) {
      if (((hx & 0xfffff) | low(x)) != 0) return A(x, x);
      return xsb == 0 ? x : 0.0;
    }
    if (x > o_thr) return M(1.0e+300, 1.0e+300);
    if (x < u_thr) return M(twom1000, twom1000);
  }
  double hi = 0.0, lo = 0.0;
  int k = 0;
  if (hx > 0x3fd62e42u) {
    if (hx < 0x3FF0A2B2u) {
      hi = xsb ? A(x, ln2HI) : S(x, ln2HI);
      lo = xsb ? -ln2LO : ln2LO;
      k = 1 - xsb - xsb;
    } else {
      k = __double2int_rz(A(M(invln2, x), xsb ? -0.5 : 0.5));
      double t = (double)k;
      hi = S(x, M(t, ln2HI));
      lo = M(t, ln2LO);
    }
    x = S(hi, lo);
  } else if (hx < 0x3e300000u) {
    if (A(1.0e+300, x) > 1.0) return A(1.0, x);
  }
  double t = M(x, x);
  double c = S(x, M(t, A(P1, M(t, A(P2, M(t, A(P3, M(t, A(P4, M(t, P5))))))))));
  if (k == 0) return S(1.0, S(D(M(x, c), S(c, 2.0)), x));
  double y = S(1.0, S(S(lo, D(M(x, c), S(2.0, c))), hi));
  if (k >= -1021) return mk((int)((unsigned)hiw(y) + ((unsigned)k << 20)), low(y));
  y = mk((int)((unsigned)hiw(y) + ((unsigned)(k + 1000) << 20)), low(y));
  return M(y, twom1000);
}

// ---- erfc (s_erf.c) -----------------------------------------------------------
__device__ __noinline__ double erfc(double x) {
  const double erx = H(0x3FEB0AC160000000ull);
  const double pp0 = H(0x3FC06EBA8214DB68ull), pp1 = H(0xBFD4CD7D691CB913ull),
               pp2 = H(0xBF9D2A51DBD7194Full), pp3 = H(0xBF77A291236668E4ull),
               pp4 = H(0xBEF8EAD6120016ACull);
  const double qq1 = H(0x3FD97779CDDADC09ull), qq2 = H(0x3FB0A54C5536CEBAull),
               qq3 = H(0x3F74D022C4D36B0Full), qq4 = H(0x3F215DC9221C1A10ull),
               qq5 = H(0xBED09C4342A26120ull);
  const double pa0 = H(0xBF6359B8BEF77538ull), pa1 = H(0x3FDA8D00AD92B34Dull),
               pa2 = H(0xBFD7D240FBB8C3F1ull), pa3 = H(0x3FD45FCA805120E4ull),
               pa4 = H(0xBFBC63983D3E28ECull), pa5 = H(0x3FA22A36599795EBull),
               pa6 = H(0xBF61BF380A96073Full);
  const double qa1 = H(0x3FBB3E6618EEE323ull), qa2 = H(0x3FE14AF092EB6F33ull),
               qa3 = H(0x3FB2635CD99FE9A7ull), qa4 = H(0x3FC02660E763351Full),
               qa5 = H(0x3F8BEDC26B51DD1Cull), qa6 = H(0x3F888B545735151Dull);
  const double ra0 = H(0xBF843412600D6435ull), ra1 = H(0xBFE63416E4BA7360ull),
               ra2 = H(0xC0251E0441B0E726ull), ra3 = H(0xC04F300AE4CBA38Dull),
               ra4 = H(0xC0644CB184282266ull), ra5 = H(0xC067135CEBCCABB2ull),
               ra6 = H(0xC054526557E4D2F2ull), ra7 = H(0xC023A0EFC69AC25Cull);
  const double sa1 = H(0x4033A6B9BD707687ull), sa2 = H(0x4061350C526AE721ull),
               sa3 = H(0x407B290DD58A1A71ull), sa4 = H(0x40842B1921EC2868ull),
               sa5 = H(0x407AD02157700314ull), sa6 = H(0x405B28A3EE48AE2Cull),
               sa7 = H(0x401A47EF8E484A93ull), sa8 = H(0xBFAEEFF2EE749A62ull);
  const double rb0 = H(0xBF84341239E86F4Aull), rb1 = H(0xBFE993BA70C285DEull),
               rb2 = H(0xC031C209555F995Aull), rb3 = H(0xC064145D43C5ED98ull),
               rb4 = H(0xC083EC881375F228ull), rb5 = H(0xC09004616A2E5992ull),
               rb6 = H(0xC07E384E9BDC383Full);
  const double sb1 = H(0x403E568B261D5190ull), sb2 = H(0x40745CAE221B9F0Aull),
               sb3 = H(0x409802EB189D5118ull), sb4 = H(0x40A8FFB7688C246Aull),
               sb5 = H(0x40A3F219CEDF3BE6ull), sb6 = H(0x407DA874E79FE763ull),
               sb7 = H(0xC03670E242712D62ull);
  const double tiny = 1e-300;
  int hx = hiw(x);
  int ix = hx & 0x7fffffff;
  if (ix >= 0x7ff00000) return A((double)(((unsigned)hx >> 31) << 1), D(1.0, x));
  if (ix < 0x3feb0000) {
    if (ix < 0x3c700000) return S(1.0, x);
    double z = M(x, x);
    double r = A(pp0, M(z, A(pp1, M(z, A(pp2, M(z, A(pp3, M(z, pp4))))))));
    double s = A(1.0, M(z, A(qq1, M(z, A(qq2, M(z, A(qq3, M(z, A(qq4, M(z, qq5))))))))));
    double y = D(r, s);
    if (hx < 0x3fd00000) return S(1.0, A(x, M(x, y)));
    r = M(x, y);
    r = A(r, S(x, 0.5));
    return S(0.5, r);
  }
  if (ix < 0x3ff40000) {
    double s = S(fabs(x), 1.0);
    double P = A(pa0, M(s, A(pa1, M(s, A(pa2, M(s, A(pa3, M(s, A(pa4, M(s, A(pa5, M(s, pa6))))))))))));
    double Q = A(1.0, M(s, A(qa1, M(s, A(qa2, M(s, A(qa3, M(s, A(qa4, M(s, A(qa5, M(s, qa6))))))))))));
    if (hx >= 0) return S(S(1.0, erx), D(P, Q));
    return A(1.0, A(erx, D(P, Q)));
  }
  if (ix < 0x403c0000) {
    x = fabs(x);
    double s = D(1.0, M(x, x));
    double R, Sv;
    if (ix < 0x4006DB6D) {
      R = A(ra0, M(s, A(ra1, M(s, A(ra2, M(s, A(ra3, M(s, A(ra4, M(s, A(ra5, M(s, A(ra6, M(s, ra7))))))))))))));
      Sv = A(1.0, M(s, A(sa1, M(s, A(sa2, M(s, A(sa3, M(s, A(sa4, M(s, A(sa5, M(s, A(sa6, M(s, A(sa7, M(s, sa8))))))))))))))));
    } else {
      if (hx < 0 && ix >= 0x40180000) return S(2.0, tiny);
      R = A(rb0, M(s, A(rb1, M(s, A(rb2, M(s, A(rb3, M(s, A(rb4, M(s, A(rb5, M(s, rb6))))))))))));
      Sv = A(1.0, M(s, A(sb1, M(s, A(sb2, M(s, A(sb3, M(s, A(sb4, M(s, A(sb5, M(s, A(sb6, M(s, sb7))))))))))))));
    }
    double z = mk(hiw(x), 0u);
    double r = M(ex(S(M(-z, z), 0.5625)), ex(A(M(S(z, x), A(z, x)), D(R, Sv))));
    if (hx > 0) return D(r, x);
    return S(2.0, D(r, x));
  }
  if (hx > 0) return M(tiny, tiny);
  return S(2.0, tiny);
}

}  // namespace dm
}  // namespace sae
