// cr_atan2.cuh — correctly rounded double atan2 for host and device.
//
// The reference's hinge angle is std::atan2(s, c) (proj/src/elements.cpp:116),
// i.e. glibc's atan2. glibc 2.39's atan2 is accurate to about half an ulp
// but not correctly rounded (its slow exact paths were removed in 2.35): on
// uniform draws about 1 in 10^3 results is the other neighbour of a
// near-midpoint value, and its exact algorithm (plus the FMA/no-FMA ifunc
// variant the host CPU selects) cannot be reproduced from here. CUDA's atan2
// is a 2-ulp approximation. This evaluates atan2 in double-double (~2^-100
// relative) and rounds once: the correctly rounded value, which is what
// glibc returns everywhere except those near-midpoint cases
// (tools/atan2_agreement.py measures the three against each other on the
// hinge inputs of real scenes; tests/test_hinge_atan2.py pins correct
// rounding against mpmath).
//
// Reduction: t = min(|y|,|x|) / max(|y|,|x|) in [0,1] as a double-double
// quotient; c = k/64 nearest t; atan(t) = atan(c) + atan((t-c)/(1+t*c)) with
// |u| <= 2^-7 and an odd Taylor polynomial through u^17; then the octant
// fix-ups pi/2 - r, pi - r and the sign of y, all in double-double.
// Zero, infinite and NaN arguments take the library atan2, whose results there
// are exact IEEE special values on both sides. The table holds atan(k/64),
// k = 0..64, as (hi, lo) pairs (tools/gen_atan_table.py, mpmath at 200 bits).
//
// Needs exact products: explicit fma() (the library is built with
// -fmad=false, which leaves explicit fma alone).
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define WEFT_HD __host__ __device__ __forceinline__
#else
#define WEFT_HD inline
#endif

namespace weft_gpu {
namespace cr {

struct DD {
  double hi, lo;
};

#ifdef __CUDA_ARCH__
#define WEFT_ATAN_TAB kAtanTabDev
#else
#define WEFT_ATAN_TAB kAtanTabHost
#endif

#ifdef __CUDACC__
static __device__ __constant__ double kAtanTabDev[130] = {  // internal linkage: one copy per TU, also under -rdc
    0x0.0p+0, 0x0.0p+0,
    0x1.fff555bbb729bp-7, -0x1.220c39d4dff50p-61,
    0x1.ffd55bba97625p-6, -0x1.5ec431444912cp-60,
    0x1.7fb818430da2ap-5, -0x1.86ef8f794f105p-63,
    0x1.ff55bb72cfdeap-5, -0x1.c934d86d23f1dp-60,
    0x1.3f59f0e7c559dp-4, 0x1.ac4ce285df847p-58,
    0x1.7ee182602f10fp-4, -0x1.cfb654c0c3d98p-58,
    0x1.be39ebe6f07c3p-4, 0x1.f7b8f29a05987p-58,
    0x1.fd5ba9aac2f6ep-4, -0x1.cd37686760c17p-59,
    0x1.1e1fafb043727p-3, -0x1.b485914dacf8cp-59,
    0x1.3d6eee8c6626cp-3, 0x1.61a3b0ce9281bp-57,
    0x1.5c9811e3ec26ap-3, -0x1.054ab2c010f3dp-58,
    0x1.7b97b4bce5b02p-3, 0x1.347b0b4f881cap-58,
    0x1.9a6a8e96c8626p-3, 0x1.cf601e7b4348ep-59,
    0x1.b90d7529260a2p-3, 0x1.17b10d2e0e5abp-61,
    0x1.d77d5df205736p-3, 0x1.c648d1534597ep-57,
    0x1.f5b75f92c80ddp-3, 0x1.8ab6e3cf7afbdp-57,
    0x1.09dc597d86362p-2, 0x1.62e47390cb865p-56,
    0x1.18bf5a30bf178p-2, 0x1.30ca4748b1bf9p-57,
    0x1.278372057ef46p-2, -0x1.077cdd36dfc81p-56,
    0x1.362773707ebccp-2, -0x1.963a544b672d8p-57,
    0x1.44aa436c2af0ap-2, -0x1.5d5e43c55b3bap-56,
    0x1.530ad9951cd4ap-2, -0x1.2566480884082p-57,
    0x1.614840309cfe2p-2, -0x1.a725715711f00p-56,
    0x1.6f61941e4def1p-2, -0x1.c63aae6f6e918p-56,
    0x1.7d5604b63b3f7p-2, 0x1.69c885c2b249ap-56,
    0x1.8b24d394a1b25p-2, 0x1.b6d0ba3748fa8p-56,
    0x1.98cd5454d6b18p-2, 0x1.9e6c988fd0a77p-56,
    0x1.a64eec3cc23fdp-2, -0x1.24dec1b50b7ffp-56,
    0x1.b3a911da65c6cp-2, 0x1.ae187b1ca5040p-56,
    0x1.c0db4c94ec9f0p-2, -0x1.cc1ce70934c34p-56,
    0x1.cde53432c1351p-2, -0x1.a2cfa4418f1adp-56,
    0x1.dac670561bb4fp-2, 0x1.a2b7f222f65e2p-56,
    0x1.e77eb7f175a34p-2, 0x1.0e53dc1bf3435p-56,
    0x1.f40dd0b541418p-2, -0x1.a3992dc382a23p-57,
    0x1.0039c73c1a40cp-1, -0x1.b32c949c9d593p-55,
    0x1.0657e94db30d0p-1, -0x1.d5b495f6349e6p-56,
    0x1.0c6145b5b43dap-1, 0x1.974fa13b5404fp-58,
    0x1.1255d9bfbd2a9p-1, -0x1.2bdaee1c0ee35p-58,
    0x1.1835a88be7c13p-1, 0x1.c621cec00c301p-55,
    0x1.1e00babdefeb4p-1, -0x1.928df287a668fp-58,
    0x1.23b71e2cc9e6ap-1, 0x1.c421c9f38224ep-57,
    0x1.2958e59308e31p-1, -0x1.09e73b0c6c087p-56,
    0x1.2ee628406cbcap-1, 0x1.c5d5e9ff0cf8dp-55,
    0x1.345f01cce37bbp-1, 0x1.1021137c71102p-55,
    0x1.39c391cd4171ap-1, -0x1.2304331d8bf46p-55,
    0x1.3f13fb89e96f4p-1, 0x1.ecf8b492644f0p-56,
    0x1.445065b795b56p-1, -0x1.f76d0163f79c8p-56,
    0x1.4978fa3269ee1p-1, 0x1.2419a87f2a458p-56,
    0x1.4e8de5bb6ec04p-1, 0x1.4a33dbeb3796cp-55,
    0x1.538f57b89061fp-1, -0x1.1bb74abda520cp-55,
    0x1.587d81f732fbbp-1, -0x1.5e5c9d8c5a950p-56,
    0x1.5d58987169b18p-1, 0x1.0028e4bc5e7cap-57,
    0x1.6220d115d7b8ep-1, -0x1.2b785350ee8c1p-57,
    0x1.66d663923e087p-1, -0x1.6ea6febe8bbbap-56,
    0x1.6b798920b3d99p-1, -0x1.a80386188c50ep-55,
    0x1.700a7c5784634p-1, -0x1.8c34d25aadef6p-56,
    0x1.748978fba8e0fp-1, 0x1.7b2a6165884a1p-59,
    0x1.78f6bbd5d315ep-1, 0x1.406a089803740p-55,
    0x1.7d528289fa093p-1, 0x1.560821e2f3aa9p-55,
    0x1.819d0b7158a4dp-1, -0x1.bf76229d3b917p-56,
    0x1.85d69576cc2c5p-1, 0x1.6b66e7fc8b8c3p-57,
    0x1.89ff5ff57f1f8p-1, -0x1.55b9a5e177a1bp-55,
    0x1.8e17aa99cc05ep-1, -0x1.ec182ab042f61p-56,
    0x1.921fb54442d18p-1, 0x1.1a62633145c07p-55,
};
#endif
static const double kAtanTabHost[130] = {
    0x0.0p+0, 0x0.0p+0,
    0x1.fff555bbb729bp-7, -0x1.220c39d4dff50p-61,
    0x1.ffd55bba97625p-6, -0x1.5ec431444912cp-60,
    0x1.7fb818430da2ap-5, -0x1.86ef8f794f105p-63,
    0x1.ff55bb72cfdeap-5, -0x1.c934d86d23f1dp-60,
    0x1.3f59f0e7c559dp-4, 0x1.ac4ce285df847p-58,
    0x1.7ee182602f10fp-4, -0x1.cfb654c0c3d98p-58,
    0x1.be39ebe6f07c3p-4, 0x1.f7b8f29a05987p-58,
    0x1.fd5ba9aac2f6ep-4, -0x1.cd37686760c17p-59,
    0x1.1e1fafb043727p-3, -0x1.b485914dacf8cp-59,
    0x1.3d6eee8c6626cp-3, 0x1.61a3b0ce9281bp-57,
    0x1.5c9811e3ec26ap-3, -0x1.054ab2c010f3dp-58,
    0x1.7b97b4bce5b02p-3, 0x1.347b0b4f881cap-58,
    0x1.9a6a8e96c8626p-3, 0x1.cf601e7b4348ep-59,
    0x1.b90d7529260a2p-3, 0x1.17b10d2e0e5abp-61,
    0x1.d77d5df205736p-3, 0x1.c648d1534597ep-57,
    0x1.f5b75f92c80ddp-3, 0x1.8ab6e3cf7afbdp-57,
    0x1.09dc597d86362p-2, 0x1.62e47390cb865p-56,
    0x1.18bf5a30bf178p-2, 0x1.30ca4748b1bf9p-57,
    0x1.278372057ef46p-2, -0x1.077cdd36dfc81p-56,
    0x1.362773707ebccp-2, -0x1.963a544b672d8p-57,
    0x1.44aa436c2af0ap-2, -0x1.5d5e43c55b3bap-56,
    0x1.530ad9951cd4ap-2, -0x1.2566480884082p-57,
    0x1.614840309cfe2p-2, -0x1.a725715711f00p-56,
    0x1.6f61941e4def1p-2, -0x1.c63aae6f6e918p-56,
    0x1.7d5604b63b3f7p-2, 0x1.69c885c2b249ap-56,
    0x1.8b24d394a1b25p-2, 0x1.b6d0ba3748fa8p-56,
    0x1.98cd5454d6b18p-2, 0x1.9e6c988fd0a77p-56,
    0x1.a64eec3cc23fdp-2, -0x1.24dec1b50b7ffp-56,
    0x1.b3a911da65c6cp-2, 0x1.ae187b1ca5040p-56,
    0x1.c0db4c94ec9f0p-2, -0x1.cc1ce70934c34p-56,
    0x1.cde53432c1351p-2, -0x1.a2cfa4418f1adp-56,
    0x1.dac670561bb4fp-2, 0x1.a2b7f222f65e2p-56,
    0x1.e77eb7f175a34p-2, 0x1.0e53dc1bf3435p-56,
    0x1.f40dd0b541418p-2, -0x1.a3992dc382a23p-57,
    0x1.0039c73c1a40cp-1, -0x1.b32c949c9d593p-55,
    0x1.0657e94db30d0p-1, -0x1.d5b495f6349e6p-56,
    0x1.0c6145b5b43dap-1, 0x1.974fa13b5404fp-58,
    0x1.1255d9bfbd2a9p-1, -0x1.2bdaee1c0ee35p-58,
    0x1.1835a88be7c13p-1, 0x1.c621cec00c301p-55,
    0x1.1e00babdefeb4p-1, -0x1.928df287a668fp-58,
    0x1.23b71e2cc9e6ap-1, 0x1.c421c9f38224ep-57,
    0x1.2958e59308e31p-1, -0x1.09e73b0c6c087p-56,
    0x1.2ee628406cbcap-1, 0x1.c5d5e9ff0cf8dp-55,
    0x1.345f01cce37bbp-1, 0x1.1021137c71102p-55,
    0x1.39c391cd4171ap-1, -0x1.2304331d8bf46p-55,
    0x1.3f13fb89e96f4p-1, 0x1.ecf8b492644f0p-56,
    0x1.445065b795b56p-1, -0x1.f76d0163f79c8p-56,
    0x1.4978fa3269ee1p-1, 0x1.2419a87f2a458p-56,
    0x1.4e8de5bb6ec04p-1, 0x1.4a33dbeb3796cp-55,
    0x1.538f57b89061fp-1, -0x1.1bb74abda520cp-55,
    0x1.587d81f732fbbp-1, -0x1.5e5c9d8c5a950p-56,
    0x1.5d58987169b18p-1, 0x1.0028e4bc5e7cap-57,
    0x1.6220d115d7b8ep-1, -0x1.2b785350ee8c1p-57,
    0x1.66d663923e087p-1, -0x1.6ea6febe8bbbap-56,
    0x1.6b798920b3d99p-1, -0x1.a80386188c50ep-55,
    0x1.700a7c5784634p-1, -0x1.8c34d25aadef6p-56,
    0x1.748978fba8e0fp-1, 0x1.7b2a6165884a1p-59,
    0x1.78f6bbd5d315ep-1, 0x1.406a089803740p-55,
    0x1.7d528289fa093p-1, 0x1.560821e2f3aa9p-55,
    0x1.819d0b7158a4dp-1, -0x1.bf76229d3b917p-56,
    0x1.85d69576cc2c5p-1, 0x1.6b66e7fc8b8c3p-57,
    0x1.89ff5ff57f1f8p-1, -0x1.55b9a5e177a1bp-55,
    0x1.8e17aa99cc05ep-1, -0x1.ec182ab042f61p-56,
    0x1.921fb54442d18p-1, 0x1.1a62633145c07p-55,
};

WEFT_HD DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return DD{s, (a - (s - bb)) + (b - bb)};
}
WEFT_HD DD fast_two_sum(double a, double b) {
  const double s = a + b;
  return DD{s, b - (s - a)};
}
WEFT_HD DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  DD t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
WEFT_HD DD dd_neg(DD a) { return DD{-a.hi, -a.lo}; }
WEFT_HD DD dd_mul(DD a, DD b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p, e);
}
WEFT_HD DD dd_mul_d(DD a, double b) {
  const double p = a.hi * b;
  double e = fma(a.hi, b, -p);
  e += a.lo * b;
  return fast_two_sum(p, e);
}
WEFT_HD DD dd_div(DD a, DD b) {
  const double q1 = a.hi / b.hi;
  DD r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
  const double q2 = r.hi / b.hi;
  r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
  const double q3 = r.hi / b.hi;
  DD q = fast_two_sum(q1, q2);
  return dd_add(q, DD{q3, 0.0});
}

// atan(u) for |u| <= 2^-7 + tiny, as u + u^3 * P(u^2); P through the u^16 term.
WEFT_HD DD atan_small(DD u) {
  const DD u2 = dd_mul(u, u);
  // Horner over c_n = (-1)^n / (2n+1), n = 8 .. 1, in double-double.
  DD p = DD{1.0 / 17.0, 0.0};
  const double inv[8] = {-1.0 / 15.0, 1.0 / 13.0, -1.0 / 11.0, 1.0 / 9.0,
                         -1.0 / 7.0, 1.0 / 5.0, -1.0 / 3.0, 0.0};
  // Low halves of the reciprocals that are not exact doubles.
  const double inv_lo[8] = {-9.251858538542971e-19,-4.270088556250602e-18,2.523234146875356e-18,6.1679056923619804e-18,-7.93016446160826e-18,-1.1102230246251566e-17,-1.850371707708594e-17, 0.0};
  for (int i = 0; i < 7; ++i) p = dd_add(dd_mul(p, u2), DD{inv[i], inv_lo[i]});
  // p = P(u2) = -1/3 + u2/5 - ...; result u + u * u2 * p
  return dd_add(u, dd_mul(u, dd_mul(u2, p)));
}

WEFT_HD double atan2(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  if (!(ax > 0.0) || !(ay > 0.0) || !(ax < INFINITY) || !(ay < INFINITY)) return ::atan2(y, x);
  const bool swap = ay > ax;
  const double num = swap ? ax : ay;
  const double den = swap ? ay : ax;
  // t = num / den as a double-double.
  const double q = num / den;
  if (q < 0x1p-900) return ::atan2(y, x);  // ratio near underflow: not reached by the hinge angle
  const double r = fma(-q, den, num);
  const DD t = fast_two_sum(q, r / den);
  const int k = static_cast<int>(t.hi * 64.0 + 0.5);
  const double c = k * 0x1p-6;
  // u = (t - c) / (1 + t c)
  const DD numu = dd_add(t, DD{-c, 0.0});
  const DD denu = dd_add(DD{1.0, 0.0}, dd_mul_d(t, c));
  const DD u = dd_div(numu, denu);
  DD a = dd_add(DD{WEFT_ATAN_TAB[2 * k], WEFT_ATAN_TAB[2 * k + 1]}, atan_small(u));
  if (swap) a = dd_add(DD{0x1.921fb54442d18p+0, 0x1.1a62633145c07p-54}, dd_neg(a));
  if (x < 0.0) a = dd_add(DD{0x1.921fb54442d18p+1, 0x1.1a62633145c07p-53}, dd_neg(a));
  const double v = a.hi + a.lo;
  return y < 0.0 ? -v : v;
}

}  // namespace cr
}  // namespace weft_gpu
