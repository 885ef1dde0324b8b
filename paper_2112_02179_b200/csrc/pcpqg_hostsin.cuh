// The double-precision sin the reference's anisotropic weights are built on
// (std::sin in sin_power_integral, proj/core/src/numerics.cpp:174-186), restated
// operation for operation for arguments in [0, 2.426): the C library here is
// glibc 2.39, whose x86-64 ifunc selects the FMA build of the IBM Accurate
// Mathematical Library sin on every host with FMA + AVX2.  Its branches for this
// range, in the order the binary evaluates them (read from its disassembly;
// each fused multiply-add below is one in the binary):
//   |x| < 2^-26          x
//   |x| < 0.126          x + x^2 (x P(x^2))                       (odd polynomial)
//   |x| < 0.85546875     sin(x_k + r) from the table at x_k = k/128 (Ziv)
//   |x| < 2.426265       cos(pi/2 - |x|) from the same table, pi/2 as hp0 + hp1
// The table (pcpqg_sincostab.inc) is read from the C library's binary by
// tools/gen_sincostab.py.  The library checks this function against the host's
// std::sin before it trusts it (sin_port_mismatches); on any mismatch the
// weights stay on the host path.
#pragma once
#include <cstdint>
#include <cstring>

#if defined(__CUDA_ARCH__)
#define PCPQG_SIN_MUL(a, b) __dmul_rn((a), (b))
#define PCPQG_SIN_ADD(a, b) __dadd_rn((a), (b))
#define PCPQG_SIN_SUB(a, b) __dsub_rn((a), (b))
#define PCPQG_SIN_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <cmath>
#define PCPQG_SIN_MUL(a, b) ((a) * (b))
#define PCPQG_SIN_ADD(a, b) ((a) + (b))
#define PCPQG_SIN_SUB(a, b) ((a) - (b))
#define PCPQG_SIN_FMA(a, b, c) std::fma((a), (b), (c))
#endif

namespace pcpqg {

constexpr int kSinTabEntries = 110;

// x in [0, 2.426265); tab = the {sin hi, sin lo, cos hi, cos lo} table
__host__ __device__ inline double sin_port(double x, const double* __restrict__ tab) {
  constexpr double big = 0x1.8p45;
  constexpr double sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7;
  constexpr double cs2 = 0.5, cs4 = -0x1.5555555555535p-5, cs6 = 0x1.6c16bedd9e239p-10;
  constexpr double hp0 = 0x1.921fb54442d18p+0, hp1 = 0x1.1a62633145c07p-54;
  constexpr double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7, s3 = -0x1.a01a019db08b8p-13,
                   s4 = 0x1.71de27b9a7ed9p-19, s5 = -0x1.addffc2fcdf59p-26;
  uint64_t bits;
#if defined(__CUDA_ARCH__)
  bits = static_cast<uint64_t>(__double_as_longlong(x));
#else
  std::memcpy(&bits, &x, 8);
#endif
  const uint32_t hx = static_cast<uint32_t>(bits >> 32) & 0x7fffffffu;
  if (hx <= 0x3e4fffffu) return x;
  if (hx <= 0x3feb5fffu) {
    if (x < 0x1.020c49ba5e354p-3) {
      const double xx = PCPQG_SIN_MUL(x, x);
      double t = PCPQG_SIN_FMA(s5, xx, s4);
      t = PCPQG_SIN_FMA(t, xx, s3);
      t = PCPQG_SIN_FMA(t, xx, s2);
      t = PCPQG_SIN_FMA(t, xx, s1);
      t = PCPQG_SIN_FMA(x, t, -0.0);
      const double r = PCPQG_SIN_FMA(xx, t, 0.0);
      return PCPQG_SIN_ADD(x, r);
    }
    const double dx = 0.0;
    const double u = PCPQG_SIN_ADD(x, big);
    const double xr = PCPQG_SIN_SUB(x, PCPQG_SIN_SUB(u, big));
#if defined(__CUDA_ARCH__)
    const uint32_t k = static_cast<uint32_t>(__double2loint(u)) << 2;
#else
    uint64_t ub;
    std::memcpy(&ub, &u, 8);
    const uint32_t k = static_cast<uint32_t>(ub) << 2;
#endif
    const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
    const double xx = PCPQG_SIN_MUL(xr, xr);
    const double p = PCPQG_SIN_FMA(xx, sn5, sn3);
    const double x3 = PCPQG_SIN_MUL(xr, xx);
    const double s = PCPQG_SIN_FMA(x3, p, dx);
    double cp = PCPQG_SIN_FMA(xx, cs6, cs4);
    cp = PCPQG_SIN_FMA(xx, cp, cs2);
    const double sf = PCPQG_SIN_ADD(xr, s);
    const double c0 = PCPQG_SIN_MUL(xx, cp);
    const double c = PCPQG_SIN_FMA(xr, dx, c0);
    double cor = PCPQG_SIN_FMA(sf, ccs, ssn);
    cor = PCPQG_SIN_FMA(-c, sn, cor);
    cor = PCPQG_SIN_FMA(sf, cs, cor);
    return PCPQG_SIN_ADD(sn, cor);
  }
  // 0.85546875 <= x < 2.426265: cos(hp0 + hp1 - x)
  const double t = PCPQG_SIN_SUB(hp0, x);
  const double dx = t < 0.0 ? -hp1 : hp1;
  const double at = t < 0.0 ? -t : t;
  const double u = PCPQG_SIN_ADD(at, big);
  double xr = PCPQG_SIN_SUB(at, PCPQG_SIN_SUB(u, big));
#if defined(__CUDA_ARCH__)
  const uint32_t k = static_cast<uint32_t>(__double2loint(u)) << 2;
#else
  uint64_t ub;
  std::memcpy(&ub, &u, 8);
  const uint32_t k = static_cast<uint32_t>(ub) << 2;
#endif
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  xr = PCPQG_SIN_ADD(xr, dx);
  const double xx = PCPQG_SIN_MUL(xr, xr);
  const double p = PCPQG_SIN_FMA(xx, sn5, sn3);
  const double x3 = PCPQG_SIN_MUL(xr, xx);
  const double s = PCPQG_SIN_FMA(x3, p, xr);
  double cp = PCPQG_SIN_FMA(xx, cs6, cs4);
  cp = PCPQG_SIN_FMA(xx, cp, cs2);
  const double c = PCPQG_SIN_MUL(xx, cp);
  double cor = PCPQG_SIN_FMA(-s, ssn, ccs);
  cor = PCPQG_SIN_FMA(-c, cs, cor);
  cor = PCPQG_SIN_FMA(-s, sn, cor);
  return PCPQG_SIN_ADD(cs, cor);
}

}  // namespace pcpqg
