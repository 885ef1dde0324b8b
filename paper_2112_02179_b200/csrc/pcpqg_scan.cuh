// K2: the fused scan + top-K kernel template (see pcpqg_kernels.cu for the
// design notes).  Instantiated per code layout in pcpqg_scan_*.cu so the
// variants compile in parallel.
#pragma once
#include "pcpqg_device.cuh"

namespace pcpqg {
namespace {
// ------------------------------------------------------ K2: scan + top-K



// CW == 0: JOINT8 (byte = c | l << cbits), eta table + scale codebook.
// CW == 1: JOINT8 with a pre-multiplied table T[j][byte] = fl(eta[j][c] *
//          lambda[j][l]) — the reference's own eta_lambda values
//          (pq_index.cpp:195-208) indexed by the code byte; used for small
//          query groups where the table fits.  k then counts table rows.
// CW >= 4: PLANES with CW-bit centers and SW-bit scale codes / raw alpha.
template <int CW, int SW>
struct Codec {
  static constexpr bool kJoint = CW <= 1;
  static constexpr int kCenterWords = kJoint ? 2 : CW / 4;  // words per octet
  static constexpr int kScaleWords = kJoint ? 0 : SW / 4;   // words per octet
  static constexpr bool kRaw = SW >= 16;                    // alpha in the stream
  static constexpr bool kNoLambda = kRaw || CW == 1;        // no scale table in smem
};

__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// Two IEEE fp32 products in one FMUL2.  Only the multiply is packed: the
// accumulation stays a scalar __fadd_rn, which ptxas never contracts, so the
// pair keeps its two separate roundings (tests/test_capi.py checks the SASS
// of every scan kernel for FFMA/FFMA2).  A packed sum is not an option:
// ptxas 12.9 contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 in spite of
// the explicit roundings (also with --fmad=false, and it sees through
// fma(p, 1, acc) and fma(a, b, -0)); a product disguised as fma(a, b, c[-0])
// kept the bits but measured 1% at B = 2 / 4 (the scans are not bound by the
// FP32 issue slots), so it was not kept.
__device__ __forceinline__ uint64_t fmul2_rn(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Scores one point for NQ queries: the sections [0, m) in order, 8 per octet.
// Full octets (m / 8 of them) need no bounds checks — all their code words
// exist — and walk the tables with incrementing pointers; only the last,
// partial octet (m % 8 sections) is guarded.
// KT != 0 fixes k (and, for JOINT8, cbits = log2 KT) at compile time so row
// offsets become immediates; KT == 0 reads k / cbits at run time.
template <int NQ, int CW, int SW, int KT, bool kPartial, int NP>
__device__ __forceinline__ void score_octet(const uint32_t* cw_ptr, const uint32_t* sw_ptr,
                                            uint32_t pstride, uint32_t ncw, uint32_t nsw,
                                            uint32_t nsec, const float* eta_o, const float* lam_o,
                                            uint32_t k, uint32_t s, uint32_t cbits,
                                            float (&acc)[NP][NQ]) {
  using Cd = Codec<CW, SW>;
  constexpr int RS = rs_of(NQ);
  uint32_t cwd[NP][Cd::kCenterWords];
  uint32_t swd[NP][Cd::kScaleWords > 0 ? Cd::kScaleWords : 1];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
#pragma unroll
    for (int i = 0; i < Cd::kCenterWords; ++i)
      cwd[p][i] = (!kPartial || static_cast<uint32_t>(i) < ncw) ? cw_ptr[p * pstride + i * kBlockPts]
                                                                  : 0u;
    if constexpr (Cd::kScaleWords > 0) {
#pragma unroll
      for (int i = 0; i < Cd::kScaleWords; ++i)
        swd[p][i] = (!kPartial || static_cast<uint32_t>(i) < nsw)
                        ? sw_ptr[p * pstride + i * kBlockPts]
                        : 0u;
    }
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (kPartial && b >= static_cast<int>(nsec)) break;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      uint32_t c;
      float alpha = 1.0f;
      if constexpr (CW == 1) {
        c = (cwd[p][b >> 2] >> (8 * (b & 3))) & 0xFFu;  // table row = code byte
      } else if constexpr (CW == 0) {
        const uint32_t byte = (cwd[p][b >> 2] >> (8 * (b & 3))) & 0xFFu;
        c = byte & ((1u << cbits) - 1u);
        alpha = lam_o[b * s + (byte >> cbits)];
      } else {
        if constexpr (CW == 4) c = (cwd[p][0] >> (4 * b)) & 0xFu;
        else if constexpr (CW == 8) c = (cwd[p][b >> 2] >> (8 * (b & 3))) & 0xFFu;
        else c = (cwd[p][b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
        if constexpr (SW == 0) {
          alpha = lam_o[b];
        } else if constexpr (SW == 4) {
          alpha = lam_o[b * s + ((swd[p][0] >> (4 * b)) & 0xFu)];
        } else if constexpr (SW == 8) {
          alpha = lam_o[b * s + ((swd[p][b >> 2] >> (8 * (b & 3))) & 0xFFu)];
        } else if constexpr (SW == 16) {
          alpha = __half2float(__ushort_as_half(
              static_cast<unsigned short>((swd[p][b >> 1] >> (16 * (b & 1))) & 0xFFFFu)));
        } else {
          alpha = __uint_as_float(swd[p][b]);
        }
      }
      const float* row = eta_o + (b * k + c) * RS;
      PCPQG_DASSERT(c < k);
      if constexpr (CW == 1) {
        if constexpr (NQ == 1) {
          acc[p][0] = __fadd_rn(acc[p][0], row[0]);
        } else {
#pragma unroll
          for (int q2 = 0; q2 < NQ / 2; ++q2) {
            float tx, ty;
            unpack2(*reinterpret_cast<const uint64_t*>(row + 2 * q2), tx, ty);
            acc[p][2 * q2] = __fadd_rn(acc[p][2 * q2], tx);
            acc[p][2 * q2 + 1] = __fadd_rn(acc[p][2 * q2 + 1], ty);
          }
        }
      } else if constexpr (NQ == 1) {
        acc[p][0] = __fadd_rn(acc[p][0], __fmul_rn(row[0], alpha));
      } else {
        const uint64_t a2 = pack2(alpha, alpha);
#pragma unroll
        for (int q2 = 0; q2 < NQ / 2; ++q2) {
          const uint64_t e2 = *reinterpret_cast<const uint64_t*>(row + 2 * q2);
          float tx, ty;
          unpack2(fmul2_rn(e2, a2), tx, ty);
          acc[p][2 * q2] = __fadd_rn(acc[p][2 * q2], tx);
          acc[p][2 * q2 + 1] = __fadd_rn(acc[p][2 * q2 + 1], ty);
        }
      }
    }
  }
}

// Full octet for 4-bit centers with k == 16 and a query group of <= 2
// (RS in {1, 2}, so a center row is 4 * RS bytes and a section's 16 rows are
// 64 * RS bytes).  The eta block of the octet starts at the shared address
// eta_sa, aligned to 64 * RS, so the row address of section b is one LOP3
// (eta_sa | (c << log2(4 * RS))) plus an immediate; with one query the two
// products of a section pair share one FMUL2.  Same roundings, same order.
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t lds_b64(uint32_t addr) {
  uint64_t v;
  asm("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

template <int SW, int NP>
struct OctetWords {
  static constexpr int NSW = SW / 4;
  uint32_t c[NP];
  uint32_t s[NP][NSW > 0 ? NSW : 1];
  __device__ __forceinline__ void load(const uint32_t* cw_ptr, const uint32_t* sw_ptr,
                                       uint32_t pstride) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      c[p] = cw_ptr[p * pstride];
#pragma unroll
      for (int i = 0; i < NSW; ++i) s[p][i] = sw_ptr[p * pstride + i * kBlockPts];
    }
  }
};

template <int NQ, int SW, int NP>
__device__ __forceinline__ void score_octet_k16(const OctetWords<SW, NP>& wd, uint32_t eta_sa,
                                                const float* lam_o, uint32_t s,
                                                float (&acc)[NP][NQ]) {
  constexpr int RS = rs_of(NQ);
  static_assert(RS == 1 || RS == 2, "fast octet needs a power-of-two row stride");
  constexpr int L = RS == 1 ? 2 : 3;            // log2(bytes per center row)
  constexpr uint32_t M = 0xFu << L;             // center field, scaled
  constexpr uint32_t SEC = 16u * RS * 4u;       // bytes per section block
  auto row = [&](uint32_t w, int b) -> uint32_t {
    const uint32_t off = b == 0 ? ((w << L) & M) : ((w >> (4 * b - L)) & M);
    return (eta_sa | off) + static_cast<uint32_t>(b) * SEC;
  };
  auto alpha_of = [&](int p, int b) -> float {
    if constexpr (SW == 16) {
      return __half2float(__ushort_as_half(
          static_cast<unsigned short>((wd.s[p][b >> 1] >> (16 * (b & 1))) & 0xFFFFu)));
    } else if constexpr (SW == 32) {
      return __uint_as_float(wd.s[p][b]);
    } else if constexpr (SW == 8) {
      return lam_o[b * s + ((wd.s[p][b >> 2] >> (8 * (b & 3))) & 0xFFu)];
    } else if constexpr (SW == 4) {
      return lam_o[b * s + ((wd.s[p][0] >> (4 * b)) & 0xFu)];
    } else {
      return lam_o[b];
    }
  };
#pragma unroll
  for (int b = 0; b < 8; b += 2) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if constexpr (NQ == 1) {
        const float e0 = lds_f32(row(wd.c[p], b));
        const float e1 = lds_f32(row(wd.c[p], b + 1));
        float t0, t1;
        unpack2(fmul2_rn(pack2(e0, e1), pack2(alpha_of(p, b), alpha_of(p, b + 1))), t0, t1);
        acc[p][0] = __fadd_rn(acc[p][0], t0);
        acc[p][0] = __fadd_rn(acc[p][0], t1);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float al = alpha_of(p, b + h);
          float tx, ty;
          unpack2(fmul2_rn(lds_b64(row(wd.c[p], b + h)), pack2(al, al)), tx, ty);
          acc[p][0] = __fadd_rn(acc[p][0], tx);
          acc[p][1] = __fadd_rn(acc[p][1], ty);
        }
      }
    }
  }
}

// Scores NP points (word pointers wp + p * pstride) for NQ queries: the
// sections [0, m) in order, 8 per octet.  NP > 1 interleaves independent
// points so a thread carries NP dependent add chains at once (small query
// groups are otherwise latency bound on the single chain).
template <int NQ, int CW, int SW, int KT, int NP = 1>
__device__ __forceinline__ void score_point(const uint32_t* wp, uint32_t pstride, uint32_t eta_sa,
                                            const float* s_eta,
                                            const float* s_lam, uint32_t k_rt, uint32_t s,
                                            uint32_t cbits_rt, uint32_t W, uint32_t Wc, uint32_t m,
                                            float (&acc)[NP][NQ]) {
  using Cd = Codec<CW, SW>;
  constexpr int RS = rs_of(NQ);
  const uint32_t k = KT ? static_cast<uint32_t>(KT) : k_rt;
  const uint32_t cbits = KT ? static_cast<uint32_t>(__builtin_ctz(KT)) : cbits_rt;
#pragma unroll
  for (int p = 0; p < NP; ++p)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[p][q] = -0.0f;  // identity of RN addition
  const uint32_t full = m >> 3;
  const uint32_t* cw_ptr = wp;
  const uint32_t* sw_ptr = wp + (Cd::kJoint ? 0u : Wc) * kBlockPts;
  const float* eta_o = s_eta;
  const float* lam_o = s_lam;
  const uint32_t eta_step = 8 * k * RS, lam_step = 8 * s;
  if constexpr (CW == 4 && KT == 16 && NQ <= 2) {
    for (uint32_t o = 0; o < full; ++o) {
      OctetWords<SW, NP> wd;
      wd.load(cw_ptr, sw_ptr, pstride);
      score_octet_k16<NQ, SW, NP>(wd, eta_sa, lam_o, s, acc);
      cw_ptr += Cd::kCenterWords * kBlockPts;
      sw_ptr += Cd::kScaleWords * kBlockPts;
      eta_sa += eta_step * 4;
      eta_o += eta_step;
      lam_o += lam_step;
    }
  } else {
    for (uint32_t o = 0; o < full; ++o) {
      score_octet<NQ, CW, SW, KT, false, NP>(cw_ptr, sw_ptr, pstride, 0, 0, 8, eta_o, lam_o, k, s,
                                             cbits, acc);
      cw_ptr += Cd::kCenterWords * kBlockPts;
      sw_ptr += Cd::kScaleWords * kBlockPts;
      eta_o += eta_step;
      lam_o += lam_step;
    }
  }
  if (m & 7u) {
    // words of the last octet that exist in the row
    const uint32_t cw0 = full * Cd::kCenterWords;
    const uint32_t ncw = (Cd::kJoint ? W : Wc) - cw0;
    const uint32_t nsw = Cd::kScaleWords > 0 ? W - (Wc + full * Cd::kScaleWords) : 0u;
    score_octet<NQ, CW, SW, KT, true, NP>(cw_ptr, sw_ptr, pstride, ncw, nsw, m & 7u, eta_o, lam_o,
                                          k, s, cbits, acc);
  }
}

// ---- filter (FT): a cheap upper-precision-bounded pre-score that decides
// which points need the exact score.  Per (point, section) one fp16 lambda_hat
// and 16 fp16 eta_hat values (four conflict-free LDS.64), 8 HFMA2: products
// and sums in fp16 within an octet, fp32 across octets.  eta_hat =
// fp16(eta * sigma_q / tau_j), lambda_hat = fp16(lambda * tau_j) with powers of
// two sigma_q, tau_j that keep every octet sum far from fp16 overflow.  The
// filter score f_q then satisfies |f_q - sigma_q * score_q| <= sigma_q * eps_q
// (bound and proof in DESIGN.md §4, K2-F), so a point is scored exactly iff
// some query has f_q >= fl_down(fl_down(tau_q - eps_q) * sigma_q): every point
// that can reach a query's top-K is scored exactly, and only those.
__device__ __forceinline__ void unpack_h2(uint64_t v, __half2& a, __half2& b) {
  uint32_t lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
  a = *reinterpret_cast<__half2*>(&lo);
  b = *reinterpret_cast<__half2*>(&hi);
}

template <bool kPartial>
__device__ __forceinline__ void filter_octet16(const uint32_t* cw_ptr, uint32_t ncw, uint32_t nsec,
                                               uint32_t eh_sa, const __half* lam_o, uint32_t s,
                                               float (&f)[16]) {
  uint32_t w[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) w[i] = (!kPartial || static_cast<uint32_t>(i) < ncw) ? cw_ptr[i * kBlockPts] : 0u;
  __half2 h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = __float2half2_rn(0.0f);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (kPartial && b >= static_cast<int>(nsec)) break;
    const uint32_t byte = (w[b >> 2] >> (8 * (b & 3))) & 0xFFu;
    const __half2 lam2 = __half2half2(lam_o[b * s + (byte >> 4)]);
    const uint32_t row = eh_sa + ((b * 16u + (byte & 15u)) * kFRS) * 2u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __half2 e0, e1;
      unpack_h2(lds_b64(row + 8u * j), e0, e1);
      h[2 * j] = __hfma2(e0, lam2, h[2 * j]);
      h[2 * j + 1] = __hfma2(e1, lam2, h[2 * j + 1]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 v = __half22float2(h[i]);
    f[2 * i] += v.x;
    f[2 * i + 1] += v.y;
  }
}

// filter scores of one point (16 queries); wp: the point's first code word
__device__ __forceinline__ void filter_point16(const uint32_t* wp, uint32_t eh_sa, const __half* s_flam,
                                               uint32_t s, uint32_t W, uint32_t m, float (&f)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) f[q] = 0.0f;
  const uint32_t full = m >> 3;
  for (uint32_t o = 0; o < full; ++o)
    filter_octet16<false>(wp + 2u * o * kBlockPts, 2, 8, eh_sa + o * (8u * 16u * kFRS * 2u), s_flam + o * 8u * s,
                          s, f);
  if (m & 7u)
    filter_octet16<true>(wp + 2u * full * kBlockPts, W - 2u * full, m & 7u, eh_sa + full * (8u * 16u * kFRS * 2u),
                         s_flam + full * 8u * s, s, f);
}

// PLANES with 4-bit centers (k = 16) and raw fp16 alpha (config 3), groups of
// 16: the stored alpha is an fp16 value, used as is (no rounding); the eta_hat
// rows are those of the JOINT8 variant.  Point words: [Wc center words (8
// codes each)][alpha words (2 each)].
__device__ __forceinline__ void filter_point16_raw(const uint32_t* wp, uint32_t eh_sa, uint32_t Wc, uint32_t m,
                                                   float (&f)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) f[q] = 0.0f;
  for (uint32_t o = 0; 8 * o < m; ++o) {
    const uint32_t nsec = min(8u, m - 8 * o);
    const uint32_t cw = wp[o * kBlockPts];
    uint32_t aw[4];
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) aw[i] = 2 * i < nsec ? wp[(Wc + 4 * o + i) * kBlockPts] : 0u;
    __half2 h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = __float2half2_rn(0.0f);
#pragma unroll
    for (uint32_t b = 0; b < 8; ++b) {
      if (b >= nsec) break;
      const __half al = __ushort_as_half(static_cast<unsigned short>(aw[b >> 1] >> (16 * (b & 1))));
      const __half2 a2 = __half2half2(al);
      const uint32_t row = eh_sa + (((8 * o + b) * 16u + ((cw >> (4 * b)) & 0xFu)) * kFRS) * 2u;
      PCPQG_DASSERT(8 * o + b < m);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __half2 e0, e1;
        unpack_h2(lds_b64(row + 8u * j), e0, e1);
        h[2 * j] = __hfma2(e0, a2, h[2 * j]);
        h[2 * j + 1] = __hfma2(e1, a2, h[2 * j + 1]);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 v = __half22float2(h[i]);
      f[2 * i] += v.x;
      f[2 * i + 1] += v.y;
    }
  }
}

// exact score of one (point, query) pair, raw fp16 alpha: the reference's
// fl(alpha * eta) terms (pq_index.cpp:230-236) added in section order
template <int RS>
__device__ __forceinline__ float exact_pair_raw16(const uint32_t* wp, uint32_t q, const float* s_eta, uint32_t Wc,
                                                  uint32_t m) {
  // all code words in flight first (m <= 64: 8 center words, 32 alpha words)
  uint32_t cw[8], aw[32];
#pragma unroll
  for (uint32_t w = 0; w < 8; ++w) cw[w] = 8 * w < m ? wp[w * kBlockPts] : 0u;
#pragma unroll
  for (uint32_t w = 0; w < 32; ++w) aw[w] = 2 * w < m ? wp[(Wc + w) * kBlockPts] : 0u;
  float acc = -0.0f;
#pragma unroll
  for (uint32_t j = 0; j < 64; ++j) {
    if (j >= m) break;
    const uint32_t c = (cw[j >> 3] >> (4 * (j & 7))) & 0xFu;
    const float al = __half2float(__ushort_as_half(static_cast<unsigned short>(aw[j >> 1] >> (16 * (j & 1)))));
    acc = __fadd_rn(acc, __fmul_rn(s_eta[(j * 16 + c) * RS + q], al));
  }
  return acc;
}

// PLANES with 8-bit centers and 4-bit scale codes (config 4, k <= 256), groups
// of 4 queries: eta_hat rows of 4 halves (one LDS.64), same products and sums.
// Point words: [Wc center words (4 codes each)][scale words (8 codes each)].
__device__ __forceinline__ void filter_point_p8s4(const uint32_t* wp, uint32_t eh_sa, const __half* s_flam,
                                                  uint32_t s, uint32_t k, uint32_t Wc, uint32_t m, float (&f)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) f[q] = 0.0f;
  for (uint32_t o = 0; 8 * o < m; ++o) {
    const uint32_t nsec = min(8u, m - 8 * o);
    const uint32_t c0 = wp[(2 * o) * kBlockPts];
    const uint32_t c1 = nsec > 4 ? wp[(2 * o + 1) * kBlockPts] : 0u;
    const uint32_t sw = wp[(Wc + o) * kBlockPts];
    __half2 h0 = __float2half2_rn(0.0f), h1 = __float2half2_rn(0.0f);
#pragma unroll
    for (uint32_t b = 0; b < 8; ++b) {
      if (b >= nsec) break;
      const uint32_t j = 8 * o + b;
      const uint32_t c = ((b < 4 ? c0 : c1) >> (8 * (b & 3))) & 0xFFu;
      const __half2 lam2 = __half2half2(s_flam[j * s + ((sw >> (4 * b)) & 0xFu)]);
      __half2 e0, e1;
      unpack_h2(lds_b64(eh_sa + (j * k + c) * 8u), e0, e1);
      h0 = __hfma2(e0, lam2, h0);
      h1 = __hfma2(e1, lam2, h1);
    }
    const float2 v0 = __half22float2(h0), v1 = __half22float2(h1);
    f[0] += v0.x;
    f[1] += v0.y;
    f[2] += v1.x;
    f[3] += v1.y;
  }
}

// exact score of one (point, query) pair, PLANES 8-bit centers / 4-bit scales,
// the eta rows read from the group's table in global memory (L2)
__device__ __forceinline__ float exact_pair_p8s4(const uint32_t* wp, uint32_t q, const float* geta, int rs,
                                                 const float* s_lam, uint32_t s, uint32_t k, uint32_t Wc,
                                                 uint32_t m) {
  // all code words in flight first (m <= 64: 16 center words, 8 scale words),
  // then the eta rows (each depends only on its code) before the ordered adds
  uint32_t cw[16], sw[8];
#pragma unroll
  for (uint32_t w = 0; w < 16; ++w) cw[w] = 4 * w < m ? wp[w * kBlockPts] : 0u;
#pragma unroll
  for (uint32_t w = 0; w < 8; ++w) sw[w] = 8 * w < m ? wp[(Wc + w) * kBlockPts] : 0u;
  float acc = -0.0f;
#pragma unroll
  for (uint32_t j = 0; j < 64; ++j) {
    if (j >= m) break;
    const uint32_t c = (cw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t l = (sw[j >> 3] >> (4 * (j & 7))) & 0xFu;
    acc = __fadd_rn(acc, __fmul_rn(__ldg(geta + (static_cast<size_t>(j) * k + c) * rs + q), s_lam[j * s + l]));
  }
  return acc;
}

// exact score of one (point, query) pair, JOINT8 with k = 16: the reference's
// fl(eta * lambda) terms added in section order (same bits as score_point)
template <int RS>
__device__ __forceinline__ float exact_pair_joint8_k16(const uint32_t* wp, uint32_t q, const float* s_eta,
                                                       const float* s_lam, uint32_t s, uint32_t m) {
  // the point's code words come from L2: all of them in flight first (m <= 64)
  uint32_t wd[16];
#pragma unroll
  for (uint32_t w = 0; w < 16; ++w) wd[w] = 4 * w < m ? wp[w * kBlockPts] : 0u;
  float acc = -0.0f;
#pragma unroll
  for (uint32_t j = 0; j < 64; ++j) {
    if (j >= m) break;
    const uint32_t byte = (wd[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    acc = __fadd_rn(acc, __fmul_rn(s_eta[(j * 16 + (byte & 15u)) * RS + q], s_lam[j * s + (byte >> 4)]));
  }
  return acc;
}

// one candidate for one query (the per-lane branch of try_insert); false if
// the buffer is full (the caller retries after a flush)
__device__ __forceinline__ bool insert_one(float sc, uint32_t id, uint32_t q, uint64_t* s_buf,
                                           const uint64_t* s_tau, uint32_t* s_cnt, uint32_t* s_flag,
                                           uint32_t cap, uint32_t reserve, uint32_t first_flush) {
  const uint64_t key = make_key(sc, id);
  if (key <= s_tau[q]) return true;
  const uint32_t slot = atomicAdd(&s_cnt[q], 1u);
  if (slot < cap) {
    s_buf[q * cap + slot] = key;
    if (slot + 1 > cap - reserve || (slot + 1 > first_flush && s_tau[q] == 0ull)) atomicOr(s_flag, 1u);
    return true;
  }
  atomicOr(s_flag, 2u);
  return false;
}

// Candidate buffers.  Per query: cap keys, a running K-th-best key tau and a
// count.  A candidate is appended only if its key beats tau.  A buffer that
// reaches cap - reserve is compacted to its K best keys behind the tile
// barrier.  With ppt > 1 the reserve covers a whole tile, so nothing can
// overflow; with ppt == 1 (large batches, where shared memory is tight) the
// reserve is small and a rare overflowing insert is retried after the flush.
template <int NQ>
__device__ __forceinline__ uint32_t try_insert(const float (&acc)[NQ], uint32_t want, uint32_t id,
                                               const float (&tauf)[NQ], uint64_t* s_buf,
                                               const uint64_t* s_tau, uint32_t* s_cnt,
                                               uint32_t* s_flag, uint32_t cap, uint32_t reserve,
                                               uint32_t first_flush) {
  // Warp-aggregated: one shared atomic per (warp, query) with candidates, so
  // the warm-up tiles (where every point is a candidate) do not serialise on
  // a single counter.
  if constexpr (NQ >= 8) {
    // wide query groups: candidates are spread thin over 16 queries, so a
    // per-lane atomic on the few passing (lane, query) pairs is cheaper
    uint32_t pend = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (((want >> q) & 1u) && acc[q] >= tauf[q]) {
        const uint64_t key = make_key(acc[q], id);
        if (key > s_tau[q]) {
          const uint32_t slot = atomicAdd(&s_cnt[q], 1u);
          if (slot < cap) {
            s_buf[q * cap + slot] = key;
            if (slot + 1 > cap - reserve || (slot + 1 > first_flush && s_tau[q] == 0ull))
              atomicOr(s_flag, 1u);
          } else {
            pend |= 1u << q;
            atomicOr(s_flag, 2u);
          }
        }
      }
    }
    return pend;
  }
  const uint32_t active = __activemask();
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t pend = 0, cand = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (((want >> q) & 1u) && acc[q] >= tauf[q]) cand |= 1u << q;
  const uint32_t wq = __reduce_or_sync(active, cand);  // queries with a candidate in this warp
  if (wq == 0u) return 0u;                               // the common case after warm-up
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (!((wq >> q) & 1u)) continue;  // warp-uniform
    bool ins = false;
    uint64_t key = 0ull;
    if ((cand >> q) & 1u) {
      key = make_key(acc[q], id);
      ins = key > s_tau[q];
    }
    const uint32_t bal = __ballot_sync(active, ins);
    if (bal == 0u) continue;
    const uint32_t leader = __ffs(bal) - 1u;
    uint32_t base = 0;
    if (lane == leader) {
      const uint32_t cnt = __popc(bal);
      base = atomicAdd(&s_cnt[q], cnt);
      const uint32_t after = base + cnt;
      // compact when the next tile could overflow, and early (at 2K keys)
      // while this query has no threshold yet
      if (after > cap - reserve || (after > first_flush && s_tau[q] == 0ull)) atomicOr(s_flag, 1u);
      if (after > cap) atomicOr(s_flag, 2u);
    }
    base = __shfl_sync(active, base, leader);
    if (ins) {
      const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
      if (slot < cap) s_buf[q * cap + slot] = key;
      else pend |= 1u << q;
    }
  }
  return pend;
}

// WS (warp-specialised, top-K with ppt > 1 only): the last warp is a TMA
// producer that refills a stage once every compute warp has released it
// (per-stage "empty" mbarriers), so compute warps never meet at a per-tile
// CTA barrier; they meet (named barrier 15, above the compaction groups' 1..4) only when a candidate buffer needs
// compaction.  A warp checks the flag before each tile, so after a flag is
// raised every warp scores at most the rest of its current tile: the one-tile
// reserve still bounds every buffer.
template <int NQ, int CW, int SW, int KT, bool WS = false, bool FT = false>
__global__ void __launch_bounds__(512, 1)
    scan_topk_kernel(const ScanArgs a) {
  static_assert(!FT || (!WS && ((NQ == 16 && CW == 0 && KT == 16) || (NQ == 4 && CW == 8 && SW == 4) ||
                                 (NQ == 16 && CW == 4 && SW == 16 && KT == 16))),
                "filter: JOINT8 k = 16 or raw fp16 alpha k = 16 in groups of 16, or PLANES 8-bit centers / "
                "4-bit scales in groups of 4");
  constexpr bool FTR = FT && CW == 4;  // raw fp16 alpha
  // FTP (PLANES, k up to 256): the exact eta table does not fit next to the
  // fp16 one, so exact re-scores read it from global memory and the queue is
  // drained early enough never to overflow (no direct path)
  constexpr bool FTP = FT && CW == 8;
  constexpr int FRS = FTP ? NQ : kFRS;  // halves per eta_hat row
  using Cd = Codec<CW, SW>;
  constexpr int RS = rs_of(NQ);
  extern __shared__ __align__(128) uint8_t smem[];

  const uint32_t k = a.k, s = a.s, W = a.W;
  const int nthr = WS ? static_cast<int>(blockDim.x) - 32 : static_cast<int>(blockDim.x);
  const uint32_t g = blockIdx.x;  // query group
  const uint32_t nq_valid = min(static_cast<uint32_t>(NQ), a.B - g * NQ);
  const uint32_t want_all = nq_valid >= 32 ? 0xFFFFFFFFu : ((1u << nq_valid) - 1u);
  const bool topk = a.scores == nullptr;

  // ---- shared memory carve-up (every region 16-byte aligned):
  //  [code tiles x stages][candidates NQ*cap][eta m8*k*RS][lambda m8*s][hist][header]
  const uint32_t tile_pts = nthr * a.ppt;
  const uint32_t tile_words = tile_pts * W;
  const int ngroups = scan_ngroups(NQ, nthr);
  uint8_t* ptr = smem;
  uint32_t* s_tile = reinterpret_cast<uint32_t*>(ptr);
  ptr += static_cast<size_t>(a.stages) * tile_words * 4;
  uint64_t* s_buf = reinterpret_cast<uint64_t*>(ptr);
  ptr += topk ? static_cast<size_t>(NQ) * a.cap * 8 : 0;
  ptr += (128u - (static_cast<uint32_t>(__cvta_generic_to_shared(ptr)) & 127u)) & 127u;
  float* s_eta = reinterpret_cast<float*>(ptr);  // 128-byte aligned (score_octet_k16)
  const uint32_t eta_sa0 = smem_u32(s_eta);
  ptr += FTP ? 0 : (static_cast<size_t>(a.m8) * k * RS * 4 + 15) & ~static_cast<size_t>(15);
  float* s_lam = reinterpret_cast<float*>(ptr);
  ptr += Cd::kNoLambda ? 0 : ((a.m8 * s * 4 + 15u) & ~15u);
  __half* s_fh = reinterpret_cast<__half*>(ptr);     // FT: eta_hat rows [m8*k][FRS]
  ptr += FT ? static_cast<size_t>(a.m8) * k * FRS * 2 : 0;
  __half* s_flam = reinterpret_cast<__half*>(ptr);   // FT: lambda_hat [m8][s]
  ptr += FT ? ((a.m8 * s * 2 + 15u) & ~15u) : 0;
  float* s_thr = reinterpret_cast<float*>(ptr);      // FT: per-query filter threshold
  ptr += FT ? 64 : 0;
  uint32_t* s_qcnt = reinterpret_cast<uint32_t*>(ptr);  // FT: queue length (+ pad)
  ptr += FT ? 16 : 0;
  uint32_t* s_queue = reinterpret_cast<uint32_t*>(ptr);  // FT: re-score queue
  ptr += FT ? kFQCap * 4 : 0;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(ptr);  // ngroups x kGroupScratch words
  ptr += topk ? static_cast<size_t>(ngroups) * (kGroupScratch) * 4 : 0;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(ptr);        // up to 4 mbarriers
  uint64_t* s_tau = reinterpret_cast<uint64_t*>(ptr + 32);   // 16 x u64
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(ptr + 160);  // 16 x u32
  uint32_t* s_flag = reinterpret_cast<uint32_t*>(ptr + 224);
  uint64_t* s_empty = reinterpret_cast<uint64_t*>(ptr + 256);  // WS: up to 4 mbarriers
#ifdef PCPQG_DEBUG
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    PCPQG_DASSERT(static_cast<size_t>(ptr + 320 - smem) <= dyn);  // the carve-up fits the launch
  }
#endif

  const int tid = threadIdx.x;
  const uint32_t reserve = a.ppt > 1 ? tile_pts : min(64u, a.cap - a.K);

  // ---- point range of this CTA: blocks [b0, b1)
  const uint32_t cx = blockIdx.y, ncx = gridDim.y;
  const uint32_t b0 = static_cast<uint32_t>((static_cast<uint64_t>(a.n_blocks) * cx) / ncx);
  const uint32_t b1 = static_cast<uint32_t>((static_cast<uint64_t>(a.n_blocks) * (cx + 1)) / ncx);
  const uint32_t tile_blocks = tile_pts / kBlockPts;
  const uint32_t ntiles = (b1 - b0 + tile_blocks - 1) / tile_blocks;
  const uint64_t p_end = min(a.n_local, static_cast<uint64_t>(b1) * kBlockPts);

  if (tid == 0) {
    for (uint32_t i = 0; i < a.stages; ++i) mbar_init(&s_bar[i], 1);
    if constexpr (WS)
      for (uint32_t i = 0; i < a.stages; ++i) mbar_init(&s_empty[i], static_cast<uint32_t>(nthr / 32));
    fence_mbar_init();
    *s_flag = 0;
  }
  auto issue_tile = [&](uint32_t t) {
    const uint32_t blk = b0 + t * tile_blocks;
    const uint32_t nb = min(tile_blocks, b1 - blk);
    const uint32_t bytes = nb * W * kBlockPts * 4;
    uint64_t* bar = &s_bar[t % a.stages];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(s_tile + static_cast<size_t>(t % a.stages) * tile_words,
             a.codes + static_cast<size_t>(blk) * W * kBlockPts, bytes, bar);
  };
  if constexpr (WS) {
    // The code stream does not depend on the LUT kernel: with a programmatic
    // dependent launch the producer warp starts streaming tiles while the LUT
    // kernel drains; only the table staging below waits for it.
    __syncthreads();  // the mbarriers are initialised
    if (tid >= nthr) {  // producer warp: one elected lane streams every tile
      if (tid == nthr) {
        for (uint32_t t = 0; t < ntiles; ++t) {
          if (t >= a.stages) {
            mbar_wait(&s_empty[t % a.stages], ((t / a.stages) - 1) & 1u);
            fence_proxy_async();  // WAR: the compute warps' reads precede the async write
          }
          issue_tile(t);
        }
      }
      return;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no-op without a programmatic launch)
  {
    if (WS && a.lut_mode) {
      // K1 inside the scan: this group's tables straight into shared memory, with
      // lut_kernel's operations in its order (build_lookup_table, pq_index.cpp:183-208)
      const uint32_t rows = k, total = a.m8 * rows * NQ;
      const uint32_t cmask = (1u << a.cbits) - 1u;
      for (uint32_t t = tid; t < total; t += nthr) {
        const uint32_t r = t % rows, j = (t / rows) % a.m8, qi = t / (rows * a.m8);
        const uint64_t q = static_cast<uint64_t>(g) * NQ + qi;
        const uint32_t c = a.lut_mode == 2 ? (r & cmask) : r;
        const uint32_t l = a.lut_mode == 2 ? (r >> a.cbits) : 0u;
        float acc = 0.0f;
        if (j >= a.m) {
          acc = -0.0f;
        } else if (q < a.B && c < a.kc) {
          const float* row = a.cb + (static_cast<uint64_t>(j) * a.kc + c) * a.dbar;
          const float* qq = a.Q + q * a.d;
          for (uint32_t e = 0; e < a.dbar; ++e) {
            const uint32_t col = j * a.dbar + e;
            const float qa = col < a.d ? __ldg(qq + col) : 0.0f;
            acc = __fadd_rn(acc, __fmul_rn(__ldg(row + e), qa));
          }
          if (a.lut_mode == 2) acc = l < s ? __fmul_rn(acc, __ldg(a.lam + static_cast<uint64_t>(j) * s + l)) : 0.0f;
        }
        s_eta[(static_cast<size_t>(j) * rows + r) * RS + qi] = acc;
      }
    }
    const float4* src = reinterpret_cast<const float4*>(a.eta + static_cast<size_t>(g) * a.gstride);
    float4* dst = reinterpret_cast<float4*>(s_eta);
    const uint32_t n4 = (FTP || (WS && a.lut_mode)) ? 0u : (a.m8 * k * RS + 3) / 4;
    for (uint32_t i = tid; i < n4; i += nthr) dst[i] = __ldg(src + i);
    if constexpr (!Cd::kNoLambda)
      for (uint32_t i = tid; i < a.m8 * s; i += nthr) s_lam[i] = __ldg(a.lam + i);
    if constexpr (FT) {
      const float4* fsrc = reinterpret_cast<const float4*>(a.fh + static_cast<size_t>(g) * a.fgstride);
      float4* fdst = reinterpret_cast<float4*>(s_fh);
      const uint32_t f4 = a.m8 * k * FRS * 2 / 16;
      for (uint32_t i = tid; i < f4; i += nthr) fdst[i] = __ldg(fsrc + i);
      for (uint32_t i = tid; i < a.m8 * s; i += nthr) s_flam[i] = a.flam[i];
      if (tid < NQ) s_thr[tid] = tid < static_cast<int>(nq_valid) ? -INFINITY : INFINITY;
      if (tid == 0) *s_qcnt = 0u;
    }
  }
  if (topk && tid < NQ) {
    s_tau[tid] = 0ull;
    s_cnt[tid] = 0u;
  }
  if constexpr (WS) {
    asm volatile("bar.sync 14, %0;" ::"r"(nthr) : "memory");  // the compute warps (the producer left)
  } else {
    __syncthreads();
    if (tid == 0)
      for (uint32_t t = 0; t < min(ntiles, a.stages - 1); ++t) issue_tile(t);
  }
  // a dependent grid (the small-batch merge) may be made resident from here on;
  // it waits for this grid's completion before it reads the lists
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // flush: compact every buffer at or over cap - reserve to its K best keys,
  // publish the new K-th key to the other CTAs of this query group
  auto flush = [&](bool force = false) {
    const int gsz = nthr / ngroups;
    Group grp{tid / gsz, gsz, tid % gsz};
    uint32_t* hist = s_hist + grp.id * (kGroupScratch);
    for (uint32_t q = grp.id; q < nq_valid; q += ngroups) {
      const uint32_t cnt = s_cnt[q];
      if (cnt + reserve > a.cap || (cnt > 2 * a.K && s_tau[q] == 0ull) || (force && cnt >= a.K)) {
        const uint32_t n = min(cnt, a.cap);
        uint64_t* buf = s_buf + q * a.cap;
        const uint64_t tau = group_select(buf, n, a.K, hist, hist + kHistWords, grp);
        group_compact(buf, n, tau, hist + kHistWords + kSvWords, grp);
        if (grp.gtid == 0) {
          s_cnt[q] = a.K;
          if (tau > s_tau[q]) s_tau[q] = tau;
          atomicMax(reinterpret_cast<unsigned long long*>(a.gtau + g * NQ + q),
                    static_cast<unsigned long long>(tau));
        }
      }
    }
  };

  // WS: all compute warps meet on named barrier 15; a raised flag is handled
  // by every warp in the same sequence (it stays raised until all have met)
  auto ws_bar = [&]() { asm volatile("bar.sync 15, %0;" ::"r"(nthr) : "memory"); };
  auto ws_meet = [&]() -> bool {
    ws_bar();
    const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(s_flag);
    if (fl) {
      flush();
      ws_bar();
      if (tid == 0) *s_flag = 0u;
      ws_bar();
    }
    return fl != 0u;
  };

  // FT: inherit the previous range's top-K once it is published (checked
  // before the first tile and after every tile; never waits).  Inserted like
  // candidates, then every buffer is compacted so tau becomes the union's K-th
  // best; only keys of this CTA's own range are emitted at the end.
  // Keys of the CTA's own range are never inherited (it scores them itself).
  bool inherited = !FT || cx == 0;
  const uint64_t own_lo = a.id_base + static_cast<uint64_t>(b0) * kBlockPts;
  const uint64_t own_hi = a.id_base + p_end;
  auto try_inherit = [&]() {
    if (inherited) return;  // CTA-uniform
    const size_t pred = static_cast<size_t>(g) * ncx + cx - 1;
    if (tid == 0) {
      uint32_t ready;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(ready) : "l"(a.carry_done + pred) : "memory");
      for (uint32_t q = 0; ready && q < nq_valid; ++q)
        if (s_cnt[q] + __ldcg(a.carry_cnt + pred * NQ + q) > a.cap) ready = 0u;  // room next time
      s_qcnt[1] = ready;
    }
    __syncthreads();
    if (!s_qcnt[1]) return;
    inherited = true;
    const uint64_t* src = a.carry + pred * NQ * a.K;
    for (uint32_t i = tid; i < nq_valid * a.K; i += nthr) {
      const uint32_t q = i / a.K;
      if (i - q * a.K >= __ldcg(a.carry_cnt + pred * NQ + q)) continue;
      const uint64_t key = __ldcg(reinterpret_cast<const unsigned long long*>(src + i));
      const uint64_t id = static_cast<uint64_t>(key_id(key));
      if (key > s_tau[q] && (id < own_lo || id >= own_hi)) s_buf[q * a.cap + atomicAdd(&s_cnt[q], 1u)] = key;
    }
    __syncthreads();
    flush(true);
    __syncthreads();
    if (tid == 0) *s_flag = 0u;
    __syncthreads();
  };

  // FT: exact re-score of the queued pairs, one pair per thread per round,
  // codes read from global memory (the tile that held them is gone); an
  // insert into a full buffer waits for the flush and is retried
  auto drain = [&](uint32_t nqe) {
    for (uint32_t r0 = 0; r0 < nqe; r0 += static_cast<uint32_t>(nthr)) {  // CTA-uniform
      const uint32_t i = r0 + tid;
      bool pending = false;
      float sc = 0.0f;
      uint32_t q = 0, pid = 0;
      const uint32_t e = i < nqe ? s_queue[i] : ~0u;
      if (e != ~0u) {
        const uint32_t pl = b0 * kBlockPts + (e >> 4);  // local point index
        q = e & 15u;
        const uint32_t* qwp = a.codes + static_cast<size_t>(pl >> 5) * W * kBlockPts + (pl & 31);
        if constexpr (FTP)
          sc = exact_pair_p8s4(qwp, q, a.eta + static_cast<size_t>(g) * a.gstride, RS, s_lam, s, k, a.Wc, a.m);
        else if constexpr (FTR)
          sc = exact_pair_raw16<RS>(qwp, q, s_eta, a.Wc, a.m);
        else
          sc = exact_pair_joint8_k16<RS>(qwp, q, s_eta, s_lam, s, a.m);
        pid = static_cast<uint32_t>(a.id_base + pl);
        pending = !insert_one(sc, pid, q, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve, 2 * a.K);
      }
      __syncthreads();
      uint32_t fl = *s_flag;
      while (fl) {  // CTA-uniform
        flush();
        __syncthreads();
        if (tid == 0) *s_flag = 0u;
        __syncthreads();
        if (!(fl & 2u)) break;
        if (pending) pending = !insert_one(sc, pid, q, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve, 2 * a.K);
        __syncthreads();
        fl = *s_flag;
      }
    }
    __syncthreads();
    if (tid == 0) *s_qcnt = 0u;
    __syncthreads();  // later appends follow the reset
  };

  float tauf[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) tauf[q] = -INFINITY;
  if constexpr (FT) {
    try_inherit();
#pragma unroll
    for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
  }

  uint32_t stage = 0, phase = 0;  // t % stages, (t / stages) & 1
  for (uint32_t t = 0; t < ntiles; ++t, stage = stage + 1 == a.stages ? 0 : stage + 1,
                phase ^= stage == 0 ? 1u : 0u) {
    if constexpr (WS) {
      if (*reinterpret_cast<volatile uint32_t*>(s_flag)) ws_meet();
    } else if (tid == 0 && t + a.stages - 1 < ntiles) {
      fence_proxy_async();  // WAR: generic-proxy reads of the reused stage precede the async write
      issue_tile(t + a.stages - 1);
    }
    // The K-th key published by the other CTAs of this group is loaded now
    // and adopted after the tile's scoring (never lowers tau: a key below any
    // CTA's K-th best cannot reach the global top-K), so the L2 round trip
    // overlaps the compute instead of holding warp 0 — and with it the tile
    // barrier — for its latency.
    // (Only the warp-specialised kernel defers: in the wide-group kernels the
    // value live across the tile costs ~28 registers per thread.)
    uint64_t gt_pref = 0ull;
    if (topk) {
      if (tid < static_cast<int>(nq_valid)) {
        const uint64_t gt = __ldcg(reinterpret_cast<const unsigned long long*>(a.gtau + g * NQ + tid));
        if constexpr (WS) gt_pref = gt;
        else if (gt > s_tau[tid]) s_tau[tid] = gt;
        if constexpr (FT) {
          // filter threshold of this query, rounded down twice (any tau read
          // by a racing thread is an older, lower one: still a valid bound)
          const float2 se = __ldg(a.fse + g * NQ + tid);
          s_thr[tid] = se.x == 0.0f ? -INFINITY : __fmul_rd(__fsub_rd(key_score(s_tau[tid]), se.y), se.x);
        }
      }
      if constexpr (!FT) {  // (FT reads tau only on its rare direct path)
#pragma unroll
        for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
      }
    }
    mbar_wait(&s_bar[stage], phase);
    const uint32_t* tile = s_tile + static_cast<size_t>(stage) * tile_words;
    const uint32_t tile_p0 = (b0 + t * tile_blocks) * kBlockPts;

    float acc[NQ];
    uint32_t pend = 0, id = 0;
    // emit one scored point: scores-only row or a top-K candidate
    auto emit = [&](const float (&sc)[NQ], uint64_t p) {
      if (!topk) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < static_cast<int>(nq_valid))
            a.scores[static_cast<size_t>(g * NQ + q) * a.n_local + p] = sc[q];
        return;
      }
      id = static_cast<uint32_t>(a.id_base + p);
      pend = try_insert<NQ>(sc, want_all, id, tauf, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve,
                            2 * a.K);
    };
    uint32_t r = 0;
    if constexpr (NQ <= 2) {
      // two points per thread in flight (points r*nthr + tid and (r+1)*nthr + tid)
      const uint32_t pstride = static_cast<uint32_t>(nthr) * W;
      for (; r + 1 < a.ppt; r += 2) {
        const uint32_t lp = r * nthr + tid;
        const uint64_t p = static_cast<uint64_t>(tile_p0) + lp;
        const uint32_t* wp = tile + (lp >> 5) * W * kBlockPts + (lp & 31);
        if (p + nthr < p_end) {
          float acc2[2][NQ];
          score_point<NQ, CW, SW, KT, 2>(wp, pstride, eta_sa0, s_eta, s_lam, k, s, a.cbits, W, a.Wc, a.m,
                                         acc2);
          emit(acc2[0], p);
          emit(acc2[1], p + nthr);
        } else {
          // tile tail: lanes past the end hold stale words, never decode them
#pragma unroll 1
          for (uint32_t h = 0; h < 2; ++h) {
            const uint64_t ph = p + h * nthr;
            if (ph < p_end) {
              float acc1[1][NQ];
              score_point<NQ, CW, SW, KT, 1>(wp + h * pstride, 0, eta_sa0, s_eta, s_lam, k, s, a.cbits, W,
                                             a.Wc, a.m, acc1);
              emit(acc1[0], ph);
            }
          }
        }
      }
    }
    for (; r < a.ppt; ++r) {
      const uint32_t lp = r * nthr + tid;                      // point within tile
      const uint64_t p = static_cast<uint64_t>(tile_p0) + lp;  // local point id
      const bool valid = p < p_end;  // inside this CTA's blocks and the shard
      const uint32_t* wp = tile + (lp >> 5) * W * kBlockPts + (lp & 31);
      PCPQG_DASSERT((lp >> 5) * W * kBlockPts + (lp & 31) < tile_words);
      // lanes past the end of a partial tile hold stale words: never decode them
      // (a stale center code can exceed k and index outside the table)
      if constexpr (FT) {
        // (warp-uniform: ppt == 1, every lane runs this once per tile)
        uint32_t mask = 0;
        if (valid) {
          float f[NQ];
          if constexpr (FTP) filter_point_p8s4(wp, smem_u32(s_fh), s_flam, s, k, a.Wc, a.m, f);
          else if constexpr (FTR) filter_point16_raw(wp, smem_u32(s_fh), a.Wc, a.m, f);
          else filter_point16(wp, smem_u32(s_fh), s_flam, s, W, a.m, f);
#pragma unroll
          // !(f < thr): a NaN pre-score (never expected) fails safe, to the exact score
          for (int q = 0; q < NQ; ++q) mask |= (f[q] < s_thr[q] ? 0u : 1u) << q;
          if (a.fmode != 1) {  // diagnostics only
            if (a.fmode == 2) mask = 0;
            if (a.fmode == 3 && mask) {
              atomicAdd(a.fcount, static_cast<unsigned long long>(__popc(mask)));
              atomicAdd(a.fcount + 2 + min(blockIdx.y, 63u), static_cast<unsigned long long>(__popc(mask)));
            }
          }
        }
        if (!__any_sync(0xFFFFFFFFu, mask != 0u)) continue;  // the common case
        // queue the passing (point, query) pairs, one shared atomic per warp
        const uint32_t lane = tid & 31u;
        const uint32_t cnt = __popc(mask);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= static_cast<uint32_t>(o)) incl += v;
        }
        const uint32_t wtot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        uint32_t base = 0;
        if (lane == 31 && wtot) base = atomicAdd(s_qcnt, wtot);
        base = __shfl_sync(0xFFFFFFFFu, base, 31);
        const uint32_t slot0 = base + incl - cnt;
        if (mask) {
          if (slot0 + cnt <= static_cast<uint32_t>(kFQCap)) {
            uint32_t mm = mask, sl = slot0;
            while (mm) {
              const uint32_t q = __ffs(mm) - 1u;
              mm &= mm - 1u;
              s_queue[sl++] = ((static_cast<uint32_t>(p) - b0 * kBlockPts) << 4) | q;
            }
          } else if constexpr (!FTP) {  // queue full (warm-up): score this point now, every query
            for (uint32_t sl = slot0; sl < min(slot0 + cnt, static_cast<uint32_t>(kFQCap)); ++sl) s_queue[sl] = ~0u;
            if (a.fmode == 3) atomicAdd(a.fcount + 1, 1ull);
#pragma unroll
            for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
            float acc1[1][NQ];
            score_point<NQ, CW, SW, KT, 1>(wp, 0, eta_sa0, s_eta, s_lam, k, s, a.cbits, W, a.Wc, a.m, acc1);
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = acc1[0][q];
            emit(acc, p);
          } else {
            PCPQG_DASSERT(false);  // FTP drains before a tile could overflow the queue
          }
        }
        continue;  // pairs that failed the filter are provably outside the top-K
      }
      if (valid) {
        float acc1[1][NQ];
        score_point<NQ, CW, SW, KT, 1>(wp, 0, eta_sa0, s_eta, s_lam, k, s, a.cbits, W, a.Wc, a.m, acc1);
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = acc1[0][q];
        emit(acc, p);
      }
    }
    if (WS && topk && tid < static_cast<int>(nq_valid) && gt_pref > s_tau[tid]) s_tau[tid] = gt_pref;
    if constexpr (WS) {
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&s_empty[stage]);  // release the stage
      continue;
    }
    __syncthreads();  // tile consumed; candidate writes visible
    if (topk) {
      uint32_t fl = *s_flag;
      while (fl) {  // CTA-uniform
        flush();
        __syncthreads();
        if (tid == 0) *s_flag = 0u;
#pragma unroll
        for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
        __syncthreads();
        if (!(fl & 2u)) break;
        // an insert overflowed (ppt == 1 only): retry it against the new tau
        if (pend)
          pend = try_insert<NQ>(acc, pend, id, tauf, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve,
                                2 * a.K);
        __syncthreads();
        fl = *s_flag;
      }
    }
    if constexpr (FT) {
      // (s_qcnt is read after the tile barrier: CTA-uniform)
      const uint32_t qn = *s_qcnt;
      // FTP: room for a whole tile of pairs must remain (the planner keeps
      // tile_pts * NQ <= kFQCap / 2)
      const uint32_t drain_at = FTP ? static_cast<uint32_t>(kFQCap) - tile_pts * NQ : static_cast<uint32_t>(kFQCap) / 2;
      if (qn > drain_at || t + 1 == ntiles) drain(min(qn, static_cast<uint32_t>(kFQCap)));
      try_inherit();
    }
  }

  if (!topk) return;
  if constexpr (WS) {
    while (ws_meet()) {
    }
  }
  // ---- final: reduce every query's buffer to (at most) its K best keys
  const int gsz = nthr / ngroups;
  const Group grp{tid / gsz, gsz, tid % gsz};
  uint32_t* hist = s_hist + grp.id * (kGroupScratch);
  for (uint32_t q = grp.id; q < NQ; q += ngroups) {
    uint64_t* buf = s_buf + q * a.cap;
    uint32_t n = q < nq_valid ? min(s_cnt[q], a.cap) : 0u;
    if (n > a.K) {
      const uint64_t tau = group_select(buf, n, a.K, hist, hist + kHistWords, grp);
      n = group_compact(buf, n, tau, hist + kHistWords + kSvWords, grp);
      if (grp.gtid == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.gtau + g * NQ + q),
                  static_cast<unsigned long long>(tau));
    }
    if constexpr (FT) {
      // publish this CTA's top-K for the next range, then keep only own keys
      // (inherited ones were emitted by the CTA that scored them)
      const size_t me = static_cast<size_t>(g) * ncx + cx;
      if (q < nq_valid) {
        for (uint32_t i = grp.gtid; i < n; i += grp.size) a.carry[(me * NQ + q) * a.K + i] = buf[i];
        if (grp.gtid == 0) a.carry_cnt[me * NQ + q] = n;
      }
      grp.sync();
      for (uint32_t i = grp.gtid; i < n; i += grp.size) {
        const uint64_t id = static_cast<uint64_t>(key_id(buf[i]));
        if (id < own_lo || id >= own_hi) buf[i] = 0ull;
      }
      grp.sync();
    }
    // Emit only keys that can still reach the global top-K: all CTAs of a
    // query group run concurrently, so by now gtau is close to the final
    // K-th key and most CTAs emit almost nothing.  Survivors are compacted
    // to the front of the row, followed by empty keys, with their count.
    grp.sync();
    const uint64_t gt = q < nq_valid ? __ldcg(reinterpret_cast<const unsigned long long*>(
                                          a.gtau + g * NQ + q))
                                    : 0ull;
    if (n) n = group_compact(buf, n, gt > 1 ? gt : 1, hist + kHistWords + kSvWords, grp);
    // sort the survivors descending so the merge can run a tournament
    {
      uint32_t P = 1;
      while (P < n) P <<= 1;
      for (uint32_t i = n + grp.gtid; i < P; i += grp.size) buf[i] = 0ull;
      grp.sync();
      for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
          for (uint32_t i = grp.gtid; i < P / 2; i += grp.size) {
            const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
            const uint32_t hi = lo + stride;
            const uint64_t x = buf[lo], y = buf[hi];
            if ((x < y) == ((lo & size) == 0)) {
              buf[lo] = y;
              buf[hi] = x;
            }
          }
          grp.sync();
        }
      }
    }
    uint64_t* out = a.partial + (static_cast<size_t>(cx) * a.Bpad + g * NQ + q) * a.Ks;
    // with counts (pcnt) the merges read only the survivors, rounded up to an
    // even count (16-byte TMA pieces; the pad key must be empty): skip the rest
    const uint32_t wr = a.pcnt ? min(a.Ks, (n + 1u) & ~1u) : a.Ks;
    for (uint32_t i = grp.gtid; i < wr; i += grp.size) out[i] = i < n ? buf[i] : 0ull;
    if (a.pcnt && grp.gtid == 0) a.pcnt[static_cast<size_t>(cx) * a.Bpad + g * NQ + q] = n;
    grp.sync();
  }
  if constexpr (FT) {
    __syncthreads();  // every query's carry row is written
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.carry_done + static_cast<size_t>(g) * ncx + cx),
                   "r"(1u)
                   : "memory");
    }
  }
  if (a.done == nullptr) return;  // lists are merged by merge_kernel

  // ---- fused merge: the last CTA of this query group to finish merges the
  // group's ncx lists (still in L2) into the final rows (threadfence + ticket)
  __shared__ uint32_t s_ticket;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_ticket = atomicAdd(a.done + g, 1u);
  }
  __syncthreads();
  if (s_ticket != ncx - 1) return;
  __threadfence();
  const uint32_t total = ncx * a.K;
  const uint32_t lane = tid & 31;
  for (uint32_t q = grp.id; q < nq_valid; q += ngroups) {
    uint64_t* buf = s_buf + q * a.cap;
    const uint32_t b = g * NQ + q;
    uint64_t thr = max(1ull, static_cast<unsigned long long>(__ldcg(
                                 reinterpret_cast<const unsigned long long*>(a.gtau + b))));
    auto fetch = [&](uint32_t i) -> uint64_t {
      const uint32_t l = i / a.K, r = i - l * a.K;
      const uint64_t key = __ldcg(reinterpret_cast<const unsigned long long*>(
          a.partial + (static_cast<size_t>(l) * a.Bpad + b) * a.Ks + r));
      return key >= thr ? key : 0ull;
    };
    uint32_t* s_n = hist + kHistWords + 3;  // sv[3]
    uint32_t* wsum = hist + kHistWords + kSvWords;
    // fallback gather over the zero-padded rows (only if survivors overflow)
    auto gather = [&]() {
      if (grp.gtid == 0) *s_n = 0;
      grp.sync();
      for (uint32_t i0 = 0; i0 < total; i0 += grp.size) {
        const uint32_t i = i0 + grp.gtid;
        const uint64_t key = i < total ? fetch(i) : 0ull;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, key != 0ull);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(s_n, static_cast<uint32_t>(__popc(bal)));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
        if (key && slot < a.cap) buf[slot] = key;
      }
      grp.sync();
      const uint32_t r = *s_n;
      grp.sync();
      return r;
    };
    // Gather the lists' survivors (compacted rows, padded to even counts so
    // every piece is a 16-byte multiple) with TMA bulk copies: all lists in
    // flight at once on this group's mbarrier.  Pass 1 sums the counts, pass 2
    // issues the copies at the exclusive-scan offsets.
    const uint32_t nw = grp.size >> 5, w = grp.gtid >> 5;
    auto scan_lists = [&](bool issue, uint64_t* mb) -> uint32_t {
      uint32_t n2 = 0;
      for (uint32_t l0 = 0; l0 < ncx; l0 += grp.size) {
        const uint32_t l = l0 + grp.gtid;
        const uint32_t c = l < ncx ? (__ldcg(a.pcnt + static_cast<size_t>(l) * a.Bpad + b) + 1u) & ~1u : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= static_cast<uint32_t>(o)) incl += v;
        }
        if (lane == 31) wsum[w] = incl;
        grp.sync();
        uint32_t before = 0, chunk = 0;
        for (uint32_t t = 0; t < nw; ++t) {
          before += t < w ? wsum[t] : 0u;
          chunk += wsum[t];
        }
        grp.sync();
        const uint32_t off = n2 + before + incl - c;
        if (issue && c)
          bulk_g2s(buf + off, a.partial + (static_cast<size_t>(l) * a.Bpad + b) * a.Ks, c * 8, mb);
        n2 += chunk;
      }
      return n2;
    };
    uint32_t n = scan_lists(false, nullptr);
    if (n <= a.cap && n > 0) {
      uint64_t* mb = reinterpret_cast<uint64_t*>(hist + kHistWords + 6);  // sv[6..7]
      if (grp.gtid == 0) {
        mbar_init(mb, 1);
        fence_mbar_init();
        fence_proxy_async();  // generic-proxy use of buf precedes the async writes
        mbar_expect_tx(mb, n * 8);
      }
      grp.sync();
      scan_lists(true, mb);
      mbar_wait(mb, 0u);
      grp.sync();
      if (grp.gtid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(mb)));
    }
    if (n > a.cap) {  // rare: find the K-th key over the (zero-padded) lists first
      thr = group_select_by(fetch, total, a.K, hist, hist + kHistWords, grp);
      n = gather();  // exactly K keys are >= the K-th
    } else if (n > a.K) {
      const uint64_t tau = group_select(buf, n, a.K, hist, hist + kHistWords, grp);
      n = group_compact(buf, n, tau, hist + kHistWords + kSvWords, grp);
    }
    // sort the <= K survivors (bitonic over P <= cap keys, descending)
    uint32_t P = 1;
    while (P < n) P <<= 1;
    for (uint32_t i = n + grp.gtid; i < P; i += grp.size) buf[i] = 0ull;
    grp.sync();
    for (uint32_t size = 2; size <= P; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = grp.gtid; i < P / 2; i += grp.size) {
          const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
          const uint32_t hi = lo + stride;
          const uint64_t x = buf[lo], y = buf[hi];
          if ((x < y) == ((lo & size) == 0)) {
            buf[lo] = y;
            buf[hi] = x;
          }
        }
        grp.sync();
      }
    }
    for (uint32_t i = grp.gtid; i < a.out_stride; i += grp.size) {
      const uint64_t key = i < n ? buf[i] : 0ull;
      if (a.out_keys) a.out_keys[static_cast<size_t>(b) * a.out_stride + i] = key;
      if (a.out_ids) a.out_ids[static_cast<size_t>(b) * a.out_stride + i] = key_id(key);
      if (a.out_scores) a.out_scores[static_cast<size_t>(b) * a.out_stride + i] = key_score(key);
    }
  }
}

template <int CW, int SW, int KT = 0>
ScanFn pick_nq(int nq) {
  // nq | kWsFlag: the warp-specialised variant (query groups of 1, 2 or 4)
  switch (nq) {
    case 1 | kWsFlag: return scan_topk_kernel<1, CW, SW, KT, true>;
    case 2 | kWsFlag: return scan_topk_kernel<2, CW, SW, KT, true>;
    case 4 | kWsFlag: return scan_topk_kernel<4, CW, SW, KT, true>;
    case 1: return scan_topk_kernel<1, CW, SW, KT>;
    case 2: return scan_topk_kernel<2, CW, SW, KT>;
    case 4: return scan_topk_kernel<4, CW, SW, KT>;
    case 8: return scan_topk_kernel<8, CW, SW, KT>;
    default: return scan_topk_kernel<16, CW, SW, KT>;
  }
}


}  // namespace
}  // namespace pcpqg
