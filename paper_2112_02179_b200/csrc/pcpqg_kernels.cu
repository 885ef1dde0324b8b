// CUDA kernels of the PCPQ query-time scoring path, written for sm_100a.
//
//   lut_kernel        K1  eta[q][j][c] = fixed-order fp32 <q_j, C_j[c]>
//                         (reference build_lookup_table, proj/core/src/pq_index.cpp:183-192)
//   scan_topk_kernel  K2  fused code scan + per-CTA top-K
//                         (score_all pq_index.cpp:212-244 + the partial_sort of
//                          proj/tools/main.cpp:233-237)
//   merge_kernel      K3  merge of per-CTA / per-shard top-K lists
//
// Exactness: every score is the reference's own sequence of IEEE fp32
// operations — fl(eta * alpha) per section (pq_index.cpp:203, :232-234),
// accumulated section 0 -> m-1 (pq_index.cpp:224-226, :232-234) with
// __fmul_rn / __fadd_rn so nothing is contracted into FMA.  The accumulator
// starts at -0.0f, which is the identity of IEEE round-to-nearest addition
// (-0 + x == x bit-for-bit, including x = +-0), so the result equals the
// reference's "first term, then add the rest".
//
// Scan organisation (lanes over points, queries per thread):
//   * A CTA owns NQ queries (a "group") and a contiguous range of points.
//   * The group's eta tables sit in shared memory as rows (j*k + c) of NQ
//     floats with an odd row stride RS, so the 32 lanes of a warp — 32 points
//     at the same section j and query q, each with its own center code c —
//     hit 32 distinct banks for any k <= 32 (or share a word: broadcast).
//   * Per (point, section) the thread decodes (c, alpha) once and reuses it
//     for all NQ queries: NQ table reads + 1 scale read per NQ lookups.
//   * Code tiles (256*PPT points, contiguous in the blocked layout) are
//     streamed global -> shared with cp.async.bulk (TMA bulk copies) into a
//     3-stage mbarrier pipeline, so HBM reads overlap the table lookups.
//   * Top-K: per query a shared candidate buffer of CAP >= K + 256*PPT keys;
//     a thread appends a candidate only if it beats the query's current K-th
//     best key.  Buffers that could overflow in the next step are compacted
//     (warp bitonic sort, keep K) behind the step barrier.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "pcpqg_internal.hpp"

namespace pcpqg {

namespace {

constexpr int kThreads = 256;
constexpr int kStages = 3;

// ------------------------------------------------------------------ keys
// 64-bit candidate key, larger = better:
//   [63:32] order-preserving image of the score (-0 canonicalised to +0, so
//           -0 and +0 compare equal as floats do in the reference comparator)
//   [31:1]  0x7FFFFFFF - id  (equal scores -> lower id first)
//   [0]     1 iff the score is -0.0 (restores the exact bits on decode)
// Key 0 is "empty" and sorts below every real key.
__device__ __forceinline__ uint32_t ord_of(float s) {
  uint32_t b = __float_as_uint(s);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t make_key(float s, uint32_t id) {
  const uint64_t negz = (__float_as_uint(s) == 0x80000000u) ? 1ull : 0ull;
  return (static_cast<uint64_t>(ord_of(s)) << 32) |
         (static_cast<uint64_t>(0x7FFFFFFFu - id) << 1) | negz;
}
__device__ __forceinline__ float key_score(uint64_t key) {
  if (key == 0ull) return -INFINITY;
  if (key & 1ull) return -0.0f;
  const uint32_t o = static_cast<uint32_t>(key >> 32);
  const uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ int32_t key_id(uint64_t key) {
  if (key == 0ull) return -1;
  return static_cast<int32_t>(0x7FFFFFFFu - static_cast<uint32_t>((key >> 1) & 0x7FFFFFFFu));
}

// ------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
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

// ----------------------------------------------------------- K1: LUT
// One thread per (query, section, center).  Grouped layout (scan input):
// eta[g*gstride + (j*k + c)*rs + qi] for sections j < m8 = m rounded up to 8;
// sections j >= m get -0.0f so the scan's branch-free octets add exactly -0.
// Plain layout (parity API): eta[q*m*k + j*k + c] for j < m.
__global__ void lut_kernel(const float* __restrict__ Q, uint32_t B, uint64_t total, uint32_t d,
                           const float* __restrict__ cb, uint32_t m, uint32_t msec, uint32_t k,
                           uint32_t dbar, int nq, int rs, uint64_t gstride, int grouped,
                           float* __restrict__ eta) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const uint32_t c = static_cast<uint32_t>(t % k);
  const uint32_t j = static_cast<uint32_t>((t / k) % msec);
  const uint64_t q = t / (static_cast<uint64_t>(k) * msec);
  float acc = 0.0f;  // fixed-order fp32 accumulation from 0.0f (pq_index.cpp:186-190)
  if (j >= m) {
    acc = -0.0f;
  } else if (q < B) {
    const float* row = cb + (static_cast<uint64_t>(j) * k + c) * dbar;
    const float* qq = Q + q * d;
    for (uint32_t a = 0; a < dbar; ++a) {
      const uint32_t col = j * dbar + a;
      const float qa = col < d ? __ldg(qq + col) : 0.0f;  // pad_vector (types.cpp:83-88)
      acc = __fadd_rn(acc, __fmul_rn(__ldg(row + a), qa));
    }
  }
  if (grouped) {
    const uint64_t g = q / nq, qi = q % nq;
    eta[g * gstride + (static_cast<uint64_t>(j) * k + c) * rs + qi] = acc;
  } else {
    eta[q * m * k + static_cast<uint64_t>(j) * k + c] = acc;
  }
}

__global__ void eta_lambda_kernel(const float* __restrict__ eta, const float* __restrict__ lam,
                                  uint64_t total, uint32_t m, uint32_t k, uint32_t s,
                                  float* __restrict__ out) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const uint32_t l = static_cast<uint32_t>(t % s);
  const uint64_t jc = t / s;  // = q*m*k + j*k + c
  const uint32_t j = static_cast<uint32_t>((jc / k) % m);
  out[t] = __fmul_rn(eta[jc], lam[static_cast<uint64_t>(j) * s + l]);  // pq_index.cpp:203
}

// ------------------------------------------------------ K2: scan + top-K
struct ScanArgs {
  const uint32_t* codes;  // [n_blocks][W][32]
  const float* eta;       // grouped tables [G][m8*k rows][RS] (group stride gstride)
  const float* lam;       // [m8][s], pad sections 1.0
  uint64_t* partial;      // [ctas_x][Bpad][K]
  uint64_t* gtau;         // [Bpad] best known K-th key per query (shared across CTAs)
  float* scores;          // score_all mode: [B][n_local]
  uint64_t n_local;
  uint32_t n_blocks, W, Wc, m, m8, k, s, cbits;
  uint32_t B, Bpad, K, cap, ppt, stages;
  uint64_t gstride;       // floats per group table (multiple of 4)
  uint64_t id_base;
};

// Row stride (floats) of the shared eta table: rows are read with LDS.64
// (query pairs), so RS is even with RS/2 odd; then 16 lanes with 16 different
// center codes c of the same section hit 16 distinct bank pairs (k <= 16).
__host__ __device__ constexpr int rs_of(int nq) {
  return nq == 1 ? 1 : (((nq / 2) & 1) ? nq : nq + 2);
}

template <int CW, int SW>
struct Codec {
  static constexpr int kCenterWords = CW == 0 ? 2 : CW / 4;  // words per octet
  static constexpr int kScaleWords = CW == 0 ? 0 : SW / 4;   // words per octet
  static constexpr bool kRaw = SW >= 16;                     // alpha in the stream
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
// of every scan kernel for FFMA/FFMA2).
__device__ __forceinline__ uint64_t fmul2_rn(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Thread group that compacts candidate buffers: `size` threads (a multiple of
// 32), synchronised by __syncwarp or a named barrier.
struct Group {
  int id, size, gtid;
  __device__ __forceinline__ void sync() const {
    if (size == 32)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(size) : "memory");
  }
};

// Histogram bins are padded by one word every 8 so that the digit scan below
// (lane l reads bins 255-8l .. 255-8l-7) touches 32 distinct banks.
__device__ __forceinline__ uint32_t hidx(uint32_t b) { return b + (b >> 3); }
constexpr int kHistWords = 288;  // 256 bins + 32 pad

// Exact K-th largest of buf[0, n) (keys are unique), MSB-first radix select
// with 8-bit digits over the group.  hist: kHistWords counters, sv: 2 words.
template <class Get>
__device__ uint64_t group_select_by(Get get, uint32_t n, uint32_t K, uint32_t* hist, uint32_t* sv,
                                    const Group& g) {
  uint64_t prefix = 0ull, mask = 0ull;
  uint32_t need = K;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = g.gtid; i < kHistWords; i += g.size) hist[i] = 0u;
    g.sync();
    // keys concentrate in a few top-byte bins: aggregate equal digits per
    // warp (__match_any_sync) so each bin gets one atomic per warp
    for (uint32_t i0 = 0; i0 < n; i0 += g.size) {
      const uint32_t i = i0 + g.gtid;
      const uint64_t key = i < n ? get(i) : 0ull;
      const bool ok = i < n && (key & mask) == prefix;
      const uint32_t digit = ok ? (static_cast<uint32_t>(key >> shift) & 0xFFu) : 0x100u;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, digit);
      if (ok && (g.gtid & 31) == __ffs(peers) - 1) atomicAdd(&hist[hidx(digit)], __popc(peers));
    }
    g.sync();
    if (g.gtid < 32) {
      const int lane = g.gtid;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        c[t] = hist[hidx(255 - 8 * lane - t)];
        tot += c[t];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const uint32_t above = incl - tot;
      if (above < need && need <= incl) {
        uint32_t acc = above;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (need <= acc + c[t]) {
            sv[0] = 255u - 8u * lane - t;
            sv[1] = need - acc;
            break;
          }
          acc += c[t];
        }
      }
    }
    g.sync();
    prefix |= static_cast<uint64_t>(sv[0]) << shift;
    mask |= 0xFFull << shift;
    need = sv[1];
  }
  return prefix;
}

__device__ __forceinline__ uint64_t group_select(const uint64_t* buf, uint32_t n, uint32_t K,
                                                 uint32_t* hist, uint32_t* sv, const Group& g) {
  return group_select_by([buf](uint32_t i) { return buf[i]; }, n, K, hist, sv, g);
}

// Order-preserving in-place compaction of buf[0, n) to the keys >= tau.
// Destinations never exceed sources and each chunk is fully read before it
// is written, so no key is overwritten before it is moved.
__device__ uint32_t group_compact(uint64_t* buf, uint32_t n, uint64_t tau, uint32_t* wsum,
                                  const Group& g) {
  const int lane = g.gtid & 31, w = g.gtid >> 5, nw = g.size >> 5;
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += g.size) {
    const uint32_t i = c0 + g.gtid;
    const uint64_t key = i < n ? buf[i] : 0ull;
    const bool keep = i < n && key >= tau;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
    uint32_t rank = __popc(bal & ((1u << lane) - 1u)), total = __popc(bal);
    if (nw > 1) {
      if (lane == 0) wsum[w] = total;
      g.sync();
      uint32_t before = 0;
      total = 0;
      for (int t = 0; t < nw; ++t) {
        const uint32_t v = wsum[t];
        before += t < w ? v : 0u;
        total += v;
      }
      rank += before;
      g.sync();
    } else {
      __syncwarp();
    }
    if (keep) buf[base + rank] = key;
    base += total;
  }
  g.sync();
  return base;
}

// Scores one point for NQ queries: the sections [0, m) in order, 8 per octet.
// Full octets are branch-free; the last, partial octet (m % 8 sections) is
// guarded by a uniform predicate.
// KT != 0 fixes k (and, for JOINT8, cbits = log2 KT) at compile time so row
// offsets become immediates; KT == 0 reads k / cbits at run time.
template <int NQ, int CW, int SW, int KT>
__device__ __forceinline__ void score_point(const uint32_t* wp, const float* s_eta,
                                            const float* s_lam, uint32_t k_rt, uint32_t s,
                                            uint32_t cbits_rt, uint32_t W, uint32_t Wc, uint32_t m,
                                            float (&acc)[NQ]) {
  const uint32_t k = KT ? static_cast<uint32_t>(KT) : k_rt;
  const uint32_t cbits = KT ? static_cast<uint32_t>(__builtin_ctz(KT)) : cbits_rt;
  using Cd = Codec<CW, SW>;
  constexpr int RS = rs_of(NQ);
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = -0.0f;  // identity of RN addition
  const uint32_t noct = (m + 7) >> 3;
  for (uint32_t o = 0; o < noct; ++o) {
    const uint32_t nsec = min(8u, m - o * 8);  // 8 except in the last octet
    uint32_t cwd[Cd::kCenterWords];
    uint32_t swd[Cd::kScaleWords > 0 ? Cd::kScaleWords : 1];
    const uint32_t cbase = o * Cd::kCenterWords;
#pragma unroll
    for (int i = 0; i < Cd::kCenterWords; ++i)
      cwd[i] = (cbase + i < (CW == 0 ? W : Wc)) ? wp[(cbase + i) * kBlockPts] : 0u;
    if constexpr (Cd::kScaleWords > 0) {
      const uint32_t sbase = Wc + o * Cd::kScaleWords;
#pragma unroll
      for (int i = 0; i < Cd::kScaleWords; ++i)
        swd[i] = (sbase + i < W) ? wp[(sbase + i) * kBlockPts] : 0u;
    }
    const float* eta_o = s_eta + static_cast<size_t>(o) * 8 * k * RS;
    const float* lam_o = s_lam + o * 8 * s;
    auto section = [&](int b) {
      uint32_t c;
      float alpha;
      if constexpr (CW == 0) {
        const uint32_t byte = (cwd[b >> 2] >> (8 * (b & 3))) & 0xFFu;
        c = byte & ((1u << cbits) - 1u);
        alpha = lam_o[b * s + (byte >> cbits)];
      } else {
        if constexpr (CW == 4) c = (cwd[0] >> (4 * b)) & 0xFu;
        else if constexpr (CW == 8) c = (cwd[b >> 2] >> (8 * (b & 3))) & 0xFFu;
        else c = (cwd[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
        if constexpr (SW == 0) {
          alpha = lam_o[b];
        } else if constexpr (SW == 4) {
          alpha = lam_o[b * s + ((swd[0] >> (4 * b)) & 0xFu)];
        } else if constexpr (SW == 8) {
          alpha = lam_o[b * s + ((swd[b >> 2] >> (8 * (b & 3))) & 0xFFu)];
        } else if constexpr (SW == 16) {
          alpha = __half2float(__ushort_as_half(
              static_cast<unsigned short>((swd[b >> 1] >> (16 * (b & 1))) & 0xFFFFu)));
        } else {
          alpha = __uint_as_float(swd[b]);
        }
      }
      const float* row = eta_o + (b * k + c) * RS;
      if constexpr (NQ == 1) {
        acc[0] = __fadd_rn(acc[0], __fmul_rn(row[0], alpha));
      } else {
        const uint64_t a2 = pack2(alpha, alpha);
#pragma unroll
        for (int q2 = 0; q2 < NQ / 2; ++q2) {
          const uint64_t e2 = *reinterpret_cast<const uint64_t*>(row + 2 * q2);
          float tx, ty;
          unpack2(fmul2_rn(e2, a2), tx, ty);
          acc[2 * q2] = __fadd_rn(acc[2 * q2], tx);
          acc[2 * q2 + 1] = __fadd_rn(acc[2 * q2 + 1], ty);
        }
      }
    };
    if (nsec == 8) {
#pragma unroll
      for (int b = 0; b < 8; ++b) section(b);
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b < static_cast<int>(nsec)) section(b);
    }
  }
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
                                               uint32_t* s_flag, uint32_t cap, uint32_t reserve) {
  uint32_t pend = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (((want >> q) & 1u) && acc[q] >= tauf[q]) {
      const uint64_t key = make_key(acc[q], id);
      if (key > s_tau[q]) {
        const uint32_t slot = atomicAdd(&s_cnt[q], 1u);
        if (slot < cap) {
          s_buf[q * cap + slot] = key;
          if (slot + 1 > cap - reserve) atomicOr(s_flag, 1u);
        } else {
          pend |= 1u << q;
          atomicOr(s_flag, 2u);
        }
      }
    }
  }
  return pend;
}

template <int NQ, int CW, int SW, int KT>
__global__ void __launch_bounds__(512)
    scan_topk_kernel(const ScanArgs a) {
  using Cd = Codec<CW, SW>;
  constexpr int RS = rs_of(NQ);
  extern __shared__ __align__(128) uint8_t smem[];

  const uint32_t k = a.k, s = a.s, W = a.W;
  const int nthr = blockDim.x;
  const uint32_t g = blockIdx.x;  // query group
  const uint32_t nq_valid = min(static_cast<uint32_t>(NQ), a.B - g * NQ);
  const uint32_t want_all = nq_valid >= 32 ? 0xFFFFFFFFu : ((1u << nq_valid) - 1u);
  const bool topk = a.scores == nullptr;

  // ---- shared memory carve-up (every region 16-byte aligned):
  //  [code tiles x stages][candidates NQ*cap][eta m8*k*RS][lambda m8*s][hist][header]
  const uint32_t tile_pts = nthr * a.ppt;
  const uint32_t tile_words = tile_pts * W;
  const int ngroups = min(NQ, nthr / 32);
  uint8_t* ptr = smem;
  uint32_t* s_tile = reinterpret_cast<uint32_t*>(ptr);
  ptr += static_cast<size_t>(a.stages) * tile_words * 4;
  uint64_t* s_buf = reinterpret_cast<uint64_t*>(ptr);
  ptr += topk ? static_cast<size_t>(NQ) * a.cap * 8 : 0;
  float* s_eta = reinterpret_cast<float*>(ptr);
  ptr += (static_cast<size_t>(a.m8) * k * RS * 4 + 15) & ~static_cast<size_t>(15);
  float* s_lam = reinterpret_cast<float*>(ptr);
  ptr += Cd::kRaw ? 0 : ((a.m8 * s * 4 + 15u) & ~15u);
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(ptr);  // ngroups x (hist + 2 sv + 14 wsum)
  ptr += topk ? static_cast<size_t>(ngroups) * (kHistWords + 16) * 4 : 0;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(ptr);        // up to 4 mbarriers
  uint64_t* s_tau = reinterpret_cast<uint64_t*>(ptr + 32);   // 16 x u64
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(ptr + 160);  // 16 x u32
  uint32_t* s_flag = reinterpret_cast<uint32_t*>(ptr + 224);

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
    fence_mbar_init();
    *s_flag = 0;
  }
  {
    const float4* src = reinterpret_cast<const float4*>(a.eta + static_cast<size_t>(g) * a.gstride);
    float4* dst = reinterpret_cast<float4*>(s_eta);
    const uint32_t n4 = (a.m8 * k * RS + 3) / 4;
    for (uint32_t i = tid; i < n4; i += nthr) dst[i] = __ldg(src + i);
    if constexpr (!Cd::kRaw)
      for (uint32_t i = tid; i < a.m8 * s; i += nthr) s_lam[i] = __ldg(a.lam + i);
  }
  if (topk && tid < NQ) {
    s_tau[tid] = 0ull;
    s_cnt[tid] = 0u;
  }
  __syncthreads();

  auto issue_tile = [&](uint32_t t) {
    const uint32_t blk = b0 + t * tile_blocks;
    const uint32_t nb = min(tile_blocks, b1 - blk);
    const uint32_t bytes = nb * W * kBlockPts * 4;
    uint64_t* bar = &s_bar[t % a.stages];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(s_tile + static_cast<size_t>(t % a.stages) * tile_words,
             a.codes + static_cast<size_t>(blk) * W * kBlockPts, bytes, bar);
  };
  if (tid == 0)
    for (uint32_t t = 0; t < min(ntiles, a.stages - 1); ++t) issue_tile(t);

  // flush: compact every buffer at or over cap - reserve to its K best keys,
  // publish the new K-th key to the other CTAs of this query group
  auto flush = [&]() {
    const int gsz = nthr / ngroups;
    Group grp{tid / gsz, gsz, tid % gsz};
    uint32_t* hist = s_hist + grp.id * (kHistWords + 16);
    for (uint32_t q = grp.id; q < nq_valid; q += ngroups) {
      const uint32_t cnt = s_cnt[q];
      if (cnt + reserve > a.cap) {
        const uint32_t n = min(cnt, a.cap);
        uint64_t* buf = s_buf + q * a.cap;
        const uint64_t tau = group_select(buf, n, a.K, hist, hist + kHistWords, grp);
        group_compact(buf, n, tau, hist + kHistWords + 2, grp);
        if (grp.gtid == 0) {
          s_cnt[q] = a.K;
          if (tau > s_tau[q]) s_tau[q] = tau;
          atomicMax(reinterpret_cast<unsigned long long*>(a.gtau + g * NQ + q),
                    static_cast<unsigned long long>(tau));
        }
      }
    }
  };

  float tauf[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) tauf[q] = -INFINITY;

  for (uint32_t t = 0; t < ntiles; ++t) {
    if (tid == 0 && t + a.stages - 1 < ntiles) {
      fence_proxy_async();  // WAR: generic-proxy reads of the reused stage precede the async write
      issue_tile(t + a.stages - 1);
    }
    if (topk) {
      // adopt a better K-th key found by another CTA (never lowers tau: a key
      // below any CTA's K-th best cannot reach the global top-K)
      if (tid < static_cast<int>(nq_valid)) {
        const uint64_t gt = __ldcg(reinterpret_cast<const unsigned long long*>(a.gtau + g * NQ + tid));
        if (gt > s_tau[tid]) s_tau[tid] = gt;
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
    }
    mbar_wait(&s_bar[t % a.stages], (t / a.stages) & 1u);
    const uint32_t* tile = s_tile + static_cast<size_t>(t % a.stages) * tile_words;
    const uint32_t tile_p0 = (b0 + t * tile_blocks) * kBlockPts;

    float acc[NQ];
    uint32_t pend = 0, id = 0;
    for (uint32_t r = 0; r < a.ppt; ++r) {
      const uint32_t lp = r * nthr + tid;                      // point within tile
      const uint64_t p = static_cast<uint64_t>(tile_p0) + lp;  // local point id
      const bool valid = p < p_end;  // inside this CTA's blocks and the shard
      const uint32_t* wp = tile + (lp >> 5) * W * kBlockPts + (lp & 31);
      score_point<NQ, CW, SW, KT>(wp, s_eta, s_lam, k, s, a.cbits, W, a.Wc, a.m, acc);
      if (!topk) {
        if (valid) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < static_cast<int>(nq_valid))
              a.scores[static_cast<size_t>(g * NQ + q) * a.n_local + p] = acc[q];
        }
        continue;
      }
      if (valid) {
        id = static_cast<uint32_t>(a.id_base + p);
        pend = try_insert<NQ>(acc, want_all, id, tauf, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve);
      }
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
        if (pend) pend = try_insert<NQ>(acc, pend, id, tauf, s_buf, s_tau, s_cnt, s_flag, a.cap, reserve);
        __syncthreads();
        fl = *s_flag;
      }
    }
  }

  if (!topk) return;
  // ---- final: reduce every query's buffer to (at most) its K best keys
  {
    const int gsz = nthr / ngroups;
    Group grp{tid / gsz, gsz, tid % gsz};
    uint32_t* hist = s_hist + grp.id * (kHistWords + 16);
    for (uint32_t q = grp.id; q < NQ; q += ngroups) {
      uint64_t* buf = s_buf + q * a.cap;
      uint32_t n = q < nq_valid ? min(s_cnt[q], a.cap) : 0u;
      if (n > a.K) {
        const uint64_t tau = group_select(buf, n, a.K, hist, hist + kHistWords, grp);
        n = group_compact(buf, n, tau, hist + kHistWords + 2, grp);
        if (grp.gtid == 0)
          atomicMax(reinterpret_cast<unsigned long long*>(a.gtau + g * NQ + q),
                    static_cast<unsigned long long>(tau));
      }
      uint64_t* out = a.partial + (static_cast<size_t>(cx) * a.Bpad + g * NQ + q) * a.K;
      for (uint32_t i = grp.gtid; i < a.K; i += grp.size) out[i] = i < n ? buf[i] : 0ull;
    }
  }
}

// ------------------------------------------------------------- K3: merge
// One CTA per query b merges L lists of Kin keys (layout [L][in_rows][Kin]).
// gtau[b] (optional) is a lower bound on the query's final K-th key — the
// best K-th key any scan CTA saw — so keys below it are dropped on load.  The
// survivors are gathered into shared memory (capacity `cap`), cut to the best
// Kout by radix select, sorted (bitonic over <= pow2(Kout) keys) and written
// as rows of out_stride keys (ranks >= Kout empty: id -1, score -inf).  Only
// if more than `cap` keys survive is the K-th key selected from the lists in
// global memory first.
constexpr uint32_t kMergeMaxCap = 24576;  // 192 KB of keys

__global__ void __launch_bounds__(512)
    merge_kernel(const uint64_t* __restrict__ in, uint32_t L, uint32_t in_rows, uint32_t Kin,
                 uint32_t Kout, uint32_t out_stride, const uint64_t* __restrict__ gtau,
                 uint32_t cap, uint64_t* __restrict__ out, int32_t* __restrict__ ids,
                 float* __restrict__ scores) {
  extern __shared__ uint64_t sk[];
  __shared__ uint32_t hist[kHistWords + 16];
  __shared__ uint32_t s_n;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const Group grp{0, static_cast<int>(nthr), static_cast<int>(tid)};
  uint64_t thr = 1ull;  // drops empty keys
  if (gtau) thr = max(thr, static_cast<uint64_t>(gtau[b]));
  const uint32_t total = L * Kin;
  auto fetch = [&](uint32_t i) -> uint64_t {
    const uint32_t l = i / Kin, r = i - l * Kin;
    const uint64_t key = in[(static_cast<size_t>(l) * in_rows + b) * Kin + r];
    return key >= thr ? key : 0ull;
  };
  // gather survivors (warp-aggregated slot allocation, 4 loads in flight)
  auto gather = [&]() {
    for (uint32_t i0 = 0; i0 < total; i0 += 4 * nthr) {
      uint64_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * nthr + tid;
        v[u] = i < total ? fetch(i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v[u] != 0ull);
        uint32_t base = 0;
        if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, static_cast<uint32_t>(__popc(bal)));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        const uint32_t slot = base + __popc(bal & ((1u << (tid & 31)) - 1u));
        if (v[u] && slot < cap) sk[slot] = v[u];
      }
    }
  };
  if (tid == 0) s_n = 0;
  __syncthreads();
  gather();
  __syncthreads();
  uint32_t n = s_n;
  if (n > cap) {  // rare: select the Kout-th key over the lists first
    thr = group_select_by(fetch, total, Kout, hist, hist + kHistWords, grp);
    __syncthreads();
    if (tid == 0) s_n = 0;
    __syncthreads();
    gather();  // exactly Kout keys are >= the Kout-th
    __syncthreads();
    n = s_n;
  } else if (n > Kout) {
    const uint64_t tau = group_select(sk, n, Kout, hist, hist + kHistWords, grp);
    n = group_compact(sk, n, tau, hist + kHistWords + 2, grp);
  }
  uint32_t P = 1;
  while (P < n) P <<= 1;
  for (uint32_t i = n + tid; i < P; i += nthr) sk[i] = 0ull;
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < P / 2; i += nthr) {
        const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
        const uint32_t hi = lo + stride;
        const uint64_t x = sk[lo], y = sk[hi];
        const bool desc = (lo & size) == 0;
        if ((x < y) == desc) {
          sk[lo] = y;
          sk[hi] = x;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = tid; i < out_stride; i += nthr) {
    const uint64_t key = (i < Kout && i < n) ? sk[i] : 0ull;
    if (out) out[static_cast<size_t>(b) * out_stride + i] = key;
    if (ids) ids[static_cast<size_t>(b) * out_stride + i] = key_id(key);
    if (scores) scores[static_cast<size_t>(b) * out_stride + i] = key_score(key);
  }
}

using ScanFn = void (*)(ScanArgs);

template <int CW, int SW, int KT = 0>
ScanFn pick_nq(int nq) {
  switch (nq) {
    case 1: return scan_topk_kernel<1, CW, SW, KT>;
    case 2: return scan_topk_kernel<2, CW, SW, KT>;
    case 4: return scan_topk_kernel<4, CW, SW, KT>;
    case 8: return scan_topk_kernel<8, CW, SW, KT>;
    default: return scan_topk_kernel<16, CW, SW, KT>;
  }
}

ScanFn pick_kernel(const DeviceIndex& x, int nq) {
  const bool k16 = x.h.k == 16;
  if (x.format == PCPQG_FMT_JOINT8) return k16 ? pick_nq<0, 0, 16>(nq) : pick_nq<0, 0>(nq);
  if (k16 && x.cw == 4 && x.sw == 16) return pick_nq<4, 16, 16>(nq);
  if (k16 && x.cw == 4 && x.sw == 32) return pick_nq<4, 32, 16>(nq);
  if (k16 && x.cw == 4 && x.sw == 8) return pick_nq<4, 8, 16>(nq);
#define PCPQG_CASE(CW_, SW_) \
  if (x.cw == CW_ && x.sw == SW_) return pick_nq<CW_, SW_>(nq);
  PCPQG_CASE(4, 4) PCPQG_CASE(4, 8) PCPQG_CASE(4, 16) PCPQG_CASE(4, 32)
  PCPQG_CASE(8, 0) PCPQG_CASE(8, 4) PCPQG_CASE(8, 8) PCPQG_CASE(8, 16) PCPQG_CASE(8, 32)
  PCPQG_CASE(16, 0) PCPQG_CASE(16, 4) PCPQG_CASE(16, 8) PCPQG_CASE(16, 16) PCPQG_CASE(16, 32)
#undef PCPQG_CASE
  fail(PCPQG_E_UNSUPPORTED, "no scan kernel for this code layout");
}

size_t scan_smem_bytes(const DeviceIndex& x, int nq, uint32_t cap, uint32_t ppt, bool topk,
                       int nthr, int stages) {
  const int rs = rs_of(nq);
  const bool raw = x.format == PCPQG_FMT_PLANES && x.sw >= 16;
  const uint32_t m8 = (x.h.m + 7) & ~7u;
  const int ngroups = std::min(nq, nthr / 32);
  size_t b = static_cast<size_t>(stages) * nthr * ppt * x.W * 4;
  b += topk ? static_cast<size_t>(nq) * cap * 8 : 0;
  b += (static_cast<size_t>(m8) * x.h.k * rs * 4 + 15) & ~static_cast<size_t>(15);
  b += raw ? 0 : ((m8 * std::max(x.h.scales, 1u) * 4 + 15u) & ~15u);
  b += topk ? static_cast<size_t>(ngroups) * (kHistWords + 16) * 4 : 0;
  b += 256;
  return b;
}

int g_max_smem = 0;

}  // namespace

uint64_t group_stride(const DeviceIndex& x, int rs) {
  const uint64_t m8 = (x.h.m + 7) & ~7u;
  return (m8 * x.h.k * rs + 3) & ~static_cast<uint64_t>(3);
}

int num_sms(int device) {
  int v = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

SearchPlan plan_search(const DeviceIndex& x, uint32_t B, uint32_t topn, bool scores_only) {
  int max_smem = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, x.device));
  g_max_smem = max_smem;
  const size_t budget = static_cast<size_t>(max_smem) - 1024;
  const bool topk = !scores_only;
  SearchPlan p;
  p.topn = topn;
  // (threads, points per thread per tile, pipeline stages) in order of preference
  struct Shape { int thr, ppt, stages; };
  static const Shape big[] = {{512, 1, 2}, {256, 1, 3}, {256, 1, 2}, {128, 1, 2}};
  static const Shape small[] = {{512, 2, 2}, {256, 4, 2}, {256, 2, 2}, {256, 1, 2}, {128, 1, 2}};
  int nq = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : 16;
  bool found = false;
  while (!found) {
    const Shape* shapes = nq >= 8 ? big : small;
    const int nshape = nq >= 8 ? 4 : 5;
    for (int i = 0; i < nshape && !found; ++i) {
      const Shape sh = shapes[i];
      // ppt > 1: room for a whole tile of inserts (no overflow possible);
      // ppt == 1: 2K + 64 keys and the rare overflow is retried (see try_insert)
      const uint32_t ins_max = static_cast<uint32_t>(sh.thr * sh.ppt);
      // (ppt > 1 also keeps a tile of slack so a flush is needed only after
      // another tile's worth of inserts, not after every insert)
      const uint32_t cap = !topk ? 0 : sh.ppt > 1 ? ((topn + 2 * ins_max + 1) & ~1u) : ((2 * topn + 64 + 1) & ~1u);
      const size_t sm = scan_smem_bytes(x, nq, cap, sh.ppt, topk, sh.thr, sh.stages);
      if (sm <= budget) {
        p.nq = nq;
        p.rs = rs_of(nq);
        p.cap = cap;
        p.smem = sm;
        p.threads = sh.thr;
        p.ppt = sh.ppt;
        p.stages = sh.stages;
        found = true;
      }
    }
    if (!found) {
      if (nq == 1) fail(PCPQG_E_UNSUPPORTED, "search configuration does not fit in shared memory");
      nq >>= 1;
    }
  }
  p.groups = (B + p.nq - 1) / p.nq;
  ScanFn fn = pick_kernel(x, p.nq);
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(p.smem)));
  int occ = 0;
  PCPQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn),
                                                           p.threads, p.smem));
  occ = std::max(occ, 1);
  const uint64_t slots = static_cast<uint64_t>(num_sms(x.device)) * occ;
  const uint32_t tile_blocks = p.threads * p.ppt / kBlockPts;
  // CTAs per group along the points: every CTA gets at least one full tile;
  // pick the count that makes the last wave as full as possible.
  uint32_t cmax = std::max<uint32_t>(1, x.n_blocks / tile_blocks);
  if (!scores_only) cmax = std::min<uint32_t>(cmax, 4096);
  uint32_t best_cx = 1;
  double best_eff = -1.0;
  const uint32_t lim = static_cast<uint32_t>(std::min<uint64_t>(cmax, std::max<uint64_t>(1, 4 * slots)));
  for (uint32_t cx = 1; cx <= lim; ++cx) {
    const uint64_t ctas = static_cast<uint64_t>(p.groups) * cx;
    const uint64_t waves = (ctas + slots - 1) / slots;
    const double eff = static_cast<double>(ctas) / static_cast<double>(waves * slots);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best_cx = cx;
    }
    if (eff > 0.999) break;
  }
  p.ctas_x = best_cx;
  return p;
}

void launch_lut(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t Bpad, int nq, int rs,
                bool grouped, float* eta, cudaStream_t st) {
  const uint32_t msec = grouped ? ((x.h.m + 7) & ~7u) : x.h.m;
  const uint64_t total = static_cast<uint64_t>(Bpad) * msec * x.h.k;
  if (total == 0) return;
  const uint32_t threads = 256;
  const uint64_t blocks = (total + threads - 1) / threads;
  lut_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
      dQ, B, total, x.h.d, x.d_codebooks, x.h.m, msec, x.h.k, x.h.dbar, nq, rs,
      group_stride(x, rs), grouped ? 1 : 0, eta);
  PCPQG_CUDA(cudaGetLastError());
}

void launch_eta_lambda(const DeviceIndex& x, const float* eta_plain, uint32_t B, float* etal,
                       cudaStream_t st) {
  const uint64_t total = static_cast<uint64_t>(B) * x.h.m * x.h.k * x.h.scales;
  if (total == 0) return;
  eta_lambda_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      eta_plain, x.d_lambda, total, x.h.m, x.h.k, x.h.scales, etal);
  PCPQG_CUDA(cudaGetLastError());
}

void launch_scan(const DeviceIndex& x, const SearchPlan& p, const float* eta_grouped, uint32_t B,
                 uint64_t* partial, uint64_t* gtau, float* scores, cudaStream_t st) {
  ScanArgs a{};
  a.codes = x.d_codes;
  a.eta = eta_grouped;
  a.lam = x.d_lambda;
  a.partial = partial;
  a.gtau = gtau;
  a.scores = scores;
  a.n_local = x.n_local;
  a.n_blocks = x.n_blocks;
  a.W = x.W;
  a.Wc = x.Wc;
  a.m = x.h.m;
  a.m8 = (x.h.m + 7) & ~7u;
  a.k = x.h.k;
  a.s = std::max(x.h.scales, 1u);
  a.cbits = x.format == PCPQG_FMT_JOINT8 ? x.cw : 0;
  a.B = B;
  a.Bpad = p.groups * p.nq;
  a.K = p.topn;
  a.cap = p.cap;
  a.ppt = p.ppt;
  a.stages = p.stages;
  a.gstride = group_stride(x, p.rs);
  a.id_base = x.shard_begin;
  ScanFn fn = pick_kernel(x, p.nq);
  dim3 grid(p.groups, p.ctas_x);
  fn<<<grid, p.threads, p.smem, st>>>(a);
  PCPQG_CUDA(cudaGetLastError());
}

void merge_lists(const uint64_t* keys, uint32_t L, uint32_t in_rows, uint32_t B, uint32_t K,
                 uint32_t out_stride, const uint64_t* gtau, uint64_t* keys_out, int32_t* ids,
                 float* scores, cudaStream_t st) {
  if (B == 0 || L == 0) return;
  if (K == 0 || K > 4096) fail(PCPQG_E_UNSUPPORTED, "topn outside the merge limits (1..4096)");
  uint32_t p2 = 1;
  while (p2 < K) p2 <<= 1;
  const uint32_t cap = std::max<uint32_t>(std::min<uint64_t>(static_cast<uint64_t>(L) * K, kMergeMaxCap), p2);
  static bool attr_set[64] = {};  // per device; racing threads set the same value
  int dev = 0;
  PCPQG_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    PCPQG_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kMergeMaxCap * 8)));
    attr_set[dev] = true;
  }
  const int thr = B < 1024 ? 512 : 256;  // few queries: more threads per query
  merge_kernel<<<B, thr, cap * 8, st>>>(keys, L, in_rows, K, std::min(K, out_stride), out_stride,
                                        gtau, cap, keys_out, ids, scores);
  PCPQG_CUDA(cudaGetLastError());
}

}  // namespace pcpqg
