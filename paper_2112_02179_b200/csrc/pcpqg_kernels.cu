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
constexpr uint32_t kMergeMaxKeys = 8192;

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
__global__ void lut_kernel(const float* __restrict__ Q, uint32_t B, uint64_t total, uint32_t d,
                           const float* __restrict__ cb, uint32_t m, uint32_t k, uint32_t dbar,
                           int nq, int rs, uint64_t gstride, int grouped, float* __restrict__ eta) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const uint32_t c = static_cast<uint32_t>(t % k);
  const uint32_t j = static_cast<uint32_t>((t / k) % m);
  const uint64_t q = t / (static_cast<uint64_t>(k) * m);
  float acc = 0.0f;  // fixed-order fp32 accumulation from 0.0f (pq_index.cpp:186-190)
  if (q < B) {
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
  const float* eta;       // grouped tables
  const float* lam;       // [m][s]
  uint64_t* partial;      // [ctas_x][Bpad][K]
  float* scores;          // score_all mode: [B][n_local]
  uint64_t n_local;
  uint32_t n_blocks, W, Wc, m, k, s, cbits;
  uint32_t B, Bpad, K, cap, ppt;
  uint64_t gstride;       // floats per group table (multiple of 4)
  uint64_t id_base;
};

// Decode of one octet of sections (8 sections) from the staged words.
// CW == 0 selects JOINT8 (byte = c | l << cbits); otherwise PLANES with
// compile-time center width CW and scale width SW.
template <int CW, int SW>
struct Codec {
  static constexpr int kCenterWords = CW == 0 ? 2 : CW / 4;       // words per octet
  static constexpr int kScaleWords = CW == 0 ? 0 : SW / 4;        // words per octet
  static constexpr bool kRaw = SW >= 16;                          // alpha in the stream
};

template <int NQ, int CW, int SW>
__global__ void __launch_bounds__(kThreads)
    scan_topk_kernel(const ScanArgs a) {
  using Cd = Codec<CW, SW>;
  constexpr int RS = NQ | 1;
  extern __shared__ __align__(128) uint8_t smem[];

  const uint32_t m = a.m, k = a.k, s = a.s, W = a.W;
  const uint32_t g = blockIdx.x;                // query group
  const uint32_t nq_valid = min(static_cast<uint32_t>(NQ), a.B - g * NQ);
  const bool topk = a.scores == nullptr;

  // ---- shared memory carve-up (every region 16-byte aligned):
  //      [code tiles x kStages][candidate keys NQ*cap][eta m*k*RS][lambda][header]
  const uint32_t tile_pts = kThreads * a.ppt;
  const uint32_t tile_words = tile_pts * W;
  uint8_t* ptr = smem;
  uint32_t* s_tile = reinterpret_cast<uint32_t*>(ptr);
  ptr += static_cast<size_t>(kStages) * tile_words * 4;
  uint64_t* s_buf = reinterpret_cast<uint64_t*>(ptr);
  ptr += topk ? static_cast<size_t>(NQ) * a.cap * 8 : 0;
  float* s_eta = reinterpret_cast<float*>(ptr);
  ptr += (static_cast<size_t>(m) * k * RS * 4 + 15) & ~static_cast<size_t>(15);
  float* s_lam = reinterpret_cast<float*>(ptr);
  ptr += ((m * (Cd::kRaw ? 1u : s) * 4 + 15u) & ~15u);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(ptr);   // kStages mbarriers (32 B)
  uint64_t* s_tau = reinterpret_cast<uint64_t*>(ptr + 32);   // 16 x u64
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(ptr + 160);  // 16 x u32
  uint32_t* s_flag = reinterpret_cast<uint32_t*>(ptr + 224);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t ins_max = tile_pts;

  // ---- point range of this CTA: blocks [b0, b1)
  const uint32_t cx = blockIdx.y, ncx = gridDim.y;
  const uint32_t b0 = static_cast<uint32_t>((static_cast<uint64_t>(a.n_blocks) * cx) / ncx);
  const uint32_t b1 = static_cast<uint32_t>((static_cast<uint64_t>(a.n_blocks) * (cx + 1)) / ncx);
  const uint32_t tile_blocks = tile_pts / kBlockPts;
  const uint32_t ntiles = (b1 - b0 + tile_blocks - 1) / tile_blocks;
  const uint64_t p_end = min(a.n_local, static_cast<uint64_t>(b1) * kBlockPts);

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&s_bar[i], 1);
    fence_mbar_init();
    *s_flag = 0;
  }
  // tables: eta of this group (m*k rows of RS floats) and the scale codebook
  {
    const float4* src = reinterpret_cast<const float4*>(a.eta + static_cast<size_t>(g) * a.gstride);
    float4* dst = reinterpret_cast<float4*>(s_eta);
    const uint32_t n4 = (m * k * RS + 3) / 4;
    for (uint32_t i = tid; i < n4; i += kThreads) dst[i] = __ldg(src + i);
    if constexpr (!Cd::kRaw)
      for (uint32_t i = tid; i < m * s; i += kThreads) s_lam[i] = __ldg(a.lam + i);
  }
  if (topk) {
    for (uint32_t i = tid; i < NQ * a.cap; i += kThreads) s_buf[i] = 0ull;
    if (tid < NQ) {
      s_tau[tid] = 0ull;
      s_cnt[tid] = 0u;
    }
  }
  __syncthreads();

  auto issue_tile = [&](uint32_t t) {
    const uint32_t blk = b0 + t * tile_blocks;
    const uint32_t nb = min(tile_blocks, b1 - blk);
    const uint32_t bytes = nb * W * kBlockPts * 4;
    uint64_t* bar = &s_bar[t % kStages];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(s_tile + static_cast<size_t>(t % kStages) * tile_words,
             a.codes + static_cast<size_t>(blk) * W * kBlockPts, bytes, bar);
  };
  if (tid == 0)
    for (uint32_t t = 0; t < min(ntiles, static_cast<uint32_t>(kStages - 1)); ++t) issue_tile(t);

  float tauf[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) tauf[q] = -INFINITY;

  for (uint32_t t = 0; t < ntiles; ++t) {
    if (tid == 0 && t + kStages - 1 < ntiles) {
      fence_proxy_async();  // WAR: generic-proxy reads of the reused stage precede the async write
      issue_tile(t + kStages - 1);
    }
    mbar_wait(&s_bar[t % kStages], (t / kStages) & 1u);
    const uint32_t* tile = s_tile + static_cast<size_t>(t % kStages) * tile_words;
    const uint32_t tile_p0 = (b0 + t * tile_blocks) * kBlockPts;

    for (uint32_t r = 0; r < a.ppt; ++r) {
      const uint32_t lp = r * kThreads + tid;      // point within tile
      const uint64_t p = static_cast<uint64_t>(tile_p0) + lp;  // local point id
      const bool valid = p < p_end;  // inside this CTA's blocks and the shard
      // word w of this point: tile[(lp/32)*W*32 + w*32 + lane]
      const uint32_t* wp = tile + (lp >> 5) * W * kBlockPts + (lp & 31);

      float acc[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] = -0.0f;

      const uint32_t noct = (m + 7) >> 3;
      for (uint32_t o = 0; o < noct; ++o) {
        uint32_t cwd[Cd::kCenterWords];
        uint32_t swd[Cd::kScaleWords > 0 ? Cd::kScaleWords : 1];
        const uint32_t cbase = o * Cd::kCenterWords;
#pragma unroll
        for (int i = 0; i < Cd::kCenterWords; ++i)
          cwd[i] = (cbase + i < (CW == 0 ? W : a.Wc)) ? wp[(cbase + i) * kBlockPts] : 0u;
        if constexpr (Cd::kScaleWords > 0) {
          const uint32_t sbase = a.Wc + o * Cd::kScaleWords;
#pragma unroll
          for (int i = 0; i < Cd::kScaleWords; ++i)
            swd[i] = (sbase + i < W) ? wp[(sbase + i) * kBlockPts] : 0u;
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const uint32_t j = o * 8 + b;
          if (j >= m) break;
          uint32_t c;
          float alpha;
          if constexpr (CW == 0) {
            const uint32_t byte = (cwd[b >> 2] >> (8 * (b & 3))) & 0xFFu;
            c = byte & ((1u << a.cbits) - 1u);
            alpha = s_lam[j * s + (byte >> a.cbits)];
          } else {
            if constexpr (CW == 4) c = (cwd[0] >> (4 * b)) & 0xFu;
            else if constexpr (CW == 8) c = (cwd[b >> 2] >> (8 * (b & 3))) & 0xFFu;
            else c = (cwd[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
            if constexpr (SW == 0) {
              alpha = s_lam[j];
            } else if constexpr (SW == 4) {
              alpha = s_lam[j * s + ((swd[0] >> (4 * b)) & 0xFu)];
            } else if constexpr (SW == 8) {
              alpha = s_lam[j * s + ((swd[b >> 2] >> (8 * (b & 3))) & 0xFFu)];
            } else if constexpr (SW == 16) {
              alpha = __half2float(__ushort_as_half(
                  static_cast<unsigned short>((swd[b >> 1] >> (16 * (b & 1))) & 0xFFFFu)));
            } else {
              alpha = __uint_as_float(swd[b]);
            }
          }
          const float* row = s_eta + (j * k + c) * RS;
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(row[q], alpha));
        }
      }

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
        const uint32_t id = static_cast<uint32_t>(a.id_base + p);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (q < static_cast<int>(nq_valid) && acc[q] >= tauf[q]) {
            const uint64_t key = make_key(acc[q], id);
            if (key > s_tau[q]) {
              const uint32_t slot = atomicAdd(&s_cnt[q], 1u);
              s_buf[q * a.cap + slot] = key;
              if (slot + 1 > a.cap - ins_max) *s_flag = 1u;
            }
          }
        }
      }
    }
    __syncthreads();  // tile consumed; candidate writes visible
    if (topk && *s_flag) {
      // Compact every buffer that could overflow during the next tile.
      for (uint32_t q = warp; q < nq_valid; q += kThreads / 32) {
        if (s_cnt[q] > a.cap - ins_max) {
          uint64_t* buf = s_buf + q * a.cap;
          const uint32_t P = a.cap;
          for (uint32_t size = 2; size <= P; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
              for (uint32_t i = lane; i < P / 2; i += 32) {
                const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
                const uint32_t hi = lo + stride;
                const uint64_t x = buf[lo], y = buf[hi];
                const bool desc = (lo & size) == 0;
                if ((x < y) == desc) {
                  buf[lo] = y;
                  buf[hi] = x;
                }
              }
              __syncwarp();
            }
          }
          for (uint32_t i = a.K + lane; i < P; i += 32) buf[i] = 0ull;
          if (lane == 0) {
            s_cnt[q] = a.K;
            s_tau[q] = buf[a.K - 1];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (tid == 0) *s_flag = 0u;
#pragma unroll
      for (int q = 0; q < NQ; ++q) tauf[q] = key_score(s_tau[q]);
    }
  }

  if (!topk) return;
  // ---- final: sort every query's buffer, emit the best K keys
  for (uint32_t q = warp; q < NQ; q += kThreads / 32) {
    uint64_t* buf = s_buf + q * a.cap;
    const uint32_t n = min(s_cnt[q], a.cap);
    uint32_t P = 1;
    while (P < n) P <<= 1;
    for (uint32_t size = 2; size <= P; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = lane; i < P / 2; i += 32) {
          const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
          const uint32_t hi = lo + stride;
          const uint64_t x = buf[lo], y = buf[hi];
          const bool desc = (lo & size) == 0;
          if ((x < y) == desc) {
            buf[lo] = y;
            buf[hi] = x;
          }
        }
        __syncwarp();
      }
    }
    uint64_t* out = a.partial + (static_cast<size_t>(cx) * a.Bpad + g * NQ + q) * a.K;
    for (uint32_t i = lane; i < a.K; i += 32) out[i] = (q < nq_valid && i < n) ? buf[i] : 0ull;
  }
}

// ------------------------------------------------------------- K3: merge
// One CTA per (query b, output list).  Loads F input lists of Kin keys
// (input layout [L][in_rows][Kin]), sorts them descending (bitonic, P <= 8192
// keys in shared memory) and writes rows of out_stride keys of which the best
// Kout are real and the rest empty (id -1, score -inf).
__global__ void __launch_bounds__(256)
    merge_kernel(const uint64_t* __restrict__ in, uint32_t L, uint32_t in_rows, uint32_t B,
                 uint32_t Kin, uint32_t Kout, uint32_t F, uint32_t P, uint32_t out_stride,
                 uint64_t* __restrict__ out, int32_t* __restrict__ ids,
                 float* __restrict__ scores) {
  extern __shared__ uint64_t sk[];
  const uint32_t b = blockIdx.x, lo_list = blockIdx.y * F;
  const uint32_t nl = min(F, L - lo_list);
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    uint64_t v = 0ull;
    if (i < nl * Kin) {
      const uint32_t l = lo_list + i / Kin, r = i % Kin;
      v = in[(static_cast<size_t>(l) * in_rows + b) * Kin + r];
    }
    sk[i] = v;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < P / 2; i += blockDim.x) {
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
  for (uint32_t i = threadIdx.x; i < out_stride; i += blockDim.x) {
    const uint64_t key = (i < Kout && i < P) ? sk[i] : 0ull;
    if (out) out[(static_cast<size_t>(blockIdx.y) * B + b) * out_stride + i] = key;
    if (ids) ids[static_cast<size_t>(b) * out_stride + i] = key_id(key);
    if (scores) scores[static_cast<size_t>(b) * out_stride + i] = key_score(key);
  }
}

using ScanFn = void (*)(ScanArgs);

template <int CW, int SW>
ScanFn pick_nq(int nq) {
  switch (nq) {
    case 1: return scan_topk_kernel<1, CW, SW>;
    case 2: return scan_topk_kernel<2, CW, SW>;
    case 4: return scan_topk_kernel<4, CW, SW>;
    case 8: return scan_topk_kernel<8, CW, SW>;
    default: return scan_topk_kernel<16, CW, SW>;
  }
}

ScanFn pick_kernel(const DeviceIndex& x, int nq) {
  if (x.format == PCPQG_FMT_JOINT8) return pick_nq<0, 0>(nq);
#define PCPQG_CASE(CW_, SW_) \
  if (x.cw == CW_ && x.sw == SW_) return pick_nq<CW_, SW_>(nq);
  PCPQG_CASE(4, 4) PCPQG_CASE(4, 8) PCPQG_CASE(4, 16) PCPQG_CASE(4, 32)
  PCPQG_CASE(8, 0) PCPQG_CASE(8, 4) PCPQG_CASE(8, 8) PCPQG_CASE(8, 16) PCPQG_CASE(8, 32)
  PCPQG_CASE(16, 0) PCPQG_CASE(16, 4) PCPQG_CASE(16, 8) PCPQG_CASE(16, 16) PCPQG_CASE(16, 32)
#undef PCPQG_CASE
  fail(PCPQG_E_UNSUPPORTED, "no scan kernel for this code layout");
}

size_t scan_smem_bytes(const DeviceIndex& x, int nq, uint32_t cap, uint32_t ppt, bool topk) {
  const int rs = nq | 1;
  const bool raw = x.format == PCPQG_FMT_PLANES && x.sw >= 16;
  size_t b = static_cast<size_t>(kStages) * kThreads * ppt * x.W * 4;
  b += topk ? static_cast<size_t>(nq) * cap * 8 : 0;
  b += (static_cast<size_t>(x.h.m) * x.h.k * rs * 4 + 15) & ~static_cast<size_t>(15);
  b += (x.h.m * (raw ? 1u : std::max(x.h.scales, 1u)) * 4 + 15u) & ~15u;
  b += 256;
  return b;
}

int g_max_smem = 0;

}  // namespace

uint64_t group_stride(const DeviceIndex& x, int rs) {
  return (static_cast<uint64_t>(x.h.m) * x.h.k * rs + 3) & ~static_cast<uint64_t>(3);
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
  SearchPlan p;
  p.topn = topn;
  int nq = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : 16;
  uint32_t ppt = nq >= 8 ? 1 : (nq >= 4 ? 2 : 4);
  const bool topk = !scores_only;
  for (;;) {
    uint32_t cap = 0;
    if (topk) {
      const uint64_t need = static_cast<uint64_t>(topn) + static_cast<uint64_t>(kThreads) * ppt;
      cap = 64;
      while (cap < need) cap <<= 1;
    }
    const size_t sm = scan_smem_bytes(x, nq, cap, ppt, topk);
    if (sm <= budget) {
      p.nq = nq;
      p.rs = nq | 1;
      p.cap = cap;
      p.smem = sm;
      p.steps_per_sync = ppt;  // reused as points-per-thread
      break;
    }
    if (ppt > 1) {
      ppt >>= 1;
    } else if (nq > 1) {
      nq >>= 1;
    } else {
      fail(PCPQG_E_UNSUPPORTED, "search configuration does not fit in shared memory");
    }
  }
  p.groups = (B + p.nq - 1) / p.nq;
  ScanFn fn = pick_kernel(x, p.nq);
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(p.smem)));
  int occ = 0;
  PCPQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn),
                                                           kThreads, p.smem));
  occ = std::max(occ, 1);
  const uint64_t slots = static_cast<uint64_t>(num_sms(x.device)) * occ;
  const uint32_t tile_blocks = kThreads * p.steps_per_sync / kBlockPts;
  // CTAs per group along the points: as many as keep every CTA busy with at
  // least one full tile, chosen to make the last wave as full as possible.
  uint32_t cmax = std::max<uint32_t>(1, x.n_blocks / tile_blocks);
  if (!scores_only) cmax = std::min<uint32_t>(cmax, 4096);
  uint32_t best_cx = 1;
  double best_eff = -1.0;
  const uint32_t lim = std::min<uint64_t>(cmax, std::max<uint64_t>(1, 4 * slots));
  for (uint32_t cx = 1; cx <= lim; ++cx) {
    const uint64_t ctas = static_cast<uint64_t>(p.groups) * cx;
    const uint64_t waves = (ctas + slots - 1) / slots;
    double eff = static_cast<double>(ctas) / static_cast<double>(waves * slots);
    // prefer fewer waves of bigger CTAs when equally efficient (fewer lists to merge)
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best_cx = cx;
    }
    if (waves == 1 && eff > 0.97) break;
  }
  p.ctas_x = best_cx;
  return p;
}

void launch_lut(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t Bpad, int nq, int rs,
                bool grouped, float* eta, cudaStream_t st) {
  const uint64_t total = static_cast<uint64_t>(Bpad) * x.h.m * x.h.k;
  if (total == 0) return;
  const uint32_t threads = 256;
  const uint64_t blocks = (total + threads - 1) / threads;
  lut_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(dQ, B, total, x.h.d, x.d_codebooks,
                                                              x.h.m, x.h.k, x.h.dbar, nq, rs,
                                                              group_stride(x, rs), grouped ? 1 : 0,
                                                              eta);
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
                 uint64_t* partial, float* scores, cudaStream_t st) {
  ScanArgs a{};
  a.codes = x.d_codes;
  a.eta = eta_grouped;
  a.lam = x.d_lambda;
  a.partial = partial;
  a.scores = scores;
  a.n_local = x.n_local;
  a.n_blocks = x.n_blocks;
  a.W = x.W;
  a.Wc = x.Wc;
  a.m = x.h.m;
  a.k = x.h.k;
  a.s = std::max(x.h.scales, 1u);
  a.cbits = x.format == PCPQG_FMT_JOINT8 ? x.cw : 0;
  a.B = B;
  a.Bpad = p.groups * p.nq;
  a.K = p.topn;
  a.cap = p.cap;
  a.ppt = p.steps_per_sync;
  a.gstride = group_stride(x, p.rs);
  a.id_base = x.shard_begin;
  ScanFn fn = pick_kernel(x, p.nq);
  dim3 grid(p.groups, p.ctas_x);
  fn<<<grid, kThreads, p.smem, st>>>(a);
  PCPQG_CUDA(cudaGetLastError());
}

size_t merge_scratch_elems(uint32_t L, uint32_t B, uint32_t K) {
  const uint32_t F = std::max<uint32_t>(2, kMergeMaxKeys / std::max<uint32_t>(K, 1));
  const uint32_t L1 = (L + F - 1) / F;
  return static_cast<size_t>(2) * std::max<uint32_t>(L1, 1) * B * std::max<uint32_t>(K, 1);
}

void merge_lists(const uint64_t* keys, uint32_t L, uint32_t in_rows, uint32_t B, uint32_t K,
                 uint32_t out_stride, uint64_t* keys_out, int32_t* ids, float* scores,
                 uint64_t* scratch, size_t scratch_elems, cudaStream_t st) {
  if (B == 0 || L == 0) return;
  if (K == 0 || K > kMergeMaxKeys / 2) fail(PCPQG_E_UNSUPPORTED, "topn outside the merge limits");
  static bool attr_set[64] = {};  // per device; racing threads set the same value
  int dev = 0;
  PCPQG_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    PCPQG_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kMergeMaxKeys * 8)));
    attr_set[dev] = true;
  }
  const uint32_t F = std::max<uint32_t>(2, kMergeMaxKeys / K);
  const uint64_t* cur = keys;
  uint32_t curL = L, rows = in_rows;
  int ping = 0;
  while (curL > F) {
    const uint32_t Lout = (curL + F - 1) / F;
    uint64_t* dst = scratch + static_cast<size_t>(ping) * (scratch_elems / 2);
    if (static_cast<size_t>(Lout) * B * K > scratch_elems / 2)
      fail(PCPQG_E_USAGE, "merge scratch too small");
    uint32_t P = 1;
    while (P < F * K) P <<= 1;
    merge_kernel<<<dim3(B, Lout), 256, P * 8, st>>>(cur, curL, rows, B, K, K, F, P, K, dst,
                                                    nullptr, nullptr);
    PCPQG_CUDA(cudaGetLastError());
    cur = dst;
    curL = Lout;
    rows = B;
    ping ^= 1;
  }
  uint32_t P = 1;
  while (P < curL * K) P <<= 1;
  merge_kernel<<<dim3(B, 1), 256, P * 8, st>>>(cur, curL, rows, B, K, std::min(K, out_stride),
                                               curL, P, out_stride, keys_out, ids, scores);
  PCPQG_CUDA(cudaGetLastError());
}

}  // namespace pcpqg
