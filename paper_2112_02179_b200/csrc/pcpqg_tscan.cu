// K2-T — the batch scan as a tensor-core pre-score filter (tcgen05) in front
// of the exact fp32 re-score.
//
// The reference scores a point as a fixed-order fp32 sum of per-section LUT
// terms (score_all, proj/core/src/pq_index.cpp:212-244):
//     score(q, p) = sum_j fl(eta_j[c_pj] * lambda_j[l_pj]),
//     eta_j[c]    = fold_a fl(C_j[c][a] * q[j*dbar + a])     (pq_index.cpp:183-192)
// In exact arithmetic that is a dot product, score = <q, x_p> with the decoded
// point x_p[j*dbar + a] = lambda_{j,l_pj} * C_j[c_pj][a] (raw alpha: alpha_pj).
// So a whole query batch against a tile of points is a GEMM.  K2-T runs it on
// the 5th-generation tensor cores in fp16 (fp32 accumulation in TMEM) and uses
// the result only to decide which (query, point) pairs can reach the top-K;
// every reported score is the exact fp32 chain of the reference, recomputed
// for the surviving pairs, so results stay bit-identical.
//
// Scaling (powers of two, exact): per section tau_j with X_j * tau_j in
// [0.5, 1), X_j = max_l |lambda_j,l| * max_{c,a} |C_j[c][a]|; per query sigma_q
// with max_i |q_i / tau_j(i)| * sigma_q in [0.5, 1).  Operands:
//     x'_i = fp16(fl(lambda * C_j[c][a]) * tau_j)   (|x'| < 1)
//     q'_i = fp16(q_i * sigma_q / tau_j)            (|q'| < 1)
// and sum_i q'_i x'_i approximates sigma_q * score.  The error bound eps_q
// (scaled units; tq_prep_kernel) covers fp16 rounding of both operands (normal
// and subnormal), the fp32 product lambda*C, the tensor core's fp32
// accumulation (taken as 2^-22 of the magnitude sum per addition) and the
// reference's own fp32 roundings, with A_q = sum_j max_l|lambda_j,l| *
// max_c sum_a |q_j,a| |C_j[c][a]| >= sum_i |q_i x_i| for every point.
//
// Pruning.  For every query each CTA keeps the candidates whose approximate
// score reaches its threshold thr_q in a list (global memory).  When a list
// fills, the warp selects its K-th best approximate score t; at least K points
// score >= t - eps exactly, so the final K-th best exact score is >= t - eps and
// every point of the final top-K (ties included) has approximate score
// >= t - 2 eps: thr_q rises to t - 2 eps, and it is shared through gthr[q]
// (atomicMax) with the other CTAs of the query.  tscan_finish_kernel then
// merges a query's lists, keeps the approximate scores >= (K-th best of the
// union) - 2 eps, re-scores those exactly in the reference order and selects
// the top-K by (score desc, id asc).  A query whose operands would leave the
// scaling range, or whose list cannot be pruned below capacity (more than a
// list of points within 2 eps of each other), is scanned exactly in full by
// the finish kernel instead — slower, never wrong.
//
// Kernel shape (one CTA per SM; grid = query tiles x point ranges):
//   warps 0-3   epilogue: warp w drains TMEM lanes 32w.. (its 32 queries) with
//               tcgen05.ld, 32 points per load, compares the chunk's max to
//               the query's threshold, appends the rare passing pairs;
//   warp 4      one thread issues tcgen05.mma.kind::f16 (M = 128 queries,
//               N = points per tile, K = 16) into a double-buffered TMEM
//               accumulator and commits to mbarriers;
//   warps 5-12  decode the next point tile from the blocked code stream into
//               shared memory (UMMA K-major layout, no swizzle), double
//               buffered.  The 128-query operand tile is one TMA bulk copy.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "pcpqg_device.cuh"

namespace pcpqg {

// per-index tables of the tensor scan (built once per index, see tc_tables)
struct TcIndex {
  bool ok = false;
  bool joint = false;
  uint32_t dbar = 0, kpad = 0, msec = 0;  // msec: sections covered by the code words (W*4 or m8)
  uint32_t rows = 0;                      // JOINT8 table rows per section (2^(cbits+lbits))
  float* d_tau = nullptr;                 // [msec] power-of-two section scales
  float* d_lam_max = nullptr;             // [msec] max_l |lambda_j,l| (raw: max |alpha_j|)
  __half* d_jtab = nullptr;               // JOINT8: [msec][rows][dbar] fp16(tau * fl(lambda*C))
  float* d_cprime = nullptr;              // PLANES: [msec][k][dbar] C * tau (exact)
  // decoded point operands, built once (tc_cache): tile-major [tile of cache_tile points][kpad/8][tile][16 B]
  // fp16 — each N-point tile of a slab is one contiguous TMA copy that lands
  // in shared memory in the UMMA K-major layout
  std::mutex cache_mu;
  bool cache_tried = false;
  uint8_t* d_xhat = nullptr;
  uint64_t npad = 0;
  uint32_t cache_tile = 0;  // points per cache tile = the cached kernel's N
  double xnorm_max = 0.0;  // max_p ||x'_p||_2 over the cached fp16 operands (0: unknown)
  ~TcIndex() {
    if (d_xhat) cudaFree(d_xhat);
    if (d_tau) cudaFree(d_tau);
    if (d_lam_max) cudaFree(d_lam_max);
    if (d_jtab) cudaFree(d_jtab);
    if (d_cprime) cudaFree(d_cprime);
  }
};

namespace {

constexpr int kTM = 128;           // queries per CTA (UMMA M = TMEM lanes)
constexpr int kEpiWarps = 8;   // two per TMEM lane quadrant (column halves)
constexpr int kMmaWarp = 8;
constexpr int kProdWarp = 9;
constexpr int kDecWarp0 = 10;
constexpr int kDecWarps = 8;
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kTThreads = (kEpiWarps + 2 + kDecWarps) * 32;  // 576
constexpr int kFinThreads = 256;
constexpr uint32_t kFinCap = 8192;  // finish kernel: keys staged per query

__host__ __device__ constexpr uint32_t umma_idesc_f16(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format = F32
         | (0u << 7)          // a_format = F16
         | (0u << 10)         // b_format = F16
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

// Shared-memory matrix descriptor, K-major, SWIZZLE_NONE: core matrices of
// 8 rows x 16 bytes; LBO = byte step between the two 16-byte K chunks of one
// instruction, SBO = byte step between 8-row groups.  SM100 version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  return d;
}

__device__ __forceinline__ float ord_to_float(uint32_t o) {
  const uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __uint_as_float(r);
}

// mbarrier wait that suspends the warp instead of spinning on try_wait
__device__ __forceinline__ void mbar_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

struct TScanArgs {
  const uint32_t* codes;    // [n_blocks][W][32]
  const uint8_t* qa;        // query operand tiles [Bpad/128][kpad/8][128][16 B]
  const float2* fse;        // [Bpad] (sigma, eps) scaled units; eps = inf: not filtered here
  const __half* jtab;       // JOINT8 decode table
  const float* cprime;      // PLANES C * tau
  const float* lam;         // [m8][s]
  uint64_t* lists;          // [ranges][Bpad][Lc] approximate keys (ord(score) << 32 | point)
  uint32_t* counts;         // [ranges][Bpad]
  uint32_t* gthr;           // [Bpad] shared threshold, ord_of(float) (0 = none)
  uint32_t* ovf;            // [Bpad] 1: list overflow -> exact full scan
  uint64_t n_local;
  uint32_t W, Wc, m, k, s, cbits, cw, sw, kpad, msec, rows, K, Lc, B, Bpad;
  uint32_t tiles_per_range;  // point tiles (of N) per CTA range
  uint32_t cprime_smem;      // 1: C * tau staged in shared memory
  uint32_t lam_smem;         // 1: scale codebooks staged in shared memory (else read through L1)
  // seed pass (mode 1): the points are sblocks blocks spread evenly over the
  // nbfull full blocks; the epilogue writes each block's best approximate
  // score to cmax[q][block] instead of appending candidates
  uint32_t mode, sblocks, nbfull, cm_stride;
  uint32_t exp;  // experiments (option scan_tc_exp): 1 = epilogue only waits and releases, 2 = no appends,
                 // 3 = no operand loads after the first fill, 4 = 1 + 3
  float* cmax;
  // per-query counts of appended candidates in 32 bins of width eps above the
  // seed threshold base[q], shared by every CTA: a bin whose suffix count
  // reaches K lifts the threshold of every range to its lower edge - 2 eps
  uint32_t* bins;      // [Bpad][32]
  const float* base;   // [Bpad] seed threshold (scaled), -inf = none
};

// ---- decode of one (point, 16-byte slab) into 8 fp16 operands
// JOINT8: a slab holds 8/DB sections; the table row of (section, code byte)
// holds the section's DB operands.
template <int DB, int RB>
__device__ __forceinline__ uint4 decode_joint(const uint32_t* wp, uint32_t slab, const __half* stab, uint32_t rows_rt) {
  constexpr int SPS = 8 / DB;  // sections per slab
  const uint32_t rows = RB ? (1u << RB) : rows_rt;
  uint32_t out[4];
  const uint32_t j0 = slab * SPS;
  if constexpr (DB == 2) {
    const uint32_t word = wp[(j0 >> 2) * kBlockPts];
    const uint32_t* t32 = reinterpret_cast<const uint32_t*>(stab) + j0 * rows;
#pragma unroll
    for (int b = 0; b < 4; ++b) out[b] = t32[b * rows + ((word >> (8 * b)) & 0xFFu)];
  } else if constexpr (DB == 4) {
    const uint32_t word = wp[(j0 >> 2) * kBlockPts] >> (8 * (j0 & 3));
    const uint2* t64 = reinterpret_cast<const uint2*>(stab) + j0 * rows;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const uint2 v = t64[b * rows + ((word >> (8 * b)) & 0xFFu)];
      out[2 * b] = v.x;
      out[2 * b + 1] = v.y;
    }
  } else if constexpr (DB == 8) {
    const uint32_t word = wp[(j0 >> 2) * kBlockPts];
    const uint4 v = reinterpret_cast<const uint4*>(stab)[j0 * rows + ((word >> (8 * (j0 & 3))) & 0xFFu)];
    out[0] = v.x, out[1] = v.y, out[2] = v.z, out[3] = v.w;
  } else {  // DB == 1: 8 sections, two code words
    const uint32_t w0 = wp[(j0 >> 2) * kBlockPts];
    const uint32_t w1 = wp[((j0 >> 2) + 1) * kBlockPts];
    const uint16_t* t16 = reinterpret_cast<const uint16_t*>(stab) + j0 * rows;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t wd = b < 2 ? w0 : w1;
      const uint32_t lo = t16[(2 * b) * rows + ((wd >> (16 * (b & 1))) & 0xFFu)];
      const uint32_t hi = t16[(2 * b + 1) * rows + ((wd >> (16 * (b & 1) + 8)) & 0xFFu)];
      out[b] = lo | (hi << 16);
    }
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

// PLANES: center code (cw bits) and scale (sw: 0 -> lambda_j[0], 4/8 -> code,
// 16 -> fp16 alpha, 32 -> fp32 alpha) of section j.  CW / SW = 0: widths
// read at run time; else compile-time (the configs' layouts).
template <int CW, int SW>
__device__ __forceinline__ void planes_cs(const uint32_t* wp, uint32_t j, const TScanArgs& a, const float* slam,
                                          uint32_t& c, float& mult) {
  const uint32_t cw = CW ? CW : a.cw, sw = CW ? SW : a.sw;
  if (cw == 4) c = (wp[(j >> 3) * kBlockPts] >> (4 * (j & 7))) & 0xFu;
  else if (cw == 8) c = (wp[(j >> 2) * kBlockPts] >> (8 * (j & 3))) & 0xFFu;
  else c = (wp[(j >> 1) * kBlockPts] >> (16 * (j & 1))) & 0xFFFFu;
  const uint32_t* sp = wp + a.Wc * kBlockPts;
  if (sw == 0) {
    mult = slam[j * a.s];
  } else if (sw == 4) {
    mult = slam[j * a.s + ((sp[(j >> 3) * kBlockPts] >> (4 * (j & 7))) & 0xFu)];
  } else if (sw == 8) {
    mult = slam[j * a.s + ((sp[(j >> 2) * kBlockPts] >> (8 * (j & 3))) & 0xFFu)];
  } else if (sw == 16) {
    mult = __half2float(__ushort_as_half(
        static_cast<unsigned short>((sp[(j >> 1) * kBlockPts] >> (16 * (j & 1))) & 0xFFFFu)));
  } else {
    mult = __uint_as_float((sp[j * kBlockPts]));
  }
}

template <int DB, int CW, int SW>
__device__ __forceinline__ uint4 decode_planes(const uint32_t* wp, uint32_t slab, const TScanArgs& a,
                                               const float* ctab, const float* slam) {
  constexpr int SPS = 8 / DB;
  float v[8];
#pragma unroll
  for (int t = 0; t < SPS; ++t) {
    const uint32_t j = slab * SPS + t;
    if (j < a.m) {
      uint32_t c;
      float mult;
      planes_cs<CW, SW>(wp, j, a, slam, c, mult);
      const float* row = ctab + (static_cast<size_t>(j) * a.k + c) * DB;
      if constexpr (DB == 4) {
        const float4 r = a.cprime_smem ? *reinterpret_cast<const float4*>(row)
                                       : __ldg(reinterpret_cast<const float4*>(row));
        v[4 * t + 0] = __fmul_rn(mult, r.x);
        v[4 * t + 1] = __fmul_rn(mult, r.y);
        v[4 * t + 2] = __fmul_rn(mult, r.z);
        v[4 * t + 3] = __fmul_rn(mult, r.w);
      } else {
#pragma unroll
        for (int e = 0; e < DB; ++e) v[DB * t + e] = __fmul_rn(mult, a.cprime_smem ? row[e] : __ldg(row + e));
      }
    } else {
#pragma unroll
      for (int e = 0; e < DB; ++e) v[DB * t + e] = 0.0f;
    }
  }
  uint32_t out[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    out[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

template <bool JOINT, int DB, int N, int CW = 0, int SW = 0, int RB = 0>
__global__ void __launch_bounds__(kTThreads, 1) tscan_kernel(TScanArgs a) {
  extern __shared__ __align__(128) uint8_t smem_t[];
  const uint32_t kb = a.kpad * 2;                       // bytes per operand row
  uint8_t* sA = smem_t;                                 // [kpad/8][128][16]
  uint8_t* sX = sA + kTM * kb;                          // 2 x [kpad/8][N][16]
  const uint32_t cbytes = N * a.W * 4;                  // one code tile (N / 32 blocks)
  uint8_t* sC = sX + 2 * N * kb;                        // 2 x staged code tiles
  uint8_t* sT = sC + 2 * cbytes;                        // decode tables
  const uint32_t tab_bytes = JOINT ? a.msec * a.rows * DB * 2
                                   : (a.cprime_smem ? a.msec * a.k * DB * 4 : 0u) + (a.lam_smem ? a.msec * a.s * 4 : 0u);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sT + ((tab_bytes + 15) & ~15u));  // epilogue select scratch
  __shared__ __align__(8) uint64_t bar_a, bar_xfull[2], bar_xempty[2], bar_afull[2], bar_aempty[2],
      bar_cfull[2], bar_cempty[2];
  __shared__ uint32_t tmem_base;

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t qt = blockIdx.x, r = blockIdx.y;
  // point space: the index (main pass) or the sample's blocks (seed pass)
  const uint64_t space = a.mode ? static_cast<uint64_t>(a.sblocks) * kBlockPts : a.n_local;
  const uint64_t pbeg = static_cast<uint64_t>(r) * a.tiles_per_range * N;
  const uint64_t pend = min(space, pbeg + static_cast<uint64_t>(a.tiles_per_range) * N);
  const uint32_t ntiles = pend > pbeg ? static_cast<uint32_t>((pend - pbeg + N - 1) / N) : 0u;

  // ---- tables -> shared memory
  if constexpr (JOINT) {
    const uint4* src = reinterpret_cast<const uint4*>(a.jtab);
    uint4* dst = reinterpret_cast<uint4*>(sT);
    for (uint32_t i = tid; i < tab_bytes / 16; i += kTThreads) dst[i] = __ldg(src + i);
  } else {
    float* st = reinterpret_cast<float*>(sT);
    uint32_t o = 0;
    if (a.cprime_smem) {
      for (uint32_t i = tid; i < a.msec * a.k * DB; i += kTThreads) st[i] = __ldg(a.cprime + i);
      o = a.msec * a.k * DB;
    }
    if (a.lam_smem)
      for (uint32_t i = tid; i < a.msec * a.s; i += kTThreads) st[o + i] = i < a.m * a.s ? __ldg(a.lam + i) : 0.0f;
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(2u * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      mbar_init(&bar_a, 1);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&bar_xfull[i], kDecWarps);
        mbar_init(&bar_xempty[i], 1);
        mbar_init(&bar_afull[i], 1);
        mbar_init(&bar_aempty[i], kEpiWarps);
        mbar_init(&bar_cfull[i], 1);
        mbar_init(&bar_cempty[i], kDecWarps);
      }
      fence_mbar_init();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      mbar_expect_tx(&bar_a, kTM * kb);
      bulk_g2s(sA, a.qa + static_cast<size_t>(qt) * kTM * kb, kTM * kb, &bar_a);
      mbar_wait(&bar_a, 0u);
      const uint32_t a0 = smem_u32(sA);
      const uint32_t idesc = umma_idesc_f16(kTM, N);
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t s = t & 1u, ph = (t >> 1) & 1u;
        mbar_sleep(&bar_xfull[s], ph);
        mbar_sleep(&bar_aempty[s], ph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t x0 = smem_u32(sX + s * N * kb);
        const uint32_t dt = tmem + s * N;
        for (uint32_t ks = 0; ks < a.kpad / 16; ++ks) {
          const uint64_t da = sdesc(a0 + ks * 2 * (kTM * 16), kTM * 16, 128);
          const uint64_t db = sdesc(x0 + ks * 2 * (N * 16), N * 16, 128);
          const uint32_t acc = ks > 0 ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar_xempty[s]))
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar_afull[s]))
                     : "memory");
      }
    }
    __syncwarp();
  } else if (warp == kProdWarp) {
    // ------------------------------------------------------------ code tiles (TMA)
    if (lane == 0) {
      const uint64_t nblk_all = (a.n_local + kBlockPts - 1) / kBlockPts;
      const uint32_t wb = a.W * kBlockPts * 4;  // bytes per 32-point block
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t s = t & 1u, ph = (t >> 1) & 1u;
        mbar_sleep(&bar_cempty[s], ph ^ 1u);
        const uint64_t j0 = (pbeg + static_cast<uint64_t>(t) * N) / kBlockPts;  // first block of the tile
        if (a.mode == 0) {
          const uint64_t left = nblk_all - j0;
          const uint32_t nb = left < N / kBlockPts ? static_cast<uint32_t>(left) : N / kBlockPts;
          mbar_expect_tx(&bar_cfull[s], nb * wb);
          bulk_g2s(sC + s * cbytes, a.codes + j0 * a.W * kBlockPts, nb * wb, &bar_cfull[s]);
        } else {
          // seed pass: the tile's blocks are spread evenly over the full blocks
          const uint64_t left = a.sblocks - j0;
          const uint32_t nb = left < N / kBlockPts ? static_cast<uint32_t>(left) : N / kBlockPts;
          mbar_expect_tx(&bar_cfull[s], nb * wb);
          for (uint32_t c = 0; c < nb; ++c) {
            const uint64_t blk = (j0 + c) * a.nbfull / a.sblocks;
            bulk_g2s(sC + s * cbytes + c * wb, a.codes + blk * a.W * kBlockPts, wb, &bar_cfull[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= kDecWarp0) {
    // ------------------------------------------------------------ decoders
    const uint32_t dt = tid - kDecWarp0 * 32;
    const uint32_t nslab = a.kpad / 8;
    const uint32_t pi = dt % N;                     // this thread's point in the tile
    constexpr uint32_t kStep = kDecThreads >= N ? kDecThreads / N : 1;
    const uint32_t s0 = kDecThreads >= N ? dt / N : 0;
    const float* slam = nullptr;
    const float* ctab = a.cprime;
    if constexpr (!JOINT) {
      const float* st = reinterpret_cast<const float*>(sT);
      if (a.cprime_smem) ctab = st;
      slam = a.lam_smem ? st + (a.cprime_smem ? a.msec * a.k * DB : 0u) : a.lam;
    }
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t s = t & 1u, ph = (t >> 1) & 1u;
      mbar_sleep(&bar_xempty[s], ph ^ 1u);
      mbar_sleep(&bar_cfull[s], ph);
      uint8_t* xs = sX + s * N * kb;
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(sC + s * cbytes);
      const uint64_t p0 = pbeg + static_cast<uint64_t>(t) * N;
      for (uint32_t pp = pi; pp < N; pp += (kDecThreads >= N ? N : kDecThreads)) {
        const uint32_t* wp = cs + (pp >> 5) * (a.W * kBlockPts) + (pp & 31u);
        uint8_t* dst = xs + pp * 16;
        uint32_t sl = s0;
        if (p0 + pp < pend) {
          // slabs with code words (JOINT8: the W words hold 4 sections each)
          const uint32_t ndata = JOINT ? min(nslab, (a.W * 4 * DB + 7) / 8) : nslab;
#pragma unroll 2
          for (; sl < ndata; sl += kStep) {
            uint4 v;
            if constexpr (JOINT) v = decode_joint<DB, RB>(wp, sl, reinterpret_cast<const __half*>(sT), a.rows);
            else v = decode_planes<DB, CW, SW>(wp, sl, a, ctab, slam);
            *reinterpret_cast<uint4*>(dst + sl * (N * 16)) = v;
          }
        }
        for (; sl < nslab; sl += kStep) *reinterpret_cast<uint4*>(dst + sl * (N * 16)) = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_cempty[s]);
        mbar_arrive(&bar_xfull[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp w: TMEM lanes 32*(w%4).. (its 32 queries), columns [half*N/2, (half+1)*N/2)
    const uint32_t quad = warp & 3u, half = warp >> 2;
    const uint32_t row = quad * 32 + lane;
    const uint32_t q = qt * kTM + row;
    const float2 se = a.fse[q];
    bool live = q < a.B && isfinite(se.y);
    const float eps2 = 2.0f * se.y;
    const float bbase = (a.mode == 0 && live) ? a.base[q] : -INFINITY;
    const bool use_bins = a.mode == 0 && live && bbase > -INFINITY;  // (NaN: no seed)
    const float delta = se.y;  // bin width: eps
    const float inv_delta = __frcp_rd(delta);  // rounded down: bins never overstate a value
    uint32_t* qbins = a.bins + static_cast<size_t>(q) * 32;
    float thr = -INFINITY;
    uint32_t cnt = 0;
    const size_t li = (static_cast<size_t>(r) * a.Bpad + q) * 2 + half;  // this thread's list
    uint64_t* list = a.lists + li * a.Lc;
    uint32_t* hist = scratch + warp * (kHistWords + kSvWords);
    const Group g{0, 32, static_cast<int>(lane)};
    constexpr uint32_t kHalf = N / 2;
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t s = t & 1u, ph = (t >> 1) & 1u;
      const uint64_t p0 = pbeg + static_cast<uint64_t>(t) * N;
      const uint32_t valid = pend - p0 < static_cast<uint64_t>(N) ? static_cast<uint32_t>(pend - p0) : static_cast<uint32_t>(N);
      if (a.mode == 0 && (t & 3u) == 0u && live) {  // other CTAs' pruning of this query
        const uint32_t go = __ldcg(a.gthr + q);
        if (go) thr = fmaxf(thr, ord_to_float(go));
        if (use_bins) {  // the highest bin whose suffix count reaches K
          uint32_t cnts[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint4 v4 = __ldcg(reinterpret_cast<const uint4*>(qbins) + i);
            cnts[4 * i] = v4.x, cnts[4 * i + 1] = v4.y, cnts[4 * i + 2] = v4.z, cnts[4 * i + 3] = v4.w;
          }
          uint32_t suf = 0;
          int hb = -1;
#pragma unroll
          for (int i = 31; i >= 0; --i) {
            suf += cnts[i];
            if (hb < 0 && suf >= a.K) hb = i;
          }
          if (hb > 0) {
            const float tc = __double2float_rd(static_cast<double>(bbase) + hb * static_cast<double>(delta) -
                                               static_cast<double>(eps2));
            thr = fmaxf(thr, tc);
          }
        }
      }
      mbar_sleep(&bar_afull[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tb = tmem + ((quad * 32u) << 16) + s * N + half * kHalf;
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < kHalf; c0 += 64) {
        float v0[32], v1[32];
        tmem_ld32(tb + c0, v0);
        tmem_ld32(tb + c0 + 32, v1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float(&v)[32] = h ? v1 : v0;
          const uint32_t cb = half * kHalf + c0 + 32 * h;  // column of v[0] in the tile
          if (cb + 32 > valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (cb + i >= valid) v[i] = -INFINITY;
          }
          float mx = fmax3(v[0], v[1], v[2]);
#pragma unroll
          for (int i = 3; i < 31; i += 2) mx = fmax3(mx, v[i], v[i + 1]);
          mx = fmaxf(mx, v[31]);
          if (a.mode) {  // seed pass: the block's best approximate score
            if (q < a.Bpad && cb < valid) a.cmax[static_cast<size_t>(q) * a.cm_stride + (p0 + cb) / kBlockPts] = mx;
            continue;
          }
          const bool lp = live && mx >= thr;
          if (__any_sync(0xFFFFFFFFu, lp)) {
            // this lane's passing columns, then one TMEM re-read per column
            // that passes for some lane (warp-uniform loop)
            uint32_t mask = 0;
            if (lp) {
#pragma unroll
              for (int i = 0; i < 32; ++i) mask |= (v[i] >= thr ? 1u : 0u) << i;
            }
            uint32_t um = __reduce_or_sync(0xFFFFFFFFu, mask);
            while (um) {
              const int i = __ffs(um) - 1;
              um &= um - 1u;
              const float vi = tmem_ld1(tb + c0 + 32 * h + i);
              if ((mask >> i) & 1u) {
                list[cnt++] = (static_cast<uint64_t>(ord_of(vi)) << 32) | static_cast<uint32_t>(p0 + cb + i);
                if (use_bins) {
                  // rounded down, so bin i only holds values >= base + i * delta
                  const float bf = __fmul_rd(__fsub_rd(vi, bbase), inv_delta);
                  const int bi = bf >= 31.0f ? 31 : (bf <= 0.0f ? 0 : static_cast<int>(bf));
                  atomicAdd(qbins + bi, 1u);
                }
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_aempty[s]);
      if (a.mode) continue;
      // overflow guard: prune a full list (warp-cooperative select of its K-th key)
      uint32_t need = __ballot_sync(0xFFFFFFFFu, live && cnt > a.Lc - kHalf);
      while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1u;
        uint64_t* L = reinterpret_cast<uint64_t*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(list), src));
        const uint32_t n = __shfl_sync(0xFFFFFFFFu, cnt, src);
        const float e2 = __shfl_sync(0xFFFFFFFFu, eps2, src);
        float th = __shfl_sync(0xFFFFFFFFu, thr, src);
        const uint64_t kth = group_select_by([L](uint32_t i) { return L[i]; }, n, a.K, hist, hist + kHistWords, g);
        const float tk = ord_to_float(static_cast<uint32_t>(kth >> 32));
        const float nt = __double2float_rd(static_cast<double>(tk) - static_cast<double>(e2));
        uint32_t nn = n;
        if (nt > th) {
          th = nt;
          nn = group_compact(L, n, static_cast<uint64_t>(ord_of(th)) << 32, nullptr, g);  // (one warp: no scratch)
        }
        if (static_cast<int>(lane) == src) {
          cnt = nn;
          thr = th;
          if (cnt > a.Lc - kHalf) {  // cannot prune below capacity: exact full scan later
            live = false;
            a.ovf[q] = 1u;
          } else {
            atomicMax(a.gthr + q, ord_of(th));
          }
        }
      }
    }
    if (a.mode == 0 && q < a.Bpad) a.counts[li] = cnt;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2u * N));
}

// ---- K2-T over the decoded operand cache: TMA -> shared memory -> tcgen05 ->
// epilogue, no decode warps.  Warps 0-7 epilogue (as tscan_kernel), warp 8
// MMA issuer, warp 9 TMA producer (kpad/8 slab copies of N*16 bytes per tile),
// warp 10 keeps the 128 queries' pruning thresholds fresh in shared memory.

// uint4 index of (point p, slab sl) in the tile-major operand cache
__host__ __device__ inline uint64_t xhat_u4_index(uint64_t p, uint32_t sl, uint32_t nslab, uint32_t T) {
  return ((p / T) * nslab + sl) * T + p % T;
}

struct XArgs {
  // tile-major operand cache [tile of N points][kpad/8][N][16 B]: a tile is one
  // contiguous run of N * kpad * 2 bytes, already in the shared-memory (UMMA
  // K-major) order, so the producer fetches it with ONE bulk copy instead of one
  // per 16-byte K slab (kpad / 8 small copies per tile kept the producer, not the
  // tensor pipe, on the critical path: exp 4 vs exp 1 in tools/tc_exp.py)
  const uint8_t* xhat;
  uint64_t npad;
  uint32_t stiles_all;   // seed pass: tiles of the whole index the sample tiles spread over
};

constexpr int kCWarps = kEpiWarps + 3;
constexpr int kCThreads = kCWarps * 32;  // 352
constexpr int kCMma = kEpiWarps, kCProd = kEpiWarps + 1, kCThr = kEpiWarps + 2;

// QT query tiles (of 128 queries) per CTA share every point tile: the operand
// stream from L2 — the limiter of the 1-tile kernel on every config (exp 4 vs
// exp 1 in tools/tc_exp.py) — is read once per QT * 128 queries.  The tiles'
// accumulators alternate in the two TMEM buffers (virtual tile v = QT * t + h
// uses buffer v & 1), so the MMA of (t, h + 1) overlaps the epilogue of (t, h).
// AT: the query operand lives in TMEM (tcgen05.st once, then the .ts form of the
// MMA): the tensor core re-reads A for every instruction, and with long K and
// 128-column point tiles (C4) those shared-memory reads are as large as B's.
// QH: the query operand carries a second fp16 half, q = q_hi + q_lo (the tile has
// 2 * kpad K columns: hi slabs, then lo slabs), and every point slab is used by
// two MMAs.  The query's fp16 rounding — half of the filter's error bound —
// drops to 2^-22, so eps and with it the candidate appends shrink; the doubled
// tensor work is free where reading the accumulators out of TMEM bounds the
// tile anyway (kpad <= 112 at N = 256).
template <int N, int ST, int QT = 1, bool AT = false, bool QH = false>
__global__ void __launch_bounds__(kCThreads, 1) tscan_cached_kernel(TScanArgs a, XArgs xa) {
  static_assert(!AT || QT == 1, "the TMEM query operand holds one tile");
  static_assert(!QH || (!AT && QT == 1), "the hi/lo query operand is a shared-memory tile");
  constexpr uint32_t AK = QH ? 2u : 1u;  // K extent of the query tile in units of kpad
  extern __shared__ __align__(128) uint8_t smem_c[];
  const uint32_t kb = a.kpad * 2;
  const uint32_t nslab = a.kpad / 8;
  uint8_t* sA = smem_c;                    // [kpad/8][128][16]
  uint8_t* sX = sA + (AT ? 0 : QT * AK * kTM * kb);  // ST x [kpad/8][N][16]   (sA: QT tiles, none with AT)
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sX + ST * N * kb);
  __shared__ __align__(8) uint64_t bar_a, bar_xfull[ST], bar_xempty[ST], bar_afull[2], bar_aempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float s_thr[QT * kTM];   // per-query threshold, kept fresh by the threshold warp
  __shared__ float s_eps[2][QT * kTM], s_bb[2][QT * kTM];  // per (column half, query): eps, seed base
  __shared__ volatile uint32_t s_done;  // epilogue warps finished
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t qt = blockIdx.x * QT, r = blockIdx.y;  // first query tile of this CTA
  // main pass: points of the index; seed pass (mode 1): sample tiles, each a
  // whole tile of the index, spread evenly over its stiles_all tiles
  const uint64_t space = a.mode ? static_cast<uint64_t>(a.sblocks) * kBlockPts : a.n_local;
  const uint64_t pbeg = static_cast<uint64_t>(r) * a.tiles_per_range * N;
  const uint64_t pend = min(space, pbeg + static_cast<uint64_t>(a.tiles_per_range) * N);
  const uint32_t ntiles = pend > pbeg ? static_cast<uint32_t>((pend - pbeg + N - 1) / N) : 0u;
  const uint32_t stiles = a.mode ? a.sblocks / (N / kBlockPts) : 0u;

  if (tid < QT * kTM) {  // start from the seed threshold (or another CTA's bound)
    const uint32_t q0 = qt * kTM + tid;
    const uint32_t go = (a.mode == 0 && q0 < a.B) ? __ldcg(a.gthr + q0) : 0u;
    s_thr[tid] = go ? ord_to_float(go) : -INFINITY;
  }
  if (tid == 0) s_done = 0;
  if (warp == kCMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(AT ? 512u : 2u * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      mbar_init(&bar_a, AT ? 4 : 1);
      for (int i = 0; i < ST; ++i) {
        mbar_init(&bar_xfull[i], 1);
        mbar_init(&bar_xempty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&bar_afull[i], 1);
        mbar_init(&bar_aempty[i], kEpiWarps);
      }
      fence_mbar_init();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == kCMma) {
    if (lane == 0) {
      if constexpr (!AT) {
        mbar_expect_tx(&bar_a, QT * AK * kTM * kb);
        for (int h = 0; h < QT; ++h)
          bulk_g2s(sA + h * AK * kTM * kb, a.qa + static_cast<size_t>(qt + h) * AK * kTM * kb, AK * kTM * kb,
                   &bar_a);
      }
      mbar_wait(&bar_a, 0u);  // (AT: the four quadrant warps have stored the tile into TMEM)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = umma_idesc_f16(kTM, N);
      for (uint32_t v = 0; v < QT * ntiles; ++v) {
        const uint32_t t = v / QT, h = v % QT;
        const uint32_t s = t % ST, ph = (t / ST) & 1u;
        const uint32_t sa = v & 1u, pa = (v >> 1) & 1u;
        if (h == 0) mbar_sleep(&bar_xfull[s], ph);
        mbar_sleep(&bar_aempty[sa], pa ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + h * AK * kTM * kb);
        const uint32_t x0 = smem_u32(sX + s * N * kb);
        const uint32_t dt = tmem + sa * N;
        const uint32_t nks = a.kpad / 16;
        for (uint32_t ks = 0; ks < AK * nks; ++ks) {
          const uint32_t kx = QH ? (ks >= nks ? ks - nks : ks) : ks;  // lo slabs meet the same point slabs
          const uint64_t db = sdesc(x0 + kx * 2 * (N * 16), N * 16, 128);
          const uint32_t acc = ks > 0 ? 1u : 0u;
          if constexpr (AT) {
            const uint32_t ta = tmem + 2u * N + ks * 8u;  // 16 fp16 of K = 8 columns
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
                "r"(ta), "l"(db), "r"(idesc), "r"(acc));
          } else {
            const uint64_t da = sdesc(a0 + ks * 2 * (kTM * 16), kTM * 16, 128);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        if (h == QT - 1)  // the point tile's last reader
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&bar_xempty[s]))
                       : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar_afull[sa]))
                     : "memory");
      }
    }
    __syncwarp();
  } else if (warp == kCProd) {
    if (lane == 0) {
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t s = t % ST, ph = (t / ST) & 1u;
        mbar_sleep(&bar_xempty[s], ph ^ 1u);
        if ((a.exp == 3 || a.exp == 4) && t >= ST) {  // experiment: no operand traffic after the first fill
          mbar_arrive(&bar_xfull[s]);
          continue;
        }
        const uint64_t gt = pbeg / N + t;  // tile of the point space
        const uint64_t src_tile = a.mode ? gt * xa.stiles_all / stiles : gt;
        mbar_expect_tx(&bar_xfull[s], N * kb);
        {  // the tile: one contiguous run, fetched in a few large pieces
          const uint32_t bytes = N * kb, piece = a.exp >= 16 ? a.exp * 1024u : 16384u;
          const uint8_t* src = xa.xhat + src_tile * static_cast<uint64_t>(bytes);
          for (uint32_t o = 0; o < bytes; o += piece)
            bulk_g2s(sX + s * bytes + o, src + o, min(piece, bytes - o), &bar_xfull[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == kCThr) {
    // ------------------------------------------------------------ threshold warp
    // for the CTA's 128 queries: the shared pruning bound gthr and the highest
    // bin whose suffix count reaches K, refreshed until the epilogue is done
    // (its loads' latency stays off the epilogue's critical path)
    if (a.mode == 0) {
      while (true) {
        const bool last = s_done >= static_cast<uint32_t>(kEpiWarps);
        for (uint32_t rr = lane; rr < QT * kTM; rr += 32) {
          const uint32_t q = qt * kTM + rr;
          if (q >= a.B) continue;
          const float2 se = a.fse[q];
          if (!isfinite(se.y)) continue;
          float th = -INFINITY;
          const uint32_t go = __ldcg(a.gthr + q);
          if (go) th = ord_to_float(go);
          const float bbase = a.base[q];
          if (bbase > -INFINITY) {
            const uint4* qb = reinterpret_cast<const uint4*>(a.bins + static_cast<size_t>(q) * 32);
            uint32_t cnts[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint4 v4 = __ldcg(qb + i);
              cnts[4 * i] = v4.x, cnts[4 * i + 1] = v4.y, cnts[4 * i + 2] = v4.z, cnts[4 * i + 3] = v4.w;
            }
            uint32_t suf = 0;
            int hb = -1;
#pragma unroll
            for (int i = 31; i >= 0; --i) {
              suf += cnts[i];
              if (hb < 0 && suf >= a.K) hb = i;
            }
            if (hb > 0)
              th = fmaxf(th, __double2float_rd(static_cast<double>(bbase) + hb * static_cast<double>(se.y) -
                                               2.0 * static_cast<double>(se.y)));
          }
          if (th > s_thr[rr]) s_thr[rr] = th;
        }
        if (last) break;
        __nanosleep(500);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (as tscan_kernel)
    const uint32_t quad = warp & 3u, half = warp >> 2;
    const uint32_t row = quad * 32 + lane;
    // per query tile h: the mutable state in registers, the constants in shared
    // memory (each thread reads back only what it wrote)
    float thr_h[QT];
    uint32_t cnt_h[QT];
    bool live_h[QT];
#pragma unroll
    for (int h = 0; h < QT; ++h) {
      const uint32_t qh = (qt + h) * kTM + row;
      const float2 se = a.fse[qh];
      live_h[h] = qh < a.B && isfinite(se.y);
      thr_h[h] = -INFINITY;
      cnt_h[h] = 0;
      s_eps[half][h * kTM + row] = se.y;
      s_bb[half][h * kTM + row] = (a.mode == 0 && live_h[h]) ? a.base[qh] : -INFINITY;
    }
    if constexpr (AT) {
      if (half == 0) {  // one warp per lane quadrant: row i of the tile -> TMEM lane i
        const uint8_t* src = a.qa + static_cast<size_t>(qt) * kTM * kb + static_cast<size_t>(row) * 16;
        for (uint32_t sl = 0; sl < nslab; ++sl) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(sl) * (kTM * 16));
          const uint32_t ta = tmem + ((quad * 32u) << 16) + 2u * N + sl * 4u;
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(w4.x),
                       "r"(w4.y), "r"(w4.z), "r"(w4.w)
                       : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_a);
      }
    }
    uint32_t* hist = scratch + warp * (kHistWords + kSvWords);
    const Group g{0, 32, static_cast<int>(lane)};
    constexpr uint32_t kHalf = N / 2;
    for (uint32_t v = 0; v < QT * ntiles; ++v) {
      const uint32_t t = v / QT, h = v % QT;
      const uint32_t sa = v & 1u, pa = (v >> 1) & 1u;
      const uint32_t q = (qt + h) * kTM + row;
      const float delta = s_eps[half][h * kTM + row];
      const float eps2 = 2.0f * delta;
      const float bbase = s_bb[half][h * kTM + row];
      const float inv_delta = __frcp_rd(delta);
      bool live = live_h[0];
      float thr = thr_h[0];
      uint32_t cnt = cnt_h[0];
      if (QT > 1 && h) {
        live = live_h[QT - 1];
        thr = thr_h[QT - 1];
        cnt = cnt_h[QT - 1];
      }
      const bool use_bins = a.mode == 0 && live && bbase > -INFINITY;  // (NaN: no seed)
      uint32_t* qbins = a.bins + static_cast<size_t>(q) * 32;
      uint64_t* list = a.lists + ((static_cast<size_t>(r) * a.Bpad + q) * 2 + half) * a.Lc;
      const uint64_t p0 = pbeg + static_cast<uint64_t>(t) * N;
      const uint32_t valid = pend - p0 < static_cast<uint64_t>(N) ? static_cast<uint32_t>(pend - p0) : static_cast<uint32_t>(N);
      if (a.mode == 0 && live) thr = fmaxf(thr, s_thr[h * kTM + row]);  // (threshold warp)
      mbar_sleep(&bar_afull[sa], pa);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (a.exp == 1 || a.exp == 4) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_aempty[sa]);
        continue;
      }
      const uint32_t tb = tmem + ((quad * 32u) << 16) + sa * N + half * kHalf;
      // 32-column chunks; the next chunk's TMEM load is in flight while this
      // one is tested
      float vb[2][32];
      float seed_mx = -INFINITY;  // seed pass: the maximum of this (tile, column half)
      tmem_ld32(tb, vb[0]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (uint32_t ch = 0; ch < kHalf / 32; ++ch) {
        float(&v)[32] = vb[ch & 1];
        if (ch + 1 < kHalf / 32) tmem_ld32(tb + (ch + 1) * 32, vb[(ch + 1) & 1]);
        {
          const uint32_t cb = half * kHalf + ch * 32;  // column of v[0] in the tile
          if (cb + 32 > valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (cb + i >= valid) v[i] = -INFINITY;
          }
          // maxima of the four 8-column groups, then of the chunk
          float gm[4];
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            float m8 = fmax3(v[8 * g8], v[8 * g8 + 1], v[8 * g8 + 2]);
            m8 = fmax3(m8, v[8 * g8 + 3], v[8 * g8 + 4]);
            m8 = fmax3(m8, v[8 * g8 + 5], v[8 * g8 + 6]);
            gm[g8] = fmaxf(m8, v[8 * g8 + 7]);
          }
          const float mx = fmaxf(fmax3(gm[0], gm[1], gm[2]), gm[3]);
          if (a.mode) {
            if (cb < valid) seed_mx = fmaxf(seed_mx, mx);
          } else {
            const bool lp = live && mx >= thr && a.exp != 2;
            if (__any_sync(0xFFFFFFFFu, lp)) {
              // rare.  The pass mask comes from the passing 8-column groups; the
              // warp then walks the union of the lanes' masks column by column
              // (uniform), so a dense tile costs 32 rounds, not 32 per lane
              uint32_t mask = 0;
              if (lp) {
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8)
                  if (gm[g8] >= thr) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) mask |= (v[8 * g8 + i] >= thr ? 1u : 0u) << (8 * g8 + i);
                  }
              }
              uint32_t um = __reduce_or_sync(0xFFFFFFFFu, mask);
#pragma unroll 1
              while (um) {
                const int i = __ffs(um) - 1;
                um &= um - 1u;
                const float vi = tmem_ld1(tb + ch * 32 + i);  // (measured: faster than selecting it from the registers)
                if ((mask >> i) & 1u) {
                  list[cnt++] = (static_cast<uint64_t>(ord_of(vi)) << 32) | static_cast<uint32_t>(p0 + cb + i);
                  if (use_bins) {
                    const float bf = __fmul_rd(__fsub_rd(vi, bbase), inv_delta);
                    const int bi = bf >= 31.0f ? 31 : (bf <= 0.0f ? 0 : static_cast<int>(bf));
                    atomicAdd(qbins + bi, 1u);
                  }
                }
              }
            }
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_aempty[sa]);
      if (a.mode) {
        // one entry per (sample tile, column half): the K-th largest of them still
        // stands for K distinct points, with a quarter of the per-block entries
        if (q < a.Bpad) a.cmax[static_cast<size_t>(q) * a.cm_stride + (p0 / N) * 2 + half] = seed_mx;
        continue;
      }
      uint32_t need = __ballot_sync(0xFFFFFFFFu, live && cnt > a.Lc - kHalf);
      while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1u;
        uint64_t* L = reinterpret_cast<uint64_t*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(list), src));
        const uint32_t n = __shfl_sync(0xFFFFFFFFu, cnt, src);
        const float e2 = __shfl_sync(0xFFFFFFFFu, eps2, src);
        float th = __shfl_sync(0xFFFFFFFFu, thr, src);
        const uint64_t kth = group_select_by([L](uint32_t i) { return L[i]; }, n, a.K, hist, hist + kHistWords, g);
        const float tk = ord_to_float(static_cast<uint32_t>(kth >> 32));
        const float nt = __double2float_rd(static_cast<double>(tk) - static_cast<double>(e2));
        uint32_t nn = n;
        if (nt > th) {
          th = nt;
          nn = group_compact(L, n, static_cast<uint64_t>(ord_of(th)) << 32, nullptr, g);
        }
        if (static_cast<int>(lane) == src) {
          cnt = nn;
          thr = th;
          if (cnt > a.Lc - kHalf) {
            live = false;
            a.ovf[q] = 1u;
          } else {
            atomicMax(a.gthr + q, ord_of(th));
          }
        }
      }
      if (QT > 1 && h) {
        live_h[QT - 1] = live;
        thr_h[QT - 1] = thr;
        cnt_h[QT - 1] = cnt;
      } else {
        live_h[0] = live;
        thr_h[0] = thr;
        cnt_h[0] = cnt;
      }
    }
    if (a.mode == 0) {
#pragma unroll
      for (int h = 0; h < QT; ++h) {
        const uint32_t qh = (qt + h) * kTM + row;
        if (qh < a.Bpad) a.counts[(static_cast<size_t>(r) * a.Bpad + qh) * 2 + half] = cnt_h[h];
      }
    }
    __syncwarp();
    if (lane == 0) atomicAdd(const_cast<uint32_t*>(&s_done), 1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kCMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(AT ? 512u : 2u * N));
}

// decode every point once into the cache: thread per (point, slab)
template <bool JOINT, int DB, int CW = 0, int SW = 0, int RB = 0>
__global__ void xhat_build_kernel(TScanArgs a, const __half* jtab, const float* ctab, const float* slam,
                                  uint8_t* xhat, uint64_t npad, uint32_t T) {
  const uint32_t nslab = a.kpad / 8;
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p = i % npad;
  const uint32_t sl = static_cast<uint32_t>(i / npad);
  if (sl >= nslab) return;
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t ndata = JOINT ? min(nslab, (a.W * 4 * DB + 7) / 8) : nslab;
  if (p < a.n_local && sl < ndata) {
    const uint32_t* wp = a.codes + (p >> 5) * (static_cast<uint64_t>(a.W) * kBlockPts) + (p & 31u);
    if constexpr (JOINT) v = decode_joint<DB, RB>(wp, sl, jtab, a.rows);
    else v = decode_planes<DB, CW, SW>(wp, sl, a, ctab, slam);
  }
  reinterpret_cast<uint4*>(xhat)[xhat_u4_index(p, sl, nslab, T)] = v;
}

// max over the points of the L2 norm of their cached fp16 operand vector (the
// Cauchy-Schwarz side of the error bound, see tq_prep_kernel)
__global__ void xhat_norm_kernel(const uint8_t* __restrict__ xhat, uint64_t n, uint32_t T, uint32_t nslab,
                                 unsigned long long* __restrict__ out_bits) {
  const uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (p < n)
    for (uint32_t sl = 0; sl < nslab; ++sl) {
      const uint4 v = reinterpret_cast<const uint4*>(xhat)[xhat_u4_index(p, sl, nslab, T)];
      const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(h[i]);
        sq = fma(static_cast<double>(f.x), static_cast<double>(f.x), sq);
        sq = fma(static_cast<double>(f.y), static_cast<double>(f.y), sq);
      }
    }
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(sqrt(sq) * (1.0 + 1e-12)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, b);
}

// ---- per-query operand tile, scale and error bound
struct PrepArgs {
  const float* Q;
  uint32_t B, Bpad, d, m, dbar, kpad, k, msec;
  const float* tau;
  const float* lam_max;
  const float* cb;  // [m][k][dbar] fp32 codebooks
  double rho;       // relative error factor (see tc_rho)
  uint32_t qh;      // 1: the operand tile carries q_hi and q_lo (2 * kpad columns)
  double xnorm_max;  // max_p ||x'_p||_2 of the operand cache (0: not available)
  uint8_t* qa;
  float2* fse;
};

__global__ void tq_prep_kernel(PrepArgs a) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (row >= a.Bpad) return;
  const float* qq = a.Q + static_cast<size_t>(row) * a.d;
  const uint32_t dim = a.m * a.dbar;
  double mx = 0.0;
  for (uint32_t i = lane; i < dim; i += 32) {
    const float qi = (row < a.B && i < a.d) ? qq[i] : 0.0f;
    mx = fmax(mx, fabs(static_cast<double>(qi)) / static_cast<double>(a.tau[i / a.dbar]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  int e = 0;
  const double f = frexp(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
  const bool ok = row < a.B && mx > 0.0 && isfinite(mx) && e >= -120 && e <= 120;
  const double sigma = ok ? ldexp(1.0, -e) : 0.0;
  (void)f;
  // operand row in the UMMA K-major layout of its 128-row tile
  const uint32_t ak = a.qh ? 2u : 1u;
  uint8_t* tile = a.qa + static_cast<size_t>(row / kTM) * kTM * a.kpad * 2 * ak;
  const uint32_t rr = row % kTM;
  double qn2 = 0.0;  // ||q~||^2, q~_i = q_i sigma / tau_j(i)
  for (uint32_t i = lane; i < a.kpad; i += 32) {
    __half h = __float2half(0.0f), hl = __float2half(0.0f);
    if (ok && i < dim && i < a.d) {
      const double qt = static_cast<double>(qq[i]) * sigma / static_cast<double>(a.tau[i / a.dbar]);
      h = __double2half(qt);
      hl = __double2half(qt - static_cast<double>(__half2float(h)));  // (exact difference, then one rounding)
      qn2 = fma(qt, qt, qn2);
    }
    *reinterpret_cast<__half*>(tile + (i / 8) * (kTM * 16) + rr * 16 + (i % 8) * 2) = h;
    if (a.qh) *reinterpret_cast<__half*>(tile + (a.kpad / 8 + i / 8) * (kTM * 16) + rr * 16 + (i % 8) * 2) = hl;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qn2 += __shfl_xor_sync(0xFFFFFFFFu, qn2, o);
  // A_q = sum_j max_l|lambda_j,l| * max_c sum_a |q_j,a| |C_j[c][a]|
  double A = 0.0;
  if (ok && a.k <= 32 && (a.k & (a.k - 1)) == 0) {
    // k a power of two <= 32: lanes over the (section, center) pairs (coalesced
    // codebook reads), the max over a section's centers by xor-shuffles inside
    // its k-lane group
    // (four 32-pair steps at a time: their loads are independent, the warp is
    // alone with its query and otherwise pays one L2 round trip per step)
    const uint32_t pairs = a.m * a.k;
    for (uint32_t i0 = 0; i0 < pairs; i0 += 128) {
      double s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t idx = i0 + 32u * u + lane;
        const uint32_t j = idx / a.k;
        double s = 0.0;
        if (idx < pairs)
          for (uint32_t t = 0; t < a.dbar; ++t) {
            const uint32_t col = j * a.dbar + t;
            const float qi = col < a.d ? qq[col] : 0.0f;
            s += fabs(static_cast<double>(qi)) * fabs(static_cast<double>(a.cb[static_cast<size_t>(idx) * a.dbar + t]));
          }
        s4[u] = s;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t idx = i0 + 32u * u + lane;
        double s = s4[u];
        for (uint32_t o = a.k >> 1; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xFFFFFFFFu, s, o));
        if (idx < pairs && (lane & (a.k - 1)) == 0) A += s * static_cast<double>(a.lam_max[idx / a.k]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) A += __shfl_xor_sync(0xFFFFFFFFu, A, o);
  } else if (ok) {
    for (uint32_t j = 0; j < a.m; ++j) {
      double best = 0.0;
      for (uint32_t c = lane; c < a.k; c += 32) {
        double s = 0.0;
        for (uint32_t t = 0; t < a.dbar; ++t) {
          const uint32_t col = j * a.dbar + t;
          const float qi = col < a.d ? qq[col] : 0.0f;
          s += fabs(static_cast<double>(qi)) * fabs(static_cast<double>(a.cb[(static_cast<size_t>(j) * a.k + c) * a.dbar + t]));
        }
        best = fmax(best, s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
      A += best * static_cast<double>(a.lam_max[j]);
    }
  }
  if (lane == 0) {
    float eps = INFINITY;
    if (ok) {
      // scaled units; 1.25x margin over the derived bound
      const double abs_sub = static_cast<double>(a.kpad) * (a.qh ? 2.0 : 1.0) * ldexp(1.0, -23) +
                             sigma * a.m * (a.dbar + 2.0) * ldexp(1.0, -149);
      double eb = 1.25 * (a.rho * A * (1.0 + 1e-12) * sigma + abs_sub);
      if (a.xnorm_max > 0.0) {
        // Cauchy-Schwarz: sum_i |q~_i x~_i| <= ||q~|| ||x~_p|| for every point, with
        // ||x~_p|| <= ||x'_p|| (1 + 2^-10) + sqrt(kpad) 2^-25 (x' = the cached fp16
        // operands).  A_q above takes the largest scale level in every section at
        // once, which no point does; this bound is the tighter one on trained
        // (anisotropic) indexes whose scale codebooks have a few large levels.
        const double xn = a.xnorm_max * (1.0 + ldexp(1.0, -10)) + sqrt(static_cast<double>(a.kpad)) * ldexp(1.0, -25);
        const double ecs = 1.25 * (a.rho * sqrt(qn2) * xn * (1.0 + 1e-12) + abs_sub);
        eb = fmin(eb, ecs);
      }
      eps = __double2float_ru(eb);
      if (!isfinite(eps)) eps = INFINITY;
    }
    a.fse[row] = make_float2(static_cast<float>(sigma), eps);
  }
}

// ---- finish: exact re-score of the surviving pairs, top-K by (score desc, id asc)
struct FinishArgs {
  const uint32_t* codes;
  const float* Q;
  const float* cb;
  const float* lam;  // [m8][s]
  const uint64_t* lists;
  const uint32_t* counts;
  const uint32_t* gthr;
  const uint32_t* ovf;
  const float2* fse;
  uint64_t n_local, id_base;
  uint32_t W, Wc, m, k, s, cbits, cw, sw, fmt, d, dbar, ranges, Lc, Bpad, K, out_stride;
  uint32_t cap;  // keys staged per query (shared memory): 4096 or kFinCap
  // queries that need the exact scan of every point are handed to the parallel
  // fallback kernels (tscan_fb_*): fb_list[atomicAdd(fb_count)] = b, up to fb_cap
  uint32_t* fb_count;
  uint32_t* fb_list;
  uint32_t fb_cap;
  uint64_t* out_keys;
  int32_t* out_ids;
  float* out_scores;
  unsigned int* diag;  // optional: [0] max |approx - sigma*exact| / eps (float bits), [1] exact-scan queries
  // seed mode: gthr[b] = (K-th largest of the seed pass's block maxima
  // cmax[b][0, seed_blocks)) - 2 eps (scaled units)
  uint32_t seed, seed_blocks, cm_stride;
  const float* cmax;
  uint32_t* gthr_out;
  float* base_out;  // seed threshold (scaled) per query, the bins' origin
};

__device__ __forceinline__ float exact_score_point(const FinishArgs& a, uint64_t p, const float* eta,
                                                   const float* slam) {
  const uint32_t* wp = a.codes + (p >> 5) * (static_cast<uint64_t>(a.W) * kBlockPts) + (p & 31u);
  float acc = -0.0f;  // identity of the first fl(acc + term) (pq_index.cpp:221-236)
  for (uint32_t j = 0; j < a.m; ++j) {
    uint32_t c;
    float mult;
    if (a.fmt == PCPQG_FMT_JOINT8) {
      const uint32_t byte = (__ldg(wp + (j >> 2) * kBlockPts) >> (8 * (j & 3))) & 0xFFu;
      c = byte & ((1u << a.cbits) - 1u);
      mult = slam[j * a.s + (byte >> a.cbits)];
    } else {
      if (a.cw == 4) c = (__ldg(wp + (j >> 3) * kBlockPts) >> (4 * (j & 7))) & 0xFu;
      else if (a.cw == 8) c = (__ldg(wp + (j >> 2) * kBlockPts) >> (8 * (j & 3))) & 0xFFu;
      else c = (__ldg(wp + (j >> 1) * kBlockPts) >> (16 * (j & 1))) & 0xFFFFu;
      const uint32_t* sp = wp + a.Wc * kBlockPts;
      if (a.sw == 0) mult = slam[j * a.s];
      else if (a.sw == 4) mult = slam[j * a.s + ((__ldg(sp + (j >> 3) * kBlockPts) >> (4 * (j & 7))) & 0xFu)];
      else if (a.sw == 8) mult = slam[j * a.s + ((__ldg(sp + (j >> 2) * kBlockPts) >> (8 * (j & 3))) & 0xFFu)];
      else if (a.sw == 16)
        mult = __half2float(__ushort_as_half(
            static_cast<unsigned short>((__ldg(sp + (j >> 1) * kBlockPts) >> (16 * (j & 1))) & 0xFFFFu)));
      else mult = __uint_as_float(__ldg(sp + j * kBlockPts));
    }
    // fl(eta * lambda) (pq_index.cpp:203, 224-226) or fl(alpha * eta) (:232-234)
    acc = __fadd_rn(acc, __fmul_rn(eta[j * a.k + c], mult));
  }
  return acc;
}

// FLAT: the list gather by flat index (many short lists: small and mid batches)
template <bool FLAT>
__global__ void __launch_bounds__(kFinThreads, FLAT ? 1 : 8) tscan_finish_kernel(FinishArgs a) {
  extern __shared__ __align__(16) uint8_t smem_f[];
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_f);              // a.cap keys
  float* eta = reinterpret_cast<float*>(buf + a.cap);             // [m][k]
  float* slam = eta + static_cast<size_t>(a.m) * a.k;               // [m][s]
  __shared__ __align__(16) uint32_t scr[kGroupScratch];
  __shared__ uint32_t s_n, s_full;
  const uint32_t b = blockIdx.x, tid = threadIdx.x;
  const Group grp{0, kFinThreads, static_cast<int>(tid)};
  const float eps = a.fse[b].y;
  const bool full_scan = !isfinite(eps) || a.ovf[b] != 0u;

  if (tid == 0) s_n = 0;
  __syncthreads();

  // append keys >= floor into buf (warp-aggregated); when buf cannot take
  // another round, cut it to its best K (or, for approximate keys, to those
  // within 2 eps of the K-th) — `mk` maps an item to its key (0 = skip)
  uint64_t floor_key = 1ull;
  auto cut = [&](bool approx) {
    const uint32_t n = s_n;
    if (n <= a.K) return;
    const uint64_t kth = group_select(buf, n, a.K, scr, scr + kHistWords, grp);
    uint64_t f = kth;
    if (approx) {
      const float tk = ord_to_float(static_cast<uint32_t>(kth >> 32));
      const float th = __double2float_rd(static_cast<double>(tk) - 2.0 * static_cast<double>(eps));
      f = static_cast<uint64_t>(ord_of(th)) << 32;
    }
    floor_key = floor_key > f ? floor_key : f;
    const uint32_t nn = group_compact(buf, n, floor_key, scr + kHistWords + kSvWords, grp);
    if (tid == 0) s_n = nn;
    __syncthreads();
  };
  auto push = [&](uint64_t key) {
    const bool take = key >= floor_key && key != 0ull;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, take);
    uint32_t base = 0;
    if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, static_cast<uint32_t>(__popc(bal)));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (take) buf[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = key;
  };

  if (a.seed) {
    // K distinct points have approximate scores >= the K-th largest block
    // maximum t of the seed pass, so >= K points score >= t - eps exactly and
    // every point of the final top-K has approximate score >= t - 2 eps
    if (full_scan) return;
    const float* cm = a.cmax + static_cast<size_t>(b) * a.cm_stride;
    const uint32_t ns = a.seed_blocks;
    if (ns < a.K) return;
    for (uint32_t i0 = 0; i0 < ns; i0 += kFinThreads) {
      if (s_n + kFinThreads > a.cap) cut(false);
      const uint32_t i = i0 + tid;
      push(i < ns ? (static_cast<uint64_t>(ord_of(cm[i])) << 32) | i : 0ull);
      __syncthreads();
    }
    cut(false);
    const uint32_t n = s_n;
    __shared__ unsigned long long s_min;
    if (tid == 0) s_min = ~0ull;
    __syncthreads();
    unsigned long long mn = ~0ull;
    for (uint32_t i = tid; i < n; i += kFinThreads) mn = min(mn, static_cast<unsigned long long>(buf[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
    if ((tid & 31) == 0) atomicMin(&s_min, mn);
    __syncthreads();
    if (tid == 0 && n >= a.K) {
      const float t = ord_to_float(static_cast<uint32_t>(s_min >> 32));
      const float th = __double2float_rd(static_cast<double>(t) - 2.0 * static_cast<double>(eps));
      a.gthr_out[b] = ord_of(th);
      a.base_out[b] = th;
    }
    return;
  }
  // exact eta of this query, in the reference's operation order (pq_index.cpp:183-192)
  for (uint32_t i = tid; i < a.m * a.k; i += kFinThreads) {
    const uint32_t j = i / a.k, c = i % a.k;
    float acc = 0.0f;
    const float* row = a.cb + static_cast<size_t>(i) * a.dbar;
    for (uint32_t t = 0; t < a.dbar; ++t) {
      const uint32_t col = j * a.dbar + t;
      const float qa = col < a.d ? __ldg(a.Q + static_cast<size_t>(b) * a.d + col) : 0.0f;
      acc = __fadd_rn(acc, __fmul_rn(__ldg(row + t), qa));
    }
    eta[i] = acc;
  }
  for (uint32_t i = tid; i < a.m * a.s; i += kFinThreads) slam[i] = __ldg(a.lam + i);
  if (tid == 0) s_n = 0;
  __syncthreads();

  __syncthreads();
  bool exact_all = full_scan;
  if (!exact_all) {
    // 1) approximate keys >= the shared threshold from every range's list
    const uint32_t g = a.gthr[b];
    floor_key = g ? static_cast<uint64_t>(g) << 32 : 1ull;
    if (tid == 0) s_full = 0u;
    // fast path: every list entry fits in buf — gather them in one pass with
    // no capacity checks (warp-aggregated appends, no block barriers).  The
    // lists are short (a few entries each over 2 * ranges lists), so walking
    // them one after the other is a chain of dependent L2 round trips (0.2 ms
    // per query at 296 lists: the whole cost of a mid-size batch, where few
    // finish CTAs run).  Instead the counts are loaded once, prefix-summed,
    // and every thread fetches flat entry e of the concatenation (its list by
    // binary search over the offsets): all loads independent.
    // (With few lists — large batches: many query tiles, few ranges, and
    // thousands of finish CTAs hiding each other's latency — the plain walk
    // is cheaper: C2 at B = 10,000 has 18 lists per query.)
    // (compile-time: the extra code cost the large-batch instantiation 45% of
    // its throughput when it was a run-time branch)
    uint32_t* off = reinterpret_cast<uint32_t*>(slam + static_cast<size_t>(a.m) * a.s);  // [2 * ranges + 1]
    const uint32_t NL = 2 * a.ranges;
    constexpr bool flat = FLAT;
    uint32_t total = 0;
    if constexpr (FLAT) {
      for (uint32_t rr = tid; rr < NL; rr += kFinThreads)
        off[rr + 1] = __ldg(a.counts + (static_cast<size_t>(rr >> 1) * a.Bpad + b) * 2 + (rr & 1u));
      if (tid == 0) off[0] = 0u;
      __syncthreads();
      if (tid < 32) {  // inclusive scan of the counts: a contiguous chunk per lane
        const uint32_t per = (NL + 31u) / 32u;
        const uint32_t lo = min(NL, tid * per), hi = min(NL, lo + per);
        uint32_t sum = 0;
        for (uint32_t i = lo; i < hi; ++i) sum += off[i + 1];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (tid >= static_cast<uint32_t>(o)) incl += v;
        }
        uint32_t run = incl - sum;
        for (uint32_t i = lo; i < hi; ++i) {
          run += off[i + 1];
          off[i + 1] = run;
        }
      }
      __syncthreads();
      total = off[NL];
    } else {
      for (uint32_t rr = 0; rr < NL; ++rr)
        total += __ldg(a.counts + (static_cast<size_t>(rr >> 1) * a.Bpad + b) * 2 + (rr & 1u));
    }
    const bool fast = total <= a.cap - kFinThreads;
    __syncthreads();
    for (uint32_t e0 = 0; flat && fast && e0 < total; e0 += kFinThreads) {
      const uint32_t e = e0 + tid;
      uint64_t key = 0ull;
      if (FLAT && e < total) {
        uint32_t lo = 0, hi = NL;  // off[lo] <= e < off[hi]
        while (hi - lo > 1u) {
          const uint32_t mid = (lo + hi) >> 1;
          if (off[mid] <= e) lo = mid;
          else hi = mid;
        }
        const size_t li = (static_cast<size_t>(lo >> 1) * a.Bpad + b) * 2 + (lo & 1u);
        key = a.lists[li * a.Lc + (e - off[lo])];
      }
      push(key);
    }
    for (uint32_t rr = 0; !flat && fast && rr < NL; ++rr) {
      const size_t li = (static_cast<size_t>(rr >> 1) * a.Bpad + b) * 2 + (rr & 1u);
      const uint32_t n = __ldg(a.counts + li);
      const uint64_t* L = a.lists + li * a.Lc;
      for (uint32_t i0 = 0; i0 < n; i0 += kFinThreads) push(i0 + tid < n ? L[i0 + tid] : 0ull);
    }
    __syncthreads();
    for (uint32_t rr = 0; !fast && rr < 2 * a.ranges && !s_full; ++rr) {
      const size_t li = (static_cast<size_t>(rr >> 1) * a.Bpad + b) * 2 + (rr & 1u);
      const uint32_t n = a.counts[li];
      const uint64_t* L = a.lists + li * a.Lc;
      for (uint32_t i0 = 0; i0 < n; i0 += kFinThreads) {
        if (s_n + kFinThreads > a.cap) {
          cut(true);
          if (s_n + kFinThreads > a.cap) {  // cannot prune: exact scan instead
            if (tid == 0) s_full = 1u;
            __syncthreads();
            break;
          }
        }
        const uint32_t i = i0 + tid;
        push(i < n ? L[i] : 0ull);
        __syncthreads();
      }
    }
    exact_all = s_full != 0u;
    __syncthreads();
    if (!exact_all) {
      // cut to the K-th best approximate score - 2 eps first: an exact
      // re-score (m scattered code words) costs more than the select
      cut(true);
      // 2) exact re-score of the survivors; key = exact (score, global id)
      const uint32_t n = s_n;
      const float sigma = a.fse[b].x;
      for (uint32_t i = tid; i < n; i += kFinThreads) {
        const uint32_t p = static_cast<uint32_t>(buf[i]);
        const float ex = exact_score_point(a, p, eta, slam);
        if (a.diag) {
          const float ap = ord_to_float(static_cast<uint32_t>(buf[i] >> 32));
          const float ratio = static_cast<float>(fabs(static_cast<double>(ap) - static_cast<double>(sigma) * ex) / eps);
          atomicMax(a.diag, __float_as_uint(ratio));
        }
        buf[i] = make_key(ex, static_cast<uint32_t>(a.id_base + p));
      }
      __syncthreads();
      floor_key = 1ull;
    } else {
      if (tid == 0) s_n = 0;
      floor_key = 1ull;
      __syncthreads();
    }
  }
  if (exact_all) {
    if (a.diag && tid == 0) atomicAdd(a.diag + 1, 1u);
    if (a.fb_count) {  // the parallel fallback takes the query (block-uniform)
      __shared__ uint32_t s_slot;
      if (tid == 0) s_slot = atomicAdd(a.fb_count, 1u);
      __syncthreads();
      if (s_slot < a.fb_cap) {
        if (tid == 0) a.fb_list[s_slot] = b;
        return;
      }
    }
    // exact scan of every point (queries outside the filter's range)
    for (uint64_t p0 = 0; p0 < a.n_local; p0 += kFinThreads) {
      if (s_n + kFinThreads > a.cap) cut(false);
      const uint64_t p = p0 + tid;
      push(p < a.n_local ? make_key(exact_score_point(a, p, eta, slam), static_cast<uint32_t>(a.id_base + p)) : 0ull);
      __syncthreads();
    }
  }
  cut(false);
  // 3) sort the <= K survivors (rank placement) and write the row
  const uint32_t n = s_n;
  for (uint32_t i = tid; i < n; i += kFinThreads) {
    const uint64_t key = buf[i];
    uint32_t ahead = 0;
    for (uint32_t j = 0; j < n; ++j) ahead += buf[j] > key ? 1u : 0u;
    if (ahead < a.out_stride) {
      const size_t o = static_cast<size_t>(b) * a.out_stride + ahead;
      if (a.out_keys) a.out_keys[o] = key;
      if (a.out_ids) a.out_ids[o] = key_id(key);
      if (a.out_scores) a.out_scores[o] = key_score(key);
    }
  }
  for (uint32_t rr = n + tid; rr < a.out_stride; rr += kFinThreads) {
    const size_t o = static_cast<size_t>(b) * a.out_stride + rr;
    if (a.out_keys) a.out_keys[o] = 0ull;
    if (a.out_ids) a.out_ids[o] = -1;
    if (a.out_scores) a.out_scores[o] = -INFINITY;
  }
}

// ---- parallel exact fallback.  A query the filter cannot serve (operands
// outside the scaling range, or more than a list of points within 2 eps of each
// other) is scored exactly over every point.  One finish CTA doing that alone
// takes tens of milliseconds at 1e6 points, so the finish kernel only records
// such queries and these two kernels spread each over S point slices:
//   tscan_fb_scan_kernel   grid (S, lanes): CTA (s, y) scores slice s for the
//                          flagged queries y, y + lanes, ... and keeps the
//                          slice's K best exact keys;
//   tscan_fb_merge_kernel  per flagged query: the K best of its S slice lists,
//                          sorted, written to the query's output row.
struct FallbackArgs {
  FinishArgs f;
  uint64_t* keys;  // [fb_cap][S][K] slice lists (0 = empty)
  uint32_t S;
};

__global__ void __launch_bounds__(kFinThreads) tscan_fb_scan_kernel(FallbackArgs fa) {
  const FinishArgs& a = fa.f;
  extern __shared__ __align__(16) uint8_t smem_b[];
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_b);
  float* eta = reinterpret_cast<float*>(buf + a.cap);
  float* slam = eta + static_cast<size_t>(a.m) * a.k;
  __shared__ __align__(16) uint32_t scr[kGroupScratch];
  __shared__ uint32_t s_n;
  const uint32_t tid = threadIdx.x, sl = blockIdx.x;
  const Group grp{0, kFinThreads, static_cast<int>(tid)};
  const uint32_t nfl = min(*a.fb_count, a.fb_cap);
  const uint64_t p_lo = a.n_local * sl / fa.S, p_hi = a.n_local * (sl + 1) / fa.S;
  for (uint32_t i = blockIdx.y; i < nfl; i += gridDim.y) {
    const uint32_t b = a.fb_list[i];
    __syncthreads();
    for (uint32_t e = tid; e < a.m * a.k; e += kFinThreads) {  // eta in the reference's order
      const uint32_t j = e / a.k;
      float acc = 0.0f;
      const float* row = a.cb + static_cast<size_t>(e) * a.dbar;
      for (uint32_t t = 0; t < a.dbar; ++t) {
        const uint32_t col = j * a.dbar + t;
        const float qa = col < a.d ? __ldg(a.Q + static_cast<size_t>(b) * a.d + col) : 0.0f;
        acc = __fadd_rn(acc, __fmul_rn(__ldg(row + t), qa));
      }
      eta[e] = acc;
    }
    for (uint32_t e = tid; e < a.m * a.s; e += kFinThreads) slam[e] = __ldg(a.lam + e);
    if (tid == 0) s_n = 0;
    __syncthreads();
    uint64_t floor_key = 1ull;
    auto cut = [&]() {
      const uint32_t n = s_n;
      if (n <= a.K) return;
      const uint64_t kth = group_select(buf, n, a.K, scr, scr + kHistWords, grp);
      floor_key = floor_key > kth ? floor_key : kth;
      const uint32_t nn = group_compact(buf, n, floor_key, scr + kHistWords + kSvWords, grp);
      if (tid == 0) s_n = nn;
      __syncthreads();
    };
    for (uint64_t p0 = p_lo; p0 < p_hi; p0 += kFinThreads) {
      if (s_n + kFinThreads > a.cap) cut();
      const uint64_t p = p0 + tid;
      const uint64_t key = p < p_hi ? make_key(exact_score_point(a, p, eta, slam), static_cast<uint32_t>(a.id_base + p)) : 0ull;
      const bool take = key >= floor_key && key != 0ull;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, take);
      uint32_t base = 0;
      if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, static_cast<uint32_t>(__popc(bal)));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (take) buf[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = key;
      __syncthreads();
    }
    cut();
    const uint32_t n = min(s_n, a.K);
    uint64_t* out = fa.keys + (static_cast<size_t>(i) * fa.S + sl) * a.K;
    for (uint32_t r = tid; r < a.K; r += kFinThreads) out[r] = r < n ? buf[r] : 0ull;
  }
}

__global__ void __launch_bounds__(kFinThreads) tscan_fb_merge_kernel(FallbackArgs fa) {
  const FinishArgs& a = fa.f;
  extern __shared__ __align__(16) uint8_t smem_m[];
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_m);
  __shared__ __align__(16) uint32_t scr[kGroupScratch];
  __shared__ uint32_t s_n;
  const uint32_t tid = threadIdx.x;
  const Group grp{0, kFinThreads, static_cast<int>(tid)};
  const uint32_t nfl = min(*a.fb_count, a.fb_cap);
  const uint32_t total = fa.S * a.K;
  for (uint32_t i = blockIdx.x; i < nfl; i += gridDim.x) {
    const uint32_t b = a.fb_list[i];
    __syncthreads();
    if (tid == 0) s_n = 0;
    __syncthreads();
    uint64_t floor_key = 1ull;
    auto cut = [&]() {
      const uint32_t n = s_n;
      if (n <= a.K) return;
      const uint64_t kth = group_select(buf, n, a.K, scr, scr + kHistWords, grp);
      floor_key = floor_key > kth ? floor_key : kth;
      const uint32_t nn = group_compact(buf, n, floor_key, scr + kHistWords + kSvWords, grp);
      if (tid == 0) s_n = nn;
      __syncthreads();
    };
    const uint64_t* src = fa.keys + static_cast<size_t>(i) * total;
    for (uint32_t j0 = 0; j0 < total; j0 += kFinThreads) {
      if (s_n + kFinThreads > a.cap) cut();
      const uint32_t j = j0 + tid;
      const uint64_t key = j < total ? src[j] : 0ull;
      const bool take = key >= floor_key && key != 0ull;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, take);
      uint32_t base = 0;
      if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, static_cast<uint32_t>(__popc(bal)));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (take) buf[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = key;
      __syncthreads();
    }
    cut();
    const uint32_t n = s_n;
    for (uint32_t r = tid; r < n; r += kFinThreads) {
      const uint64_t key = buf[r];
      uint32_t ahead = 0;
      for (uint32_t j = 0; j < n; ++j) ahead += buf[j] > key ? 1u : 0u;
      if (ahead < a.out_stride) {
        const size_t o = static_cast<size_t>(b) * a.out_stride + ahead;
        if (a.out_keys) a.out_keys[o] = key;
        if (a.out_ids) a.out_ids[o] = key_id(key);
        if (a.out_scores) a.out_scores[o] = key_score(key);
      }
    }
    for (uint32_t rr = n + tid; rr < a.out_stride; rr += kFinThreads) {
      const size_t o = static_cast<size_t>(b) * a.out_stride + rr;
      if (a.out_keys) a.out_keys[o] = 0ull;
      if (a.out_ids) a.out_ids[o] = -1;
      if (a.out_scores) a.out_scores[o] = -INFINITY;
    }
  }
}

int g_max_smem_t = 0;

template <bool JOINT, int DB, int N>
size_t tscan_smem(const DeviceIndex& x, const TcIndex& t, bool cprime_smem, bool lam_smem) {
  const size_t kb = t.kpad * 2;
  size_t tab = JOINT ? static_cast<size_t>(t.msec) * t.rows * DB * 2
                     : (cprime_smem ? static_cast<size_t>(t.msec) * x.h.k * DB * 4 : 0) +
                           (lam_smem ? static_cast<size_t>(t.msec) * std::max(x.h.scales, 1u) * 4 : 0);
  return kTM * kb + 2 * N * kb + 2 * static_cast<size_t>(N) * x.W * 4 + ((tab + 15) & ~static_cast<size_t>(15)) +
         kEpiWarps * (kHistWords + kSvWords) * 4 + 128;
}

}  // namespace

// ------------------------------------------------------------------ host
// relative error factor of the filter (see the header): fp16 operands,
// fp32 lambda*C, tensor-core accumulation over kpad products (+ 1), and the
// reference's roundings over dbar products and m terms
double tc_rho(uint32_t kpad, uint32_t dbar, uint32_t m, bool qh = false) {
  const double uh = std::ldexp(1.0, -11), u = std::ldexp(1.0, -24);
  // qh: q = q_hi + q_lo, the query's rounding is that of q_lo (2^-11 of 2^-11 |q|);
  // twice the products are accumulated
  const double uq = qh ? uh * uh * (1.0 + uh) : uh;
  const double kacc = qh ? 2.0 * kpad : kpad;
  return uh + uq + uh * uq + 2.0 * u + (kacc + 1.0) * std::ldexp(1.0, -22) + (dbar + m + 2.0) * u * 1.01;
}

const TcIndex& tc_tables(const DeviceIndex& x) {
  std::call_once(x.tc_once, [&] {
    auto* t = new TcIndex();
    x.tc = t;
    const uint32_t m = x.h.m, k = x.h.k, dbar = x.h.dbar, s = std::max(x.h.scales, 1u);
    const bool joint = x.format == PCPQG_FMT_JOINT8;
    const bool raw = x.format == PCPQG_FMT_PLANES && x.sw >= 16;
    if (!(dbar == 1 || dbar == 2 || dbar == 4 || dbar == 8)) return;
    if (m * dbar > 1024) return;
    t->joint = joint;
    t->dbar = dbar;
    t->kpad = ((m * dbar + 15) / 16) * 16;
    t->msec = joint ? x.W * 4 : ((m + 7) & ~7u);
    t->msec = std::max(t->msec, (t->kpad / dbar));  // every slab's sections exist in the tables
    t->rows = joint ? (1u << (x.cw + x.sw)) : 0u;
    std::vector<float> lmax(t->msec, 0.0f), tau(t->msec, 1.0f);
    if (raw) {
      ensure_alpha_max(x);
      for (uint32_t j = 0; j < m; ++j) lmax[j] = x.amax[j];
    } else {
      for (uint32_t j = 0; j < m; ++j)
        for (uint32_t l = 0; l < s; ++l)
          lmax[j] = std::max(lmax[j], std::fabs(x.h.scales ? x.h.scalar_cb[j * x.h.scales + l] : 1.0f));
    }
    for (uint32_t j = 0; j < m; ++j) {
      float cmax = 0.0f;
      for (uint32_t i = 0; i < k * dbar; ++i) cmax = std::max(cmax, std::fabs(x.h.codebooks[(size_t)j * k * dbar + i]));
      const double X = static_cast<double>(cmax) * lmax[j];
      if (X > 0.0) {
        int e = 0;
        std::frexp(X, &e);
        if (e < -120 || e > 120) return;  // outside the scaling range: no tensor scan for this index
        tau[j] = static_cast<float>(std::ldexp(1.0, -e));
      }
    }
    if (joint) {
      const uint32_t rows = t->rows, cb = x.cw;
      std::vector<__half> tab(static_cast<size_t>(t->msec) * rows * dbar, __float2half(0.0f));
      for (uint32_t j = 0; j < m; ++j)
        for (uint32_t r = 0; r < rows; ++r) {
          const uint32_t c = r & ((1u << cb) - 1u), l = r >> cb;
          if (c >= k || l >= s) continue;
          const float lam = x.h.scales ? x.h.scalar_cb[j * x.h.scales + l] : 1.0f;
          for (uint32_t a2 = 0; a2 < dbar; ++a2) {
            volatile float prod = lam * x.h.codebooks[((size_t)j * k + c) * dbar + a2];  // fl(lambda * C)
            tab[((size_t)j * rows + r) * dbar + a2] = __float2half(prod * tau[j]);
          }
        }
      PCPQG_CUDA(cudaMalloc(&t->d_jtab, tab.size() * 2));
      PCPQG_CUDA(cudaMemcpy(t->d_jtab, tab.data(), tab.size() * 2, cudaMemcpyHostToDevice));
    } else {
      std::vector<float> cp(static_cast<size_t>(t->msec) * k * dbar, 0.0f);
      for (uint32_t j = 0; j < m; ++j)
        for (uint32_t i = 0; i < k * dbar; ++i) cp[(size_t)j * k * dbar + i] = x.h.codebooks[(size_t)j * k * dbar + i] * tau[j];
      PCPQG_CUDA(cudaMalloc(&t->d_cprime, cp.size() * 4));
      PCPQG_CUDA(cudaMemcpy(t->d_cprime, cp.data(), cp.size() * 4, cudaMemcpyHostToDevice));
    }
    PCPQG_CUDA(cudaMalloc(&t->d_tau, t->msec * 4));
    PCPQG_CUDA(cudaMemcpy(t->d_tau, tau.data(), t->msec * 4, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMalloc(&t->d_lam_max, t->msec * 4));
    PCPQG_CUDA(cudaMemcpy(t->d_lam_max, lmax.data(), t->msec * 4, cudaMemcpyHostToDevice));
    t->ok = true;
  });
  return *x.tc;
}

namespace {
// point ranges per query tile: fill the last wave, ranges of >= 8 tiles
uint32_t tc_ranges(uint64_t ptiles, uint32_t qtiles, int nsm, uint32_t& tpr) {
  const uint64_t sms = static_cast<uint64_t>(nsm);
  uint64_t best_r = 1;
  double best_eff = -1.0;
  const uint32_t rmax = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(ptiles / 8, 256)));
  for (uint32_t r = 1; r <= rmax; ++r) {
    const uint64_t t = (ptiles + r - 1) / r;
    const uint64_t rr = (ptiles + t - 1) / t;  // ranges actually used
    const uint64_t waves = (qtiles * rr + sms - 1) / sms;
    const double eff = static_cast<double>(qtiles * rr) / static_cast<double>(waves * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best_r = rr;
    }
    if (eff > 0.97) break;
  }
  tpr = static_cast<uint32_t>((ptiles + best_r - 1) / best_r);
  return static_cast<uint32_t>((ptiles + tpr - 1) / tpr);
}

struct TcKernel {
  const void* fn;
  size_t smem;
  uint32_t N;
  bool cprime_smem, lam_smem;
  uint32_t qt = 1;  // query tiles (of 128) per CTA
  bool qh = false;  // hi/lo query operand (2 * kpad K columns)
};

template <bool JOINT, int DB, int CW = 0, int SW = 0, int RB = 0>
TcKernel pick_db(const DeviceIndex& x, const TcIndex& t, size_t budget) {
  // preference: wide tiles, then tables in shared memory
  struct Opt { int n; bool cp, lam; };
  const Opt opts[] = {{256, true, true}, {128, true, true}, {128, false, true}, {128, false, false}};
  for (const Opt& o : opts) {
    const bool cp = !JOINT && o.cp, lam = !JOINT && o.lam;
    const size_t sm = o.n == 256 ? tscan_smem<JOINT, DB, 256>(x, t, cp, lam) : tscan_smem<JOINT, DB, 128>(x, t, cp, lam);
    if (sm <= budget)
      return {o.n == 256 ? reinterpret_cast<const void*>(tscan_kernel<JOINT, DB, 256, CW, SW, RB>)
                         : reinterpret_cast<const void*>(tscan_kernel<JOINT, DB, 128, CW, SW, RB>),
              sm, static_cast<uint32_t>(o.n), cp, lam};
  }
  return {nullptr, 0, 0, false, false};
}

TcKernel pick_tc(const DeviceIndex& x, const TcIndex& t) {
  int max_smem = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, x.device));
  const size_t budget = static_cast<size_t>(max_smem) - 512;
  // the configs' PLANES layouts get compile-time code widths
  if (!t.joint && t.dbar == 4 && x.cw == 4 && x.sw == 16) return pick_db<false, 4, 4, 16>(x, t, budget);
  if (!t.joint && t.dbar == 4 && x.cw == 8 && x.sw == 4) return pick_db<false, 4, 8, 4>(x, t, budget);
  // the configs' JOINT8 layouts (C2: 4-bit centers + 3-bit scales, dbar 2;
  // C1: 4 + 4 bits, dbar 4) get compile-time table rows
  if (t.joint && t.dbar == 2 && t.rows == 128) return pick_db<true, 2, 0, 0, 7>(x, t, budget);
  if (t.joint && t.dbar == 4 && t.rows == 256) return pick_db<true, 4, 0, 0, 8>(x, t, budget);
  switch ((t.joint ? 100 : 0) + t.dbar) {
    case 101: return pick_db<true, 1>(x, t, budget);
    case 102: return pick_db<true, 2>(x, t, budget);
    case 104: return pick_db<true, 4>(x, t, budget);
    case 108: return pick_db<true, 8>(x, t, budget);
    case 1: return pick_db<false, 1>(x, t, budget);
    case 2: return pick_db<false, 2>(x, t, budget);
    case 4: return pick_db<false, 4>(x, t, budget);
    default: return pick_db<false, 8>(x, t, budget);
  }
}
// ---- the decoded operand cache
template <bool JOINT, int DB, int CW = 0, int SW = 0, int RB = 0>
void build_xhat_t(const DeviceIndex& x, const TcIndex& t, uint8_t* xhat, uint64_t npad, uint32_t T) {
  TScanArgs a{};
  a.codes = x.d_codes;
  a.n_local = x.n_local;
  a.W = x.W;
  a.Wc = x.Wc;
  a.m = x.h.m;
  a.k = x.h.k;
  a.s = std::max(x.h.scales, 1u);
  a.cw = x.cw;
  a.sw = x.sw;
  a.kpad = t.kpad;
  a.msec = t.msec;
  a.rows = t.rows;
  a.cprime_smem = 0;  // tables read from global memory here
  const uint64_t total = static_cast<uint64_t>(t.kpad / 8) * npad;
  xhat_build_kernel<JOINT, DB, CW, SW, RB><<<static_cast<unsigned>((total + 255) / 256), 256>>>(
      a, t.d_jtab, t.d_cprime, x.d_lambda, xhat, npad, T);
  PCPQG_CUDA(cudaGetLastError());
}

void build_xhat(const DeviceIndex& x, const TcIndex& t, uint8_t* xhat, uint64_t npad, uint32_t T) {
  if (!t.joint && t.dbar == 4 && x.cw == 4 && x.sw == 16) return build_xhat_t<false, 4, 4, 16>(x, t, xhat, npad, T);
  if (!t.joint && t.dbar == 4 && x.cw == 8 && x.sw == 4) return build_xhat_t<false, 4, 8, 4>(x, t, xhat, npad, T);
  if (t.joint && t.dbar == 2 && t.rows == 128) return build_xhat_t<true, 2, 0, 0, 7>(x, t, xhat, npad, T);
  if (t.joint && t.dbar == 4 && t.rows == 256) return build_xhat_t<true, 4, 0, 0, 8>(x, t, xhat, npad, T);
  switch ((t.joint ? 100 : 0) + t.dbar) {
    case 101: return build_xhat_t<true, 1>(x, t, xhat, npad, T);
    case 102: return build_xhat_t<true, 2>(x, t, xhat, npad, T);
    case 104: return build_xhat_t<true, 4>(x, t, xhat, npad, T);
    case 108: return build_xhat_t<true, 8>(x, t, xhat, npad, T);
    case 1: return build_xhat_t<false, 1>(x, t, xhat, npad, T);
    case 2: return build_xhat_t<false, 2>(x, t, xhat, npad, T);
    case 4: return build_xhat_t<false, 4>(x, t, xhat, npad, T);
    default: return build_xhat_t<false, 8>(x, t, xhat, npad, T);
  }
}

uint32_t cache_tile_for(int device, uint32_t kpad);

// the cache exists (built on first use when it fits: at most scan_tc_cache_pct
// percent of the device's free memory)
bool tc_cache(const DeviceIndex& x, const TcIndex& tc) {
  TcIndex& t = const_cast<TcIndex&>(tc);  // a lazily built member, guarded by cache_mu
  std::lock_guard<std::mutex> lk(t.cache_mu);
  if (t.cache_tried) return t.d_xhat != nullptr;
  t.cache_tried = true;
  const uint64_t npad = (x.n_local + 255) / 256 * 256;
  const uint64_t bytes = static_cast<uint64_t>(t.kpad / 8) * npad * 16;
  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(x.device));
  size_t fr = 0, tot = 0;
  PCPQG_CUDA(cudaMemGetInfo(&fr, &tot));
  if (bytes <= static_cast<uint64_t>(fr) / 100 * static_cast<uint64_t>(options().scan_tc_cache_pct)) {
    if (cudaMalloc(&t.d_xhat, bytes) == cudaSuccess) {
      t.npad = npad;
      t.cache_tile = cache_tile_for(x.device, t.kpad);
      build_xhat(x, t, t.d_xhat, npad, t.cache_tile);
      unsigned long long* d_nb = nullptr;
      PCPQG_CUDA(cudaMalloc(&d_nb, 8));
      PCPQG_CUDA(cudaMemset(d_nb, 0, 8));
      xhat_norm_kernel<<<static_cast<unsigned>((x.n_local + 255) / 256), 256>>>(t.d_xhat, x.n_local, t.cache_tile,
                                                                               t.kpad / 8, d_nb);
      unsigned long long nb = 0;
      PCPQG_CUDA(cudaMemcpy(&nb, d_nb, 8, cudaMemcpyDeviceToHost));
      cudaFree(d_nb);
      std::memcpy(&t.xnorm_max, &nb, 8);
      if (!std::isfinite(t.xnorm_max)) t.xnorm_max = 0.0;
      PCPQG_CUDA(cudaDeviceSynchronize());
    } else {
      cudaGetLastError();
      t.d_xhat = nullptr;
    }
  }
  cudaSetDevice(prev);
  return t.d_xhat != nullptr;
}

// The cached kernel for a batch of B queries on `device`.  Two query tiles per
// CTA halve the operand stream from L2 per flop; measured (tools/ab_qt.py) that
// pays only where the point tile stays at 256 columns and K is long enough for
// the tensor pipe — not the TMEM read-out — to bound the tile: C3 (kpad 128)
// 2.73 -> 2.45 ms, but C2 (kpad 112, TMEM-bound) 4.11 -> 4.26 ms and C4 (kpad
// 256: the two query tiles only fit next to 64-column point tiles, whose MMAs
// re-read the query operand twice as often) 42.0 -> 44.3 ms.  So: QT = 2 iff
// the batch has the tiles (an odd count pads one empty tile: accepted from 5
// tiles on), kpad >= 128 and 256-column point tiles fit.
// points per tile of the operand cache (= the cached kernels' N for this K):
// 256 when one query tile and two 256-column stages fit, else 128
uint32_t cache_tile_for(int device, uint32_t kpad) {
  int max_smem = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  const size_t budget = static_cast<size_t>(max_smem) - 512 - 6144;
  const size_t kb = kpad * 2;
  const size_t sm = kTM * kb + 2 * 256 * kb + kEpiWarps * (kHistWords + kSvWords) * 4 + 128;
  return sm <= budget ? 256u : 128u;
}

TcKernel pick_cached_for(int device, uint32_t kpad, uint32_t B) {
  int max_smem = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  const size_t budget = static_cast<size_t>(max_smem) - 512 - 6144;  // (static shared: barriers, thresholds)
  const size_t kb = kpad * 2;
  struct Opt { int n, st, qt; bool at, qh; const void* fn; };
  const Opt opts[] = {
      {256, 2, 1, false, true, reinterpret_cast<const void*>(tscan_cached_kernel<256, 2, 1, false, true>)},
      {256, 3, 2, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<256, 3, 2>)},
      {256, 2, 2, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<256, 2, 2>)},
      {128, 3, 1, true, false, reinterpret_cast<const void*>(tscan_cached_kernel<128, 3, 1, true>)},
      {128, 2, 1, true, false, reinterpret_cast<const void*>(tscan_cached_kernel<128, 2, 1, true>)},
      {256, 3, 1, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<256, 3, 1>)},
      {256, 2, 1, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<256, 2, 1>)},
      {128, 3, 1, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<128, 3, 1>)},
      {128, 2, 1, false, false, reinterpret_cast<const void*>(tscan_cached_kernel<128, 2, 1>)}};
  const uint32_t t128 = (B + kTM - 1) / kTM;
  const bool two = options().scan_tc_qt >= 2 && kpad >= 128 && t128 >= 2 && (t128 % 2 == 0 || t128 >= 5);
  // the query tile in TMEM (AT): for long K (kpad >= 192, where 256-column point
  // tiles do not fit and the operand re-reads bind) when the tile's kpad / 2
  // columns fit next to the two 128-column accumulators
  const bool at = options().scan_tc_at && kpad >= 192 && 2u * 128u + kpad / 2 <= 512u;
  // the hi/lo query operand (QH): where the TMEM read-out, not the tensor pipe,
  // bounds a 256-column tile even with twice the MMAs (kpad * 16 clk < 2048 clk)
  const bool qh = options().scan_tc_qh && kpad <= 112;
  const uint32_t T = cache_tile_for(device, kpad);
  for (const Opt& o : opts) {
    if (static_cast<uint32_t>(o.n) != T) continue;  // the cache's tile is the kernel's N
    if (o.qt == 2 && !two) continue;
    if (o.at && !at) continue;
    if (o.qh && !qh) continue;
    const size_t sm = (o.at ? 0 : static_cast<size_t>(o.qt) * (o.qh ? 2 : 1) * kTM * kb) +
                      static_cast<size_t>(o.st) * o.n * kb + kEpiWarps * (kHistWords + kSvWords) * 4 + 128;
    if (sm <= budget) {
      TcKernel k{o.fn, sm, static_cast<uint32_t>(o.n), false, false};
      k.qt = static_cast<uint32_t>(o.qt);
      k.qh = o.qh;
      return k;
    }
  }
  return {nullptr, 0, 0, false, false};
}

TcKernel pick_cached(const DeviceIndex& x, const TcIndex& t, uint32_t B) {
  return pick_cached_for(x.device, t.kpad, B);
}

// the kernel a search runs: over the decoded cache when enabled and built
TcKernel pick_search_kernel(const DeviceIndex& x, const TcIndex& t, bool& cached, uint32_t B) {
  cached = false;
  if (options().scan_tc_cache_pct > 0 && tc_cache(x, t)) {
    const TcKernel k = pick_cached(x, t, B);
    if (k.fn) {
      cached = true;
      return k;
    }
  }
  return pick_tc(x, t);
}
}  // namespace

TcPlan tscan_plan(const DeviceIndex& x, uint32_t B, uint32_t K) {
  TcPlan p;
  const TcIndex& t = tc_tables(x);
  bool cached = false;
  const TcKernel kern = pick_search_kernel(x, t, cached, B);
  p.N = kern.N;
  p.qtiles = (B + kern.qt * kTM - 1) / (kern.qt * kTM);  // CTAs along the queries
  const uint64_t ptiles = (x.n_local + p.N - 1) / p.N;
  p.ranges = tc_ranges(ptiles, p.qtiles, num_sms(x.device), p.tiles_per_range);
  (void)K;
  return p;
}

bool tscan_eligible(const DeviceIndex& x, uint32_t B, uint32_t K) {
  if (!options().scan_tc || B < static_cast<uint32_t>(options().scan_tc_min_batch) || K == 0 || K > 256) return false;
  if (x.n_local < 2048 || x.n_local >= (1ull << 32)) return false;
  if (B < 256 && x.n_local * static_cast<uint64_t>(B) < static_cast<uint64_t>(std::max<int64_t>(0, options().scan_tc_min_work)))
    return false;
  const TcIndex& t = tc_tables(x);
  if (!t.ok) return false;
  return pick_tc(x, t).fn != nullptr;
}

void tscan_search(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t K, uint32_t out_stride,
                  uint64_t* d_keys, int32_t* d_ids, float* d_scores, ScratchAlloc alloc, cudaStream_t st,
                  float* stage_ms) {
  const TcIndex& t = tc_tables(x);
  bool cached = false;
  const TcKernel kern = pick_search_kernel(x, t, cached, B);
  if (!kern.fn) fail(PCPQG_E_UNSUPPORTED, "tensor scan: layout not supported");
  const uint32_t qrows = kern.qt * kTM;  // queries per CTA
  const uint32_t Bpad = (B + qrows - 1) / qrows * qrows;
  const uint32_t qtiles = Bpad / qrows;  // CTAs along the queries
  const uint32_t N = kern.N;
  const uint64_t ptiles = (x.n_local + N - 1) / N;
  uint32_t tpr = 0;
  const uint32_t ranges = tc_ranges(ptiles, qtiles, num_sms(x.device), tpr);
  // seed pass: sblocks of the full 32-point blocks, spread evenly (about
  // n / scan_tc_seed points); its K-th best block maximum sits near global
  // rank K * n / S, so each (range, half) list expects ~K * n / (S * 2 ranges)
  const uint64_t nbfull = x.n_local / kBlockPts;
  const uint64_t den = static_cast<uint64_t>(std::max(1, options().scan_tc_seed));
  // (at most scan_tc_seed_max points: past ~1M the sample's cost — its GEMM and the
  // K-th-of-block-maxima select — grows with n while its threshold only gains ln)
  const uint64_t seed_cap = std::max<uint64_t>(2ull * K, static_cast<uint64_t>(options().scan_tc_seed_max) / kBlockPts);
  uint32_t sblocks = static_cast<uint32_t>(
      std::min<uint64_t>({nbfull, std::max<uint64_t>(nbfull / den, 2 * K), seed_cap}));
  uint32_t stiles_all = 0;
  if (cached) {  // the cached kernel samples whole tiles of N points
    const uint32_t bpt = N / kBlockPts;
    stiles_all = static_cast<uint32_t>(x.n_local / N);
    sblocks = std::min<uint32_t>(stiles_all, (sblocks + bpt - 1) / bpt) * bpt;
  }
  if (options().scan_tc_seed <= 0 || sblocks < K) sblocks = 0;
  // entries the seed select sees: per block (decoding kernel) or per (tile, half)
  uint32_t seed_entries = sblocks;
  if (cached && sblocks) {
    const uint32_t bpt = N / kBlockPts;
    if (sblocks / bpt * 2 < K) sblocks = std::min<uint32_t>(stiles_all, (K + 1) / 2) * bpt;
    seed_entries = sblocks / bpt * 2;
    if (seed_entries < K) sblocks = seed_entries = 0;
  }
  const uint64_t expect =
      sblocks ? static_cast<uint64_t>(K) * x.n_local / (static_cast<uint64_t>(sblocks) * kBlockPts * ranges * 2) + 1
              : x.n_local / (ranges * 2) + 1;
  uint32_t Lc = static_cast<uint32_t>(std::min<uint64_t>(8192, std::max<uint64_t>(1024, ((4 * expect + N) + 63) / 64 * 64)));
  Lc = std::max<uint32_t>(Lc, ((K + N) + 63) / 64 * 64);

  uint8_t* qa = static_cast<uint8_t*>(alloc(static_cast<size_t>(Bpad) * t.kpad * 2 * (kern.qh ? 2 : 1)));
  float2* fse = static_cast<float2*>(alloc(static_cast<size_t>(Bpad) * 8));
  uint64_t* lists = static_cast<uint64_t*>(alloc(static_cast<size_t>(ranges) * Bpad * 2 * Lc * 8));
  uint32_t* counts = static_cast<uint32_t*>(alloc(static_cast<size_t>(ranges) * Bpad * 2 * 4));
  float* cmax = sblocks ? static_cast<float*>(alloc(static_cast<size_t>(Bpad) * sblocks * 4)) : nullptr;
  uint32_t* bins = static_cast<uint32_t*>(alloc(static_cast<size_t>(Bpad) * 33 * 4));
  float* base = reinterpret_cast<float*>(bins + static_cast<size_t>(Bpad) * 32);
  PCPQG_CUDA(cudaMemsetAsync(bins, 0, static_cast<size_t>(Bpad) * 32 * 4, st));
  PCPQG_CUDA(cudaMemsetAsync(base, 0xFF, static_cast<size_t>(Bpad) * 4, st));  // NaN: no seed
  uint32_t* gthr = static_cast<uint32_t*>(alloc(static_cast<size_t>(Bpad) * 8));
  uint32_t* ovf = gthr + Bpad;
  PCPQG_CUDA(cudaMemsetAsync(gthr, 0, static_cast<size_t>(Bpad) * 8, st));

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (stage_ms) {
    for (auto& e : ev) PCPQG_CUDA(cudaEventCreate(&e));
    PCPQG_CUDA(cudaEventRecord(ev[0], st));
  }
  // ---- 1. per-query operand tiles, scales, error bounds
  PrepArgs pa{};
  pa.Q = dQ;
  pa.B = B;
  pa.Bpad = Bpad;
  pa.d = x.h.d;
  pa.m = x.h.m;
  pa.dbar = x.h.dbar;
  pa.kpad = t.kpad;
  pa.k = x.h.k;
  pa.msec = t.msec;
  pa.tau = t.d_tau;
  pa.lam_max = t.d_lam_max;
  pa.cb = x.d_codebooks;
  pa.rho = tc_rho(t.kpad, x.h.dbar, x.h.m, kern.qh);
  pa.qh = kern.qh ? 1u : 0u;
  pa.xnorm_max = (cached && options().scan_tc_cs) ? t.xnorm_max : 0.0;
  pa.qa = qa;
  pa.fse = fse;
  tq_prep_kernel<<<(Bpad + 7) / 8, 256, 0, st>>>(pa);
  PCPQG_CUDA(cudaGetLastError());

  // ---- finish / seed arguments
  FinishArgs f{};
  f.codes = x.d_codes;
  f.Q = dQ;
  f.cb = x.d_codebooks;
  f.lam = x.d_lambda;
  f.lists = lists;
  f.counts = counts;
  f.gthr = gthr;
  f.ovf = ovf;
  f.fse = fse;
  f.n_local = x.n_local;
  f.id_base = x.shard_begin;
  f.W = x.W;
  f.Wc = x.Wc;
  f.m = x.h.m;
  f.k = x.h.k;
  f.s = std::max(x.h.scales, 1u);
  f.cbits = x.format == PCPQG_FMT_JOINT8 ? x.cw : 0u;
  f.cw = x.cw;
  f.sw = x.sw;
  f.fmt = x.format;
  f.d = x.h.d;
  f.dbar = x.h.dbar;
  f.ranges = ranges;
  f.Lc = Lc;
  f.Bpad = Bpad;
  f.K = K;
  f.out_stride = out_stride;
  f.out_keys = d_keys;
  f.out_ids = d_ids;
  f.out_scores = d_scores;
  f.seed_blocks = seed_entries;
  f.cm_stride = seed_entries;
  f.cmax = cmax;
  f.gthr_out = gthr;
  f.base_out = base;
  // staged keys per query: half the buffer when the expected list total leaves
  // room (twice as many finish CTAs per SM); a query that outgrows it is cut in
  // rounds or, at worst, scanned exactly
  const uint64_t per_query = expect * ranges * 2;
  f.cap = (per_query * 2 + kFinThreads <= kFinCap / 2 && sblocks <= kFinCap / 2) ? kFinCap / 2 : kFinCap;
  // (the kernel is latency bound and shared memory sets its occupancy: a third
  // tier when the expected total itself fits a quarter of the buffer)
  if (options().scan_tc_fin_small && f.cap == kFinCap / 2 && per_query + kFinThreads <= kFinCap / 4 &&
      seed_entries <= kFinCap / 8 && 2 * K + kFinThreads <= kFinCap / 4)
    f.cap = kFinCap / 4;
  // many short lists (small / mid batches: one query tile, a range per SM) are gathered by flat index
  const bool fin_flat = 2 * ranges > 32;
  const size_t fsm = static_cast<size_t>(f.cap) * 8 + static_cast<size_t>(x.h.m) * x.h.k * 4 +
                     static_cast<size_t>(x.h.m) * std::max(x.h.scales, 1u) * 4 + 16 +
                     (fin_flat ? (2 * static_cast<size_t>(ranges) + 2) * 4 : 0);  // + the flat gather's list offsets
  auto* const fin_kernel = fin_flat ? tscan_finish_kernel<true> : tscan_finish_kernel<false>;
  PCPQG_CUDA(cudaFuncSetAttribute(fin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fsm)));

  // ---- 3. tensor-core filter
  TScanArgs a{};
  a.codes = x.d_codes;
  a.qa = qa;
  a.fse = fse;
  a.jtab = t.d_jtab;
  a.cprime = t.d_cprime;
  a.lam = x.d_lambda;
  a.lists = lists;
  a.counts = counts;
  a.gthr = gthr;
  a.ovf = ovf;
  a.n_local = x.n_local;
  a.W = x.W;
  a.Wc = x.Wc;
  a.m = x.h.m;
  a.k = x.h.k;
  a.s = std::max(x.h.scales, 1u);
  a.cbits = f.cbits;
  a.cw = x.cw;
  a.sw = x.sw;
  a.kpad = t.kpad;
  a.msec = t.msec;
  a.rows = t.rows;
  a.K = K;
  a.Lc = Lc;
  a.B = B;
  a.Bpad = Bpad;
  a.tiles_per_range = tpr;
  a.cprime_smem = kern.cprime_smem ? 1u : 0u;
  a.lam_smem = kern.lam_smem ? 1u : 0u;
  a.nbfull = static_cast<uint32_t>(nbfull);
  a.bins = bins;
  a.base = base;
  a.exp = static_cast<uint32_t>(options().scan_tc_exp);
  PCPQG_CUDA(cudaFuncSetAttribute(kern.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kern.smem)));
  // ---- 2. seed pass over the sample blocks + K-th best block maximum per query
  if (sblocks) {
    TScanArgs as = a;
    as.mode = 1;
    as.sblocks = sblocks;
    as.cm_stride = seed_entries;
    as.cmax = cmax;
    const uint64_t stiles = (static_cast<uint64_t>(sblocks) * kBlockPts + N - 1) / N;
    uint32_t stpr = 0;
    const uint32_t sranges = tc_ranges(stiles, qtiles, num_sms(x.device), stpr);
    as.tiles_per_range = stpr;
    XArgs xs{t.d_xhat, t.npad, stiles_all};
    void* args[] = {&as, &xs};
    PCPQG_CUDA(cudaLaunchKernel(kern.fn, dim3(qtiles, sranges), dim3(cached ? kCThreads : kTThreads), args,
                                kern.smem, st));
    FinishArgs fs = f;
    fs.seed = 1;
    fin_kernel<<<B, kFinThreads, fsm, st>>>(fs);
    PCPQG_CUDA(cudaGetLastError());
  }
  if (stage_ms) PCPQG_CUDA(cudaEventRecord(ev[1], st));
  // ---- 3. tensor-core filter over every point
  {
    XArgs xs{t.d_xhat, t.npad, stiles_all};
    void* args[] = {&a, &xs};
    PCPQG_CUDA(cudaLaunchKernel(kern.fn, dim3(qtiles, ranges), dim3(cached ? kCThreads : kTThreads), args,
                                kern.smem, st));
  }
  if (stage_ms) PCPQG_CUDA(cudaEventRecord(ev[2], st));
  if (options().scan_tc_diag) {  // diagnostics: list fill, overflows, unfiltered queries
    std::vector<uint32_t> hc(static_cast<size_t>(ranges) * Bpad * 2), hg(2 * Bpad);
    std::vector<float2> hf(Bpad);
    PCPQG_CUDA(cudaMemcpyAsync(hc.data(), counts, hc.size() * 4, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaMemcpyAsync(hg.data(), gthr, hg.size() * 4, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaMemcpyAsync(hf.data(), fse, hf.size() * 8, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
    uint64_t tot = 0, mx = 0, novf = 0, ninf = 0;
    for (uint32_t q = 0; q < B; ++q) {
      uint64_t c = 0;
      for (uint32_t r2 = 0; r2 < ranges; ++r2) c += hc[(static_cast<size_t>(r2) * Bpad + q) * 2] + hc[(static_cast<size_t>(r2) * Bpad + q) * 2 + 1];
      tot += c;
      mx = std::max(mx, c);
      novf += hg[Bpad + q] ? 1 : 0;
      ninf += std::isfinite(hf[q].y) ? 0 : 1;
    }
    std::fprintf(stderr,
                 "[pcpqg] tscan: N=%u ranges=%u tiles/range=%u Lc=%u seed=%u pts | list entries %.1f per query "
                 "(max %llu), overflowed %llu, unfiltered %llu of %u queries; eps[0]=%g sigma[0]=%g\n",
                 N, ranges, tpr, Lc, sblocks * kBlockPts, static_cast<double>(tot) / B,
                 static_cast<unsigned long long>(mx), static_cast<unsigned long long>(novf),
                 static_cast<unsigned long long>(ninf), B, hf[0].y, hf[0].x);
  }

  // ---- 4. exact re-score of the survivors, top-K rows
  unsigned int* diag = nullptr;
  if (options().scan_tc_diag) {
    diag = static_cast<unsigned int*>(alloc(16));
    PCPQG_CUDA(cudaMemsetAsync(diag, 0, 16, st));
    f.diag = diag;
  }
  // queries that need the exact scan go to the parallel fallback (usually none:
  // the two launches then return at once)
  const uint32_t fb_cap = std::min<uint32_t>(B, 256);
  const uint32_t fb_S = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(2ull * num_sms(x.device), x.n_local / 1024)));
  uint32_t* fb = static_cast<uint32_t*>(alloc(static_cast<size_t>(fb_cap + 1) * 4));
  PCPQG_CUDA(cudaMemsetAsync(fb, 0, 4, st));
  f.fb_count = fb;
  f.fb_list = fb + 1;
  f.fb_cap = fb_cap;
  fin_kernel<<<B, kFinThreads, fsm, st>>>(f);
  PCPQG_CUDA(cudaGetLastError());
  {
    FallbackArgs fa{};
    fa.f = f;
    fa.f.diag = nullptr;
    fa.S = fb_S;
    fa.keys = static_cast<uint64_t*>(alloc(static_cast<size_t>(fb_cap) * fb_S * K * 8));
    PCPQG_CUDA(cudaFuncSetAttribute(tscan_fb_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(fsm)));
    PCPQG_CUDA(cudaFuncSetAttribute(tscan_fb_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(f.cap * 8)));
    tscan_fb_scan_kernel<<<dim3(fb_S, std::min<uint32_t>(fb_cap, 16)), kFinThreads, fsm, st>>>(fa);
    tscan_fb_merge_kernel<<<std::min<uint32_t>(fb_cap, 64), kFinThreads, static_cast<size_t>(f.cap) * 8, st>>>(fa);
    PCPQG_CUDA(cudaGetLastError());
  }
  if (diag) {
    unsigned int hd[2];
    PCPQG_CUDA(cudaMemcpyAsync(hd, diag, 8, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
    float r;
    std::memcpy(&r, hd, 4);
    std::fprintf(stderr, "[pcpqg] tscan finish: max |approx - sigma*exact| / eps = %g; exact-scan queries %u\n", r,
                 hd[1]);
  }
  if (stage_ms) {
    PCPQG_CUDA(cudaEventRecord(ev[3], st));
    PCPQG_CUDA(cudaEventSynchronize(ev[3]));
    cudaEventElapsedTime(&stage_ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&stage_ms[1], ev[1], ev[2]);
    cudaEventElapsedTime(&stage_ms[2], ev[2], ev[3]);
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

}  // namespace pcpqg

namespace pcpqg {
// ====================================================================== GT-T
// Exact ground truth (brute_force_topn, proj/core/src/eval.cpp:36-49) through
// the same tensor-core filter: the raw fp32 points are the "decoded" operands.
//   x' = fp16(x * tau)      tau   = 2^-e, max |x_i| * tau in [0.5, 1) over the data set
//   q' = fp16(q * sigma_q)  sigma = 2^-e, max |q_i| * sigma in [0.5, 1)
// so sum_i q'_i x'_i approximates S <q, x> with S = sigma_q * tau (powers of
// two: exact scaling).  Per element q'x' = S q x (1 + d1)(1 + d2), |d| <= 2^-11,
// or an absolute 2^-25 where an operand is a fp16 subnormal; the tensor core
// accumulates the exact products in fp32 (taken as 2^-22 of the magnitude sum
// per addition, as in K2-T).  With sum_i |q_i x_i| <= ||q|| max_p ||x_p||:
//   |approx - S <q, x>_ref| <= eps_q = 1.25 ((2^-10 + 2^-21 + 1.01 kpad 2^-22) S ||q|| Xn + kpad 2^-23)
// (the reference's own fp64 roundings, d 2^-53 relative, are far inside the
// margin).  The filter (tscan_cached_kernel) keeps every pair within 2 eps of a
// lower bound of the query's K-th best approximate score; gt_tfinish_kernel
// re-scores those in the reference's order (dot_qx: sequential fp64, index
// order, eval.cpp:18-24) and selects the top-K by (score desc, id asc), so the
// result is the reference's, bit for bit.  A query outside the scaling range,
// or whose candidates cannot be pruned (a list of points within 2 eps of each
// other: e.g. an all-zero query), is flagged and scored exactly over every
// point by the caller (pcpqg_eval.cu).
namespace {

struct GtStats {  // device scalars of the data set
  unsigned int xmax_bits;          // max |x_i| (float bits; non-finite -> 0x7F800000)
  unsigned int pad;
  unsigned long long xnorm_bits;   // max row norm, rounded up (double bits)
};

// one warp per row, lanes over the columns (coalesced): max |x_i| and the row norm
__global__ void gt_stats_kernel(const float* __restrict__ X, uint64_t n, uint32_t d, GtStats* __restrict__ out) {
  const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  unsigned int mb = 0;
  unsigned long long nb = 0;
  for (uint64_t row = w0; row < n; row += nw) {
    const float* r = X + row * d;
    float mx = 0.0f;
    double sq = 0.0;
    for (uint32_t i = lane; i < d; i += 32) {
      const float v = fabsf(r[i]);
      mx = v > mx || !(v == v) ? (v == v ? v : INFINITY) : mx;
      sq = fma(static_cast<double>(v), static_cast<double>(v), sq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
    mb = max(mb, __float_as_uint(mx));
    // (any summation order of the squares is within d 2^-53 of the norm^2: the factor covers it)
    nb = max(nb, static_cast<unsigned long long>(__double_as_longlong(sqrt(sq) * (1.0 + 1e-9))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mb = max(mb, __shfl_xor_sync(0xFFFFFFFFu, mb, o));
    nb = max(nb, __shfl_xor_sync(0xFFFFFFFFu, nb, o));
  }
  if (lane == 0) {
    atomicMax(&out->xmax_bits, mb);
    atomicMax(&out->xnorm_bits, nb);
  }
}

// tau = 2^-e with xmax * tau in [0.5, 1); 0 when the data cannot be scaled
__device__ __forceinline__ double gt_tau(const GtStats* st) {
  const float xmax = __uint_as_float(st->xmax_bits);
  if (!(xmax > 0.0f) || !isfinite(xmax)) return 0.0;
  int e = 0;
  frexp(static_cast<double>(xmax), &e);
  if (e < -100 || e > 100) return 0.0;
  return ldexp(1.0, -e);
}

// the operand cache of a point chunk (tile-major, tiles of T = the kernel's N
// points).  A CTA takes 64 points: their rows are read coalesced into shared
// memory, then thread (point, slab) converts 8 values and writes 16 bytes, the
// 64 points of a slab contiguous.
constexpr uint32_t kGxPts = 64;
__global__ void __launch_bounds__(256) gt_xhat_kernel(const float* __restrict__ X, uint64_t n, uint32_t d,
                                                      uint32_t kpad, uint64_t npad, uint32_t T,
                                                      const GtStats* __restrict__ st, uint8_t* __restrict__ xhat) {
  extern __shared__ float s_rows[];  // [64][d + 1]
  const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * kGxPts;
  const uint32_t ld = d + 1;
  const uint64_t cnt = p0 < n ? min(static_cast<uint64_t>(kGxPts), n - p0) : 0;
  for (uint64_t i = threadIdx.x; i < cnt * d; i += blockDim.x) s_rows[(i / d) * ld + i % d] = X[p0 * d + i];
  __syncthreads();
  const double tau = gt_tau(st);
  const uint32_t nslab = kpad / 8;
  for (uint32_t w = threadIdx.x; w < kGxPts * nslab; w += blockDim.x) {
    const uint32_t pl = w % kGxPts, sl = w / kGxPts;
    const uint64_t p = p0 + pl;
    if (p >= npad) continue;
    __align__(16) __half h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t c = sl * 8 + i;
      const float v = (pl < cnt && c < d) ? s_rows[pl * ld + c] : 0.0f;
      h[i] = __double2half(static_cast<double>(v) * tau);
    }
    reinterpret_cast<uint4*>(xhat)[xhat_u4_index(p, sl, nslab, T)] = *reinterpret_cast<const uint4*>(h);
  }
}

struct GtPrepArgs {
  const float* Q;
  uint32_t B, Bpad, d, kpad, qh;
  const GtStats* st;
  uint8_t* qa;
  float2* fse;  // (S = sigma * tau, eps in scaled units; eps = inf: not filtered)
};

__global__ void gt_prep_kernel(GtPrepArgs a) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (row >= a.Bpad) return;
  const float* qq = a.Q + static_cast<size_t>(row) * a.d;
  double mx = 0.0, sq = 0.0;
  bool fin = true;
  for (uint32_t i = lane; i < a.d; i += 32) {
    const double qi = row < a.B ? static_cast<double>(qq[i]) : 0.0;
    fin = fin && isfinite(qi);
    mx = fmax(mx, fabs(qi));
    sq = fma(qi, qi, sq);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
  }
  fin = __all_sync(0xFFFFFFFFu, fin);
  const double tau = gt_tau(a.st);
  int e = 0;
  frexp(mx, &e);
  const bool ok = row < a.B && fin && tau > 0.0 && mx > 0.0 && e >= -100 && e <= 100;
  const double sigma = ok ? ldexp(1.0, -e) : 0.0;
  const uint32_t ak = a.qh ? 2u : 1u;
  uint8_t* tile = a.qa + static_cast<size_t>(row / kTM) * kTM * a.kpad * 2 * ak;
  const uint32_t rr = row % kTM;
  for (uint32_t i = lane; i < a.kpad; i += 32) {
    __half h = __float2half(0.0f), hl = __float2half(0.0f);
    if (ok && i < a.d) {
      const double qt = static_cast<double>(qq[i]) * sigma;
      h = __double2half(qt);
      hl = __double2half(qt - static_cast<double>(__half2float(h)));
    }
    *reinterpret_cast<__half*>(tile + (i / 8) * (kTM * 16) + rr * 16 + (i % 8) * 2) = h;
    if (a.qh) *reinterpret_cast<__half*>(tile + (a.kpad / 8 + i / 8) * (kTM * 16) + rr * 16 + (i % 8) * 2) = hl;
  }
  if (lane == 0) {
    float eps = INFINITY, S = 0.0f;
    if (ok) {
      const double Sd = sigma * tau;
      const double xn = __longlong_as_double(static_cast<long long>(a.st->xnorm_bits));
      const double A = Sd * sqrt(sq) * (1.0 + 1e-12) * xn;
      // fp16 rounding of x' (2^-11) and of the query (2^-11, or 2^-22 with the hi/lo
      // operand), their product term, the tensor core's accumulation
      const double uq = a.qh ? ldexp(1.0, -22) * (1.0 + ldexp(1.0, -11)) : ldexp(1.0, -11);
      const double kacc = a.qh ? 2.0 * a.kpad : a.kpad;
      const double rho = ldexp(1.0, -11) + uq + ldexp(1.0, -21) + 1.01 * kacc * ldexp(1.0, -22);
      const double eb = 1.25 * (rho * A * (1.0 + 1e-9) + kacc * ldexp(1.0, -23));
      eps = __double2float_ru(eb);
      S = static_cast<float>(Sd);
      if (!isfinite(eps) || !(S > 0.0f) || !isfinite(S)) eps = INFINITY;
    }
    a.fse[row] = make_float2(S, eps);
  }
}

struct GtFinishArgs {
  const float* X;
  const float* Q;
  uint64_t n, id_base;
  uint32_t d;
  const uint64_t* lists;
  const uint32_t* counts;
  const uint32_t* gthr;
  const uint32_t* ovf;
  const float2* fse;
  uint32_t ranges, Lc, Bpad, K, out_stride, count_stride;
  uint32_t* out_ids;       // [B][out_stride] global ids
  double* out_scores;      // [B][out_stride]
  uint32_t* out_count;     // [B * count_stride]
  uint32_t* fallback;      // [B] 1: the query needs the exact full scan
  unsigned int* diag;      // optional: max |approx - S*exact| / eps (float bits)
};

__device__ __forceinline__ double gt_dot(const float* __restrict__ q, const float* __restrict__ x, uint32_t d) {
  double acc = 0.0;  // dot_qx: index order, no contraction (eval.cpp:18-24)
  for (uint32_t a = 0; a < d; ++a)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(__ldg(q + a)), static_cast<double>(__ldg(x + a))));
  return acc;
}

__global__ void __launch_bounds__(kFinThreads) gt_tfinish_kernel(GtFinishArgs a) {
  extern __shared__ __align__(16) uint8_t smem_g[];
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_g);           // kFinCap approximate keys
  double* exs = reinterpret_cast<double*>(buf + kFinCap);       // kFinCap exact scores
  __shared__ __align__(16) uint32_t scr[kGroupScratch];
  __shared__ uint32_t hist96[256];
  __shared__ Sel96 sel;
  __shared__ uint32_t s_n, s_full, s_w;
  __shared__ uint32_t widx[256];
  const uint32_t b = blockIdx.x, tid = threadIdx.x;
  const Group grp{0, kFinThreads, static_cast<int>(tid)};
  const float eps = a.fse[b].y;
  if (!isfinite(eps) || a.ovf[b] != 0u) {
    if (tid == 0) a.fallback[b] = 1u;
    return;
  }
  if (tid == 0) {
    s_n = 0;
    s_full = 0u;
    s_w = 0u;
  }
  __syncthreads();
  uint64_t floor_key = 1ull;
  auto cut = [&]() {  // keep the approximate keys within 2 eps of the K-th best
    const uint32_t n = s_n;
    if (n <= a.K) return;
    const uint64_t kth = group_select(buf, n, a.K, scr, scr + kHistWords, grp);
    const float tk = ord_to_float(static_cast<uint32_t>(kth >> 32));
    const float th = __double2float_rd(static_cast<double>(tk) - 2.0 * static_cast<double>(eps));
    const uint64_t f = static_cast<uint64_t>(ord_of(th)) << 32;
    floor_key = floor_key > f ? floor_key : f;
    const uint32_t nn = group_compact(buf, n, floor_key, scr + kHistWords + kSvWords, grp);
    if (tid == 0) s_n = nn;
    __syncthreads();
  };
  auto push = [&](uint64_t key) {
    const bool take = key >= floor_key && key != 0ull;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, take);
    uint32_t base = 0;
    if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, static_cast<uint32_t>(__popc(bal)));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (take) buf[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = key;
  };
  {
    const uint32_t g = a.gthr[b];
    floor_key = g ? static_cast<uint64_t>(g) << 32 : 1ull;
    for (uint32_t rr = 0; rr < 2 * a.ranges && !s_full; ++rr) {
      const size_t li = (static_cast<size_t>(rr >> 1) * a.Bpad + b) * 2 + (rr & 1u);
      const uint32_t n = a.counts[li];
      const uint64_t* L = a.lists + li * a.Lc;
      for (uint32_t i0 = 0; i0 < n; i0 += kFinThreads) {
        if (s_n + kFinThreads > kFinCap) {
          cut();
          if (s_n + kFinThreads > kFinCap) {  // cannot prune: exact scan instead
            if (tid == 0) s_full = 1u;
            __syncthreads();
            break;
          }
        }
        const uint32_t i = i0 + tid;
        push(i < n ? L[i] : 0ull);
        __syncthreads();
      }
    }
    __syncthreads();
    if (s_full) {
      if (tid == 0) a.fallback[b] = 1u;
      return;
    }
    cut();
  }
  // exact re-score of the survivors in the reference's order
  const uint32_t n = s_n;
  const float* q = a.Q + static_cast<size_t>(b) * a.d;
  const float S = a.fse[b].x;
  for (uint32_t i = tid; i < n; i += kFinThreads) {
    const uint32_t p = static_cast<uint32_t>(buf[i]);
    const double ex = gt_dot(q, a.X + static_cast<uint64_t>(p) * a.d, a.d);
    exs[i] = ex;
    if (a.diag) {
      const float ap = ord_to_float(static_cast<uint32_t>(buf[i] >> 32));
      const float ratio = static_cast<float>(fabs(static_cast<double>(ap) - static_cast<double>(S) * ex) / eps);
      atomicMax(a.diag, __float_as_uint(ratio));
    }
  }
  __syncthreads();
  // the top-K by (score desc, id asc): exact 96-bit selection, then rank placement
  const uint32_t keep = min(a.K, n);
  auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) {
    h = ord64(exs[i]);
    l = ~static_cast<uint32_t>(a.id_base + static_cast<uint32_t>(buf[i]));
    return true;
  };
  select96(get, n, keep, n, hist96, sel);
  for (uint32_t i = tid; i < n; i += kFinThreads) {
    uint64_t h;
    uint32_t l;
    get(i, h, l);
    if (!sel96_take(sel, h, l)) continue;
    const uint32_t slot = atomicAdd(&s_w, 1u);
    if (slot < 256u) widx[slot] = i;
  }
  __syncthreads();
  const uint32_t nw = min(s_w, keep);
  for (uint32_t w = tid; w < nw; w += kFinThreads) {
    const uint32_t i = widx[w];
    const uint64_t hi = ord64(exs[i]);
    const uint32_t id = static_cast<uint32_t>(a.id_base + static_cast<uint32_t>(buf[i]));
    uint32_t ahead = 0;
    for (uint32_t v = 0; v < nw; ++v) {
      const uint32_t j = widx[v];
      const uint64_t hj = ord64(exs[j]);
      const uint32_t idj = static_cast<uint32_t>(a.id_base + static_cast<uint32_t>(buf[j]));
      ahead += (hj > hi || (hj == hi && idj < id)) ? 1u : 0u;
    }
    const size_t o = static_cast<size_t>(b) * a.out_stride + ahead;
    a.out_ids[o] = id;
    a.out_scores[o] = exs[i];
  }
  if (tid == 0) a.out_count[static_cast<size_t>(b) * a.count_stride] = nw;
}

struct GtKernel {
  const void* fn;
  size_t smem;
  uint32_t N;
  uint32_t qt;
  bool qh;
};

GtKernel gt_pick(int device, uint32_t kpad, uint32_t B) {
  const TcKernel k = pick_cached_for(device, kpad, B);
  return {k.fn, k.smem, k.N, k.qt, k.qh};
}

}  // namespace

bool gt_tscan_eligible(uint64_t n, uint32_t d, uint32_t B, uint32_t K, int device) {
  if (!options().gt_tc || K == 0 || K > 256 || B < static_cast<uint32_t>(options().gt_tc_min_batch)) return false;
  if (n < 4096 || d == 0) return false;
  const uint32_t kpad = (d + 15) / 16 * 16;
  return gt_pick(device, kpad, B).fn != nullptr;
}

uint64_t gt_tscan_chunk_points(uint64_t n, uint32_t d, int device) {
  const uint32_t kpad = (d + 15) / 16 * 16;
  size_t fr = 0, tot = 0;
  PCPQG_CUDA(cudaMemGetInfo(&fr, &tot));
  const uint64_t budget = static_cast<uint64_t>(fr) / 100 * 35;  // operand cache: at most 35% of free memory
  uint64_t pc = std::min<uint64_t>(n, std::max<uint64_t>(65536, budget / (kpad * 2ull)));
  pc = std::min<uint64_t>(pc, (1ull << 32) - 512);
  if (options().gt_chunk > 0) pc = std::min<uint64_t>(n, std::max<uint64_t>(4096, options().gt_chunk));
  (void)device;
  return pc / 256 * 256 >= 4096 && pc < n ? pc / 256 * 256 : pc;
}

// One point chunk [p0, p0 + pc) of the data set: per query the chunk's exact
// top-K (global ids, double scores, sorted by (score desc, id asc)) into
// out_ids / out_scores [B][out_stride] + out_count [B]; fallback[b] = 1 where
// the query must be scored exactly over the chunk by the caller.
void gt_tscan_chunk(const float* dXc, uint64_t pc, uint64_t p0, uint32_t d, const float* dQ, uint32_t B, uint32_t K,
                    const void* d_stats, uint32_t* out_ids, double* out_scores, uint32_t* out_count,
                    uint32_t out_stride, uint32_t count_stride, uint32_t* fallback, int device, ScratchAlloc alloc,
                    cudaStream_t st, float* stage_ms) {
  const uint32_t kpad = (d + 15) / 16 * 16;
  const GtKernel kern = gt_pick(device, kpad, B);
  if (!kern.fn) fail(PCPQG_E_UNSUPPORTED, "ground truth tensor filter: dimension too large");
  const GtStats* stats = static_cast<const GtStats*>(d_stats);
  const uint32_t qrows = kern.qt * kTM;
  const uint32_t Bpad = (B + qrows - 1) / qrows * qrows;
  const uint32_t qtiles = Bpad / qrows;  // CTAs along the queries
  const uint32_t N = kern.N;
  const uint64_t npad = (pc + 255) / 256 * 256;
  const uint64_t ptiles = (pc + N - 1) / N;
  uint32_t tpr = 0;
  const uint32_t ranges = tc_ranges(ptiles, qtiles, num_sms(device), tpr);
  // seed pass over whole tiles spread evenly (about pc / scan_tc_seed points)
  const uint32_t bpt = N / kBlockPts;
  const uint64_t nbfull = pc / kBlockPts;
  const uint64_t den = static_cast<uint64_t>(std::max(1, options().scan_tc_seed));
  // (at most scan_tc_seed_max points: past ~1M the sample's cost — its GEMM and the
  // K-th-of-block-maxima select — grows with n while its threshold only gains ln)
  const uint64_t seed_cap = std::max<uint64_t>(2ull * K, static_cast<uint64_t>(options().scan_tc_seed_max) / kBlockPts);
  uint32_t sblocks = static_cast<uint32_t>(
      std::min<uint64_t>({nbfull, std::max<uint64_t>(nbfull / den, 2 * K), seed_cap}));
  const uint32_t stiles_all = static_cast<uint32_t>(pc / N);
  sblocks = std::min<uint32_t>(stiles_all, (sblocks + bpt - 1) / bpt) * bpt;
  if (options().scan_tc_seed <= 0 || sblocks < K) sblocks = 0;
  uint32_t seed_entries = 0;  // one per (sample tile, column half)
  if (sblocks) {
    if (sblocks / bpt * 2 < K) sblocks = std::min<uint32_t>(stiles_all, (K + 1) / 2) * bpt;
    seed_entries = sblocks / bpt * 2;
    if (seed_entries < K) sblocks = seed_entries = 0;
  }
  const uint64_t expect =
      sblocks ? static_cast<uint64_t>(K) * pc / (static_cast<uint64_t>(sblocks) * kBlockPts * ranges * 2) + 1
              : pc / (ranges * 2) + 1;
  uint32_t Lc = static_cast<uint32_t>(std::min<uint64_t>(8192, std::max<uint64_t>(1024, ((4 * expect + N) + 63) / 64 * 64)));
  Lc = std::max<uint32_t>(Lc, ((K + N) + 63) / 64 * 64);

  uint8_t* xhat = static_cast<uint8_t*>(alloc(static_cast<size_t>(kpad / 8) * npad * 16));
  uint8_t* qa = static_cast<uint8_t*>(alloc(static_cast<size_t>(Bpad) * kpad * 2 * (kern.qh ? 2 : 1)));
  float2* fse = static_cast<float2*>(alloc(static_cast<size_t>(Bpad) * 8));
  uint64_t* lists = static_cast<uint64_t*>(alloc(static_cast<size_t>(ranges) * Bpad * 2 * Lc * 8));
  uint32_t* counts = static_cast<uint32_t*>(alloc(static_cast<size_t>(ranges) * Bpad * 2 * 4));
  float* cmax = sblocks ? static_cast<float*>(alloc(static_cast<size_t>(Bpad) * sblocks * 4)) : nullptr;
  uint32_t* bins = static_cast<uint32_t*>(alloc(static_cast<size_t>(Bpad) * 33 * 4));
  float* base = reinterpret_cast<float*>(bins + static_cast<size_t>(Bpad) * 32);
  PCPQG_CUDA(cudaMemsetAsync(bins, 0, static_cast<size_t>(Bpad) * 32 * 4, st));
  PCPQG_CUDA(cudaMemsetAsync(base, 0xFF, static_cast<size_t>(Bpad) * 4, st));  // NaN: no seed
  uint32_t* gthr = static_cast<uint32_t*>(alloc(static_cast<size_t>(Bpad) * 8));
  uint32_t* ovf = gthr + Bpad;
  PCPQG_CUDA(cudaMemsetAsync(gthr, 0, static_cast<size_t>(Bpad) * 8, st));
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (stage_ms) {
    for (auto& e : ev) PCPQG_CUDA(cudaEventCreate(&e));
    PCPQG_CUDA(cudaEventRecord(ev[0], st));
  }
  {
    const size_t xsm = static_cast<size_t>(kGxPts) * (d + 1) * 4;
    PCPQG_CUDA(cudaFuncSetAttribute(gt_xhat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(xsm)));
    gt_xhat_kernel<<<static_cast<unsigned>((npad + kGxPts - 1) / kGxPts), 256, xsm, st>>>(dXc, pc, d, kpad, npad, N,
                                                                                         stats, xhat);
  }
  GtPrepArgs pa{dQ, B, Bpad, d, kpad, kern.qh ? 1u : 0u, stats, qa, fse};
  gt_prep_kernel<<<(Bpad + 7) / 8, 256, 0, st>>>(pa);
  PCPQG_CUDA(cudaGetLastError());

  TScanArgs a{};
  a.qa = qa;
  a.fse = fse;
  a.lists = lists;
  a.counts = counts;
  a.gthr = gthr;
  a.ovf = ovf;
  a.n_local = pc;
  a.kpad = kpad;
  a.K = K;
  a.Lc = Lc;
  a.B = B;
  a.Bpad = Bpad;
  a.tiles_per_range = tpr;
  a.nbfull = static_cast<uint32_t>(nbfull);
  a.bins = bins;
  a.base = base;
  PCPQG_CUDA(cudaFuncSetAttribute(kern.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kern.smem)));
  if (sblocks) {  // seed: the K-th best block maximum of the sample, per query
    TScanArgs as = a;
    as.mode = 1;
    as.sblocks = sblocks;
    as.cm_stride = seed_entries;
    as.cmax = cmax;
    const uint64_t stiles = (static_cast<uint64_t>(sblocks) * kBlockPts + N - 1) / N;
    uint32_t stpr = 0;
    const uint32_t sranges = tc_ranges(stiles, qtiles, num_sms(device), stpr);
    as.tiles_per_range = stpr;
    XArgs xs{xhat, npad, stiles_all};
    void* args[] = {&as, &xs};
    PCPQG_CUDA(cudaLaunchKernel(kern.fn, dim3(qtiles, sranges), dim3(kCThreads), args, kern.smem, st));
    FinishArgs fs{};
    fs.seed = 1;
    fs.fse = fse;
    fs.ovf = ovf;
    fs.K = K;
    fs.seed_blocks = seed_entries;
    fs.cm_stride = seed_entries;
    fs.cmax = cmax;
    fs.gthr_out = gthr;
    fs.base_out = base;
    fs.cap = kFinCap;
    const size_t fsm = kFinCap * 8 + 16;
    PCPQG_CUDA(cudaFuncSetAttribute(tscan_finish_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kFinCap * 8 + 64 * 1024)));
    tscan_finish_kernel<false><<<B, kFinThreads, fsm, st>>>(fs);
    PCPQG_CUDA(cudaGetLastError());
  }
  if (stage_ms) PCPQG_CUDA(cudaEventRecord(ev[1], st));
  {
    XArgs xs{xhat, npad, stiles_all};
    void* args[] = {&a, &xs};
    PCPQG_CUDA(cudaLaunchKernel(kern.fn, dim3(qtiles, ranges), dim3(kCThreads), args, kern.smem, st));
  }
  if (stage_ms) PCPQG_CUDA(cudaEventRecord(ev[2], st));
  GtFinishArgs f{};
  f.X = dXc;
  f.Q = dQ;
  f.n = pc;
  f.id_base = p0;
  f.d = d;
  f.lists = lists;
  f.counts = counts;
  f.gthr = gthr;
  f.ovf = ovf;
  f.fse = fse;
  f.ranges = ranges;
  f.Lc = Lc;
  f.Bpad = Bpad;
  f.K = K;
  f.out_stride = out_stride;
  f.count_stride = count_stride;
  f.out_ids = out_ids;
  f.out_scores = out_scores;
  f.out_count = out_count;
  f.fallback = fallback;
  unsigned int* diag = nullptr;
  if (options().scan_tc_diag) {
    diag = static_cast<unsigned int*>(alloc(16));
    PCPQG_CUDA(cudaMemsetAsync(diag, 0, 16, st));
    f.diag = diag;
  }
  const size_t gsm = static_cast<size_t>(kFinCap) * 16;
  PCPQG_CUDA(cudaFuncSetAttribute(gt_tfinish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(gsm)));
  gt_tfinish_kernel<<<B, kFinThreads, gsm, st>>>(f);
  PCPQG_CUDA(cudaGetLastError());
  if (diag) {
    unsigned int hd[2];
    std::vector<uint32_t> hc(static_cast<size_t>(ranges) * Bpad * 2);
    PCPQG_CUDA(cudaMemcpyAsync(hd, diag, 8, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaMemcpyAsync(hc.data(), counts, hc.size() * 4, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
    uint64_t tot = 0;
    for (uint32_t q = 0; q < B; ++q)
      for (uint32_t r2 = 0; r2 < ranges; ++r2)
        tot += hc[(static_cast<size_t>(r2) * Bpad + q) * 2] + hc[(static_cast<size_t>(r2) * Bpad + q) * 2 + 1];
    float r;
    std::memcpy(&r, hd, 4);
    std::fprintf(stderr,
                 "[pcpqg] gt tscan: N=%u ranges=%u Lc=%u seed=%u pts | list entries %.1f per query; "
                 "max |approx - S*exact| / eps = %g\n",
                 N, ranges, Lc, sblocks * kBlockPts, static_cast<double>(tot) / B, r);
  }
  if (stage_ms) {
    PCPQG_CUDA(cudaEventRecord(ev[3], st));
    PCPQG_CUDA(cudaEventSynchronize(ev[3]));
    cudaEventElapsedTime(&stage_ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&stage_ms[1], ev[1], ev[2]);
    cudaEventElapsedTime(&stage_ms[2], ev[2], ev[3]);
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

size_t gt_stats_bytes() { return sizeof(GtStats); }

void gt_stats(const float* dX, uint64_t n, uint32_t d, void* d_stats, cudaStream_t st) {
  PCPQG_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(GtStats), st));
  gt_stats_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 7) / 8, 148ull * 64)), 256, 0, st>>>(
      dX, n, d, static_cast<GtStats*>(d_stats));
  PCPQG_CUDA(cudaGetLastError());
}

}  // namespace pcpqg

namespace pcpqg {
void free_tc(TcIndex* t) { delete t; }
}  // namespace pcpqg
