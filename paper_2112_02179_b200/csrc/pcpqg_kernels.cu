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
#include <cassert>
#include <cstdio>


#include "pcpqg_device.cuh"

namespace pcpqg {

ScanFn scan_fn_joint8(bool k16, int nq);
ScanFn scan_fn_joint8_table(int nq);
ScanFn scan_fn_joint8_filter();
ScanFn scan_fn_p8_filter();
ScanFn scan_fn_p4_raw16_filter();
ScanFn scan_fn_p4(uint32_t sw, bool k16, int nq);
ScanFn scan_fn_p8(uint32_t sw, int nq);
ScanFn scan_fn_p16(uint32_t sw, int nq);

namespace {

ScanFn pick_kernel(const DeviceIndex& x, int nq, bool table = false, bool filter = false) {
  const bool k16 = x.h.k == 16;
  ScanFn f = nullptr;
  if (filter) f = x.format == PCPQG_FMT_JOINT8 ? scan_fn_joint8_filter()
                  : x.cw == 8                   ? scan_fn_p8_filter()
                                                : scan_fn_p4_raw16_filter();
  else if (table) f = scan_fn_joint8_table(nq);
  else if (x.format == PCPQG_FMT_JOINT8) f = scan_fn_joint8(k16, nq);
  else if (x.cw == 4) f = scan_fn_p4(x.sw, k16, nq);
  else if (x.cw == 8) f = scan_fn_p8(x.sw, nq);
  else if (x.cw == 16) f = scan_fn_p16(x.sw, nq);
  if (!f) fail(PCPQG_E_UNSUPPORTED, "no scan kernel for this code layout");
  return f;
}

// ----------------------------------------------------------- K1: LUT
// One thread per (query, section, center).  Grouped layout (scan input):
// eta[g*gstride + (j*k + c)*rs + qi] for sections j < m8 = m rounded up to 8;
// sections j >= m get -0.0f so the scan's branch-free octets add exactly -0.
// Plain layout (parity API): eta[q*m*k + j*k + c] for j < m.
__global__ void lut_kernel(const float* __restrict__ Q, uint32_t B, uint64_t total, uint32_t d,
                           const float* __restrict__ cb, const float* __restrict__ lam, uint32_t m,
                           uint32_t msec, uint32_t k, uint32_t rows, uint32_t cbits, uint32_t s,
                           uint32_t dbar, int nq, int rs, uint64_t gstride, int mode,
                           float* __restrict__ eta, uint64_t* __restrict__ zero, uint32_t nzero) {
  // a small-batch scan launched as a programmatic dependent may start now; it
  // waits for this grid's completion before it reads eta
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < nzero) zero[t] = 0ull;  // the scan's shared K-th keys and tickets (saves a memset)
  if (t >= total) return;
  const uint32_t r = static_cast<uint32_t>(t % rows);  // center (modes 0/1) or code byte (mode 2)
  const uint32_t j = static_cast<uint32_t>((t / rows) % msec);
  const uint64_t q = t / (static_cast<uint64_t>(rows) * msec);
  const uint32_t c = mode == 2 ? (r & ((1u << cbits) - 1u)) : r;
  const uint32_t l = mode == 2 ? (r >> cbits) : 0u;
  float acc = 0.0f;  // fixed-order fp32 accumulation from 0.0f (pq_index.cpp:186-190)
  if (j >= m) {
    acc = -0.0f;
  } else if (q < B && c < k) {
    const float* row = cb + (static_cast<uint64_t>(j) * k + c) * dbar;
    const float* qq = Q + q * d;
    for (uint32_t a = 0; a < dbar; ++a) {
      const uint32_t col = j * dbar + a;
      const float qa = col < d ? __ldg(qq + col) : 0.0f;  // pad_vector (types.cpp:83-88)
      acc = __fadd_rn(acc, __fmul_rn(__ldg(row + a), qa));
    }
    // eta * lambda, the stored eta_lambda entry (pq_index.cpp:203)
    if (mode == 2) acc = l < s ? __fmul_rn(acc, __ldg(lam + static_cast<uint64_t>(j) * s + l)) : 0.0f;
  }
  if (mode != 0) {
    const uint64_t g = q / nq, qi = q % nq;
    eta[g * gstride + (static_cast<uint64_t>(j) * rows + r) * rs + qi] = acc;
  } else {
    eta[q * m * k + static_cast<uint64_t>(j) * k + c] = acc;
  }
}

// per-section max |alpha| of a raw fp16 alpha plane (PLANES, 16-bit scale
// words: 2 alphas per word); one thread per (point, scale word)
__global__ void alpha_max_kernel(const uint32_t* __restrict__ codes, uint64_t n, uint32_t W, uint32_t Wc,
                                 uint32_t m, uint32_t* __restrict__ amax_bits) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t Ws = W - Wc;
  if (t >= n * Ws) return;
  const uint64_t p = t / Ws;
  const uint32_t w = static_cast<uint32_t>(t % Ws);
  const uint32_t word = codes[((p >> 5) * W + Wc + w) * kBlockPts + (p & 31)];
#pragma unroll
  for (uint32_t h = 0; h < 2; ++h) {
    const uint32_t j = 2 * w + h;
    if (j >= m) break;
    const float a = fabsf(__half2float(__ushort_as_half(static_cast<unsigned short>(word >> (16 * h)))));
    atomicMax(amax_bits + j, __float_as_uint(a));  // non-negative floats order like their bits
  }
}

// K2-F eligibility of the raw fp16 alpha layout: alpha is used unscaled, so
// every section's max |alpha| must keep fp16(eta * sigma) in range
bool raw_alpha_filter_ok(const DeviceIndex& x) {
  if (!(x.format == PCPQG_FMT_PLANES && x.cw == 4 && x.sw == 16 && x.h.k == 16)) return false;
  ensure_alpha_max(x);
  for (uint32_t j = 0; j < x.h.m; ++j)
    if (x.amax[j] != 0.0f && (x.amax[j] < 0.0625f || x.amax[j] > 16.0f)) return false;
  return true;
}

// ------------------------------------------------- K2-F: filter tables
// raw alpha: tau_j = 1, maxlam_j = max |alpha_j| (no lambda_hat table)
__global__ void ftab_alpha_kernel(const float* __restrict__ amax, uint32_t m8, float* __restrict__ tau,
                                  float* __restrict__ maxlam) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m8) return;
  tau[j] = 1.0f;
  maxlam[j] = amax[j];
}

// Section scales: tau_j = 2^-e with max_l |lambda_j[l]| = f * 2^e, f in
// [0.5, 1) (1 if every lambda is 0); lambda_hat = fp16(lambda * tau_j).
__global__ void ftab_lambda_kernel(const float* __restrict__ lam, uint32_t m8, uint32_t s,
                                   __half* __restrict__ flam, float* __restrict__ tau,
                                   float* __restrict__ maxlam) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m8) return;
  float mx = 0.0f;
  for (uint32_t l = 0; l < s; ++l) mx = fmaxf(mx, fabsf(lam[j * s + l]));
  int e = 0;
  if (mx > 0.0f) frexpf(mx, &e);
  e = max(e, -125);  // (all-subnormal scales: tau stays finite)
  const float t = ldexpf(1.0f, -e);
  for (uint32_t l = 0; l < s; ++l) flam[j * s + l] = __float2half_rn(lam[j * s + l] * t);
  tau[j] = t;
  maxlam[j] = mx;
}

// Per query: sigma = 2^(10 - e) with M = max_j (max_c |eta_j[c]|) * max_l |lambda_j[l]|
// = f * 2^e (so M * sigma < 2^10: every product < 2^10, every octet sum < 2^13),
// A = sum_j of the same per-section maxima (>= sum_j |term_j| of any point), and
//   eps = (12u + 2^-20) A + m 1e-4 / sigma + (m + 1) 1.02 2^-24 A,  u = 2^-11:
// fp16 rounding of eta_hat, lambda_hat, each HFMA2 and the octet sums (<= 12u
// per unit of sum |term|), subnormal absolute errors (<= 1e-4 per section in
// scaled units), the fp32 octet adds (2^-20), and the distance between the
// reference's fp32 score and the real sum of the terms ((m+1) 2^-24 A).
__global__ void ftab_query_kernel(const float* __restrict__ eta, uint64_t gstride, int rs, int nq,
                                  uint32_t m, uint32_t k, uint32_t Bpad, const float* __restrict__ maxlam,
                                  float2* __restrict__ fse) {
  // one warp per query, lanes over the sections
  const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (q >= Bpad) return;
  const uint64_t g = q / nq, qi = q % nq;
  const float* eg = eta + g * gstride + qi;
  double M = 0.0, A = 0.0;
  for (uint32_t j = lane; j < m; j += 32) {
    float me = 0.0f;
    for (uint32_t c = 0; c < k; ++c) me = fmaxf(me, fabsf(eg[(static_cast<uint64_t>(j) * k + c) * rs]));
    const double pr = static_cast<double>(me) * static_cast<double>(maxlam[j]);
    M = fmax(M, pr);
    A += pr;  // (any order: A only scales the bound, which has slack for its rounding)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    M = fmax(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
    A += __shfl_xor_sync(0xFFFFFFFFu, A, o);
  }
  if (lane != 0) return;
  int e = 0;
  if (M > 0.0) frexp(M, &e);
  // sigma outside [2^-100, 2^120] (terms near fp32's range limits, where the
  // reference's own products under/overflow): no filter for this query —
  // (0, inf) makes every point pass to the exact score
  if (e < -110 || e > 110) {
    fse[q] = make_float2(0.0f, INFINITY);
    return;
  }
  const double sigma = ldexp(1.0, 10 - e);
  const double u = ldexp(1.0, -11);
  const double eps = (12.0 * u + ldexp(1.0, -20)) * A + m * 1e-4 / sigma +
                     (m + 1.0) * 1.02 * ldexp(1.0, -24) * A;
  fse[q] = make_float2(static_cast<float>(sigma), __double2float_ru(eps * (1.0 + 1e-6)));
}

// eta_hat[g][(j*rows + c)*frs + qi] = fp16(eta * sigma_q / tau_j) (exact
// scaling by a power of two, one rounding); 0 for pad columns and lambda-free
// sections
__global__ void ftab_eta_kernel(const float* __restrict__ eta, uint64_t gstride, int rs, uint32_t m8,
                                uint32_t rows, uint32_t frs, uint32_t nq, uint64_t total,
                                const float* __restrict__ tau, const float* __restrict__ maxlam,
                                const float2* __restrict__ fse, __half* __restrict__ fh, uint64_t fgstride) {
  // one thread per eta_hat row (g, j, c): frs halves, written as words
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const uint32_t c = static_cast<uint32_t>(t % rows);
  const uint32_t j = static_cast<uint32_t>((t / rows) % m8);
  const uint64_t g = t / (static_cast<uint64_t>(rows) * m8);
  const float* er = eta + g * gstride + (static_cast<uint64_t>(j) * rows + c) * rs;
  uint32_t* out = reinterpret_cast<uint32_t*>(fh + g * fgstride + (static_cast<uint64_t>(j) * rows + c) * frs);
  const bool live = maxlam[j] > 0.0f;
  const float tj = tau[j];
  for (uint32_t qi = 0; qi < frs; qi += 2) {
    float v[2] = {0.0f, 0.0f};
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h)
      if (live && qi + h < nq)  // sigma / tau_j: powers of two, applied in double (no fp32 over/underflow)
        v[h] = static_cast<float>(static_cast<double>(er[qi + h]) * static_cast<double>(fse[g * nq + qi + h].x) /
                                  static_cast<double>(tj));
    const __half2 hv = __floats2half2_rn(v[0], v[1]);
    out[qi / 2] = *reinterpret_cast<const uint32_t*>(&hv);
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
                 float* __restrict__ scores, const uint32_t* __restrict__ counts) {
  extern __shared__ uint64_t sk[];
  __shared__ __align__(16) uint32_t hist[kGroupScratch];
  __shared__ uint32_t s_n;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const Group grp{0, static_cast<int>(nthr), static_cast<int>(tid)};
  uint64_t thr = 1ull;  // drops empty keys
  if (gtau) thr = max(thr, static_cast<uint64_t>(gtau[b]));
  const uint32_t total = L * Kin;
  auto fetch = [&](uint32_t i) -> uint64_t {
    const uint32_t l = i / Kin, r = i - l * Kin;
    // (counts: a list's keys past its length are not keys)
    if (counts && r >= counts[static_cast<size_t>(l) * in_rows + b]) return 0ull;
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
#ifdef PCPQG_DEBUG
  if (tid == 0 && b < 2) printf("merge b=%u L=%u Kin=%u total=%u survivors=%u cap=%u thr=%llx\n", b, L, Kin, total, n, cap, (unsigned long long)thr);
#endif
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
    n = group_compact(sk, n, tau, hist + kHistWords + kSvWords, grp);
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

// K3b: merge of SORTED lists (the scan's per-CTA survivor lists and the
// per-GPU result rows are both sorted descending).  One CTA per query: the
// lists' survivors are staged in shared memory at exclusive-scan offsets by
// TMA bulk copies (every list in flight at once), then warp 0 runs a K-step
// tournament: each lane keeps the current heads of its <= 8 lists in
// registers, the warp arg-max picks the winner, only the winning lane
// advances one list (one shared load).  counts (optional) gives each list's
// length; without it a list ends at its first empty (0) key.
constexpr int kTourListsPerLane = 8;  // L <= 256

// NT = 128: the warp-0 tournament (many queries: one small CTA each).
// NT = 512: few queries — the whole CTA radix-selects the Kout-th key over the
// staged survivors, compacts and bitonic-sorts (no serial K-step loop).
template <int NT>
__global__ void __launch_bounds__(NT)
    merge_sorted_kernel(const uint64_t* __restrict__ in, const uint32_t* __restrict__ counts,
                        uint32_t L, uint32_t in_rows, uint32_t Ks, uint32_t Kout,
                        uint32_t out_stride, uint32_t cap, uint64_t* __restrict__ out,
                        int32_t* __restrict__ ids, float* __restrict__ scores) {
  extern __shared__ __align__(16) uint64_t s_key[];  // cap keys
  __shared__ uint32_t s_off[257];
  __shared__ uint32_t wsum[NT / 32];
  __shared__ __align__(8) uint64_t s_bar;
  const uint32_t b = blockIdx.x, tid = threadIdx.x;
  const uint32_t lane = tid & 31, w = tid >> 5;
  const bool tma = (Ks & 1u) == 0u;  // 16-byte aligned rows
  auto row = [&](uint32_t l) { return in + (static_cast<size_t>(l) * in_rows + b) * Ks; };
  auto list_len = [&](uint32_t l) -> uint32_t {
    if (counts) return counts[static_cast<size_t>(l) * in_rows + b];
    const uint64_t* r = row(l);  // first empty key ends the list
    uint32_t lo = 0, hi = Ks;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (r[mid] != 0ull) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  // Wide path with L >= Kout lists: the Kout-th largest list head T is a lower
  // bound of the Kout-th key overall (Kout heads are >= T), so each sorted list
  // only contributes its prefix of keys >= T.
  uint64_t T = 0ull;
  if constexpr (NT > 128) {
    static_assert(NT >= 256, "one thread per list head");
    __shared__ uint64_t s_head[256];
    __shared__ uint64_t s_T;
    if (L >= Kout && L <= 256) {
      const uint64_t h = tid < L && list_len(tid) > 0 ? row(tid)[0] : 0ull;
      if (tid < L) s_head[tid] = h;
      if (tid == 0) s_T = 0ull;
      __syncthreads();
      // T = the head with exactly Kout - 1 heads ahead of it (larger, or equal
      // at a lower list index): the Kout-th of the heads sorted descending, or
      // 0 with fewer than Kout non-empty lists.  One barrier instead of a sort.
      if (tid < L && h != 0ull) {
        uint32_t ahead = 0;
        for (uint32_t j = 0; j < L; ++j) {
          const uint64_t v = s_head[j];
          ahead += (v > h || (v == h && j < tid)) ? 1u : 0u;
        }
        if (ahead == Kout - 1) s_T = h;
      }
      __syncthreads();
      T = s_T;
    }
  }
  // list lengths (padded to even) -> exclusive offsets
  uint32_t base = 0;
  for (uint32_t l0 = 0; l0 < L; l0 += NT) {
    const uint32_t l = l0 + tid;
    uint32_t c = 0;
    if (l < L) {
      c = list_len(l);
      c = min(c, Kout);             // a sorted list contributes at most Kout keys
      if (T) {                      // keys >= T: a prefix of the descending list
        const uint64_t* r = row(l);
        uint32_t lo = 0, hi = c;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (r[mid] >= T) lo = mid + 1;
          else hi = mid;
        }
        c = lo;
      }
      if (tma) c = (c + 1u) & ~1u;  // 16-byte pieces; the pad key is empty or beyond Kout
    }
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    uint32_t before = 0, chunk = 0;
    for (uint32_t t = 0; t < NT / 32; ++t) {
      before += t < w ? wsum[t] : 0u;
      chunk += wsum[t];
    }
    if (l < L) s_off[l] = base + before + incl - c;
    base += chunk;
    __syncthreads();
  }
  if (tid == 0) s_off[L] = base;
  const uint32_t total = min(base, cap);
  if (tma) {
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      fence_mbar_init();
      mbar_expect_tx(&s_bar, total * 8);
    }
    __syncthreads();
    for (uint32_t l = tid; l < L; l += NT) {
      const uint32_t o = s_off[l], c = min(s_off[l + 1], total) - min(o, total);
      if (c) bulk_g2s(s_key + o, row(l), c * 8, &s_bar);
    }
    mbar_wait(&s_bar, 0u);
  } else {
    __syncthreads();
    for (uint32_t l = w; l < L; l += NT / 32) {
      const uint32_t o = s_off[l], c = min(s_off[l + 1], total) - min(o, total);
      const uint64_t* r = row(l);
      for (uint32_t i = lane; i < c; i += 32) s_key[o + i] = r[i];
    }
    __syncthreads();
  }
  if constexpr (NT > 128) {
    // block-parallel: Kout-th key by radix select, keep the keys at or above it
    // (pad / empty keys sort last), bitonic sort, write
    __shared__ __align__(16) uint32_t scratch[kGroupScratch];
    const Group grp{0, NT, static_cast<int>(tid)};
    uint32_t n = total;
    // up to 256 staged keys: the rank placement below selects and orders them
    // in one pass (cheaper than the radix select's ~24 barriers)
    if (n > Kout && n > 256u) {
      const uint64_t tau = group_select(s_key, n, Kout, scratch, scratch + kHistWords, grp);
      n = group_compact(s_key, n, tau, scratch + kHistWords + kSvWords, grp);
    }
    auto put = [&](uint32_t r, uint64_t key) {
      if (out) out[static_cast<size_t>(b) * out_stride + r] = key;
      if (ids) ids[static_cast<size_t>(b) * out_stride + r] = key_id(key);
      if (scores) scores[static_cast<size_t>(b) * out_stride + r] = key_score(key);
    };
    if (n <= static_cast<uint32_t>(NT)) {
      // one key per thread: its output row is the number of keys ahead of it
      // (larger, or equal at a lower index) — the row the descending sort
      // below would give it, without the sort's ~28 barriers
      __syncthreads();
      if (tid < n) {
        const uint64_t key = s_key[tid];
        uint32_t ahead = 0;
        for (uint32_t j = 0; j < n; ++j) {
          const uint64_t v = s_key[j];
          ahead += (v > key || (v == key && j < tid)) ? 1u : 0u;
        }
        if (ahead < out_stride) put(ahead, ahead < Kout ? key : 0ull);
      }
      for (uint32_t r = n + tid; r < out_stride; r += NT) put(r, 0ull);
      return;
    }
    uint32_t P = 1;
    while (P < n) P <<= 1;
    for (uint32_t i = n + tid; i < P; i += NT) s_key[i] = 0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = tid; i < P / 2; i += NT) {
          const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
          const uint32_t hi = lo + stride;
          const uint64_t x = s_key[lo], y = s_key[hi];
          if ((x < y) == ((lo & size) == 0)) {
            s_key[lo] = y;
            s_key[hi] = x;
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t r = tid; r < out_stride; r += NT) {
      const uint64_t key = r < Kout && r < n ? s_key[r] : 0ull;
      if (out) out[static_cast<size_t>(b) * out_stride + r] = key;
      if (ids) ids[static_cast<size_t>(b) * out_stride + r] = key_id(key);
      if (scores) scores[static_cast<size_t>(b) * out_stride + r] = key_score(key);
    }
    return;
  }
  if (w != 0) return;
  // tournament
  uint32_t pos[kTourListsPerLane], end[kTourListsPerLane];
  uint64_t hd[kTourListsPerLane];
#pragma unroll
  for (int j = 0; j < kTourListsPerLane; ++j) {
    const uint32_t l = lane + 32u * j;
    pos[j] = l < L ? min(s_off[l], total) : 0u;
    end[j] = l < L ? min(s_off[l + 1], total) : 0u;
    hd[j] = pos[j] < end[j] ? s_key[pos[j]] : 0ull;
  }
  auto best_of = [&](uint64_t& best, int& jb) {
    best = hd[0];
    jb = 0;
#pragma unroll
    for (int j = 1; j < kTourListsPerLane; ++j)
      if (hd[j] > best) {
        best = hd[j];
        jb = j;
      }
  };
  uint64_t best;
  int jb;
  best_of(best, jb);
  for (uint32_t r = 0; r < out_stride; ++r) {
    uint64_t m = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, m, o);
      m = v > m ? v : m;
    }
    const uint64_t key = r < Kout ? m : 0ull;
    if (lane == (r & 31u)) {  // spread the output stores over the lanes
      if (out) out[static_cast<size_t>(b) * out_stride + r] = key;
      if (ids) ids[static_cast<size_t>(b) * out_stride + r] = key_id(key);
      if (scores) scores[static_cast<size_t>(b) * out_stride + r] = key_score(key);
    }
    if (m != 0ull && best == m) {  // keys are unique: exactly one winner
#pragma unroll
      for (int j = 0; j < kTourListsPerLane; ++j)
        if (j == jb) {
          pos[j] += 1;
          hd[j] = pos[j] < end[j] ? s_key[pos[j]] : 0ull;
        }
      best_of(best, jb);
    }
  }
}

// K3c: the sorted merge for few queries (B < #SMs) in ONE round trip to global
// memory.  merge_sorted_kernel<512> walks a latency chain there (list lengths ->
// heads -> a binary search over L2 per list -> TMA staging); here every list
// row is staged whole by one bulk copy per list, issued together with the
// count loads, and everything else — the head threshold T (the Kout-th largest
// head bounds the answer), each list's prefix >= T, the compaction and the
// rank placement — runs on shared memory.  Launched with programmatic stream
// serialization: the CTA is resident before the scan drains and waits in
// griddepcontrol.wait.
constexpr uint32_t kOneDense = 2048;   // dense staging for the usual case (prefix total <= 2048)
constexpr uint32_t kOneMaxKeys = 23000;  // L * Ks limit (shared memory)
__global__ void __launch_bounds__(512)
    merge_oneshot_kernel(const uint64_t* __restrict__ in, const uint32_t* __restrict__ counts, uint32_t L,
                         uint32_t in_rows, uint32_t Ks, uint32_t Kout, uint32_t out_stride,
                         uint64_t* __restrict__ out, int32_t* __restrict__ ids, float* __restrict__ scores) {
  constexpr uint32_t NT = 512;
  extern __shared__ __align__(16) uint64_t s_one[];  // [L * Ks] staged rows | [kOneDense] dense
  uint64_t* s_all = s_one;
  uint64_t* s_dense = s_one + static_cast<size_t>(L) * Ks;
  __shared__ uint32_t s_len[256], s_off[257], wsum[NT / 32];
  __shared__ uint64_t s_head[256];
  __shared__ uint64_t s_T;
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ __align__(16) uint32_t scratch[kGroupScratch];
  const uint32_t b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&s_bar, L * Ks * 8);
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scan's lists and counts are complete
  for (uint32_t l = tid; l < L; l += NT) {
    bulk_g2s(s_all + static_cast<size_t>(l) * Ks, in + (static_cast<size_t>(l) * in_rows + b) * Ks, Ks * 8, &s_bar);
    s_len[l] = min(counts[static_cast<size_t>(l) * in_rows + b], min(Ks, Kout));
  }
  mbar_wait(&s_bar, 0u);
  __syncthreads();
  // T = the Kout-th largest list head (0 with fewer than Kout non-empty lists)
  uint64_t T = 0ull;
  if (L >= Kout) {
    const uint64_t h = tid < L && s_len[tid] > 0 ? s_all[static_cast<size_t>(tid) * Ks] : 0ull;
    if (tid < L) s_head[tid] = h;
    if (tid == 0) s_T = 0ull;
    __syncthreads();
    if (tid < L && h != 0ull) {
      uint32_t ahead = 0;
      for (uint32_t j = 0; j < L; ++j) {
        const uint64_t v = s_head[j];
        ahead += (v > h || (v == h && j < tid)) ? 1u : 0u;
      }
      if (ahead == Kout - 1) s_T = h;
    }
    __syncthreads();
    T = s_T;
  }
  // each list's prefix of keys >= T (descending lists), exclusive offsets
  uint32_t c = 0;
  if (tid < L) {
    c = s_len[tid];
    if (T) {
      const uint64_t* r = s_all + static_cast<size_t>(tid) * Ks;
      uint32_t lo = 0, hi = c;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (r[mid] >= T) lo = mid + 1;
        else hi = mid;
      }
      c = lo;
    }
  }
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += v;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t before = 0, total = 0;
  for (uint32_t t = 0; t < NT / 32; ++t) {
    before += t < w ? wsum[t] : 0u;
    total += wsum[t];
  }
  if (tid < L) s_off[tid] = before + incl - c;
  if (tid == 0) s_off[L] = total;
  __syncthreads();
  const Group grp{0, static_cast<int>(NT), static_cast<int>(tid)};
  uint64_t* key = s_dense;
  uint32_t n = total;
  if (total <= kOneDense) {
    for (uint32_t l = w; l < L; l += NT / 32) {
      const uint32_t o = s_off[l], cl = s_off[l + 1] - o;
      const uint64_t* r = s_all + static_cast<size_t>(l) * Ks;
      for (uint32_t i = lane; i < cl; i += 32) s_dense[o + i] = r[i];
    }
    __syncthreads();
  } else {  // rare: empty the tails and compact the staged rows in place
    for (uint32_t l = w; l < L; l += NT / 32) {
      const uint32_t cl = s_off[l + 1] - s_off[l];
      uint64_t* r = s_all + static_cast<size_t>(l) * Ks;
      for (uint32_t i = cl + lane; i < Ks; i += 32) r[i] = 0ull;
    }
    __syncthreads();
    key = s_all;
    n = group_compact(s_all, L * Ks, 1ull, scratch + kHistWords + kSvWords, grp);
  }
  if (n > NT) {  // more than one key per thread: cut to the Kout best first (Kout <= 512)
    const uint64_t tau = group_select(key, n, Kout, scratch, scratch + kHistWords, grp);
    n = group_compact(key, n, tau, scratch + kHistWords + kSvWords, grp);
  }
  auto put = [&](uint32_t r, uint64_t kk) {
    if (out) out[static_cast<size_t>(b) * out_stride + r] = kk;
    if (ids) ids[static_cast<size_t>(b) * out_stride + r] = key_id(kk);
    if (scores) scores[static_cast<size_t>(b) * out_stride + r] = key_score(kk);
  };
  if (tid < n) {  // a key's output row = the number of keys ahead of it
    const uint64_t kk = key[tid];
    uint32_t ahead = 0;
    for (uint32_t j = 0; j < n; ++j) {
      const uint64_t v = key[j];
      ahead += (v > kk || (v == kk && j < tid)) ? 1u : 0u;
    }
    if (ahead < out_stride) put(ahead, ahead < Kout ? kk : 0ull);
  }
  for (uint32_t r = min(n, Kout) + tid; r < out_stride; r += NT) put(r, 0ull);
}

// filter (K2-F) variants: JOINT8 k = 16 in groups of 16 (eta rows of kFRS
// halves, exact table in shared memory) or PLANES 8-bit centers / 4-bit scales
// in groups of 4 (rows of 4 halves, exact table left in global memory)
bool filter_layout(const DeviceIndex& x) {
  if (x.h.m > 64) return false;  // (the exact re-score keeps a point's words in registers)
  return (x.format == PCPQG_FMT_JOINT8 && x.h.k == 16) ||
         (x.format == PCPQG_FMT_PLANES && x.cw == 8 && x.sw == 4) || raw_alpha_filter_ok(x);
}
// groups of 16 with the exact table in shared memory (JOINT8, raw alpha) or
// groups of 4 with it in global memory (PLANES 8/4)
bool filter_nq16(const DeviceIndex& x) { return !(x.format == PCPQG_FMT_PLANES && x.cw == 8); }
uint32_t filter_frs(const DeviceIndex& x) { return filter_nq16(x) ? kFRS : 4u; }

size_t scan_smem_bytes(const DeviceIndex& x, int nq, uint32_t cap, uint32_t ppt, bool topk,
                       int nthr, int stages, uint32_t rows, bool table, bool filter = false) {
  const int rs = rs_of(nq);
  const bool nolam = table || (x.format == PCPQG_FMT_PLANES && x.sw >= 16);
  const uint32_t m8 = (x.h.m + 7) & ~7u;
  const int ngroups = scan_ngroups(nq, nthr);
  const bool eta_global = filter && !filter_nq16(x);  // the groups-of-4 variant reads eta from L2
  size_t b = static_cast<size_t>(stages) * nthr * ppt * x.W * 4;
  b += topk ? static_cast<size_t>(nq) * cap * 8 : 0;
  b += eta_global ? 0 : (static_cast<size_t>(m8) * rows * rs * 4 + 15) & ~static_cast<size_t>(15);
  b += nolam ? 0 : ((m8 * std::max(x.h.scales, 1u) * 4 + 15u) & ~15u);
  b += topk ? static_cast<size_t>(ngroups) * kGroupScratch * 4 : 0;
  if (filter)
    b += static_cast<size_t>(m8) * rows * filter_frs(x) * 2 + ((m8 * std::max(x.h.scales, 1u) * 2 + 15u) & ~15u) +
         64 + 16 + kFQCap * 4;
  b += 320 + 128;  // header + alignment of the eta block
  return b;
}

int g_max_smem = 0;

}  // namespace

uint64_t group_stride(const DeviceIndex& x, int rs, uint32_t rows) {
  const uint64_t m8 = (x.h.m + 7) & ~7u;
  return (m8 * rows * rs + 3) & ~static_cast<uint64_t>(3);
}

int num_sms(int device) {
  int v = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

SearchPlan plan_search_uncached(const DeviceIndex& x, uint32_t B, uint32_t topn, bool scores_only);

// plans are pure functions of (index, B, topn, options): cached per index,
// so a per-query loop pays the planning (attribute queries, occupancy) once
SearchPlan plan_search(const DeviceIndex& x, uint32_t B, uint32_t topn, bool scores_only) {
  const auto key = std::make_tuple(B, topn, scores_only, options_version());
  {
    std::lock_guard<std::mutex> lk(x.plan_mu);
    auto it = x.plans.find(key);
    if (it != x.plans.end()) return *it->second;
  }
  const SearchPlan p = plan_search_uncached(x, B, topn, scores_only);
  std::lock_guard<std::mutex> lk(x.plan_mu);
  if (x.plans.size() > 256) {
    for (auto& kv : x.plans) delete kv.second;
    x.plans.clear();
  }
  auto*& slot = x.plans[key];
  if (!slot) slot = new SearchPlan(p);
  return p;
}

SearchPlan plan_search_uncached(const DeviceIndex& x, uint32_t B, uint32_t topn, bool scores_only) {
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
  // JOINT8 with a query group of <= 2: read the pre-multiplied eta*lambda table
  // (one shared load + one add per section) when it fits next to the tiles.
  const uint32_t trows = x.format == PCPQG_FMT_JOINT8 ? (1u << (x.cw + x.sw)) : 0u;
  bool found = false;
  // K2-F for PLANES 8-bit centers / 4-bit scales: groups of 4 over the fp16
  // table (the exact fp32 table of k = 256 admits only groups of 2)
  if (topk && options().scan_filter && !filter_nq16(x) && filter_layout(x) && B >= 3 && options().scan_shape == 0) {
    static const Shape fsh[] = {{256, 1, 3}, {256, 1, 2}, {128, 1, 2}};
    for (const Shape& sh : fsh) {
      uint32_t p2 = 1;
      while (p2 < topn) p2 <<= 1;
      const uint32_t cap = std::max<uint32_t>((2 * topn + 64 + 1) & ~1u, p2);
      if (static_cast<uint32_t>(sh.thr) * sh.ppt * 4 > static_cast<uint32_t>(kFQCap) / 2) continue;
      const size_t sm = scan_smem_bytes(x, 4, cap, sh.ppt, true, sh.thr, sh.stages, x.h.k, false, true);
      if (sm <= budget) {
        p.filter = true;
        p.table = false;
        p.rows = x.h.k;
        p.nq = 4;
        p.rs = rs_of(4);
        p.cap = cap;
        p.smem = sm;
        p.threads = sh.thr;
        p.ws = false;
        p.ppt = sh.ppt;
        p.stages = sh.stages;
        found = true;
        break;
      }
    }
  }
  while (!found) {
    const int forced = options().scan_shape;
    const Shape fshape[] = {{forced / 10000, (forced / 100) % 100, forced % 100}};
    const Shape* shapes = forced ? fshape : nq >= 8 ? big : small;
    const int nshape = forced ? 1 : nq >= 8 ? 4 : 5;
    // (ppt > 1: a tile of slack first, then only 256 keys — a smaller
    // candidate buffer beats dropping to fewer threads)
    for (int i = 0, sv = 0; i < nshape && !found; sv = sv ? 0 : 1, i += sv ? 0 : 1) {
      const Shape sh0 = shapes[i];
      if (sv == 1 && sh0.ppt == 1) continue;
      // warp-specialised variant: the last warp of the CTA is the TMA producer
      const bool ws = topk && nq <= options().scan_ws_max_nq && sh0.ppt > 1 && options().scan_ws &&
                      !options().fused_merge;
      const Shape sh{ws ? sh0.thr - 32 : sh0.thr, sh0.ppt, sh0.stages};
      // ppt > 1: room for a whole tile of inserts (no overflow possible);
      // ppt == 1: 2K + 64 keys and the rare overflow is retried (see try_insert)
      const uint32_t ins_max = static_cast<uint32_t>(sh.thr * sh.ppt);
      // (ppt > 1 also keeps a tile of slack so a flush is needed only after
      // another tile's worth of inserts, not after every insert)
      uint32_t p2 = 1;
      while (p2 < topn) p2 <<= 1;
      const uint32_t slack = sv == 0 ? ins_max : 256u;
      uint32_t cap = !topk ? 0 : sh.ppt > 1 ? ((topn + ins_max + slack + 1) & ~1u) : ((2 * topn + 64 + 1) & ~1u);
      if (topk) cap = std::max(cap, p2);  // the fused merge sorts pow2(K) keys in place
      const bool table = trows && nq <= 2 &&
                         scan_smem_bytes(x, nq, cap, sh.ppt, topk, sh.thr, sh.stages, trows, true) <= budget;
      const uint32_t rows = table ? trows : x.h.k;
      // K2-F: the fp16 pre-score filter for full groups of 16 over JOINT8 k = 16
      const bool filter = options().scan_filter && topk && nq == 16 && !table && !ws && sh.ppt == 1 &&
                          filter_nq16(x) && filter_layout(x) &&
                          scan_smem_bytes(x, nq, cap, sh.ppt, topk, sh.thr, sh.stages, rows, table, true) <= budget;
      const size_t sm = scan_smem_bytes(x, nq, cap, sh.ppt, topk, sh.thr, sh.stages, rows, table, filter);
      if (sm <= budget) {
        p.filter = filter;
        p.table = table;
        p.rows = rows;
        p.nq = nq;
        p.rs = rs_of(nq);
        p.cap = cap;
        p.smem = sm;
        p.threads = sh0.thr;
        p.ws = ws;
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
  ScanFn fn = pick_kernel(x, p.nq | (p.ws ? kWsFlag : 0), p.table, p.filter);
  // the device maximum, not p.smem: plans are cached, and a later plan of the
  // same kernel must not shrink the limit under an earlier one
  cudaFuncAttributes fa{};
  PCPQG_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(fn)));
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_smem - static_cast<int>(fa.sharedSizeBytes)));
  int occ = 0;
  PCPQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn),
                                                           p.threads, p.smem));
  occ = std::max(occ, 1);
  const uint64_t slots = static_cast<uint64_t>(num_sms(x.device)) * occ;
  const uint32_t tile_blocks = (p.threads - (p.ws ? 32 : 0)) * p.ppt / kBlockPts;
  // CTAs per group along the points: every CTA gets at least one full tile;
  // pick the count that makes the last wave as full as possible.
  uint32_t cmax = std::max<uint32_t>(1, x.n_blocks / tile_blocks);
  // the sorted merge stages up to 24000 survivor keys per query
  if (!scores_only)
    cmax = std::min<uint32_t>({cmax, 256u, std::max<uint32_t>(1, 24000 / std::max(topn + 1, 2u))});
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
                int mode, uint32_t rows, float* eta, cudaStream_t st, uint64_t* zero, uint32_t nzero) {
  const uint32_t msec = mode ? ((x.h.m + 7) & ~7u) : x.h.m;
  if (mode == 0) rows = x.h.k;
  const uint64_t total = static_cast<uint64_t>(Bpad) * msec * rows;
  if (total < nzero) {  // (never for a search: Bpad * m8 * rows >= Bpad + groups)
    PCPQG_CUDA(cudaMemsetAsync(zero, 0, 8ull * nzero, st));
    nzero = 0;
  }
  if (total == 0) return;
  const uint32_t threads = 256;
  const uint64_t blocks = (total + threads - 1) / threads;
  lut_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
      dQ, B, total, x.h.d, x.d_codebooks, x.d_lambda, x.h.m, msec, x.h.k, rows, x.cw,
      std::max(x.h.scales, 1u), x.h.dbar, nq, rs, mode ? group_stride(x, rs, rows) : 0, mode, eta, zero, nzero);
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

void ensure_alpha_max(const DeviceIndex& x) {
  std::call_once(x.amax_once, [&] {
    const uint32_t m8 = (x.h.m + 7) & ~7u;
    int prev = 0;
    PCPQG_CUDA(cudaGetDevice(&prev));
    PCPQG_CUDA(cudaSetDevice(x.device));
    float* d = nullptr;
    PCPQG_CUDA(cudaMalloc(&d, m8 * 4ull));
    PCPQG_CUDA(cudaMemset(d, 0, m8 * 4ull));
    const uint64_t total = x.n_local * (x.W - x.Wc);
    if (total)
      alpha_max_kernel<<<static_cast<unsigned>((total + 255) / 256), 256>>>(x.d_codes, x.n_local, x.W, x.Wc, x.h.m,
                                                                             reinterpret_cast<uint32_t*>(d));
    PCPQG_CUDA(cudaGetLastError());
    x.amax.assign(m8, 0.0f);
    PCPQG_CUDA(cudaMemcpy(x.amax.data(), d, m8 * 4ull, cudaMemcpyDeviceToHost));
    x.d_amax = d;
    cudaSetDevice(prev);
  });
}

uint64_t filter_group_stride(const DeviceIndex& x) {
  const uint64_t rows = filter_nq16(x) ? 16u : x.h.k;
  return (static_cast<uint64_t>((x.h.m + 7) & ~7u) * rows * filter_frs(x) + 7) & ~static_cast<uint64_t>(7);
}

void launch_filter_tables(const DeviceIndex& x, const SearchPlan& p, const float* eta_grouped,
                          const FilterTables& ft, cudaStream_t st) {
  const uint32_t m8 = (x.h.m + 7) & ~7u, s = std::max(x.h.scales, 1u);
  const uint32_t Bpad = p.groups * p.nq;
  const uint64_t gs = group_stride(x, p.rs, p.rows);
  float* tau = ft.work;
  float* maxlam = ft.work + m8;
  if (x.format == PCPQG_FMT_PLANES && x.sw == 16)
    ftab_alpha_kernel<<<(m8 + 63) / 64, 64, 0, st>>>(x.d_amax, m8, tau, maxlam);
  else
    ftab_lambda_kernel<<<(m8 + 63) / 64, 64, 0, st>>>(x.d_lambda, m8, s, ft.flam, tau, maxlam);
  ftab_query_kernel<<<(Bpad * 32 + 127) / 128, 128, 0, st>>>(eta_grouped, gs, p.rs, p.nq, x.h.m, p.rows, Bpad,
                                                             maxlam, ft.fse);
  const uint64_t total = static_cast<uint64_t>(p.groups) * m8 * p.rows;
  ftab_eta_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      eta_grouped, gs, p.rs, m8, p.rows, filter_frs(x), p.nq, total, tau, maxlam, ft.fse, ft.fh,
      filter_group_stride(x));
  PCPQG_CUDA(cudaGetLastError());
}

void launch_scan(const DeviceIndex& x, const SearchPlan& p, const float* eta_grouped, uint32_t B,
                 uint64_t* partial, uint64_t* gtau, float* scores, cudaStream_t st,
                 const FusedMerge* fm, const FilterTables* ft, const float* dQ) {
  ScanArgs a{};
  if (dQ) {  // the scan builds its tables itself (warp-specialised scans only)
    if (!p.ws) fail(PCPQG_E_USAGE, "in-kernel LUT needs the warp-specialised scan");
    a.Q = dQ;
    a.cb = x.d_codebooks;
    a.lut_mode = p.table ? 2u : 1u;
    a.kc = x.h.k;
    a.d = x.h.d;
    a.dbar = x.h.dbar;
  }
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
  a.k = p.rows;  // eta rows per section: centers, or code bytes in table mode
  a.s = std::max(x.h.scales, 1u);
  a.cbits = x.format == PCPQG_FMT_JOINT8 ? x.cw : 0;
  a.B = B;
  a.Bpad = p.groups * p.nq;
  a.K = p.topn;
  a.Ks = (p.topn + 1) & ~1u;
  a.cap = p.cap;
  a.ppt = p.ppt;
  a.stages = p.stages;
  a.gstride = group_stride(x, p.rs, p.rows);
  a.id_base = x.shard_begin;
  if (fm) {
    a.pcnt = fm->pcnt;
    a.done = fm->done;
    a.out_keys = fm->keys;
    a.out_ids = fm->ids;
    a.out_scores = fm->scores;
    a.out_stride = fm->out_stride;
  }
  if (p.ws && a.done) fail(PCPQG_E_USAGE, "the fused merge needs the non-specialised scan");
  if (p.filter) {
    if (!ft) fail(PCPQG_E_USAGE, "filter plan without filter tables");
    a.fh = ft->fh;
    a.flam = ft->flam;
    a.fse = ft->fse;
    a.fgstride = filter_group_stride(x);
    a.fmode = static_cast<uint32_t>(options().scan_filter);
    a.fcount = ft->count;
    a.carry = ft->carry;
    a.carry_cnt = ft->carry_cnt;
    a.carry_done = ft->carry_done;
  }
  ScanFn fn = pick_kernel(x, p.nq | (p.ws ? kWsFlag : 0), p.table, p.filter);
  dim3 grid(p.groups, p.ctas_x);
  if (p.ws && options().pdl && !dQ) {
    // small batches: the scan may start while the LUT kernel drains (it waits in
    // griddepcontrol.wait before it reads the tables; its code stream does not
    // depend on them)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PCPQG_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  } else {
    fn<<<grid, p.threads, p.smem, st>>>(a);
  }
  PCPQG_CUDA(cudaGetLastError());
}

namespace {
void launch_merge_kernel(const uint64_t* keys, const uint32_t* counts, uint32_t L, uint32_t in_rows, uint32_t B,
                         uint32_t Kin, uint32_t kout, uint32_t out_stride, const uint64_t* gtau,
                         uint64_t* keys_out, int32_t* ids, float* scores, cudaStream_t st);
}  // namespace

void merge_sorted_lists(const uint64_t* keys, const uint32_t* counts, uint32_t L, uint32_t in_rows,
                        uint32_t B, uint32_t Ks, uint32_t Kout, uint32_t out_stride,
                        uint64_t* keys_out, int32_t* ids, float* scores, cudaStream_t st) {
  if (B == 0 || L == 0) return;
  const uint64_t per = std::min(Ks, Kout) + 1;
  if (L > 32u * kTourListsPerLane || static_cast<uint64_t>(L) * per > kMergeMaxCap) {
    // more survivors than the staging buffer holds (many lists, or long
    // ones): the unsorted merge selects the Kout-th key over the lists in
    // global memory first, so no list is dropped
    if (Kout == 0 || Kout > 4096) fail(PCPQG_E_UNSUPPORTED, "topn outside the merge limits (1..4096)");
    launch_merge_kernel(keys, counts, L, in_rows, B, Ks, Kout, out_stride, nullptr, keys_out, ids, scores, st);
    return;
  }
  const uint32_t cap = static_cast<uint32_t>(L * per);
  static bool attr_set[64] = {};
  int dev = 0;
  PCPQG_CUDA(cudaGetDevice(&dev));
  if (counts && options().merge_oneshot && (Ks & 1u) == 0u && L <= 256 && Kout <= 512 &&
      static_cast<uint64_t>(L) * Ks <= kOneMaxKeys && B < static_cast<uint32_t>(num_sms(dev))) {
    const size_t sm = (static_cast<size_t>(L) * Ks + kOneDense) * 8;
    static bool one_set[64] = {};
    if (dev < 64 && !one_set[dev]) {
      PCPQG_CUDA(cudaFuncSetAttribute(merge_oneshot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((kOneMaxKeys + kOneDense) * 8)));
      one_set[dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(B);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = options().pdl ? 1 : 0;
    PCPQG_CUDA(cudaLaunchKernelEx(&cfg, merge_oneshot_kernel, keys, counts, L, in_rows, Ks, Kout, out_stride,
                                  keys_out, ids, scores));
    return;
  }
  if (dev < 64 && !attr_set[dev]) {
    PCPQG_CUDA(cudaFuncSetAttribute(merge_sorted_kernel<128>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 24576 * 8));
    PCPQG_CUDA(cudaFuncSetAttribute(merge_sorted_kernel<512>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 24576 * 8));
    attr_set[dev] = true;
  }
  // few queries: one wide CTA each selects in parallel; many: the tournament.
  // The bitonic sort of the wide path needs pow2(min(total, cap)) slots.
  uint32_t p2 = 1;
  while (p2 < cap) p2 <<= 1;
  const bool wide = B < static_cast<uint32_t>(num_sms(dev)) && p2 <= 24576 && options().merge_wide != 0;
  if (wide)
    merge_sorted_kernel<512><<<B, 512, static_cast<size_t>(p2) * 8, st>>>(
        keys, counts, L, in_rows, Ks, Kout, out_stride, cap, keys_out, ids, scores);
  else
    merge_sorted_kernel<128><<<B, 128, static_cast<size_t>(cap) * 8, st>>>(
        keys, counts, L, in_rows, Ks, Kout, out_stride, cap, keys_out, ids, scores);
  PCPQG_CUDA(cudaGetLastError());
}

void merge_lists(const uint64_t* keys, uint32_t L, uint32_t in_rows, uint32_t B, uint32_t K,
                 uint32_t out_stride, const uint64_t* gtau, uint64_t* keys_out, int32_t* ids,
                 float* scores, cudaStream_t st, uint32_t keep) {
  if (B == 0 || L == 0) return;
  if (K == 0 || K > 4096) fail(PCPQG_E_UNSUPPORTED, "topn outside the merge limits (1..4096)");
  launch_merge_kernel(keys, nullptr, L, in_rows, B, K, std::min(keep ? keep : K, out_stride), out_stride, gtau,
                      keys_out, ids, scores, st);
}

namespace {
// merge_kernel over L lists of Kin keys (optionally only their first
// counts[l][b]) -> the best Kout (<= 4096) keys per query
void launch_merge_kernel(const uint64_t* keys, const uint32_t* counts, uint32_t L, uint32_t in_rows, uint32_t B,
                         uint32_t Kin, uint32_t kout, uint32_t out_stride, const uint64_t* gtau,
                         uint64_t* keys_out, int32_t* ids, float* scores, cudaStream_t st) {
  uint32_t p2 = 1;
  while (p2 < kout) p2 <<= 1;
  const uint32_t cap = std::max<uint32_t>(std::min<uint64_t>(static_cast<uint64_t>(L) * Kin, kMergeMaxCap), p2);
  static bool attr_set[64] = {};  // per device; racing threads set the same value
  int dev = 0;
  PCPQG_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    PCPQG_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kMergeMaxCap * 8)));
    attr_set[dev] = true;
  }
  const int thr = B < 1024 ? 512 : 256;  // few queries: more threads per query
  merge_kernel<<<B, thr, cap * 8, st>>>(keys, L, in_rows, Kin, kout, out_stride, gtau, cap, keys_out,
                                        ids, scores, counts);
  PCPQG_CUDA(cudaGetLastError());
}
}  // namespace

}  // namespace pcpqg
