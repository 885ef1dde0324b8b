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
ScanFn scan_fn_p4(uint32_t sw, bool k16, int nq);
ScanFn scan_fn_p8(uint32_t sw, int nq);
ScanFn scan_fn_p16(uint32_t sw, int nq);

namespace {

ScanFn pick_kernel(const DeviceIndex& x, int nq) {
  const bool k16 = x.h.k == 16;
  ScanFn f = nullptr;
  if (x.format == PCPQG_FMT_JOINT8) f = scan_fn_joint8(k16, nq);
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
  __shared__ uint32_t hist[kGroupScratch];
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
  b += topk ? static_cast<size_t>(ngroups) * (kGroupScratch) * 4 : 0;
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
