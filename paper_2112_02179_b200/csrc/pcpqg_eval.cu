// Exact ground truth and recall on the GPU:
//
//   brute_force_topn (proj/core/src/eval.cpp:36-49): for every query, the
//     topn points by the exact inner product dot_qx — a double accumulation of
//     float x float products in index order (eval.cpp:18-24) — ties toward
//     the lower id.
//   recall1_single (eval.cpp:57-66): 1 iff the best exact dot over the
//     retrieved ids reaches the exact top-1 score.
//
// B200 design: a tensor-core pre-score filter, then an exact re-rank.
//   E1  GT-T (pcpqg_tscan.cu): the raw points, scaled by a power of two and
//       rounded to fp16, are the operands of the K2-T filter kernel (TMA ->
//       shared memory -> tcgen05.mma kind::f16, fp32 accumulators in TMEM); per
//       query it keeps the points whose approximate score lies within 2*eps of
//       a lower bound of the K-th best, eps a proven bound on |approx - exact|.
//   E2  gt_tfinish_kernel re-scores those pairs in the reference's order
//       (sequential fp64, index order) and keeps the chunk's exact top-n by
//       (score desc, id asc).  Queries the filter cannot serve (outside the
//       scaling range, or more than a list of points within 2*eps of each
//       other: an all-zero query) are flagged; gt_chunk_exact_kernel scores
//       every point of the chunk for them.  The same kernel is the whole path
//       for small inputs, N > 256 and dimensions above the filter's tile.
//   E3  per query: exact top-n by (score desc, id asc) over the chunks'
//       candidates, bitonic-sorted.
// No library GEMM: the contraction is the repo's own tcgen05 kernel.
#include <algorithm>
#include <cmath>

#include "pcpqg_internal.hpp"
#include "pcpqg_device.cuh"

namespace pcpqg {
namespace {

__device__ __forceinline__ double dot_qx(const float* q, const float* x, uint32_t d) {
  double acc = 0.0;  // dot_qx: index order, no contraction (eval.cpp:18-24)
  for (uint32_t a = 0; a < d; ++a)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(q[a]), static_cast<double>(x[a])));
  return acc;
}

constexpr uint32_t kGtMaxTop = 4096;
constexpr uint32_t kGtSub = 4096;    // points scored per round of the exact kernel
constexpr uint32_t kGtThreads = 512;
constexpr uint32_t kGtPerThread = (kGtMaxTop + kGtSub) / kGtThreads;  // 16

// E2': one CTA per query over one chunk of pc points, every point scored in
// the reference's order.  The CTA keeps its best `keep` (score, id) pairs in
// shared memory; a round scores kGtSub points and appends those that beat the
// current keep-th best, and an exact 96-bit selection trims the set when it
// outgrows keep.  With fallback != nullptr only the flagged queries run.
__global__ void __launch_bounds__(kGtThreads)
    gt_chunk_exact_kernel(const float* __restrict__ X, uint64_t pc, uint64_t p0, uint32_t d,
                          const float* __restrict__ Q, uint32_t topn, const uint32_t* __restrict__ fallback,
                          uint32_t* __restrict__ cand, double* __restrict__ cand_s, uint32_t* __restrict__ ccount,
                          uint32_t out_stride, uint32_t count_stride) {
  extern __shared__ __align__(16) uint8_t smem_e[];
  __shared__ uint32_t hist[256];
  __shared__ Sel96 sel;
  __shared__ uint32_t s_n, s_w, s_minl;
  __shared__ unsigned long long s_minh;
  const uint32_t b = blockIdx.x, tid = threadIdx.x;
  if (fallback && !fallback[b]) return;
  const uint32_t keep = static_cast<uint32_t>(min(static_cast<uint64_t>(topn), pc));
  double* sc = reinterpret_cast<double*>(smem_e);            // keep + kGtSub scores
  uint32_t* id = reinterpret_cast<uint32_t*>(sc + keep + kGtSub);
  const float* q = Q + static_cast<uint64_t>(b) * d;
  if (tid == 0) s_n = 0;
  __syncthreads();
  bool full = false;      // the set holds keep pairs and (th, tl) is its worst key
  uint64_t th = 0;
  uint32_t tl = 0;
  for (uint64_t sub0 = 0; sub0 < pc; sub0 += kGtSub) {
    const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(kGtSub), pc - sub0));
    for (uint32_t i = tid; i < cnt; i += kGtThreads) {
      const uint64_t p = sub0 + i;
      const double s = dot_qx(q, X + p * d, d);
      const uint64_t h = ord64(s);
      const uint32_t gid = static_cast<uint32_t>(p0 + p);
      const uint32_t l = ~gid;
      if (!full || h > th || (h == th && l > tl)) {
        const uint32_t slot = atomicAdd(&s_n, 1u);
        sc[slot] = s;
        id[slot] = gid;
      }
    }
    __syncthreads();
    const uint32_t n = s_n;
    if (n <= keep) {
      if (n < keep || full) continue;  // (n == keep, first time full: fall through for the threshold)
    }
    auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) {
      h = ord64(sc[i]);
      l = ~id[i];
      return true;
    };
    if (n > keep) {
      select96(get, n, keep, n, hist, sel);
      // in-place compaction through registers (n <= keep + kGtSub <= 16 per thread)
      double rs[kGtPerThread];
      uint32_t ri[kGtPerThread], rslot[kGtPerThread];
      if (tid == 0) s_w = 0;
      __syncthreads();
#pragma unroll
      for (uint32_t u = 0; u < kGtPerThread; ++u) {
        const uint32_t i = tid + u * kGtThreads;
        rslot[u] = 0xFFFFFFFFu;
        if (i < n) {
          uint64_t h;
          uint32_t l;
          get(i, h, l);
          if (sel96_take(sel, h, l)) {
            rs[u] = sc[i];
            ri[u] = id[i];
            rslot[u] = atomicAdd(&s_w, 1u);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (uint32_t u = 0; u < kGtPerThread; ++u)
        if (rslot[u] != 0xFFFFFFFFu && rslot[u] < keep) {
          sc[rslot[u]] = rs[u];
          id[rslot[u]] = ri[u];
        }
      if (tid == 0) s_n = min(s_w, keep);
      __syncthreads();
    }
    // the worst key of the (now full) set
    if (tid == 0) {
      s_minh = ~0ull;
      s_minl = ~0u;
    }
    __syncthreads();
    {
      unsigned long long mh = ~0ull;
      for (uint32_t i = tid; i < keep; i += kGtThreads) mh = min(mh, static_cast<unsigned long long>(ord64(sc[i])));
      atomicMin(&s_minh, mh);
      __syncthreads();
      uint32_t ml = ~0u;
      for (uint32_t i = tid; i < keep; i += kGtThreads)
        if (ord64(sc[i]) == s_minh) ml = min(ml, ~id[i]);
      atomicMin(&s_minl, ml);
      __syncthreads();
    }
    full = true;
    th = s_minh;
    tl = s_minl;
    __syncthreads();
  }
  const uint32_t n = min(s_n, keep);
  const uint64_t base = static_cast<uint64_t>(b) * out_stride;
  for (uint32_t i = tid; i < n; i += kGtThreads) {
    cand[base + i] = id[i];
    cand_s[base + i] = sc[i];
  }
  if (tid == 0) ccount[static_cast<uint64_t>(b) * count_stride] = n;
}

// E3: the exact top-n over the chunks' exact candidates, sorted.

__global__ void __launch_bounds__(512)
    gt_final_kernel(const uint32_t* __restrict__ cand, const double* __restrict__ cand_s,
                    const uint32_t* __restrict__ ccount, uint32_t nchunks, uint32_t topn,
                    int32_t* __restrict__ ids, double* __restrict__ scores) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t hist[256];
  __shared__ Sel96 sel;
  __shared__ uint32_t s_n, s_valid;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t base = static_cast<uint64_t>(b) * nchunks * topn;
  const uint64_t nslots = static_cast<uint64_t>(nchunks) * topn;
  if (tid == 0) {
    s_n = 0;
    s_valid = 0;
  }
  __syncthreads();
  {
    uint32_t v = 0;
    for (uint32_t c = tid; c < nchunks; c += nthr) v += ccount[static_cast<uint64_t>(b) * nchunks + c];
    atomicAdd(&s_valid, v);
  }
  __syncthreads();
  auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) {
    const uint32_t c = static_cast<uint32_t>(i / topn), j = static_cast<uint32_t>(i % topn);
    if (j >= ccount[static_cast<uint64_t>(b) * nchunks + c]) return false;
    h = ord64(cand_s[base + i]);
    l = ~cand[base + i];
    return true;
  };
  const uint32_t nvalid = s_valid;
  const uint32_t keep = min(topn, nvalid);
  select96(get, nslots, keep, nvalid, hist, sel);
  uint64_t* k_hi = reinterpret_cast<uint64_t*>(smem);
  uint32_t* k_id = reinterpret_cast<uint32_t*>(k_hi + kGtMaxTop);
  uint32_t* k_ix = k_id + kGtMaxTop;
  for (uint64_t i = tid; i < nslots; i += nthr) {
    uint64_t h;
    uint32_t l;
    if (!get(i, h, l) || !sel96_take(sel, h, l)) continue;
    const uint32_t slot = atomicAdd(&s_n, 1u);
    if (slot < keep) {
      k_hi[slot] = h;
      k_id[slot] = ~l;
      k_ix[slot] = static_cast<uint32_t>(i);
    }
  }
  __syncthreads();
  uint32_t P2 = 1;
  while (P2 < keep) P2 <<= 1;
  for (uint32_t i = keep + tid; i < P2; i += nthr) {
    k_hi[i] = 0ull;
    k_id[i] = 0xFFFFFFFFu;
    k_ix[i] = 0u;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P2; size <<= 1)
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < P2 / 2; i += nthr) {
        const uint32_t lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool hi_better = k_hi[hi] > k_hi[lo] || (k_hi[hi] == k_hi[lo] && k_id[hi] < k_id[lo]);
        if (hi_better == ((lo & size) == 0)) {
          const uint64_t th = k_hi[lo];
          k_hi[lo] = k_hi[hi];
          k_hi[hi] = th;
          const uint32_t ti = k_id[lo];
          k_id[lo] = k_id[hi];
          k_id[hi] = ti;
          const uint32_t tx = k_ix[lo];
          k_ix[lo] = k_ix[hi];
          k_ix[hi] = tx;
        }
      }
      __syncthreads();
    }
  for (uint32_t i = tid; i < topn; i += nthr) {
    const uint64_t o = static_cast<uint64_t>(b) * topn + i;
    ids[o] = i < keep ? static_cast<int32_t>(k_id[i]) : -1;
    scores[o] = i < keep ? cand_s[base + k_ix[i]] : __longlong_as_double(0x7FF8000000000000ll);
  }
}

// recall1_single: best exact dot over the retrieved ids vs the exact top-1
__global__ void recall1_kernel(const float* __restrict__ X, uint64_t n, uint32_t d,
                               const float* __restrict__ Q, uint32_t B, const uint32_t* __restrict__ ret,
                               uint32_t R, const double* __restrict__ top1, int32_t* __restrict__ hits,
                               uint32_t* __restrict__ err) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const float* q = Q + static_cast<uint64_t>(b) * d;
  double best = -INFINITY;
  for (uint32_t i = 0; i < R; ++i) {
    const uint32_t id = ret[static_cast<uint64_t>(b) * R + i];
    if (id >= n) {
      atomicOr(err, 1u);
      return;
    }
    const float* x = X + static_cast<uint64_t>(id) * d;
    double acc = 0.0;
    for (uint32_t a = 0; a < d; ++a)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(q[a]), static_cast<double>(x[a])));
    best = acc > best ? acc : best;
  }
  hits[b] = best >= top1[b] ? 1 : 0;
}

template <class T>
T* galloc(std::vector<void*>& keep, size_t n, cudaStream_t st) {
  void* p = nullptr;
  PCPQG_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
  keep.push_back(p);
  return static_cast<T*>(p);
}

}  // namespace

void brute_force_topn(const float* dX, uint64_t n, uint32_t d, const float* dQ, uint32_t B,
                      uint32_t topn, int32_t* d_ids, double* d_scores, int device, cudaStream_t st) {
  if (topn < 1 || topn > n) fail(PCPQG_E_DATA, "brute_force_topn: need 1 <= N <= n");
  if (topn > kGtMaxTop) fail(PCPQG_E_UNSUPPORTED, "brute_force_topn: N above 4096");
  if (B == 0) return;
  keep_mempool(device);
  const bool tc = gt_tscan_eligible(n, d, B, topn, device);
  // point chunks: the tensor filter's fp16 operand cache bounds a chunk; the
  // exact kernel's ids are 32-bit
  uint64_t P = tc ? gt_tscan_chunk_points(n, d, device) : std::min<uint64_t>(n, 1ull << 31);
  if (!tc && options().gt_chunk > 0) P = std::min<uint64_t>(n, std::max<int>(1, options().gt_chunk));
  const uint64_t nchunks = (n + P - 1) / P;
  if (nchunks > 0xFFFFull) fail(PCPQG_E_UNSUPPORTED, "brute_force_topn: too many chunks");
  if (n > 0xFFFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "brute_force_topn: more than 2^32 points");
  std::vector<void*> keep;
  const uint64_t slots = static_cast<uint64_t>(B) * nchunks * topn;
  uint32_t* cand = galloc<uint32_t>(keep, slots, st);
  double* cand_s = galloc<double>(keep, slots, st);
  uint32_t* ccount = galloc<uint32_t>(keep, static_cast<uint64_t>(B) * nchunks, st);
  uint32_t* fallback = galloc<uint32_t>(keep, B, st);
  void* stats = nullptr;
  if (tc) {
    stats = galloc<uint8_t>(keep, gt_stats_bytes(), st);
    gt_stats(dX, n, d, stats, st);
  }
  const uint32_t ostride = static_cast<uint32_t>(nchunks * topn);
  const size_t esm = (static_cast<size_t>(std::min<uint64_t>(topn, P)) + kGtSub) * 12 + 16;
  PCPQG_CUDA(cudaFuncSetAttribute(gt_chunk_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>((kGtMaxTop + kGtSub) * 12 + 16)));
  uint32_t chunk = 0;
  for (uint64_t p0 = 0; p0 < n; p0 += P, ++chunk) {
    const uint64_t pc = std::min<uint64_t>(P, n - p0);
    uint32_t* c_ids = cand + static_cast<uint64_t>(chunk) * topn;
    double* c_sc = cand_s + static_cast<uint64_t>(chunk) * topn;
    const bool tcc = tc && pc >= 4096;  // (a short last chunk is scored exactly)
    if (tcc) {
      std::vector<void*> scratch;
      PCPQG_CUDA(cudaMemsetAsync(fallback, 0, 4ull * B, st));
      gt_tscan_chunk(dX + p0 * d, pc, p0, d, dQ, B, topn, stats, c_ids, c_sc, ccount + chunk, ostride,
                     static_cast<uint32_t>(nchunks), fallback, device,
                     [&](size_t bytes) { return static_cast<void*>(galloc<uint8_t>(scratch, bytes, st)); }, st,
                     nullptr);
      for (void* p : scratch) PCPQG_CUDA(cudaFreeAsync(p, st));
    }
    gt_chunk_exact_kernel<<<B, kGtThreads, esm, st>>>(dX + p0 * d, pc, p0, d, dQ, topn, tcc ? fallback : nullptr, c_ids,
                                                      c_sc, ccount + chunk, ostride, static_cast<uint32_t>(nchunks));
    PCPQG_CUDA(cudaGetLastError());
  }
  PCPQG_CUDA(cudaFuncSetAttribute(gt_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGtMaxTop * 16)));
  gt_final_kernel<<<B, 512, kGtMaxTop * 16, st>>>(cand, cand_s, ccount, static_cast<uint32_t>(nchunks),
                                                  topn, d_ids, d_scores);
  PCPQG_CUDA(cudaGetLastError());
  for (void* p : keep) PCPQG_CUDA(cudaFreeAsync(p, st));
}

void recall1(const float* dX, uint64_t n, uint32_t d, const float* dQ, uint32_t B,
             const uint32_t* d_ret, uint32_t R, const double* d_top1, int32_t* d_hits, cudaStream_t st) {
  if (B == 0) return;
  std::vector<void*> keep;
  uint32_t* err = galloc<uint32_t>(keep, 1, st);
  PCPQG_CUDA(cudaMemsetAsync(err, 0, 4, st));
  recall1_kernel<<<(B + 127) / 128, 128, 0, st>>>(dX, n, d, dQ, B, d_ret, R, d_top1, d_hits, err);
  PCPQG_CUDA(cudaGetLastError());
  uint32_t h = 0;
  PCPQG_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
  for (void* p : keep) PCPQG_CUDA(cudaFreeAsync(p, st));
  PCPQG_CUDA(cudaStreamSynchronize(st));
  if (h) fail(PCPQG_E_DATA, "recall1_single: id out of range");
}

}  // namespace pcpqg
