// Exact ground truth and recall on the GPU:
//
//   brute_force_topn (proj/core/src/eval.cpp:36-49): for every query, the
//     topn points by the exact inner product dot_qx — a double accumulation of
//     float x float products in index order (eval.cpp:18-24) — ties toward
//     the lower id.
//   recall1_single (eval.cpp:57-66): 1 iff the best exact dot over the
//     retrieved ids reaches the exact top-1 score.
//
// B200 design: an approximate pass, then an exact re-rank.
//   E1  a cuBLAS DGEMM S = Q X^T over a chunk of points (a plain library GEMM:
//       float inputs widened to double, so every product is exact; only the
//       summation order differs from the reference).
//   E2  per (query, chunk): the topn-th largest approximate score t and every
//       point with s~ >= t - 2*eps becomes a candidate.  Any summation order of
//       d exact products is within gamma_{d-1} * sum|q_j x_j| <= gamma *
//       ||q|| ||x|| of the exact sum, so the GEMM's sum and the reference's
//       sequential sum differ by at most eps = 2*gamma*||q||*max||x||.  The
//       topn points with the largest s~ all have a reference score >= t - eps,
//       so every point of the chunk's reference top-n has s~ >= t - 2*eps: the
//       rule keeps the chunk's exact top-n (ties included).
//       Every band point is rescored in the reference order right there and
//       the chunk keeps its exact top-n, so a chunk contributes <= topn
//       candidates whatever the ties.
//   E3  per query: exact top-n by (score desc, id asc) over the chunks'
//       candidates, bitonic-sorted.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "pcpqg_internal.hpp"
#include "pcpqg_device.cuh"

namespace pcpqg {
namespace {

__global__ void to_double_kernel(const float* __restrict__ x, uint64_t cnt, double* __restrict__ y) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < cnt) y[t] = static_cast<double>(x[t]);
}

// ||row||_2 (rounded up a little: a bound, not a value)
__global__ void row_norm_kernel(const float* __restrict__ x, uint64_t rows, uint32_t d,
                                double* __restrict__ out, unsigned long long* __restrict__ max_bits) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows) return;
  const float* r = x + t * d;
  double s = 0.0;
  for (uint32_t i = 0; i < d; ++i) s = fma(static_cast<double>(r[i]), static_cast<double>(r[i]), s);
  const double nrm = sqrt(s) * (1.0 + 1e-12);
  if (out) out[t] = nrm;
  if (max_bits) atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(nrm)));
}

__device__ __forceinline__ double dot_qx(const float* q, const float* x, uint32_t d) {
  double acc = 0.0;  // dot_qx: index order, no contraction (eval.cpp:18-24)
  for (uint32_t a = 0; a < d; ++a)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(q[a]), static_cast<double>(x[a])));
  return acc;
}

// E2: one CTA per query over one chunk of P approximate scores S[b][.]:
//  1. t = the keep-th largest approximate score;
//  2. every point of the band s~ >= t - 2*eps gets its exact (reference-order)
//     score, written over its S entry; the others become -inf (excluded);
//  3. the chunk's exact top-keep by (score desc, id asc) among the band —
//     which is the chunk's exact top-keep — goes to the candidate slots
//     [b][chunk][0, keep) with its exact scores.  At most topn per chunk, so
//     massive ties (an all-zero query) cannot overflow anything.
__global__ void __launch_bounds__(512)
    gt_chunk_select_kernel(double* __restrict__ S, uint32_t P, uint64_t p0, uint32_t topn,
                           const float* __restrict__ X, uint32_t d, const float* __restrict__ Q,
                           const double* __restrict__ qnorm, const unsigned long long* __restrict__ xmax_bits,
                           double gamma, uint32_t chunk, uint32_t nchunks, uint32_t* __restrict__ cand,
                           double* __restrict__ cand_s, uint32_t* __restrict__ ccount) {
  __shared__ uint32_t hist[256];
  __shared__ Sel96 sel;
  __shared__ unsigned long long s_min;
  __shared__ uint32_t s_band, s_n;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  double* s = S + static_cast<uint64_t>(b) * P;
  const float* q = Q + static_cast<uint64_t>(b) * d;
  const uint32_t keep = min(topn, P);
  double thr = -INFINITY;
  if (keep < P) {
    select96(
        [&](uint64_t i, uint64_t& h, uint32_t& l) {
          h = ord64(s[i]);
          l = static_cast<uint32_t>(i);  // unique keys; only the value order matters
          return true;
        },
        P, keep, P, hist, sel);
    if (tid == 0) s_min = ~0ull;
    __syncthreads();
    unsigned long long mn = ~0ull;
    for (uint32_t i = tid; i < P; i += nthr) {
      const uint64_t h = ord64(s[i]);
      if (sel96_take(sel, h, i)) mn = min(mn, static_cast<unsigned long long>(h));
    }
    atomicMin(&s_min, mn);
    __syncthreads();
    const uint64_t o = s_min;  // the keep-th largest approximate score
    const double t = __longlong_as_double(static_cast<long long>((o >> 63) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o));
    // eps bounds |GEMM sum - reference sum|: two summation orders, each within
    // gamma * ||q|| * ||x|| of the exact value
    const double eps = 2.0 * gamma * qnorm[b] * __longlong_as_double(static_cast<long long>(*xmax_bits));
    thr = t - 2.0 * eps * (1.0 + 1e-6);
  }
  if (tid == 0) {
    s_band = 0;
    s_n = 0;
  }
  __syncthreads();
  uint32_t band = 0;
  for (uint32_t i = tid; i < P; i += nthr) {
    if (s[i] >= thr) {
      s[i] = dot_qx(q, X + (p0 + i) * d, d);
      ++band;
    } else {
      s[i] = -INFINITY;
    }
  }
  atomicAdd(&s_band, band);
  __syncthreads();
  const uint32_t nband = s_band;
  const uint32_t kk = min(keep, nband);
  auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) {
    h = ord64(s[i]);
    l = ~static_cast<uint32_t>(p0 + i);
    return s[i] != -INFINITY;
  };
  select96(get, P, kk, nband, hist, sel);
  const uint64_t base = (static_cast<uint64_t>(b) * nchunks + chunk) * topn;
  for (uint32_t i = tid; i < P; i += nthr) {
    uint64_t h;
    uint32_t l;
    if (!get(i, h, l) || !sel96_take(sel, h, l)) continue;
    const uint32_t slot = atomicAdd(&s_n, 1u);
    if (slot < kk) {
      cand[base + slot] = ~l;
      cand_s[base + slot] = s[i];
    }
  }
  __syncthreads();
  if (tid == 0) ccount[static_cast<uint64_t>(b) * nchunks + chunk] = min(s_n, kk);
}

// E3: the exact top-n over the chunks' exact candidates, sorted.
constexpr uint32_t kGtMaxTop = 4096;

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

cublasHandle_t cublas_for(int device) {
  static std::mutex mu;
  static cublasHandle_t h[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) fail(PCPQG_E_USAGE, "bad device ordinal");
  if (!h[device]) {
    if (cublasCreate(&h[device]) != CUBLAS_STATUS_SUCCESS) fail(PCPQG_E_CUDA, "cublasCreate failed");
  }
  return h[device];
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
  cublasHandle_t h = cublas_for(device);
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) fail(PCPQG_E_CUDA, "cublasSetStream failed");
  // gamma_{d-1} = (d-1)u / (1 - (d-1)u), u = 2^-53, with a safety factor
  const double u = std::ldexp(1.0, -53);
  const double gamma = 1.01 * (d * u) / (1.0 - d * u);
  // point chunk: the approximate score block [B][P] stays within ~4 GB
  uint64_t P = std::max<uint64_t>(4096, std::min<uint64_t>({n, (4ull << 30) / (8ull * B), 1ull << 20}));
  if (options().gt_chunk > 0) P = static_cast<uint64_t>(options().gt_chunk);
  const uint64_t nchunks = (n + P - 1) / P;
  if (nchunks > 0xFFFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "brute_force_topn: too many chunks");
  std::vector<void*> keep;
  double* Q64 = galloc<double>(keep, static_cast<size_t>(B) * d, st);
  double* X64 = galloc<double>(keep, P * d, st);
  double* S = galloc<double>(keep, P * B, st);
  double* qn = galloc<double>(keep, B, st);
  unsigned long long* xmax = galloc<unsigned long long>(keep, 2, st);
  const uint64_t slots = static_cast<uint64_t>(B) * nchunks * topn;
  uint32_t* cand = galloc<uint32_t>(keep, slots, st);
  double* cand_s = galloc<double>(keep, slots, st);
  uint32_t* ccount = galloc<uint32_t>(keep, static_cast<uint64_t>(B) * nchunks, st);
  PCPQG_CUDA(cudaMemsetAsync(xmax, 0, 16, st));
  const uint64_t bd = static_cast<uint64_t>(B) * d;
  to_double_kernel<<<static_cast<unsigned>((bd + 255) / 256), 256, 0, st>>>(dQ, bd, Q64);
  row_norm_kernel<<<(B + 255) / 256, 256, 0, st>>>(dQ, B, d, qn, nullptr);
  row_norm_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(dX, n, d, nullptr, xmax);
  PCPQG_CUDA(cudaGetLastError());
  const double one = 1.0, zero = 0.0;
  uint32_t chunk = 0;
  for (uint64_t p0 = 0; p0 < n; p0 += P, ++chunk) {
    const uint32_t pc = static_cast<uint32_t>(std::min<uint64_t>(P, n - p0));
    const uint64_t cnt = static_cast<uint64_t>(pc) * d;
    to_double_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(dX + p0 * d, cnt, X64);
    PCPQG_CUDA(cudaGetLastError());
    // row-major S[B][pc] = Q64[B][d] X64[pc][d]^T: column-major S^T = op(X64) * Q64^T
    if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(pc), static_cast<int>(B),
                    static_cast<int>(d), &one, X64, static_cast<int>(d), Q64, static_cast<int>(d), &zero, S,
                    static_cast<int>(pc)) != CUBLAS_STATUS_SUCCESS)
      fail(PCPQG_E_CUDA, "cublasDgemm failed");
    gt_chunk_select_kernel<<<B, 512, 0, st>>>(S, pc, p0, topn, dX, d, dQ, qn, xmax, gamma, chunk,
                                              static_cast<uint32_t>(nchunks), cand, cand_s, ccount);
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
