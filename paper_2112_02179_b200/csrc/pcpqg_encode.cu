// Encode path (secondary, config 5): per-point center assignment and
// score-aware scale codes, in fp64 with the reference's operation order so
// the codes are bit-identical.  Every multiply/add/divide is an explicit
// round-to-nearest intrinsic: no FMA contraction (the reference is built
// without -march, so GCC emits separate mulsd/addsd).
//
//   assign_projective_kernel   pcpq::assign_projective   clustering.cpp:250-289
//   assign_aniso_kernel        pcpq::assign_anisotropic  clustering.cpp:298-368
//                              (allow_scaling true or false, optional previous
//                              assignment: assign_aniso_impl)
//   aniso_alpha_codes_kernel   quantize_anisotropic code assignment
//                              scalar_quant.cpp:121-150 (+ nearest_code :28-39)
//
// Layout: one section's vectors x[n][dbar] (fp32) and centers[k][dbar]; one
// thread per point; the k center rows and their squared norms are staged in
// shared memory once per CTA.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "pcpqg_internal.hpp"

namespace pcpqg {
namespace {

constexpr int kEncThreads = 256;

// dotf of clustering.cpp:14-19: widen to double, sequential from 0.0
__device__ __forceinline__ double dotf(const float* a, const float* b, uint32_t n) {
  double acc = 0.0;
  for (uint32_t i = 0; i < n; ++i)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(a[i]), static_cast<double>(b[i])));
  return acc;
}

// std::max(v, 0.0) returns v unless v < 0 (so -0.0 stays -0.0)
__device__ __forceinline__ double clamp0(double v) { return v < 0.0 ? 0.0 : v; }

// opt_alpha_from, clustering.cpp:36-40
__device__ __forceinline__ double opt_alpha_from(double ip, double nx2, double c2, double hp,
                                                 double hb) {
  const double denom =
      __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), ip), ip), nx2), __dmul_rn(hb, c2));
  if (fabs(denom) <= 1e-30) return 0.0;
  return __ddiv_rn(__dmul_rn(hp, ip), denom);
}

// stage centers + squared norms in shared memory
__device__ void stage_centers(const float* centers, uint32_t k, uint32_t dbar, float* s_c,
                              double* s_c2) {
  for (uint32_t i = threadIdx.x; i < k * dbar; i += blockDim.x) s_c[i] = centers[i];
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) s_c2[j] = dotf(s_c + j * dbar, s_c + j * dbar, dbar);
  __syncthreads();
}

__global__ void __launch_bounds__(kEncThreads)
    assign_projective_kernel(const float* __restrict__ x, uint64_t n, uint32_t dbar,
                             const float* __restrict__ centers, uint32_t k,
                             uint32_t* __restrict__ assign, double* __restrict__ alpha,
                             double* __restrict__ loss) {
  extern __shared__ double s_mem[];
  double* s_c2 = s_mem;
  float* s_c = reinterpret_cast<float*>(s_mem + k);
  stage_centers(centers, k, dbar, s_c, s_c2);
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* xi = x + i * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) {
      assign[i] = 0;
      alpha[i] = 0.0;
      if (loss) loss[i] = 0.0;
      continue;
    }
    double best = INFINITY, bip = 0.0;
    uint32_t bj = 0;
    for (uint32_t j = 0; j < k; ++j) {
      const double ip = dotf(xi, s_c + j * dbar, dbar);
      const double l = __dsub_rn(nx2, __ddiv_rn(__dmul_rn(ip, ip), s_c2[j]));
      if (l < best) {  // strict: ties keep the lowest index
        best = l;
        bj = j;
        bip = ip;
      }
    }
    assign[i] = bj;
    alpha[i] = __ddiv_rn(bip, s_c2[bj]);
    if (loss) loss[i] = clamp0(best);
  }
}

__global__ void __launch_bounds__(kEncThreads)
    assign_aniso_kernel(const float* __restrict__ x, uint64_t n, uint32_t dbar,
                        const float* __restrict__ centers, uint32_t k,
                        const double* __restrict__ h_par, const double* __restrict__ h_bot,
                        const uint32_t* __restrict__ prev, bool scaling, uint32_t* __restrict__ assign,
                        double* __restrict__ alpha, double* __restrict__ loss) {
  extern __shared__ double s_mem[];
  double* s_c2 = s_mem;
  float* s_c = reinterpret_cast<float*>(s_mem + k);
  stage_centers(centers, k, dbar, s_c, s_c2);
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* xi = x + i * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) {
      assign[i] = 0;
      alpha[i] = 0.0;
      if (loss) loss[i] = 0.0;
      continue;
    }
    const double hp = h_par[i], hb = h_bot[i];
    double bdist = INFINITY, balpha = 1.0;
    uint32_t bj = 0;
    if (!scaling) {
      // fixed unit scale (anisotropic_k_clustering): argmin quad_at(point_quad, 1.0)
      const double qb = __dmul_rn(hp, nx2);
      double bloss = INFINITY;
      for (uint32_t j = 0; j < k; ++j) {
        const double ip = dotf(xi, s_c + j * dbar, dbar);
        const double w = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), ip), ip), nx2),
                                   __dmul_rn(hb, s_c2[j]));
        const double qa = __dmul_rn(__dmul_rn(-2.0, hp), ip);
        const double l = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(w, 1.0), qa), 1.0), qb);
        if (l < bloss) {
          bloss = l;
          bj = j;
        }
      }
      assign[i] = bj;
      alpha[i] = 1.0;
      if (loss) loss[i] = clamp0(bloss);
      continue;
    }
    for (uint32_t j = 0; j < k; ++j) {
      const double ip = dotf(xi, s_c + j * dbar, dbar);
      const double beta = opt_alpha_from(ip, nx2, s_c2[j], hp, hb);
      // nx2 - 2.0 * beta * ip + beta * beta * c2   (left to right)
      const double dist = __dadd_rn(__dsub_rn(nx2, __dmul_rn(__dmul_rn(2.0, beta), ip)),
                                    __dmul_rn(__dmul_rn(beta, beta), s_c2[j]));
      if (dist < bdist) {
        bdist = dist;
        bj = j;
        balpha = beta;
      }
    }
    // quad_at(point_quad(bip, nx2, c2, w), balpha), clustering.cpp:29-34
    const double bip = dotf(xi, s_c + bj * dbar, dbar);
    const double c2 = s_c2[bj];
    const double w = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), bip), bip), nx2),
                               __dmul_rn(hb, c2));
    const double qa = __dmul_rn(__dmul_rn(-2.0, hp), bip);
    const double qb = __dmul_rn(hp, nx2);
    double bloss = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(w, balpha), qa), balpha), qb);
    // keep the previous center if switching would raise this point's own
    // score-aware loss (clustering.cpp:339-349)
    if (prev && prev[i] != bj) {
      const uint32_t pj = prev[i];
      const double pip = dotf(xi, s_c + pj * dbar, dbar);
      const double pc2 = s_c2[pj];
      const double pbeta = opt_alpha_from(pip, nx2, pc2, hp, hb);
      const double pw = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), pip), pip), nx2),
                                  __dmul_rn(hb, pc2));
      const double pa = __dmul_rn(__dmul_rn(-2.0, hp), pip);
      const double ploss = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(pw, pbeta), pa), pbeta), qb);
      if (ploss < bloss) {
        bj = pj;
        balpha = pbeta;
        bloss = ploss;
      }
    }
    assign[i] = bj;
    alpha[i] = balpha;
    if (loss) loss[i] = clamp0(bloss);
  }
}

__global__ void __launch_bounds__(kEncThreads)
    aniso_alpha_codes_kernel(const float* __restrict__ x, uint64_t n, uint32_t dbar,
                             const float* __restrict__ centers, const uint32_t* __restrict__ assign,
                             const double* __restrict__ h_par, const double* __restrict__ h_bot,
                             const float* __restrict__ values, uint32_t s,
                             uint8_t* __restrict__ codes) {
  __shared__ float s_v[256];
  for (uint32_t l = threadIdx.x; l < s; l += blockDim.x) s_v[l] = values[l];
  __syncthreads();
  // nearest_code(values, 0.0): argmin |v - 0|, strict <
  uint32_t zero_code = 0;
  double bd = INFINITY;
  for (uint32_t l = 0; l < s; ++l) {
    const double dd = fabs(__dsub_rn(static_cast<double>(s_v[l]), 0.0));
    if (dd < bd) {
      bd = dd;
      zero_code = l;
    }
  }
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* xi = x + i * dbar;
    const float* c = centers + static_cast<uint64_t>(assign[i]) * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) {
      codes[i] = static_cast<uint8_t>(zero_code);
      continue;
    }
    const double c2 = dotf(c, c, dbar);
    const double ip = dotf(xi, c, dbar);
    const double hp = h_par[i], hb = h_bot[i];
    const double wq = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), ip), ip), nx2),
                                __dmul_rn(hb, c2));
    if (!(wq > 0.0)) {
      codes[i] = static_cast<uint8_t>(zero_code);
      continue;
    }
    const double qa = __dmul_rn(__dmul_rn(-2.0, hp), ip);
    const double qb = __dmul_rn(hp, nx2);
    double best = INFINITY;
    uint32_t bl = 0;
    for (uint32_t l = 0; l < s; ++l) {
      const double lam = s_v[l];
      const double v = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(wq, lam), qa), lam), qb);
      if (v < best) {
        best = v;
        bl = l;
      }
    }
    codes[i] = static_cast<uint8_t>(bl);
  }
}

// center_anisotropic statistics (clustering.cpp:382-402).  Only the final
// additions depend on order, so the work splits in two:
//   center_terms_kernel  (parallel)  every member's S terms, written in
//                        cluster-sorted (id-ordered) position: fl(fl(coef*xa)*xb),
//                        fl(fl(alpha*h_par)*xa), fl(alpha^2*h_bot) — zeros for a
//                        zero-norm point, which the reference skips (adding +0.0
//                        to a sum that started at +0.0 never changes its bits)
//   center_chain_kernel  (sequential per (section, cluster, stat)) adds the
//                        terms in member order onto the incoming partial, the
//                        reference's exact summation order.
// Stats per cluster: M upper triangle (a <= b, row-major), rhs[dbar], diag.
__global__ void center_terms_kernel(const float* __restrict__ x, uint32_t dbar, uint64_t n,
                                    uint64_t sec_stride, uint32_t sec0, uint32_t nsec,
                                    const uint32_t* __restrict__ order,
                                    const double* __restrict__ alpha, const double* __restrict__ hp,
                                    const double* __restrict__ hb, double* __restrict__ terms) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(nsec) * n) return;
  const uint32_t jl = static_cast<uint32_t>(t / n);  // section within this batch
  const uint64_t p = t % n;                          // sorted position
  const uint32_t j = sec0 + jl;
  const uint32_t S = dbar * (dbar + 1) / 2 + dbar + 1;
  const uint32_t id = order[static_cast<size_t>(j) * n + p];
  const float* xi = x + static_cast<size_t>(j) * sec_stride + static_cast<size_t>(id) * dbar;
  // stat-major: terms[jl][s][p] with rows of n2 = n rounded up to even (16-byte
  // aligned), so a chain reads one contiguous, vector-loadable run
  const uint64_t n2 = (n + 1) & ~1ull;
  double* out = terms + static_cast<size_t>(jl) * S * n2 + p;
  double nx2 = 0.0;
  for (uint32_t a = 0; a < dbar; ++a)
    nx2 = __dadd_rn(nx2, __dmul_rn(static_cast<double>(xi[a]), static_cast<double>(xi[a])));
  if (nx2 == 0.0) {
    for (uint32_t s = 0; s < S; ++s) out[static_cast<size_t>(s) * n2] = 0.0;
    return;
  }
  const size_t gi = static_cast<size_t>(j) * n + id;
  const double al = alpha[gi], h_par = hp[gi], h_bot = hb[gi];
  const double a2 = __dmul_rn(al, al);
  const double coef = __ddiv_rn(__dmul_rn(a2, __dsub_rn(h_par, h_bot)), nx2);
  const double ah = __dmul_rn(al, h_par);
  uint32_t s = 0;
  for (uint32_t a = 0; a < dbar; ++a) {
    const double cx = __dmul_rn(coef, static_cast<double>(xi[a]));
    for (uint32_t b = a; b < dbar; ++b) out[static_cast<size_t>(s++) * n2] = __dmul_rn(cx, static_cast<double>(xi[b]));
  }
  for (uint32_t a = 0; a < dbar; ++a) out[static_cast<size_t>(s++) * n2] = __dmul_rn(ah, static_cast<double>(xi[a]));
  out[static_cast<size_t>(s) * n2] = __dmul_rn(a2, h_bot);
}

__global__ void center_chain_kernel(const double* __restrict__ terms, uint64_t n, uint32_t S,
                                    uint32_t k, uint32_t sec0, uint32_t nsec,
                                    const uint32_t* __restrict__ starts,
                                    const double* __restrict__ init, double* __restrict__ stats) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // (section, cluster, stat)
  if (t >= nsec * k * S) return;
  const uint32_t s = t % S, c = (t / S) % k, jl = t / (S * k);
  const uint32_t j = sec0 + jl;
  const size_t o = (static_cast<size_t>(j) * k + c) * S + s;
  double acc = init ? init[o] : 0.0;
  const uint32_t* st = starts + static_cast<size_t>(j) * (k + 1);
  const double* tp = terms + (static_cast<size_t>(jl) * S + s) * ((n + 1) & ~1ull);
  uint32_t p = st[c];
  const uint32_t p1 = st[c + 1];
  if ((p & 1u) && p < p1) acc = __dadd_rn(acc, __ldg(tp + p++));  // align to 16 bytes
  // 32 doubles in flight (16 x 16-byte loads), then the ordered adds
  const double2* tp2 = reinterpret_cast<const double2*>(tp);
  for (; p + 32 <= p1; p += 32) {
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(tp2 + (p >> 1) + u);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      acc = __dadd_rn(acc, v[u].x);
      acc = __dadd_rn(acc, v[u].y);
    }
  }
  for (; p < p1; ++p) acc = __dadd_rn(acc, __ldg(tp + p));
  stats[o] = acc;
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}

__global__ void cluster_starts_kernel(const uint32_t* sorted_keys, uint64_t n, uint32_t k,
                                      uint32_t* starts) {
  // starts[c] = first position with key >= c (binary search), starts[k] = n
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > k) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sorted_keys[mid] < c) lo = mid + 1; else hi = mid;
  }
  starts[c] = static_cast<uint32_t>(lo);
}

unsigned enc_grid(uint64_t n) {
  const uint64_t blocks = (n + kEncThreads - 1) / kEncThreads;
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(blocks, 1), 148ull * 16));
}

}  // namespace

void launch_assign_projective(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                              uint32_t k, uint32_t* assign, double* alpha, double* loss,
                              cudaStream_t st) {
  if (n == 0) return;
  const size_t smem = k * 8 + k * dbar * 4;
  if (smem > 200 * 1024) fail(PCPQG_E_UNSUPPORTED, "assign: codebook too large for shared memory");
  if (smem > 48 * 1024)
    PCPQG_CUDA(cudaFuncSetAttribute(assign_projective_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  assign_projective_kernel<<<enc_grid(n), kEncThreads, smem, st>>>(x, n, dbar, centers, k, assign,
                                                                   alpha, loss);
  PCPQG_CUDA(cudaGetLastError());
}

void launch_assign_anisotropic(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                               uint32_t k, const double* hp, const double* hb, const uint32_t* prev,
                               uint32_t* assign, double* alpha, double* loss, cudaStream_t st,
                               bool scaling) {
  if (n == 0) return;
  const size_t smem = k * 8 + k * dbar * 4;
  if (smem > 200 * 1024) fail(PCPQG_E_UNSUPPORTED, "assign: codebook too large for shared memory");
  if (smem > 48 * 1024)
    PCPQG_CUDA(cudaFuncSetAttribute(assign_aniso_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  assign_aniso_kernel<<<enc_grid(n), kEncThreads, smem, st>>>(x, n, dbar, centers, k, hp, hb,
                                                              prev, scaling, assign, alpha, loss);
  PCPQG_CUDA(cudaGetLastError());
}

void launch_aniso_alpha_codes(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                              const uint32_t* assign, const double* hp, const double* hb,
                              const float* values, uint32_t s, uint8_t* codes, cudaStream_t st) {
  if (n == 0) return;
  aniso_alpha_codes_kernel<<<enc_grid(n), kEncThreads, 0, st>>>(x, n, dbar, centers, assign, hp,
                                                                hb, values, s, codes);
  PCPQG_CUDA(cudaGetLastError());
}

void launch_center_stats(const float* x, uint64_t n, uint32_t dbar, uint32_t nsec,
                         uint64_t sec_stride, const uint32_t* assign, const double* alpha,
                         const double* hp, const double* hb, uint32_t k, const double* init,
                         double* stats, cudaStream_t st) {
  if (dbar == 0 || dbar > 16) fail(PCPQG_E_UNSUPPORTED, "center stats: section width must be 1..16");
  if (n > 0xFFFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "center stats: more than 2^32 points");
  uint32_t *ids = nullptr, *order = nullptr, *keys_out = nullptr, *starts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int bits = 1;
  while ((1u << bits) < k) ++bits;
  PCPQG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, assign, keys_out, ids, order,
                                             static_cast<int>(n), 0, bits, st));
  PCPQG_CUDA(cudaMallocAsync(&ids, std::max<uint64_t>(n, 1) * 4, st));
  PCPQG_CUDA(cudaMallocAsync(&keys_out, std::max<uint64_t>(n, 1) * 4, st));
  PCPQG_CUDA(cudaMallocAsync(&order, std::max<uint64_t>(n, 1) * 4 * nsec, st));
  PCPQG_CUDA(cudaMallocAsync(&starts, static_cast<size_t>(k + 1) * 4 * nsec, st));
  PCPQG_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), st));
  if (n) iota_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(ids, n);
  for (uint32_t j = 0; j < nsec; ++j) {
    // stable sort of point ids by cluster: members in increasing id order
    PCPQG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, assign + static_cast<size_t>(j) * n,
                                               keys_out, ids, order + static_cast<size_t>(j) * n,
                                               static_cast<int>(n), 0, bits, st));
    cluster_starts_kernel<<<(k + 1 + 127) / 128, 128, 0, st>>>(keys_out, n, k,
                                                                starts + static_cast<size_t>(j) * (k + 1));
  }
  // terms for as many sections at a time as fit in ~4 GB
  const uint32_t S = dbar * (dbar + 1) / 2 + dbar + 1;
  const uint64_t per_sec = std::max<uint64_t>(((n + 1) & ~1ull), 2) * S * 8;
  size_t free_b = 0, total_b = 0;
  PCPQG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t budget = std::max<uint64_t>(free_b / 3, per_sec);  // more sections -> more chains in flight
  const uint32_t batch = static_cast<uint32_t>(std::clamp<uint64_t>(budget / per_sec, 1, nsec));
  double* terms = nullptr;
  PCPQG_CUDA(cudaMallocAsync(&terms, per_sec * batch, st));
  for (uint32_t s0 = 0; s0 < nsec; s0 += batch) {
    const uint32_t nb = std::min(batch, nsec - s0);
    const uint64_t tot = static_cast<uint64_t>(nb) * n;
    if (tot)
      center_terms_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
          x, dbar, n, sec_stride, s0, nb, order, alpha, hp, hb, terms);
    const uint32_t chains = nb * k * S;
    center_chain_kernel<<<(chains + 127) / 128, 128, 0, st>>>(terms, n, S, k, s0, nb, starts, init,
                                                              stats);
  }
  PCPQG_CUDA(cudaGetLastError());
  cudaFreeAsync(terms, st);
  cudaFreeAsync(ids, st);
  cudaFreeAsync(keys_out, st);
  cudaFreeAsync(order, st);
  cudaFreeAsync(starts, st);
  cudaFreeAsync(tmp, st);
}

}  // namespace pcpqg
