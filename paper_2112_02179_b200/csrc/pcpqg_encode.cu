// Encode path (secondary, config 5): per-point center assignment and
// score-aware scale codes, in fp64 with the reference's operation order so
// the codes are bit-identical.  Every multiply/add/divide is an explicit
// round-to-nearest intrinsic: no FMA contraction (the reference is built
// without -march, so GCC emits separate mulsd/addsd).
//
//   assign_projective_kernel   pcpq::assign_projective   clustering.cpp:250-289
//   assign_aniso_kernel        pcpq::assign_anisotropic  clustering.cpp:298-368
//                              (allow_scaling = true, no previous assignment)
//   aniso_alpha_codes_kernel   quantize_anisotropic code assignment
//                              scalar_quant.cpp:121-150 (+ nearest_code :28-39)
//
// Layout: one section's vectors x[n][dbar] (fp32) and centers[k][dbar]; one
// thread per point; the k center rows and their squared norms are staged in
// shared memory once per CTA.
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
    const double hp = h_par[i], hb = h_bot[i];
    double bdist = INFINITY, balpha = 1.0;
    uint32_t bj = 0;
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
    const double bloss = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(w, balpha), qa), balpha), qb);
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
                               uint32_t k, const double* hp, const double* hb, uint32_t* assign,
                               double* alpha, double* loss, cudaStream_t st) {
  if (n == 0) return;
  const size_t smem = k * 8 + k * dbar * 4;
  if (smem > 200 * 1024) fail(PCPQG_E_UNSUPPORTED, "assign: codebook too large for shared memory");
  if (smem > 48 * 1024)
    PCPQG_CUDA(cudaFuncSetAttribute(assign_aniso_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  assign_aniso_kernel<<<enc_grid(n), kEncThreads, smem, st>>>(x, n, dbar, centers, k, hp, hb,
                                                              assign, alpha, loss);
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

}  // namespace pcpqg
