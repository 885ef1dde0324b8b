// Anisotropic weights on the GPU: aniso_weights
// (proj/core/src/clustering.cpp:204-217) -> sin_power_integral
// (proj/core/src/numerics.cpp:174-186), the largest fixed cost of an apcpq /
// aniso build (2 x 1025 std::sin per (point, section); 6.6e11 at config 5).
//
// One thread per (section, point) row.  The Simpson sums are sequential in the
// reference (sum += 4 f or 2 f for i = 1..1023), so a thread keeps both running
// sums in registers and walks i in order; the sin of every node is sin_port
// (pcpqg_hostsin.cuh), which reproduces the host C library's sin bit for bit
// with explicit round-to-nearest multiplies, adds and fused multiply-adds.
// Nodes i*h of neighbouring rows fall into the same sin branch for most i, so
// the warps stay converged; the 3.5 KB table sits in shared memory.
//
// The GPU path is used only after sin_port has been compared with the host's
// std::sin — on the host (the restatement itself) and on the device (the
// compiled kernel) — over a fixed argument set that covers every branch and
// the branch edges; a mismatch (another C library, a host without FMA) leaves
// the weights on the host-thread path (aniso_weights_host).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "pcpqg_hostsin.cuh"
#include "pcpqg_internal.hpp"

namespace pcpqg {
namespace {

const double kSinTabHost[4 * kSinTabEntries] = {
#include "pcpqg_sincostab.inc"
};
__device__ const double kSinTabDev[4 * kSinTabEntries] = {
#include "pcpqg_sincostab.inc"
};

// ipow (numerics.cpp:22-29): square-and-multiply, r first
__device__ __forceinline__ double ipow_dev(double base, int p) {
  double r = 1.0, b = base;
  for (int e = p; e > 0; e >>= 1) {
    if (e & 1) r = __dmul_rn(r, b);
    b = __dmul_rn(b, b);
  }
  return r;
}

constexpr int kPanels = 1024;  // kSimpsonPanels (numerics.cpp)

__global__ void __launch_bounds__(128) aniso_weights_kernel(const float* __restrict__ x, uint64_t n, uint32_t dbar,
                                                            double t, double* __restrict__ h_par,
                                                            double* __restrict__ h_bot) {
  __shared__ double tab[4 * kSinTabEntries];
  for (int i = threadIdx.x; i < 4 * kSinTabEntries; i += blockDim.x) tab[i] = kSinTabDev[i];
  __syncthreads();
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double nx2 = 0.0;  // dotf (clustering.cpp:14-19)
  for (uint32_t a = 0; a < dbar; ++a) {
    const double v = static_cast<double>(x[row * dbar + a]);
    nx2 = __dadd_rn(nx2, __dmul_rn(v, v));
  }
  if (!(nx2 > 0.0)) {
    h_par[row] = 0.0;
    h_bot[row] = 0.0;
    return;
  }
  const double theta = __ddiv_rn(t, __dsqrt_rn(nx2));
  const double half_pi = 3.141592653589793 / 2.0;
  const double tc = theta < 0.0 ? 0.0 : (half_pi < theta ? half_pi : theta);  // std::clamp
  const int p_lo = static_cast<int>(dbar) - 2, p_hi = static_cast<int>(dbar);
  double i_lo = 0.0, i_hi = 0.0;
  if (tc != 0.0) {
    const double h = __ddiv_rn(tc, static_cast<double>(kPanels));
    const double s0 = sin_port(0.0, tab), st = sin_port(tc, tab);
    double sum_lo = __dadd_rn(ipow_dev(s0, p_lo), ipow_dev(st, p_lo));
    double sum_hi = __dadd_rn(ipow_dev(s0, p_hi), ipow_dev(st, p_hi));
    for (int i = 1; i < kPanels; ++i) {
      const double si = sin_port(__dmul_rn(static_cast<double>(i), h), tab);
      const double w = (i & 1) ? 4.0 : 2.0;
      sum_lo = __dadd_rn(sum_lo, __dmul_rn(w, ipow_dev(si, p_lo)));
      sum_hi = __dadd_rn(sum_hi, __dmul_rn(w, ipow_dev(si, p_hi)));
    }
    i_lo = __ddiv_rn(__dmul_rn(sum_lo, h), 3.0);
    i_hi = __ddiv_rn(__dmul_rn(sum_hi, h), 3.0);
  }
  const double hb = i_hi < 0.0 ? 0.0 : i_hi;  // std::max(i_hi, 0.0)
  const double hp = __dmul_rn(static_cast<double>(static_cast<int>(dbar) - 1), __dsub_rn(i_lo, i_hi));
  h_bot[row] = hb;
  h_par[row] = hp < hb ? hb : hp;  // std::max(hp, hb)
}

__global__ void sin_port_kernel(const double* __restrict__ x, uint32_t n, double* __restrict__ out) {
  __shared__ double tab[4 * kSinTabEntries];
  for (int i = threadIdx.x; i < 4 * kSinTabEntries; i += blockDim.x) tab[i] = kSinTabDev[i];
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = sin_port(x[i], tab);
}

// the fixed self-check argument set: uniform over [0, pi/2], every binade down
// to 2^-40, Simpson node grids, and the branch edges with their neighbours
std::vector<double> check_args() {
  std::vector<double> a;
  uint64_t s = 0x9E3779B97F4A7C15ull;
  auto next = [&] {  // splitmix64
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const double half_pi = 3.141592653589793 / 2.0;
  auto unit = [&] { return static_cast<double>(next() >> 11) * 0x1p-53; };
  for (int i = 0; i < 200000; ++i) a.push_back(unit() * half_pi);
  for (int e = -40; e <= 0; ++e)
    for (int i = 0; i < 1000; ++i) a.push_back(std::min(half_pi, std::ldexp(1.0 + unit(), e)));
  for (int r = 0; r < 60; ++r) {
    const double h = unit() * half_pi / kPanels;
    for (int i = 0; i <= kPanels; ++i) a.push_back(i * h);
  }
  for (double edge : {0x1p-26, 0x1.020c49ba5e354p-3, 0.85546875, half_pi})
    for (double v : {std::nextafter(edge, 0.0), edge, std::nextafter(edge, 2.0)})
      if (v <= half_pi) a.push_back(v);
  a.push_back(0.0);
  return a;
}

}  // namespace

uint64_t sin_port_mismatches(int device, uint64_t* total) {
  const std::vector<double> a = check_args();
  if (total) *total = a.size();
  std::vector<double> got(a.size());
  if (device < 0) {
    for (size_t i = 0; i < a.size(); ++i) got[i] = sin_port(a[i], kSinTabHost);
  } else {
    int prev = 0;
    PCPQG_CUDA(cudaGetDevice(&prev));
    PCPQG_CUDA(cudaSetDevice(device));
    double *dx = nullptr, *dy = nullptr;
    PCPQG_CUDA(cudaMalloc(&dx, a.size() * 8));
    PCPQG_CUDA(cudaMalloc(&dy, a.size() * 8));
    PCPQG_CUDA(cudaMemcpy(dx, a.data(), a.size() * 8, cudaMemcpyHostToDevice));
    sin_port_kernel<<<static_cast<unsigned>((a.size() + 255) / 256), 256>>>(dx, static_cast<uint32_t>(a.size()), dy);
    const cudaError_t e1 = cudaGetLastError();
    const cudaError_t e2 = cudaMemcpy(got.data(), dy, a.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    cudaSetDevice(prev);
    PCPQG_CUDA(e1);
    PCPQG_CUDA(e2);
  }
  uint64_t bad = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double want = std::sin(a[i]);
    bad += std::memcmp(&want, &got[i], 8) != 0;
  }
  return bad;
}

bool aniso_weights_gpu_ok(int device) {
  static std::mutex mu;
  static int state[64] = {};  // per device: 0 unknown, 1 ok, 2 mismatch
  std::lock_guard<std::mutex> lock(mu);
  const int slot = std::max(0, std::min(63, device));
  if (state[slot] == 0)
    state[slot] = (sin_port_mismatches(-1) == 0 && sin_port_mismatches(device) == 0) ? 1 : 2;
  return state[slot] == 1;
}

void launch_aniso_weights(const float* dX, uint64_t n, uint32_t dbar, double t, double* dHp, double* dHb,
                          cudaStream_t st) {
  if (n == 0) return;
  const uint64_t blocks = (n + 127) / 128;
  if (blocks > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "aniso_weights: too many rows for one launch");
  aniso_weights_kernel<<<static_cast<unsigned>(blocks), 128, 0, st>>>(dX, n, dbar, t, dHp, dHb);
  PCPQG_CUDA(cudaGetLastError());
}

void aniso_weights_gpu(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot,
                       int device) {
  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  struct Restore {
    int dv;
    ~Restore() { cudaSetDevice(dv); }
  } restore{prev};
  if (!aniso_weights_gpu_ok(device))
    fail(PCPQG_E_UNSUPPORTED, "aniso_weights: the GPU sin does not reproduce this host's std::sin bits");
  // row chunks bound the device footprint (20 B per row at dbar = 4 ... 48 B at dbar = 8)
  const uint64_t chunk = std::min<uint64_t>(n, 1ull << 26);
  float* dX = nullptr;
  double *dHp = nullptr, *dHb = nullptr;
  struct Free {
    float*& a;
    double*& b;
    double*& c;
    ~Free() {
      cudaFree(a);
      cudaFree(b);
      cudaFree(c);
    }
  } fr{dX, dHp, dHb};
  if (n == 0) return;
  PCPQG_CUDA(cudaMalloc(&dX, chunk * dbar * 4));
  PCPQG_CUDA(cudaMalloc(&dHp, chunk * 8));
  PCPQG_CUDA(cudaMalloc(&dHb, chunk * 8));
  for (uint64_t b = 0; b < n; b += chunk) {
    const uint64_t c = std::min(chunk, n - b);
    PCPQG_CUDA(cudaMemcpy(dX, x + b * dbar, c * dbar * 4, cudaMemcpyHostToDevice));
    launch_aniso_weights(dX, c, dbar, t, dHp, dHb, nullptr);
    PCPQG_CUDA(cudaMemcpy(h_par + b, dHp, c * 8, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(h_bot + b, dHb, c * 8, cudaMemcpyDeviceToHost));
  }
}

}  // namespace pcpqg
