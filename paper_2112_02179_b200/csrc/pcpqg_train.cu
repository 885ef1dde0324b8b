// GPU index training, method kmeans (first solver):
// pcpq::build_pq_index(method = kmeans) (proj/core/src/pq_index.cpp:62-168)
// with kmeans_pp (proj/core/src/clustering.cpp:478-550) per section, producing
// the same PCPQIDX1 image byte for byte.
//
// Host: validate_config + mean_l2_norm (types.cpp:25-69), the per-section
//   seeds Rng::mix(seed, 2j+1) and k-means++ seeding (clustering.cpp:70-144;
//   the D^2 sampling scan is inherently sequential and cheap at these widths),
//   the rare empty-cluster reseed (clustering.cpp:156-185), the convergence
//   test (clustering.cpp:146-151) and the serialization (pq_index.cpp:372-407).
// GPU, all m sections at once (sections are independent):
//   T1  assignment: per (section, point) the first nearest center by the
//       double squared distance summed in coordinate order
//   T2  member lists: stable segmented radix sort of (cluster, point) per
//       section = members_of's increasing-id order
//   T3  centers: per (section, cluster, coordinate) the double sum over the
//       members in order, / count, rounded to float
//   T4  loss: per point the distance to its new center, then per section one
//       sequential chain over clusters and members in order (the reference's
//       loop order, so the loss trace — and the convergence decisions — are
//       bit-identical)
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>

#include <chrono>

#include "pcpqg_train_common.cuh"

namespace pcpqg {
namespace {

// k-means++ over all rows of one section x [n][dbar] (kmeanspp_ids with
// candidates = every row, then seed_centers' copy; clustering.cpp:70-144)
void seed_kmeanspp(const float* x, uint64_t n, uint32_t dbar, uint32_t k, uint64_t seed, float* centers) {
  Rng rng(seed);
  std::vector<uint32_t> seeds;
  seeds.push_back(static_cast<uint32_t>(rng.next_index(n)));
  std::vector<double> d2(n, std::numeric_limits<double>::infinity());
  while (seeds.size() < k) {
    const float* last = x + static_cast<uint64_t>(seeds.back()) * dbar;
    double total = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      double dd = 0.0;
      const float* xi = x + i * dbar;
      for (uint32_t j = 0; j < dbar; ++j) {
        const double diff = static_cast<double>(xi[j]) - static_cast<double>(last[j]);
        dd += diff * diff;
      }
      d2[i] = std::min(d2[i], dd);
      total += d2[i];
    }
    if (total <= 0.0) {
      seeds.push_back(static_cast<uint32_t>(rng.next_index(n)));
      continue;
    }
    double target = rng.next_double() * total;
    uint64_t pick = n - 1;
    for (uint64_t i = 0; i < n; ++i) {
      target -= d2[i];
      if (target <= 0.0) {
        pick = i;
        break;
      }
    }
    seeds.push_back(static_cast<uint32_t>(pick));
  }
  for (uint32_t j = 0; j < k; ++j)
    std::memcpy(centers + static_cast<uint64_t>(j) * dbar, x + static_cast<uint64_t>(seeds[j]) * dbar,
                4ull * dbar);
}

// T1: one thread per (active section, point); centers of the section in smem
__global__ void km_assign_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                                 const float* __restrict__ C, const uint32_t* __restrict__ active,
                                 uint32_t* __restrict__ assign, double* __restrict__ ploss,
                                 uint32_t* __restrict__ counts) {
  extern __shared__ float s_c[];
  const uint32_t sec = active[blockIdx.y];
  for (uint32_t t = threadIdx.x; t < k * dbar; t += blockDim.x) s_c[t] = C[static_cast<uint64_t>(sec) * k * dbar + t];
  __syncthreads();
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* xi = X + (static_cast<uint64_t>(sec) * n + i) * dbar;
  double best = INFINITY;
  uint32_t bj = 0;
  for (uint32_t j = 0; j < k; ++j) {
    double dd = 0.0;
    for (uint32_t a = 0; a < dbar; ++a) {
      const double diff = __dsub_rn(static_cast<double>(xi[a]), static_cast<double>(s_c[j * dbar + a]));
      dd = __dadd_rn(dd, __dmul_rn(diff, diff));
    }
    if (dd < best) {
      best = dd;
      bj = j;
    }
  }
  assign[static_cast<uint64_t>(sec) * n + i] = bj;
  ploss[static_cast<uint64_t>(sec) * n + i] = best;
  atomicAdd(&counts[static_cast<uint64_t>(sec) * k + bj], 1u);
}

// T3: one thread per (section, cluster, coordinate): the member-order mean
__global__ void km_center_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                                 const uint32_t* __restrict__ active, uint32_t nact,
                                 const uint32_t* __restrict__ members, const uint32_t* __restrict__ counts,
                                 const uint64_t* __restrict__ offs, float* __restrict__ C) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(nact) * k * dbar) return;
  const uint32_t a = static_cast<uint32_t>(t % dbar);
  const uint32_t c = static_cast<uint32_t>((t / dbar) % k);
  const uint32_t sec = active[t / (static_cast<uint64_t>(k) * dbar)];
  const uint32_t cnt = counts[static_cast<uint64_t>(sec) * k + c];
  if (cnt == 0) return;  // an empty cluster keeps its center
  const uint32_t* mem = members + static_cast<uint64_t>(sec) * n + offs[static_cast<uint64_t>(sec) * k + c];
  const float* xs = X + static_cast<uint64_t>(sec) * n * dbar;
  double sum = 0.0;
  uint32_t i = 0;
  for (; i + 8 <= cnt; i += 8) {  // eight independent loads in flight, adds in order
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = xs[static_cast<uint64_t>(mem[i + u]) * dbar + a];
#pragma unroll
    for (int u = 0; u < 8; ++u) sum = __dadd_rn(sum, static_cast<double>(v[u]));
  }
  for (; i < cnt; ++i) sum = __dadd_rn(sum, static_cast<double>(xs[static_cast<uint64_t>(mem[i]) * dbar + a]));
  C[(static_cast<uint64_t>(sec) * k + c) * dbar + a] =
      static_cast<float>(__ddiv_rn(sum, static_cast<double>(cnt)));
}

// T4a: per (section, sorted position) the squared distance of that member to its new center
__global__ void km_dist_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                               const uint32_t* __restrict__ active, const uint32_t* __restrict__ members,
                               const uint32_t* __restrict__ sorted_assign, const float* __restrict__ C,
                               double* __restrict__ dist) {
  const uint32_t sec = active[blockIdx.y];
  const uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i = members[static_cast<uint64_t>(sec) * n + p];
  const uint32_t c = sorted_assign[static_cast<uint64_t>(sec) * n + p];
  const float* xi = X + (static_cast<uint64_t>(sec) * n + i) * dbar;
  const float* cj = C + (static_cast<uint64_t>(sec) * k + c) * dbar;
  double dd = 0.0;
  for (uint32_t a = 0; a < dbar; ++a) {
    const double diff = __dsub_rn(static_cast<double>(xi[a]), static_cast<double>(cj[a]));
    dd = __dadd_rn(dd, __dmul_rn(diff, diff));
  }
  dist[static_cast<uint64_t>(sec) * n + p] = dd;
}

}  // namespace

std::vector<uint8_t> train_kmeans(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                  double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device) {
  const double t = validate_train(X, n, d, m, k, s, t_frac, max_iters, tol, false);
  const uint32_t padded_d = ((d + m - 1) / m) * m, dbar = padded_d / m;

  // ---- sections [m][n][dbar] (pad_columns + split_sections) and k-means++ seeds
  std::vector<float> secs(static_cast<uint64_t>(m) * n * dbar, 0.0f);
  std::vector<float> centers(static_cast<uint64_t>(m) * k * dbar, 0.0f);
  {
    const unsigned nt = std::max(1u, std::min(m, std::min(32u, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (uint32_t j = w; j < m; j += nt) {
          float* sj = secs.data() + static_cast<uint64_t>(j) * n * dbar;
          for (uint64_t i = 0; i < n; ++i)
            for (uint32_t a = 0; a < dbar; ++a) {
              const uint32_t col = j * dbar + a;
              sj[i * dbar + a] = col < d ? X[i * d + col] : 0.0f;
            }
          // solver_seed = Rng::mix(seed, 2j + 1) (pq_index.cpp:83); kmeans_pp: Rng rng(solver_seed)
          seed_kmeanspp(sj, n, dbar, k, Rng::mix(seed, 2ull * j + 1),
                        centers.data() + static_cast<uint64_t>(j) * k * dbar);
        }
      });
    for (auto& x : th) x.join();
  }

  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  struct Restore {
    int dv;
    ~Restore() { cudaSetDevice(dv); }
  } restore{prev};
  std::vector<void*> keep;
  struct Free {
    std::vector<void*>* k;
    ~Free() {
      for (void* p : *k) cudaFree(p);
    }
  } fr{&keep};
  const uint64_t mn = static_cast<uint64_t>(m) * n;
  float* dX = talloc<float>(keep, mn * dbar);
  float* dC = talloc<float>(keep, static_cast<uint64_t>(m) * k * dbar);
  uint32_t* dA = talloc<uint32_t>(keep, mn);
  double* dL = talloc<double>(keep, mn);
  uint32_t* dCnt = talloc<uint32_t>(keep, static_cast<uint64_t>(m) * k);
  uint64_t* dOff = talloc<uint64_t>(keep, static_cast<uint64_t>(m) * k);
  uint32_t* dIdx = talloc<uint32_t>(keep, mn);
  uint32_t* dMem = talloc<uint32_t>(keep, mn);
  uint32_t* dSA = talloc<uint32_t>(keep, mn);
  double* dDist = talloc<double>(keep, mn);
  double* dLoss = talloc<double>(keep, m);
  uint32_t* dAct = talloc<uint32_t>(keep, m);
  int* dSeg = talloc<int>(keep, m + 1);
  PCPQG_CUDA(cudaMemcpy(dX, secs.data(), 4 * mn * dbar, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dC, centers.data(), centers.size() * 4, cudaMemcpyHostToDevice));
  std::vector<int> seg(m + 1);
  for (uint32_t j = 0; j <= m; ++j) seg[j] = static_cast<int>(static_cast<uint64_t>(j) * n);
  PCPQG_CUDA(cudaMemcpy(dSeg, seg.data(), 4ull * (m + 1), cudaMemcpyHostToDevice));
  if (mn > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "m x n above 2^31 for the member sort");
  int kbits = 1;
  while ((1u << kbits) < k) ++kbits;
  size_t tmp_bytes = 0;
  PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp_bytes, dA, dSA, dIdx, dMem, static_cast<int>(mn),
                                                      static_cast<int>(m), dSeg, dSeg + 1, 0, kbits));
  void* dTmp = talloc<uint8_t>(keep, tmp_bytes);
  const size_t csmem = 4ull * k * dbar;
  if (csmem > 48 * 1024)
    PCPQG_CUDA(cudaFuncSetAttribute(km_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(csmem)));

  // assignment (+ counts) for the listed sections, then host reseed if any
  // cluster came out empty
  auto assign = [&](const std::vector<uint32_t>& act) {
    PCPQG_CUDA(cudaMemcpy(dAct, act.data(), 4 * act.size(), cudaMemcpyHostToDevice));
    for (uint32_t sj : act) PCPQG_CUDA(cudaMemset(dCnt + static_cast<uint64_t>(sj) * k, 0, 4ull * k));
    dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(act.size()));
    km_assign_kernel<<<grid, 256, csmem>>>(dX, n, dbar, k, dC, dAct, dA, dL, dCnt);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<uint32_t> cnt(static_cast<uint64_t>(m) * k);
    PCPQG_CUDA(cudaMemcpy(cnt.data(), dCnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    for (uint32_t sj : act) {
      bool empty = false;
      for (uint32_t c = 0; c < k; ++c) empty |= cnt[static_cast<uint64_t>(sj) * k + c] == 0;
      if (!empty) continue;
      std::vector<uint32_t> as(n);
      std::vector<double> pl(n);
      float* cs = centers.data() + static_cast<uint64_t>(sj) * k * dbar;
      PCPQG_CUDA(cudaMemcpy(cs, dC + static_cast<uint64_t>(sj) * k * dbar, 4ull * k * dbar, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(as.data(), dA + static_cast<uint64_t>(sj) * n, 4 * n, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(pl.data(), dL + static_cast<uint64_t>(sj) * n, 8 * n, cudaMemcpyDeviceToHost));
      reseed_host(secs.data() + static_cast<uint64_t>(sj) * n * dbar, n, dbar, k, cs, as.data(), pl.data());
      std::vector<uint32_t> c2(k, 0);
      for (uint64_t i = 0; i < n; ++i) ++c2[as[i]];
      PCPQG_CUDA(cudaMemcpy(dC + static_cast<uint64_t>(sj) * k * dbar, cs, 4ull * k * dbar, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dA + static_cast<uint64_t>(sj) * n, as.data(), 4 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dL + static_cast<uint64_t>(sj) * n, pl.data(), 8 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dCnt + static_cast<uint64_t>(sj) * k, c2.data(), 4ull * k, cudaMemcpyHostToDevice));
    }
  };

  std::vector<uint32_t> active(m);
  for (uint32_t j = 0; j < m; ++j) active[j] = j;
  std::vector<std::vector<double>> trace(m);
  for (uint32_t iter = 0; iter < max_iters && !active.empty(); ++iter) {
    assign(active);
    // member lists of every section (sorting converged ones too is harmless)
    km_iota_kernel<<<static_cast<unsigned>((mn + 255) / 256), 256>>>(dIdx, n, m);
    PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(dTmp, tmp_bytes, dA, dSA, dIdx, dMem, static_cast<int>(mn),
                                                        static_cast<int>(m), dSeg, dSeg + 1, 0, kbits));
    km_offsets_kernel<<<(m + 127) / 128, 128>>>(dCnt, m, k, dOff);
    PCPQG_CUDA(cudaMemcpy(dAct, active.data(), 4 * active.size(), cudaMemcpyHostToDevice));
    const uint32_t nact = static_cast<uint32_t>(active.size());
    const uint64_t nc = static_cast<uint64_t>(nact) * k * dbar;
    km_center_kernel<<<static_cast<unsigned>((nc + 127) / 128), 128>>>(dX, n, dbar, k, dAct, nact, dMem, dCnt, dOff, dC);
    dim3 g2(static_cast<unsigned>((n + 255) / 256), nact);
    km_dist_kernel<<<g2, 256>>>(dX, n, dbar, k, dAct, dMem, dSA, dC, dDist);
    km_loss_kernel<<<(nact + 3) / 4, 128>>>(dDist, n, dAct, nact, dLoss);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<double> loss(m);
    PCPQG_CUDA(cudaMemcpy(loss.data(), dLoss, 8ull * m, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> still;
    for (uint32_t sj : active) {
      auto& tr = trace[sj];
      tr.push_back(loss[sj]);
      bool conv = false;  // converged (clustering.cpp:146-151)
      if (tr.size() >= 2) {
        const double p = tr[tr.size() - 2], c = tr.back();
        conv = std::fabs(p - c) <= tol * std::max(std::fabs(p), 1e-300);
      }
      if (!conv) still.push_back(sj);
    }
    active.swap(still);
  }
  std::vector<uint32_t> all(m);
  for (uint32_t j = 0; j < m; ++j) all[j] = j;
  assign(all);  // final memberships against the final centers (+ reseed)

  std::vector<uint32_t> codes(mn);
  PCPQG_CUDA(cudaMemcpy(codes.data(), dA, 4 * mn, cudaMemcpyDeviceToHost));
  PCPQG_CUDA(cudaMemcpy(centers.data(), dC, centers.size() * 4, cudaMemcpyDeviceToHost));

  // ---- serialize (pq_index.cpp:372-407): method 0, scales 1, scale codebook {1}
  const bool wide = k > 256;
  const uint64_t row = static_cast<uint64_t>(m) * (wide ? 2 : 1) + m;
  std::vector<uint8_t> out;
  out.reserve(48 + centers.size() * 4 + 4ull * m + n * row);
  auto u32 = [&](uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  };
  const char magic[8] = {'P', 'C', 'P', 'Q', 'I', 'D', 'X', '1'};
  out.insert(out.end(), magic, magic + 8);
  u32(1);
  u32(0);  // Method::kmeans
  u32(static_cast<uint32_t>(n));
  u32(d);
  u32(padded_d);
  u32(m);
  u32(k);
  u32(1);
  uint64_t tb;
  std::memcpy(&tb, &t, 8);
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<uint8_t>(tb >> (8 * i)));
  const size_t cb0 = out.size();
  out.resize(cb0 + centers.size() * 4);
  std::memcpy(out.data() + cb0, centers.data(), centers.size() * 4);  // [m][k][dbar], little-endian
  const float one = 1.0f;
  for (uint32_t j = 0; j < m; ++j) {
    uint32_t u;
    std::memcpy(&u, &one, 4);
    u32(u);
  }
  const size_t b0 = out.size();
  out.resize(b0 + n * row, 0);
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t* r = out.data() + b0 + i * row;
    for (uint32_t j = 0; j < m; ++j) {
      const uint32_t c = codes[static_cast<uint64_t>(j) * n + i];
      if (wide) {
        r[2 * j] = static_cast<uint8_t>(c);
        r[2 * j + 1] = static_cast<uint8_t>(c >> 8);
      } else {
        r[j] = static_cast<uint8_t>(c);
      }
    }
    // scale codes are all 0 (the rest of the row is already zero)
  }
  return out;
}

}  // namespace pcpqg

// =====================================================================
// method pcpq: projective_k_clustering (clustering.cpp:552-622) per section,
// unit-norm directions with the norms folded into the scales, then
// quantize_projective (scalar_quant.cpp:51-70) or raw alphas.
namespace pcpqg {
namespace {

// v of top_singular_pair (numerics.cpp:46-136) from the Gram matrix g [cols][cols]
std::vector<double> top_direction(const std::vector<double>& g, uint32_t cols) {
  std::vector<double> v(cols, 0.0), w(cols);
  bool all_zero = true;
  for (uint32_t a = 0; a < cols; ++a) all_zero &= g[a * cols + a] == 0.0;
  if (all_zero) {
    v[0] = 1.0;
    return v;
  }
  const int max_iters = 500;
  const double tol = 1e-10;
  Rng rng(0x5157A1B2C3D4E5F6ull);
  double rho = 0.0;
  for (int attempt = 0;; ++attempt) {
    double nv = 0.0;
    for (uint32_t a = 0; a < cols; ++a) {
      v[a] = 2.0 * rng.next_double() - 1.0;
      nv += v[a] * v[a];
    }
    nv = std::sqrt(nv);
    for (auto& x : v) x /= nv;
    bool live = false;
    rho = 0.0;
    for (int it = 0; it < max_iters; ++it) {
      double nw = 0.0, rayleigh = 0.0;
      for (uint32_t a = 0; a < cols; ++a) {
        double acc = 0.0;
        for (uint32_t b = 0; b < cols; ++b) acc += g[a * cols + b] * v[b];
        w[a] = acc;
        nw += acc * acc;
        rayleigh += v[a] * acc;
      }
      nw = std::sqrt(nw);
      if (nw == 0.0) break;
      for (uint32_t a = 0; a < cols; ++a) v[a] = w[a] / nw;
      if (live && std::fabs(rayleigh - rho) <= tol * std::max(rayleigh, 1e-300)) {
        rho = rayleigh;
        break;
      }
      rho = rayleigh;
      live = true;
    }
    if (live) break;
    if (attempt >= 4) {
      std::fill(v.begin(), v.end(), 0.0);
      v[attempt % cols] = 1.0;
      break;
    }
  }
  uint32_t pivot = 0;  // sign convention: largest-|entry| (first on ties) non-negative
  double best_abs = -1.0;
  for (uint32_t a = 0; a < cols; ++a)
    if (std::fabs(v[a]) > best_abs) {
      best_abs = std::fabs(v[a]);
      pivot = a;
    }
  if (v[pivot] < 0.0)
    for (auto& x : v) x = -x;
  return v;
}

// kmeans_1d (numerics.cpp:211-326) for a section with <= s distinct values
// (the only case handled on the host; quantize_projective_all sends the rest to
// the GPU): the codebook is the sorted distinct values, each value's code its
// rank; then quantize_projective's codebook padding to s floats
void trivial_1d_codes(const std::vector<double>& values, uint32_t s, std::vector<float>& cb,
                      std::vector<uint8_t>& codes) {
  const uint64_t n = values.size();
  std::vector<double> distinct(values.begin(), values.end());
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  cb.clear();  // pad_codebook
  for (double v : distinct) cb.push_back(static_cast<float>(v));
  while (cb.size() < s) cb.push_back(cb.empty() ? 0.0f : cb.back());
  codes.resize(n);
  for (uint64_t i = 0; i < n; ++i)
    codes[i] = static_cast<uint8_t>(std::lower_bound(distinct.begin(), distinct.end(), values[i]) - distinct.begin());
}

// Gram chains: per (active section, cluster, a <= b) the member-order sum of x_a x_b
__global__ void tp_gram_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                               const uint32_t* __restrict__ active, uint32_t nact,
                               const uint32_t* __restrict__ members, const uint32_t* __restrict__ counts,
                               const uint64_t* __restrict__ offs, double* __restrict__ G) {
  const uint32_t np = dbar * (dbar + 1) / 2;
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(nact) * k * np) return;
  uint32_t pi = static_cast<uint32_t>(t % np);
  const uint32_t c = static_cast<uint32_t>((t / np) % k);
  const uint32_t sec = active[t / (static_cast<uint64_t>(k) * np)];
  uint32_t a = 0;
  while (pi >= dbar - a) {
    pi -= dbar - a;
    ++a;
  }
  const uint32_t b = a + pi;
  const uint32_t cnt = counts[static_cast<uint64_t>(sec) * k + c];
  const uint32_t* mem = members + static_cast<uint64_t>(sec) * n + offs[static_cast<uint64_t>(sec) * k + c];
  const float* xs = X + static_cast<uint64_t>(sec) * n * dbar;
  double g = 0.0;
  uint32_t i = 0;
  for (; i + 8 <= cnt; i += 8) {
    float va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* r = xs + static_cast<uint64_t>(mem[i + u]) * dbar;
      va[u] = r[a];
      vb[u] = r[b];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) g = __dadd_rn(g, __dmul_rn(static_cast<double>(va[u]), static_cast<double>(vb[u])));
  }
  for (; i < cnt; ++i) {
    const float* r = xs + static_cast<uint64_t>(mem[i]) * dbar;
    g = __dadd_rn(g, __dmul_rn(static_cast<double>(r[a]), static_cast<double>(r[b])));
  }
  G[(static_cast<uint64_t>(sec) * k + c) * dbar * dbar + a * dbar + b] = g;
}

__device__ __forceinline__ double tp_dot(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(a[i]), static_cast<double>(b[i])));
  return acc;
}

// per sorted member: the projective loss under the old center and the candidate
__global__ void tp_loss_terms_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                                     const uint32_t* __restrict__ active, const uint32_t* __restrict__ members,
                                     const uint32_t* __restrict__ sorted_assign, const float* __restrict__ C,
                                     const float* __restrict__ Cand, double* __restrict__ lo,
                                     double* __restrict__ ln) {
  const uint32_t sec = active[blockIdx.y];
  const uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i = members[static_cast<uint64_t>(sec) * n + p];
  const uint32_t c = sorted_assign[static_cast<uint64_t>(sec) * n + p];
  const float* xi = X + (static_cast<uint64_t>(sec) * n + i) * dbar;
  const float* co = C + (static_cast<uint64_t>(sec) * k + c) * dbar;
  const float* cn = Cand + (static_cast<uint64_t>(sec) * k + c) * dbar;
  const double nx2 = tp_dot(xi, xi, dbar);
  // cluster_loss (clustering.cpp:561-570): max(|x|^2 - ip^2 / |c|^2, 0)
  const double io = tp_dot(xi, co, dbar), in = tp_dot(xi, cn, dbar);
  const double lo_v = __dsub_rn(nx2, __ddiv_rn(__dmul_rn(io, io), tp_dot(co, co, dbar)));
  const double ln_v = __dsub_rn(nx2, __ddiv_rn(__dmul_rn(in, in), tp_dot(cn, cn, dbar)));
  lo[static_cast<uint64_t>(sec) * n + p] = lo_v > 0.0 ? lo_v : 0.0;
  ln[static_cast<uint64_t>(sec) * n + p] = ln_v > 0.0 ? ln_v : 0.0;
}


// ---- kmeans_1d on the GPU (numerics.cpp:211-326) for every (section,
// restart) at once.  Sequential parts stay sequential: k-means++'s D^2 total
// and the `target -= d2[i]` pick scan, the round loss and the per-group sums
// are ordered chains (one warp per chain, adds in lane order); the RNG, the
// center updates, the rare empty-group reseed (which reads partially updated
// centers) and the best restart are on the host.
// KI1: d2[i] = min(d2[i], (v - c)^2) for the newest seed center (std::min order)
__global__ void k1_d2_kernel(const double* __restrict__ V, const uint64_t* __restrict__ poff,
                             const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                             const uint32_t* __restrict__ act, const double* __restrict__ newc, int first,
                             double* __restrict__ d2) {
  const uint32_t p = act[blockIdx.y];
  const uint64_t n = pcnt[p], o = poff[p], ab = pbase[p];
  const double c = newc[p];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double df = __dsub_rn(V[o + i], c);
    const double x = __dmul_rn(df, df);
    const double old = first ? INFINITY : d2[ab + i];
    d2[ab + i] = x < old ? x : old;
  }
}

// KI2: per problem one warp: mode 0 the ordered total of d2; mode 1 the pick
// scan (target -= d2[i] until <= 0; n - 1 if it never is)
__global__ void k1_seed_chain_kernel(const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                                     const uint32_t* __restrict__ act, uint32_t nact, const double* __restrict__ d2,
                                     int mode, double* __restrict__ total, const double* __restrict__ target,
                                     uint64_t* __restrict__ pick) {
  const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (w >= nact) return;
  const uint32_t p = act[w];
  const uint64_t n = pcnt[p], ab = pbase[p];
  double acc = mode == 0 ? 0.0 : target[p];
  uint64_t pk = n - 1;
  bool done = false;
  for (uint64_t b0 = 0; b0 < n && !done; b0 += 32) {
    const uint64_t i = b0 + lane;
    const double v = i < n ? d2[ab + i] : 0.0;
    const uint32_t cnt = n - b0 < 32 ? static_cast<uint32_t>(n - b0) : 32u;
    for (uint32_t l = 0; l < cnt; ++l) {
      const double x = __shfl_sync(0xFFFFFFFFu, v, l);
      if (mode == 0) {
        acc = __dadd_rn(acc, x);
      } else {
        acc = __dsub_rn(acc, x);
        if (acc <= 0.0) {
          pk = b0 + l;
          done = true;
          break;
        }
      }
    }
  }
  if (lane == 0) {
    if (mode == 0) total[p] = acc;
    else pick[p] = pk;
  }
}

// KR1: assignment to the first nearest center ((v - c)^2, strict <), its
// distance for the loss chain, and whether it changed
__global__ void k1_assign_kernel(const double* __restrict__ V, const uint64_t* __restrict__ poff,
                                 const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                                 const uint32_t* __restrict__ act, uint32_t s, const double* __restrict__ cen,
                                 const uint8_t* __restrict__ prev, uint8_t* __restrict__ cur, int check,
                                 uint32_t* __restrict__ changed, double* __restrict__ bdo) {
  __shared__ double sc[256];
  const uint32_t p = act[blockIdx.y];
  for (uint32_t t = threadIdx.x; t < s; t += blockDim.x) sc[t] = cen[static_cast<uint64_t>(p) * s + t];
  __syncthreads();
  const uint64_t n = pcnt[p], o = poff[p], ab = pbase[p];
  int diff = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = V[o + i];
    double bd = INFINITY;
    uint32_t bj = 0;
    for (uint32_t j = 0; j < s; ++j) {
      const double df = __dsub_rn(v, sc[j]);
      const double dd = __dmul_rn(df, df);
      if (dd < bd) {
        bd = dd;
        bj = j;
      }
    }
    cur[ab + i] = static_cast<uint8_t>(bj);
    bdo[ab + i] = bd;
    diff |= check && prev[ab + i] != bj;
  }
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(changed + p, 1u);
}

// KR2: one warp per chain: the round loss (bd in order) or one group's sum
// of values and count (its members in order)
__global__ void k1_chain_kernel(const double* __restrict__ V, const uint64_t* __restrict__ poff,
                                const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                                const uint32_t* __restrict__ act, uint32_t nact, uint32_t s,
                                const uint8_t* __restrict__ cur, const double* __restrict__ bd,
                                double* __restrict__ loss, double* __restrict__ sums, uint64_t* __restrict__ cnts) {
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (wid >= static_cast<uint64_t>(nact) * (s + 1)) return;
  const uint32_t p = act[wid / (s + 1)];
  const uint32_t st = static_cast<uint32_t>(wid % (s + 1));
  const uint64_t n = pcnt[p], o = poff[p], ab = pbase[p];
  if (st == 0) {
    double acc = 0.0;
    for (uint64_t b0 = 0; b0 < n; b0 += 32) {
      const uint64_t i = b0 + lane;
      const double v = i < n ? bd[ab + i] : 0.0;
      const uint32_t cnt = n - b0 < 32 ? static_cast<uint32_t>(n - b0) : 32u;
      for (uint32_t l = 0; l < cnt; ++l) acc = __dadd_rn(acc, __shfl_sync(0xFFFFFFFFu, v, l));
    }
    if (lane == 0) loss[p] = acc;
    return;
  }
  const uint32_t g = st - 1;
  double sum = 0.0;
  uint64_t cn = 0;
  for (uint64_t b0 = 0; b0 < n; b0 += 32) {
    const uint64_t i = b0 + lane;
    const bool mine = i < n && cur[ab + i] == g;
    uint32_t mm = __ballot_sync(0xFFFFFFFFu, mine);
    cn += __popc(mm);
    const double v = mine ? V[o + i] : 0.0;
    while (mm) {
      const uint32_t l = __ffs(mm) - 1u;
      mm &= mm - 1u;
      sum = __dadd_rn(sum, __shfl_sync(0xFFFFFFFFu, v, l));
    }
  }
  if (lane == 0) {
    sums[static_cast<uint64_t>(p) * s + g] = sum;
    cnts[static_cast<uint64_t>(p) * s + g] = cn;
  }
}

// quantize_projective (scalar_quant.cpp:50-70) for every section: kmeans_1d
// (trivial sections, <= s distinct values, on the host; the rest on the GPU),
// canonical codebook padded to s floats, and the codes
void quantize_projective_all(const std::vector<std::vector<double>>& vals, uint32_t s,
                             const std::vector<uint64_t>& seeds, std::vector<std::vector<float>>& cbs,
                             std::vector<std::vector<uint8_t>>& codes, unsigned nthreads) {
  const uint32_t m = static_cast<uint32_t>(vals.size());
  std::vector<uint8_t> trivial(m, 0);
  {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nthreads; ++w)
      th.emplace_back([&, w] {
        for (uint32_t j = w; j < m; j += nthreads) {
          std::vector<double> distinct(vals[j]);
          std::sort(distinct.begin(), distinct.end());
          distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
          if (distinct.size() <= s) {
            trivial[j] = 1;
            trivial_1d_codes(vals[j], s, cbs[j], codes[j]);
          }
        }
      });
    for (auto& x : th) x.join();
  }
  std::vector<uint32_t> secs;
  std::vector<uint64_t> soff(m, 0);
  uint64_t total = 0;
  for (uint32_t j = 0; j < m; ++j)
    if (!trivial[j]) {
      secs.push_back(j);
      soff[j] = total;
      total += vals[j].size();
    }
  if (secs.empty()) return;
  constexpr uint32_t R = 10;
  const uint32_t P = static_cast<uint32_t>(secs.size()) * R;
  std::vector<double> hv(total);
  for (uint32_t j : secs) std::copy(vals[j].begin(), vals[j].end(), hv.begin() + soff[j]);
  std::vector<uint64_t> poff(P), pcnt(P), pbase(P);
  for (uint32_t si = 0; si < secs.size(); ++si)
    for (uint32_t r = 0; r < R; ++r) {
      poff[si * R + r] = soff[secs[si]];
      pcnt[si * R + r] = vals[secs[si]].size();
      pbase[si * R + r] = r * total + soff[secs[si]];
    }
  std::vector<void*> keep;
  struct Free {
    std::vector<void*>* k;
    ~Free() {
      for (void* p : *k) cudaFree(p);
    }
  } fr{&keep};
  double* dV = talloc<double>(keep, total);
  uint64_t* dOff = talloc<uint64_t>(keep, P);
  uint64_t* dCnt = talloc<uint64_t>(keep, P);
  uint64_t* dBase = talloc<uint64_t>(keep, P);
  uint32_t* dAct = talloc<uint32_t>(keep, P);
  double* dD2 = talloc<double>(keep, R * total);  // seeding d2, then the round distances
  uint8_t* dAs[2] = {talloc<uint8_t>(keep, R * total), talloc<uint8_t>(keep, R * total)};
  double* dC = talloc<double>(keep, static_cast<uint64_t>(P) * s);
  double* dNew = talloc<double>(keep, P);
  double* dTot = talloc<double>(keep, P);
  double* dTgt = talloc<double>(keep, P);
  uint64_t* dPick = talloc<uint64_t>(keep, P);
  uint32_t* dChg = talloc<uint32_t>(keep, P);
  double* dLoss = talloc<double>(keep, P);
  double* dSum = talloc<double>(keep, static_cast<uint64_t>(P) * s);
  uint64_t* dNum = talloc<uint64_t>(keep, static_cast<uint64_t>(P) * s);
  PCPQG_CUDA(cudaMemcpy(dV, hv.data(), 8 * total, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dOff, poff.data(), 8ull * P, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dCnt, pcnt.data(), 8ull * P, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dBase, pbase.data(), 8ull * P, cudaMemcpyHostToDevice));
  uint64_t max_n = 0;
  for (uint32_t j : secs) max_n = std::max<uint64_t>(max_n, vals[j].size());
  const unsigned bx = static_cast<unsigned>(std::min<uint64_t>((max_n + 255) / 256, 64));
  std::vector<uint32_t> all(P);
  for (uint32_t p = 0; p < P; ++p) all[p] = p;
  PCPQG_CUDA(cudaMemcpy(dAct, all.data(), 4ull * P, cudaMemcpyHostToDevice));
  auto valof = [&](uint32_t p, uint64_t i) { return vals[secs[p / R]][i]; };

  // k-means++ seeding of every problem (root.split(restart) streams)
  std::vector<Rng> rngs;
  rngs.reserve(P);
  std::vector<double> cen(static_cast<uint64_t>(P) * s), newc(P), tot(P), tgt(P);
  std::vector<uint64_t> pick(P);
  for (uint32_t p = 0; p < P; ++p) {
    rngs.emplace_back(Rng::mix(seeds[secs[p / R]], p % R));
    cen[static_cast<uint64_t>(p) * s] = newc[p] = valof(p, rngs[p].next_index(pcnt[p]));
  }
  const unsigned wblocks = (P * 32 + 127) / 128;
  for (uint32_t t = 1; t < s; ++t) {
    PCPQG_CUDA(cudaMemcpy(dNew, newc.data(), 8ull * P, cudaMemcpyHostToDevice));
    k1_d2_kernel<<<dim3(bx, P), 256>>>(dV, dOff, dCnt, dBase, dAct, dNew, t == 1, dD2);
    k1_seed_chain_kernel<<<wblocks, 128>>>(dCnt, dBase, dAct, P, dD2, 0, dTot, nullptr, nullptr);
    PCPQG_CUDA(cudaGetLastError());
    PCPQG_CUDA(cudaMemcpy(tot.data(), dTot, 8ull * P, cudaMemcpyDeviceToHost));
    std::vector<uint8_t> scan(P, 0);
    for (uint32_t p = 0; p < P; ++p) {
      if (tot[p] <= 0.0) {
        newc[p] = valof(p, rngs[p].next_index(pcnt[p]));
      } else {
        tgt[p] = rngs[p].next_double() * tot[p];
        scan[p] = 1;
      }
    }
    PCPQG_CUDA(cudaMemcpy(dTgt, tgt.data(), 8ull * P, cudaMemcpyHostToDevice));
    k1_seed_chain_kernel<<<wblocks, 128>>>(dCnt, dBase, dAct, P, dD2, 1, nullptr, dTgt, dPick);
    PCPQG_CUDA(cudaGetLastError());
    PCPQG_CUDA(cudaMemcpy(pick.data(), dPick, 8ull * P, cudaMemcpyDeviceToHost));
    for (uint32_t p = 0; p < P; ++p) {
      if (scan[p]) newc[p] = valof(p, pick[p]);
      cen[static_cast<uint64_t>(p) * s + t] = newc[p];
    }
  }

  // Lloyd rounds
  std::vector<uint32_t> active = all, final_buf(P, 0), chg(P);
  std::vector<double> loss(P, 0.0), sums(static_cast<uint64_t>(P) * s);
  std::vector<uint64_t> cnts(static_cast<uint64_t>(P) * s);
  for (int round = 0; round < 100 && !active.empty(); ++round) {
    const uint32_t nact = static_cast<uint32_t>(active.size());
    const int cb = round & 1;
    PCPQG_CUDA(cudaMemcpy(dAct, active.data(), 4ull * nact, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemcpy(dC, cen.data(), 8ull * P * s, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemset(dChg, 0, 4ull * P));
    k1_assign_kernel<<<dim3(bx, nact), 256>>>(dV, dOff, dCnt, dBase, dAct, s, dC, dAs[cb ^ 1], dAs[cb], round > 0,
                                               dChg, dD2);
    const uint64_t nt = static_cast<uint64_t>(nact) * (s + 1) * 32;
    k1_chain_kernel<<<static_cast<unsigned>((nt + 127) / 128), 128>>>(dV, dOff, dCnt, dBase, dAct, nact, s, dAs[cb],
                                                                       dD2, dLoss, dSum, dNum);
    PCPQG_CUDA(cudaGetLastError());
    PCPQG_CUDA(cudaMemcpy(loss.data(), dLoss, 8ull * P, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(chg.data(), dChg, 4ull * P, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(sums.data(), dSum, sums.size() * 8, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(cnts.data(), dNum, cnts.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> still;
    for (uint32_t p : active) {
      final_buf[p] = static_cast<uint32_t>(cb);
      if (round > 0 && !chg[p]) continue;  // prev == assign
      double* cp = cen.data() + static_cast<uint64_t>(p) * s;
      std::vector<uint8_t> as;  // fetched only for an empty group
      for (uint32_t j = 0; j < s; ++j) {
        const uint64_t c = cnts[static_cast<uint64_t>(p) * s + j];
        if (c > 0) {
          cp[j] = sums[static_cast<uint64_t>(p) * s + j] / static_cast<double>(c);
        } else {  // the farthest value from its (possibly already updated) center
          if (as.empty()) {
            as.resize(pcnt[p]);
            PCPQG_CUDA(cudaMemcpy(as.data(), dAs[cb] + pbase[p], pcnt[p], cudaMemcpyDeviceToHost));
          }
          uint64_t far = 0;
          double fd = -1.0;
          for (uint64_t i = 0; i < pcnt[p]; ++i) {
            const double v = valof(p, i);
            const double dd = (v - cp[as[i]]) * (v - cp[as[i]]);
            if (dd > fd) {
              fd = dd;
              far = i;
            }
          }
          cp[j] = valof(p, far);
        }
      }
      still.push_back(p);
    }
    active.swap(still);
  }
  // best restart per section (strict <), canonical codebook, padding, codes
  for (uint32_t si = 0; si < secs.size(); ++si) {
    const uint32_t j = secs[si];
    uint32_t bp = si * R;
    double best = std::numeric_limits<double>::infinity();
    for (uint32_t r = 0; r < R; ++r)
      if (loss[si * R + r] < best) {
        best = loss[si * R + r];
        bp = si * R + r;
      }
    const uint64_t n = pcnt[bp];
    std::vector<uint8_t> as(n);
    PCPQG_CUDA(cudaMemcpy(as.data(), dAs[final_buf[bp]] + pbase[bp], n, cudaMemcpyDeviceToHost));
    std::vector<double> bv(cen.begin() + static_cast<uint64_t>(bp) * s, cen.begin() + static_cast<uint64_t>(bp + 1) * s);
    std::vector<uint32_t> order(s);
    for (uint32_t i = 0; i < s; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return bv[a] < bv[b]; });
    std::vector<double> sorted;
    std::vector<uint32_t> remap(s, 0);
    for (uint32_t pos = 0; pos < s; ++pos) {
      const double val = bv[order[pos]];
      if (sorted.empty() || val != sorted.back()) sorted.push_back(val);
      remap[order[pos]] = static_cast<uint32_t>(sorted.size() - 1);
    }
    cbs[j].clear();
    for (double v : sorted) cbs[j].push_back(static_cast<float>(v));
    while (cbs[j].size() < s) cbs[j].push_back(cbs[j].empty() ? 0.0f : cbs[j].back());
    codes[j].resize(n);
    for (uint64_t i = 0; i < n; ++i) codes[j][i] = static_cast<uint8_t>(remap[as[i]]);
  }
}

}  // namespace

std::vector<uint8_t> train_pcpq(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                bool quantize, double t_frac, uint32_t max_iters, double tol, uint64_t seed,
                                int device) {
  using clk = std::chrono::steady_clock;
  auto tick = clk::now();
  auto phase = [&](int i) {
    const auto now = clk::now();
    g_train_phases[i] = std::chrono::duration<double>(now - tick).count();
    tick = now;
  };
  for (double& v : g_train_phases) v = 0.0;
  const double t = validate_train(X, n, d, m, k, s, t_frac, max_iters, tol, false);
  const uint32_t scales = quantize ? s : 0;  // effective_scales (pq_index.cpp:35-38)
  if (quantize && s > 256) fail(PCPQG_E_DATA, "scalar quantization: need 1 <= s <= 256");
  const uint32_t padded_d = ((d + m - 1) / m) * m, dbar = padded_d / m;
  const uint64_t mn = static_cast<uint64_t>(m) * n;
  std::vector<float> secs(mn * dbar, 0.0f);
  std::vector<float> centers(static_cast<uint64_t>(m) * k * dbar, 0.0f);
  const unsigned nt = std::max(1u, std::min(m, std::min(32u, std::thread::hardware_concurrency())));
  auto par_sections = [&](auto&& f) {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (uint32_t j = w; j < m; j += nt) f(j);
      });
    for (auto& x : th) x.join();
  };
  par_sections([&](uint32_t j) {
    float* sj = secs.data() + static_cast<uint64_t>(j) * n * dbar;
    for (uint64_t i = 0; i < n; ++i)
      for (uint32_t a = 0; a < dbar; ++a) {
        const uint32_t col = j * dbar + a;
        sj[i * dbar + a] = col < d ? X[i * d + col] : 0.0f;
      }
    seed_nonzero(sj, n, dbar, k, Rng::mix(seed, 2ull * j + 1), true, centers.data() + static_cast<uint64_t>(j) * k * dbar);
  });
  auto check_nonzero = [&](uint32_t j) {  // check_centers_nonzero (clustering.cpp:42-45)
    for (uint32_t c = 0; c < k; ++c) {
      double acc = 0.0;
      const float* r = centers.data() + (static_cast<uint64_t>(j) * k + c) * dbar;
      for (uint32_t a = 0; a < dbar; ++a) acc += static_cast<double>(r[a]) * static_cast<double>(r[a]);
      if (acc == 0.0) fail(PCPQG_E_DATA, "zero center row");
    }
  };
  for (uint32_t j = 0; j < m; ++j) check_nonzero(j);

  phase(0);
  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  struct Restore {
    int dv;
    ~Restore() { cudaSetDevice(dv); }
  } restore{prev};
  std::vector<void*> keep;
  struct Free {
    std::vector<void*>* k;
    ~Free() {
      for (void* p : *k) cudaFree(p);
    }
  } fr{&keep};
  float* dX = talloc<float>(keep, mn * dbar);
  float* dC = talloc<float>(keep, static_cast<uint64_t>(m) * k * dbar);
  float* dCand = talloc<float>(keep, static_cast<uint64_t>(m) * k * dbar);
  uint32_t* dA = talloc<uint32_t>(keep, mn);
  double* dAl = talloc<double>(keep, mn);
  double* dL = talloc<double>(keep, mn);
  uint32_t* dCnt = talloc<uint32_t>(keep, static_cast<uint64_t>(m) * k);
  uint64_t* dOff = talloc<uint64_t>(keep, static_cast<uint64_t>(m) * k);
  uint32_t* dIdx = talloc<uint32_t>(keep, mn);
  uint32_t* dMem = talloc<uint32_t>(keep, mn);
  uint32_t* dSA = talloc<uint32_t>(keep, mn);
  double* dLo = talloc<double>(keep, mn);
  double* dLn = talloc<double>(keep, mn);
  double* dG = talloc<double>(keep, static_cast<uint64_t>(m) * k * dbar * dbar);
  double* dCL = talloc<double>(keep, static_cast<uint64_t>(m) * k * 2);
  uint32_t* dAct = talloc<uint32_t>(keep, m);
  int* dSeg = talloc<int>(keep, m + 1);
  PCPQG_CUDA(cudaMemcpy(dX, secs.data(), 4 * mn * dbar, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dC, centers.data(), centers.size() * 4, cudaMemcpyHostToDevice));
  std::vector<int> seg(m + 1);
  for (uint32_t j = 0; j <= m; ++j) seg[j] = static_cast<int>(static_cast<uint64_t>(j) * n);
  PCPQG_CUDA(cudaMemcpy(dSeg, seg.data(), 4ull * (m + 1), cudaMemcpyHostToDevice));
  if (mn > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "m x n above 2^31 for the member sort");
  int kbits = 1;
  while ((1u << kbits) < k) ++kbits;
  size_t tmp_bytes = 0;
  PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp_bytes, dA, dSA, dIdx, dMem, static_cast<int>(mn),
                                                      static_cast<int>(m), dSeg, dSeg + 1, 0, kbits));
  void* dTmp = talloc<uint8_t>(keep, tmp_bytes);

  // assign_projective (+ counts) for the listed sections, host reseed of empty clusters
  auto assign = [&](const std::vector<uint32_t>& act) {
    for (uint32_t sj : act) {
      launch_assign_projective(dX + static_cast<uint64_t>(sj) * n * dbar, n, dbar,
                               dC + static_cast<uint64_t>(sj) * k * dbar, k, dA + static_cast<uint64_t>(sj) * n,
                               dAl + static_cast<uint64_t>(sj) * n, dL + static_cast<uint64_t>(sj) * n, 0);
      PCPQG_CUDA(cudaMemset(dCnt + static_cast<uint64_t>(sj) * k, 0, 4ull * k));
    }
    PCPQG_CUDA(cudaMemcpy(dAct, act.data(), 4 * act.size(), cudaMemcpyHostToDevice));
    tp_count_kernel<<<dim3(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(act.size())), 256>>>(
        dA, n, k, dAct, dCnt);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<uint32_t> cnt(static_cast<uint64_t>(m) * k);
    PCPQG_CUDA(cudaMemcpy(cnt.data(), dCnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    for (uint32_t sj : act) {
      bool empty = false;
      for (uint32_t c = 0; c < k; ++c) empty |= cnt[static_cast<uint64_t>(sj) * k + c] == 0;
      if (!empty) continue;
      std::vector<uint32_t> as(n);
      std::vector<double> pl(n), al(n);
      float* cs = centers.data() + static_cast<uint64_t>(sj) * k * dbar;
      PCPQG_CUDA(cudaMemcpy(as.data(), dA + static_cast<uint64_t>(sj) * n, 4 * n, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(pl.data(), dL + static_cast<uint64_t>(sj) * n, 8 * n, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(al.data(), dAl + static_cast<uint64_t>(sj) * n, 8 * n, cudaMemcpyDeviceToHost));
      // reseed_empty_clusters (clustering.cpp:156-185), alphas of moved points become 1
      std::vector<uint64_t> counts(k, 0);
      for (uint64_t i = 0; i < n; ++i) ++counts[as[i]];
      const float* xs = secs.data() + static_cast<uint64_t>(sj) * n * dbar;
      for (bool changed = true; changed;) {
        changed = false;
        for (uint32_t j = 0; j < k; ++j) {
          if (counts[j] > 0) continue;
          uint64_t far = 0;
          double fl = 0.0;
          for (uint64_t i = 0; i < n; ++i)
            if (pl[i] > fl) {
              fl = pl[i];
              far = i;
            }
          if (!(fl > 0.0)) continue;
          std::memcpy(cs + static_cast<uint64_t>(j) * dbar, xs + far * dbar, 4ull * dbar);
          --counts[as[far]];
          ++counts[j];
          as[far] = j;
          al[far] = 1.0;
          pl[far] = 0.0;
          changed = true;
        }
      }
      std::vector<uint32_t> c2(k);
      for (uint32_t c = 0; c < k; ++c) c2[c] = static_cast<uint32_t>(counts[c]);
      PCPQG_CUDA(cudaMemcpy(dC + static_cast<uint64_t>(sj) * k * dbar, cs, 4ull * k * dbar, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dA + static_cast<uint64_t>(sj) * n, as.data(), 4 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dL + static_cast<uint64_t>(sj) * n, pl.data(), 8 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dAl + static_cast<uint64_t>(sj) * n, al.data(), 8 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dCnt + static_cast<uint64_t>(sj) * k, c2.data(), 4ull * k, cudaMemcpyHostToDevice));
    }
  };

  std::vector<uint32_t> active(m);
  for (uint32_t j = 0; j < m; ++j) active[j] = j;
  std::vector<std::vector<double>> trace(m);
  const uint32_t np = dbar * (dbar + 1) / 2;
  for (uint32_t iter = 0; iter < max_iters && !active.empty(); ++iter) {
    assign(active);
    km_iota_kernel<<<static_cast<unsigned>((mn + 255) / 256), 256>>>(dIdx, n, m);
    PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(dTmp, tmp_bytes, dA, dSA, dIdx, dMem, static_cast<int>(mn),
                                                        static_cast<int>(m), dSeg, dSeg + 1, 0, kbits));
    km_offsets_kernel<<<(m + 127) / 128, 128>>>(dCnt, m, k, dOff);
    PCPQG_CUDA(cudaMemcpy(dAct, active.data(), 4 * active.size(), cudaMemcpyHostToDevice));
    const uint32_t nact = static_cast<uint32_t>(active.size());
    const uint64_t ng = static_cast<uint64_t>(nact) * k * np;
    tp_gram_kernel<<<static_cast<unsigned>((ng + 127) / 128), 128>>>(dX, n, dbar, k, dAct, nact, dMem, dCnt, dOff, dG);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<double> G(static_cast<uint64_t>(m) * k * dbar * dbar);
    std::vector<uint32_t> cnt(static_cast<uint64_t>(m) * k);
    PCPQG_CUDA(cudaMemcpy(G.data(), dG, G.size() * 8, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(cnt.data(), dCnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    // center_projective per non-empty cluster (host power iteration on the
    // d̄ x d̄ Gram matrix), rounded to float: the candidate centers
    std::vector<float> cand(centers);
    {
      std::vector<std::thread> th;
      for (unsigned w = 0; w < nt; ++w)
        th.emplace_back([&, w] {
          for (uint32_t ai = w; ai < nact; ai += nt) {
            const uint32_t sj = active[ai];
            for (uint32_t c = 0; c < k; ++c) {
              if (cnt[static_cast<uint64_t>(sj) * k + c] == 0) continue;
              std::vector<double> g(dbar * dbar);
              const double* gs = G.data() + (static_cast<uint64_t>(sj) * k + c) * dbar * dbar;
              for (uint32_t a = 0; a < dbar; ++a)
                for (uint32_t b = a; b < dbar; ++b) g[a * dbar + b] = g[b * dbar + a] = gs[a * dbar + b];
              const std::vector<double> v = top_direction(g, dbar);
              float* out = cand.data() + (static_cast<uint64_t>(sj) * k + c) * dbar;
              for (uint32_t a = 0; a < dbar; ++a) out[a] = static_cast<float>(v[a]);
            }
          }
        });
      for (auto& x : th) x.join();
    }
    PCPQG_CUDA(cudaMemcpy(dCand, cand.data(), cand.size() * 4, cudaMemcpyHostToDevice));
    dim3 g2(static_cast<unsigned>((n + 255) / 256), nact);
    tp_loss_terms_kernel<<<g2, 256>>>(dX, n, dbar, k, dAct, dMem, dSA, dC, dCand, dLo, dLn);
    const uint64_t nl = static_cast<uint64_t>(nact) * k * 2;
    tp_loss_chain_kernel<<<static_cast<unsigned>((nl + 127) / 128), 128>>>(dLo, dLn, n, k, dAct, nact, dCnt, dOff, dCL);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<double> CL(static_cast<uint64_t>(m) * k * 2);
    PCPQG_CUDA(cudaMemcpy(CL.data(), dCL, CL.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> still;
    for (uint32_t sj : active) {
      double loss = 0.0;
      for (uint32_t c = 0; c < k; ++c) {
        if (cnt[static_cast<uint64_t>(sj) * k + c] == 0) continue;
        const double old_l = CL[(static_cast<uint64_t>(sj) * k + c) * 2], new_l = CL[(static_cast<uint64_t>(sj) * k + c) * 2 + 1];
        if (new_l < old_l) {  // keep the old center unless the rounded update helps
          std::memcpy(centers.data() + (static_cast<uint64_t>(sj) * k + c) * dbar,
                      cand.data() + (static_cast<uint64_t>(sj) * k + c) * dbar, 4ull * dbar);
          loss += new_l;
        } else {
          loss += old_l;
        }
      }
      auto& tr = trace[sj];
      tr.push_back(loss);
      bool conv = false;
      if (tr.size() >= 2) {
        const double p = tr[tr.size() - 2], c = tr.back();
        conv = std::fabs(p - c) <= tol * std::max(std::fabs(p), 1e-300);
      }
      if (!conv) still.push_back(sj);
    }
    PCPQG_CUDA(cudaMemcpy(dC, centers.data(), centers.size() * 4, cudaMemcpyHostToDevice));
    active.swap(still);
  }
  std::vector<uint32_t> all(m);
  for (uint32_t j = 0; j < m; ++j) all[j] = j;
  assign(all);
  std::vector<uint32_t> codes(mn);
  std::vector<double> alphas(mn);
  PCPQG_CUDA(cudaMemcpy(codes.data(), dA, 4 * mn, cudaMemcpyDeviceToHost));
  PCPQG_CUDA(cudaMemcpy(alphas.data(), dAl, 8 * mn, cudaMemcpyDeviceToHost));
  PCPQG_CUDA(cudaMemcpy(centers.data(), dC, centers.size() * 4, cudaMemcpyDeviceToHost));

  phase(1);
  // unit directions, norms folded into the scales (pq_index.cpp:102-117); then
  // quantize_projective (scale_seed = Rng::mix(seed, 2j + 2)) or raw alphas
  std::vector<std::vector<float>> scb(m);
  std::vector<std::vector<uint8_t>> scodes(m);
  par_sections([&](uint32_t j) {
    std::vector<double> norms(k, 1.0);
    for (uint32_t c = 0; c < k; ++c) {
      float* row = centers.data() + (static_cast<uint64_t>(j) * k + c) * dbar;
      double acc = 0.0;
      for (uint32_t a = 0; a < dbar; ++a) acc += static_cast<double>(row[a]) * static_cast<double>(row[a]);
      const double nrm = std::sqrt(acc);
      if (nrm > 0.0) {
        norms[c] = nrm;
        for (uint32_t a = 0; a < dbar; ++a) row[a] = static_cast<float>(row[a] / nrm);
      }
    }
    double* al = alphas.data() + static_cast<uint64_t>(j) * n;
    const uint32_t* cj = codes.data() + static_cast<uint64_t>(j) * n;
    for (uint64_t i = 0; i < n; ++i) al[i] *= norms[cj[i]];
  });
  if (quantize) {
    std::vector<std::vector<double>> vals(m);
    std::vector<uint64_t> sseeds(m);
    for (uint32_t j = 0; j < m; ++j) {
      vals[j].assign(alphas.begin() + static_cast<uint64_t>(j) * n, alphas.begin() + static_cast<uint64_t>(j + 1) * n);
      sseeds[j] = Rng::mix(seed, 2ull * j + 2);
    }
    quantize_projective_all(vals, s, sseeds, scb, scodes, nt);
  }

  phase(2);
  // serialize (pq_index.cpp:372-407), method 2 (pcpq)
  const bool wide = k > 256;
  const uint64_t cbytes = static_cast<uint64_t>(m) * (wide ? 2 : 1);
  const uint64_t row = cbytes + (scales == 0 ? 4ull * m : m);
  std::vector<uint8_t> out;
  out.reserve(48 + centers.size() * 4 + 4ull * m * scales + n * row);
  auto u32 = [&](uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  };
  const char magic[8] = {'P', 'C', 'P', 'Q', 'I', 'D', 'X', '1'};
  out.insert(out.end(), magic, magic + 8);
  u32(1);
  u32(2);  // Method::pcpq
  u32(static_cast<uint32_t>(n));
  u32(d);
  u32(padded_d);
  u32(m);
  u32(k);
  u32(scales);
  uint64_t tb;
  std::memcpy(&tb, &t, 8);
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<uint8_t>(tb >> (8 * i)));
  size_t at = out.size();
  out.resize(at + centers.size() * 4);
  std::memcpy(out.data() + at, centers.data(), centers.size() * 4);
  for (uint32_t j = 0; j < m && quantize; ++j) {
    at = out.size();
    out.resize(at + 4ull * s);
    std::memcpy(out.data() + at, scb[j].data(), 4ull * s);
  }
  at = out.size();
  out.resize(at + n * row, 0);
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t* r = out.data() + at + i * row;
    for (uint32_t j = 0; j < m; ++j) {
      const uint32_t c = codes[static_cast<uint64_t>(j) * n + i];
      if (wide) {
        r[2 * j] = static_cast<uint8_t>(c);
        r[2 * j + 1] = static_cast<uint8_t>(c >> 8);
      } else {
        r[j] = static_cast<uint8_t>(c);
      }
      if (quantize) {
        r[cbytes + j] = scodes[j][i];
      } else {
        const float a = static_cast<float>(alphas[static_cast<uint64_t>(j) * n + i]);
        std::memcpy(r + cbytes + 4ull * j, &a, 4);
      }
    }
  }
  phase(3);
  return out;
}

}  // namespace pcpqg
