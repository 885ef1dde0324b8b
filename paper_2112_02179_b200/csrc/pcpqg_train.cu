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

#include "pcpqg_internal.hpp"

namespace pcpqg {
namespace {

// ---- the reference's RNG (proj/core/src/rng.cpp): xoshiro256++ seeded by splitmix64
uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) w = splitmix64(sm);
  }
  uint64_t next_u64() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  size_t next_index(size_t bound) {
    return static_cast<size_t>((static_cast<unsigned __int128>(next_u64()) * bound) >> 64);
  }
  static uint64_t mix(uint64_t seed, uint64_t tag) {
    uint64_t state = seed ^ (0x9E3779B97F4A7C15ull + (tag << 1));
    const uint64_t a = splitmix64(state);
    state ^= tag;
    return a ^ splitmix64(state);
  }
};

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

__global__ void km_iota_kernel(uint32_t* __restrict__ v, uint64_t n, uint32_t nsec) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n * nsec) v[t] = static_cast<uint32_t>(t % n);
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

// T4b: one thread per active section: the sequential loss chain
__global__ void km_loss_kernel(const double* __restrict__ dist, uint64_t n, const uint32_t* __restrict__ active,
                               uint32_t nact, double* __restrict__ loss) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nact) return;
  const uint32_t sec = active[t];
  const double* d = dist + static_cast<uint64_t>(sec) * n;
  double acc = 0.0;
  uint64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = d[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; i < n; ++i) acc = __dadd_rn(acc, d[i]);
  loss[sec] = acc;
}

// exclusive offsets of the cluster counts per section
__global__ void km_offsets_kernel(const uint32_t* __restrict__ counts, uint32_t nsec, uint32_t k,
                                  uint64_t* __restrict__ offs) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsec) return;
  uint64_t o = 0;
  for (uint32_t c = 0; c < k; ++c) {
    offs[static_cast<uint64_t>(s) * k + c] = o;
    o += counts[static_cast<uint64_t>(s) * k + c];
  }
}

template <class T>
T* talloc(std::vector<void*>& keep, size_t cnt) {
  void* p = nullptr;
  PCPQG_CUDA(cudaMalloc(&p, std::max<size_t>(cnt, 1) * sizeof(T)));
  keep.push_back(p);
  return static_cast<T*>(p);
}

// reseed_empty_clusters (clustering.cpp:156-185) for one section on the host
void reseed_host(const float* x, uint64_t n, uint32_t dbar, uint32_t k, float* centers,
                 uint32_t* assignment, double* ploss) {
  std::vector<uint64_t> counts(k, 0);
  for (uint64_t i = 0; i < n; ++i) ++counts[assignment[i]];
  for (bool changed = true; changed;) {
    changed = false;
    for (uint32_t j = 0; j < k; ++j) {
      if (counts[j] > 0) continue;
      uint64_t far = 0;
      double fl = 0.0;
      for (uint64_t i = 0; i < n; ++i)
        if (ploss[i] > fl) {
          fl = ploss[i];
          far = i;
        }
      if (!(fl > 0.0)) continue;
      std::memcpy(centers + static_cast<uint64_t>(j) * dbar, x + far * dbar, 4ull * dbar);
      --counts[assignment[far]];
      ++counts[j];
      assignment[far] = j;
      ploss[far] = 0.0;
      changed = true;
    }
  }
}

}  // namespace

std::vector<uint8_t> train_kmeans(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                  double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device) {
  // ---- validate_config (types.cpp:35-69) and build_pq_index's own check
  for (uint64_t i = 0; i < n * d; ++i)
    if (!std::isfinite(X[i])) fail(PCPQG_E_DATA, "dataset contains non-finite values");
  if (n == 0) fail(PCPQG_E_DATA, "empty dataset");
  if (d == 0) fail(PCPQG_E_DATA, "zero-dimensional dataset");
  if (m == 0) fail(PCPQG_E_DATA, "m must be >= 1");
  if (m > d) fail(PCPQG_E_DATA, "m exceeds dimensionality");
  if (k < 2) fail(PCPQG_E_DATA, "k must be >= 2");
  if (s < 1) fail(PCPQG_E_DATA, "s must be >= 1");
  if (s >= (1u << 16)) fail(PCPQG_E_DATA, "s out of range");
  if (!std::isfinite(t_frac) || t_frac < 0.0) fail(PCPQG_E_DATA, "t_frac must be finite and non-negative");
  if (max_iters < 1) fail(PCPQG_E_DATA, "max_iters must be >= 1");
  if (!(tol > 0.0)) fail(PCPQG_E_DATA, "tol must be positive");
  if (k > n) fail(PCPQG_E_DATA, "build_pq_index: k exceeds point count");
  if (k > 65536) fail(PCPQG_E_DATA, "serialize: k too large for the code width");
  if (n > 0xFFFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "more than 2^32 points");
  double total = 0.0;  // mean_l2_norm (types.cpp:25-33)
  for (uint64_t i = 0; i < n; ++i) {
    double sq = 0.0;
    for (uint32_t a = 0; a < d; ++a) sq += static_cast<double>(X[i * d + a]) * X[i * d + a];
    total += std::sqrt(sq);
  }
  const double t = t_frac * (total / static_cast<double>(n));
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
    km_loss_kernel<<<(nact + 31) / 32, 32>>>(dDist, n, dAct, nact, dLoss);
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
