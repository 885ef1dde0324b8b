// Shared pieces of the GPU trainers (pcpqg_train.cu: kmeans / pcpq,
// pcpqg_train_aniso.cu: aniso / apcpq): the reference's RNG, validate_config,
// the host reseed and the chain kernels every solver uses.  Everything sits in
// an anonymous namespace, so each trainer TU has its own copy.
#pragma once
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

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

__global__ void km_iota_kernel(uint32_t* __restrict__ v, uint64_t n, uint32_t nsec) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n * nsec) v[t] = static_cast<uint32_t>(t % n);
}

// acc + v[0] + v[1] + ... + v[n-1] with sequential round-to-nearest adds (the
// reference's loop order), by one warp: the lanes load 32*U values per step
// (coalesced, the next step's loads in flight while this step adds) and the
// adds run in index order on values broadcast by shuffles, so the only
// dependent chain is the DADD itself.  Every lane returns the sum.
template <int U>
__device__ __forceinline__ double warp_ordered_sum(const double* __restrict__ v, uint64_t n, double acc) {
  const uint32_t lane = threadIdx.x & 31u;
  constexpr uint64_t SB = 32ull * U;
  double cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = static_cast<uint64_t>(u) * 32 + lane;
    cur[u] = i < n ? v[i] : 0.0;
  }
  for (uint64_t b0 = 0; b0 < n; b0 += SB) {
    const uint64_t nb = b0 + SB;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = nb + static_cast<uint64_t>(u) * 32 + lane;
      nxt[u] = i < n ? v[i] : 0.0;
    }
    if (nb <= n) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int l = 0; l < 32; ++l) acc = __dadd_rn(acc, __shfl_sync(0xFFFFFFFFu, cur[u], l));
    } else {  // the last, partial step: no padding is added (-0.0 + 0.0 would lose the sign)
      const uint32_t rem = static_cast<uint32_t>(n - b0);
#pragma unroll
      for (int u = 0; u < U; ++u)
        for (uint32_t l = 0; l < 32 && static_cast<uint32_t>(u) * 32 + l < rem; ++l)
          acc = __dadd_rn(acc, __shfl_sync(0xFFFFFFFFu, cur[u], l));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  return acc;
}

// T4b: one warp per active section: the sequential (id-order) loss chain
__global__ void km_loss_kernel(const double* __restrict__ dist, uint64_t n, const uint32_t* __restrict__ active,
                               uint32_t nact, double* __restrict__ loss) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nact) return;  // warp-uniform
  const uint32_t sec = active[w];
  const double acc = warp_ordered_sum<4>(dist + static_cast<uint64_t>(sec) * n, n, 0.0);
  if ((threadIdx.x & 31u) == 0) loss[sec] = acc;
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

// validate_config (types.cpp:35-69) + build_pq_index's k <= n check; returns
// the frozen t = t_frac * mean_l2_norm(data) (types.cpp:25-33)
double validate_train(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s, double t_frac,
                      uint32_t max_iters, double tol, bool score_aware) {
  // the finite check and the row norms on host threads; the norm sum below stays
  // sequential in row order (mean_l2_norm's order)
  std::vector<double> norms(n);
  {
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const uint64_t chunk = (n + nt - 1) / nt;
    std::vector<uint8_t> bad(nt, 0);
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        const uint64_t e = std::min(n, (w + 1) * chunk);
        for (uint64_t i = w * chunk; i < e; ++i) {
          double sq = 0.0;
          for (uint32_t a = 0; a < d; ++a) {
            const float v = X[i * d + a];
            if (!std::isfinite(v)) bad[w] = 1;
            sq += static_cast<double>(v) * v;
          }
          norms[i] = std::sqrt(sq);
        }
      });
    for (auto& x : th) x.join();
    for (uint8_t b : bad)
      if (b) fail(PCPQG_E_DATA, "dataset contains non-finite values");
  }
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
  for (uint64_t i = 0; i < n; ++i) total += norms[i];
  if (score_aware && (((d + m - 1) / m) * m) / m < 2)
    fail(PCPQG_E_DATA, "score-aware methods need section width >= 2");
  return t_frac * (total / static_cast<double>(n));
}

__global__ void tp_count_kernel(const uint32_t* __restrict__ assign, uint64_t n, uint32_t k,
                                const uint32_t* __restrict__ active, uint32_t* __restrict__ counts) {
  const uint32_t sec = active[blockIdx.y];
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&counts[static_cast<uint64_t>(sec) * k + assign[static_cast<uint64_t>(sec) * n + i]], 1u);
}

// per (active section, cluster): the member-order sums of both loss terms
__global__ void tp_loss_chain_kernel(const double* __restrict__ lo, const double* __restrict__ ln, uint64_t n,
                                     uint32_t k, const uint32_t* __restrict__ active, uint32_t nact,
                                     const uint32_t* __restrict__ counts, const uint64_t* __restrict__ offs,
                                     double* __restrict__ out) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(nact) * k * 2) return;
  const uint32_t which = static_cast<uint32_t>(t & 1);
  const uint32_t c = static_cast<uint32_t>((t >> 1) % k);
  const uint32_t sec = active[(t >> 1) / k];
  const uint64_t o = static_cast<uint64_t>(sec) * n + offs[static_cast<uint64_t>(sec) * k + c];
  const uint32_t cnt = counts[static_cast<uint64_t>(sec) * k + c];
  const double* v = (which ? ln : lo) + o;
  double acc = 0.0;
  uint32_t i = 0;
  for (; i + 8 <= cnt; i += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = v[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, x[u]);
  }
  for (; i < cnt; ++i) acc = __dadd_rn(acc, v[i]);
  out[(static_cast<uint64_t>(sec) * k + c) * 2 + which] = acc;
}

// seed_centers(require_nonzero = true) (clustering.cpp:118-144): k-means++ over
// the nonzero rows, of canonical_rows(x) (clustering.cpp:50-66) for the
// projective solver, of x itself for the score-aware ones
void seed_nonzero(const float* x, uint64_t n, uint32_t dbar, uint32_t k, uint64_t seed, bool canonical,
                  float* centers) {
  std::vector<float> canon(x, x + n * dbar);
  for (uint64_t i = 0; i < n && canonical; ++i) {
    float* row = canon.data() + i * dbar;
    uint32_t piv = 0;
    float best = -1.0f;
    for (uint32_t j = 0; j < dbar; ++j) {
      const float a = std::fabs(row[j]);
      if (a > best) {
        best = a;
        piv = j;
      }
    }
    if (row[piv] < 0.0f)
      for (uint32_t j = 0; j < dbar; ++j) row[j] = -row[j];
  }
  std::vector<uint32_t> cand;
  for (uint64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (uint32_t j = 0; j < dbar; ++j)
      acc += static_cast<double>(canon[i * dbar + j]) * static_cast<double>(canon[i * dbar + j]);
    if (acc > 0.0) cand.push_back(static_cast<uint32_t>(i));
  }
  std::memset(centers, 0, 4ull * k * dbar);
  std::vector<uint32_t> seeds;
  if (!cand.empty()) {
    Rng rng(seed);
    const uint64_t nc = cand.size();
    seeds.push_back(cand[rng.next_index(nc)]);
    std::vector<double> d2(nc, std::numeric_limits<double>::infinity());
    while (seeds.size() < k) {
      const float* last = canon.data() + static_cast<uint64_t>(seeds.back()) * dbar;
      double total = 0.0;
      for (uint64_t i = 0; i < nc; ++i) {
        double dd = 0.0;
        const float* xi = canon.data() + static_cast<uint64_t>(cand[i]) * dbar;
        for (uint32_t j = 0; j < dbar; ++j) {
          const double diff = static_cast<double>(xi[j]) - static_cast<double>(last[j]);
          dd += diff * diff;
        }
        d2[i] = std::min(d2[i], dd);
        total += d2[i];
      }
      if (total <= 0.0) {
        seeds.push_back(cand[rng.next_index(nc)]);
        continue;
      }
      double target = rng.next_double() * total;
      uint64_t pick = nc - 1;
      for (uint64_t i = 0; i < nc; ++i) {
        target -= d2[i];
        if (target <= 0.0) {
          pick = i;
          break;
        }
      }
      seeds.push_back(cand[pick]);
    }
  }
  for (uint32_t j = 0; j < seeds.size(); ++j)
    std::memcpy(centers + static_cast<uint64_t>(j) * dbar, canon.data() + static_cast<uint64_t>(seeds[j]) * dbar,
                4ull * dbar);
  for (uint32_t j = static_cast<uint32_t>(seeds.size()); j < k; ++j)
    centers[static_cast<uint64_t>(j) * dbar + (j % dbar)] = 1.0f;  // deterministic nonzero fill
}

}  // namespace
}  // namespace pcpqg
