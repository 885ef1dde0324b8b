// GPU index training, methods aniso (ScaNN baseline) and apcpq (SURVEY.md §8(f)
// row 3; BASELINE config 5): pcpq::build_pq_index(method = aniso / apcpq)
// (proj/core/src/pq_index.cpp:62-168) with the score-aware solver aniso_solver
// (proj/core/src/clustering.cpp:622-722) per section, producing the reference's
// PCPQIDX1 image byte for byte.
//
// Host: validate_config, the per-section seeds (seed_centers with
//   require_nonzero, Rng::mix(seed, 2j+1)), the anisotropic weights
//   (aniso_weights, clustering.cpp:204-217: Simpson sums of the C library's sin,
//   computed once on host threads and reused by the quantizer, which the
//   reference recomputes bit-identically), the empty-cluster reseed, the
//   d̄ x d̄ Cholesky solves of center_anisotropic (numerics.cpp:138-172), the
//   convergence test; for quantized apcpq the quadratics and the final code
//   snapping per section on host threads.
// GPU, all active sections at once:
//   A1  assign_aniso_impl (launch_assign_anisotropic, fixed or optimal scale,
//       keep-previous fallback after the first iteration)
//   A2  member lists: stable segmented radix sort (members_of order)
//   A3  center_anisotropic statistics: exact member-order fp64 sums
//       (launch_center_stats)
//   A4  cluster_loss of the old center and the candidate: per-member terms in
//       parallel, member-order chains per cluster (clustering.cpp:655-666, :700-702)
//   A5  the scale refresh and loss trace: per-point terms, one id-order chain
//       per section (clustering.cpp:705-718)
//   MQ  minimize_quadratic_scalars (numerics.cpp:328-404) for every (section,
//       restart) at once: assignment rounds in parallel, the objective and the
//       per-level sums as ordered chains; RNG and level updates on the host
// Every fp64 operation is an explicit round-to-nearest intrinsic in the
// reference's evaluation order, so the assignment, the centers, the loss trace
// and with them every convergence decision are bit-identical.
#include <chrono>

#include "pcpqg_train_common.cuh"

namespace pcpqg {
namespace {

// PCPQG_TRAIN_TRACE=1: wall time of the trainer's sub-phases on stderr
struct TrainTrace {
  bool on = std::getenv("PCPQG_TRAIN_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pcpqg train] %-28s %.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

// ---- host numerics (proj/core/src/numerics.cpp)
double ipow_host(double base, int p) {  // numerics.cpp:22-29
  double r = 1.0, b = base;
  for (int e = p; e > 0; e >>= 1) {
    if (e & 1) r *= b;
    b *= b;
  }
  return r;
}

// sin_power_integral (numerics.cpp:174-186: composite Simpson, 1024 panels) for
// p_lo and p_hi in one pass: both sums see
// the same sin(i*h) values and keep their own order, so each is bit-identical
// to a separate call — at half the sin evaluations
void sin_power_integral_pair(int p_lo, int p_hi, double theta_max, double& i_lo, double& i_hi) {
  const double hi = 3.141592653589793 / 2.0;
  const double t = std::clamp(theta_max, 0.0, hi);
  if (t == 0.0) {
    i_lo = i_hi = 0.0;
    return;
  }
  const double h = t / 1024;
  const double s0 = std::sin(0.0), st = std::sin(t);
  double sum_lo = ipow_host(s0, p_lo) + ipow_host(st, p_lo);
  double sum_hi = ipow_host(s0, p_hi) + ipow_host(st, p_hi);
  for (int i = 1; i < 1024; ++i) {
    const double si = std::sin(i * h);
    const double f_lo = ipow_host(si, p_lo), f_hi = ipow_host(si, p_hi);
    sum_lo += (i & 1) ? 4.0 * f_lo : 2.0 * f_lo;
    sum_hi += (i & 1) ? 4.0 * f_hi : 2.0 * f_hi;
  }
  i_lo = sum_lo * h / 3.0;
  i_hi = sum_hi * h / 3.0;
}

// aniso_weights (clustering.cpp:204-217) for norm_x > 0
void aniso_weights_one(double norm_x, double t, int dbar, double& h_par, double& h_bot) {
  const double theta = t / norm_x;
  double i_lo, i_hi;
  sin_power_integral_pair(dbar - 2, dbar, theta, i_lo, i_hi);
  h_bot = std::max(i_hi, 0.0);
  h_par = std::max((dbar - 1) * (i_lo - i_hi), h_bot);
}

// solve_spd (numerics.cpp:138-172) for the d x d system a (row-major, full);
// false where the reference throws errc::numeric (not positive definite)
bool solve_spd_host(std::vector<double> l, const double* b, uint32_t d, double ridge, double* x) {
  for (uint32_t i = 0; i < d; ++i) l[i * d + i] += ridge;
  for (uint32_t j = 0; j < d; ++j) {
    double diag = l[j * d + j];
    for (uint32_t c = 0; c < j; ++c) diag -= l[j * d + c] * l[j * d + c];
    if (!(diag > 0.0)) return false;
    diag = std::sqrt(diag);
    l[j * d + j] = diag;
    for (uint32_t i = j + 1; i < d; ++i) {
      double acc = l[i * d + j];
      for (uint32_t c = 0; c < j; ++c) acc -= l[i * d + c] * l[j * d + c];
      l[i * d + j] = acc / diag;
    }
  }
  std::vector<double> y(d);
  for (uint32_t i = 0; i < d; ++i) {
    double acc = b[i];
    for (uint32_t c = 0; c < i; ++c) acc -= l[i * d + c] * y[c];
    y[i] = acc / l[i * d + i];
  }
  for (uint32_t ii = d; ii-- > 0;) {
    double acc = y[ii];
    for (uint32_t c = ii + 1; c < d; ++c) acc -= l[c * d + ii] * x[c];
    x[ii] = acc / l[ii * d + ii];
  }
  return true;
}

struct Quad {
  double w, a, b;
};
void canonicalize(std::vector<double>& values, std::vector<uint32_t>& best_assign);

// canonicalize_codebook (numerics.cpp:188-209): ascending (stable), exact
// duplicates merged, the assignment remapped
void canonicalize(std::vector<double>& values, std::vector<uint32_t>& best_assign) {
  const uint32_t ns = static_cast<uint32_t>(values.size());
  std::vector<uint32_t> order(ns);
  for (uint32_t i = 0; i < ns; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return values[a] < values[b]; });
  std::vector<double> sorted;
  std::vector<uint32_t> remap(ns, 0);
  for (uint32_t pos = 0; pos < ns; ++pos) {
    const double val = values[order[pos]];
    if (sorted.empty() || val != sorted.back()) sorted.push_back(val);
    remap[order[pos]] = static_cast<uint32_t>(sorted.size() - 1);
  }
  values = sorted;
  for (auto& a : best_assign) a = remap[a];
}

double dot_host(const float* a, const float* b, uint32_t n) {  // dotf, clustering.cpp:14-19
  double acc = 0.0;
  for (uint32_t i = 0; i < n; ++i) acc += static_cast<double>(a[i]) * static_cast<double>(b[i]);
  return acc;
}

// quantize_anisotropic (scalar_quant.cpp:72-150), split around the fit:
// the per-point quadratics of one section (points with zero norm or no
// curvature excluded) ...
struct QuantSection {
  std::vector<Quad> quads;
  std::vector<uint64_t> quad_of;   // point id per quad
  std::vector<double> values;      // fitted codebook (canonical)
  std::vector<uint32_t> assign;    // per quad
};

void build_quads(const float* x, uint64_t n, uint32_t dbar, const float* centers, uint32_t k, const uint32_t* assign,
                 const double* hp, const double* hb, QuantSection& qs) {
  std::vector<double> c2(k);
  for (uint32_t j = 0; j < k; ++j) c2[j] = dot_host(centers + static_cast<uint64_t>(j) * dbar,
                                                    centers + static_cast<uint64_t>(j) * dbar, dbar);
  qs.quads.clear();
  qs.quad_of.clear();
  qs.quads.reserve(n);
  qs.quad_of.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    const float* xi = x + i * dbar;
    const double nx2 = dot_host(xi, xi, dbar);
    if (nx2 == 0.0) continue;
    const double ip = dot_host(xi, centers + static_cast<uint64_t>(assign[i]) * dbar, dbar);
    const double wq = (hp[i] - hb[i]) * ip * ip / nx2 + hb[i] * c2[assign[i]];
    if (!(wq > 0.0)) continue;
    qs.quads.push_back({wq, -2.0 * hp[i] * ip, hp[i] * nx2});
    qs.quad_of.push_back(i);
  }
}

// ... and, after minimize_quadratic_scalars, the padded float codebook and
// the codes: every quad snapped against the float codebook (ties to the lower
// code), excluded points to nearest_code(values, 0.0)
void finish_quantize(const QuantSection& qs, uint64_t n, uint32_t s, std::vector<float>& cb,
                     std::vector<uint8_t>& codes) {
  codes.assign(n, 0);
  cb.clear();
  if (qs.quads.empty()) {  // nothing carries loss: one zero scale
    cb.assign(s, 0.0f);
    return;
  }
  for (double v : qs.values) cb.push_back(static_cast<float>(v));  // pad_codebook
  while (cb.size() < s) cb.push_back(cb.empty() ? 0.0f : cb.back());
  for (uint64_t qi = 0; qi < qs.quads.size(); ++qi) {
    double best = std::numeric_limits<double>::infinity();
    uint8_t bl = 0;
    for (uint32_t l = 0; l < s; ++l) {
      const double lam = cb[l];
      const double v = (qs.quads[qi].w * lam + qs.quads[qi].a) * lam + qs.quads[qi].b;
      if (v < best) {
        best = v;
        bl = static_cast<uint8_t>(l);
      }
    }
    codes[qs.quad_of[qi]] = bl;
  }
  if (qs.quads.size() != n) {
    uint8_t zero_code = 0;
    double bd = std::numeric_limits<double>::infinity();
    for (uint32_t l = 0; l < s; ++l) {
      const double dd = std::fabs(static_cast<double>(cb[l]) - 0.0);
      if (dd < bd) {
        bd = dd;
        zero_code = static_cast<uint8_t>(l);
      }
    }
    std::vector<bool> fitted(n, false);
    for (auto i : qs.quad_of) fitted[i] = true;
    for (uint64_t i = 0; i < n; ++i)
      if (!fitted[i]) codes[i] = zero_code;
  }
}

// ---- device pieces
__device__ __forceinline__ double ta_dot(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(a[i]), static_cast<double>(b[i])));
  return acc;
}

// quad_at(point_quad(ip, nx2, c2, {hp, hb}), l)  (clustering.cpp:29-34)
__device__ __forceinline__ double ta_quad_at(double ip, double nx2, double c2, double hp, double hb, double l) {
  const double w = __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), ip), ip), nx2), __dmul_rn(hb, c2));
  const double a = __dmul_rn(__dmul_rn(-2.0, hp), ip);
  const double b = __dmul_rn(hp, nx2);
  return __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(w, l), a), l), b);
}

// opt_alpha_from (clustering.cpp:36-40)
__device__ __forceinline__ double ta_opt_alpha(double ip, double nx2, double c2, double hp, double hb) {
  const double denom =
      __dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(__dsub_rn(hp, hb), ip), ip), nx2), __dmul_rn(hb, c2));
  if (fabs(denom) <= 1e-30) return 0.0;
  return __ddiv_rn(__dmul_rn(hp, ip), denom);
}

// A4: per sorted member, cluster_loss terms under the old center and the candidate
__global__ void ta_cluster_terms_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                                        const uint32_t* __restrict__ active, const uint32_t* __restrict__ members,
                                        const uint32_t* __restrict__ sorted_assign, const float* __restrict__ C,
                                        const float* __restrict__ Cand, const double* __restrict__ hp,
                                        const double* __restrict__ hb, const double* __restrict__ alpha,
                                        double* __restrict__ lo, double* __restrict__ ln) {
  const uint32_t sec = active[blockIdx.y];
  const uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t so = static_cast<uint64_t>(sec) * n;
  const uint32_t i = members[so + p];
  const uint32_t c = sorted_assign[so + p];
  const float* xi = X + (so + i) * dbar;
  const double nx2 = ta_dot(xi, xi, dbar);
  if (nx2 == 0.0) {  // skipped by the reference: +0.0 never changes the chain
    lo[so + p] = 0.0;
    ln[so + p] = 0.0;
    return;
  }
  const float* co = C + (static_cast<uint64_t>(sec) * k + c) * dbar;
  const float* cn = Cand + (static_cast<uint64_t>(sec) * k + c) * dbar;
  const double h1 = hp[so + i], h0 = hb[so + i], al = alpha[so + i];
  lo[so + p] = ta_quad_at(ta_dot(xi, co, dbar), nx2, ta_dot(co, co, dbar), h1, h0, al);
  ln[so + p] = ta_quad_at(ta_dot(xi, cn, dbar), nx2, ta_dot(cn, cn, dbar), h1, h0, al);
}

// A5: per point (id order), the refreshed scale and its loss term
__global__ void ta_refresh_kernel(const float* __restrict__ X, uint64_t n, uint32_t dbar, uint32_t k,
                                  const uint32_t* __restrict__ active, const uint32_t* __restrict__ assign,
                                  const float* __restrict__ C, const double* __restrict__ hp,
                                  const double* __restrict__ hb, bool scaling, double* __restrict__ alpha,
                                  double* __restrict__ term) {
  const uint32_t sec = active[blockIdx.y];
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g = static_cast<uint64_t>(sec) * n + i;
  const float* xi = X + g * dbar;
  const double nx2 = ta_dot(xi, xi, dbar);
  if (nx2 == 0.0) {
    alpha[g] = scaling ? 0.0 : 1.0;
    term[g] = 0.0;
    return;
  }
  const float* cj = C + (static_cast<uint64_t>(sec) * k + assign[g]) * dbar;
  const double ip = ta_dot(xi, cj, dbar), c2 = ta_dot(cj, cj, dbar);
  double al = alpha[g];
  if (scaling) al = ta_opt_alpha(ip, nx2, c2, hp[g], hb[g]);
  alpha[g] = al;
  term[g] = ta_quad_at(ip, nx2, c2, hp[g], hb[g], al);
}

// ---- minimize_quadratic_scalars on the GPU (numerics.cpp:328-404): every
// (section, restart) is an independent problem; per round
//   MQ1  assignment: per (problem, quad) the first minimum of
//        ((w*l)*l + a*l) + b over the problem's s levels, and whether it
//        differs from the previous round's
//   MQ2  the per-level sums of w and a (one chain per level, in quad order)
// and, once after the rounds,
//   MQ3  every problem's objective: the chain over its last round's minima in
//        quad order (the reference recomputes it each round and reads only
//        the last)
// The host keeps each restart's RNG (initial picks, empty-level reseeds),
// the level update -sa / (2 sw), the convergence test and the best restart,
// so every value and decision is the reference's.
__device__ __forceinline__ double mq_eval(double w, double a, double b, double l) {
  return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(w, l), l), __dmul_rn(a, l)), b);
}

__global__ void mq_assign_kernel(const double* __restrict__ W, const double* __restrict__ A,
                                 const double* __restrict__ Bq, const uint64_t* __restrict__ poff,
                                 const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                                 const uint32_t* __restrict__ act, uint32_t s, const double* __restrict__ lam,
                                 const uint8_t* __restrict__ prev, uint8_t* __restrict__ cur, int check,
                                 uint32_t* __restrict__ changed, double* __restrict__ bvout) {
  __shared__ double sl[256];
  const uint32_t p = act[blockIdx.y];
  for (uint32_t t = threadIdx.x; t < s; t += blockDim.x) sl[t] = lam[static_cast<uint64_t>(p) * s + t];
  __syncthreads();
  const uint64_t n = pcnt[p], o = poff[p], ab = pbase[p];
  int diff = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double w = W[o + i], a = A[o + i], b = Bq[o + i];
    double bv = INFINITY;
    uint32_t bj = 0;
    for (uint32_t j = 0; j < s; ++j) {
      const double v = mq_eval(w, a, b, sl[j]);
      if (v < bv) {  // strict: ties keep the lower level
        bv = v;
        bj = j;
      }
    }
    cur[ab + i] = static_cast<uint8_t>(bj);
    bvout[ab + i] = bv;
    diff |= check && prev[ab + i] != bj;
  }
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(changed + p, 1u);
}

// One warp per (problem, level g): sw[g] += w, sa[g] += a over the level's quads
// in index order (numerics.cpp:387-390).  The warp walks the assignment in
// steps of 256 quads (8 coalesced byte loads per lane, the next step's in
// flight), compacts the step's members — in index order, by ballot ranks —
// into a shared buffer, and adds them sequentially from there.
constexpr int kMqWarps = 4;
__global__ void __launch_bounds__(32 * kMqWarps)
    mq_sums_kernel(const double* __restrict__ W, const double* __restrict__ A, const uint64_t* __restrict__ poff,
                   const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                   const uint32_t* __restrict__ act, uint32_t nact, uint32_t s, const uint8_t* __restrict__ cur,
                   double* __restrict__ sums) {
  __shared__ double2 buf_all[kMqWarps][256];
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (wid >= static_cast<uint64_t>(nact) * s) return;  // warp-uniform
  double2* buf = buf_all[threadIdx.x >> 5];
  const uint32_t p = act[wid / s];
  const uint32_t g = static_cast<uint32_t>(wid % s);
  const uint64_t n = pcnt[p], o = poff[p], ab = pbase[p];
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t cn[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint64_t i = static_cast<uint64_t>(u) * 32 + lane;
    cn[u] = i < n ? cur[ab + i] : 0xFFFFu;
  }
  double sw = 0.0, sa = 0.0;
  for (uint64_t b0 = 0; b0 < n; b0 += 256) {
    uint32_t cc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) cc[u] = cn[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = b0 + 256 + static_cast<uint64_t>(u) * 32 + lane;
      cn[u] = i < n ? cur[ab + i] : 0xFFFFu;
    }
    uint32_t base = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool mine = cc[u] == g;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mine);
      if (mine) {
        const uint64_t i = o + b0 + static_cast<uint64_t>(u) * 32 + lane;
        buf[base + __popc(bal & lt)] = make_double2(W[i], A[i]);
      }
      base += __popc(bal);
    }
    __syncwarp();
    uint32_t r = 0;
    for (; r + 4 <= base; r += 4) {
      const double2 v0 = buf[r], v1 = buf[r + 1], v2 = buf[r + 2], v3 = buf[r + 3];
      sw = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sw, v0.x), v1.x), v2.x), v3.x);
      sa = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sa, v0.y), v1.y), v2.y), v3.y);
    }
    for (; r < base; ++r) {
      const double2 v = buf[r];
      sw = __dadd_rn(sw, v.x);
      sa = __dadd_rn(sa, v.y);
    }
    __syncwarp();
  }
  if (lane == 0) {
    sums[(static_cast<uint64_t>(p) * s + g) * 2] = sw;
    sums[(static_cast<uint64_t>(p) * s + g) * 2 + 1] = sa;
  }
}

// ---- per-level sums through a stable counting sort (s <= 16).  mq_sums_kernel
// makes every level's warp walk the whole assignment (s-fold redundant reads,
// ~8 instructions per quad); here the quads of a problem are stably partitioned
// by level — index order kept inside a level — so each level's ordered sum
// reads only its own contiguous run:
//   mq_lcount_kernel    per (chunk of 4096 quads, problem): per-level counts
//   mq_loffsets_kernel  per problem: the chunks' offsets inside each level's run,
//                       the runs' bases and lengths
//   mq_lscatter_kernel  per (chunk, problem): w and a to their sorted positions
//                       (a thread owns 16 consecutive quads; its rank inside a
//                       level = a block-wide exclusive scan of packed counters)
//   mq_lsum_kernel      per (problem, level): the two ordered sums over the run
constexpr uint32_t kMqChunk = 4096;
constexpr uint32_t kMqLv = 16;  // levels the packed counters hold (4 x u64, 16-bit fields)

struct LvCnt {
  uint64_t c[4];
};
__device__ __forceinline__ void lv_add(LvCnt& x, uint32_t lv) {
  const uint64_t one = 1ull << (16u * (lv & 3u));
  const uint32_t w = lv >> 2;
  x.c[0] += w == 0 ? one : 0ull;
  x.c[1] += w == 1 ? one : 0ull;
  x.c[2] += w == 2 ? one : 0ull;
  x.c[3] += w == 3 ? one : 0ull;
}
__device__ __forceinline__ uint32_t lv_get(const LvCnt& x, uint32_t lv) {
  const uint32_t w = lv >> 2;
  const uint64_t v = w == 0 ? x.c[0] : (w == 1 ? x.c[1] : (w == 2 ? x.c[2] : x.c[3]));
  return static_cast<uint32_t>(v >> (16u * (lv & 3u))) & 0xFFFFu;
}

// the 16 assignment bytes of thread t of a chunk (0xFF past the end)
__device__ __forceinline__ void mq_load_levels(const uint8_t* __restrict__ cur, uint64_t i0, uint64_t n,
                                               uint8_t (&lv)[16]) {
  if (i0 + 16 <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(cur + i0);  // (regions are 16-byte aligned)
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) lv[j] = static_cast<uint8_t>(w4[j >> 2] >> (8 * (j & 3)));
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) lv[j] = i0 + j < n ? cur[i0 + j] : static_cast<uint8_t>(0xFF);
  }
}

__global__ void __launch_bounds__(256)
    mq_lcount_kernel(const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                     const uint32_t* __restrict__ act, const uint8_t* __restrict__ cur, uint32_t nch,
                     uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[kMqLv];
  const uint32_t p = act[blockIdx.y], chunk = blockIdx.x;
  const uint64_t n = pcnt[p], c0 = static_cast<uint64_t>(chunk) * kMqChunk;
  if (c0 >= n) return;  // block-uniform
  if (threadIdx.x < kMqLv) h[threadIdx.x] = 0;
  __syncthreads();
  uint8_t lv[16];
  mq_load_levels(cur + pbase[p], c0 + 16ull * threadIdx.x, n, lv);
  LvCnt c{{0, 0, 0, 0}};
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (lv[j] < kMqLv) lv_add(c, lv[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) c.c[k4] += __shfl_xor_sync(0xFFFFFFFFu, c.c[k4], o);
  if ((threadIdx.x & 31) == 0)
    for (uint32_t l = 0; l < kMqLv; ++l) {
      const uint32_t v = lv_get(c, l);
      if (v) atomicAdd(&h[l], v);
    }
  __syncthreads();
  if (threadIdx.x < kMqLv) counts[(static_cast<uint64_t>(p) * nch + chunk) * kMqLv + threadIdx.x] = h[threadIdx.x];
}

// one warp per active problem, lane = level: counts -> the chunk's offset inside
// the level's run (in place); lbase / lcnt = the runs' bases and lengths
__global__ void mq_loffsets_kernel(const uint64_t* __restrict__ pcnt, const uint32_t* __restrict__ act,
                                   uint32_t nact, uint32_t nch, uint32_t* __restrict__ counts,
                                   uint64_t* __restrict__ lbase, uint64_t* __restrict__ lcnt) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nact) return;
  const uint32_t p = act[w];
  const uint32_t used = static_cast<uint32_t>((pcnt[p] + kMqChunk - 1) / kMqChunk);
  uint64_t run = 0;
  if (lane < kMqLv) {
    uint32_t* c = counts + static_cast<uint64_t>(p) * nch * kMqLv + lane;
    for (uint32_t ch = 0; ch < used; ++ch) {
      const uint32_t v = c[static_cast<uint64_t>(ch) * kMqLv];
      c[static_cast<uint64_t>(ch) * kMqLv] = static_cast<uint32_t>(run);
      run += v;
    }
  }
  uint64_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += v;
  }
  if (lane < kMqLv) {
    lbase[static_cast<uint64_t>(p) * kMqLv + lane] = incl - run;
    lcnt[static_cast<uint64_t>(p) * kMqLv + lane] = run;
  }
}

// The chunk's quads are first placed level-major in shared memory (a thread owns
// 16 consecutive quads; its rank inside a level = a block-wide exclusive scan of
// packed counters), then every level's run leaves as consecutive 16-byte {w, a}
// stores — the sorted copy is written coalesced.
__global__ void __launch_bounds__(256)
    mq_lscatter_kernel(const double* __restrict__ W, const double* __restrict__ A, const uint64_t* __restrict__ poff,
                       const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase,
                       const uint32_t* __restrict__ act, const uint8_t* __restrict__ cur, uint32_t nch,
                       const uint32_t* __restrict__ choff, const uint64_t* __restrict__ lbase, uint64_t npad,
                       double2* __restrict__ SWA) {
  extern __shared__ __align__(16) uint8_t smem_ls[];
  double2* stage = reinterpret_cast<double2*>(smem_ls);                      // [kMqChunk] level-major
  uint8_t* slev = smem_ls + static_cast<size_t>(kMqChunk) * sizeof(double2);  // [kMqChunk] level of a staged slot
  __shared__ uint64_t sbase[kMqLv];
  __shared__ uint32_t lstart[kMqLv + 1];
  __shared__ LvCnt wtot[8];
  const uint32_t p = act[blockIdx.y], chunk = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t n = pcnt[p], c0 = static_cast<uint64_t>(chunk) * kMqChunk;
  if (c0 >= n) return;  // block-uniform
  if (tid < kMqLv)
    sbase[tid] = lbase[static_cast<uint64_t>(p) * kMqLv + tid] +
                 choff[(static_cast<uint64_t>(p) * nch + chunk) * kMqLv + tid];
  const uint64_t i0 = c0 + 16ull * tid;
  uint8_t lv[16];
  mq_load_levels(cur + pbase[p], i0, n, lv);
  double w[16], a[16];
  {
    const double* wp = W + poff[p] + i0;
    const double* ap = A + poff[p] + i0;
    if (i0 + 16 <= n) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const double2 w2 = *reinterpret_cast<const double2*>(wp + j), a2 = *reinterpret_cast<const double2*>(ap + j);
        w[j] = w2.x, w[j + 1] = w2.y, a[j] = a2.x, a[j + 1] = a2.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        w[j] = i0 + j < n ? wp[j] : 0.0;
        a[j] = i0 + j < n ? ap[j] : 0.0;
      }
    }
  }
  LvCnt c{{0, 0, 0, 0}};
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (lv[j] < kMqLv) lv_add(c, lv[j]);
  // exclusive scan over the block's threads (quad order = thread order)
  LvCnt incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, incl.c[k4], o);
      if (lane >= static_cast<uint32_t>(o)) incl.c[k4] += v;
    }
  if (lane == 31) wtot[wid] = incl;
  __syncthreads();
  LvCnt run{{0, 0, 0, 0}}, tot{{0, 0, 0, 0}};
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    uint64_t before = 0, all = 0;
    for (uint32_t t = 0; t < 8; ++t) {
      before += t < wid ? wtot[t].c[k4] : 0ull;
      all += wtot[t].c[k4];
    }
    run.c[k4] = before + incl.c[k4] - c.c[k4];
    tot.c[k4] = all;
  }
  if (tid == 0) {  // where each level's run starts in the staged chunk
    uint32_t acc = 0;
    for (uint32_t l = 0; l < kMqLv; ++l) {
      lstart[l] = acc;
      acc += lv_get(tot, l);
    }
    lstart[kMqLv] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t l = lv[j];
    if (l < kMqLv) {
      const uint32_t slot = lstart[l] + lv_get(run, l);
      lv_add(run, l);
      stage[slot] = make_double2(w[j], a[j]);
      slev[slot] = static_cast<uint8_t>(l);
    }
  }
  __syncthreads();
  double2* out = SWA + static_cast<uint64_t>(p) * npad;
  const uint32_t cnt = lstart[kMqLv];
  for (uint32_t i = tid; i < cnt; i += 256) {
    const uint32_t l = slev[i];
    out[sbase[l] + (i - lstart[l])] = stage[i];
  }
}

// One warp per (problem, level): the two ordered sums over the level's run of
// {w, a} pairs.  The warp stages 128 pairs at a time in shared memory
// (coalesced 16-byte loads, the next step's in flight) and adds them in order
// from there: one broadcast LDS.128 and two DADDs per pair.  (Broadcasting the
// values by shuffles instead — warp_ordered_sum — is shuffle-throughput bound
// once thousands of warps do it: 72 ms per round at n = 1e7.)
constexpr int kLsWarps = 4;
__global__ void __launch_bounds__(32 * kLsWarps)
    mq_lsum_kernel(const uint32_t* __restrict__ act, uint32_t nact, uint32_t s, const uint64_t* __restrict__ lbase,
                   const uint64_t* __restrict__ lcnt, uint64_t npad, const double2* __restrict__ SWA,
                   double* __restrict__ sums) {
  __shared__ __align__(16) double2 buf_all[kLsWarps][128];
  const uint64_t wid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (wid >= static_cast<uint64_t>(nact) * s) return;  // warp-uniform
  double2* buf = buf_all[threadIdx.x >> 5];
  const uint32_t p = act[wid / s], g = static_cast<uint32_t>(wid % s);
  const double2* src = SWA + static_cast<uint64_t>(p) * npad + lbase[static_cast<uint64_t>(p) * kMqLv + g];
  const uint64_t n = lcnt[static_cast<uint64_t>(p) * kMqLv + g];
  double sw = 0.0, sa = 0.0;
  double2 nx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint64_t i = static_cast<uint64_t>(u) * 32 + lane;
    nx[u] = i < n ? src[i] : make_double2(0.0, 0.0);
  }
  for (uint64_t b0 = 0; b0 < n; b0 += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) buf[u * 32 + lane] = nx[u];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = b0 + 128 + static_cast<uint64_t>(u) * 32 + lane;
      nx[u] = i < n ? src[i] : make_double2(0.0, 0.0);
    }
    __syncwarp();
    const uint32_t cnt = n - b0 < 128 ? static_cast<uint32_t>(n - b0) : 128u;
    if (cnt == 128) {
#pragma unroll 16
      for (uint32_t r = 0; r < 128; ++r) {
        const double2 v = buf[r];
        sw = __dadd_rn(sw, v.x);
        sa = __dadd_rn(sa, v.y);
      }
    } else {
      for (uint32_t r = 0; r < cnt; ++r) {
        const double2 v = buf[r];
        sw = __dadd_rn(sw, v.x);
        sa = __dadd_rn(sa, v.y);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    sums[(static_cast<uint64_t>(p) * s + g) * 2] = sw;
    sums[(static_cast<uint64_t>(p) * s + g) * 2 + 1] = sa;
  }
}

// One warp per problem: obj = the sum of the last round's bv in index order
// (numerics.cpp:371-383; only the final round's value is ever read, so it is
// computed once, after the rounds)
__global__ void mq_obj_kernel(const uint64_t* __restrict__ pcnt, const uint64_t* __restrict__ pbase, uint32_t P,
                              const double* __restrict__ bv, double* __restrict__ obj) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= P) return;  // warp-uniform
  const double acc = warp_ordered_sum<4>(bv + pbase[p], pcnt[p], 0.0);
  if ((threadIdx.x & 31u) == 0) obj[p] = acc;
}

// minimize_quadratic_scalars for every section with quads (seeds[j] = the
// section's scale seed), canonicalized; fills qs[j].values / .assign
void minimize_quadratic_scalars_gpu(std::vector<QuantSection>& qs, uint32_t s, const std::vector<uint64_t>& seeds) {
  std::vector<uint32_t> secs;
  uint64_t total = 0;
  std::vector<uint64_t> soff(qs.size(), 0);
  for (uint32_t j = 0; j < qs.size(); ++j)
    if (!qs[j].quads.empty()) {
      secs.push_back(j);
      soff[j] = total;
      total += (qs[j].quads.size() + 15) / 16 * 16;  // 16-aligned regions (vector loads of the level sort)
    }
  if (secs.empty()) return;
  TrainTrace tr;
  constexpr uint32_t R = 10;  // kRestarts1D
  const uint32_t P = static_cast<uint32_t>(secs.size()) * R;
  std::vector<double> hw(total), ha(total), hbq(total);
  {  // structure-of-arrays copy of the quads, one host thread per section
    std::vector<std::thread> th;
    const unsigned nt = std::max(1u, std::min<unsigned>(static_cast<unsigned>(secs.size()),
                                                        std::min(32u, std::thread::hardware_concurrency())));
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (size_t si = w; si < secs.size(); si += nt) {
          const uint32_t j = secs[si];
          for (uint64_t i = 0; i < qs[j].quads.size(); ++i) {
            hw[soff[j] + i] = qs[j].quads[i].w;
            ha[soff[j] + i] = qs[j].quads[i].a;
            hbq[soff[j] + i] = qs[j].quads[i].b;
          }
        }
      });
    for (auto& x : th) x.join();
  }
  // problem p = (section secs[p / R], restart p % R); assignment regions
  // [restart][section items]
  std::vector<uint64_t> poff(P), pcnt(P), pbase(P);
  // minima[i] = -a / (2 w) (numerics.cpp:334-338), evaluated where it is read
  // (initial picks, empty-level reseeds): the same expression, no n-sized array
  auto minimum_of = [&](uint32_t j, uint64_t i) { return -qs[j].quads[i].a / (2.0 * qs[j].quads[i].w); };
  for (uint32_t si = 0; si < secs.size(); ++si) {
    const uint32_t j = secs[si];
    const uint64_t n = qs[j].quads.size();
    for (uint32_t r = 0; r < R; ++r) {
      poff[si * R + r] = soff[j];
      pcnt[si * R + r] = n;
      pbase[si * R + r] = r * total + soff[j];
    }
  }
  std::vector<Rng> rngs;
  rngs.reserve(P);
  std::vector<double> lam(static_cast<uint64_t>(P) * s);
  for (uint32_t p = 0; p < P; ++p) {
    const uint32_t j = secs[p / R];
    const uint64_t n = qs[j].quads.size();
    rngs.emplace_back(Rng::mix(seeds[j], p % R));  // root.split(restart)
    Rng& rng = rngs.back();
    double* lp = lam.data() + static_cast<uint64_t>(p) * s;
    if (n >= s) {
      std::vector<uint64_t> picked;
      while (picked.size() < s) {
        const uint64_t c = rng.next_index(n);
        if (std::find(picked.begin(), picked.end(), c) == picked.end()) picked.push_back(c);
      }
      for (uint32_t l = 0; l < s; ++l) lp[l] = minimum_of(j, picked[l]);
    } else {
      for (uint32_t l = 0; l < s; ++l) lp[l] = minimum_of(j, l < n ? l : rng.next_index(n));
    }
  }
  tr.mark("mq: SoA copy + seeds");
  std::vector<void*> keep;
  struct Free {
    std::vector<void*>* k;
    ~Free() {
      for (void* p : *k) cudaFree(p);
    }
  } fr{&keep};
  double* dW = talloc<double>(keep, total);
  double* dA = talloc<double>(keep, total);
  double* dB = talloc<double>(keep, total);
  uint64_t* dOff = talloc<uint64_t>(keep, P);
  uint64_t* dCnt = talloc<uint64_t>(keep, P);
  uint64_t* dBase = talloc<uint64_t>(keep, P);
  uint32_t* dAct = talloc<uint32_t>(keep, P);
  double* dLam = talloc<double>(keep, static_cast<uint64_t>(P) * s);
  uint8_t* dAs[2] = {talloc<uint8_t>(keep, R * total), talloc<uint8_t>(keep, R * total)};
  double* dBv = talloc<double>(keep, R * total);
  uint32_t* dChg = talloc<uint32_t>(keep, P);
  double* dObj = talloc<double>(keep, P);
  double* dSums = talloc<double>(keep, static_cast<uint64_t>(P) * s * 2);
  // the level sort (s <= 16, when its sorted copies of w and a fit the free memory)
  uint64_t max_n0 = 0;
  for (uint32_t j : secs) max_n0 = std::max<uint64_t>(max_n0, qs[j].quads.size());
  const uint64_t npad = (max_n0 + 15) / 16 * 16;
  const uint32_t nch = static_cast<uint32_t>((max_n0 + kMqChunk - 1) / kMqChunk);
  double2* dSWA = nullptr;
  uint32_t* dLc = nullptr;
  uint64_t *dLbase = nullptr, *dLcnt = nullptr;
  bool lsort = false;
  if (s <= kMqLv && options().train_level_sort) {
    size_t fr = 0, tot = 0;
    PCPQG_CUDA(cudaMemGetInfo(&fr, &tot));
    const uint64_t need = 2ull * P * npad * 8 + static_cast<uint64_t>(P) * nch * kMqLv * 4 + (64ull << 20);
    if (tr.on) std::fprintf(stderr, "[pcpqg train] level sort needs %.1f GB, %.1f GB free\n", need / 1e9, fr / 1e9);
    if (need < fr / 10 * 9) {
      dSWA = talloc<double2>(keep, static_cast<uint64_t>(P) * npad);
      dLc = talloc<uint32_t>(keep, static_cast<uint64_t>(P) * nch * kMqLv);
      dLbase = talloc<uint64_t>(keep, static_cast<uint64_t>(P) * kMqLv);
      dLcnt = talloc<uint64_t>(keep, static_cast<uint64_t>(P) * kMqLv);
      lsort = true;
      PCPQG_CUDA(cudaFuncSetAttribute(mq_lscatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kMqChunk * (sizeof(double2) + 1))));
    }
  }
  PCPQG_CUDA(cudaMemcpy(dW, hw.data(), 8 * total, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dA, ha.data(), 8 * total, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dB, hbq.data(), 8 * total, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dOff, poff.data(), 8ull * P, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dCnt, pcnt.data(), 8ull * P, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dBase, pbase.data(), 8ull * P, cudaMemcpyHostToDevice));
  tr.mark("mq: alloc + H2D");
  uint64_t max_n = 0;
  for (uint32_t j : secs) max_n = std::max<uint64_t>(max_n, qs[j].quads.size());
  std::vector<uint32_t> active(P), final_buf(P, 0);
  for (uint32_t p = 0; p < P; ++p) active[p] = p;
  std::vector<double> obj(P, 0.0), sums(static_cast<uint64_t>(P) * s * 2);
  std::vector<uint32_t> chg(P);
  for (int round = 0; round < 100 && !active.empty(); ++round) {  // kMaxRounds1D
    const uint32_t nact = static_cast<uint32_t>(active.size());
    const int cb = round & 1;
    PCPQG_CUDA(cudaMemcpy(dAct, active.data(), 4ull * nact, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemcpy(dLam, lam.data(), 8ull * P * s, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemset(dChg, 0, 4ull * P));
    const unsigned bx = static_cast<unsigned>(std::min<uint64_t>((max_n + 255) / 256, 64));
    mq_assign_kernel<<<dim3(bx, nact), 256>>>(dW, dA, dB, dOff, dCnt, dBase, dAct, s, dLam, dAs[cb ^ 1], dAs[cb],
                                               round > 0, dChg, dBv);
    const uint64_t nw = static_cast<uint64_t>(nact) * s;
    if (lsort) {
      mq_lcount_kernel<<<dim3(nch, nact), 256>>>(dCnt, dBase, dAct, dAs[cb], nch, dLc);
      mq_loffsets_kernel<<<(nact + 3) / 4, 128>>>(dCnt, dAct, nact, nch, dLc, dLbase, dLcnt);
      constexpr size_t kLsSmem = static_cast<size_t>(kMqChunk) * (sizeof(double2) + 1);
      mq_lscatter_kernel<<<dim3(nch, nact), 256, kLsSmem>>>(dW, dA, dOff, dCnt, dBase, dAct, dAs[cb], nch, dLc,
                                                            dLbase, npad, dSWA);
      mq_lsum_kernel<<<static_cast<unsigned>((nw + kLsWarps - 1) / kLsWarps), 32 * kLsWarps>>>(
          dAct, nact, s, dLbase, dLcnt, npad, dSWA, dSums);
    } else {
      mq_sums_kernel<<<static_cast<unsigned>((nw + kMqWarps - 1) / kMqWarps), 32 * kMqWarps>>>(
          dW, dA, dOff, dCnt, dBase, dAct, nact, s, dAs[cb], dSums);
    }
    PCPQG_CUDA(cudaGetLastError());
    PCPQG_CUDA(cudaMemcpy(chg.data(), dChg, 4ull * P, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(sums.data(), dSums, sums.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> still;
    for (uint32_t p : active) {
      final_buf[p] = static_cast<uint32_t>(cb);
      if (round > 0 && !chg[p]) continue;  // prev == assign: converged, lambda unchanged
      const uint32_t j = secs[p / R];
      const uint64_t n = qs[j].quads.size();
      double* lp = lam.data() + static_cast<uint64_t>(p) * s;
      for (uint32_t l = 0; l < s; ++l) {
        const double sw = sums[(static_cast<uint64_t>(p) * s + l) * 2], sa = sums[(static_cast<uint64_t>(p) * s + l) * 2 + 1];
        if (sw > 0.0)
          lp[l] = -sa / (2.0 * sw);
        else
          lp[l] = minimum_of(j, rngs[p].next_index(n));  // empty group: reseed
      }
      still.push_back(p);
    }
    active.swap(still);
  }
  tr.mark("mq: rounds");
  // every problem's objective: its last round's bv (finished problems are not
  // assigned again, so their bv stays)
  mq_obj_kernel<<<(P + 3) / 4, 128>>>(dCnt, dBase, P, dBv, dObj);
  PCPQG_CUDA(cudaGetLastError());
  PCPQG_CUDA(cudaMemcpy(obj.data(), dObj, 8ull * P, cudaMemcpyDeviceToHost));
  tr.mark("mq: objective");
  // the best restart per section (strict <, earlier restarts win ties)
  for (uint32_t si = 0; si < secs.size(); ++si) {
    const uint32_t j = secs[si];
    uint32_t bp = si * R;
    double best = std::numeric_limits<double>::infinity();
    bool any = false;
    for (uint32_t r = 0; r < R; ++r)
      if (obj[si * R + r] < best) {
        best = obj[si * R + r];
        bp = si * R + r;
        any = true;
      }
    if (!any) continue;  // (the reference keeps an empty codebook: obj never < inf)
    const uint64_t n = qs[j].quads.size();
    std::vector<uint8_t> as(n);
    PCPQG_CUDA(cudaMemcpy(as.data(), dAs[final_buf[bp]] + pbase[bp], n, cudaMemcpyDeviceToHost));
    qs[j].values.assign(lam.begin() + static_cast<uint64_t>(bp) * s, lam.begin() + static_cast<uint64_t>(bp + 1) * s);
    qs[j].assign.assign(as.begin(), as.end());
    canonicalize(qs[j].values, qs[j].assign);
  }
  tr.mark("mq: D2H + canonicalize");
}

}  // namespace

void aniso_weights_host(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot) {
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  const uint64_t chunk = (n + nt - 1) / nt;
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      const uint64_t e = std::min(n, (w + 1) * chunk);
      for (uint64_t i = w * chunk; i < e; ++i) {
        const double nx2 = dot_host(x + i * dbar, x + i * dbar, dbar);
        h_par[i] = h_bot[i] = 0.0;
        if (nx2 > 0.0) aniso_weights_one(std::sqrt(nx2), t, static_cast<int>(dbar), h_par[i], h_bot[i]);
      }
    });
  for (auto& x : th) x.join();
}

namespace {

// One device's share of an aniso / apcpq build: the sections listed in
// `sections` (global ids; sections are independent problems — their own seeds
// Rng::mix(seed, 2j+1) / (seed, 2j+2), weights, Lloyd loop and scale quantizer).
struct AnisoPart {
  std::vector<uint32_t> sections;
  std::vector<float> centers;              // [ml][k][dbar]
  std::vector<uint32_t> codes;             // [ml][n]
  std::vector<double> alphas;              // [ml][n]
  std::vector<std::vector<float>> scb;     // [ml] scale codebooks (quantized)
  std::vector<std::vector<uint8_t>> scodes;  // [ml][n] scale codes (quantized)
  double phases[3] = {0, 0, 0};
  int weights_gpu = 0;
};

void train_aniso_part(const float* X, uint64_t n, uint32_t d, uint32_t dbar, uint32_t k, uint32_t s, bool scaling,
                      bool quant, double t, uint32_t max_iters, double tol, uint64_t seed, int device,
                      AnisoPart& part) {
  using clk = std::chrono::steady_clock;
  auto tick = clk::now();
  auto phase = [&](int i) {
    const auto now = clk::now();
    part.phases[i] = std::chrono::duration<double>(now - tick).count();
    tick = now;
  };
  const std::vector<uint32_t>& gsec = part.sections;
  const uint32_t m = static_cast<uint32_t>(gsec.size());  // sections of this part
  const uint64_t mn = static_cast<uint64_t>(m) * n;
  std::vector<float> secs(mn * dbar, 0.0f);
  std::vector<float>& centers = part.centers;
  centers.assign(static_cast<uint64_t>(m) * k * dbar, 0.0f);
  std::vector<double> hp(mn), hb(mn);
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
        const uint32_t col = gsec[j] * dbar + a;
        sj[i * dbar + a] = col < d ? X[i * d + col] : 0.0f;
      }
    seed_nonzero(sj, n, dbar, k, Rng::mix(seed, 2ull * gsec[j] + 1), false,
                 centers.data() + static_cast<uint64_t>(j) * k * dbar);
  });
  int prev_dev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev_dev));
  PCPQG_CUDA(cudaSetDevice(device));
  struct Restore {
    int dv;
    ~Restore() { cudaSetDevice(dv); }
  } restore{prev_dev};
  // weights once per (section, point); the quantizer's recomputation is identical.
  // On the GPU when its sin reproduces this host's std::sin bits (pcpqg_weights.cu),
  // else on host threads.
  const bool gpu_weights = options().weights_gpu && aniso_weights_gpu_ok(device);
  part.weights_gpu = gpu_weights ? 1 : 0;
  if (!gpu_weights) aniso_weights_host(secs.data(), mn, dbar, t, hp.data(), hb.data());
  std::vector<void*> keep;
  struct Free {
    std::vector<void*>* k;
    ~Free() {
      for (void* p : *k) cudaFree(p);
    }
  } fr{&keep};
  const uint32_t np = dbar * (dbar + 1) / 2, S = np + dbar + 1;
  float* dX = talloc<float>(keep, mn * dbar);
  float* dC = talloc<float>(keep, static_cast<uint64_t>(m) * k * dbar);
  float* dCand = talloc<float>(keep, static_cast<uint64_t>(m) * k * dbar);
  double* dHp = talloc<double>(keep, mn);
  double* dHb = talloc<double>(keep, mn);
  uint32_t* dA = talloc<uint32_t>(keep, mn);
  uint32_t* dPrev = talloc<uint32_t>(keep, mn);
  double* dAl = talloc<double>(keep, mn);
  double* dL = talloc<double>(keep, mn);
  uint32_t* dCnt = talloc<uint32_t>(keep, static_cast<uint64_t>(m) * k);
  uint64_t* dOff = talloc<uint64_t>(keep, static_cast<uint64_t>(m) * k);
  uint32_t* dIdx = talloc<uint32_t>(keep, mn);
  uint32_t* dMem = talloc<uint32_t>(keep, mn);
  uint32_t* dSA = talloc<uint32_t>(keep, mn);
  double* dLo = talloc<double>(keep, mn);
  double* dLn = talloc<double>(keep, mn);
  double* dStats = talloc<double>(keep, static_cast<uint64_t>(m) * k * S);
  double* dCL = talloc<double>(keep, static_cast<uint64_t>(m) * k * 2);
  double* dLoss = talloc<double>(keep, m);
  uint32_t* dAct = talloc<uint32_t>(keep, m);
  int* dSeg = talloc<int>(keep, m + 1);
  PCPQG_CUDA(cudaMemcpy(dX, secs.data(), 4 * mn * dbar, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMemcpy(dC, centers.data(), centers.size() * 4, cudaMemcpyHostToDevice));
  if (gpu_weights) {
    launch_aniso_weights(dX, mn, dbar, t, dHp, dHb, nullptr);
    PCPQG_CUDA(cudaMemcpy(hp.data(), dHp, 8 * mn, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(hb.data(), dHb, 8 * mn, cudaMemcpyDeviceToHost));
  } else {
    PCPQG_CUDA(cudaMemcpy(dHp, hp.data(), 8 * mn, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemcpy(dHb, hb.data(), 8 * mn, cudaMemcpyHostToDevice));
  }
  std::vector<uint32_t> live;  // sections with a nonzero weight (else model.degenerate)
  for (uint32_t j = 0; j < m; ++j) {
    bool any = false;
    for (uint64_t i = 0; i < n && !any; ++i)
      any = hp[static_cast<uint64_t>(j) * n + i] > 0.0 || hb[static_cast<uint64_t>(j) * n + i] > 0.0;
    if (any) live.push_back(j);
  }
  phase(0);
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

  // A1 for the listed sections (+ counts), then reseed_empty_clusters on the host
  auto assign = [&](const std::vector<uint32_t>& act, bool first) {
    for (uint32_t sj : act) {
      const uint64_t o = static_cast<uint64_t>(sj) * n;
      if (!first) PCPQG_CUDA(cudaMemcpyAsync(dPrev + o, dA + o, 4 * n, cudaMemcpyDeviceToDevice));
      launch_assign_anisotropic(dX + o * dbar, n, dbar, dC + static_cast<uint64_t>(sj) * k * dbar, k, dHp + o,
                                dHb + o, first ? nullptr : dPrev + o, dA + o, dAl + o, dL + o, 0, scaling);
      PCPQG_CUDA(cudaMemsetAsync(dCnt + static_cast<uint64_t>(sj) * k, 0, 4ull * k));
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
      const uint64_t o = static_cast<uint64_t>(sj) * n;
      std::vector<uint32_t> as(n);
      std::vector<double> pl(n), al(n);
      float* cs = centers.data() + static_cast<uint64_t>(sj) * k * dbar;
      PCPQG_CUDA(cudaMemcpy(as.data(), dA + o, 4 * n, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(pl.data(), dL + o, 8 * n, cudaMemcpyDeviceToHost));
      PCPQG_CUDA(cudaMemcpy(al.data(), dAl + o, 8 * n, cudaMemcpyDeviceToHost));
      // reseed_empty_clusters (clustering.cpp:156-185): moved points get scale 1
      std::vector<uint64_t> counts(k, 0);
      for (uint64_t i = 0; i < n; ++i) ++counts[as[i]];
      const float* xs = secs.data() + o * dbar;
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
      PCPQG_CUDA(cudaMemcpy(dA + o, as.data(), 4 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dL + o, pl.data(), 8 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dAl + o, al.data(), 8 * n, cudaMemcpyHostToDevice));
      PCPQG_CUDA(cudaMemcpy(dCnt + static_cast<uint64_t>(sj) * k, c2.data(), 4ull * k, cudaMemcpyHostToDevice));
    }
  };

  std::vector<uint32_t> active = live;
  std::vector<std::vector<double>> trace(m);
  for (uint32_t iter = 0; iter < max_iters && !active.empty(); ++iter) {
    assign(active, iter == 0);
    const uint32_t nact = static_cast<uint32_t>(active.size());
    // A2 member lists (all sections; inactive ones are left as they were)
    km_iota_kernel<<<static_cast<unsigned>((mn + 255) / 256), 256>>>(dIdx, n, m);
    PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(dTmp, tmp_bytes, dA, dSA, dIdx, dMem, static_cast<int>(mn),
                                                        static_cast<int>(m), dSeg, dSeg + 1, 0, kbits));
    km_offsets_kernel<<<(m + 127) / 128, 128>>>(dCnt, m, k, dOff);
    // A3 center statistics, all sections in one batched call (the inactive
    // sections' results are not read)
    launch_center_stats(dX, n, dbar, m, n * dbar, dA, dAl, dHp, dHb, k, nullptr, dStats, 0);
    std::vector<double> st(static_cast<uint64_t>(m) * k * S);
    std::vector<uint32_t> cnt(static_cast<uint64_t>(m) * k);
    PCPQG_CUDA(cudaMemcpy(st.data(), dStats, st.size() * 8, cudaMemcpyDeviceToHost));
    PCPQG_CUDA(cudaMemcpy(cnt.data(), dCnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    // center_anisotropic per non-empty cluster: the ridge-regularised d̄ x d̄
    // Cholesky solve, rounded to float; a singular system or a zero candidate
    // keeps the previous center (clustering.cpp:686-697)
    std::vector<float> cand(centers);
    std::vector<uint8_t> solved(static_cast<uint64_t>(m) * k, 0);
    for (uint32_t sj : active)
      for (uint32_t c = 0; c < k; ++c) {
        const uint64_t sc = static_cast<uint64_t>(sj) * k + c;
        if (cnt[sc] == 0) continue;
        const double* sv = st.data() + sc * S;
        std::vector<double> M(dbar * dbar, 0.0), rhs(dbar), sol(dbar);
        uint32_t q = 0;
        for (uint32_t a = 0; a < dbar; ++a)
          for (uint32_t b = a; b < dbar; ++b) M[a * dbar + b] = sv[q++];
        for (uint32_t a = 0; a < dbar; ++a) rhs[a] = sv[np + a];
        const double diag = sv[np + dbar];
        for (uint32_t a = 0; a < dbar; ++a) {
          M[a * dbar + a] += diag;
          for (uint32_t b = 0; b < a; ++b) M[a * dbar + b] = M[b * dbar + a];
        }
        double tr = 0.0;
        for (uint32_t a = 0; a < dbar; ++a) tr += M[a * dbar + a];
        if (!solve_spd_host(M, rhs.data(), dbar, 1e-9 * tr / static_cast<double>(dbar), sol.data())) continue;
        float* out = cand.data() + sc * dbar;
        for (uint32_t a = 0; a < dbar; ++a) out[a] = static_cast<float>(sol[a]);
        if (dot_host(out, out, dbar) == 0.0) {
          std::memcpy(out, centers.data() + sc * dbar, 4ull * dbar);
          continue;
        }
        solved[sc] = 1;
      }
    PCPQG_CUDA(cudaMemcpy(dCand, cand.data(), cand.size() * 4, cudaMemcpyHostToDevice));
    PCPQG_CUDA(cudaMemcpy(dAct, active.data(), 4 * active.size(), cudaMemcpyHostToDevice));
    dim3 g2(static_cast<unsigned>((n + 255) / 256), nact);
    ta_cluster_terms_kernel<<<g2, 256>>>(dX, n, dbar, k, dAct, dMem, dSA, dC, dCand, dHp, dHb, dAl, dLo, dLn);
    const uint64_t nl = static_cast<uint64_t>(nact) * k * 2;
    tp_loss_chain_kernel<<<static_cast<unsigned>((nl + 127) / 128), 128>>>(dLo, dLn, n, k, dAct, nact, dCnt, dOff,
                                                                          dCL);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<double> CL(static_cast<uint64_t>(m) * k * 2);
    PCPQG_CUDA(cudaMemcpy(CL.data(), dCL, CL.size() * 8, cudaMemcpyDeviceToHost));
    for (uint32_t sj : active)
      for (uint32_t c = 0; c < k; ++c) {
        const uint64_t sc = static_cast<uint64_t>(sj) * k + c;
        if (solved[sc] && CL[sc * 2 + 1] < CL[sc * 2])
          std::memcpy(centers.data() + sc * dbar, cand.data() + sc * dbar, 4ull * dbar);
      }
    PCPQG_CUDA(cudaMemcpy(dC, centers.data(), centers.size() * 4, cudaMemcpyHostToDevice));
    // A5 scale refresh + the id-order loss chain
    ta_refresh_kernel<<<g2, 256>>>(dX, n, dbar, k, dAct, dA, dC, dHp, dHb, scaling, dAl, dLo);
    km_loss_kernel<<<(nact + 3) / 4, 128>>>(dLo, n, dAct, nact, dLoss);
    PCPQG_CUDA(cudaGetLastError());
    std::vector<double> loss(m);
    PCPQG_CUDA(cudaMemcpy(loss.data(), dLoss, 8ull * m, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> still;
    for (uint32_t sj : active) {
      auto& tr = trace[sj];
      tr.push_back(loss[sj]);
      bool conv = false;
      if (tr.size() >= 2) {
        const double p = tr[tr.size() - 2], c = tr.back();
        conv = std::fabs(p - c) <= tol * std::max(std::fabs(p), 1e-300);
      }
      if (!conv) still.push_back(sj);
    }
    active.swap(still);
  }
  // the final assignment against the trained centers, keep-previous on
  if (!live.empty()) assign(live, false);
  std::vector<uint32_t>& codes = part.codes;
  std::vector<double>& alphas = part.alphas;
  codes.assign(mn, 0);
  alphas.assign(mn, 1.0);
  PCPQG_CUDA(cudaMemcpy(centers.data(), dC, centers.size() * 4, cudaMemcpyDeviceToHost));
  for (uint32_t sj : live) {
    const uint64_t o = static_cast<uint64_t>(sj) * n;
    PCPQG_CUDA(cudaMemcpy(codes.data() + o, dA + o, 4 * n, cudaMemcpyDeviceToHost));
    if (scaling) PCPQG_CUDA(cudaMemcpy(alphas.data() + o, dAl + o, 8 * n, cudaMemcpyDeviceToHost));
  }

  phase(1);
  // scales: {1} for aniso, raw alphas, or quantize_anisotropic with
  // scale_seed = Rng::mix(seed, 2j + 2)
  std::vector<std::vector<float>>& scb = part.scb;
  std::vector<std::vector<uint8_t>>& scodes = part.scodes;
  scb.assign(m, {});
  scodes.assign(m, {});
  if (quant) {
    TrainTrace tr;
    std::vector<QuantSection> qs(m);
    std::vector<uint64_t> sseeds(m);
    par_sections([&](uint32_t j) {
      const uint64_t o = static_cast<uint64_t>(j) * n;
      build_quads(secs.data() + o * dbar, n, dbar, centers.data() + static_cast<uint64_t>(j) * k * dbar, k,
                  codes.data() + o, hp.data() + o, hb.data() + o, qs[j]);
      sseeds[j] = Rng::mix(seed, 2ull * gsec[j] + 2);
    });
    tr.mark("scales: build_quads");
    minimize_quadratic_scalars_gpu(qs, s, sseeds);
    tr.t = std::chrono::steady_clock::now();
    par_sections([&](uint32_t j) { finish_quantize(qs[j], n, s, scb[j], scodes[j]); });
    tr.mark("scales: finish_quantize");
  }

  phase(2);
}

}  // namespace

std::vector<uint8_t> train_aniso(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                 bool scaling, bool quantize, double t_frac, uint32_t max_iters, double tol,
                                 uint64_t seed, const int* devices, int ndev) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  for (double& v : g_train_phases) v = 0.0;
  if (!devices || ndev < 1) fail(PCPQG_E_USAGE, "train_aniso: need at least one device");
  const double t = validate_train(X, n, d, m, k, s, t_frac, max_iters, tol, true);
  const bool quant = scaling && quantize;
  const uint32_t scales = !scaling ? 1 : (quant ? s : 0);  // effective_scales (pq_index.cpp:35-38)
  if (quant && s > 256) fail(PCPQG_E_DATA, "scalar quantization: need 1 <= s <= 256");
  const uint32_t padded_d = ((d + m - 1) / m) * m, dbar = padded_d / m;
  // sections are dealt round-robin to the devices; each device thread trains its
  // sections end to end, so nothing is exchanged until the image is assembled
  const uint32_t np = std::min<uint32_t>(static_cast<uint32_t>(ndev), m);
  std::vector<AnisoPart> parts(np);
  for (uint32_t j = 0; j < m; ++j) parts[j % np].sections.push_back(j);
  const double prep0 = std::chrono::duration<double>(clk::now() - t0).count();
  std::vector<std::exception_ptr> errs(np);
  {
    std::vector<std::thread> th;
    for (uint32_t g = 0; g < np; ++g)
      th.emplace_back([&, g] {
        try {
          train_aniso_part(X, n, d, dbar, k, s, scaling, quant, t, max_iters, tol, seed, devices[g], parts[g]);
        } catch (...) {
          errs[g] = std::current_exception();
        }
      });
    for (auto& x : th) x.join();
  }
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  g_train_weights_gpu = 1;
  for (const AnisoPart& p : parts) {
    for (int i = 0; i < 3; ++i) g_train_phases[i] = std::max(g_train_phases[i], p.phases[i]);
    g_train_weights_gpu &= p.weights_gpu;
  }
  g_train_phases[0] += prep0;
  const auto t1 = clk::now();
  // where section j lives: (part, local index)
  std::vector<const AnisoPart*> owner(m);
  std::vector<uint32_t> local(m);
  for (const AnisoPart& p : parts)
    for (uint32_t jl = 0; jl < p.sections.size(); ++jl) {
      owner[p.sections[jl]] = &p;
      local[p.sections[jl]] = jl;
    }
  // serialize (pq_index.cpp:372-407): method 1 (aniso) or 3 (apcpq)
  const bool wide = k > 256;
  const uint64_t cbytes = static_cast<uint64_t>(m) * (wide ? 2 : 1);
  const uint64_t row = cbytes + (scales == 0 ? 4ull * m : m);
  const uint64_t cb_floats = static_cast<uint64_t>(k) * dbar;
  std::vector<uint8_t> out;
  out.reserve(48 + 4ull * m * cb_floats + 4ull * m * scales + n * row);
  auto u32 = [&](uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  };
  const char magic[8] = {'P', 'C', 'P', 'Q', 'I', 'D', 'X', '1'};
  out.insert(out.end(), magic, magic + 8);
  u32(1);
  u32(scaling ? 3 : 1);
  u32(static_cast<uint32_t>(n));
  u32(d);
  u32(padded_d);
  u32(m);
  u32(k);
  u32(scales);
  uint64_t tb;
  std::memcpy(&tb, &t, 8);
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<uint8_t>(tb >> (8 * i)));
  size_t at = 0;
  for (uint32_t j = 0; j < m; ++j) {
    at = out.size();
    out.resize(at + cb_floats * 4);
    std::memcpy(out.data() + at, owner[j]->centers.data() + local[j] * cb_floats, cb_floats * 4);
  }
  for (uint32_t j = 0; j < m && scales >= 1; ++j) {
    at = out.size();
    out.resize(at + 4ull * scales);
    if (quant) {
      std::memcpy(out.data() + at, owner[j]->scb[local[j]].data(), 4ull * s);
    } else {
      const float one = 1.0f;
      std::memcpy(out.data() + at, &one, 4);
    }
  }
  at = out.size();
  out.resize(at + n * row, 0);
  // rows are written by host threads over point ranges
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const uint64_t chunk = (n + nt - 1) / nt;
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      const uint64_t e = std::min(n, (w + 1) * chunk);
      for (uint64_t i = w * chunk; i < e; ++i) {
        uint8_t* r = out.data() + at + i * row;
        for (uint32_t j = 0; j < m; ++j) {
          const AnisoPart& p = *owner[j];
          const uint64_t o = static_cast<uint64_t>(local[j]) * n + i;
          const uint32_t c = p.codes[o];
          if (wide) {
            r[2 * j] = static_cast<uint8_t>(c);
            r[2 * j + 1] = static_cast<uint8_t>(c >> 8);
          } else {
            r[j] = static_cast<uint8_t>(c);
          }
          if (quant) {
            r[cbytes + j] = p.scodes[local[j]][i];
          } else if (scales == 0) {
            const float a = static_cast<float>(p.alphas[o]);
            std::memcpy(r + cbytes + 4ull * j, &a, 4);
          }  // aniso: scale codes stay 0
        }
      }
    });
  for (auto& x : th) x.join();
  g_train_phases[3] = std::chrono::duration<double>(clk::now() - t1).count();
  return out;
}

}  // namespace pcpqg
