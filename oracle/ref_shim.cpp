// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (pcpq, compiled
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libpcpq_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's reference / cpu_baseline legs load it, and only as the checker
// or as the timed reference CPU arm.
//
// Entry points mirror the reference calls they wrap:
//   ref_build_index     -> pcpq::build_pq_index + pcpq::serialize
//                          (proj/core/src/pq_index.cpp:62-168, :372-407)
//   ref_index_open      -> pcpq::deserialize (pq_index.cpp:409-488)
//   ref_build_lut       -> pcpq::build_lookup_table (pq_index.cpp:170-210)
//   ref_score_query     -> pcpq::score_query (pq_index.cpp:246-250)
//   ref_search          -> the flat query loop of proj/tools/main.cpp:229-243
//                          (score_query + iota + partial_sort by (score desc,
//                          id asc)), optionally spread over a std::thread pool
//                          (harness-level; the functions are reentrant).
//   ref_assign_*        -> pcpq::assign_projective / assign_anisotropic
//                          (proj/core/src/clustering.cpp:250-368)
//   ref_aniso_weights   -> pcpq::aniso_weights (clustering.cpp:204-217)
//   ref_generate_dataset-> pcpq::generate_dataset (datagen.cpp:70-89)
//   ref_brute_force_topn-> pcpq::brute_force_topn per query (eval.cpp:36-49)
//   ref_recall1         -> pcpq::recall1_single per query (eval.cpp:57-66)
//   ref_build_ivf       -> pcpq::build_ivf + serialize (proj/core/src/ivf.cpp:46-87, :229-255)
//   ref_ivf_query       -> pcpq::deserialize_ivf + query_ivf per query
//                          (ivf.cpp:256-316, :89-153)
// Status codes: 0 ok, errc+1 on pcpq::error, 99 on any other exception.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "pcpq/clustering.hpp"
#include "pcpq/datagen.hpp"
#include "pcpq/eval.hpp"
#include "pcpq/ivf.hpp"
#include "pcpq/pq_index.hpp"
#include "pcpq/scalar_quant.hpp"
#include "pcpq/types.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const pcpq::error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

void fill_counters(const pcpq::ScoreCounters& c, std::uint64_t* out) {
  if (!out) return;
  out[0] = c.table_madds;
  out[1] = c.scalar_mults;
  out[2] = c.point_mults;
  out[3] = c.lookups;
  out[4] = c.adds;
}

pcpq::MatrixF to_matrix(const float* x, std::uint64_t rows, std::uint32_t cols) {
  pcpq::MatrixF m(rows, cols);
  std::memcpy(m.data.data(), x, sizeof(float) * rows * cols);
  return m;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

int ref_build_index(const float* data, std::uint64_t n, std::uint32_t d, int method,
                    int quantize, std::uint32_t m, std::uint32_t k, std::uint32_t s,
                    double t_frac, std::uint32_t max_iters, double tol, std::uint64_t seed,
                    std::uint8_t** out, std::uint64_t* out_len) {
  return guarded([&] {
    pcpq::PQConfig cfg;
    cfg.method = static_cast<pcpq::Method>(method);
    cfg.quantize_scalars = quantize != 0;
    cfg.m = m;
    cfg.k = k;
    cfg.s = s;
    cfg.t_frac = t_frac;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.seed = seed;
    const pcpq::PQIndex idx = pcpq::build_pq_index(to_matrix(data, n, d), cfg);
    const std::vector<std::uint8_t> bytes = pcpq::serialize(idx);
    *out = static_cast<std::uint8_t*>(std::malloc(bytes.size()));
    std::memcpy(*out, bytes.data(), bytes.size());
    *out_len = bytes.size();
  });
}

void* ref_index_open(const std::uint8_t* bytes, std::uint64_t len, int* status) {
  pcpq::PQIndex* h = nullptr;
  *status = guarded([&] {
    h = new pcpq::PQIndex(pcpq::deserialize(std::span<const std::uint8_t>(bytes, len)));
  });
  return h;
}

void ref_index_close(void* h) { delete static_cast<pcpq::PQIndex*>(h); }

int ref_index_shape(void* h, std::uint64_t* out6) {
  return guarded([&] {
    const auto& idx = *static_cast<pcpq::PQIndex*>(h);
    out6[0] = idx.n();
    out6[1] = idx.config.d;
    out6[2] = idx.m();
    out6[3] = idx.k();
    out6[4] = idx.scales;
    out6[5] = idx.config.padded_d;
  });
}

int ref_serialize(void* h, std::uint8_t** out, std::uint64_t* out_len) {
  return guarded([&] {
    const auto bytes = pcpq::serialize(*static_cast<pcpq::PQIndex*>(h));
    *out = static_cast<std::uint8_t*>(std::malloc(bytes.size()));
    std::memcpy(*out, bytes.data(), bytes.size());
    *out_len = bytes.size();
  });
}

int ref_build_lut(void* h, const float* q, std::uint32_t d, float* eta, float* etal,
                  std::uint64_t* counters) {
  return guarded([&] {
    pcpq::ScoreCounters c;
    const auto lut = pcpq::build_lookup_table(*static_cast<pcpq::PQIndex*>(h),
                                              std::span<const float>(q, d), &c);
    std::memcpy(eta, lut.eta.data(), sizeof(float) * lut.eta.size());
    if (etal && !lut.eta_lambda.empty())
      std::memcpy(etal, lut.eta_lambda.data(), sizeof(float) * lut.eta_lambda.size());
    fill_counters(c, counters);
  });
}

int ref_score_query(void* h, const float* q, std::uint32_t d, float* scores,
                    std::uint64_t* counters) {
  return guarded([&] {
    pcpq::ScoreCounters c;
    const auto s = pcpq::score_query(*static_cast<pcpq::PQIndex*>(h),
                                     std::span<const float>(q, d), &c);
    std::memcpy(scores, s.data(), sizeof(float) * s.size());
    fill_counters(c, counters);
  });
}

// The flat-index query loop of proj/tools/main.cpp:229-243, per query:
// score_query, iota, partial_sort(topn) by (score desc, id asc).  `threads`
// > 1 spreads queries over a std::thread pool (one query per task).
int ref_search(void* h, const float* Q, std::uint64_t B, std::uint32_t d, std::uint32_t topn_req,
               int threads, std::int32_t* ids, float* out_scores) {
  return guarded([&] {
    const auto& index = *static_cast<pcpq::PQIndex*>(h);
    if (d != index.config.d) pcpq::fail(pcpq::errc::data, "query dimension does not match index");
    const std::uint32_t topn = std::min<std::uint32_t>(topn_req, index.n());
    std::atomic<std::uint64_t> next{0};
    std::string first_err;
    std::atomic<int> err_code{0};
    auto worker = [&] {
      std::vector<std::uint32_t> order(index.n());
      for (;;) {
        const std::uint64_t qi = next.fetch_add(1);
        if (qi >= B || err_code.load()) return;
        const int st = guarded([&] {
          const std::vector<float> scores =
              pcpq::score_query(index, std::span<const float>(Q + qi * d, d));
          std::iota(order.begin(), order.end(), 0u);
          std::partial_sort(order.begin(), order.begin() + topn, order.end(),
                            [&](std::uint32_t x, std::uint32_t y) {
                              if (scores[x] != scores[y]) return scores[x] > scores[y];
                              return x < y;
                            });
          for (std::uint32_t i = 0; i < topn; ++i) {
            ids[qi * topn_req + i] = static_cast<std::int32_t>(order[i]);
            if (out_scores) out_scores[qi * topn_req + i] = scores[order[i]];
          }
          for (std::uint32_t i = topn; i < topn_req; ++i) {
            ids[qi * topn_req + i] = -1;
            if (out_scores) out_scores[qi * topn_req + i] = -__builtin_inff();
          }
        });
        if (st) err_code.store(st);
      }
    };
    const int nt = std::max(1, threads);
    if (nt == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    if (err_code.load()) pcpq::fail(static_cast<pcpq::errc>(err_code.load() - 1), g_err);
  });
}

std::uint64_t ref_logical_payload_bits(std::uint64_t n, std::uint32_t m, std::uint32_t k,
                                       std::uint32_t scales) {
  return pcpq::logical_payload_bits(n, m, k, scales);
}

int ref_generate_dataset(int dist, std::uint64_t n, std::uint32_t d, std::uint64_t seed,
                         float* out) {
  return guarded([&] {
    const auto x = pcpq::generate_dataset(static_cast<pcpq::Dist>(dist), n, d, seed);
    std::memcpy(out, x.data.data(), sizeof(float) * x.data.size());
  });
}

int ref_aniso_weights(double norm_x, double t, int dbar, double* h_par, double* h_bot) {
  return guarded([&] {
    const auto w = pcpq::aniso_weights(norm_x, t, dbar);
    *h_par = w.h_par;
    *h_bot = w.h_bot;
  });
}

int ref_assign_projective(const float* x, std::uint64_t n, std::uint32_t dbar,
                          const float* centers, std::uint32_t k, std::uint32_t* assign,
                          double* alphas, double* point_loss) {
  return guarded([&] {
    const auto r = pcpq::assign_projective(to_matrix(x, n, dbar), to_matrix(centers, k, dbar));
    std::copy(r.assignment.begin(), r.assignment.end(), assign);
    std::copy(r.alphas.begin(), r.alphas.end(), alphas);
    if (point_loss) std::copy(r.point_loss.begin(), r.point_loss.end(), point_loss);
  });
}

int ref_assign_anisotropic(const float* x, std::uint64_t n, std::uint32_t dbar,
                           const float* centers, std::uint32_t k, const double* h_par,
                           const double* h_bot, int allow_scaling, std::uint32_t* assign,
                           double* alphas, double* point_loss) {
  return guarded([&] {
    std::vector<pcpq::AnisoWeights> w(n);
    for (std::uint64_t i = 0; i < n; ++i) w[i] = {h_par[i], h_bot[i]};
    const auto r = pcpq::assign_anisotropic(to_matrix(x, n, dbar), to_matrix(centers, k, dbar),
                                            w, allow_scaling != 0);
    std::copy(r.assignment.begin(), r.assignment.end(), assign);
    std::copy(r.alphas.begin(), r.alphas.end(), alphas);
    if (point_loss) std::copy(r.point_loss.begin(), r.point_loss.end(), point_loss);
  });
}

// pcpq::center_anisotropic (proj/core/src/clustering.cpp:382-410) over the
// member rows x[members[i]] in the given order.
int ref_center_anisotropic(const float* x, std::uint32_t dbar, const std::uint32_t* members,
                           std::uint64_t cnt, const double* alpha, const double* h_par,
                           const double* h_bot, double* center) {
  return guarded([&] {
    std::vector<const float*> rows(cnt);
    std::vector<double> al(cnt);
    std::vector<pcpq::AnisoWeights> w(cnt);
    for (std::uint64_t i = 0; i < cnt; ++i) {
      rows[i] = x + static_cast<std::uint64_t>(members[i]) * dbar;
      al[i] = alpha[members[i]];
      w[i] = {h_par[members[i]], h_bot[members[i]]};
    }
    const auto c = pcpq::center_anisotropic(rows, dbar, al, w);
    std::copy(c.begin(), c.end(), center);
  });
}

// pcpq::quantize_anisotropic (proj/core/src/scalar_quant.cpp:72-152): fitted
// codebook (s floats) and the per-point codes.
int ref_quantize_anisotropic(const float* x, std::uint64_t n, std::uint32_t dbar,
                             const float* centers, std::uint32_t k, const std::uint32_t* assign,
                             const double* h_par, const double* h_bot, std::uint32_t s,
                             std::uint64_t seed, float* values, std::uint8_t* codes) {
  return guarded([&] {
    std::vector<pcpq::AnisoWeights> w(n);
    for (std::uint64_t i = 0; i < n; ++i) w[i] = {h_par[i], h_bot[i]};
    const std::vector<std::uint32_t> a(assign, assign + n);
    const auto q = pcpq::quantize_anisotropic(to_matrix(x, n, dbar), to_matrix(centers, k, dbar),
                                              a, w, s, seed);
    std::copy(q.values.begin(), q.values.end(), values);
    std::copy(q.codes.begin(), q.codes.end(), codes);
  });
}


int ref_build_ivf(const float* data, std::uint64_t n, std::uint32_t d, std::uint32_t kbar,
                  int method, int quantize, std::uint32_t m, std::uint32_t k, std::uint32_t s,
                  std::uint32_t max_iters, std::uint64_t seed, std::uint8_t** out,
                  std::uint64_t* out_len) {
  return guarded([&] {
    pcpq::PQConfig cfg;
    cfg.method = static_cast<pcpq::Method>(method);
    cfg.quantize_scalars = quantize != 0;
    cfg.m = m;
    cfg.k = k;
    cfg.s = s;
    cfg.max_iters = max_iters;
    cfg.seed = seed;
    const pcpq::IVFIndex idx = pcpq::build_ivf(to_matrix(data, n, d), kbar, cfg, seed);
    const std::vector<std::uint8_t> bytes = pcpq::serialize(idx);
    *out = static_cast<std::uint8_t*>(std::malloc(bytes.size()));
    std::memcpy(*out, bytes.data(), bytes.size());
    *out_len = bytes.size();
  });
}

// One query_ivf per query row.  ids/scores: B x topn (id -1 / NaN past the
// returned length), counts[b] = returned length, short_flags[b], requested
// scores B x R (R requested ids per query, row-major), counters5 summed.
int ref_ivf_query(const std::uint8_t* bytes, std::uint64_t len, const float* Q, std::uint64_t B,
                  std::uint32_t d, std::uint32_t k_probe, std::uint32_t topn,
                  const std::uint32_t* requested, std::uint32_t R, std::int32_t* ids,
                  double* scores, std::uint32_t* counts, std::uint8_t* short_flags,
                  double* req_scores, std::uint64_t* counters5) {
  return guarded([&] {
    const pcpq::IVFIndex idx = pcpq::deserialize_ivf({bytes, static_cast<std::size_t>(len)});
    pcpq::ScoreCounters c;
    for (std::uint64_t b = 0; b < B; ++b) {
      std::span<const std::uint32_t> req;
      if (R) req = {requested + b * R, R};
      const auto res = pcpq::query_ivf(idx, {Q + b * d, d}, k_probe, topn, req, &c);
      for (std::uint32_t i = 0; i < topn; ++i) {
        ids[b * topn + i] = i < res.top.size() ? static_cast<std::int32_t>(res.top[i].id) : -1;
        scores[b * topn + i] =
            i < res.top.size() ? res.top[i].score : std::numeric_limits<double>::quiet_NaN();
      }
      counts[b] = static_cast<std::uint32_t>(res.top.size());
      short_flags[b] = res.short_result ? 1 : 0;
      for (std::uint32_t i = 0; i < R; ++i) req_scores[b * R + i] = res.requested[i];
    }
    fill_counters(c, counters5);
  });
}

// deserialize_ivf alone (status = errc + 1), for the container error classes
int ref_ivf_validate(const std::uint8_t* bytes, std::uint64_t len) {
  return guarded([&] { (void)pcpq::deserialize_ivf({bytes, static_cast<std::size_t>(len)}); });
}

// Handle-based IVF for timing: deserialize once, then query_ivf per query row
// spread over a std::thread pool (the reference call is reentrant).
void* ref_ivf_open(const std::uint8_t* bytes, std::uint64_t len, int* status) {
  pcpq::IVFIndex* out = nullptr;
  *status = guarded([&] {
    out = new pcpq::IVFIndex(pcpq::deserialize_ivf({bytes, static_cast<std::size_t>(len)}));
  });
  return out;
}

void ref_ivf_close(void* h) { delete static_cast<pcpq::IVFIndex*>(h); }

int ref_ivf_query_h(void* h, const float* Q, std::uint64_t B, std::uint32_t d, std::uint32_t k_probe,
                    std::uint32_t topn, int threads, std::int32_t* ids, double* scores) {
  return guarded([&] {
    const auto& idx = *static_cast<pcpq::IVFIndex*>(h);
    std::atomic<std::uint64_t> next{0};
    std::atomic<int> err_code{0};
    auto worker = [&] {
      for (;;) {
        const std::uint64_t qi = next.fetch_add(1);
        if (qi >= B || err_code.load()) return;
        const int st = guarded([&] {
          const auto res = pcpq::query_ivf(idx, {Q + qi * d, d}, k_probe, topn);
          for (std::uint32_t i = 0; i < topn; ++i) {
            ids[qi * topn + i] = i < res.top.size() ? static_cast<std::int32_t>(res.top[i].id) : -1;
            scores[qi * topn + i] =
                i < res.top.size() ? res.top[i].score : std::numeric_limits<double>::quiet_NaN();
          }
        });
        if (st) err_code.store(st);
      }
    };
    const int nt = std::max(1, threads);
    if (nt == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    if (err_code.load()) pcpq::fail(static_cast<pcpq::errc>(err_code.load() - 1), g_err);
  });
}

int ref_brute_force_topn(const float* X, std::uint64_t n, std::uint32_t d, const float* Q,
                         std::uint64_t B, std::uint32_t topn, int threads, std::int32_t* ids,
                         double* scores) {
  return guarded([&] {
    const pcpq::MatrixF data = to_matrix(X, n, d);
    std::atomic<std::uint64_t> next{0};
    std::atomic<int> err_code{0};
    auto worker = [&] {
      for (;;) {
        const std::uint64_t b = next.fetch_add(1);
        if (b >= B || err_code.load()) return;
        const int st = guarded([&] {
          const auto top = pcpq::brute_force_topn(data, {Q + b * d, d}, topn);
          for (std::uint32_t i = 0; i < topn; ++i) {
            ids[b * topn + i] = static_cast<std::int32_t>(top[i].id);
            scores[b * topn + i] = top[i].score;
          }
        });
        if (st) err_code.store(st);
      }
    };
    const int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    if (err_code.load()) pcpq::fail(static_cast<pcpq::errc>(err_code.load() - 1), g_err);
  });
}

int ref_recall1(const float* X, std::uint64_t n, std::uint32_t d, const float* Q, std::uint64_t B,
                const std::uint32_t* retrieved, std::uint32_t R, const double* exact_top1,
                std::int32_t* hits) {
  return guarded([&] {
    const pcpq::MatrixF data = to_matrix(X, n, d);
    for (std::uint64_t b = 0; b < B; ++b)
      hits[b] = pcpq::recall1_single(data, {Q + b * d, d}, {retrieved + b * R, R}, exact_top1[b]);
  });
}
}  // extern "C"
