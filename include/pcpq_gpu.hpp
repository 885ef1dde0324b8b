// Header-only C++ drop-in over libpcpqg.so for code written against the
// reference scoring API (namespace pcpq, proj/core/include/pcpq/pq_index.hpp).
//
//   reference (CPU)                              this shim (B200)
//   pcpq::read_pq_index(path)                    pcpq::gpu::read_pq_index(path, device)
//   pcpq::deserialize(bytes)                     pcpq::gpu::deserialize(bytes, device)
//   pcpq::build_lookup_table(index, q, counters) pcpq::gpu::build_lookup_table(...)
//   pcpq::score_all(index, lut, counters)        pcpq::gpu::score_all(...)
//   pcpq::score_query(index, q, counters)        pcpq::gpu::score_query(...)
//   the CLI's flat top-n (tools/main.cpp:229-243) pcpq::gpu::search(index, Q, B, topn)
//
// Same argument meaning and results (bit-identical scores, identical top-n
// with the (score desc, id asc) tie rule); errors are thrown as
// pcpq::gpu::error carrying the reference errc (types.hpp:14-34).
#pragma once

#include <cstdint>
#include <filesystem>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pcpqg.h"

namespace pcpq::gpu {

enum class errc {
  usage, data, numeric, bad_magic, bad_version, truncated, code_out_of_range, size_mismatch,
  cuda = 99, unsupported = 100
};

class error : public std::runtime_error {
 public:
  error(int status, const std::string& what)
      : std::runtime_error(what),
        code_(status >= 1 && status <= 8 ? static_cast<errc>(status - 1)
                                         : (status == PCPQG_E_CUDA ? errc::cuda : errc::unsupported)) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

inline void check(int status) {
  if (status != PCPQG_OK) throw error(status, pcpqg_last_error());
}

struct ScoreCounters {  // pcpq::ScoreCounters (pq_index.hpp:49-55)
  std::uint64_t table_madds = 0, scalar_mults = 0, point_mults = 0, lookups = 0, adds = 0;
  std::uint64_t* raw() { return &table_madds; }
};
static_assert(sizeof(ScoreCounters) == 5 * sizeof(std::uint64_t));

struct LookupTable {  // pcpq::LookupTable (pq_index.hpp:39-43) + the query it was built for
  std::uint32_t m = 0, k = 0, scales = 0;
  std::vector<float> eta, eta_lambda;
  std::vector<float> q;
};

// A PCPQIDX1 index (or a shard of it) resident in one GPU's HBM.
class Index {
 public:
  Index() = default;
  explicit Index(pcpqg_index* h) : h_(h) { check(pcpqg_index_info(h_, &info_)); }
  Index(Index&& o) noexcept : h_(std::exchange(o.h_, nullptr)), info_(o.info_) {}
  Index& operator=(Index&& o) noexcept {
    std::swap(h_, o.h_);
    info_ = o.info_;
    return *this;
  }
  Index(const Index&) = delete;
  Index& operator=(const Index&) = delete;
  ~Index() {
    if (h_) pcpqg_index_free(h_);
  }

  std::size_t n() const { return info_.shard_end - info_.shard_begin; }
  std::uint32_t m() const { return info_.m; }
  std::uint32_t k() const { return info_.k; }
  std::uint32_t d() const { return info_.d; }
  std::uint32_t scales() const { return info_.scales; }
  const pcpqg_info& info() const { return info_; }
  const pcpqg_index* handle() const { return h_; }

 private:
  pcpqg_index* h_ = nullptr;
  pcpqg_info info_{};
};

inline Index deserialize(std::span<const std::uint8_t> bytes, int device = 0,
                         std::uint64_t shard_begin = 0, std::uint64_t shard_end = 0) {
  pcpqg_index* h = nullptr;
  check(pcpqg_index_load(bytes.data(), bytes.size(), device, shard_begin, shard_end, &h));
  return Index(h);
}

inline Index read_pq_index(const std::filesystem::path& path, int device = 0,
                           std::uint64_t shard_begin = 0, std::uint64_t shard_end = 0) {
  pcpqg_index* h = nullptr;
  check(pcpqg_index_load_file(path.string().c_str(), device, shard_begin, shard_end, &h));
  return Index(h);
}

inline LookupTable build_lookup_table(const Index& index, std::span<const float> q,
                                      ScoreCounters* counters = nullptr) {
  LookupTable lut;
  lut.m = index.m();
  lut.k = index.k();
  lut.scales = index.scales();
  lut.eta.resize(static_cast<std::size_t>(lut.m) * lut.k);
  lut.eta_lambda.resize(static_cast<std::size_t>(lut.m) * lut.k * lut.scales);
  check(pcpqg_build_lut(index.handle(), q.data(), 1, static_cast<std::uint32_t>(q.size()),
                        lut.eta.data(), lut.scales ? lut.eta_lambda.data() : nullptr,
                        counters ? counters->raw() : nullptr));
  lut.q.assign(q.begin(), q.end());
  return lut;
}

inline std::vector<float> score_all(const Index& index, const LookupTable& lut,
                                    ScoreCounters* counters = nullptr) {
  if (lut.m != index.m() || lut.k != index.k() || lut.scales != index.scales())
    throw error(PCPQG_E_SIZE_MISMATCH, "score_all: table does not match index");
  std::vector<float> out(index.n());
  ScoreCounters tmp;
  check(pcpqg_score_all(index.handle(), lut.q.data(), 1, static_cast<std::uint32_t>(lut.q.size()),
                        out.data(), tmp.raw()));
  if (counters) {  // the table stage was already counted by build_lookup_table
    counters->point_mults += tmp.point_mults;
    counters->lookups += tmp.lookups;
    counters->adds += tmp.adds;
  }
  return out;
}

inline std::vector<float> score_query(const Index& index, std::span<const float> q,
                                      ScoreCounters* counters = nullptr) {
  std::vector<float> out(index.n());
  check(pcpqg_score_all(index.handle(), q.data(), 1, static_cast<std::uint32_t>(q.size()),
                        out.data(), counters ? counters->raw() : nullptr));
  return out;
}

struct SearchResult {
  std::uint32_t topn = 0;
  std::vector<std::int32_t> ids;  // B x topn, -1 past min(topn, n)
  std::vector<float> scores;      // B x topn, -inf past min(topn, n)
};

// Batched flat top-n: Q is B x d row-major.
inline SearchResult search(const Index& index, std::span<const float> Q, std::uint32_t B,
                           std::uint32_t topn) {
  SearchResult r;
  r.topn = topn;
  r.ids.resize(static_cast<std::size_t>(B) * topn);
  r.scores.resize(static_cast<std::size_t>(B) * topn);
  const std::uint32_t d = B ? static_cast<std::uint32_t>(Q.size() / B) : index.d();
  check(pcpqg_search(index.handle(), Q.data(), B, d, topn, r.ids.data(), r.scores.data()));
  return r;
}

// One index sharded over several GPUs of this process (pcpqg_multi_*): shard r
// = points [r*n/ndev, (r+1)*n/ndev) on devices[r]; search() gathers the per-shard
// top-n key rows (NCCL AllGather or peer copies) and merges them on devices[0],
// so it equals search() on the whole index.
class MultiIndex {
 public:
  MultiIndex(std::span<const std::uint8_t> bytes, std::span<const int> devices,
             int transport = PCPQG_TRANSPORT_AUTO) {
    check(pcpqg_multi_load(bytes.data(), bytes.size(), devices.data(), static_cast<int>(devices.size()),
                           transport, &h_));
    check(pcpqg_multi_info(h_, info_));
  }
  MultiIndex(MultiIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {
    for (int i = 0; i < 4; ++i) info_[i] = o.info_[i];
  }
  MultiIndex(const MultiIndex&) = delete;
  MultiIndex& operator=(const MultiIndex&) = delete;
  ~MultiIndex() {
    if (h_) pcpqg_multi_free(h_);
  }
  std::size_t n() const { return info_[0]; }
  std::size_t devices() const { return info_[1]; }
  int transport() const { return static_cast<int>(info_[2]); }
  std::uint32_t d() const { return static_cast<std::uint32_t>(info_[3]); }

  SearchResult search(std::span<const float> Q, std::uint32_t B, std::uint32_t topn) const {
    SearchResult r;
    r.topn = topn;
    r.ids.resize(static_cast<std::size_t>(B) * topn);
    r.scores.resize(static_cast<std::size_t>(B) * topn);
    const std::uint32_t dd = B ? static_cast<std::uint32_t>(Q.size() / B) : d();
    check(pcpqg_multi_search(h_, Q.data(), B, dd, topn, r.ids.data(), r.scores.data()));
    return r;
  }

 private:
  pcpqg_multi* h_ = nullptr;
  std::uint64_t info_[4] = {0, 0, 0, 0};
};

inline std::uint64_t logical_payload_bits(std::uint64_t n, std::uint32_t m, std::uint32_t k,
                                          std::uint32_t scales) {
  return pcpqg_logical_payload_bits(n, m, k, scales);
}

}  // namespace pcpq::gpu
