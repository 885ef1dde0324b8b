// Index ingest: parse + validate a PCPQIDX1 image and repack one shard of it
// into the blocked device code stream.
//
// Validation mirrors pcpq::deserialize (proj/core/src/pq_index.cpp:409-488):
// same checks, same error classes, and — because the reference reads the
// payload strictly front to back — the *first* offending byte decides which
// error is reported (a bad code before the end of a truncated file is
// code_out_of_range, not truncated).  The payload is validated and repacked
// by a pool of host threads, one contiguous range of 32-point blocks each.
#include <cuda_fp16.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <fstream>
#include <thread>

#include "pcpqg_internal.hpp"

namespace pcpqg {

void fail(int code, const std::string& what) { throw Error{code, what}; }

void check_cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess)
    fail(PCPQG_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void keep_mempool(int device) {
  // Stream-ordered scratch (cudaMallocAsync) comes from the device's default
  // pool; by default the pool returns freed memory to the driver at every
  // synchronisation, so a query's multi-GB scratch would be re-mapped on
  // every call.  Keep it cached instead (once per device).
  static std::atomic<uint64_t> done{0};
  if (device < 0 || device >= 64 || (done.load() >> device) & 1ull) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.fetch_or(1ull << device);
}

DeviceIndex::~DeviceIndex() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (d_codebooks) cudaFree(d_codebooks);
  if (d_lambda) cudaFree(d_lambda);
  if (d_codes) cudaFree(d_codes);
  if (d_amax) cudaFree(d_amax);
  if (tc) free_tc(tc);
  for (auto& kv : plans) delete kv.second;
  cudaSetDevice(prev);
}

namespace {

uint32_t ceil_log2(uint64_t v) {
  uint32_t b = 0;
  if (v <= 1) return 0;
  v -= 1;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

struct Cursor {
  const uint8_t* p;
  uint64_t len, pos = 0;
  void need(uint64_t n) {
    if (pos + n > len)
      fail(PCPQG_E_TRUNCATED, "index stream truncated at byte " + std::to_string(pos));
  }
  uint32_t u32() {
    need(4);
    const uint8_t* b = p + pos;
    pos += 4;
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
  }
  float f32() {
    const uint32_t u = u32();
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  double f64() {
    const uint64_t lo = u32(), hi = u32();
    const uint64_t u = lo | (hi << 32);
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
};

inline uint32_t rd_u32le(const uint8_t* b) {
  return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

bool fp16_exact(float a) {
  const __half h = __float2half_rn(a);
  const float back = __half2float(h);
  uint32_t x, y;
  std::memcpy(&x, &a, 4);
  std::memcpy(&y, &back, 4);
  return x == y;
}

int pool_size() {
  const unsigned hc = std::thread::hardware_concurrency();
  return static_cast<int>(std::clamp<unsigned>(hc, 1u, 64u));
}

template <class F>
void parallel_ranges(uint64_t n, F&& f) {
  const int T = static_cast<int>(std::min<uint64_t>(pool_size(), std::max<uint64_t>(1, n / 4096)));
  if (T <= 1) {
    f(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const uint64_t a = n * t / T, b = n * (t + 1) / T;
    th.emplace_back([&, a, b, t] { f(a, b, t); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

ParsedIndex parse_header(const uint8_t* bytes, uint64_t len) {
  Cursor r{bytes, len};
  r.need(8);
  if (std::memcmp(bytes, "PCPQIDX1", 8) != 0) fail(PCPQG_E_BAD_MAGIC, "not an index file");
  r.pos = 8;
  const uint32_t version = r.u32();
  if (version != 1) fail(PCPQG_E_BAD_VERSION, "unsupported index version " + std::to_string(version));
  ParsedIndex P;
  P.bytes = bytes;
  HostIndex& h = P.h;
  h.method = r.u32();
  if (h.method > 3) fail(PCPQG_E_DATA, "unknown method tag");
  h.n = r.u32();
  h.d = r.u32();
  h.padded_d = r.u32();
  h.m = r.u32();
  h.k = r.u32();
  h.scales = r.u32();
  h.t = r.f64();
  if (h.n == 0 || h.d == 0 || h.m == 0 || h.k < 2) fail(PCPQG_E_DATA, "bad header field");
  if (h.k > 65536) fail(PCPQG_E_DATA, "bad header field: k");
  if (h.scales > 256) fail(PCPQG_E_DATA, "bad header field: scale count");
  if (h.padded_d < h.d || h.padded_d % h.m != 0)
    fail(PCPQG_E_DATA, "bad header field: padded dimension");
  h.dbar = h.padded_d / h.m;
  const uint64_t m = h.m;
  const uint64_t ncb = m * h.k * h.dbar;
  // codebooks and scale codebooks (truncation reported at the first missing byte)
  if (r.pos + 4 * (ncb + m * h.scales) > len) {
    r.pos += ((len - r.pos) / 4) * 4;
    fail(PCPQG_E_TRUNCATED, "index stream truncated at byte " + std::to_string(r.pos));
  }
  h.codebooks.resize(ncb);
  for (uint64_t i = 0; i < ncb; ++i) h.codebooks[i] = r.f32();
  h.scalar_cb.resize(m * h.scales);
  for (uint64_t i = 0; i < m * h.scales; ++i) h.scalar_cb[i] = r.f32();

  P.wide = h.k > 256;
  P.cbytes = m * (P.wide ? 2 : 1);
  P.row = P.cbytes + (h.scales == 0 ? 4 * m : m);
  P.body = bytes + r.pos;
  return P;
}

uint64_t full_rows_of(const ParsedIndex& P, uint64_t len) {
  const uint64_t body = static_cast<uint64_t>(P.body - P.bytes);
  return std::min<uint64_t>(P.h.n, (len - body) / P.row);
}

void check_tail(const ParsedIndex& P, uint64_t len, const uint8_t* tail) {
  const HostIndex& h = P.h;
  const uint64_t m = h.m, n = h.n, row = P.row, cbytes = P.cbytes;
  const bool wide = P.wide;
  const uint64_t body = static_cast<uint64_t>(P.body - P.bytes);
  const uint64_t avail = len - body;
  const uint64_t full_rows = full_rows_of(P, len);
  if (full_rows < n) {
    // partial row: codes present before the end are still checked in order
    const uint8_t* pr = tail;
    const uint64_t left = avail - full_rows * row;
    const uint64_t cw = wide ? 2 : 1;
    for (uint64_t j = 0; j < m && (j + 1) * cw <= left; ++j) {
      const uint32_t c = wide ? (uint32_t(pr[2 * j]) | (uint32_t(pr[2 * j + 1]) << 8)) : pr[j];
      if (c >= h.k)
        fail(PCPQG_E_CODE_OUT_OF_RANGE, "center code out of range at point " + std::to_string(full_rows));
    }
    if (h.scales && left > cbytes)
      for (uint64_t j = 0; cbytes + j < left && j < m; ++j)
        if (pr[cbytes + j] >= h.scales)
          fail(PCPQG_E_CODE_OUT_OF_RANGE, "scale code out of range at point " + std::to_string(full_rows));
    const uint64_t unit = h.scales == 0 && left >= cbytes ? 4 : (wide && left < cbytes ? 2 : 1);
    const uint64_t at = body + full_rows * row + (left < cbytes ? (left / unit) * unit
                                                                : cbytes + ((left - cbytes) / unit) * unit);
    fail(PCPQG_E_TRUNCATED, "index stream truncated at byte " + std::to_string(at));
  }
  if (body + n * row != len)
    fail(PCPQG_E_SIZE_MISMATCH,
         "trailing bytes after index payload at byte " + std::to_string(body + n * row));
}

[[noreturn]] void fail_bad_code(const ParsedIndex& P, uint64_t pos) {
  const bool center = (pos % P.row) < P.cbytes;
  fail(PCPQG_E_CODE_OUT_OF_RANGE, std::string(center ? "center" : "scale") +
                                      " code out of range at point " + std::to_string(pos / P.row));
}

namespace {
void validate_rows(const ParsedIndex& P, const uint8_t* bytes, uint64_t len);
}

ParsedIndex parse_index(const uint8_t* bytes, uint64_t len) {
  ParsedIndex P = parse_header(bytes, len);
  validate_rows(P, bytes, len);
  return P;
}

namespace {
// the reference's row checks (pq_index.cpp:455-486) over P.h.n rows, then the
// tail checks: partial row, truncation, trailing bytes
void validate_rows(const ParsedIndex& P, const uint8_t* bytes, uint64_t len) {
  const HostIndex& h = P.h;
  const uint64_t m = h.m;
  const uint64_t row = P.row, cbytes = P.cbytes;
  const bool wide = P.wide;
  const uint64_t body = static_cast<uint64_t>(P.body - bytes);
  const uint64_t full_rows = full_rows_of(P, len);

  // ---- validate the complete rows in parallel; earliest bad code wins
  std::atomic<uint64_t> first_bad{UINT64_MAX};
  parallel_ranges(full_rows, [&](uint64_t a, uint64_t b, int) {
    for (uint64_t i = a; i < b && i * row < first_bad.load(std::memory_order_relaxed); ++i) {
      const uint8_t* pr = bytes + body + i * row;
      for (uint64_t j = 0; j < m; ++j) {
        const uint32_t c = wide ? (uint32_t(pr[2 * j]) | (uint32_t(pr[2 * j + 1]) << 8)) : pr[j];
        if (c >= h.k) {
          uint64_t pos = i * row + j, cur = first_bad.load();
          while (pos < cur && !first_bad.compare_exchange_weak(cur, pos)) {}
          return;
        }
      }
      if (h.scales) {
        for (uint64_t j = 0; j < m; ++j) {
          if (pr[cbytes + j] >= h.scales) {
            uint64_t pos = i * row + cbytes + j, cur = first_bad.load();
            while (pos < cur && !first_bad.compare_exchange_weak(cur, pos)) {}
            return;
          }
        }
      }
    }
  });
  if (first_bad.load() != UINT64_MAX) fail_bad_code(P, first_bad.load());
  check_tail(P, len, P.body + full_rows * row);
}
}  // namespace

bool alphas_fp16_exact(const ParsedIndex& P, uint64_t begin, uint64_t end) {
  if (P.h.scales != 0) return true;
  const uint64_t m = P.h.m;
  std::atomic<bool> exact{true};
  parallel_ranges(end - begin, [&](uint64_t a, uint64_t b, int) {
    for (uint64_t i = a; i < b && exact.load(std::memory_order_relaxed); ++i) {
      const uint8_t* pr = P.body + (begin + i) * P.row + P.cbytes;
      for (uint64_t j = 0; j < m; ++j) {
        const uint32_t u = rd_u32le(pr + 4 * j);
        float f;
        std::memcpy(&f, &u, 4);
        if (!fp16_exact(f)) {
          exact.store(false);
          return;
        }
      }
    }
  });
  return exact.load();
}

CodeLayout choose_layout(uint32_t k, uint32_t scales, uint32_t m, bool fp16_exact_alphas) {
  CodeLayout L;
  const uint32_t cbits = ceil_log2(k);
  if (scales >= 1) {
    const uint32_t lbits = ceil_log2(scales);
    if (cbits + lbits <= 8) {
      L.format = PCPQG_FMT_JOINT8;
      L.cw = cbits;
      L.sw = lbits;
      L.W = (m + 3) / 4;
      L.Wc = L.W;
      return L;
    }
    L.format = PCPQG_FMT_PLANES;
    L.cw = cbits <= 4 ? 4 : cbits <= 8 ? 8 : 16;
    L.sw = lbits == 0 ? 0 : lbits <= 4 ? 4 : 8;
  } else {
    L.format = PCPQG_FMT_PLANES;
    L.cw = cbits <= 4 ? 4 : cbits <= 8 ? 8 : 16;
    // fp16 plane only when every alpha round-trips exactly
    L.sw = fp16_exact_alphas ? 16 : 32;
  }
  L.Wc = (m * L.cw + 31) / 32;
  L.W = L.Wc + (m * L.sw + 31) / 32;
  return L;
}

void repack(const ParsedIndex& P, const CodeLayout& L, uint64_t begin, uint64_t n_local,
            uint32_t* dst_words) {
  const uint64_t m = P.h.m;
  const uint32_t n_blocks = static_cast<uint32_t>((n_local + kBlockPts - 1) / kBlockPts);
  const uint32_t W = L.W, Wc = L.Wc, cwb = L.cw, swb = L.sw;
  const bool wide = P.wide;
  const uint64_t cbytes = P.cbytes, row = P.row;
  const uint32_t scales = P.h.scales;
  parallel_ranges(n_blocks, [&](uint64_t ba, uint64_t bb, int) {
    for (uint64_t blk = ba; blk < bb; ++blk) {
      uint32_t* dst = dst_words + blk * W * kBlockPts;
      for (uint32_t lane = 0; lane < kBlockPts; ++lane) {
        const uint64_t p = blk * kBlockPts + lane;
        if (p >= n_local) break;
        const uint8_t* pr = P.body + (begin + p) * row;
        for (uint64_t j = 0; j < m; ++j) {
          const uint32_t c = wide ? (uint32_t(pr[2 * j]) | (uint32_t(pr[2 * j + 1]) << 8)) : pr[j];
          if (L.format == PCPQG_FMT_JOINT8) {
            const uint32_t l = scales ? pr[cbytes + j] : 0u;
            const uint32_t byte = c | (l << cwb);
            dst[(j / 4) * kBlockPts + lane] |= byte << (8 * (j % 4));
          } else {
            const uint64_t cbit = j * cwb;
            dst[(cbit / 32) * kBlockPts + lane] |= c << (cbit % 32);
            uint32_t sval = 0;
            if (swb == 4 || swb == 8) {
              sval = pr[cbytes + j];
            } else if (swb == 16) {
              const uint32_t u = rd_u32le(pr + cbytes + 4 * j);
              float f;
              std::memcpy(&f, &u, 4);
              sval = __half_as_ushort(__float2half_rn(f));
            } else if (swb == 32) {
              sval = rd_u32le(pr + cbytes + 4 * j);
            }
            if (swb) {
              const uint64_t sbit = j * swb;
              dst[(Wc + sbit / 32) * kBlockPts + lane] |= sval << (sbit % 32);
            }
          }
        }
      }
    }
  });
}

namespace {
DeviceIndex* load_parsed(ParsedIndex& P, int device, uint64_t begin, uint64_t end, uint64_t id_base,
                         uint64_t total_n);
}

DeviceIndex* load_index(const uint8_t* bytes, uint64_t len, int device, uint64_t begin,
                        uint64_t end) {
  ParsedIndex P = parse_index(bytes, len);
  const uint64_t n = P.h.n;
  if (end == 0 || end > n) end = n;
  return load_parsed(P, device, begin, end, begin, n);
}

std::vector<DeviceIndex*> load_index_shards(const uint8_t* bytes, uint64_t len, const int* devices, int ndev) {
  const ParsedIndex P0 = parse_index(bytes, len);  // validated once
  const uint64_t n = P0.h.n;
  if (ndev < 1 || static_cast<uint64_t>(ndev) > n) fail(PCPQG_E_USAGE, "bad device count for the index");
  std::vector<std::unique_ptr<DeviceIndex>> out;
  for (int r = 0; r < ndev; ++r) {
    ParsedIndex P = P0;  // (load_parsed consumes the host copy)
    const uint64_t b = n * r / ndev, e = n * (r + 1) / ndev;
    out.emplace_back(load_parsed(P, devices[r], b, e, b, n));
  }
  std::vector<DeviceIndex*> raw;
  for (auto& x : out) raw.push_back(x.release());
  return raw;
}

DeviceIndex* load_index_part(const uint8_t* bytes, uint64_t len, uint64_t row_begin, int device) {
  ParsedIndex P = parse_header(bytes, len);
  const uint64_t total = P.h.n;
  const uint64_t body = static_cast<uint64_t>(P.body - bytes);
  const uint64_t count = (len - body) / P.row;
  if (count == 0 || row_begin + count > total)
    fail(PCPQG_E_USAGE, "part image rows [" + std::to_string(row_begin) + ", " + std::to_string(row_begin + count) +
                            ") outside the index's " + std::to_string(total) + " points");
  // the part's rows validate like a whole index of `count` points; count is
  // the number of whole rows, so a partial last row is trailing bytes
  // (size_mismatch)
  P.h.n = static_cast<uint32_t>(count);
  validate_rows(P, bytes, len);
  return load_parsed(P, device, 0, count, row_begin, total);
}

namespace {
DeviceIndex* load_parsed(ParsedIndex& P, int device, uint64_t begin, uint64_t end, uint64_t id_base,
                         uint64_t total_n) {
  const uint64_t n = P.h.n, m = P.h.m;
  // ---- shard + layout
  if (begin >= end || end > n) fail(PCPQG_E_USAGE, "empty shard range");
  if (total_n > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "more than 2^31-1 points");
  auto* x = new DeviceIndex();
  std::unique_ptr<DeviceIndex> guard(x);
  x->device = device;
  x->shard_begin = id_base;
  x->n_local = end - begin;
  x->n_blocks = static_cast<uint32_t>((x->n_local + kBlockPts - 1) / kBlockPts);
  const CodeLayout L = choose_layout(P.h.k, P.h.scales, P.h.m,
                                     P.h.scales == 0 && alphas_fp16_exact(P, begin, end));
  x->format = L.format;
  x->cw = L.cw;
  x->sw = L.sw;
  x->W = L.W;
  x->Wc = L.Wc;
  const uint64_t words = static_cast<uint64_t>(x->n_blocks) * x->W * kBlockPts;
  x->code_bytes = words * 4;
  std::vector<uint32_t> packed(words, 0u);
  repack(P, L, begin, x->n_local, packed.data());

  x->h = std::move(P.h);
  x->h.n = static_cast<uint32_t>(total_n);
  const HostIndex& H = x->h;
  const uint64_t ncb = m * H.k * H.dbar;
  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  PCPQG_CUDA(cudaMalloc(&x->d_codes, std::max<uint64_t>(x->code_bytes, 128)));
  PCPQG_CUDA(cudaMemcpy(x->d_codes, packed.data(), x->code_bytes, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaMalloc(&x->d_codebooks, std::max<uint64_t>(ncb, 1) * 4));
  PCPQG_CUDA(cudaMemcpy(x->d_codebooks, H.codebooks.data(), ncb * 4, cudaMemcpyHostToDevice));
  // scale codebooks padded to m8 = m rounded up to 8 sections (pad rows 1.0)
  const uint64_t m8 = (m + 7) & ~7ull;
  std::vector<float> lam(m8 * std::max(H.scales, 1u), 1.0f);
  if (H.scales) std::copy(H.scalar_cb.begin(), H.scalar_cb.end(), lam.begin());
  PCPQG_CUDA(cudaMalloc(&x->d_lambda, lam.size() * 4));
  PCPQG_CUDA(cudaMemcpy(x->d_lambda, lam.data(), lam.size() * 4, cudaMemcpyHostToDevice));
  PCPQG_CUDA(cudaSetDevice(prev));
  return guard.release();
}
}  // namespace

}  // namespace pcpqg
