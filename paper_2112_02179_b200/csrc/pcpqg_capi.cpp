// C ABI of libpcpqg.so (declared in include/pcpqg.h).  Every entry point
// catches internal errors and returns a status; nothing throws across the ABI.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "pcpqg.h"

#include "pcpqg_internal.hpp"

namespace pcpqg {
thread_local double g_train_phases[4] = {0, 0, 0, 0};
thread_local int g_train_weights_gpu = 0;
}

struct pcpqg_index {
  std::unique_ptr<pcpqg::DeviceIndex> x;
};
struct pcpqg_ivf {
  std::unique_ptr<pcpqg::DeviceIvf> v;
};
// One index sharded over several devices of this process (pcpqg_multi_*).
struct pcpqg_multi {
  std::vector<std::unique_ptr<pcpqg::DeviceIndex>> shards;
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;  // NCCL transport; empty: peer copies
  uint64_t n = 0;
  uint32_t d = 0;
  ~pcpqg_multi();
};

namespace pcpqg {
namespace {
std::atomic<uint64_t> g_opt_version{0};
}
uint64_t options_version() { return g_opt_version.load(std::memory_order_relaxed); }
void bump_options_version() { g_opt_version.fetch_add(1, std::memory_order_relaxed); }
Options& options() {
  static Options o = [] {
    Options v;
    if (const char* e = std::getenv("PCPQG_FUSED_MERGE")) v.fused_merge = e[0] == '1';
    if (const char* e = std::getenv("PCPQG_LUT_TENSOR_CORES")) v.lut_tensor_cores = e[0] == '1';
    if (const char* e = std::getenv("PCPQG_SCAN_FILTER")) v.scan_filter = e[0] - '0';
    if (const char* e = std::getenv("PCPQG_SCAN_WS_MAX_NQ")) v.scan_ws_max_nq = std::atoi(e);
    if (const char* e = std::getenv("PCPQG_IVF_GROUPED")) v.ivf_grouped = e[0] == '1';
    return v;
  }();
  return o;
}
}  // namespace pcpqg

namespace {

thread_local std::string g_err;
thread_local bool g_profile = false;
thread_local float g_timings[3] = {0, 0, 0};
}  // namespace
namespace pcpqg {
bool profiling_enabled() { return g_profile; }
void set_last_timings(const float* t3) {
  for (int i = 0; i < 3; ++i) g_timings[i] = t3[i];
}
}  // namespace pcpqg
namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PCPQG_OK;
  } catch (const pcpqg::Error& e) {
    g_err = e.what;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return PCPQG_E_DATA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PCPQG_E_DATA;
  }
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    PCPQG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) PCPQG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Stream-ordered scratch allocation (cudaMallocAsync pool).
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* get(size_t n) {
    void* p = nullptr;
    PCPQG_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

void check_query_dim(const pcpqg::DeviceIndex& x, uint32_t d) {
  // build_lookup_table rejects a wrong query width with size_mismatch
  // (proj/core/src/pq_index.cpp:174-175)
  if (d != x.h.d) pcpqg::fail(PCPQG_E_SIZE_MISMATCH, "build_lookup_table: query dimension mismatch");
}

void check_finite(const float* Q, uint64_t cnt) {
  for (uint64_t i = 0; i < cnt; ++i)
    if (!std::isfinite(Q[i])) pcpqg::fail(PCPQG_E_DATA, "query contains non-finite values");
}

struct Events {
  cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
  bool on;
  cudaStream_t st;
  Events(bool enable, cudaStream_t s) : on(enable), st(s) {
    if (on)
      for (auto& x : e) PCPQG_CUDA(cudaEventCreate(&x));
  }
  void rec(int i) {
    if (on) PCPQG_CUDA(cudaEventRecord(e[i], st));
  }
  void finish() {
    if (!on) return;
    PCPQG_CUDA(cudaEventSynchronize(e[3]));
    for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&g_timings[i], e[i], e[i + 1]);
  }
  ~Events() {
    for (auto& x : e)
      if (x) cudaEventDestroy(x);
  }
};

// LUT -> fused scan/top-K -> merge, all on `st`.
void search_impl(const pcpqg::DeviceIndex& x, const float* dQ, uint32_t B, uint32_t topn,
                 int32_t* d_ids, float* d_scores, uint64_t* d_keys, cudaStream_t st) {
  const uint32_t K = std::min<uint32_t>(topn, x.h.n);
  if (K == 0) {
    if (d_ids) PCPQG_CUDA(cudaMemsetAsync(d_ids, 0xFF, sizeof(int32_t) * B * topn, st));
    return;
  }
  pcpqg::keep_mempool(x.device);
  if (pcpqg::tscan_eligible(x, B, K)) {  // K2-T: tensor-core pre-score filter + exact re-score
    Scratch ws(st);
    float t3[3] = {0.0f, 0.0f, 0.0f};
    pcpqg::tscan_search(x, dQ, B, K, topn, d_keys, d_ids, d_scores,
                        [&ws](size_t bytes) -> void* { return ws.get<uint8_t>(bytes); }, st,
                        g_profile ? t3 : nullptr);
    if (g_profile) pcpqg::set_last_timings(t3);
    return;
  }
  const pcpqg::SearchPlan p = pcpqg::plan_search(x, B, K, false);
  const uint32_t Bpad = p.groups * p.nq;
  Scratch ws(st);
  // PCPQG_SYNC_TRACE=1: synchronise and report after every stage (finds the kernel a hang is in)
  static const bool trace = std::getenv("PCPQG_SYNC_TRACE") != nullptr;
  auto mark = [&](const char* what) {
    if (!trace) return;
    std::fprintf(stderr, "[pcpqg trace] B=%u nq=%d ws=%d filter=%d ctas_x=%u: %s ...", B, p.nq, p.ws ? 1 : 0, p.filter,
                 p.ctas_x, what);
    std::fflush(stderr);
    const cudaError_t e = cudaStreamSynchronize(st);
    std::fprintf(stderr, " %s\n", cudaGetErrorString(e));
    std::fflush(stderr);
  };
  float* eta = ws.get<float>(static_cast<size_t>(p.groups) * pcpqg::group_stride(x, p.rs, p.rows) + 4);
  uint64_t* partial = ws.get<uint64_t>(static_cast<size_t>(p.ctas_x) * Bpad * ((K + 1) & ~1u));
  // shared K-th keys [Bpad] and the fused merge's per-group tickets, one memset
  uint64_t* gtau = ws.get<uint64_t>(Bpad + (p.groups + 1) / 2);
  uint32_t* done = reinterpret_cast<uint32_t*>(gtau + Bpad);
  const uint32_t nzero = Bpad + (p.groups + 1) / 2;
  Events ev(g_profile, st);
  ev.rec(0);
  // small batches (warp-specialised scan): the scan CTAs build their tables themselves
  const bool lut_in_scan = p.ws && !p.filter && pcpqg::options().scan_lut_fused != 0;
  if (lut_in_scan) {
    PCPQG_CUDA(cudaMemsetAsync(gtau, 0, sizeof(uint64_t) * nzero, st));
  } else if (pcpqg::options().lut_tensor_cores && !p.table && B >= 128 && pcpqg::lut_tc_supported(x)) {
    PCPQG_CUDA(cudaMemsetAsync(gtau, 0, sizeof(uint64_t) * nzero, st));
    pcpqg::launch_lut_tc(x, dQ, B, Bpad, p.nq, p.rs, p.rows, eta, st);
  } else {
    pcpqg::launch_lut(x, dQ, B, Bpad, p.nq, p.rs, p.table ? 2 : 1, p.rows, eta, st, gtau, nzero);
  }
  ev.rec(1);
  mark("lut");
  // default: the scan emits sorted survivor lists + counts, a tournament
  // kernel merges them; PCPQG_FUSED_MERGE=1 merges inside the scan instead
  const bool fused = pcpqg::options().fused_merge != 0;
  pcpqg::FusedMerge fm;
  fm.pcnt = ws.get<uint32_t>(static_cast<size_t>(p.ctas_x) * Bpad);
  if (fused) {
    fm.done = done;
    fm.keys = d_keys;
    fm.ids = d_ids;
    fm.scores = d_scores;
    fm.out_stride = topn;
  }
  pcpqg::FilterTables ft;
  if (p.filter) {
    const uint32_t m8 = (x.h.m + 7) & ~7u;
    ft.fh = reinterpret_cast<__half*>(ws.get<float>(p.groups * pcpqg::filter_group_stride(x) / 2 + 4));
    ft.flam = reinterpret_cast<__half*>(ws.get<float>(m8 * std::max(x.h.scales, 1u) / 2 + 4));
    ft.fse = reinterpret_cast<float2*>(ws.get<float>(2ull * Bpad + 4));
    ft.work = ws.get<float>(2ull * m8 + 4);
    ft.count = ws.get<unsigned long long>(66);
    PCPQG_CUDA(cudaMemsetAsync(ft.count, 0, 66 * 8, st));
    pcpqg::launch_filter_tables(x, p, eta, ft, st);
    mark("filter tables");
    const size_t ranges = static_cast<size_t>(p.groups) * p.ctas_x;
    ft.carry = ws.get<uint64_t>(ranges * p.nq * K);
    ft.carry_cnt = ws.get<uint32_t>(ranges * p.nq);
    ft.carry_done = ws.get<uint32_t>(ranges);
    PCPQG_CUDA(cudaMemsetAsync(ft.carry_done, 0, ranges * 4, st));
  }
  pcpqg::launch_scan(x, p, eta, B, partial, gtau, nullptr, st, &fm, &ft, lut_in_scan ? dQ : nullptr);
  mark("scan");
  if (p.filter && pcpqg::options().scan_filter == 3) {
    unsigned long long c[66] = {};
    PCPQG_CUDA(cudaMemcpyAsync(c, ft.count, 66 * 8, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[pcpqg] filter: %llu of %llu (point, query) pairs passed; %llu points scored directly; by range:",
                 c[0], static_cast<unsigned long long>(x.n_local) * p.groups * p.nq, c[1]);
    for (uint32_t y = 0; y < std::min<uint32_t>(p.ctas_x, 64); ++y) std::fprintf(stderr, " %llu", c[2 + y]);
    std::fprintf(stderr, "\n");
  }
  ev.rec(2);
  if (!fused)
    pcpqg::merge_sorted_lists(partial, fm.pcnt, p.ctas_x, Bpad, B, (K + 1) & ~1u, K, topn, d_keys,
                              d_ids, d_scores, st);
  mark("merge");
  ev.rec(3);
  ev.finish();
}

// ------------------------------------------------------------- multi-GPU
// libnccl, resolved at first use (dlopen): the library needs it only for
// multi-device handles, and then binds whichever libnccl.so.2 the process has.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!lib) return a;
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(lib, "ncclCommInitAll"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(lib, "ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(lib, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(lib, "ncclGroupEnd"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(lib, "ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(lib, "ncclGetErrorString"));
    a.ok = a.CommInitAll && a.CommDestroy && a.GroupStart && a.GroupEnd && a.AllGather && a.GetErrorString;
    return a;
  }();
  return api;
}
void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    pcpqg::fail(PCPQG_E_CUDA, std::string(what) + ": " + nccl_api().GetErrorString(r));
}

thread_local cudaStream_t g_streams[64] = {};
cudaStream_t host_stream(int dev) {
  if (dev < 0 || dev >= 64) pcpqg::fail(PCPQG_E_USAGE, "bad device ordinal");
  if (!g_streams[dev]) PCPQG_CUDA(cudaStreamCreateWithFlags(&g_streams[dev], cudaStreamNonBlocking));
  return g_streams[dev];
}

}  // namespace

extern "C" {

const char* pcpqg_last_error(void) { return g_err.c_str(); }

int pcpqg_index_load(const uint8_t* bytes, uint64_t len, int device, uint64_t shard_begin,
                     uint64_t shard_end, pcpqg_index** out) {
  return guarded([&] {
    if (!out) pcpqg::fail(PCPQG_E_USAGE, "null output handle");
    *out = nullptr;
    std::unique_ptr<pcpqg::DeviceIndex> xi(pcpqg::load_index(bytes, len, device, shard_begin, shard_end));  // (no handle leak on a throw)
    auto* h = new pcpqg_index();
    h->x = std::move(xi);
    *out = h;
  });
}

int pcpqg_index_load_part(const uint8_t* bytes, uint64_t len, uint64_t row_begin, int device, pcpqg_index** out) {
  return guarded([&] {
    if (!out) pcpqg::fail(PCPQG_E_USAGE, "null output handle");
    *out = nullptr;
    if (!bytes && len) pcpqg::fail(PCPQG_E_USAGE, "null image");
    std::unique_ptr<pcpqg::DeviceIndex> xi(pcpqg::load_index_part(bytes, len, row_begin, device));  // (no handle leak on a throw)
    auto* h = new pcpqg_index();
    h->x = std::move(xi);
    *out = h;
  });
}

int pcpqg_index_load_file(const char* path, int device, uint64_t shard_begin, uint64_t shard_end,
                          pcpqg_index** out) {
  std::vector<uint8_t> buf;
  const int st = guarded([&] {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) pcpqg::fail(PCPQG_E_DATA, std::string("cannot open: ") + path);
    const std::streamsize n = in.tellg();
    in.seekg(0);
    buf.resize(static_cast<size_t>(n));
    if (n && !in.read(reinterpret_cast<char*>(buf.data()), n))
      pcpqg::fail(PCPQG_E_DATA, std::string("read failed: ") + path);
  });
  if (st) return st;
  return pcpqg_index_load(buf.data(), buf.size(), device, shard_begin, shard_end, out);
}

int pcpqg_index_load_gpu(const uint8_t* bytes, uint64_t len, int device, uint64_t shard_begin,
                         uint64_t shard_end, pcpqg_index** out) {
  return guarded([&] {
    if (!out) pcpqg::fail(PCPQG_E_USAGE, "null output handle");
    *out = nullptr;
    static const uint8_t empty = 0;
    auto h = std::make_unique<pcpqg_index>();
    h->x.reset(pcpqg::load_index_gpu(bytes ? bytes : &empty, len, device, shard_begin, shard_end));
    *out = h.release();
  });
}

int pcpqg_index_load_file_gpu(const char* path, int device, uint64_t shard_begin, uint64_t shard_end,
                              pcpqg_index** out) {
  return guarded([&] {
    if (!out || !path) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    *out = nullptr;
    auto h = std::make_unique<pcpqg_index>();
    h->x.reset(pcpqg::load_index_file_gpu(path, device, shard_begin, shard_end));
    *out = h.release();
  });
}

int pcpqg_index_codes(const pcpqg_index* idx, void* out, uint64_t bytes) {
  return guarded([&] {
    if (!idx || !out) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    const auto& x = *idx->x;
    if (bytes < x.code_bytes) pcpqg::fail(PCPQG_E_USAGE, "output buffer too small");
    DeviceGuard dg(x.device);
    PCPQG_CUDA(cudaMemcpy(out, x.d_codes, x.code_bytes, cudaMemcpyDeviceToHost));
  });
}

void pcpqg_index_free(pcpqg_index* idx) { delete idx; }

int pcpqg_index_info(const pcpqg_index* idx, pcpqg_info* o) {
  return guarded([&] {
    if (!idx || !o) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    const auto& x = *idx->x;
    o->method = x.h.method;
    o->n = x.h.n;
    o->d = x.h.d;
    o->padded_d = x.h.padded_d;
    o->m = x.h.m;
    o->k = x.h.k;
    o->scales = x.h.scales;
    o->dbar = x.h.dbar;
    o->t = x.h.t;
    o->shard_begin = x.shard_begin;
    o->shard_end = x.shard_begin + x.n_local;
    o->format = x.format;
    o->center_bits = x.cw;
    o->scale_bits = x.sw;
    o->words_per_point = x.W;
    o->code_bytes = x.code_bytes;
    o->device = x.device;
  });
}

int pcpqg_plan_info(const pcpqg_index* idx, uint32_t B, uint32_t topn, uint32_t* out8) {
  return guarded([&] {
    if (!idx || !out8) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    const pcpqg::DeviceIndex& x = *idx->x;
    PCPQG_CUDA(cudaSetDevice(x.device));
    const uint32_t K = std::max(1u, std::min<uint32_t>(topn, x.h.n));
    if (pcpqg::tscan_eligible(x, std::max(B, 1u), K)) {
      // K2-T: (128 queries per CTA, threads, points per tile, 2 stages, point
      // ranges, query tiles, filter = 2 (tensor-core pre-score), table = 0)
      const pcpqg::TcPlan t = pcpqg::tscan_plan(x, std::max(B, 1u), K);
      const uint32_t v[8] = {128u, 416u, t.N, 2u, t.ranges, t.qtiles, 2u, 0u};
      std::memcpy(out8, v, sizeof(v));
      return;
    }
    const pcpqg::SearchPlan p = pcpqg::plan_search(x, std::max(B, 1u), K, false);
    const uint32_t v[8] = {static_cast<uint32_t>(p.nq), static_cast<uint32_t>(p.threads), p.ppt, p.stages, p.ctas_x,
                           p.groups, p.filter ? 1u : 0u, p.table ? 1u : 0u};
    std::memcpy(out8, v, sizeof(v));
  });
}

int pcpqg_counters(const pcpqg_index* idx, uint32_t B, uint64_t* out) {
  return guarded([&] {
    const auto& x = *idx->x;
    const uint64_t n = x.n_local, m = x.h.m, k = x.h.k, s = x.h.scales;
    out[0] += static_cast<uint64_t>(B) * k * x.h.padded_d;
    out[1] += s >= 1 ? static_cast<uint64_t>(B) * s * k * m : 0;
    out[2] += s == 0 ? static_cast<uint64_t>(B) * n * m : 0;
    out[3] += static_cast<uint64_t>(B) * n * m;
    out[4] += static_cast<uint64_t>(B) * n * (m - 1);
  });
}

uint64_t pcpqg_logical_payload_bits(uint64_t n, uint32_t m, uint32_t k, uint32_t scales) {
  auto clog2 = [](uint64_t v) -> uint64_t {
    uint64_t b = 0;
    if (v <= 1) return 0;
    v -= 1;
    while (v) {
      ++b;
      v >>= 1;
    }
    return b;
  };
  const uint64_t sb = scales == 0 ? 32 : clog2(scales);
  return n * m * (clog2(k) + sb);
}

int pcpqg_build_lut(const pcpqg_index* idx, const float* Q, uint32_t B, uint32_t d, float* eta,
                    float* eta_lambda, uint64_t* counters) {
  return guarded([&] {
    const auto& x = *idx->x;
    check_query_dim(x, d);
    if (B == 0) return;
    DeviceGuard dg(x.device);
    cudaStream_t st = host_stream(x.device);
    Scratch ws(st);
    float* dQ = ws.get<float>(static_cast<size_t>(B) * d);
    const size_t ne = static_cast<size_t>(B) * x.h.m * x.h.k;
    float* de = ws.get<float>(ne);
    PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, sizeof(float) * B * d, cudaMemcpyHostToDevice, st));
    pcpqg::launch_lut(x, dQ, B, B, 1, 1, 0, 0, de, st);
    PCPQG_CUDA(cudaMemcpyAsync(eta, de, sizeof(float) * ne, cudaMemcpyDeviceToHost, st));
    if (eta_lambda && x.h.scales) {
      float* dl = ws.get<float>(ne * x.h.scales);
      pcpqg::launch_eta_lambda(x, de, B, dl, st);
      PCPQG_CUDA(cudaMemcpyAsync(eta_lambda, dl, sizeof(float) * ne * x.h.scales,
                                 cudaMemcpyDeviceToHost, st));
    }
    PCPQG_CUDA(cudaStreamSynchronize(st));
    if (counters) {
      counters[0] += static_cast<uint64_t>(B) * x.h.k * x.h.padded_d;
      if (x.h.scales) counters[1] += static_cast<uint64_t>(B) * x.h.scales * x.h.k * x.h.m;
    }
  });
}

int pcpqg_score_all(const pcpqg_index* idx, const float* Q, uint32_t B, uint32_t d, float* scores,
                    uint64_t* counters) {
  return guarded([&] {
    const auto& x = *idx->x;
    check_query_dim(x, d);
    if (B == 0) return;
    DeviceGuard dg(x.device);
    cudaStream_t st = host_stream(x.device);
    // score in query batches so the B x n output stays bounded on the device
    const uint32_t per = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(B, (1ull << 28) / std::max<uint64_t>(x.n_local, 1))));
    for (uint32_t q0 = 0; q0 < B; q0 += per) {
      const uint32_t nb = std::min(per, B - q0);
      const pcpqg::SearchPlan p = pcpqg::plan_search(x, nb, 0, true);
      Scratch ws(st);
      float* dQ = ws.get<float>(static_cast<size_t>(nb) * d);
      float* eta = ws.get<float>(static_cast<size_t>(p.groups) * pcpqg::group_stride(x, p.rs, p.rows) + 4);
      float* ds = ws.get<float>(static_cast<size_t>(nb) * x.n_local);
      PCPQG_CUDA(cudaMemcpyAsync(dQ, Q + static_cast<size_t>(q0) * d, sizeof(float) * nb * d,
                                 cudaMemcpyHostToDevice, st));
      pcpqg::launch_lut(x, dQ, nb, p.groups * p.nq, p.nq, p.rs, p.table ? 2 : 1, p.rows, eta, st);
      pcpqg::launch_scan(x, p, eta, nb, nullptr, nullptr, ds, st);
      PCPQG_CUDA(cudaMemcpyAsync(scores + static_cast<size_t>(q0) * x.n_local, ds,
                                 sizeof(float) * nb * x.n_local, cudaMemcpyDeviceToHost, st));
      PCPQG_CUDA(cudaStreamSynchronize(st));
    }
    if (counters) {
      const uint64_t n = x.n_local, m = x.h.m;
      counters[0] += static_cast<uint64_t>(B) * x.h.k * x.h.padded_d;
      if (x.h.scales) counters[1] += static_cast<uint64_t>(B) * x.h.scales * x.h.k * m;
      else counters[2] += static_cast<uint64_t>(B) * n * m;
      counters[3] += static_cast<uint64_t>(B) * n * m;
      counters[4] += static_cast<uint64_t>(B) * n * (m - 1);
    }
  });
}

int pcpqg_search(const pcpqg_index* idx, const float* Q, uint32_t B, uint32_t d, uint32_t topn,
                 int32_t* ids, float* scores) {
  return guarded([&] {
    const auto& x = *idx->x;
    check_query_dim(x, d);
    check_finite(Q, static_cast<uint64_t>(B) * d);
    if (B == 0 || topn == 0) return;
    DeviceGuard dg(x.device);
    cudaStream_t st = host_stream(x.device);
    Scratch ws(st);
    float* dQ = ws.get<float>(static_cast<size_t>(B) * d);
    int32_t* di = ws.get<int32_t>(static_cast<size_t>(B) * topn);
    float* ds = scores ? ws.get<float>(static_cast<size_t>(B) * topn) : nullptr;
    PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, sizeof(float) * B * d, cudaMemcpyHostToDevice, st));
    search_impl(x, dQ, B, topn, di, ds, nullptr, st);
    PCPQG_CUDA(cudaMemcpyAsync(ids, di, sizeof(int32_t) * B * topn, cudaMemcpyDeviceToHost, st));
    if (scores)
      PCPQG_CUDA(cudaMemcpyAsync(scores, ds, sizeof(float) * B * topn, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
  });
}

int pcpqg_search_device(const pcpqg_index* idx, const float* dQ, uint32_t B, uint32_t d,
                        uint32_t topn, int32_t* d_ids, float* d_scores, uint64_t* d_keys,
                        void* cuda_stream) {
  return guarded([&] {
    const auto& x = *idx->x;
    check_query_dim(x, d);
    if (B == 0 || topn == 0) return;
    DeviceGuard dg(x.device);
    search_impl(x, dQ, B, topn, d_ids, d_scores, d_keys, static_cast<cudaStream_t>(cuda_stream));
  });
}

int pcpqg_merge_device(const uint64_t* d_keys, uint32_t L, uint32_t B, uint32_t topn,
                       int32_t* d_ids, float* d_scores, uint64_t* d_keys_out, int device,
                       void* cuda_stream) {
  return guarded([&] {
    if (B == 0 || topn == 0 || L == 0) return;
    DeviceGuard dg(device);
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    // the per-GPU rows are sorted descending (empty keys last)
    pcpqg::merge_sorted_lists(d_keys, nullptr, L, B, B, topn, topn, topn, d_keys_out, d_ids,
                              d_scores, st);
  });
}

int pcpqg_set_option(const char* name, int64_t value) {
  return guarded([&] {
    const std::string n = name ? name : "";
    if (n == "lut_tensor_cores") pcpqg::options().lut_tensor_cores = value != 0;
    else if (n == "fused_merge") pcpqg::options().fused_merge = value != 0;
    else if (n == "scan_ws") pcpqg::options().scan_ws = value != 0;
    else if (n == "scan_filter") pcpqg::options().scan_filter = value;
    else if (n == "scan_ws_max_nq") pcpqg::options().scan_ws_max_nq = value;
    else if (n == "ivf_grouped") pcpqg::options().ivf_grouped = value != 0;
    else if (n == "merge_wide") pcpqg::options().merge_wide = value != 0;
    else if (n == "scan_lut_fused") pcpqg::options().scan_lut_fused = value != 0;
    else if (n == "merge_oneshot") pcpqg::options().merge_oneshot = value != 0;
    else if (n == "pdl") pcpqg::options().pdl = value != 0;
    else if (n == "gt_chunk") pcpqg::options().gt_chunk = static_cast<int>(value);
    else if (n == "gt_tc") pcpqg::options().gt_tc = value != 0;
    else if (n == "gt_tc_min_batch") pcpqg::options().gt_tc_min_batch = static_cast<int>(value);
    else if (n == "scan_shape") pcpqg::options().scan_shape = static_cast<int>(value);
    else if (n == "scan_tc") pcpqg::options().scan_tc = static_cast<int>(value);
    else if (n == "scan_tc_min_batch") pcpqg::options().scan_tc_min_batch = static_cast<int>(value);
    else if (n == "scan_tc_fin_small") pcpqg::options().scan_tc_fin_small = value != 0;
    else if (n == "scan_tc_min_work") pcpqg::options().scan_tc_min_work = value;
    else if (n == "scan_tc_qh") pcpqg::options().scan_tc_qh = value != 0;
    else if (n == "scan_tc_at") pcpqg::options().scan_tc_at = value != 0;
    else if (n == "scan_tc_qt") pcpqg::options().scan_tc_qt = static_cast<int>(value);
    else if (n == "scan_tc_cs") pcpqg::options().scan_tc_cs = value != 0;
    else if (n == "scan_tc_exp") pcpqg::options().scan_tc_exp = static_cast<int>(value);
    else if (n == "scan_tc_diag") pcpqg::options().scan_tc_diag = static_cast<int>(value);
    else if (n == "train_level_sort") pcpqg::options().train_level_sort = value != 0;
    else if (n == "weights_gpu") pcpqg::options().weights_gpu = value != 0;
    else if (n == "scan_tc_seed_max") pcpqg::options().scan_tc_seed_max = static_cast<int>(value);
    else if (n == "scan_tc_seed") pcpqg::options().scan_tc_seed = static_cast<int>(value);
    else if (n == "scan_tc_cache_pct") pcpqg::options().scan_tc_cache_pct = static_cast<int>(value);
    else pcpqg::fail(PCPQG_E_USAGE, "unknown option: " + n);
    pcpqg::bump_options_version();
  });
}

int pcpqg_set_profiling(int enabled) {
  g_profile = enabled != 0;
  return PCPQG_OK;
}

int pcpqg_last_timings(float* out3) {
  for (int i = 0; i < 3; ++i) out3[i] = g_timings[i];
  return PCPQG_OK;
}

int pcpqg_assign_projective(const float* d_x, uint64_t n, uint32_t dbar, const float* d_centers,
                            uint32_t k, uint32_t* d_assign, double* d_alpha, double* d_loss,
                            int device, void* cuda_stream) {
  return guarded([&] {
    if (k == 0 || dbar == 0) pcpqg::fail(PCPQG_E_DATA, "assign_projective: bad centers");
    DeviceGuard dg(device);
    pcpqg::launch_assign_projective(d_x, n, dbar, d_centers, k, d_assign, d_alpha, d_loss,
                                    static_cast<cudaStream_t>(cuda_stream));
  });
}

int pcpqg_assign_anisotropic(const float* d_x, uint64_t n, uint32_t dbar, const float* d_centers,
                             uint32_t k, const double* d_h_par, const double* d_h_bot,
                             const uint32_t* d_prev, uint32_t* d_assign, double* d_alpha,
                             double* d_loss, int device, void* cuda_stream) {
  return guarded([&] {
    if (k == 0 || dbar == 0) pcpqg::fail(PCPQG_E_DATA, "assign_anisotropic: bad centers");
    DeviceGuard dg(device);
    pcpqg::launch_assign_anisotropic(d_x, n, dbar, d_centers, k, d_h_par, d_h_bot, d_prev,
                                     d_assign, d_alpha, d_loss,
                                     static_cast<cudaStream_t>(cuda_stream));
  });
}

int pcpqg_center_stats(const float* d_x, uint64_t n, uint32_t dbar, uint32_t nsec,
                       uint64_t sec_stride, const uint32_t* d_assign, const double* d_alpha,
                       const double* d_h_par, const double* d_h_bot, uint32_t k,
                       const double* d_init, double* d_stats, int device, void* cuda_stream) {
  return guarded([&] {
    if (k == 0 || nsec == 0) pcpqg::fail(PCPQG_E_DATA, "center_stats: empty problem");
    DeviceGuard dg(device);
    pcpqg::launch_center_stats(d_x, n, dbar, nsec, sec_stride, d_assign, d_alpha, d_h_par, d_h_bot,
                               k, d_init, d_stats, static_cast<cudaStream_t>(cuda_stream));
  });
}

int pcpqg_aniso_alpha_codes(const float* d_x, uint64_t n, uint32_t dbar, const float* d_centers,
                            const uint32_t* d_assign, const double* d_h_par,
                            const double* d_h_bot, const float* d_values, uint32_t s,
                            uint8_t* d_codes, int device, void* cuda_stream) {
  return guarded([&] {
    if (s == 0 || s > 256) pcpqg::fail(PCPQG_E_DATA, "scalar quantization: need 1 <= s <= 256");
    DeviceGuard dg(device);
    pcpqg::launch_aniso_alpha_codes(d_x, n, dbar, d_centers, d_assign, d_h_par, d_h_bot, d_values,
                                    s, d_codes, static_cast<cudaStream_t>(cuda_stream));
  });
}


// ---------------------------------------------------------------- IVF
int pcpqg_ivf_load(const uint8_t* bytes, uint64_t len, int device, pcpqg_ivf** out) {
  return guarded([&] {
    if (!out) pcpqg::fail(PCPQG_E_USAGE, "null output");
    *out = nullptr;
    if (!bytes && len) pcpqg::fail(PCPQG_E_USAGE, "null bytes");
    static const uint8_t empty = 0;
    auto h = std::make_unique<pcpqg_ivf>();  // load_ivf selects `device` for the upload
    h->v.reset(pcpqg::load_ivf(bytes ? bytes : &empty, len, device));
    *out = h.release();
  });
}

int pcpqg_ivf_load_file(const char* path, int device, pcpqg_ivf** out) {
  std::vector<uint8_t> buf;
  const int st = guarded([&] {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) pcpqg::fail(PCPQG_E_DATA, std::string("cannot open: ") + path);
    const std::streamsize n = in.tellg();
    in.seekg(0);
    buf.resize(static_cast<size_t>(n));
    if (n && !in.read(reinterpret_cast<char*>(buf.data()), n))
      pcpqg::fail(PCPQG_E_DATA, std::string("read failed: ") + path);
  });
  if (st) return st;
  return pcpqg_ivf_load(buf.data(), buf.size(), device, out);
}

void pcpqg_ivf_free(pcpqg_ivf* v) { delete v; }

int pcpqg_ivf_info(const pcpqg_ivf* h, uint64_t* o) {
  return guarded([&] {
    if (!h || !o) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    const auto& v = *h->v;
    const uint64_t vals[10] = {v.n, v.d, v.kbar, v.m, v.k_max, v.scales, v.method, v.n_raw,
                               v.code_bytes, v.n_pq ? v.lay.format : 0u};
    for (int i = 0; i < 10; ++i) o[i] = vals[i];
  });
}

namespace {
void check_ivf_args(const pcpqg::DeviceIvf& v, uint32_t d, uint32_t k_probe, uint32_t topn) {
  // query_ivf's argument checks, in its order (proj/core/src/ivf.cpp:93-98)
  if (d != v.d) pcpqg::fail(PCPQG_E_SIZE_MISMATCH, "query_ivf: dimension mismatch");
  if (k_probe < 1 || k_probe > v.kbar) pcpqg::fail(PCPQG_E_DATA, "query_ivf: need 1 <= k_probe <= kbar");
  if (topn < 1) pcpqg::fail(PCPQG_E_DATA, "query_ivf: topN must be >= 1");
}
}  // namespace

int pcpqg_ivf_query(const pcpqg_ivf* h, const float* Q, uint32_t B, uint32_t d, uint32_t k_probe,
                    uint32_t topn, const uint32_t* requested, uint32_t R, int32_t* ids,
                    double* scores, uint32_t* counts, uint8_t* short_flags, double* req_scores,
                    uint32_t* probes) {
  return guarded([&] {
    if (!h) pcpqg::fail(PCPQG_E_USAGE, "null index");
    const auto& v = *h->v;
    check_ivf_args(v, d, k_probe, topn);
    if (R && (!requested || !req_scores)) pcpqg::fail(PCPQG_E_USAGE, "null requested ids");
    for (uint64_t i = 0; i < static_cast<uint64_t>(B) * R; ++i)
      if (requested[i] >= v.n) pcpqg::fail(PCPQG_E_DATA, "query_ivf: requested id out of range");
    check_finite(Q, static_cast<uint64_t>(B) * d);
    if (B == 0) return;
    DeviceGuard dg(v.device);
    cudaStream_t st = host_stream(v.device);
    Scratch ws(st);
    const size_t bt = static_cast<size_t>(B) * topn, br = static_cast<size_t>(B) * R;
    float* dQ = ws.get<float>(static_cast<size_t>(B) * d);
    uint32_t* dreq = R ? ws.get<uint32_t>(br) : nullptr;
    int32_t* di = ws.get<int32_t>(bt);
    double* ds = ws.get<double>(bt);
    uint32_t* dc = ws.get<uint32_t>(B);
    uint8_t* dsh = ws.get<uint8_t>(B);
    double* drs = R ? ws.get<double>(br) : nullptr;
    uint32_t* dp = probes ? ws.get<uint32_t>(static_cast<size_t>(B) * k_probe) : nullptr;
    PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, sizeof(float) * B * d, cudaMemcpyHostToDevice, st));
    if (R) PCPQG_CUDA(cudaMemcpyAsync(dreq, requested, 4 * br, cudaMemcpyHostToDevice, st));
    pcpqg::ivf_query(v, dQ, B, k_probe, topn, dreq, R, di, ds, dc, dsh, drs, dp, st);
    if (ids) PCPQG_CUDA(cudaMemcpyAsync(ids, di, 4 * bt, cudaMemcpyDeviceToHost, st));
    if (scores) PCPQG_CUDA(cudaMemcpyAsync(scores, ds, 8 * bt, cudaMemcpyDeviceToHost, st));
    if (counts) PCPQG_CUDA(cudaMemcpyAsync(counts, dc, 4ull * B, cudaMemcpyDeviceToHost, st));
    if (short_flags) PCPQG_CUDA(cudaMemcpyAsync(short_flags, dsh, B, cudaMemcpyDeviceToHost, st));
    if (R) PCPQG_CUDA(cudaMemcpyAsync(req_scores, drs, 8 * br, cudaMemcpyDeviceToHost, st));
    if (probes)
      PCPQG_CUDA(cudaMemcpyAsync(probes, dp, 4ull * B * k_probe, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
  });
}

int pcpqg_ivf_query_device(const pcpqg_ivf* h, const float* dQ, uint32_t B, uint32_t d,
                           uint32_t k_probe, uint32_t topn, const uint32_t* d_requested,
                           uint32_t R, int32_t* d_ids, double* d_scores, uint32_t* d_counts,
                           uint8_t* d_short_flags, double* d_req_scores, uint32_t* d_probes,
                           void* cuda_stream) {
  return guarded([&] {
    if (!h) pcpqg::fail(PCPQG_E_USAGE, "null index");
    const auto& v = *h->v;
    check_ivf_args(v, d, k_probe, topn);
    if (B == 0) return;
    if (!d_ids || !d_scores || !d_counts || !d_short_flags)
      pcpqg::fail(PCPQG_E_USAGE, "null output");
    if (R && (!d_requested || !d_req_scores)) pcpqg::fail(PCPQG_E_USAGE, "null requested ids");
    DeviceGuard dg(v.device);
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (R && pcpqg::ivf_check_requested(d_requested, static_cast<uint64_t>(B) * R, v.n, st))
      pcpqg::fail(PCPQG_E_DATA, "query_ivf: requested id out of range");
    pcpqg::ivf_query(v, dQ, B, k_probe, topn, d_requested, R, d_ids, d_scores, d_counts,
                     d_short_flags, d_req_scores, d_probes, st);
  });
}

int pcpqg_ivf_counters(const pcpqg_ivf* h, const uint32_t* probes, uint32_t B, uint32_t k_probe,
                       uint64_t* out) {
  return guarded([&] {
    if (!h || !out || (B && !probes)) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    const auto& v = *h->v;
    // score_query's counters for every probed PQ cell (ivf.cpp:127-128;
    // pq_index.cpp:170-244), the same shape formula as pcpqg_counters
    const uint64_t m = v.m, s = v.scales;
    for (uint64_t i = 0; i < static_cast<uint64_t>(B) * k_probe; ++i) {
      const uint32_t r = probes[i];
      if (r >= v.kbar) pcpqg::fail(PCPQG_E_USAGE, "bad cell id");
      const uint64_t k = v.cell_k[r], n = v.cell_n[r];
      if (k == 0) continue;  // raw cell: no sub-index
      out[0] += k * v.padded_d;
      out[1] += s >= 1 ? s * k * m : 0;
      out[2] += s == 0 ? n * m : 0;
      out[3] += n * m;
      out[4] += n * (m - 1);
    }
  });
}

// ---------------------------------------------------------------- eval
int pcpqg_brute_force_topn(const float* X, uint64_t n, uint32_t d, const float* Q, uint32_t B,
                           uint32_t topn, int32_t* ids, double* scores, int device) {
  return guarded([&] {
    if (topn < 1 || topn > n) pcpqg::fail(PCPQG_E_DATA, "brute_force_topn: need 1 <= N <= n");
    if (B == 0) return;
    if (!X || !Q || !ids || !scores) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    DeviceGuard dg(device);
    cudaStream_t st = host_stream(device);
    Scratch ws(st);
    float* dX = ws.get<float>(n * d);
    float* dQ = ws.get<float>(static_cast<size_t>(B) * d);
    int32_t* di = ws.get<int32_t>(static_cast<size_t>(B) * topn);
    double* ds = ws.get<double>(static_cast<size_t>(B) * topn);
    PCPQG_CUDA(cudaMemcpyAsync(dX, X, 4 * n * d, cudaMemcpyHostToDevice, st));
    PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, 4ull * B * d, cudaMemcpyHostToDevice, st));
    pcpqg::brute_force_topn(dX, n, d, dQ, B, topn, di, ds, device, st);
    PCPQG_CUDA(cudaMemcpyAsync(ids, di, 4ull * B * topn, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaMemcpyAsync(scores, ds, 8ull * B * topn, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
  });
}

int pcpqg_brute_force_topn_device(const float* d_X, uint64_t n, uint32_t d, const float* d_Q,
                                  uint32_t B, uint32_t topn, int32_t* d_ids, double* d_scores,
                                  int device, void* cuda_stream) {
  return guarded([&] {
    if (topn < 1 || topn > n) pcpqg::fail(PCPQG_E_DATA, "brute_force_topn: need 1 <= N <= n");
    if (B == 0) return;
    DeviceGuard dg(device);
    pcpqg::brute_force_topn(d_X, n, d, d_Q, B, topn, d_ids, d_scores, device,
                            static_cast<cudaStream_t>(cuda_stream));
  });
}

int pcpqg_recall1(const float* X, uint64_t n, uint32_t d, const float* Q, uint32_t B,
                  const uint32_t* retrieved, uint32_t R, const double* exact_top1, int32_t* hits,
                  int device) {
  return guarded([&] {
    for (uint64_t i = 0; i < static_cast<uint64_t>(B) * R; ++i)
      if (retrieved[i] >= n) pcpqg::fail(PCPQG_E_DATA, "recall1_single: id out of range");
    if (B == 0) return;
    DeviceGuard dg(device);
    cudaStream_t st = host_stream(device);
    Scratch ws(st);
    float* dX = ws.get<float>(n * d);
    float* dQ = ws.get<float>(static_cast<size_t>(B) * d);
    uint32_t* dr = ws.get<uint32_t>(static_cast<size_t>(B) * R);
    double* dt = ws.get<double>(B);
    int32_t* dh = ws.get<int32_t>(B);
    PCPQG_CUDA(cudaMemcpyAsync(dX, X, 4 * n * d, cudaMemcpyHostToDevice, st));
    PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, 4ull * B * d, cudaMemcpyHostToDevice, st));
    if (R) PCPQG_CUDA(cudaMemcpyAsync(dr, retrieved, 4ull * B * R, cudaMemcpyHostToDevice, st));
    PCPQG_CUDA(cudaMemcpyAsync(dt, exact_top1, 8ull * B, cudaMemcpyHostToDevice, st));
    pcpqg::recall1(dX, n, d, dQ, B, dr, R, dt, dh, st);
    PCPQG_CUDA(cudaMemcpyAsync(hits, dh, 4ull * B, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
  });
}

// ---------------------------------------------------------------- training
int pcpqg_train_kmeans(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                       double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device,
                       uint8_t** out, uint64_t* out_len) {
  return guarded([&] {
    if (!out || !out_len || (!X && n && d)) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    *out = nullptr;
    *out_len = 0;
    std::vector<uint8_t> img = pcpqg::train_kmeans(X, n, d, m, k, s, t_frac, max_iters, tol, seed, device);
    auto* p = static_cast<uint8_t*>(std::malloc(std::max<size_t>(img.size(), 1)));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, img.data(), img.size());
    *out = p;
    *out_len = img.size();
  });
}

int pcpqg_train_pcpq(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s, int quantize,
                     double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device, uint8_t** out,
                     uint64_t* out_len) {
  return guarded([&] {
    if (!out || !out_len || (!X && n && d)) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    *out = nullptr;
    *out_len = 0;
    std::vector<uint8_t> img =
        pcpqg::train_pcpq(X, n, d, m, k, s, quantize != 0, t_frac, max_iters, tol, seed, device);
    auto* p = static_cast<uint8_t*>(std::malloc(std::max<size_t>(img.size(), 1)));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, img.data(), img.size());
    *out = p;
    *out_len = img.size();
  });
}

int pcpqg_train_aniso_multi(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s, int method,
                            int quantize, double t_frac, uint32_t max_iters, double tol, uint64_t seed,
                            const int* devices, int ndev, uint8_t** out, uint64_t* out_len) {
  return guarded([&] {
    if (!out || !out_len || (!X && n && d) || !devices) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    if (ndev < 1) pcpqg::fail(PCPQG_E_USAGE, "train_aniso: need at least one device");
    if (method != 1 && method != 3) pcpqg::fail(PCPQG_E_USAGE, "train_aniso: method must be 1 (aniso) or 3 (apcpq)");
    *out = nullptr;
    *out_len = 0;
    std::vector<uint8_t> img = pcpqg::train_aniso(X, n, d, m, k, s, method == 3, quantize != 0, t_frac, max_iters,
                                                  tol, seed, devices, ndev);
    auto* p = static_cast<uint8_t*>(std::malloc(std::max<size_t>(img.size(), 1)));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, img.data(), img.size());
    *out = p;
    *out_len = img.size();
  });
}

int pcpqg_train_aniso(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s, int method,
                      int quantize, double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device,
                      uint8_t** out, uint64_t* out_len) {
  return pcpqg_train_aniso_multi(X, n, d, m, k, s, method, quantize, t_frac, max_iters, tol, seed, &device, 1, out,
                                 out_len);
}

int pcpqg_aniso_weights(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot) {
  return guarded([&] {
    if ((!x && n) || (!h_par && n) || (!h_bot && n)) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    if (t < 0.0 || !std::isfinite(t)) pcpqg::fail(PCPQG_E_DATA, "aniso_weights: bad threshold");
    if (dbar < 2) pcpqg::fail(PCPQG_E_DATA, "aniso_weights: dbar must be >= 2");
    pcpqg::aniso_weights_host(x, n, dbar, t, h_par, h_bot);
  });
}

int pcpqg_aniso_weights_gpu(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot,
                            int device) {
  return guarded([&] {
    if ((!x && n) || (!h_par && n) || (!h_bot && n)) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    if (t < 0.0 || !std::isfinite(t)) pcpqg::fail(PCPQG_E_DATA, "aniso_weights: bad threshold");
    if (dbar < 2) pcpqg::fail(PCPQG_E_DATA, "aniso_weights: dbar must be >= 2");
    pcpqg::aniso_weights_gpu(x, n, dbar, t, h_par, h_bot, device);
  });
}

int pcpqg_sin_selfcheck(int device, uint64_t* mismatches, uint64_t* total) {
  return guarded([&] {
    if (!mismatches) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    *mismatches = pcpqg::sin_port_mismatches(device, total);
  });
}

int pcpqg_train_weights_on_gpu(int* out) {
  return guarded([&] {
    if (!out) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    *out = pcpqg::g_train_weights_gpu;
  });
}

int pcpqg_train_phases(double* out4) {
  return guarded([&] {
    if (!out4) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    for (int i = 0; i < 4; ++i) out4[i] = pcpqg::g_train_phases[i];
  });
}

void pcpqg_free(void* p) { std::free(p); }

int pcpqg_multi_load(const uint8_t* bytes, uint64_t len, const int* devices, int ndev, int transport,
                     pcpqg_multi** out) {
  return guarded([&] {
    if (!out || !devices || ndev < 1) pcpqg::fail(PCPQG_E_USAGE, "null argument or no devices");
    *out = nullptr;
    if (transport < PCPQG_TRANSPORT_AUTO || transport > PCPQG_TRANSPORT_PEER)
      pcpqg::fail(PCPQG_E_USAGE, "unknown transport");
    std::unique_ptr<pcpqg_multi> h(new pcpqg_multi());
    h->devices.assign(devices, devices + ndev);
    for (pcpqg::DeviceIndex* x : pcpqg::load_index_shards(bytes, len, devices, ndev)) h->shards.emplace_back(x);
    h->n = h->shards[0]->h.n;
    h->d = h->shards[0]->h.d;
    std::vector<int> sorted = h->devices;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const bool use_nccl = transport == PCPQG_TRANSPORT_NCCL ||
                          (transport == PCPQG_TRANSPORT_AUTO && ndev > 1 && distinct && nccl_api().ok);
    if (transport == PCPQG_TRANSPORT_NCCL && !(distinct && nccl_api().ok))
      pcpqg::fail(PCPQG_E_UNSUPPORTED, "NCCL transport needs distinct devices and libnccl.so.2");
    if (use_nccl) {
      h->comms.resize(ndev);
      check_nccl(nccl_api().CommInitAll(h->comms.data(), ndev, h->devices.data()), "ncclCommInitAll");
    } else {
      // peer copies into device 0's buffer (NVLink where peers can access each other)
      for (int r = 1; r < ndev; ++r) {
        if (h->devices[r] == h->devices[0]) continue;
        int can = 0;
        PCPQG_CUDA(cudaDeviceCanAccessPeer(&can, h->devices[0], h->devices[r]));
        if (can) {
          DeviceGuard dg(h->devices[0]);
          const cudaError_t e = cudaDeviceEnablePeerAccess(h->devices[r], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) PCPQG_CUDA(e);
          cudaGetLastError();
        }
      }
    }
    *out = h.release();
  });
}

void pcpqg_multi_free(pcpqg_multi* h) { delete h; }

int pcpqg_multi_info(const pcpqg_multi* h, uint64_t* out4) {
  return guarded([&] {
    if (!h || !out4) pcpqg::fail(PCPQG_E_USAGE, "null argument");
    out4[0] = h->n;
    out4[1] = h->shards.size();
    out4[2] = h->comms.empty() ? PCPQG_TRANSPORT_PEER : PCPQG_TRANSPORT_NCCL;
    out4[3] = h->d;
  });
}

int pcpqg_multi_search(const pcpqg_multi* h, const float* Q, uint32_t B, uint32_t d, uint32_t topn,
                       int32_t* ids, float* scores) {
  return guarded([&] {
    if (!h) pcpqg::fail(PCPQG_E_USAGE, "null handle");
    check_query_dim(*h->shards[0], d);
    check_finite(Q, static_cast<uint64_t>(B) * d);
    if (B == 0 || topn == 0) return;
    const int L = static_cast<int>(h->shards.size());
    const size_t rowk = static_cast<size_t>(B) * topn;
    std::vector<std::unique_ptr<Scratch>> ws(L);
    std::vector<uint64_t*> keys(L), gathered(L, nullptr);
    std::vector<cudaStream_t> st(L);
    // 1. every shard's fused search, asynchronously on its own device
    for (int r = 0; r < L; ++r) {
      DeviceGuard dg(h->devices[r]);
      st[r] = host_stream(h->devices[r]);
      ws[r].reset(new Scratch(st[r]));
      float* dQ = ws[r]->get<float>(static_cast<size_t>(B) * d);
      keys[r] = ws[r]->get<uint64_t>(rowk);
      PCPQG_CUDA(cudaMemcpyAsync(dQ, Q, sizeof(float) * B * d, cudaMemcpyHostToDevice, st[r]));
      search_impl(*h->shards[r], dQ, B, topn, nullptr, nullptr, keys[r], st[r]);
    }
    // 2. gather the [B][topn] key rows (global ids) on device 0
    const int root = h->devices[0];
    if (!h->comms.empty()) {
      for (int r = 0; r < L; ++r) {
        DeviceGuard dg(h->devices[r]);
        gathered[r] = ws[r]->get<uint64_t>(rowk * L);
      }
      check_nccl(nccl_api().GroupStart(), "ncclGroupStart");
      for (int r = 0; r < L; ++r)
        check_nccl(nccl_api().AllGather(keys[r], gathered[r], rowk, ncclUint64, h->comms[r], st[r]), "ncclAllGather");
      check_nccl(nccl_api().GroupEnd(), "ncclGroupEnd");
    } else {
      DeviceGuard dg(root);
      gathered[0] = ws[0]->get<uint64_t>(rowk * L);
      for (int r = 0; r < L; ++r) {
        if (r > 0) {
          cudaEvent_t ev;
          {
            DeviceGuard dr(h->devices[r]);
            PCPQG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            PCPQG_CUDA(cudaEventRecord(ev, st[r]));
          }
          PCPQG_CUDA(cudaStreamWaitEvent(st[0], ev, 0));
          cudaEventDestroy(ev);
        }
        PCPQG_CUDA(cudaMemcpyPeerAsync(gathered[0] + rowk * r, root, keys[r], h->devices[r], rowk * 8, st[0]));
      }
    }
    // 3. merge on device 0 (lists sorted, keys carry global ids: equals the
    // unsharded partial_sort of proj/tools/main.cpp:233-237)
    DeviceGuard dg(root);
    int32_t* di = ws[0]->get<int32_t>(rowk);
    float* ds = ws[0]->get<float>(rowk);
    pcpqg::merge_sorted_lists(gathered[0], nullptr, static_cast<uint32_t>(L), B, B, topn, topn, topn, nullptr, di,
                              ds, st[0]);
    PCPQG_CUDA(cudaMemcpyAsync(ids, di, sizeof(int32_t) * rowk, cudaMemcpyDeviceToHost, st[0]));
    if (scores) PCPQG_CUDA(cudaMemcpyAsync(scores, ds, sizeof(float) * rowk, cudaMemcpyDeviceToHost, st[0]));
    for (int r = 0; r < L; ++r) {
      DeviceGuard dr(h->devices[r]);
      PCPQG_CUDA(cudaStreamSynchronize(st[r]));
    }
    for (int r = L - 1; r >= 0; --r) {  // stream-ordered frees on each device
      DeviceGuard dr(h->devices[r]);
      ws[r].reset();
    }
  });
}

}  // extern "C"

pcpqg_multi::~pcpqg_multi() {
  for (ncclComm_t c : comms)
    if (c) nccl_api().CommDestroy(c);
}
