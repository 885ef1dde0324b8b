// GPU index ingest: pcpq::deserialize's validation
// (proj/core/src/pq_index.cpp:409-488) and the repack into the blocked device
// code stream, done in HBM instead of on host threads.
//
//   host  header + codebooks (parse_header), the partial last row / truncation
//         / trailing-byte checks (check_tail) — a few hundred bytes
//   I1    the complete code rows stream to HBM through pinned double buffers
//   I2    validation: every code byte checked in parallel, coalesced; the
//         reference's first offending byte (its sequential reader stops there)
//         is the minimum over the bad positions (atomicMin), encoded exactly as
//         the host path encodes it, so the error is the same
//   I3    raw alphas: fp16 round-trip check of the shard (the fp16 plane rule)
//   I4    repack: one warp per 32-point block stages the block's 32 rows in
//         shared memory and writes each of its W words with one coalesced
//         128-byte store — the same words as the host repack
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>
#include <fstream>
#include <memory>
#include <thread>

#include "pcpqg_internal.hpp"

namespace pcpqg {
namespace {

struct BodyDesc {
  uint64_t rows;          // complete rows on the device
  uint32_t row, cbytes, m, k, scales;
  bool wide;
};

// I2: one thread per 4 body bytes
__global__ void ingest_validate_kernel(const uint8_t* __restrict__ body, BodyDesc b,
                                       unsigned long long* __restrict__ first_bad) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t total = b.rows * b.row;
  for (uint64_t o = 4 * t; o < min(total, 4 * t + 4); ++o) {
    const uint64_t i = o / b.row;
    const uint32_t c = static_cast<uint32_t>(o - i * b.row);
    if (c < b.cbytes) {
      uint32_t code, j;
      if (b.wide) {
        if (c & 1u) continue;
        code = static_cast<uint32_t>(body[o]) | (static_cast<uint32_t>(body[o + 1]) << 8);
        j = c >> 1;
      } else {
        code = body[o];
        j = c;
      }
      // host encoding of the position: i*row + section (centers first)
      if (code >= b.k) atomicMin(first_bad, static_cast<unsigned long long>(i * b.row + j));
    } else if (b.scales && c < b.cbytes + b.m) {
      if (body[o] >= b.scales) atomicMin(first_bad, static_cast<unsigned long long>(i * b.row + c));
    }
  }
}

// I3: every alpha of rows [begin, end) round-trips through fp16 exactly?
__global__ void ingest_fp16_kernel(const uint8_t* __restrict__ body, BodyDesc b, uint64_t begin,
                                   uint64_t cnt, uint32_t* __restrict__ ok) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= cnt * b.m) return;
  const uint64_t i = begin + t / b.m;
  const uint32_t j = static_cast<uint32_t>(t % b.m);
  const uint8_t* p = body + i * b.row + b.cbytes + 4ull * j;
  const uint32_t u = static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
                     (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
  const float f = __uint_as_float(u);
  if (__float_as_uint(__half2float(__float2half_rn(f))) != u) atomicAnd(ok, 0u);
}

// I4: one warp per block of 32 points; rows staged in shared memory
__global__ void __launch_bounds__(128)
    ingest_repack_kernel(const uint8_t* __restrict__ body, BodyDesc b, uint64_t begin, uint64_t n_local,
                         uint32_t format, uint32_t cw, uint32_t sw, uint32_t W, uint32_t Wc,
                         uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t s_rows[];  // 4 warps x 32 rows
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint64_t blk = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
  const uint64_t nblk = (n_local + 31) / 32;
  if (blk >= nblk) return;
  uint8_t* rows = s_rows + static_cast<size_t>(warp) * 32 * b.row;
  const uint64_t p0 = blk * 32;
  const uint32_t np = n_local - p0 < 32 ? static_cast<uint32_t>(n_local - p0) : 32u;
  const uint8_t* src = body + (begin + p0) * b.row;
  for (uint32_t x = lane; x < np * b.row; x += 32) rows[x] = src[x];  // contiguous, coalesced
  __syncwarp();
  const uint8_t* pr = rows + static_cast<size_t>(lane) * b.row;
  const bool live = lane < np;
  auto center = [&](uint32_t j) -> uint32_t {
    return b.wide ? (static_cast<uint32_t>(pr[2 * j]) | (static_cast<uint32_t>(pr[2 * j + 1]) << 8)) : pr[j];
  };
  auto rd32 = [&](uint32_t off) -> uint32_t {
    return static_cast<uint32_t>(pr[off]) | (static_cast<uint32_t>(pr[off + 1]) << 8) |
           (static_cast<uint32_t>(pr[off + 2]) << 16) | (static_cast<uint32_t>(pr[off + 3]) << 24);
  };
  for (uint32_t w = 0; w < W; ++w) {
    uint32_t word = 0;
    if (live) {
      if (format == PCPQG_FMT_JOINT8) {
        for (uint32_t q = 0; q < 4; ++q) {
          const uint32_t j = 4 * w + q;
          if (j >= b.m) break;
          const uint32_t l = b.scales ? pr[b.cbytes + j] : 0u;
          word |= (center(j) | (l << cw)) << (8 * q);
        }
      } else if (w < Wc) {
        // center plane: sections whose cw-bit field starts in word w
        const uint32_t per = 32 / cw;
        for (uint32_t q = 0; q < per; ++q) {
          const uint32_t j = w * per + q;
          if (j >= b.m) break;
          word |= center(j) << (q * cw);
        }
      } else {
        const uint32_t per = 32 / sw;
        for (uint32_t q = 0; q < per; ++q) {
          const uint32_t j = (w - Wc) * per + q;
          if (j >= b.m) break;
          uint32_t v;
          if (sw == 4 || sw == 8) v = pr[b.cbytes + j];
          else if (sw == 16) v = __half_as_ushort(__float2half_rn(__uint_as_float(rd32(b.cbytes + 4 * j))));
          else v = rd32(b.cbytes + 4 * j);
          word |= v << (q * sw);
        }
      }
    }
    out[(blk * W + w) * 32 + lane] = word;
  }
}

// pinned double-buffered host -> device copy of `len` bytes; `read(dst, off,
// n)` fills a host staging buffer (a memcpy from the caller's image, or a
// file read)
template <class Read>
void stream_to_device(uint8_t* dst, uint64_t len, Read read, cudaStream_t st) {
  const uint64_t chunk = 64ull << 20;
  uint8_t* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  PCPQG_CUDA(cudaMallocHost(&stage[0], chunk));
  PCPQG_CUDA(cudaMallocHost(&stage[1], chunk));
  PCPQG_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  PCPQG_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  struct Free {
    uint8_t** s;
    cudaEvent_t* e;
    ~Free() {
      cudaFreeHost(s[0]);
      cudaFreeHost(s[1]);
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } guard{stage, done};
  bool used[2] = {false, false};
  int i = 0;
  for (uint64_t off = 0; off < len; off += chunk, i ^= 1) {
    const uint64_t n = std::min(chunk, len - off);
    if (used[i]) PCPQG_CUDA(cudaEventSynchronize(done[i]));  // the buffer's previous copy is done
    read(stage[i], off, n);
    PCPQG_CUDA(cudaMemcpyAsync(dst + off, stage[i], n, cudaMemcpyHostToDevice, st));
    PCPQG_CUDA(cudaEventRecord(done[i], st));
    used[i] = true;
  }
  PCPQG_CUDA(cudaStreamSynchronize(st));
}

// Ingest with the header already parsed; `read_body(dst, off, n)` supplies
// body bytes [off, off + n) of the complete rows.
template <class Read>
DeviceIndex* ingest(ParsedIndex& P, uint64_t len, const uint8_t* tail, int device, uint64_t begin,
                    uint64_t end, Read read_body) {
  const HostIndex& H = P.h;
  const uint64_t n = H.n, m = H.m;
  const uint64_t full = full_rows_of(P, len);
  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev};
  cudaStream_t st;
  PCPQG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  const uint64_t body_bytes = full * P.row;
  uint8_t* d_body = nullptr;
  PCPQG_CUDA(cudaMalloc(&d_body, std::max<uint64_t>(body_bytes, 16)));
  struct BodyFree {
    uint8_t* p;
    ~BodyFree() { cudaFree(p); }
  } bf{d_body};
  stream_to_device(d_body, body_bytes, read_body, st);
  BodyDesc b{full, static_cast<uint32_t>(P.row), static_cast<uint32_t>(P.cbytes), static_cast<uint32_t>(m),
             H.k, H.scales, P.wide};
  unsigned long long* d_flags = nullptr;  // [0] first bad position, [1] fp16 ok
  PCPQG_CUDA(cudaMalloc(&d_flags, 16));
  struct FlagFree {
    unsigned long long* p;
    ~FlagFree() { cudaFree(p); }
  } ff{d_flags};
  const unsigned long long init[2] = {~0ull, 1ull};
  PCPQG_CUDA(cudaMemcpyAsync(d_flags, init, 16, cudaMemcpyHostToDevice, st));
  if (body_bytes) {
    const uint64_t threads = (body_bytes + 3) / 4;
    ingest_validate_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(d_body, b, d_flags);
    PCPQG_CUDA(cudaGetLastError());
  }
  unsigned long long first_bad = ~0ull;
  PCPQG_CUDA(cudaMemcpyAsync(&first_bad, d_flags, 8, cudaMemcpyDeviceToHost, st));
  PCPQG_CUDA(cudaStreamSynchronize(st));
  if (first_bad != ~0ull) fail_bad_code(P, first_bad);
  check_tail(P, len, tail);  // partial row / truncation / trailing bytes, host side

  if (end == 0 || end > n) end = n;
  if (begin >= end) fail(PCPQG_E_USAGE, "empty shard range");
  if (n > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "more than 2^31-1 points");
  auto x = std::make_unique<DeviceIndex>();
  x->device = device;
  x->shard_begin = begin;
  x->n_local = end - begin;
  x->n_blocks = static_cast<uint32_t>((x->n_local + kBlockPts - 1) / kBlockPts);
  bool fp16 = false;
  if (H.scales == 0) {
    uint32_t* ok = reinterpret_cast<uint32_t*>(d_flags + 1);
    const uint64_t cnt = x->n_local * m;
    ingest_fp16_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(d_body, b, begin, x->n_local, ok);
    PCPQG_CUDA(cudaGetLastError());
    uint32_t h = 0;
    PCPQG_CUDA(cudaMemcpyAsync(&h, ok, 4, cudaMemcpyDeviceToHost, st));
    PCPQG_CUDA(cudaStreamSynchronize(st));
    fp16 = h != 0;
  }
  const CodeLayout L = choose_layout(H.k, H.scales, H.m, fp16);
  x->format = L.format;
  x->cw = L.cw;
  x->sw = L.sw;
  x->W = L.W;
  x->Wc = L.Wc;
  x->code_bytes = static_cast<uint64_t>(x->n_blocks) * x->W * kBlockPts * 4;
  PCPQG_CUDA(cudaMalloc(&x->d_codes, std::max<uint64_t>(x->code_bytes, 128)));
  const size_t smem = 4ull * 32 * P.row;
  if (smem > 200 * 1024) fail(PCPQG_E_UNSUPPORTED, "GPU ingest: code rows too long");
  PCPQG_CUDA(cudaFuncSetAttribute(ingest_repack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::max<size_t>(smem, 16))));
  const uint64_t ctas = (x->n_blocks + 3) / 4;
  ingest_repack_kernel<<<static_cast<unsigned>(ctas), 128, smem, st>>>(d_body, b, begin, x->n_local, L.format,
                                                                      L.cw, L.sw, L.W, L.Wc, x->d_codes);
  PCPQG_CUDA(cudaGetLastError());
  const uint64_t ncb = m * H.k * H.dbar;
  PCPQG_CUDA(cudaMalloc(&x->d_codebooks, std::max<uint64_t>(ncb, 1) * 4));
  PCPQG_CUDA(cudaMemcpyAsync(x->d_codebooks, H.codebooks.data(), ncb * 4, cudaMemcpyHostToDevice, st));
  const uint64_t m8 = (m + 7) & ~7ull;
  std::vector<float> lam(m8 * std::max(H.scales, 1u), 1.0f);
  if (H.scales) std::copy(H.scalar_cb.begin(), H.scalar_cb.end(), lam.begin());
  PCPQG_CUDA(cudaMalloc(&x->d_lambda, lam.size() * 4));
  PCPQG_CUDA(cudaMemcpyAsync(x->d_lambda, lam.data(), lam.size() * 4, cudaMemcpyHostToDevice, st));
  PCPQG_CUDA(cudaStreamSynchronize(st));
  x->h = std::move(P.h);
  return x.release();
}

}  // namespace

DeviceIndex* load_index_gpu(const uint8_t* bytes, uint64_t len, int device, uint64_t begin, uint64_t end) {
  ParsedIndex P = parse_header(bytes, len);
  const uint8_t* body = P.body;
  const uint8_t* tail = body + full_rows_of(P, len) * P.row;
  // staging copy split over host threads (one thread copies ~10 GB/s; the
  // PCIe copy of the previous chunk runs meanwhile)
  const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  return ingest(P, len, tail, device, begin, end, [&](uint8_t* dst, uint64_t off, uint64_t n) {
    if (n < (8u << 20) || nt == 1) {
      std::memcpy(dst, body + off, n);
      return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
      const uint64_t a = n * t / nt, b = n * (t + 1) / nt;
      th.emplace_back([=] { std::memcpy(dst + a, body + off + a, b - a); });
    }
    for (auto& x : th) x.join();
  });
}

DeviceIndex* load_index_file_gpu(const char* path, int device, uint64_t begin, uint64_t end) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) fail(PCPQG_E_DATA, std::string("cannot open: ") + path);
  const uint64_t len = static_cast<uint64_t>(in.tellg());
  // header + codebooks: read a prefix, growing it until the header parses
  // (parse_header reports truncation only when the prefix is the whole file)
  std::vector<uint8_t> head(std::min<uint64_t>(len, 1 << 20));
  ParsedIndex P;
  for (;;) {
    in.seekg(0);
    if (!head.empty() &&
        !in.read(reinterpret_cast<char*>(head.data()), static_cast<std::streamsize>(head.size())))
      fail(PCPQG_E_DATA, std::string("read failed: ") + path);
    try {
      P = parse_header(head.data(), head.size());
      break;
    } catch (const Error& e) {
      if (e.code != PCPQG_E_TRUNCATED || head.size() == len) throw;
      head.resize(std::min<uint64_t>(len, head.size() * 4));
    }
  }
  const uint64_t body_off = static_cast<uint64_t>(P.body - P.bytes);
  const uint64_t full = full_rows_of(P, len);
  const uint64_t tail_off = body_off + full * P.row;
  std::vector<uint8_t> tail(len - tail_off + 1);
  in.seekg(static_cast<std::streamoff>(tail_off));
  if (len > tail_off &&
      !in.read(reinterpret_cast<char*>(tail.data()), static_cast<std::streamsize>(len - tail_off)))
    fail(PCPQG_E_DATA, std::string("read failed: ") + path);
  in.clear();
  return ingest(P, len, tail.data(), device, begin, end, [&](uint8_t* dst, uint64_t off, uint64_t n) {
    in.seekg(static_cast<std::streamoff>(body_off + off));
    if (!in.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(n)))
      fail(PCPQG_E_DATA, std::string("read failed: ") + path);
  });
}

}  // namespace pcpqg
