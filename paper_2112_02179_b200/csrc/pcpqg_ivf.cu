// IVF query path: the two-level index of
// proj/core/include/pcpq/ivf.hpp — a coarse partition of the points and, per
// cell, a PQ index over the residuals x - c (or the raw residuals for cells
// with < 2 members) — queried as query_ivf does (proj/core/src/ivf.cpp:89-153):
//
//   K_c  coarse scores  cs[b][r] = <q_b, c_r> in double, sequential over d
//        (dotf, ivf.cpp:18-23; every product of two floats is exact in double)
//   K_o  probe order    stable descending sort of cs[b][.] (ivf.cpp:104-108):
//        CUB segmented radix sort (stable) of order-preserving 64-bit keys,
//        -0 folded onto +0 so that equal scores keep ascending r
//   K_p  pool offsets   probe p of query b owns pool[off[b][p], +|cell|) — the
//        reference's pool order (probe order, member order, ivf.cpp:113-132)
//   K_s  cell scoring   one CTA per (query, probe, chunk of the cell): the
//        cell's eta table in shared memory (the fixed-order fp32 LUT of
//        pq_index.cpp:186-190 over the cell's own codebooks), then every
//        member's score_all value in the same fp32 order as the flat scan
//        (score_point), combined as coarse + double(sub) (ivf.cpp:130); raw
//        cells score coarse + dotf(q, residual) (ivf.cpp:122-124)
//   K_t  top-n          one CTA per query: exact radix select of the keep-th
//        best (score desc, id asc) over 96-bit keys (ivf.cpp:139-146), then a
//        bitonic sort of the survivors
//   K_r  requested ids  pool lookup through point_cluster / point_slot
//        (ivf.cpp:134-137); NaN when the id's cell was not probed
//
// Every cell's codes live in one blocked stream with a common layout chosen
// from the largest cell k (codes of a cell with a lowered k are smaller, so
// they fit), codebooks and scale codebooks concatenated per cell.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>

#include "pcpqg_internal.hpp"
#include "pcpqg_scan.cuh"

namespace pcpqg {

DeviceIvf::~DeviceIvf() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (void* p : {static_cast<void*>(d_coarse), static_cast<void*>(d_cells),
                  static_cast<void*>(d_codes), static_cast<void*>(d_cb), static_cast<void*>(d_lam),
                  static_cast<void*>(d_raw), static_cast<void*>(d_members),
                  static_cast<void*>(d_pcluster), static_cast<void*>(d_pslot)})
    if (p) cudaFree(p);
  cudaSetDevice(prev);
}

namespace {

// The reference's container Reader (ivf.cpp:186-226): every short read is
// `truncated`.
struct IvfReader {
  const uint8_t* p;
  uint64_t len, pos = 0;
  void need(uint64_t n) const {
    if (pos + n > len) fail(PCPQG_E_TRUNCATED, "container truncated at byte " + std::to_string(pos));
  }
  uint32_t u32() {
    need(4);
    const uint8_t* b = p + pos;
    pos += 4;
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
  }
  uint64_t u64() {
    const uint64_t lo = u32(), hi = u32();
    return lo | (hi << 32);
  }
};

template <class T>
T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  PCPQG_CUDA(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (!v.empty()) PCPQG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

DeviceIvf* load_ivf(const uint8_t* bytes, uint64_t len, int device) {
  IvfReader r{bytes, len};
  r.need(8);
  if (std::memcmp(bytes, "PCPQIVF1", 8) != 0) fail(PCPQG_E_BAD_MAGIC, "not a container file");
  r.pos = 8;
  const uint32_t version = r.u32();
  if (version != 1)
    fail(PCPQG_E_BAD_VERSION, "unsupported container version " + std::to_string(version));
  auto v = std::make_unique<DeviceIvf>();
  v->device = device;
  v->n = r.u32();
  v->d = r.u32();
  v->kbar = r.u32();
  if (v->n == 0 || v->d == 0 || v->kbar == 0 || v->kbar > v->n)
    fail(PCPQG_E_DATA, "bad container header");
  const uint32_t kbar = v->kbar, d = v->d;
  const uint64_t kd = static_cast<uint64_t>(kbar) * d;
  r.need(4 * kd);
  std::vector<float> coarse(kd);
  std::memcpy(coarse.data(), bytes + r.pos, 4 * kd);
  r.pos += 4 * kd;
  std::vector<uint64_t> moff(kbar + 1, 0);
  std::vector<uint32_t> members;
  for (uint32_t c = 0; c < kbar; ++c) {
    const uint32_t count = r.u32();
    if (count > v->n) fail(PCPQG_E_DATA, "member count exceeds n");
    r.need(4ull * count);
    const size_t at = members.size();
    members.resize(at + count);
    std::memcpy(members.data() + at, bytes + r.pos, 4ull * count);
    r.pos += 4ull * count;
    moff[c + 1] = members.size();
  }
  // blobs: a PCPQIDX1 image (validated like pcpq::deserialize) or a raw block
  std::vector<ParsedIndex> parsed(kbar);
  std::vector<uint8_t> is_raw(kbar, 0);
  std::vector<std::pair<uint64_t, uint64_t>> raw_span(kbar, {0, 0});  // (byte offset, floats)
  for (uint32_t c = 0; c < kbar; ++c) {
    const uint64_t blen = r.u64();
    r.need(blen);
    const uint8_t* blob = bytes + r.pos;
    r.pos += blen;
    const uint64_t count = moff[c + 1] - moff[c];
    if (blen >= 8 && std::memcmp(blob, "PCPQRAW1", 8) == 0) {
      IvfReader br{blob, blen, 8};
      const uint32_t bc = br.u32();
      const uint32_t dim = br.u32();
      if (dim != d) fail(PCPQG_E_DATA, "raw block dimension mismatch");
      if (bc != count) fail(PCPQG_E_SIZE_MISMATCH, "raw block count mismatch");
      const uint64_t nf = static_cast<uint64_t>(bc) * dim;
      br.need(4 * nf);
      if (br.pos + 4 * nf != blen) fail(PCPQG_E_SIZE_MISMATCH, "trailing bytes in raw block");
      is_raw[c] = 1;
      raw_span[c] = {static_cast<uint64_t>(blob - bytes) + br.pos, nf};
    } else {
      parsed[c] = parse_index(blob, blen);
      if (parsed[c].h.n != count)
        fail(PCPQG_E_SIZE_MISMATCH, "sub-index size does not match member list");
      if (parsed[c].h.d != d) fail(PCPQG_E_DATA, "sub-index dimension mismatch");
    }
  }
  if (r.pos != len)
    fail(PCPQG_E_SIZE_MISMATCH, "trailing bytes after container at byte " + std::to_string(r.pos));
  // rebuild_point_maps (ivf.cpp:28-43)
  std::vector<uint32_t> pcluster(v->n, 0), pslot(v->n, 0);
  {
    std::vector<uint8_t> seen(v->n, 0);
    for (uint32_t c = 0; c < kbar; ++c)
      for (uint64_t pos = moff[c]; pos < moff[c + 1]; ++pos) {
        const uint32_t id = members[pos];
        if (id >= v->n || seen[id]) fail(PCPQG_E_DATA, "member lists do not partition the ids");
        seen[id] = 1;
        pcluster[id] = c;
        pslot[id] = static_cast<uint32_t>(pos - moff[c]);
      }
    for (uint8_t s : seen)
      if (!s) fail(PCPQG_E_DATA, "member lists do not partition the ids");
  }

  // ---- common layout of the PQ cells
  bool first = true, fp16 = true;
  for (uint32_t c = 0; c < kbar; ++c) {
    if (is_raw[c]) {
      ++v->n_raw;
      continue;
    }
    const HostIndex& h = parsed[c].h;
    if (first) {
      v->m = h.m;
      v->padded_d = h.padded_d;
      v->dbar = h.dbar;
      v->scales = h.scales;
      v->method = h.method;
      first = false;
    } else if (h.m != v->m || h.padded_d != v->padded_d || h.scales != v->scales) {
      fail(PCPQG_E_UNSUPPORTED, "IVF cells with different m / padded_d / scale counts");
    }
    v->k_max = std::max(v->k_max, h.k);
    ++v->n_pq;
    if (h.scales == 0 && fp16) fp16 = alphas_fp16_exact(parsed[c], 0, h.n);
  }
  if (v->n_pq) v->lay = choose_layout(v->k_max, v->scales, v->m, fp16);
  const uint32_t m8 = (v->m + 7) & ~7u;
  const uint32_t s1 = std::max(v->scales, 1u);
  std::vector<IvfCell> cells(kbar);
  uint64_t blocks = 0, cbf = 0, rawf = 0;
  uint32_t pq_i = 0;
  v->cell_n.resize(kbar);
  v->cell_k.assign(kbar, 0);
  for (uint32_t c = 0; c < kbar; ++c) {
    IvfCell& e = cells[c];
    e.n = static_cast<uint32_t>(moff[c + 1] - moff[c]);
    e.member_off = moff[c];
    v->cell_n[c] = e.n;
    if (is_raw[c]) {
      e.raw = 1;
      e.raw_off = rawf;
      rawf += raw_span[c].second;
      v->max_raw_pts = std::max(v->max_raw_pts, e.n);
    } else {
      e.k = parsed[c].h.k;
      v->cell_k[c] = e.k;
      e.block_off = blocks;
      const uint64_t nb = (e.n + kBlockPts - 1) / kBlockPts;
      blocks += nb;
      v->max_cell_blocks = std::max<uint64_t>(v->max_cell_blocks, nb);
      e.cb_off = cbf;
      cbf += static_cast<uint64_t>(v->m) * e.k * v->dbar;
      e.lam_off = static_cast<uint64_t>(pq_i) * m8 * s1;
      ++pq_i;
    }
  }
  std::vector<uint32_t> codes(blocks * v->lay.W * kBlockPts, 0u);
  std::vector<float> cb(cbf), lam(static_cast<uint64_t>(pq_i) * m8 * s1, 1.0f), raw(rawf);
  for (uint32_t c = 0; c < kbar; ++c) {
    const IvfCell& e = cells[c];
    if (e.raw) {
      std::memcpy(raw.data() + e.raw_off, bytes + raw_span[c].first, 4 * raw_span[c].second);
      continue;
    }
    const ParsedIndex& P = parsed[c];
    repack(P, v->lay, 0, e.n, codes.data() + e.block_off * v->lay.W * kBlockPts);
    std::copy(P.h.codebooks.begin(), P.h.codebooks.end(), cb.begin() + e.cb_off);
    std::copy(P.h.scalar_cb.begin(), P.h.scalar_cb.end(), lam.begin() + e.lam_off);
  }
  // sum of the p largest cells: the pool size bound for p probes
  std::vector<uint32_t> sz = v->cell_n;
  std::sort(sz.begin(), sz.end(), std::greater<uint32_t>());
  v->top_prefix.assign(kbar + 1, 0);
  for (uint32_t i = 0; i < kbar; ++i) v->top_prefix[i + 1] = v->top_prefix[i] + sz[i];

  int prev = 0;
  PCPQG_CUDA(cudaGetDevice(&prev));
  PCPQG_CUDA(cudaSetDevice(device));
  v->code_bytes = codes.size() * 4;
  v->d_coarse = upload(coarse);
  v->d_cells = upload(cells);
  v->d_codes = upload(codes);
  v->d_cb = upload(cb);
  v->d_lam = upload(lam);
  v->d_raw = upload(raw);
  v->d_members = upload(members);
  v->d_pcluster = upload(pcluster);
  v->d_pslot = upload(pslot);
  PCPQG_CUDA(cudaSetDevice(prev));
  return v.release();
}

namespace {

// order-preserving image of a double, -0 folded onto +0 (they compare equal)
__device__ __forceinline__ uint64_t ord64(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  if ((b << 1) == 0ull) b = 0ull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// K_c: cs[b][r] = sum_a double(q[a]) * double(c_r[a]) in index order
__global__ void ivf_coarse_kernel(const float* __restrict__ Q, uint32_t B, uint32_t d,
                                  const float* __restrict__ C, uint32_t kbar,
                                  double* __restrict__ cs, uint64_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(B) * kbar) return;
  const uint32_t b = static_cast<uint32_t>(t / kbar), r = static_cast<uint32_t>(t % kbar);
  const float* q = Q + static_cast<uint64_t>(b) * d;
  const float* c = C + static_cast<uint64_t>(r) * d;
  double acc = 0.0;
  for (uint32_t a = 0; a < d; ++a)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(__ldg(q + a)), static_cast<double>(__ldg(c + a))));
  cs[t] = acc;
  keys[t] = ord64(acc);
  vals[t] = r;
}

__global__ void ivf_seg_offsets_kernel(uint32_t B, uint32_t kbar, int* off) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= B) off[t] = static_cast<int>(t * kbar);
}

// K_p: probes[b][p], probe position of every cell (-1 = not probed), pool
// offsets (exclusive scan of the probed cell sizes) and pool sizes
__global__ void __launch_bounds__(256)
    ivf_probe_kernel(const uint32_t* __restrict__ sorted_r, uint32_t kbar, uint32_t kp,
                     const IvfCell* __restrict__ cells, uint32_t* __restrict__ probes,
                     int32_t* __restrict__ probe_pos, uint64_t* __restrict__ pool_off,
                     uint64_t* __restrict__ pool_n) {
  using Scan = cub::BlockScan<uint64_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t carry;
  const uint32_t b = blockIdx.x;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t p0 = 0; p0 < kp; p0 += 256) {
    const uint32_t p = p0 + threadIdx.x;
    uint32_t r = 0;
    uint64_t sz = 0;
    if (p < kp) {
      r = sorted_r[static_cast<uint64_t>(b) * kbar + p];
      sz = cells[r].n;
      probes[static_cast<uint64_t>(b) * kp + p] = r;
      probe_pos[static_cast<uint64_t>(b) * kbar + r] = static_cast<int32_t>(p);
    }
    uint64_t excl, total;
    Scan(tmp).ExclusiveSum(sz, excl, total);
    if (p < kp) pool_off[static_cast<uint64_t>(b) * kp + p] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) pool_n[b] = carry;
}

struct IvfScoreArgs {
  const float* Q;
  uint32_t d, kbar, kp, chunk_pts;
  const double* cs;
  const uint32_t* probes;
  const uint64_t* pool_off;
  const IvfCell* cells;
  const uint32_t* codes;
  const float* cb;
  const float* lam;
  const float* raw;
  const uint32_t* members;
  uint32_t m, m8, dbar, k_max, s, cbits, W, Wc;
  uint64_t pool_stride;
  double* poolD;
  uint32_t* poolI;
};

// K_s: one CTA per (query, probe, chunk of the cell's members)
template <int CW, int SW>
__global__ void __launch_bounds__(256) ivf_score_kernel(const IvfScoreArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t b = blockIdx.x / a.kp, p = blockIdx.x % a.kp;
  const uint32_t r = a.probes[static_cast<uint64_t>(b) * a.kp + p];
  const IvfCell cell = a.cells[r];
  const uint32_t pos0 = blockIdx.y * a.chunk_pts;
  if (pos0 >= cell.n) return;
  const uint32_t pos1 = min(cell.n, pos0 + a.chunk_pts);
  const double coarse = a.cs[static_cast<uint64_t>(b) * a.kbar + r];
  const float* q = a.Q + static_cast<uint64_t>(b) * a.d;
  const uint64_t out0 = static_cast<uint64_t>(b) * a.pool_stride +
                        a.pool_off[static_cast<uint64_t>(b) * a.kp + p];
  if (cell.raw) {
    // coarse + dotf(q, residual row) (ivf.cpp:122-124)
    for (uint32_t pos = pos0 + threadIdx.x; pos < pos1; pos += blockDim.x) {
      const float* x = a.raw + cell.raw_off + static_cast<uint64_t>(pos) * a.d;
      double acc = 0.0;
      for (uint32_t i = 0; i < a.d; ++i)
        acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(__ldg(q + i)), static_cast<double>(__ldg(x + i))));
      a.poolD[out0 + pos] = __dadd_rn(coarse, acc);
      a.poolI[out0 + pos] = a.members[cell.member_off + pos];
    }
    return;
  }
  using Cd = Codec<CW, SW>;
  float* s_eta = reinterpret_cast<float*>(smem);  // [m8][k_max], RS = 1
  float* s_lam = s_eta + static_cast<size_t>(a.m8) * a.k_max;
  // the cell's eta table: fixed-order fp32 dot from 0.0f (pq_index.cpp:186-190)
  const float* cbr = a.cb + cell.cb_off;
  for (uint32_t t = threadIdx.x; t < a.m8 * a.k_max; t += blockDim.x) {
    const uint32_t j = t / a.k_max, c = t % a.k_max;
    float acc = 0.0f;
    if (j >= a.m) {
      acc = -0.0f;
    } else if (c < cell.k) {
      const float* row = cbr + (static_cast<uint64_t>(j) * cell.k + c) * a.dbar;
      for (uint32_t i = 0; i < a.dbar; ++i) {
        const uint32_t col = j * a.dbar + i;
        const float qa = col < a.d ? __ldg(q + col) : 0.0f;  // pad_vector (types.cpp:83-88)
        acc = __fadd_rn(acc, __fmul_rn(__ldg(row + i), qa));
      }
    }
    s_eta[t] = acc;
  }
  if constexpr (!Cd::kNoLambda)
    for (uint32_t t = threadIdx.x; t < a.m8 * a.s; t += blockDim.x) s_lam[t] = __ldg(a.lam + cell.lam_off + t);
  __syncthreads();
  const uint32_t eta_sa = static_cast<uint32_t>(__cvta_generic_to_shared(s_eta));
  for (uint32_t pos = pos0 + threadIdx.x; pos < pos1; pos += blockDim.x) {
    const uint64_t blk = cell.block_off + pos / kBlockPts;
    const uint32_t* wp = a.codes + blk * a.W * kBlockPts + (pos % kBlockPts);
    float acc[1][1];
    score_point<1, CW, SW, 0, 1>(wp, 0, eta_sa, s_eta, s_lam, a.k_max, a.s, a.cbits, a.W, a.Wc, a.m,
                                 acc);
    a.poolD[out0 + pos] = __dadd_rn(coarse, static_cast<double>(acc[0][0]));  // ivf.cpp:130
    a.poolI[out0 + pos] = a.members[cell.member_off + pos];
  }
}

// K_t: exact top-n of each query's pool by (score desc, id asc) over the
// 96-bit keys (ord64(score), ~id): MSB-first radix select (8-bit digits,
// stops when the selected bin holds exactly the keys still needed), gather,
// bitonic sort.
constexpr uint32_t kIvfMaxTop = 8192;

__global__ void __launch_bounds__(1024)
    ivf_select_kernel(const double* __restrict__ poolD, const uint32_t* __restrict__ poolI,
                      uint64_t stride, const uint64_t* __restrict__ pool_n, uint32_t topn,
                      int32_t* __restrict__ ids, double* __restrict__ scores,
                      uint32_t* __restrict__ counts, uint8_t* __restrict__ shorts) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_phi, s_mhi;
  __shared__ uint32_t s_plo, s_mlo, s_need, s_cnt, s_done, s_n;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t n = pool_n[b];
  const uint32_t keep = static_cast<uint32_t>(n < topn ? n : static_cast<uint64_t>(topn));
  const double* D = poolD + static_cast<uint64_t>(b) * stride;
  const uint32_t* I = poolI + static_cast<uint64_t>(b) * stride;
  if (tid == 0) {
    counts[b] = keep;
    shorts[b] = n < topn ? 1 : 0;
    s_phi = 0;
    s_mhi = 0;
    s_plo = 0;
    s_mlo = 0;
    s_need = keep;
    s_done = keep == n ? 1u : 0u;  // everything is selected
    s_n = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 12 && !s_done; ++pass) {
    for (uint32_t i = tid; i < 256; i += nthr) hist[i] = 0;
    __syncthreads();
    const uint64_t phi = s_phi, mhi = s_mhi;
    const uint32_t plo = s_plo, mlo = s_mlo;
    for (uint64_t i = tid; i < n; i += nthr) {
      const uint64_t hi = ord64(D[i]);
      const uint32_t lo = ~I[i];
      if ((hi & mhi) == phi && (lo & mlo) == plo) {
        const uint32_t dg = pass < 8 ? static_cast<uint32_t>(hi >> (56 - 8 * pass)) & 0xFFu
                                     : (lo >> (24 - 8 * (pass - 8))) & 0xFFu;
        atomicAdd(&hist[dg], 1u);
      }
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t need = s_need, cum = 0;
      int sel = 255;
      for (; sel >= 0; --sel) {
        if (cum + hist[sel] >= need) break;
        cum += hist[sel];
      }
      const uint32_t cnt = hist[sel];
      s_need = need - cum;
      if (pass < 8) {
        s_phi |= static_cast<uint64_t>(sel) << (56 - 8 * pass);
        s_mhi |= 0xFFull << (56 - 8 * pass);
      } else {
        s_plo |= static_cast<uint32_t>(sel) << (24 - 8 * (pass - 8));
        s_mlo |= 0xFFu << (24 - 8 * (pass - 8));
      }
      if (cnt == s_need) s_done = 1;
    }
    __syncthreads();
  }
  // gather: keys whose masked prefix is above (or equal to) the selected one
  uint64_t* k_hi = reinterpret_cast<uint64_t*>(smem);
  uint32_t* k_id = reinterpret_cast<uint32_t*>(k_hi + kIvfMaxTop);
  uint32_t* k_ix = k_id + kIvfMaxTop;
  {
    const uint64_t phi = s_phi, mhi = s_mhi;
    const uint32_t plo = s_plo, mlo = s_mlo;
    for (uint64_t i = tid; i < n; i += nthr) {
      const uint64_t hi = ord64(D[i]);
      const uint32_t id = I[i];
      const uint64_t mh = hi & mhi;
      const uint32_t ml = ~id & mlo;
      if (mh > phi || (mh == phi && ml >= plo)) {
        const uint32_t slot = atomicAdd(&s_n, 1u);
        if (slot < keep) {
          k_hi[slot] = hi;
          k_id[slot] = id;
          k_ix[slot] = static_cast<uint32_t>(i);
        }
      }
    }
  }
  __syncthreads();
  uint32_t P = 1;
  while (P < keep) P <<= 1;
  for (uint32_t i = keep + tid; i < P; i += nthr) {
    k_hi[i] = 0ull;
    k_id[i] = 0xFFFFFFFFu;
    k_ix[i] = 0u;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
      for (uint32_t i = tid; i < P / 2; i += nthr) {
        const uint32_t lo = 2 * stride2 * (i / stride2) + (i % stride2);
        const uint32_t hi = lo + stride2;
        // "better" = score desc, id asc
        const bool hi_better = k_hi[hi] > k_hi[lo] || (k_hi[hi] == k_hi[lo] && k_id[hi] < k_id[lo]);
        if (hi_better == ((lo & size) == 0)) {
          const uint64_t th = k_hi[lo];
          k_hi[lo] = k_hi[hi];
          k_hi[hi] = th;
          const uint32_t ti = k_id[lo];
          k_id[lo] = k_id[hi];
          k_id[hi] = ti;
          const uint32_t tx = k_ix[lo];
          k_ix[lo] = k_ix[hi];
          k_ix[hi] = tx;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = tid; i < topn; i += nthr) {
    const uint64_t o = static_cast<uint64_t>(b) * topn + i;
    ids[o] = i < keep ? static_cast<int32_t>(k_id[i]) : -1;
    scores[o] = i < keep ? D[k_ix[i]] : __longlong_as_double(0x7FF8000000000000ll);
  }
}

// K_r: requested ids (ivf.cpp:134-137)
__global__ void ivf_requested_kernel(const uint32_t* __restrict__ req, uint32_t B, uint32_t R,
                                     uint32_t kbar, uint32_t kp, const uint32_t* __restrict__ pcluster,
                                     const uint32_t* __restrict__ pslot,
                                     const int32_t* __restrict__ probe_pos,
                                     const uint64_t* __restrict__ pool_off,
                                     const double* __restrict__ poolD, uint64_t stride,
                                     double* __restrict__ out) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(B) * R) return;
  const uint32_t b = static_cast<uint32_t>(t / R);
  const uint32_t id = req[t];
  const uint32_t r = pcluster[id];
  const int32_t p = probe_pos[static_cast<uint64_t>(b) * kbar + r];
  out[t] = p < 0 ? __longlong_as_double(0x7FF8000000000000ll)
                 : poolD[static_cast<uint64_t>(b) * stride +
                         pool_off[static_cast<uint64_t>(b) * kp + p] + pslot[id]];
}

__global__ void ivf_check_ids_kernel(const uint32_t* __restrict__ req, uint64_t cnt, uint32_t n,
                                     uint32_t* __restrict__ err) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < cnt && req[t] >= n) atomicOr(err, 1u);
}

using IvfScoreFn = void (*)(IvfScoreArgs);

template <int CW>
IvfScoreFn ivf_pick_sw(uint32_t sw) {
  switch (sw) {
    case 0: return ivf_score_kernel<CW, 0>;
    case 4: return ivf_score_kernel<CW, 4>;
    case 8: return ivf_score_kernel<CW, 8>;
    case 16: return ivf_score_kernel<CW, 16>;
    case 32: return ivf_score_kernel<CW, 32>;
  }
  return nullptr;
}

IvfScoreFn ivf_pick(const CodeLayout& L) {
  if (L.format == PCPQG_FMT_JOINT8) return ivf_score_kernel<0, 0>;
  if (L.cw == 4) return ivf_pick_sw<4>(L.sw);
  if (L.cw == 8) return ivf_pick_sw<8>(L.sw);
  if (L.cw == 16) return ivf_pick_sw<16>(L.sw);
  return nullptr;
}

template <class T>
T* salloc(std::vector<void*>& keep, size_t n, cudaStream_t st) {
  void* p = nullptr;
  PCPQG_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
  keep.push_back(p);
  return static_cast<T*>(p);
}

}  // namespace

uint32_t ivf_check_requested(const uint32_t* d_req, uint64_t cnt, uint32_t n, cudaStream_t st) {
  if (cnt == 0) return 0;
  std::vector<void*> keep;
  uint32_t* d_err = salloc<uint32_t>(keep, 1, st);
  PCPQG_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  ivf_check_ids_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(d_req, cnt, n, d_err);
  PCPQG_CUDA(cudaGetLastError());
  uint32_t h = 0;
  PCPQG_CUDA(cudaMemcpyAsync(&h, d_err, 4, cudaMemcpyDeviceToHost, st));
  for (void* p : keep) cudaFreeAsync(p, st);
  PCPQG_CUDA(cudaStreamSynchronize(st));
  return h;
}

void ivf_query(const DeviceIvf& v, const float* dQ, uint32_t B, uint32_t kp, uint32_t topn,
               const uint32_t* d_req, uint32_t R, int32_t* d_ids, double* d_scores,
               uint32_t* d_counts, uint8_t* d_short, double* d_req_scores, uint32_t* d_probes,
               cudaStream_t st) {
  if (B == 0) return;
  if (topn > kIvfMaxTop) fail(PCPQG_E_UNSUPPORTED, "IVF topN above 8192");
  const uint64_t stride = std::max<uint64_t>(v.top_prefix[kp], 1);
  // query chunk so that the pools stay within ~2 GB
  const uint64_t per_q = stride * 12 + static_cast<uint64_t>(v.kbar) * 32;
  const uint32_t chunk = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(B, (2ull << 30) / per_q)));
  const uint32_t s1 = std::max(v.scales, 1u);
  const uint32_t m8 = (v.m + 7) & ~7u;
  IvfScoreFn score_fn = v.n_pq ? ivf_pick(v.lay) : ivf_score_kernel<0, 0>;
  if (!score_fn) fail(PCPQG_E_UNSUPPORTED, "no IVF scoring kernel for this code layout");
  const size_t score_smem = (static_cast<size_t>(m8) * std::max(v.k_max, 1u) + m8 * s1) * 4;
  static const size_t kSelSmem = kIvfMaxTop * 16;
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(score_fn),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::max<size_t>(score_smem, 1))));
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(ivf_select_kernel),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSelSmem)));
  int max_smem = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, v.device));
  if (score_smem > static_cast<size_t>(max_smem))
    fail(PCPQG_E_UNSUPPORTED, "IVF cell eta table does not fit in shared memory");
  // members per scoring CTA: larger for big k (the eta build is per CTA)
  const uint32_t chunk_pts = v.k_max > 64 ? 8192 : 2048;
  const uint32_t max_pts = std::max<uint32_t>(
      static_cast<uint32_t>(std::min<uint64_t>(v.max_cell_blocks * kBlockPts, 0xFFFFFFFFull)),
      v.max_raw_pts);
  const uint32_t nchunks = std::max<uint32_t>(1, (max_pts + chunk_pts - 1) / chunk_pts);
  if (nchunks > 65535) fail(PCPQG_E_UNSUPPORTED, "IVF cell too large");

  for (uint32_t b0 = 0; b0 < B; b0 += chunk) {
    const uint32_t Bc = std::min(chunk, B - b0);
    const uint64_t bk = static_cast<uint64_t>(Bc) * v.kbar;
    std::vector<void*> keep;
    double* cs = salloc<double>(keep, bk, st);
    uint64_t* keys = salloc<uint64_t>(keep, bk, st);
    uint64_t* keys2 = salloc<uint64_t>(keep, bk, st);
    uint32_t* vals = salloc<uint32_t>(keep, bk, st);
    uint32_t* vals2 = salloc<uint32_t>(keep, bk, st);
    int* segoff = salloc<int>(keep, Bc + 1, st);
    uint32_t* probes = d_probes ? d_probes + static_cast<uint64_t>(b0) * kp
                                : salloc<uint32_t>(keep, static_cast<uint64_t>(Bc) * kp, st);
    int32_t* ppos = salloc<int32_t>(keep, bk, st);
    uint64_t* poff = salloc<uint64_t>(keep, static_cast<uint64_t>(Bc) * kp, st);
    uint64_t* pn = salloc<uint64_t>(keep, Bc, st);
    double* poolD = salloc<double>(keep, static_cast<uint64_t>(Bc) * stride, st);
    uint32_t* poolI = salloc<uint32_t>(keep, static_cast<uint64_t>(Bc) * stride, st);
    const float* q = dQ + static_cast<uint64_t>(b0) * v.d;

    ivf_coarse_kernel<<<static_cast<unsigned>((bk + 255) / 256), 256, 0, st>>>(
        q, Bc, v.d, v.d_coarse, v.kbar, cs, keys, vals);
    PCPQG_CUDA(cudaGetLastError());
    ivf_seg_offsets_kernel<<<(Bc + 1 + 255) / 256, 256, 0, st>>>(Bc, v.kbar, segoff);
    PCPQG_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        nullptr, tmp_bytes, keys, keys2, vals, vals2, static_cast<int>(bk), static_cast<int>(Bc), segoff,
        segoff + 1, 0, 64, st));
    void* tmp = salloc<uint8_t>(keep, tmp_bytes, st);
    PCPQG_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        tmp, tmp_bytes, keys, keys2, vals, vals2, static_cast<int>(bk), static_cast<int>(Bc), segoff,
        segoff + 1, 0, 64, st));
    PCPQG_CUDA(cudaMemsetAsync(ppos, 0xFF, bk * sizeof(int32_t), st));
    ivf_probe_kernel<<<Bc, 256, 0, st>>>(vals2, v.kbar, kp, v.d_cells, probes, ppos, poff, pn);
    PCPQG_CUDA(cudaGetLastError());

    IvfScoreArgs a{};
    a.Q = q;
    a.d = v.d;
    a.kbar = v.kbar;
    a.kp = kp;
    a.chunk_pts = chunk_pts;
    a.cs = cs;
    a.probes = probes;
    a.pool_off = poff;
    a.cells = v.d_cells;
    a.codes = v.d_codes;
    a.cb = v.d_cb;
    a.lam = v.d_lam;
    a.raw = v.d_raw;
    a.members = v.d_members;
    a.m = v.m;
    a.m8 = m8;
    a.dbar = v.dbar;
    a.k_max = std::max(v.k_max, 1u);
    a.s = s1;
    a.cbits = v.lay.format == PCPQG_FMT_JOINT8 ? v.lay.cw : 0u;
    a.W = v.lay.W;
    a.Wc = v.lay.Wc;
    a.pool_stride = stride;
    a.poolD = poolD;
    a.poolI = poolI;
    const uint64_t gx = static_cast<uint64_t>(Bc) * kp;
    if (gx > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "IVF batch x probes too large");
    score_fn<<<dim3(static_cast<unsigned>(gx), nchunks), 256, score_smem, st>>>(a);
    PCPQG_CUDA(cudaGetLastError());
    ivf_select_kernel<<<Bc, 1024, kSelSmem, st>>>(
        poolD, poolI, stride, pn, topn, d_ids + static_cast<uint64_t>(b0) * topn,
        d_scores + static_cast<uint64_t>(b0) * topn, d_counts + b0, d_short + b0);
    PCPQG_CUDA(cudaGetLastError());
    if (R && d_req_scores) {
      const uint64_t br = static_cast<uint64_t>(Bc) * R;
      ivf_requested_kernel<<<static_cast<unsigned>((br + 255) / 256), 256, 0, st>>>(
          d_req + static_cast<uint64_t>(b0) * R, Bc, R, v.kbar, kp, v.d_pcluster, v.d_pslot, ppos, poff,
          poolD, stride, d_req_scores + static_cast<uint64_t>(b0) * R);
      PCPQG_CUDA(cudaGetLastError());
    }
    for (void* p : keep) PCPQG_CUDA(cudaFreeAsync(p, st));
  }
}

}  // namespace pcpqg
