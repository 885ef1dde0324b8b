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
#include <cstdlib>

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

// K_o for kbar <= kIvfSortMax: one CTA per query sorts its kbar (key, r)
// pairs in shared memory by (key desc, r asc) — the result of the stable
// descending sort — and writes the cell order.
constexpr uint32_t kIvfSortMax = 4096;

__global__ void __launch_bounds__(1024)
    ivf_order_kernel(const uint64_t* __restrict__ keys, uint32_t kbar, uint32_t* __restrict__ order) {
  __shared__ uint64_t k[kIvfSortMax];
  __shared__ uint32_t v[kIvfSortMax];
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  uint32_t P = 1;
  while (P < kbar) P <<= 1;
  for (uint32_t i = tid; i < P; i += nthr) {
    k[i] = i < kbar ? keys[static_cast<uint64_t>(b) * kbar + i] : 0ull;
    v[i] = i < kbar ? i : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < P / 2; i += nthr) {
        const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
        const uint32_t hi = lo + stride;
        const bool hi_first = k[hi] > k[lo] || (k[hi] == k[lo] && v[hi] < v[lo]);
        if (hi_first == ((lo & size) == 0)) {
          const uint64_t tk = k[lo];
          k[lo] = k[hi];
          k[hi] = tk;
          const uint32_t tv = v[lo];
          v[lo] = v[hi];
          v[hi] = tv;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = tid; i < kbar; i += nthr) order[static_cast<uint64_t>(b) * kbar + i] = v[i];
}

__global__ void ivf_seg_offsets_kernel(uint32_t B, uint32_t kbar, int* off) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= B) off[t] = static_cast<int>(t * kbar);
}

// K_p: probes[b][p], the probe position of every cell (-1 = not probed), the
// probed population pool_n[b] (ivf.cpp:113-132), and the scoring work list:
// probe p of query b is split into ceil(|cell| / chunk) chunks whose
// query-local first index is coff[b][p]; qch[b] = the query's chunk count.
__global__ void __launch_bounds__(256)
    ivf_probe_kernel(const uint32_t* __restrict__ sorted_r, uint32_t kbar, uint32_t kp,
                     const IvfCell* __restrict__ cells, uint32_t chunk_pts,
                     uint32_t* __restrict__ probes, int32_t* __restrict__ probe_pos,
                     uint32_t* __restrict__ coff, uint32_t* __restrict__ qch,
                     uint64_t* __restrict__ pool_n) {
  using Scan = cub::BlockScan<uint32_t, 256>;
  using Red = cub::BlockReduce<uint64_t, 256>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
  } tmp;
  __shared__ uint32_t carry;
  const uint32_t b = blockIdx.x;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  uint64_t pop = 0;
  for (uint32_t p0 = 0; p0 < kp; p0 += 256) {
    const uint32_t p = p0 + threadIdx.x;
    uint32_t nch = 0;
    if (p < kp) {
      const uint32_t r = sorted_r[static_cast<uint64_t>(b) * kbar + p];
      const uint32_t n = cells[r].n;
      pop += n;
      nch = (n + chunk_pts - 1) / chunk_pts;
      probes[static_cast<uint64_t>(b) * kp + p] = r;
      probe_pos[static_cast<uint64_t>(b) * kbar + r] = static_cast<int32_t>(p);
    }
    uint32_t excl, total;
    Scan(tmp.scan).ExclusiveSum(nch, excl, total);
    if (p < kp) coff[static_cast<uint64_t>(b) * kp + p] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  const uint64_t tot = Red(tmp.red).Sum(pop);
  if (threadIdx.x == 0) {
    pool_n[b] = tot;
    qch[b] = carry;
  }
}

// qbase[b] = first chunk of query b (exclusive scan of qch), qbase[B] = total
__global__ void __launch_bounds__(1024)
    ivf_chunk_base_kernel(const uint32_t* __restrict__ qch, uint32_t B, uint64_t* __restrict__ qbase) {
  using Scan = cub::BlockScan<uint64_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < B; b0 += 1024) {
    const uint32_t b = b0 + threadIdx.x;
    const uint64_t v = b < B ? qch[b] : 0;
    uint64_t excl, total;
    Scan(tmp).ExclusiveSum(v, excl, total);
    if (b < B) qbase[b] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) qbase[B] = carry;
}

struct IvfScoreArgs {
  const float* Q;
  uint32_t B, d, kbar, kp, chunk_pts, S;  // S: candidate slots per chunk = min(topn, chunk_pts)
  const double* cs;
  const uint32_t* probes;
  const uint32_t* coff;
  const uint64_t* qbase;
  const IvfCell* cells;
  const uint32_t* codes;
  const float* cb;
  const float* lam;
  const float* raw;
  const uint32_t* members;
  uint32_t m, m8, dbar, k_max, s, cbits, W, Wc;
  double* candD;   // [chunks][S]
  uint32_t* candI;
  uint32_t* ccnt;  // [chunks]
  unsigned long long* tau;  // [B] ord64 bound on each query's topn-th best score (0 = none)
  uint32_t topn;
};

// The cell's eta table for query q: the fixed-order fp32 dot from 0.0f of
// build_lookup_table (pq_index.cpp:186-190) over the cell's own codebooks;
// rows j >= m are -0.0 (never read).  Also the cell's scale codebooks.
template <bool kLam>
__device__ void ivf_build_lut(const IvfScoreArgs& a, const IvfCell& cell, const float* q, float* s_eta,
                              float* s_lam) {
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
  if constexpr (kLam)
    for (uint32_t t = threadIdx.x; t < a.m8 * a.s; t += blockDim.x) s_lam[t] = __ldg(a.lam + cell.lam_off + t);
}

__device__ __forceinline__ double ivf_raw_score(const float* q, const float* x, uint32_t d, double coarse) {
  double acc = 0.0;  // coarse + dotf(q, residual) (ivf.cpp:122-124)
  for (uint32_t i = 0; i < d; ++i)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(__ldg(q + i)), static_cast<double>(__ldg(x + i))));
  return __dadd_rn(coarse, acc);
}

// K_s: persistent; CTA c takes the contiguous work items [T*c/G, T*(c+1)/G)
// of the (query, probe, chunk) list, so consecutive items mostly share the
// (query, cell) and its eta table.  Per chunk: score every member
// (coarse + double(sub), ivf.cpp:130), keep the chunk's exact top-S by
// (score desc, id asc) and write them as candidates.
template <int CW, int SW>
__global__ void __launch_bounds__(256) ivf_score_kernel(const IvfScoreArgs a) {
  using Cd = Codec<CW, SW>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t hist[256];
  __shared__ Sel96 sel;
  __shared__ uint32_t s_n, s_surv;
  __shared__ unsigned long long s_kmin;
  float* s_eta = reinterpret_cast<float*>(smem);  // [m8][k_max], RS = 1
  float* s_lam = s_eta + static_cast<size_t>(a.m8) * a.k_max;
  double* s_D = reinterpret_cast<double*>(
      smem + ((static_cast<size_t>(a.m8) * (a.k_max + a.s) * 4 + 15) & ~static_cast<size_t>(15)));
  uint32_t* s_id = reinterpret_cast<uint32_t*>(s_D + a.chunk_pts);
  const uint32_t eta_sa = static_cast<uint32_t>(__cvta_generic_to_shared(s_eta));
  const uint64_t T = a.qbase[a.B];
  const uint64_t w0 = T * blockIdx.x / gridDim.x, w1 = T * (blockIdx.x + 1) / gridDim.x;
  uint32_t cur_b = 0xFFFFFFFFu, cur_p = 0xFFFFFFFFu;
  for (uint64_t w = w0; w < w1; ++w) {
    // (query, probe, chunk) of work item w
    uint32_t lo = 0, hi = a.B;  // largest b with qbase[b] <= w
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (a.qbase[mid] <= w) lo = mid;
      else hi = mid;
    }
    const uint32_t b = lo;
    const uint32_t local = static_cast<uint32_t>(w - a.qbase[b]);
    const uint32_t* co = a.coff + static_cast<uint64_t>(b) * a.kp;
    uint32_t pl = 0, ph = a.kp;  // largest p with coff[p] <= local
    while (ph - pl > 1) {
      const uint32_t mid = (pl + ph) >> 1;
      if (co[mid] <= local) pl = mid;
      else ph = mid;
    }
    const uint32_t p = pl;
    const uint32_t chunk = local - co[p];
    const uint32_t r = a.probes[static_cast<uint64_t>(b) * a.kp + p];
    const IvfCell cell = a.cells[r];
    const uint32_t pos0 = chunk * a.chunk_pts;
    const uint32_t cnt = min(cell.n - pos0, a.chunk_pts);
    const double coarse = a.cs[static_cast<uint64_t>(b) * a.kbar + r];
    const float* q = a.Q + static_cast<uint64_t>(b) * a.d;
    if (!cell.raw && (b != cur_b || p != cur_p)) {
      __syncthreads();  // previous item's table reads are done
      ivf_build_lut<!Cd::kNoLambda>(a, cell, q, s_eta, s_lam);
      cur_b = b;
      cur_p = p;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t pos = pos0 + i;
      double D;
      if (cell.raw) {
        D = ivf_raw_score(q, a.raw + cell.raw_off + static_cast<uint64_t>(pos) * a.d, a.d, coarse);
      } else {
        const uint64_t blk = cell.block_off + pos / kBlockPts;
        const uint32_t* wp = a.codes + blk * a.W * kBlockPts + (pos % kBlockPts);
        float acc[1][1];
        score_point<1, CW, SW, 0, 1>(wp, 0, eta_sa, s_eta, s_lam, a.k_max, a.s, a.cbits, a.W, a.Wc,
                                     a.m, acc);
        D = __dadd_rn(coarse, static_cast<double>(acc[0][0]));  // ivf.cpp:130
      }
      s_D[i] = D;
      s_id[i] = a.members[cell.member_off + pos];
    }
    // Keys below the query's published bound cannot reach its top-n (some
    // chunk already holds topn keys at or above it); count the survivors.
    const unsigned long long tau = __ldcg(a.tau + b);
    if (threadIdx.x == 0) {
      s_surv = 0;
      s_n = 0;
      s_kmin = ~0ull;
    }
    __syncthreads();
    {
      uint32_t c = 0;
      for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) c += ord64(s_D[i]) >= tau ? 1u : 0u;
      c = __reduce_add_sync(0xFFFFFFFFu, c);
      if ((threadIdx.x & 31u) == 0 && c) atomicAdd(&s_surv, c);
    }
    __syncthreads();
    const uint32_t nsurv = s_surv;
    const uint32_t keep = min(a.S, nsurv);
    auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) -> bool {
      h = ord64(s_D[i]);
      l = ~s_id[i];
      return h >= tau;
    };
    select96(get, cnt, keep, nsurv, hist, sel);  // returns at once when nsurv <= S
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      uint64_t h;
      uint32_t l;
      if (get(i, h, l) && sel96_take(sel, h, l)) {
        const uint32_t slot = atomicAdd(&s_n, 1u);
        a.candD[w * a.S + slot] = s_D[i];
        a.candI[w * a.S + slot] = ~l;
        atomicMin(&s_kmin, static_cast<unsigned long long>(h));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      a.ccnt[w] = s_n;
      // this chunk alone holds topn keys at or above s_kmin: publish it
      if (s_n >= a.topn) atomicMax(a.tau + b, s_kmin);
    }
  }
}

// K_g: the batched multi-cell scan.  The probes are
// inverted into (cell -> probing queries); a work item is (cell, group of up
// to 16 of its queries, chunk of the cell's members).  Per (cell, group) the
// 16 queries' eta tables over the cell's codebooks are built once (the K1
// arithmetic, NQ = 16 rows), and every member is decoded once and scored for
// all 16 with the flat scan's score_point — the same fp32 order, so every
// score equals the per-(query, cell) kernel's.  Each query's chunk top-S is
// then selected exactly and written to the work slot that query's own
// (probe, chunk) owns in the per-query layout, so K_t is unchanged.
constexpr uint32_t kIvfGroupQ = 16;

struct IvfGroupArgs {
  const uint32_t* inv_bp;   // [B*kp] b*kp + p, sorted by cell (stable: by b, p)
  const uint32_t* cstart;   // [kbar+1] first inv_bp index of each cell
  const uint64_t* ibase;    // [kbar+1] first work item of each cell
};

template <int CW, int SW>
__global__ void __launch_bounds__(512) ivf_group_score_kernel(const IvfScoreArgs a, const IvfGroupArgs gi) {
  constexpr int NQ = kIvfGroupQ;
  constexpr int RS = rs_of(NQ);
  using Cd = Codec<CW, SW>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_bp[NQ];
  __shared__ double s_co[NQ];
  __shared__ uint32_t whist[NQ][256];  // per-warp selection histograms
  float* s_eta = reinterpret_cast<float*>(smem);  // [m8][k_max][RS]
  float* s_lam = s_eta + static_cast<size_t>(a.m8) * a.k_max * RS;
  double* s_D = reinterpret_cast<double*>(
      smem + ((static_cast<size_t>(a.m8) * (a.k_max * RS + a.s) * 4 + 15) & ~static_cast<size_t>(15)));
  uint32_t* s_id = reinterpret_cast<uint32_t*>(s_D + static_cast<size_t>(NQ) * a.chunk_pts);
  const uint64_t T = gi.ibase[a.kbar];
  const uint64_t w0 = T * blockIdx.x / gridDim.x, w1 = T * (blockIdx.x + 1) / gridDim.x;
  uint32_t cur_r = 0xFFFFFFFFu, cur_g = 0xFFFFFFFFu, nq = 0;
  for (uint64_t w = w0; w < w1; ++w) {
    uint32_t lo = 0, hi = a.kbar;  // largest r with ibase[r] <= w
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (gi.ibase[mid] <= w) lo = mid;
      else hi = mid;
    }
    const uint32_t r = lo;
    const IvfCell cell = a.cells[r];
    const uint32_t nch = (cell.n + a.chunk_pts - 1) / a.chunk_pts;
    const uint32_t local = static_cast<uint32_t>(w - gi.ibase[r]);
    const uint32_t g = local / nch, ch = local % nch;
    if (r != cur_r || g != cur_g) {
      __syncthreads();  // the previous item's table and slot reads are done
      const uint32_t c0 = gi.cstart[r] + g * NQ;
      nq = min(static_cast<uint32_t>(NQ), gi.cstart[r + 1] - c0);
      if (threadIdx.x < NQ) {
        const uint32_t bp = threadIdx.x < nq ? gi.inv_bp[c0 + threadIdx.x] : 0u;
        s_bp[threadIdx.x] = bp;
        s_co[threadIdx.x] = threadIdx.x < nq ? a.cs[static_cast<uint64_t>(bp / a.kp) * a.kbar + r] : 0.0;
      }
      __syncthreads();
      const float* cbr = a.cb + cell.cb_off;
      const uint32_t tot = a.m8 * a.k_max * NQ;
      for (uint32_t t = threadIdx.x; t < tot; t += blockDim.x) {
        const uint32_t qs = t % NQ, c = (t / NQ) % a.k_max, j = t / (NQ * a.k_max);
        float acc = 0.0f;  // ivf_build_lut's value for this query (pq_index.cpp:186-190)
        if (j >= a.m) {
          acc = -0.0f;
        } else if (c < cell.k && qs < nq) {
          const float* q = a.Q + static_cast<uint64_t>(s_bp[qs] / a.kp) * a.d;
          const float* row = cbr + (static_cast<uint64_t>(j) * cell.k + c) * a.dbar;
          for (uint32_t i = 0; i < a.dbar; ++i) {
            const uint32_t col = j * a.dbar + i;
            const float qa = col < a.d ? __ldg(q + col) : 0.0f;
            acc = __fadd_rn(acc, __fmul_rn(__ldg(row + i), qa));
          }
        }
        s_eta[(j * a.k_max + c) * RS + qs] = acc;
      }
      if constexpr (!Cd::kNoLambda)
        for (uint32_t t = threadIdx.x; t < a.m8 * a.s; t += blockDim.x) s_lam[t] = __ldg(a.lam + cell.lam_off + t);
      cur_r = r;
      cur_g = g;
    }
    __syncthreads();
    const uint32_t pos0 = ch * a.chunk_pts;
    const uint32_t cnt = min(cell.n - pos0, a.chunk_pts);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t pos = pos0 + i;
      const uint64_t blk = cell.block_off + pos / kBlockPts;
      const uint32_t* wp = a.codes + blk * a.W * kBlockPts + (pos % kBlockPts);
      float acc[1][NQ];
      score_point<NQ, CW, SW, 0, 1>(wp, 0, 0u, s_eta, s_lam, a.k_max, a.s, a.cbits, a.W, a.Wc, a.m, acc);
#pragma unroll
      for (int qs = 0; qs < NQ; ++qs)
        s_D[static_cast<size_t>(qs) * a.chunk_pts + i] = __dadd_rn(s_co[qs], static_cast<double>(acc[0][qs]));
      s_id[i] = a.members[cell.member_off + pos];
    }
    __syncthreads();
    {  // one warp per query slot: survivors, exact top-S, candidates (no block barriers)
      const uint32_t qs = threadIdx.x >> 5, lane = threadIdx.x & 31u;
      if (qs < nq) {
        const uint32_t bp = s_bp[qs];
        const uint32_t b = bp / a.kp;
        const uint64_t wo = a.qbase[b] + a.coff[bp] + ch;  // the query's own (probe, chunk) slot
        const double* D = s_D + static_cast<size_t>(qs) * a.chunk_pts;
        const unsigned long long tau = __ldcg(a.tau + b);
        auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) -> bool {
          h = ord64(D[i]);
          l = ~s_id[i];
          return h >= tau;
        };
        uint32_t nsurv = 0;
        for (uint32_t i = lane; i < cnt; i += 32) nsurv += ord64(D[i]) >= tau ? 1u : 0u;
        nsurv = __reduce_add_sync(0xFFFFFFFFu, nsurv);
        Sel96 sw;
        warp_select96(get, cnt, min(a.S, nsurv), nsurv, whist[qs], sw);
        const bool all = a.S >= nsurv;
        uint32_t base = 0;
        unsigned long long kmin = ~0ull;
        for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
          const uint32_t i = i0 + lane;
          uint64_t h = 0;
          uint32_t l = 0;
          const bool take = i < cnt && get(i, h, l) && (all || sel96_take(sw, h, l));
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, take);
          if (take) {
            const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
            a.candD[wo * a.S + slot] = D[i];
            a.candI[wo * a.S + slot] = ~l;
            kmin = min(kmin, static_cast<unsigned long long>(h));
          }
          base += __popc(bal);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) kmin = min(kmin, __shfl_xor_sync(0xFFFFFFFFu, kmin, o));
        if (lane == 0) {
          a.ccnt[wo] = base;
          if (base >= a.topn) atomicMax(a.tau + b, kmin);
        }
      }
    }
  }
}

// inversion helpers: cell starts of the sorted (cell, b*kp+p) pairs, and the
// per-cell work-item counts (groups x chunks)
__global__ void ivf_inv_starts_kernel(const uint32_t* __restrict__ sorted_r, uint32_t n, uint32_t kbar,
                                      uint32_t* __restrict__ cstart) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > kbar) return;
  uint32_t lo = 0, hi = n;  // first position with key >= r
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sorted_r[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  cstart[r] = lo;
}

__global__ void ivf_inv_items_kernel(const uint32_t* __restrict__ cstart, const IvfCell* __restrict__ cells,
                                     uint32_t kbar, uint32_t chunk_pts, uint64_t* __restrict__ items) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= kbar) return;
  const uint32_t nq = cstart[r + 1] - cstart[r];
  const uint32_t groups = (nq + kIvfGroupQ - 1) / kIvfGroupQ;
  items[r] = static_cast<uint64_t>(groups) * ((cells[r].n + chunk_pts - 1) / chunk_pts);
}

__global__ void ivf_iota_kernel(uint32_t* __restrict__ v, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// K_t: exact top-n of each query's candidates (the chunks' survivors) by
// (score desc, id asc) (ivf.cpp:139-146): select96, gather, bitonic sort.
constexpr uint32_t kIvfMaxTop = 8192;

__global__ void __launch_bounds__(1024)
    ivf_select_kernel(const double* __restrict__ candD, const uint32_t* __restrict__ candI,
                      const uint32_t* __restrict__ ccnt, const uint64_t* __restrict__ qbase,
                      uint32_t S, const uint64_t* __restrict__ pool_n, uint32_t topn,
                      int32_t* __restrict__ ids, double* __restrict__ scores,
                      uint32_t* __restrict__ counts, uint8_t* __restrict__ shorts) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t hist[256];
  __shared__ Sel96 sel;
  __shared__ uint32_t s_n;
  __shared__ unsigned long long s_valid;
  const uint32_t b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t c0 = qbase[b], c1 = qbase[b + 1];
  const uint64_t nslots = (c1 - c0) * S;
  const uint64_t pop = pool_n[b];
  const uint32_t keep = static_cast<uint32_t>(pop < topn ? pop : static_cast<uint64_t>(topn));
  if (tid == 0) {
    counts[b] = keep;
    shorts[b] = pop < topn ? 1 : 0;
    s_n = 0;
    s_valid = 0;
  }
  __syncthreads();
  {
    unsigned long long v = 0;
    for (uint64_t w = c0 + tid; w < c1; w += nthr) v += ccnt[w];
    atomicAdd(&s_valid, v);
  }
  __syncthreads();
  auto get = [&](uint64_t i, uint64_t& h, uint32_t& l) -> bool {
    const uint64_t w = c0 + i / S;
    const uint32_t j = static_cast<uint32_t>(i % S);
    if (j >= ccnt[w]) return false;
    h = ord64(candD[w * S + j]);
    l = ~candI[w * S + j];
    return true;
  };
  select96(get, nslots, keep, s_valid, hist, sel);
  uint64_t* k_hi = reinterpret_cast<uint64_t*>(smem);
  uint32_t* k_id = reinterpret_cast<uint32_t*>(k_hi + kIvfMaxTop);
  uint32_t* k_ix = k_id + kIvfMaxTop;  // candidate slot (for the exact score bits)
  for (uint64_t i = tid; i < nslots; i += nthr) {
    uint64_t h;
    uint32_t l;
    if (!get(i, h, l) || !sel96_take(sel, h, l)) continue;
    const uint32_t slot = atomicAdd(&s_n, 1u);
    if (slot < keep) {
      k_hi[slot] = h;
      k_id[slot] = ~l;
      k_ix[slot] = static_cast<uint32_t>(i);
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
    if (i < keep) {
      const uint64_t sl = k_ix[i];
      scores[o] = candD[(c0 + sl / S) * S + sl % S];
    } else {
      scores[o] = __longlong_as_double(0x7FF8000000000000ll);
    }
  }
}

// K_r: requested ids (ivf.cpp:134-137): one CTA per (query, id) rebuilds the
// id's cell table and scores that one member exactly like K_s; NaN when the
// cell was not probed.
template <int CW, int SW>
__global__ void __launch_bounds__(128)
    ivf_requested_kernel(const IvfScoreArgs a, const uint32_t* __restrict__ req, uint32_t R,
                         const uint32_t* __restrict__ pcluster, const uint32_t* __restrict__ pslot,
                         const int32_t* __restrict__ probe_pos, double* __restrict__ out) {
  using Cd = Codec<CW, SW>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint64_t t = blockIdx.x;
  const uint32_t b = static_cast<uint32_t>(t / R);
  const uint32_t id = req[t];
  const uint32_t r = pcluster[id];
  if (probe_pos[static_cast<uint64_t>(b) * a.kbar + r] < 0) {
    if (threadIdx.x == 0) out[t] = __longlong_as_double(0x7FF8000000000000ll);
    return;
  }
  const IvfCell cell = a.cells[r];
  const uint32_t pos = pslot[id];
  const double coarse = a.cs[static_cast<uint64_t>(b) * a.kbar + r];
  const float* q = a.Q + static_cast<uint64_t>(b) * a.d;
  if (cell.raw) {
    if (threadIdx.x == 0) out[t] = ivf_raw_score(q, a.raw + cell.raw_off + static_cast<uint64_t>(pos) * a.d, a.d, coarse);
    return;
  }
  float* s_eta = reinterpret_cast<float*>(smem);
  float* s_lam = s_eta + static_cast<size_t>(a.m8) * a.k_max;
  ivf_build_lut<!Cd::kNoLambda>(a, cell, q, s_eta, s_lam);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t blk = cell.block_off + pos / kBlockPts;
    const uint32_t* wp = a.codes + blk * a.W * kBlockPts + (pos % kBlockPts);
    float acc[1][1];
    score_point<1, CW, SW, 0, 1>(wp, 0, static_cast<uint32_t>(__cvta_generic_to_shared(s_eta)), s_eta,
                                 s_lam, a.k_max, a.s, a.cbits, a.W, a.Wc, a.m, acc);
    out[t] = __dadd_rn(coarse, static_cast<double>(acc[0][0]));
  }
}

__global__ void ivf_check_ids_kernel(const uint32_t* __restrict__ req, uint64_t cnt, uint32_t n,
                                     uint32_t* __restrict__ err) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < cnt && req[t] >= n) atomicOr(err, 1u);
}

using IvfScoreFn = void (*)(IvfScoreArgs);
using IvfReqFn = void (*)(IvfScoreArgs, const uint32_t*, uint32_t, const uint32_t*, const uint32_t*,
                          const int32_t*, double*);
using IvfGroupFn = void (*)(IvfScoreArgs, IvfGroupArgs);
struct IvfFns {
  IvfScoreFn score = nullptr;
  IvfReqFn req = nullptr;
  IvfGroupFn group = nullptr;
};

template <int CW, int SW>
IvfFns ivf_fns() {
  return {ivf_score_kernel<CW, SW>, ivf_requested_kernel<CW, SW>, ivf_group_score_kernel<CW, SW>};
}

template <int CW>
IvfFns ivf_pick_sw(uint32_t sw) {
  switch (sw) {
    case 0: return ivf_fns<CW, 0>();
    case 4: return ivf_fns<CW, 4>();
    case 8: return ivf_fns<CW, 8>();
    case 16: return ivf_fns<CW, 16>();
    case 32: return ivf_fns<CW, 32>();
  }
  return {};
}

IvfFns ivf_pick(const CodeLayout& L) {
  if (L.format == PCPQG_FMT_JOINT8) return ivf_fns<0, 0>();
  if (L.cw == 4) return ivf_pick_sw<4>(L.sw);
  if (L.cw == 8) return ivf_pick_sw<8>(L.sw);
  if (L.cw == 16) return ivf_pick_sw<16>(L.sw);
  return {};
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
  keep_mempool(v.device);
  const uint32_t s1 = std::max(v.scales, 1u);
  const uint32_t m8 = (v.m + 7) & ~7u;
  const uint32_t kmx = std::max(v.k_max, 1u);
  IvfFns fns = v.n_pq ? ivf_pick(v.lay) : ivf_fns<0, 0>();
  if (!fns.score) fail(PCPQG_E_UNSUPPORTED, "no IVF scoring kernel for this code layout");
  // K_g (batched multi-cell scan) for containers of PQ cells with small k and
  // batches large enough that cells are probed by several queries; it needs
  // 512-point chunks (its 16 score rows live in shared memory)
  const uint32_t RSg = static_cast<uint32_t>(rs_of(kIvfGroupQ));
  int max_smem0 = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem0, cudaDevAttrMaxSharedMemoryPerBlockOptin, v.device));
  const size_t lut_g = (static_cast<size_t>(m8) * (kmx * RSg + s1) * 4 + 15) & ~static_cast<size_t>(15);
  // 1024-member chunks when the 16 score rows fit (fewer candidate lists for
  // the final select), else 512; + 20 KB static (per-warp histograms)
  const uint32_t gchunk = lut_g + 1024ull * (kIvfGroupQ * 8 + 4) + 20480 <= static_cast<size_t>(max_smem0) ? 1024 : 512;
  const size_t group_smem = lut_g + static_cast<size_t>(gchunk) * (kIvfGroupQ * 8 + 4);
  const bool grouped = v.n_raw == 0 && v.n_pq > 0 && options().ivf_grouped && fns.group &&
                       static_cast<uint64_t>(B) * kp >= 4ull * v.kbar &&
                       group_smem + 20480 <= static_cast<size_t>(max_smem0);
  // (per-(query, cell) kernel: 1024-member chunks balance the persistent CTAs
  // better than 2048 — 2.14 vs 2.42 ms at 1M points, k_probe 32, B 1000)
  const uint32_t chunk_pts = grouped ? gchunk : 1024;
  const uint32_t S = std::min(topn, chunk_pts);
  const size_t lut_bytes = (static_cast<size_t>(m8) * (kmx + s1) * 4 + 15) & ~static_cast<size_t>(15);
  const size_t score_smem = lut_bytes + static_cast<size_t>(chunk_pts) * 12;
  const size_t req_smem = std::max<size_t>(lut_bytes, 16);
  static const size_t kSelSmem = kIvfMaxTop * 16;
  int max_smem = 0, sms = 0;
  PCPQG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, v.device));
  PCPQG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, v.device));
  if (score_smem + 2048 > static_cast<size_t>(max_smem))
    fail(PCPQG_E_UNSUPPORTED, "IVF cell eta table does not fit in shared memory");
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fns.score),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(score_smem)));
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fns.req),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(req_smem)));
  PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(ivf_select_kernel),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSelSmem)));
  int occ = 0;
  PCPQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fns.score),
                                                           256, score_smem));
  const uint32_t grid = static_cast<uint32_t>(sms) * std::max(occ, 1);
  // upper bound of a query's chunk count: every probe contributes its ceil
  const uint64_t max_chunks_q = kp + v.top_prefix[kp] / chunk_pts + 1;
  const uint64_t per_q = max_chunks_q * (S * 12ull + 4) + static_cast<uint64_t>(v.kbar) * 28 + kp * 8ull;
  // queries per pass: the per-query scratch within max(1 GB, free / 8)
  size_t free_b = 0, total_b = 0;
  PCPQG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t budget = std::max<uint64_t>(1ull << 30, free_b / 8);
  const uint32_t chunk = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(B, budget / per_q)));

  for (uint32_t b0 = 0; b0 < B; b0 += chunk) {
    const uint32_t Bc = std::min(chunk, B - b0);
    const uint64_t bk = static_cast<uint64_t>(Bc) * v.kbar;
    const uint64_t tmax = static_cast<uint64_t>(Bc) * max_chunks_q;
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
    uint32_t* coff = salloc<uint32_t>(keep, static_cast<uint64_t>(Bc) * kp, st);
    uint32_t* qch = salloc<uint32_t>(keep, Bc, st);
    uint64_t* qbase = salloc<uint64_t>(keep, Bc + 1, st);
    uint64_t* pn = salloc<uint64_t>(keep, Bc, st);
    double* candD = salloc<double>(keep, tmax * S, st);
    uint32_t* candI = salloc<uint32_t>(keep, tmax * S, st);
    uint32_t* ccnt = salloc<uint32_t>(keep, tmax, st);
    unsigned long long* tau = salloc<unsigned long long>(keep, Bc, st);
    PCPQG_CUDA(cudaMemsetAsync(tau, 0, 8ull * Bc, st));
    const float* q = dQ + static_cast<uint64_t>(b0) * v.d;

    // profiling (pcpqg_set_profiling): probe selection / scoring / top-n stage times
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    const bool prof = profiling_enabled();
    if (prof)
      for (auto& e : ev) {
        PCPQG_CUDA(cudaEventCreate(&e));
      }
    if (prof) PCPQG_CUDA(cudaEventRecord(ev[0], st));
    ivf_coarse_kernel<<<static_cast<unsigned>((bk + 255) / 256), 256, 0, st>>>(
        q, Bc, v.d, v.d_coarse, v.kbar, cs, keys, vals);
    PCPQG_CUDA(cudaGetLastError());
    if (v.kbar <= kIvfSortMax) {
      ivf_order_kernel<<<Bc, 1024, 0, st>>>(keys, v.kbar, vals2);
      PCPQG_CUDA(cudaGetLastError());
    } else {
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
    }
    PCPQG_CUDA(cudaMemsetAsync(ppos, 0xFF, bk * sizeof(int32_t), st));
    ivf_probe_kernel<<<Bc, 256, 0, st>>>(vals2, v.kbar, kp, v.d_cells, chunk_pts, probes, ppos, coff, qch, pn);
    PCPQG_CUDA(cudaGetLastError());
    ivf_chunk_base_kernel<<<1, 1024, 0, st>>>(qch, Bc, qbase);
    PCPQG_CUDA(cudaGetLastError());

    if (prof) PCPQG_CUDA(cudaEventRecord(ev[1], st));
    IvfScoreArgs a{};
    a.Q = q;
    a.B = Bc;
    a.d = v.d;
    a.kbar = v.kbar;
    a.kp = kp;
    a.chunk_pts = chunk_pts;
    a.S = S;
    a.cs = cs;
    a.probes = probes;
    a.coff = coff;
    a.qbase = qbase;
    a.cells = v.d_cells;
    a.codes = v.d_codes;
    a.cb = v.d_cb;
    a.lam = v.d_lam;
    a.raw = v.d_raw;
    a.members = v.d_members;
    a.m = v.m;
    a.m8 = m8;
    a.dbar = v.dbar;
    a.k_max = kmx;
    a.s = s1;
    a.cbits = v.lay.format == PCPQG_FMT_JOINT8 ? v.lay.cw : 0u;
    a.W = v.lay.W;
    a.Wc = v.lay.Wc;
    a.candD = candD;
    a.candI = candI;
    a.ccnt = ccnt;
    a.tau = tau;
    a.topn = topn;
    if (grouped) {
      // invert the probes: (cell, b*kp + p) sorted by cell, stable
      const uint32_t np = Bc * kp;
      uint32_t* ikey = salloc<uint32_t>(keep, np, st);
      uint32_t* ival = salloc<uint32_t>(keep, np, st);
      uint32_t* cstart = salloc<uint32_t>(keep, v.kbar + 1, st);
      uint64_t* items = salloc<uint64_t>(keep, v.kbar + 1, st);
      uint64_t* ibase = salloc<uint64_t>(keep, v.kbar + 1, st);
      ivf_iota_kernel<<<(np + 255) / 256, 256, 0, st>>>(vals, np);
      int bits = 1;
      while ((1u << bits) < v.kbar) ++bits;
      size_t tb = 0;
      PCPQG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, probes, ikey, vals, ival, static_cast<int>(np), 0,
                                                 bits, st));
      void* tmp = salloc<uint8_t>(keep, tb, st);
      PCPQG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, probes, ikey, vals, ival, static_cast<int>(np), 0, bits,
                                                 st));
      ivf_inv_starts_kernel<<<(v.kbar + 1 + 255) / 256, 256, 0, st>>>(ikey, np, v.kbar, cstart);
      ivf_inv_items_kernel<<<(v.kbar + 255) / 256, 256, 0, st>>>(cstart, v.d_cells, v.kbar, chunk_pts, items);
      PCPQG_CUDA(cudaMemsetAsync(items + v.kbar, 0, 8, st));
      size_t tb2 = 0;
      PCPQG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, items, ibase, v.kbar + 1, st));
      void* tmp2 = salloc<uint8_t>(keep, tb2, st);
      PCPQG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb2, items, ibase, v.kbar + 1, st));
      PCPQG_CUDA(cudaGetLastError());
      IvfGroupArgs gi{ival, cstart, ibase};
      PCPQG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fns.group),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(group_smem)));
      fns.group<<<static_cast<unsigned>(sms), 512, group_smem, st>>>(a, gi);
    } else {
      fns.score<<<grid, 256, score_smem, st>>>(a);
    }
    PCPQG_CUDA(cudaGetLastError());
    if (prof) PCPQG_CUDA(cudaEventRecord(ev[2], st));
    ivf_select_kernel<<<Bc, 1024, kSelSmem, st>>>(
        candD, candI, ccnt, qbase, S, pn, topn, d_ids + static_cast<uint64_t>(b0) * topn,
        d_scores + static_cast<uint64_t>(b0) * topn, d_counts + b0, d_short + b0);
    PCPQG_CUDA(cudaGetLastError());
    if (prof) {
      PCPQG_CUDA(cudaEventRecord(ev[3], st));
      PCPQG_CUDA(cudaEventSynchronize(ev[3]));
      float t3[3];
      for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t3[i], ev[i], ev[i + 1]);
      set_last_timings(t3);
      for (auto& e : ev) cudaEventDestroy(e);
    }
    if (R && d_req_scores) {
      const uint64_t br = static_cast<uint64_t>(Bc) * R;
      if (br > 0x7FFFFFFFull) fail(PCPQG_E_UNSUPPORTED, "too many requested ids");
      fns.req<<<static_cast<unsigned>(br), 128, req_smem, st>>>(
          a, d_req + static_cast<uint64_t>(b0) * R, R, v.d_pcluster, v.d_pslot, ppos,
          d_req_scores + static_cast<uint64_t>(b0) * R);
      PCPQG_CUDA(cudaGetLastError());
    }
    for (void* p : keep) PCPQG_CUDA(cudaFreeAsync(p, st));
  }
}

}  // namespace pcpqg
