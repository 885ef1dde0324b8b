// Device helpers shared by the kernel translation units of libpcpqg.so:
// candidate keys, mbarrier / TMA bulk-copy wrappers, thread groups and the
// group-parallel radix select + compaction used by the top-K machinery.
#pragma once
#include <cuda_fp16.h>

#include <cassert>
#include <cstdint>

#include "pcpqg_internal.hpp"

// PCPQG_DEBUG builds (make debug) check every shared-memory index.
#ifdef PCPQG_DEBUG
#define PCPQG_DASSERT(x) assert(x)
#else
#define PCPQG_DASSERT(x) ((void)0)
#endif

namespace pcpqg {

struct ScanArgs {
  const uint32_t* codes;  // [n_blocks][W][32]
  const float* eta;       // grouped tables [G][m8*k rows][RS] (group stride gstride)
  const float* lam;       // [m8][s], pad sections 1.0
  uint64_t* partial;      // [ctas_x][Bpad][K] survivors first, then empty keys
  uint32_t* pcnt;         // [ctas_x][Bpad] survivors per list (optional)
  uint64_t* gtau;         // [Bpad] best known K-th key per query (shared across CTAs)
  float* scores;          // score_all mode: [B][n_local]
  uint64_t n_local;
  uint32_t n_blocks, W, Wc, m, m8, k, s, cbits;
  uint32_t B, Bpad, K, Ks, cap, ppt, stages;  // Ks: partial row stride (K rounded up to even)
  uint64_t gstride;       // floats per group table (multiple of 4)
  uint64_t id_base;
  // fused merge (optional): per-group completion tickets and the final rows
  uint32_t* done;         // [groups], zeroed before the launch; nullptr = separate merge
  uint64_t* out_keys;     // [B][out_stride] (each optional)
  int32_t* out_ids;
  float* out_scores;
  uint32_t out_stride;
  // filter mode (JOINT8, k = 16, NQ = 16): fp16 eta_hat rows [G][m8*16][kFRS],
  // fp16 lambda_hat [m8][s] and per query (sigma, eps) [Bpad]
  const __half* fh;
  const __half* flam;
  const float2* fse;
  uint64_t fgstride;      // halves per group table
  uint32_t fmode;         // 1 filter; diagnostics: 2 never pass (filter cost), 3 count passes
  // filter mode: every CTA leaves its final top-K (of everything it saw,
  // inherited keys included) in carry[(g*ctas_x + cx)*NQ + q][K] and raises
  // carry_done[g*ctas_x + cx]; the next range's CTA inherits it, so a CTA's
  // pruning bound is the K-th best of the union of all ranges before it
  uint64_t* carry;
  uint32_t* carry_cnt;
  uint32_t* carry_done;
  unsigned long long* fcount;
  // single-launch small-batch search (warp-specialised scans): the CTA builds
  // its group's tables itself (lut_mode 1: eta, 2: the JOINT8 eta*lambda table —
  // lut_kernel's arithmetic) from the queries and codebooks, so no LUT kernel
  // runs before the scan; 0 = read a.eta
  const float* Q;         // [B][d]
  const float* cb;        // [m][kc][dbar]
  uint32_t lut_mode, kc, d, dbar;
};
using ScanFn = void (*)(ScanArgs);
// filter tables: halves per eta_hat row (16 queries + 4 pad: 40 bytes = five
// 8-byte units, odd, so 16 lanes with 16 distinct centers hit 16 bank pairs)
constexpr int kFRS = 20;
// filter mode: queue of (point, query) pairs that passed the filter
// (point within the CTA's range << 4 | query), re-scored exactly by the whole
// CTA once it is half full (and at the end), reading the codes from L2/HBM
constexpr int kFQCap = 2048;
constexpr int kWsFlag = 0x100;  // pick_* argument: nq | kWsFlag selects the WS scan

// Row stride (floats) of the shared eta table: rows are read with LDS.64
// (query pairs), so RS is even with RS/2 odd; then 16 lanes with 16 different
// center codes c of the same section hit 16 distinct bank pairs (k <= 16).
// Compaction groups of a scan CTA: the largest count <= nq that splits the
// nthr/32 warps evenly (named-barrier sizes must be warp multiples).
__host__ __device__ constexpr int scan_ngroups(int nq, int nthr) {
  int g = nq < nthr / 32 ? nq : nthr / 32;
  while (g > 1 && (nthr / 32) % g != 0) --g;
  return g;
}

__host__ __device__ constexpr int rs_of(int nq) {
  return nq == 1 ? 1 : (((nq / 2) & 1) ? nq : nq + 2);
}


namespace {

constexpr int kThreads = 256;
constexpr int kStages = 3;

// ------------------------------------------------------------------ keys
// 64-bit candidate key, larger = better:
//   [63:32] order-preserving image of the score (-0 canonicalised to +0, so
//           -0 and +0 compare equal as floats do in the reference comparator)
//   [31:1]  0x7FFFFFFF - id  (equal scores -> lower id first)
//   [0]     1 iff the score is -0.0 (restores the exact bits on decode)
// Key 0 is "empty" and sorts below every real key.
__device__ __forceinline__ uint32_t ord_of(float s) {
  uint32_t b = __float_as_uint(s);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t make_key(float s, uint32_t id) {
  const uint64_t negz = (__float_as_uint(s) == 0x80000000u) ? 1ull : 0ull;
  return (static_cast<uint64_t>(ord_of(s)) << 32) |
         (static_cast<uint64_t>(0x7FFFFFFFu - id) << 1) | negz;
}
__device__ __forceinline__ float key_score(uint64_t key) {
  if (key == 0ull) return -INFINITY;
  if (key & 1ull) return -0.0f;
  const uint32_t o = static_cast<uint32_t>(key >> 32);
  const uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ int32_t key_id(uint64_t key) {
  if (key == 0ull) return -1;
  return static_cast<int32_t>(0x7FFFFFFFu - static_cast<uint32_t>((key >> 1) & 0x7FFFFFFFu));
}

// ------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Thread group that compacts candidate buffers: `size` threads (a multiple of
// 32), synchronised by __syncwarp or a named barrier.
struct Group {
  int id, size, gtid;
  __device__ __forceinline__ void sync() const {
    if (size == 32)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(size) : "memory");
  }
};

// Histogram bins are padded by one word every 8 so that the digit scan below
// (lane l reads bins 255-8l .. 255-8l-7) touches 32 distinct banks.
__device__ __forceinline__ uint32_t hidx(uint32_t b) { return b + (b >> 3); }
constexpr int kHistWords = 288;  // 256 bins + 32 pad
// per-group scratch: histogram, 2 select words, 32 per-warp compaction counts
// (sv: digit, need, bin count, pad, u64 minimum; wsum: per-warp counts)
constexpr int kSvWords = 8;
constexpr int kGroupScratch = kHistWords + kSvWords + 32;

// Exact K-th largest of buf[0, n) (keys are unique), MSB-first radix select
// with 8-bit digits over the group; stops as soon as the selected digit's bin
// holds exactly the keys still needed (usually after 2-3 of the 8 digits) and
// returns that bin's minimum.  hist: kHistWords counters, sv: kSvWords words.
template <class Get>
__device__ uint64_t group_select_by(Get get, uint32_t n, uint32_t K, uint32_t* hist, uint32_t* sv,
                                    const Group& g) {
  uint64_t prefix = 0ull, mask = 0ull;
  uint32_t need = K;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = g.gtid; i < kHistWords; i += g.size) hist[i] = 0u;
    g.sync();
    // keys concentrate in a few top-byte bins: aggregate equal digits per
    // warp (__match_any_sync) so each bin gets one atomic per warp
    for (uint32_t i0 = 0; i0 < n; i0 += g.size) {
      const uint32_t i = i0 + g.gtid;
      const uint64_t key = i < n ? get(i) : 0ull;
      const bool ok = i < n && (key & mask) == prefix;
      const uint32_t digit = ok ? (static_cast<uint32_t>(key >> shift) & 0xFFu) : 0x100u;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, digit);
      if (ok && (g.gtid & 31) == __ffs(peers) - 1) atomicAdd(&hist[hidx(digit)], __popc(peers));
    }
    g.sync();
    if (g.gtid < 32) {
      const int lane = g.gtid;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        c[t] = hist[hidx(255 - 8 * lane - t)];
        tot += c[t];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const uint32_t above = incl - tot;
      if (above < need && need <= incl) {
        uint32_t acc = above;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (need <= acc + c[t]) {
            sv[0] = 255u - 8u * lane - t;
            sv[1] = need - acc;
            sv[2] = c[t];
            break;
          }
          acc += c[t];
        }
      }
    }
    g.sync();
    prefix |= static_cast<uint64_t>(sv[0]) << shift;
    mask |= 0xFFull << shift;
    need = sv[1];
    if (sv[2] == need) {
      // every key with this prefix is needed: the K-th is their minimum
      unsigned long long* smin = reinterpret_cast<unsigned long long*>(sv + 4);
      if (g.gtid == 0) *smin = ~0ull;
      g.sync();
      unsigned long long mn = ~0ull;
      for (uint32_t i = g.gtid; i < n; i += g.size) {
        const uint64_t key = get(i);
        if ((key & mask) == prefix && key < mn) mn = key;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
      if ((g.gtid & 31) == 0) atomicMin(smin, mn);
      g.sync();
      const uint64_t r = *smin;
      g.sync();
      return r;
    }
  }
  return prefix;
}

__device__ __forceinline__ uint64_t group_select(const uint64_t* buf, uint32_t n, uint32_t K,
                                                 uint32_t* hist, uint32_t* sv, const Group& g) {
  return group_select_by([buf](uint32_t i) { return buf[i]; }, n, K, hist, sv, g);
}

// Order-preserving in-place compaction of buf[0, n) to the keys >= tau.
// Destinations never exceed sources and each chunk is fully read before it
// is written, so no key is overwritten before it is moved.
__device__ uint32_t group_compact(uint64_t* buf, uint32_t n, uint64_t tau, uint32_t* wsum,
                                  const Group& g) {
  const int lane = g.gtid & 31, w = g.gtid >> 5, nw = g.size >> 5;
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += g.size) {
    const uint32_t i = c0 + g.gtid;
    const uint64_t key = i < n ? buf[i] : 0ull;
    const bool keep = i < n && key >= tau;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
    uint32_t rank = __popc(bal & ((1u << lane) - 1u)), total = __popc(bal);
    if (nw > 1) {
      if (lane == 0) wsum[w] = total;
      g.sync();
      uint32_t before = 0;
      total = 0;
      for (int t = 0; t < nw; ++t) {
        const uint32_t v = wsum[t];
        before += t < w ? v : 0u;
        total += v;
      }
      rank += before;
      g.sync();
    } else {
      __syncwarp();
    }
    if (keep) buf[base + rank] = key;
    base += total;
  }
  g.sync();
  return base;
}


// order-preserving image of a double, -0 folded onto +0 (they compare equal)
__device__ __forceinline__ uint64_t ord64(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  if ((b << 1) == 0ull) b = 0ull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ---- exact selection over 96-bit keys (ord64(score), ~id): the keep best by
// (score desc, id asc).  MSB-first radix select with 8-bit digits over the
// block; stops as soon as the selected digit's bin holds exactly the keys
// still needed.  Afterwards sel96_take(key) says whether a key is selected.
struct Sel96 {
  uint64_t phi, mhi;
  uint32_t plo, mlo, need, done;
};

template <class Get>
__device__ void select96(Get get, uint64_t n, uint32_t keep, uint64_t nvalid, uint32_t* hist,
                         Sel96& s) {
  __shared__ unsigned long long s_min, s_max;
  __shared__ uint32_t s_lmin, s_lmax;
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
  if (tid == 0) {
    s.phi = 0;
    s.mhi = 0;
    s.plo = 0;
    s.mlo = 0;
    s.need = keep;
    s.done = keep >= nvalid ? 1u : 0u;  // everything valid is selected
    s_min = ~0ull;
    s_max = 0ull;
    s_lmin = ~0u;
    s_lmax = 0u;
  }
  __syncthreads();
  if (s.done) return;
  // The keys of one query's chunk share their leading bytes (coarse score +
  // a small residual score): start the digit passes below the common prefix
  // of the smallest and largest key, which every key in between shares.
  {
    unsigned long long mn = ~0ull, mx = 0ull;
    for (uint64_t i = tid; i < n; i += nthr) {
      uint64_t h;
      uint32_t l;
      if (!get(i, h, l)) continue;
      mn = min(mn, static_cast<unsigned long long>(h));
      mx = max(mx, static_cast<unsigned long long>(h));
    }
    atomicMin(&s_min, mn);
    atomicMax(&s_max, mx);
  }
  __syncthreads();
  int pass0 = 0;
  const uint64_t hmin = s_min, hmax = s_max;
  if (hmin == hmax) {
    uint32_t mn = ~0u, mx = 0u;
    for (uint64_t i = tid; i < n; i += nthr) {
      uint64_t h;
      uint32_t l;
      if (!get(i, h, l)) continue;
      mn = min(mn, l);
      mx = max(mx, l);
    }
    atomicMin(&s_lmin, mn);
    atomicMax(&s_lmax, mx);
    __syncthreads();
    const uint32_t x = s_lmin ^ s_lmax;
    const int lb = x ? __clz(x) / 8 : 4;  // common leading bytes of lo
    pass0 = 8 + lb;
    if (tid == 0) {
      s.phi = hmin;
      s.mhi = ~0ull;
      const uint32_t m = lb == 0 ? 0u : (lb >= 4 ? ~0u : ~0u << (32 - 8 * lb));
      s.plo = s_lmin & m;
      s.mlo = m;
    }
  } else {
    const int hb = __clzll(static_cast<long long>(hmin ^ hmax)) / 8;  // common leading bytes of hi
    pass0 = hb;
    if (tid == 0 && hb > 0) {
      const uint64_t m = ~0ull << (64 - 8 * hb);
      s.phi = hmin & m;
      s.mhi = m;
    }
  }
  __syncthreads();
  for (int pass = pass0; pass < 12; ++pass) {
    if (s.done) break;  // block-uniform (read after a barrier)
    for (uint32_t i = tid; i < 256; i += nthr) hist[i] = 0;
    __syncthreads();
    const uint64_t phi = s.phi, mhi = s.mhi;
    const uint32_t plo = s.plo, mlo = s.mlo;
    // whole warps iterate together so the increments can be warp-aggregated
    const uint64_t nr = (n + 31) & ~31ull;
    for (uint64_t i = tid; i < nr; i += nthr) {
      uint32_t dg = 0x100u;  // no increment
      uint64_t h;
      uint32_t l;
      if (i < n && get(i, h, l) && (h & mhi) == phi && (l & mlo) == plo)
        dg = pass < 8 ? static_cast<uint32_t>(h >> (56 - 8 * pass)) & 0xFFu
                      : (l >> (24 - 8 * (pass - 8))) & 0xFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dg);
      if (dg != 0x100u && lane == static_cast<uint32_t>(__ffs(peers) - 1))
        atomicAdd(&hist[dg], static_cast<uint32_t>(__popc(peers)));
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t need = s.need;
      uint32_t cum = 0;
      int sel = 255;
      for (; sel > 0; --sel) {
        if (cum + hist[sel] >= need) break;
        cum += hist[sel];
      }
      const uint32_t cnt = hist[sel];
      s.need = need - cum;
      if (pass < 8) {
        s.phi |= static_cast<uint64_t>(sel) << (56 - 8 * pass);
        s.mhi |= 0xFFull << (56 - 8 * pass);
      } else {
        s.plo |= static_cast<uint32_t>(sel) << (24 - 8 * (pass - 8));
        s.mlo |= 0xFFu << (24 - 8 * (pass - 8));
      }
      if (cnt == s.need) s.done = 1u;
    }
    __syncthreads();
  }
}

// select96 for one warp (no block barriers): the same MSB-first digit passes
// over n <= a few hundred keys, a per-warp 256-bin histogram, the digit found
// with a lane-parallel suffix scan.  The result s is identical to select96's.
template <class Get>
__device__ void warp_select96(Get get, uint32_t n, uint32_t keep, uint32_t nvalid, uint32_t* hist, Sel96& s) {
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t phi = 0, mhi = 0;
  uint32_t plo = 0, mlo = 0, need = keep;
  bool done = keep >= nvalid;
  int pass0 = 0;
  if (!done) {
    unsigned long long mn = ~0ull, mx = 0ull;
    for (uint32_t i = lane; i < n; i += 32) {
      uint64_t h;
      uint32_t l;
      if (!get(i, h, l)) continue;
      mn = min(mn, static_cast<unsigned long long>(h));
      mx = max(mx, static_cast<unsigned long long>(h));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    if (mn == mx) {
      uint32_t lmn = ~0u, lmx = 0u;
      for (uint32_t i = lane; i < n; i += 32) {
        uint64_t h;
        uint32_t l;
        if (!get(i, h, l)) continue;
        lmn = min(lmn, l);
        lmx = max(lmx, l);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lmn = min(lmn, __shfl_xor_sync(0xFFFFFFFFu, lmn, o));
        lmx = max(lmx, __shfl_xor_sync(0xFFFFFFFFu, lmx, o));
      }
      const uint32_t x = lmn ^ lmx;
      const int lb = x ? __clz(x) / 8 : 4;
      pass0 = 8 + lb;
      phi = mn;
      mhi = ~0ull;
      mlo = lb == 0 ? 0u : (lb >= 4 ? ~0u : ~0u << (32 - 8 * lb));
      plo = lmn & mlo;
    } else {
      const int hb = __clzll(static_cast<long long>(mn ^ mx)) / 8;
      pass0 = hb;
      if (hb > 0) {
        mhi = ~0ull << (64 - 8 * hb);
        phi = mn & mhi;
      }
    }
  }
  for (int pass = pass0; pass < 12 && !done; ++pass) {
    for (uint32_t i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
      uint64_t h;
      uint32_t l;
      if (get(i, h, l) && (h & mhi) == phi && (l & mlo) == plo) {
        const uint32_t dg = pass < 8 ? static_cast<uint32_t>(h >> (56 - 8 * pass)) & 0xFFu
                                     : (l >> (24 - 8 * (pass - 8))) & 0xFFu;
        atomicAdd(&hist[dg], 1u);
      }
    }
    __syncwarp();
    // lane t owns bins 255-8t .. 248-8t (top first)
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = hist[255 - 8 * lane - k];
      sum += v[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += t;
    }
    const uint32_t hit = __ballot_sync(0xFFFFFFFFu, incl >= need);
    const uint32_t L = hit ? __ffs(hit) - 1u : 31u;
    uint32_t sel = 0, cnt = 0, cum = 0;
    if (lane == L) {
      cum = incl - sum;
      int k = 0;
      for (; k < 7; ++k) {
        if (cum + v[k] >= need) break;
        cum += v[k];
      }
      sel = 255 - 8 * lane - k;
      cnt = v[k];
    }
    sel = __shfl_sync(0xFFFFFFFFu, sel, L);
    cnt = __shfl_sync(0xFFFFFFFFu, cnt, L);
    cum = __shfl_sync(0xFFFFFFFFu, cum, L);
    need -= cum;
    if (pass < 8) {
      phi |= static_cast<uint64_t>(sel) << (56 - 8 * pass);
      mhi |= 0xFFull << (56 - 8 * pass);
    } else {
      plo |= sel << (24 - 8 * (pass - 8));
      mlo |= 0xFFu << (24 - 8 * (pass - 8));
    }
    if (cnt == need) done = true;
    __syncwarp();
  }
  s.phi = phi;
  s.mhi = mhi;
  s.plo = plo;
  s.mlo = mlo;
  s.need = need;
  s.done = 1u;
}

__device__ __forceinline__ bool sel96_take(const Sel96& s, uint64_t hi, uint32_t lo) {
  const uint64_t mh = hi & s.mhi;
  const uint32_t ml = lo & s.mlo;
  return mh > s.phi || (mh == s.phi && ml >= s.plo);
}

}  // namespace
}  // namespace pcpqg
