// K1' — the LUT build as a tcgen05 tensor-core contraction (large query
// batches, tolerance mode).
//
//   eta[q][j][c] = <q_j, C_j[c]>  for a tile of 128 queries x all k centers of
//   section j is a [128 x K] . [k x K]^T product with K = dbar.  fp32 inputs are
//   split into two tf32 halves (x = x_hi + x_lo, both round-to-nearest tf32) and
//   the four partial products are laid side by side along K:
//       A row (query)  = [q_hi | q_hi | q_lo | q_lo]      (4*dbar, zero-padded to 8)
//       B row (center) = [c_hi | c_lo | c_hi | c_lo]
//   so one accumulation in TMEM yields q_hi.c_hi + q_hi.c_lo + q_lo.c_hi + q_lo.c_lo
//   = <q, c> to ~2^-22 relative per term (tf32 keeps 11 significant bits; the
//   split keeps 22).  This is NOT the reference's sequential fp32 fold
//   (pq_index.cpp:186-190): scores built from these tables agree with the
//   reference to ~1e-6 of max|score|, inside the north-star tolerance of 1e-5;
//   the exact CUDA-core LUT (lut_kernel) stays the default.
//
// One CTA (4 warps) per (query tile, section): all threads stage the split
// operands in shared memory in the UMMA canonical K-major layout (no swizzle:
// 8-row x 16-byte core matrices), warp 0 allocates TMEM, one thread issues
// tcgen05.mma.kind::tf32 (M=128, N=k, K=8 per instruction) and commits to an
// mbarrier, then every warp drains its 32 TMEM lanes (= its 32 queries) with
// tcgen05.ld.32x32b and writes the rows in the scan's grouped table layout.
#include <cstdint>

#include "pcpqg_device.cuh"

namespace pcpqg {
namespace {

constexpr int kTcRows = 128;  // UMMA M = queries per tile

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Shared-memory matrix descriptor, K-major, SWIZZLE_NONE (canonical layout
// ((8,m),(4 tf32,2)) : ((16B, SBO), (4B, LBO))), SM100 version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format = F32
         | (2u << 7)          // a_format = TF32
         | (2u << 10)         // b_format = TF32
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

template <int KT>  // K extent (4*dbar rounded up to 8), 8 | 16 | 24 | 32
__global__ void __launch_bounds__(128)
    lut_tc_kernel(const float* __restrict__ Q, uint32_t B, uint32_t Bpad, uint32_t d,
                  const float* __restrict__ cb,
                  uint32_t m, uint32_t k, uint32_t dbar, int nq, int rs, uint64_t gstride,
                  float* __restrict__ eta) {
  // canonical K-major layout: byte(row, kk) = (kk/4) * LBO + row * 16 + (kk%4) * 4,
  // LBO = rows * 16 (next 16-byte K chunk), SBO = 128 (next 8-row core matrix)
  extern __shared__ __align__(128) float smem_tc[];
  float* sA = smem_tc;                      // KT/4 chunks x 128 rows x 4
  float* sB = smem_tc + KT * kTcRows;       // KT/4 chunks x k rows x 4
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t q0 = blockIdx.x * kTcRows, j = blockIdx.y;
  const uint64_t qrow = q0 + tid;  // this thread's query (= TMEM lane)

  if (j >= m) {  // padded sections of the grouped table: -0.0 rows
    if (qrow < Bpad) {
      const uint64_t g = qrow / nq, qi = qrow % nq;
      for (uint32_t c = 0; c < k; ++c) eta[g * gstride + (static_cast<uint64_t>(j) * k + c) * rs + qi] = -0.0f;
    }
    return;
  }
  // ---- stage A (queries) and B (centers) split operands
  {
    float v[KT];
#pragma unroll
    for (int i = 0; i < KT; ++i) v[i] = 0.0f;
    for (uint32_t a = 0; a < dbar; ++a) {
      const uint32_t col = j * dbar + a;
      const float x = (qrow < B && col < d) ? Q[qrow * d + col] : 0.0f;
      const float hi = tf32_rna(x), lo = tf32_rna(x - hi);
      v[a] = hi;
      v[dbar + a] = hi;
      v[2 * dbar + a] = lo;
      v[3 * dbar + a] = lo;
    }
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) sA[(kk / 4) * (kTcRows * 4) + tid * 4 + (kk % 4)] = v[kk];
  }
  for (uint32_t c = tid; c < k; c += blockDim.x) {
    float v[KT];
#pragma unroll
    for (int i = 0; i < KT; ++i) v[i] = 0.0f;
    for (uint32_t a = 0; a < dbar; ++a) {
      const float x = cb[(static_cast<uint64_t>(j) * k + c) * dbar + a];
      const float hi = tf32_rna(x), lo = tf32_rna(x - hi);
      v[a] = hi;
      v[dbar + a] = lo;
      v[2 * dbar + a] = hi;
      v[3 * dbar + a] = lo;
    }
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) sB[(kk / 4) * (k * 4) + c * 4 + (kk % 4)] = v[kk];
  }
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint32_t ncols = 32;
  while (ncols < k) ncols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (tid == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const uint32_t lboA = kTcRows * 16, lboB = k * 16;
    const uint32_t idesc = umma_idesc_tf32(kTcRows, k);
#pragma unroll
    for (int ks = 0; ks < KT / 8; ++ks) {  // K = 8 tf32 = two 16-byte chunks per instruction
      const uint64_t da = umma_desc(a0 + ks * 2 * lboA, lboA, 128);
      const uint64_t db = umma_desc(b0 + ks * 2 * lboB, lboB, 128);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  mbar_wait(&mbar, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- drain: warp w owns TMEM lanes 32w..32w+31 (its queries), 32 columns per load
  const uint64_t g = qrow / nq, qi = qrow % nq;
  for (uint32_t c0 = 0; c0 < k; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((warp * 32u) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (qrow < Bpad) {  // queries in [B, Bpad) get the zero rows of their zero inputs
      float* dst = eta + g * gstride + (static_cast<uint64_t>(j) * k + c0) * rs + qi;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c0 + i < k) dst[static_cast<uint64_t>(i) * rs] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  (void)lane;
}

}  // namespace

bool lut_tc_supported(const DeviceIndex& x) {
  return x.h.k >= 16 && x.h.k <= 256 && x.h.k % 16 == 0 && x.h.dbar <= 8;
}

void launch_lut_tc(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t Bpad, int nq, int rs,
                   uint32_t rows, float* eta, cudaStream_t st) {
  if (!lut_tc_supported(x)) fail(PCPQG_E_UNSUPPORTED, "tensor-core LUT needs 16 <= k <= 256, k % 16 == 0, dbar <= 8");
  const uint32_t kt = ((4 * x.h.dbar + 7) / 8) * 8;
  const uint32_t m8 = (x.h.m + 7) & ~7u;
  const dim3 grid((Bpad + kTcRows - 1) / kTcRows, m8);
  const size_t smem = static_cast<size_t>(kt) * (kTcRows + x.h.k) * 4;
  const uint64_t gs = group_stride(x, rs, rows);
  auto go = [&](auto kern) {
    PCPQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, 128, smem, st>>>(dQ, B, Bpad, x.h.d, x.d_codebooks, x.h.m, x.h.k, x.h.dbar, nq, rs, gs,
                                  eta);
  };
  switch (kt) {
    case 8: go(lut_tc_kernel<8>); break;
    case 16: go(lut_tc_kernel<16>); break;
    case 24: go(lut_tc_kernel<24>); break;
    default: go(lut_tc_kernel<32>); break;
  }
  PCPQG_CUDA(cudaGetLastError());
}

}  // namespace pcpqg
