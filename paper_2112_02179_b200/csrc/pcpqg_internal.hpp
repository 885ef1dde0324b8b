// Internal declarations shared by the host side (index load, C ABI) and the
// CUDA kernels of libpcpqg.so.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "pcpqg.h"

namespace pcpqg {

// Error with a pcpqg status code; converted to a status at the C boundary.
struct Error {
  int code;
  std::string what;
};
[[noreturn]] void fail(int code, const std::string& what);
void check_cuda(cudaError_t e, const char* where);
#define PCPQG_CUDA(call) ::pcpqg::check_cuda((call), #call)

// The device code stream is a sequence of 32-point blocks.  Inside a block
// the layout is word-major: word w of the 32 points is 128 contiguous bytes
// ([block][w][lane]), so a warp that owns a block loads each word with one
// fully coalesced 128-byte transaction.  A point's row is W 32-bit words:
//   JOINT8 : byte j = center | scale_code << cbits            (W = ceil(m/4))
//   PLANES : Wc center words (cw bits per section), then Ws scale words
//            (sw bits: 0 none, 4/8 scale codes, 16 fp16 alpha, 32 fp32 alpha)
constexpr int kBlockPts = 32;

struct HostIndex {  // parsed PCPQIDX1, point-major like pcpq::PQIndex
  uint32_t method = 0, n = 0, d = 0, padded_d = 0, m = 0, k = 0, scales = 0, dbar = 0;
  double t = 0.0;
  std::vector<float> codebooks;       // m*k*dbar
  std::vector<float> scalar_cb;       // m*scales
};

struct TcIndex;  // tensor-scan tables (pcpqg_tscan.cu)
void free_tc(TcIndex* t);

struct DeviceIndex {
  HostIndex h;
  uint64_t shard_begin = 0, n_local = 0;
  uint32_t n_blocks = 0;
  int device = 0;
  uint32_t format = 0;
  uint32_t cw = 0, sw = 0;   // PLANES widths; JOINT8: cw=cbits, sw=lbits
  uint32_t W = 0, Wc = 0;    // words per point, center words (PLANES)
  uint64_t code_bytes = 0;
  float* d_codebooks = nullptr;  // m*k*dbar
  float* d_lambda = nullptr;     // m8*max(scales,1), m8 = m rounded up to 8, pad rows 1.0
  uint32_t* d_codes = nullptr;   // n_blocks * W * 32
  // raw fp16 alpha layouts: per-section max |alpha| over the shard (K2-F bound
  // and eligibility), computed on first use
  // plan_search results by (B, topn, scores_only, options version)
  mutable std::mutex plan_mu;
  mutable std::map<std::tuple<uint32_t, uint32_t, bool, uint64_t>, struct SearchPlan*> plans;
  mutable std::once_flag amax_once;
  mutable std::vector<float> amax;  // [m8]
  mutable float* d_amax = nullptr;
  // K2-T tables (section scales, fp16 decode table), built on first use
  mutable std::once_flag tc_once;
  mutable TcIndex* tc = nullptr;
  ~DeviceIndex();
};
// fills x.amax / x.d_amax (raw fp16 alpha layouts; synchronises)
void ensure_alpha_max(const DeviceIndex& x);

// Keep the device's default stream-ordered memory pool cached across calls.
void keep_mempool(int device);

// Parse + validate a PCPQIDX1 image (pcpq::deserialize error classes and
// first-offending-byte order); body points at the first code row.
struct ParsedIndex {
  HostIndex h;
  const uint8_t* bytes = nullptr;  // the image (its first byte)
  const uint8_t* body = nullptr;
  uint64_t row = 0, cbytes = 0;  // bytes per code row, center-code bytes per row
  bool wide = false;             // two-byte center codes (k > 256)
};
ParsedIndex parse_index(const uint8_t* bytes, uint64_t len);
// The pieces of parse_index: header + codebooks (no code rows read) ...
ParsedIndex parse_header(const uint8_t* bytes, uint64_t len);
// ... the number of complete code rows present in `len` bytes ...
uint64_t full_rows_of(const ParsedIndex& P, uint64_t len);
// ... the error for a bad code at body byte `pos` (code_out_of_range) ...
[[noreturn]] void fail_bad_code(const ParsedIndex& P, uint64_t pos);
// ... and the checks after the complete rows: partial row codes, truncation,
// trailing bytes (in the reference's byte order); `tail` points at the bytes
// that follow the complete rows.
void check_tail(const ParsedIndex& P, uint64_t len, const uint8_t* tail);
// GPU ingest (pcpqg_ingest.cu): same validation and layout as load_index,
// with the code rows validated and repacked in HBM.
DeviceIndex* load_index_gpu(const uint8_t* bytes, uint64_t len, int device, uint64_t begin,
                            uint64_t end);
DeviceIndex* load_index_file_gpu(const char* path, int device, uint64_t begin, uint64_t end);
// Device code layout: JOINT8 when cbits + lbits <= 8, else PLANES.
struct CodeLayout {
  uint32_t format = 0, cw = 0, sw = 0, W = 0, Wc = 0;
};
CodeLayout choose_layout(uint32_t k, uint32_t scales, uint32_t m, bool fp16_exact_alphas);
bool alphas_fp16_exact(const ParsedIndex& P, uint64_t begin, uint64_t end);
// Repack points [begin, begin + n_local) into zeroed blocked words
// [ceil(n_local/32)][W][32] (word-interleaved by lane).
void repack(const ParsedIndex& P, const CodeLayout& L, uint64_t begin, uint64_t n_local,
            uint32_t* dst_words);

// Parse + validate (mirrors pcpq::deserialize error classes), repack the
// requested shard and upload it.
DeviceIndex* load_index(const uint8_t* bytes, uint64_t len, int device, uint64_t begin,
                        uint64_t end);
// A part image: the header and codebooks of an index of n points followed by
// the rows [row_begin, row_begin + count) only; ids stay global.
DeviceIndex* load_index_part(const uint8_t* bytes, uint64_t len, uint64_t row_begin, int device);
// Validate once, then load shard r = [r*n/ndev, (r+1)*n/ndev) on devices[r].
std::vector<DeviceIndex*> load_index_shards(const uint8_t* bytes, uint64_t len, const int* devices, int ndev);

// ---------------------------------------------------------------- IVF
// One cell of a PCPQIVF1 container on the device (see pcpqg_ivf.cu).
struct IvfCell {
  uint32_t n = 0, k = 0, raw = 0, pad = 0;  // members, cell k (PQ), raw-residual flag
  uint64_t block_off = 0;   // first 32-point block in the shared code stream (PQ)
  uint64_t member_off = 0;  // first id in the concatenated member lists
  uint64_t cb_off = 0;      // first float of the cell's codebooks [m][k][dbar] (PQ)
  uint64_t lam_off = 0;     // first float of the cell's scale codebooks [m8][max(s,1)] (PQ)
  uint64_t raw_off = 0;     // first float of the cell's residual rows [n][d] (raw)
};

struct DeviceIvf {
  uint32_t n = 0, d = 0, kbar = 0;
  int device = 0;
  // layout shared by every PQ cell (from the largest cell k)
  uint32_t m = 0, dbar = 0, padded_d = 0, scales = 0, k_max = 0, method = 0;
  uint32_t n_raw = 0, n_pq = 0, max_raw_pts = 0;
  uint64_t max_cell_blocks = 0, code_bytes = 0;
  CodeLayout lay;
  std::vector<uint32_t> cell_n;      // members per cell
  std::vector<uint32_t> cell_k;      // PQ cell k (0 for raw cells)
  std::vector<uint64_t> top_prefix;  // [p] = size of the p largest cells (pool bound)
  float* d_coarse = nullptr;         // [kbar][d]
  IvfCell* d_cells = nullptr;
  uint32_t* d_codes = nullptr;       // all PQ cells, blocked, layout `lay`
  float* d_cb = nullptr;
  float* d_lam = nullptr;
  float* d_raw = nullptr;
  uint32_t* d_members = nullptr;
  uint32_t* d_pcluster = nullptr;    // point -> cell
  uint32_t* d_pslot = nullptr;       // point -> position in its member list
  ~DeviceIvf();
};

// Parse + validate a PCPQIVF1 container (pcpq::deserialize_ivf error classes
// and order, proj/core/src/ivf.cpp:256-316) and upload it.
DeviceIvf* load_ivf(const uint8_t* bytes, uint64_t len, int device);
// query_ivf (ivf.cpp:89-153) for B device-resident queries; outputs [B][topn]
// (id -1 / NaN past counts[b]), short flags, requested scores [B][R], and
// optionally the probed cells [B][k_probe].  Arguments are validated by the caller.
void ivf_query(const DeviceIvf& v, const float* dQ, uint32_t B, uint32_t k_probe, uint32_t topn,
               const uint32_t* d_req, uint32_t R, int32_t* d_ids, double* d_scores,
               uint32_t* d_counts, uint8_t* d_short, double* d_req_scores, uint32_t* d_probes,
               cudaStream_t st);
// nonzero if any requested id is >= n (synchronises the stream)
uint32_t ivf_check_requested(const uint32_t* d_req, uint64_t cnt, uint32_t n, cudaStream_t st);

// ---------------------------------------------------------------- eval
// brute_force_topn (proj/core/src/eval.cpp:36-49) for B device queries over
// device points X [n][d]: ids [B][topn], exact double scores; synchronises.
void brute_force_topn(const float* dX, uint64_t n, uint32_t d, const float* dQ, uint32_t B,
                      uint32_t topn, int32_t* d_ids, double* d_scores, int device, cudaStream_t st);
// recall1_single (eval.cpp:57-66) per query: retrieved [B][R], exact top-1 [B]
void recall1(const float* dX, uint64_t n, uint32_t d, const float* dQ, uint32_t B,
             const uint32_t* d_ret, uint32_t R, const double* d_top1, int32_t* d_hits, cudaStream_t st);

// ---------------------------------------------------------------- training
// build_pq_index(method = kmeans) + serialize (pq_index.cpp:62-168, :372-407):
// the PCPQIDX1 image, byte-identical to the reference's.
std::vector<uint8_t> train_kmeans(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                  double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device);
// build_pq_index(method = pcpq) + serialize: projective_k_clustering per section
// (clustering.cpp:552-622), unit directions, quantize_projective or raw alphas.
std::vector<uint8_t> train_pcpq(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                bool quantize, double t_frac, uint32_t max_iters, double tol, uint64_t seed,
                                int device);

// build_pq_index(method = aniso / apcpq) + serialize: the score-aware solver
// (clustering.cpp:622-722) per section with fixed (aniso) or optimal (apcpq)
// scales, then quantize_anisotropic (scalar_quant.cpp:72-150) or raw alphas.
// The m sections are independent problems: they are dealt round-robin to the
// ndev devices (one host thread each), so a multi-GPU build exchanges nothing
// until the image is assembled and is byte-identical for every device list.
std::vector<uint8_t> train_aniso(const float* X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                                 bool scaling, bool quantize, double t_frac, uint32_t max_iters, double tol,
                                 uint64_t seed, const int* devices, int ndev);
// wall seconds of the last training call on this thread: prep (validation,
// sections, seeds, weights), Lloyd iterations, scales, serialization
extern thread_local double g_train_phases[4];
// aniso_weights (clustering.cpp:204-217) for every row of x [n][dbar] with a
// nonzero norm (zero rows get {0, 0}), on host threads with the C library's
// sin, as the reference computes them
void aniso_weights_host(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot);
// The same weights on the GPU (pcpqg_weights.cu): one thread per row, the host C
// library's sin restated bit for bit (pcpqg_hostsin.cuh).
//   sin_port_mismatches(-1 | device): the restatement on the host / the compiled
//     kernel on `device` against std::sin over the fixed self-check arguments
//   aniso_weights_gpu_ok: both are 0 (cached per device)
//   launch_aniso_weights: device rows in, device weights out
//   aniso_weights_gpu: host rows in, host weights out; fails (unsupported) when
//     the self-check does not pass
uint64_t sin_port_mismatches(int device, uint64_t* total = nullptr);
bool aniso_weights_gpu_ok(int device);
void launch_aniso_weights(const float* dX, uint64_t n, uint32_t dbar, double t, double* dHp, double* dHb,
                          cudaStream_t st);
void aniso_weights_gpu(const float* x, uint64_t n, uint32_t dbar, double t, double* h_par, double* h_bot,
                       int device);
// 1 when the last train_aniso call on this thread computed its weights on the GPU
extern thread_local int g_train_weights_gpu;

// ---------------------------------------------------------------- kernels
struct SearchPlan {
  int nq = 16;        // queries per CTA group (template NQ)
  int rs = 18;        // eta row stride in floats (see rs_of)
  uint32_t groups = 0, ctas_x = 0;  // grid: (groups, ctas_x)
  uint32_t cap = 0;   // per-query candidate buffer: K + threads*ppt
  int threads = 256;  // CTA size
  uint32_t ppt = 1;   // points per thread per code tile
  uint32_t stages = 2;  // TMA pipeline depth
  size_t smem = 0;
  uint32_t topn = 0;  // effective per-list K
  bool table = false; // JOINT8 read through a pre-multiplied eta*lambda table
  uint32_t rows = 0;  // table rows per section: k, or 2^(cbits+lbits) in table mode
  bool ws = false;    // warp-specialised scan: threads = compute threads + 1 producer warp
  bool filter = false;  // fp16 pre-score filter (K2-F) in front of the exact score
};

SearchPlan plan_search(const DeviceIndex& x, uint32_t B, uint32_t topn, bool scores_only);

// LUT build on device.  layout_grouped: eta[(g*m*k + j*k + c)*rs + qi]
// (q = g*nq + qi); otherwise plain eta[q*m*k + j*k + c].  Queries >= B get 0.
// mode 0: plain eta[q][j][c]; 1: grouped eta rows for the scan; 2: grouped
// pre-multiplied eta*lambda rows indexed by the JOINT8 code byte.
// zero / nzero: u64 words the kernel also clears (the scan's shared K-th keys)
void launch_lut(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t Bpad, int nq, int rs,
                int mode, uint32_t rows, float* eta, cudaStream_t st, uint64_t* zero = nullptr,
                uint32_t nzero = 0);
// K1' tensor-core LUT build (tolerance mode, pcpqg_lut_tc.cu)
bool lut_tc_supported(const DeviceIndex& x);
void launch_lut_tc(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t Bpad, int nq, int rs,
                   uint32_t rows, float* eta, cudaStream_t st);
// process-wide options (pcpqg_set_option)
struct Options {
  int lut_tensor_cores = 0;  // 1: tcgen05 LUT build for batches >= 128 (tolerance mode)
  int fused_merge = 0;       // 1: merge inside the scan's last CTA per query group
  int scan_ws = 1;            // warp-specialised scan for small query groups
  int scan_ws_max_nq = 4;     // ... of at most this many queries
  int merge_wide = 1;         // block-parallel sorted merge for batches < #SMs
  int scan_lut_fused = 1;     // small batches: the warp-specialised scan builds its tables itself (no LUT kernel)
  int merge_oneshot = 1;      // ... with every list staged whole in one round trip (merge_oneshot_kernel)
  int pdl = 1;                // programmatic dependent launch between LUT, small-batch scan and merge
  int gt_chunk = 0;           // !=0: points per chunk of brute_force_topn
  int gt_tc = 1;              // brute_force_topn: tensor-core pre-score filter (exact results)
  int gt_tc_min_batch = 4;    // ... for batches of at least this many queries
  int scan_shape = 0;        // !=0: force the scan shape threads*10000 + ppt*100 + stages
  // K2-F, the fp16 CUDA-core pre-score filter (exact results).  Opt-in since the last session of round 2:
  // K2-T serves the batches it was built for, and a stress run (tools/stress_mix.py: C2, batch sizes 1..255
  // in turn, L2 flushed between calls) hung inside its scan kernel in ~1 of 5 runs, while the exact scans
  // and K2-T passed 37 of 37 (profiles/r02_k2f_stress.md); the cause was not found
  int scan_filter = 0;
  int ivf_grouped = 1;        // IVF batched multi-cell scan for batches with several queries per cell
  int scan_tc = 1;            // K2-T: tensor-core pre-score filter for batch scans (exact results)
  int scan_tc_min_batch = 8;  // ... for batches of at least this many queries
  // ... with at least this many (query, point) pairs, or 256 queries: K2-T has ~0.1 ms of fixed cost
  // (prep, seed pass, finish) plus one pass over the operand cache whatever B is, the CUDA-core scans
  // cost ~ n * B; measured crossover: B ~ 80 at C1 (n = 1e5), B ~ 7 at C2 and C3 (tools/ab_midbatch.py,
  // profiles/r02_midbatch.md)
  int64_t scan_tc_min_work = 8000000;
  int scan_tc_qh = 0;         // K2-T: hi/lo fp16 query operand for kpad <= 112 (halves eps; measured slower at C2: opt-in)
  int scan_tc_at = 1;         // K2-T: query operand in TMEM for long K (kpad >= 192)
  int scan_tc_qt = 2;         // K2-T: query tiles (of 128) per CTA sharing each point tile (1 | 2)
  int scan_tc_cs = 1;         // K2-T: Cauchy-Schwarz error bound from the operand cache's largest norm
  int scan_tc_exp = 0;        // kernel experiments (wrong results): 1 = no epilogue work, 2 = no candidate appends
  int scan_tc_fin_small = 0;  // K2-T finish kernel: 2048-key staging buffer when the expected lists fit (opt-in: C2 rescore 0.67 -> 0.55 ms, but lists beyond it fall to the exact scan: minutes on the trained index)
  int scan_tc_diag = 0;       // 1: print K2-T list statistics (synchronises)
  int scan_tc_cache_pct = 40;  // K2-T decoded operand cache: built when it needs <= this % of free HBM (0: off)
  int train_level_sort = 1;   // scale quantizer: per-level sums through a stable counting sort (s <= 16)
  int weights_gpu = 1;        // anisotropic weights on the GPU when its sin reproduces the host's bits
  int scan_tc_seed_max = 1 << 20;  // ... and at most this many points
  int scan_tc_seed = 16;      // K2-T seed sample: one point in scan_tc_seed (evenly spread blocks); 0 = no seed
};
Options& options();
// pcpqg_set_profiling state, and the stage times pcpqg_last_timings returns
bool profiling_enabled();
void set_last_timings(const float* t3);
// bumped by every option change (keys the per-index plan cache)
uint64_t options_version();
void bump_options_version();
void launch_eta_lambda(const DeviceIndex& x, const float* eta_plain, uint32_t B, float* etal,
                       cudaStream_t st);
// Fused scan + per-CTA top-K (partial keys [ctas_x][Bpad][K]) or, with
// scores != nullptr, the plain score_all output [B][n_local].
// Final rows written by the scan itself: the last CTA of each query group
// merges the group's per-CTA lists (done: [groups] tickets, zeroed).
struct FusedMerge {
  uint32_t* pcnt = nullptr;  // [ctas_x][Bpad] survivor counts
  uint32_t* done = nullptr;
  uint64_t* keys = nullptr;
  int32_t* ids = nullptr;
  float* scores = nullptr;
  uint32_t out_stride = 0;
};
// Filter tables (plan.filter) built from the grouped eta tables: eta_hat
// [groups][fgstride] halves, lambda_hat [m8][s] halves, (sigma, eps) [Bpad].
struct FilterTables {
  __half* fh = nullptr;
  __half* flam = nullptr;
  float2* fse = nullptr;
  float* work = nullptr;  // [2 * m8] section scales
  unsigned long long* count = nullptr;  // diagnostics (scan_filter = 3): points scored exactly
  uint64_t* carry = nullptr;       // [groups*ctas_x*16][K] top-K handed to the next range
  uint32_t* carry_cnt = nullptr;   // [groups*ctas_x*16]
  uint32_t* carry_done = nullptr;  // [groups*ctas_x], zeroed before the scan
};
uint64_t filter_group_stride(const DeviceIndex& x);
void launch_filter_tables(const DeviceIndex& x, const SearchPlan& p, const float* eta_grouped,
                          const FilterTables& ft, cudaStream_t st);
void launch_scan(const DeviceIndex& x, const SearchPlan& p, const float* eta_grouped, uint32_t B,
                 uint64_t* partial, uint64_t* gtau, float* scores, cudaStream_t st,
                 const FusedMerge* fm = nullptr, const FilterTables* ft = nullptr, const float* dQ = nullptr);
// Merge L lists of K keys per query (layout [L][in_rows][K]) into rows of
// out_stride keys for queries [0, B): keys_out [B][out_stride] and/or decoded
// ids / scores.  gtau (optional, [B]) is a lower bound on each query's final
// K-th key used to drop hopeless keys early.
void merge_lists(const uint64_t* keys, uint32_t L, uint32_t in_rows, uint32_t B, uint32_t K,
                 uint32_t out_stride, const uint64_t* gtau, uint64_t* keys_out, int32_t* ids,
                 float* scores, cudaStream_t st, uint32_t keep = 0);
// Merge of lists sorted descending ([L][in_rows][Ks]; counts optional, else a
// list ends at its first empty key) by a K-step warp tournament per query.
void merge_sorted_lists(const uint64_t* keys, const uint32_t* counts, uint32_t L, uint32_t in_rows,
                        uint32_t B, uint32_t Ks, uint32_t Kout, uint32_t out_stride,
                        uint64_t* keys_out, int32_t* ids, float* scores, cudaStream_t st);
uint64_t group_stride(const DeviceIndex& x, int rs, uint32_t rows);

// encode kernels
void launch_assign_projective(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                              uint32_t k, uint32_t* assign, double* alpha, double* loss,
                              cudaStream_t st);
void launch_assign_anisotropic(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                               uint32_t k, const double* hp, const double* hb, const uint32_t* prev,
                               uint32_t* assign, double* alpha, double* loss, cudaStream_t st,
                               bool scaling = true);
void launch_center_stats(const float* x, uint64_t n, uint32_t dbar, uint32_t nsec,
                         uint64_t sec_stride, const uint32_t* assign, const double* alpha,
                         const double* hp, const double* hb, uint32_t k, const double* init,
                         double* stats, cudaStream_t st);
void launch_aniso_alpha_codes(const float* x, uint64_t n, uint32_t dbar, const float* centers,
                              const uint32_t* assign, const double* hp, const double* hb,
                              const float* values, uint32_t s, uint8_t* codes, cudaStream_t st);

int num_sms(int device);

// ---------------------------------------------------------------- K2-T
// device scratch for one call (stream-ordered, freed after the call)
using ScratchAlloc = std::function<void*(size_t)>;
struct TcPlan {
  uint32_t N = 0, qtiles = 0, ranges = 0, tiles_per_range = 0;
};
// the tensor-core filter scan applies (layout, batch, K <= 256, options)
bool tscan_eligible(const DeviceIndex& x, uint32_t B, uint32_t K);
TcPlan tscan_plan(const DeviceIndex& x, uint32_t B, uint32_t K);
// K2-T search: rows [B][out_stride] of the exact top-K (keys / ids / scores,
// each optional); stage_ms (optional, synchronises): prep, filter, finish
// GT-T: brute_force_topn's approximate pass on the tensor cores (pcpqg_tscan.cu):
// the raw points as fp16 operands through the K2-T filter kernel, the surviving
// pairs re-scored in the reference's fp64 order.  gt_stats: the data set's
// scaling scalars (device, gt_stats_bytes() bytes).  gt_tscan_chunk: one point
// chunk -> per query its exact top-K (global ids, scores, count), or
// fallback[b] = 1 where the caller must score the chunk exactly.
bool gt_tscan_eligible(uint64_t n, uint32_t d, uint32_t B, uint32_t K, int device);
uint64_t gt_tscan_chunk_points(uint64_t n, uint32_t d, int device);
size_t gt_stats_bytes();
void gt_stats(const float* dX, uint64_t n, uint32_t d, void* d_stats, cudaStream_t st);
void gt_tscan_chunk(const float* dXc, uint64_t pc, uint64_t p0, uint32_t d, const float* dQ, uint32_t B, uint32_t K,
                    const void* d_stats, uint32_t* out_ids, double* out_scores, uint32_t* out_count,
                    uint32_t out_stride, uint32_t count_stride, uint32_t* fallback, int device, ScratchAlloc alloc,
                    cudaStream_t st, float* stage_ms);
void tscan_search(const DeviceIndex& x, const float* dQ, uint32_t B, uint32_t K, uint32_t out_stride,
                  uint64_t* d_keys, int32_t* d_ids, float* d_scores, ScratchAlloc alloc, cudaStream_t st,
                  float* stage_ms);

}  // namespace pcpqg
