/* pcpqg — B200-native query-time scoring path for projective-clustering
 * product quantization (PCPQ, arXiv 2112.02179).  Plain C ABI: no exceptions,
 * no C++/torch types, plain pointers and sizes.
 *
 * Every entry point replaces (or, for the batched ones, extends) a piece of
 * the reference C++ API in namespace pcpq (/root/reference/proj):
 *
 *   pcpqg_index_load / _load_file  <- pcpq::deserialize / read_pq_index
 *                                     (core/src/pq_index.cpp:409-488, :499-505)
 *                                     + repack into the device code stream
 *   pcpqg_build_lut                <- pcpq::build_lookup_table
 *                                     (core/src/pq_index.cpp:170-210)
 *   pcpqg_score_all                <- pcpq::score_all / score_query
 *                                     (core/src/pq_index.cpp:212-250)
 *   pcpqg_search[_device]          <- the flat query loop of tools/main.cpp:229-243
 *                                     (score_query + partial_sort by (score desc,
 *                                     id asc)), batched over B queries, fused
 *   pcpqg_merge_device             <- no reference equivalent (its analogue is the
 *                                     global partial_sort): merges per-shard top-n
 *   pcpqg_counters                 <- pcpq::ScoreCounters (core/include/pcpq/pq_index.hpp:49-55)
 *   pcpqg_logical_payload_bits     <- pcpq::logical_payload_bits (core/src/pq_index.cpp:40-44)
 *   pcpqg_assign_projective        <- pcpq::assign_projective (core/src/clustering.cpp:250-289)
 *   pcpqg_assign_anisotropic       <- pcpq::assign_anisotropic(allow_scaling=true)
 *                                     (core/src/clustering.cpp:298-368)
 *   pcpqg_aniso_alpha_codes        <- quantize_anisotropic's code assignment
 *                                     (core/src/scalar_quant.cpp:121-150)
 *   pcpqg_center_stats             <- the member sums of pcpq::center_anisotropic
 *                                     (core/src/clustering.cpp:382-402)
 *   pcpqg_ivf_load / _load_file    <- pcpq::deserialize_ivf / read_ivf_index
 *                                     (core/src/ivf.cpp:256-316, :325-335)
 *   pcpqg_ivf_query[_device]       <- pcpq::query_ivf (core/src/ivf.cpp:89-153),
 *                                     batched over B queries
 *   pcpqg_brute_force_topn[_device]<- pcpq::brute_force_topn (core/src/eval.cpp:36-49)
 *   pcpqg_recall1[_device]         <- pcpq::recall1_single (core/src/eval.cpp:57-66)
 *   pcpqg_train_kmeans / _pcpq / _aniso <- pcpq::build_pq_index(method = kmeans / pcpq / aniso,apcpq)
 *                                  + serialize (pq_index.cpp:62-168, :372-407)
 *   pcpqg_aniso_weights[_gpu]      <- pcpq::aniso_weights (clustering.cpp:204-217)
 *                                     (core/src/pq_index.cpp:62-168, :372-407)
 *
 * Status: 0 on success, otherwise pcpq::errc + 1 (core/include/pcpq/types.hpp:14-23)
 * or one of the PCPQG_E_* codes >= 100.  The message of the last failure on the
 * calling thread is returned by pcpqg_last_error().
 *
 * Numerics: scores are bit-identical to the reference CPU path (same fp32
 * operations in the same order, no FMA contraction), so top-n lists are
 * identical including the (score desc, id asc) tie rule.
 */
#ifndef PCPQG_H
#define PCPQG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PCPQG_OK = 0,
  PCPQG_E_USAGE = 1,
  PCPQG_E_DATA = 2,
  PCPQG_E_NUMERIC = 3,
  PCPQG_E_BAD_MAGIC = 4,
  PCPQG_E_BAD_VERSION = 5,
  PCPQG_E_TRUNCATED = 6,
  PCPQG_E_CODE_OUT_OF_RANGE = 7,
  PCPQG_E_SIZE_MISMATCH = 8,
  PCPQG_E_CUDA = 100,        /* CUDA runtime failure (message has the detail) */
  PCPQG_E_UNSUPPORTED = 101  /* valid request outside this build's limits */
};

/* Device code-stream layouts. */
enum {
  PCPQG_FMT_JOINT8 = 1, /* one byte per section: center | scale_code << cbits */
  PCPQG_FMT_PLANES = 2  /* center plane (4/8/16 bit) + scale plane (0/4/8 bit codes,
                           16 = fp16-exact raw alpha, 32 = fp32 raw alpha) */
};

typedef struct pcpqg_index pcpqg_index;

typedef struct pcpqg_info {
  uint32_t method, n, d, padded_d, m, k, scales, dbar; /* PCPQIDX1 header */
  double t;
  uint64_t shard_begin, shard_end; /* global ids [begin, end) resident on this handle */
  uint32_t format;                 /* PCPQG_FMT_* */
  uint32_t center_bits, scale_bits;/* plane widths (JOINT8: cbits, lbits) */
  uint32_t words_per_point;        /* 32-bit words per point in the code stream */
  uint64_t code_bytes;             /* bytes of the resident code stream */
  int device;
} pcpqg_info;

const char *pcpqg_last_error(void);

/* Parse + validate a PCPQIDX1 image (same checks and error classes as
 * pcpq::deserialize), repack points [shard_begin, shard_end) into the device
 * layout and upload them to `device`.  shard_end == 0 means "to the end".
 * Ids reported by search are global (shard_begin + local). */
int pcpqg_index_load(const uint8_t *bytes, uint64_t len, int device, uint64_t shard_begin,
                     uint64_t shard_end, pcpqg_index **out);
int pcpqg_index_load_file(const char *path, int device, uint64_t shard_begin,
                          uint64_t shard_end, pcpqg_index **out);
/* The same load with the code rows validated and repacked on the GPU
 * (SURVEY §8(f) row 2): the rows stream to HBM through pinned buffers; errors
 * and the resulting device layout are identical to pcpqg_index_load. The
 * _file variant streams the file without holding it in host memory. */
int pcpqg_index_load_gpu(const uint8_t *bytes, uint64_t len, int device, uint64_t shard_begin,
                         uint64_t shard_end, pcpqg_index **out);
int pcpqg_index_load_file_gpu(const char *path, int device, uint64_t shard_begin,
                              uint64_t shard_end, pcpqg_index **out);
/* Load one shard from a PART image: the PCPQIDX1 header and codebooks of an
 * index of n points followed only by its rows [row_begin, row_begin + count),
 * count = (len - header bytes) / row bytes.  The rows are validated like
 * pcpq::deserialize validates a whole index (proj/core/src/pq_index.cpp:455-488:
 * code_out_of_range; bytes past the last whole row: size_mismatch); ids stay
 * global (shard_begin = row_begin).  For sharded deployments in which each
 * rank holds only its own rows. */
int pcpqg_index_load_part(const uint8_t *bytes, uint64_t len, uint64_t row_begin, int device,
                          pcpqg_index **out);
/* ---- one index sharded over several GPUs of this process (SURVEY §8(b),
 * §8(e)).  Shard r = points [r*n/ndev, (r+1)*n/ndev) is resident on
 * devices[r] (the image is validated once, like pcpq::deserialize).
 * pcpqg_multi_search runs the fused search on every device, gathers the
 * per-shard top-n key rows (global ids) on devices[0] and merges them there:
 * the result equals pcpqg_search on the whole index, i.e. the reference's
 * score_query + partial_sort (proj/core/src/pq_index.cpp:246-250,
 * proj/tools/main.cpp:229-243).  Transport of the gather: NCCL AllGather
 * (ncclCommInitAll over the devices, grouped calls; needs distinct devices
 * and libnccl.so.2) or peer copies (cudaMemcpyPeerAsync, NVLink P2P where
 * enabled; also serves repeated devices).  AUTO picks NCCL when possible. */
typedef struct pcpqg_multi pcpqg_multi;
enum { PCPQG_TRANSPORT_AUTO = 0, PCPQG_TRANSPORT_NCCL = 1, PCPQG_TRANSPORT_PEER = 2 };
int pcpqg_multi_load(const uint8_t *bytes, uint64_t len, const int *devices, int ndev, int transport,
                     pcpqg_multi **out);
void pcpqg_multi_free(pcpqg_multi *h);
/* out4: n, device count, transport in use (NCCL / PEER), d */
int pcpqg_multi_info(const pcpqg_multi *h, uint64_t *out4);
/* Host queries Q [B][d] -> ids / scores [B][topn] (synchronous). */
int pcpqg_multi_search(const pcpqg_multi *h, const float *Q, uint32_t B, uint32_t d, uint32_t topn,
                       int32_t *ids, float *scores);

/* Copy the device code stream (code_bytes of pcpqg_info) to host memory. */
int pcpqg_index_codes(const pcpqg_index *idx, void *out, uint64_t bytes);
void pcpqg_index_free(pcpqg_index *idx);
int pcpqg_index_info(const pcpqg_index *idx, pcpqg_info *out);

/* Host-buffer parity entry points (synchronous). */
/* eta: B*m*k floats, eta_lambda: B*m*k*scales floats (NULL to skip). counters
 * (5 x u64, may be NULL) accumulate like pcpq::ScoreCounters for B queries. */
int pcpqg_build_lut(const pcpqg_index *idx, const float *Q, uint32_t B, uint32_t d, float *eta,
                    float *eta_lambda, uint64_t *counters);
/* scores: B * (shard_end - shard_begin) floats, row-major by query. */
int pcpqg_score_all(const pcpqg_index *idx, const float *Q, uint32_t B, uint32_t d,
                    float *scores, uint64_t *counters);

/* Batched fused search over host buffers: H2D of Q, LUT build, fused
 * scan + top-n, merge, D2H of the result.  topn_eff = min(topn, shard size);
 * slots beyond it get id -1 and score -inf.  ids/scores: B*topn.  Non-finite
 * query values are rejected with PCPQG_E_DATA. */
int pcpqg_search(const pcpqg_index *idx, const float *Q, uint32_t B, uint32_t d, uint32_t topn,
                 int32_t *ids, float *scores);

/* Same on device-resident buffers, stream-ordered (no host synchronisation).
 * d_ids / d_scores / d_keys may each be NULL.  d_keys receives B*topn packed
 * 64-bit keys for a later cross-shard pcpqg_merge_device. */
int pcpqg_search_device(const pcpqg_index *idx, const float *dQ, uint32_t B, uint32_t d,
                        uint32_t topn, int32_t *d_ids, float *d_scores, uint64_t *d_keys,
                        void *cuda_stream);

/* Merge L lists of per-query top-n keys laid out [L][B][topn] (e.g. the
 * all-gathered per-shard results) into the global top-n. */
int pcpqg_merge_device(const uint64_t *d_keys, uint32_t L, uint32_t B, uint32_t topn,
                       int32_t *d_ids, float *d_scores, uint64_t *d_keys_out, int device,
                       void *cuda_stream);

/* Analytic ScoreCounters for scoring B queries against the resident shard. */
int pcpqg_counters(const pcpqg_index *idx, uint32_t B, uint64_t *out5);
/* The scan plan pcpqg_search would use for B queries / topn (diagnostics):
 * out8 = {queries per CTA group, threads, points per thread, pipeline stages,
 * CTAs per group along the points, groups, fp16 pre-score filter (K2-F) on,
 * pre-multiplied table mode on}. */
int pcpqg_plan_info(const pcpqg_index *idx, uint32_t B, uint32_t topn, uint32_t *out8);
uint64_t pcpqg_logical_payload_bits(uint64_t n, uint32_t m, uint32_t k, uint32_t scales);

/* Process-wide options:
 *   "lut_tensor_cores" 0|1  build the query LUT of batches >= 128 with tcgen05
 *                           tensor cores (4-way tf32 split; tolerance mode:
 *                           scores within ~1e-6 of max|score| instead of
 *                           bit-identical).  Default 0 (exact CUDA-core LUT).
 *   "fused_merge"      0|1  merge the per-CTA lists inside the scan's last CTA
 *                           of each query group instead of a merge kernel. */
int pcpqg_set_option(const char *name, int64_t value);

/* Timing of the last search on this thread (CUDA events on the launching
 * stream; milliseconds): lut, scan, merge.  Only filled when enabled. */
int pcpqg_set_profiling(int enabled);
int pcpqg_last_timings(float *out3);

/* ---- encode path (secondary; fp64, reference operation order, bit-exact) ----
 * Device pointers, stream-ordered.  x: n*dbar fp32 section vectors, centers:
 * k*dbar fp32.  Outputs: assignment (u32), alpha (f64), point loss (f64). */
int pcpqg_assign_projective(const float *d_x, uint64_t n, uint32_t dbar, const float *d_centers,
                            uint32_t k, uint32_t *d_assign, double *d_alpha, double *d_loss,
                            int device, void *cuda_stream);
/* d_prev (may be NULL): previous assignment; a point only switches centers if
 * that does not raise its own score-aware loss (clustering.cpp:339-349). */
int pcpqg_assign_anisotropic(const float *d_x, uint64_t n, uint32_t dbar,
                             const float *d_centers, uint32_t k, const double *d_h_par,
                             const double *d_h_bot, const uint32_t *d_prev, uint32_t *d_assign,
                             double *d_alpha, double *d_loss, int device, void *cuda_stream);
/* Score-aware scale codes against a float codebook of s values, given the
 * chosen centers; zero-norm / zero-curvature points get the code nearest 0. */
int pcpqg_aniso_alpha_codes(const float *d_x, uint64_t n, uint32_t dbar, const float *d_centers,
                            const uint32_t *d_assign, const double *d_h_par,
                            const double *d_h_bot, const float *d_values, uint32_t s,
                            uint8_t *d_codes, int device, void *cuda_stream);

/* Lloyd center statistics of the score-aware solver for nsec sections at
 * once: per (section, cluster) the fp64 sums of pcpq::center_anisotropic over
 * the cluster's members in increasing id order (the reference's summation
 * order), S = dbar(dbar+1)/2 + dbar + 1 doubles: M upper triangle (row-major,
 * a <= b), rhs[dbar], diag.  Section j's points are d_x + j*sec_stride
 * ([n][dbar]); d_assign/d_alpha/d_h_par/d_h_bot are [nsec][n].  d_init (may be
 * NULL) seeds the sums — the running partials of the ranks holding lower ids,
 * which makes a rank-ordered chain over GPUs bit-identical to one process. */
int pcpqg_center_stats(const float *d_x, uint64_t n, uint32_t dbar, uint32_t nsec,
                       uint64_t sec_stride, const uint32_t *d_assign, const double *d_alpha,
                       const double *d_h_par, const double *d_h_bot, uint32_t k,
                       const double *d_init, double *d_stats, int device, void *cuda_stream);

/* ---- IVF (two-level index, core/include/pcpq/ivf.hpp) ---------------------
 * A PCPQIVF1 container: coarse centers, member lists and per cell a PQ index
 * over the residuals (or raw residual rows for cells of < 2 members), held on
 * one device.  Validation and error classes follow pcpq::deserialize_ivf. */
typedef struct pcpqg_ivf pcpqg_ivf;

int pcpqg_ivf_load(const uint8_t *bytes, uint64_t len, int device, pcpqg_ivf **out);
int pcpqg_ivf_load_file(const char *path, int device, pcpqg_ivf **out);
void pcpqg_ivf_free(pcpqg_ivf *v);
/* out10: n, d, kbar, m, k (largest cell k), scales, method, raw cells,
 * device code bytes, code layout (PCPQG_FMT_*; 0 when every cell is raw) */
int pcpqg_ivf_info(const pcpqg_ivf *v, uint64_t *out10);

/* query_ivf for B queries Q [B][d] (host memory).  Per query b:
 *   ids[b][topn], scores[b][topn]   best first by (score desc, id asc); the
 *                                   first counts[b] = min(topn, probed
 *                                   population) slots are filled, the rest are
 *                                   id -1 / NaN
 *   short_flags[b]                  probed population < topn (IVFQueryOutput::short_result)
 *   req_scores[b][R]                scores of requested[b][R] (NaN when unprobed);
 *                                   requested / req_scores may be NULL when R = 0
 *   probes[b][k_probe] (optional)   the probed cells, best coarse score first
 * Scores are doubles, bit-identical to the reference: <q,c> + double(sub).
 * Errors as query_ivf: d != n-dim -> SIZE_MISMATCH; k_probe outside
 * [1, kbar], topn < 1, a requested id >= n -> DATA. */
int pcpqg_ivf_query(const pcpqg_ivf *v, const float *Q, uint32_t B, uint32_t d, uint32_t k_probe,
                    uint32_t topn, const uint32_t *requested, uint32_t R, int32_t *ids,
                    double *scores, uint32_t *counts, uint8_t *short_flags, double *req_scores,
                    uint32_t *probes);
/* The same with every array in device memory, on cuda_stream (a requested-id
 * range check synchronises the stream when R > 0). */
int pcpqg_ivf_query_device(const pcpqg_ivf *v, const float *dQ, uint32_t B, uint32_t d,
                           uint32_t k_probe, uint32_t topn, const uint32_t *d_requested,
                           uint32_t R, int32_t *d_ids, double *d_scores, uint32_t *d_counts,
                           uint8_t *d_short_flags, double *d_req_scores, uint32_t *d_probes,
                           void *cuda_stream);

/* ScoreCounters that query_ivf would add for these probes [B][k_probe]
 * (accumulated onto out5; raw cells add nothing, as in the reference). */
int pcpqg_ivf_counters(const pcpqg_ivf *v, const uint32_t *probes, uint32_t B, uint32_t k_probe,
                       uint64_t *out5);

/* ---- exact ground truth / recall (core/include/pcpq/eval.hpp) -------------
 * brute_force_topn for B queries over X [n][d] (fp32): per query the topn
 * points by the exact double inner product (index-order sum of exact
 * products, eval.cpp:18-24), ties toward the lower id; ids [B][topn] and the
 * bit-identical double scores.  topn outside [1, n] -> DATA.  Host arrays
 * (copied to `device`), or device arrays on cuda_stream (synchronised). */
int pcpqg_brute_force_topn(const float *X, uint64_t n, uint32_t d, const float *Q, uint32_t B,
                           uint32_t topn, int32_t *ids, double *scores, int device);
int pcpqg_brute_force_topn_device(const float *d_X, uint64_t n, uint32_t d, const float *d_Q,
                                  uint32_t B, uint32_t topn, int32_t *d_ids, double *d_scores,
                                  int device, void *cuda_stream);
/* recall1_single per query: hits[b] = 1 iff max over retrieved[b][0..R) of
 * the exact dot reaches exact_top1[b]; a retrieved id >= n -> DATA. */
int pcpqg_recall1(const float *X, uint64_t n, uint32_t d, const float *Q, uint32_t B,
                  const uint32_t *retrieved, uint32_t R, const double *exact_top1, int32_t *hits,
                  int device);

/* ---- training ----------------------------------------
 * build_pq_index with method = kmeans on X [n][d] (host, fp32) and the given
 * PQConfig fields; *out receives the serialized PCPQIDX1 image (byte-identical
 * to the reference's build + serialize), released with pcpqg_free.  The
 * Lloyd iterations of every section run on `device`.  Errors as
 * validate_config / build_pq_index (DATA). */
int pcpqg_train_kmeans(const float *X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                       double t_frac, uint32_t max_iters, double tol, uint64_t seed, int device,
                       uint8_t **out, uint64_t *out_len);
/* method = pcpq: projective clustering per section on the GPU, unit-norm
 * directions, scales quantized to s levels (quantize != 0) or stored raw. */
int pcpqg_train_pcpq(const float *X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                     int quantize, double t_frac, uint32_t max_iters, double tol, uint64_t seed,
                     int device, uint8_t **out, uint64_t *out_len);
/* method = aniso (1, the ScaNN baseline: fixed unit scales) or apcpq (3:
 * optimal per-point scales, quantized to s levels with
 * minimize_quadratic_scalars when quantize != 0, else stored raw): the
 * score-aware solver of clustering.cpp:622-722 per section on the GPU. */
int pcpqg_train_aniso(const float *X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                      int method, int quantize, double t_frac, uint32_t max_iters, double tol,
                      uint64_t seed, int device, uint8_t **out, uint64_t *out_len);
/* The same build on ndev GPUs of one process.  The m sections of a product
 * quantizer are independent problems (their own seed streams, weights, Lloyd
 * loop and scale quantizer), so they are dealt round-robin to the devices, one
 * host thread per device; nothing is exchanged until the image is assembled,
 * every ordered fp64 sum stays on one GPU, and the image is byte-identical to
 * the single-device (and the reference's) build for every device list.  A
 * device may be listed more than once. */
int pcpqg_train_aniso_multi(const float *X, uint64_t n, uint32_t d, uint32_t m, uint32_t k, uint32_t s,
                            int method, int quantize, double t_frac, uint32_t max_iters, double tol,
                            uint64_t seed, const int *devices, int ndev, uint8_t **out, uint64_t *out_len);
/* pcpq::aniso_weights (clustering.cpp:204-217) for every row of x [n][dbar]:
 * rows with a zero norm get {0, 0} (AnisoWeights' defaults, as the solvers
 * leave them).  Host threads, the C library's sin: bit-identical to the
 * reference.  DATA for t < 0 / non-finite or dbar < 2. */
int pcpqg_aniso_weights(const float *x, uint64_t n, uint32_t dbar, double t, double *h_par, double *h_bot);
/* The same weights computed by a CUDA kernel on `device` (one thread per row;
 * the Simpson sums in the reference's order over a bit-for-bit restatement of
 * the host C library's sin, csrc/pcpqg_hostsin.cuh): bit-identical to
 * pcpqg_aniso_weights.  UNSUPPORTED when the restated sin does not reproduce
 * this host's std::sin on the library's self-check arguments (another C
 * library, or a host without FMA); the trainers then keep the host path. */
int pcpqg_aniso_weights_gpu(const float *x, uint64_t n, uint32_t dbar, double t, double *h_par, double *h_bot,
                            int device);
/* Self-check of the restated sin against this host's std::sin: mismatches of
 * the host-evaluated restatement (device < 0) or of the kernel on `device`,
 * out of *total arguments (uniform over [0, pi/2], every binade down to 2^-40,
 * Simpson node grids, the branch edges). */
int pcpqg_sin_selfcheck(int device, uint64_t *mismatches, uint64_t *total);
/* 1 when the last pcpqg_train_aniso call on this thread computed its weights
 * on the GPU, 0 for host threads. */
int pcpqg_train_weights_on_gpu(int *out);
/* wall seconds of the last training call on this thread: [prep (validation,
 * sections, seeds, weights), Lloyd iterations, scales, serialization]. */
int pcpqg_train_phases(double *out4);
void pcpqg_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* PCPQG_H */
