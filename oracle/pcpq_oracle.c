/* TEST INFRASTRUCTURE ONLY — CPU oracle ("port") restating the reference
 * PCPQ scoring path in plain C.  See pcpq_oracle.h for the pinning story.
 *
 * Compiled with -ffp-contract=off and no -march so every float/double
 * operation is a separately rounded IEEE mul or add in the reference's order,
 * exactly like the reference build (proj/CMakeLists.txt:4-14).
 */
#define _GNU_SOURCE
#include "pcpq_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { E_OK = 0, E_USAGE = 1, E_DATA = 2, E_NUMERIC = 3, E_MAGIC = 4, E_VERSION = 5,
       E_TRUNC = 6, E_RANGE = 7, E_SIZE = 8 };

static int set_err(char *err, size_t errlen, int code, const char *msg) {
  if (err && errlen) snprintf(err, errlen, "%s", msg);
  return code;
}

/* ---------------------------------------------------------------- reader */
typedef struct { const uint8_t *p; uint64_t len, pos; int bad; } rd_t;

static int rd_raw(rd_t *r, void *dst, uint64_t n) {
  if (r->pos + n > r->len) { r->bad = 1; return 0; }
  memcpy(dst, r->p + r->pos, n);
  r->pos += n;
  return 1;
}
static uint32_t rd_u32(rd_t *r) {
  uint8_t b[4] = {0, 0, 0, 0};
  rd_raw(r, b, 4);
  return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}
static float rd_f32(rd_t *r) { uint32_t u = rd_u32(r); float f; memcpy(&f, &u, 4); return f; }
static double rd_f64(rd_t *r) {
  uint64_t lo = rd_u32(r), hi = rd_u32(r);
  uint64_t u = lo | (hi << 32);
  double v; memcpy(&v, &u, 8); return v;
}

void orc_free(orc_index *idx) {
  if (!idx) return;
  free(idx->codebooks); free(idx->scalar_cb); free(idx->center_codes);
  free(idx->scalar_codes); free(idx->raw_alphas); free(idx);
}
void orc_free_bytes(void *p) { free(p); }

/* Same validation order and error classes as pcpq::deserialize
 * (proj/core/src/pq_index.cpp:409-488). */
int orc_parse(const uint8_t *bytes, uint64_t len, orc_index **out, char *err, size_t errlen) {
  rd_t r = {bytes, len, 0, 0};
  char magic[8];
  *out = NULL;
  if (!rd_raw(&r, magic, 8)) return set_err(err, errlen, E_TRUNC, "truncated");
  if (memcmp(magic, "PCPQIDX1", 8) != 0) return set_err(err, errlen, E_MAGIC, "not an index file");
  uint32_t version = rd_u32(&r);
  if (r.bad) return set_err(err, errlen, E_TRUNC, "truncated");
  if (version != 1) return set_err(err, errlen, E_VERSION, "unsupported index version");
  uint32_t method = rd_u32(&r);
  if (r.bad) return set_err(err, errlen, E_TRUNC, "truncated");
  if (method > 3) return set_err(err, errlen, E_DATA, "unknown method tag");
  orc_index *x = calloc(1, sizeof(orc_index));
  x->method = method;
  x->n = rd_u32(&r); x->d = rd_u32(&r); x->padded_d = rd_u32(&r);
  x->m = rd_u32(&r); x->k = rd_u32(&r); x->scales = rd_u32(&r);
  x->t = rd_f64(&r);
  if (r.bad) { orc_free(x); return set_err(err, errlen, E_TRUNC, "truncated"); }
  if (x->n == 0 || x->d == 0 || x->m == 0 || x->k < 2) { orc_free(x); return set_err(err, errlen, E_DATA, "bad header field"); }
  if (x->k > 65536) { orc_free(x); return set_err(err, errlen, E_DATA, "bad header field: k"); }
  if (x->scales > 256) { orc_free(x); return set_err(err, errlen, E_DATA, "bad header field: scale count"); }
  if (x->padded_d < x->d || x->padded_d % x->m != 0) { orc_free(x); return set_err(err, errlen, E_DATA, "bad header field: padded dimension"); }
  x->dbar = x->padded_d / x->m;
  const uint64_t n = x->n, m = x->m, k = x->k;
  const int wide = x->k > 256;
  x->codebooks = malloc(sizeof(float) * m * k * x->dbar + 4);
  for (uint64_t i = 0; i < m * k * x->dbar; ++i) x->codebooks[i] = rd_f32(&r);
  x->scalar_cb = malloc(sizeof(float) * m * x->scales + 4);
  for (uint64_t i = 0; i < m * x->scales; ++i) x->scalar_cb[i] = rd_f32(&r);
  if (r.bad) { orc_free(x); return set_err(err, errlen, E_TRUNC, "truncated"); }
  x->center_codes = malloc(sizeof(uint32_t) * n * m);
  if (x->scales == 0) x->raw_alphas = malloc(sizeof(float) * n * m);
  else x->scalar_codes = malloc(n * m);
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j < m; ++j) {
      uint32_t c;
      if (wide) {
        uint8_t b[2] = {0, 0};
        rd_raw(&r, b, 2);
        c = (uint32_t)b[0] | ((uint32_t)b[1] << 8);
      } else {
        uint8_t b = 0;
        rd_raw(&r, &b, 1);
        c = b;
      }
      if (r.bad) { orc_free(x); return set_err(err, errlen, E_TRUNC, "truncated"); }
      if (c >= x->k) { orc_free(x); return set_err(err, errlen, E_RANGE, "center code out of range"); }
      x->center_codes[i * m + j] = c;
    }
    if (x->scales == 0) {
      for (uint64_t j = 0; j < m; ++j) x->raw_alphas[i * m + j] = rd_f32(&r);
      if (r.bad) { orc_free(x); return set_err(err, errlen, E_TRUNC, "truncated"); }
    } else {
      for (uint64_t j = 0; j < m; ++j) {
        uint8_t b = 0;
        rd_raw(&r, &b, 1);
        if (r.bad) { orc_free(x); return set_err(err, errlen, E_TRUNC, "truncated"); }
        if (b >= x->scales) { orc_free(x); return set_err(err, errlen, E_RANGE, "scale code out of range"); }
        x->scalar_codes[i * m + j] = b;
      }
    }
  }
  if (r.pos != r.len) { orc_free(x); return set_err(err, errlen, E_SIZE, "trailing bytes after index payload"); }
  *out = x;
  return E_OK;
}

/* ------------------------------------------------------------- writer */
typedef struct { uint8_t *p; uint64_t len, cap; } wr_t;
static void wr_raw(wr_t *w, const void *src, uint64_t n) {
  if (w->len + n > w->cap) {
    w->cap = (w->len + n) * 2 + 64;
    w->p = realloc(w->p, w->cap);
  }
  memcpy(w->p + w->len, src, n);
  w->len += n;
}
static void wr_u32(wr_t *w, uint32_t v) {
  uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
  wr_raw(w, b, 4);
}
static void wr_f32(wr_t *w, float f) { uint32_t u; memcpy(&u, &f, 4); wr_u32(w, u); }

int orc_serialize(const orc_index *x, uint8_t **out, uint64_t *len) {
  wr_t w = {NULL, 0, 0};
  const uint64_t n = x->n, m = x->m, k = x->k;
  wr_raw(&w, "PCPQIDX1", 8);
  wr_u32(&w, 1); wr_u32(&w, x->method); wr_u32(&w, x->n); wr_u32(&w, x->d);
  wr_u32(&w, x->padded_d); wr_u32(&w, x->m); wr_u32(&w, x->k); wr_u32(&w, x->scales);
  uint64_t tb; memcpy(&tb, &x->t, 8);
  wr_u32(&w, (uint32_t)tb); wr_u32(&w, (uint32_t)(tb >> 32));
  for (uint64_t i = 0; i < m * k * x->dbar; ++i) wr_f32(&w, x->codebooks[i]);
  for (uint64_t i = 0; i < m * x->scales; ++i) wr_f32(&w, x->scalar_cb[i]);
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j < m; ++j) {
      uint32_t c = x->center_codes[i * m + j];
      if (k > 256) { uint8_t b[2] = {(uint8_t)c, (uint8_t)(c >> 8)}; wr_raw(&w, b, 2); }
      else { uint8_t b = (uint8_t)c; wr_raw(&w, &b, 1); }
    }
    if (x->scales == 0) for (uint64_t j = 0; j < m; ++j) wr_f32(&w, x->raw_alphas[i * m + j]);
    else wr_raw(&w, x->scalar_codes + i * m, m);
  }
  *out = w.p;
  *len = w.len;
  return E_OK;
}

/* ------------------------------------------------------------ scoring */
int orc_build_lut(const orc_index *x, const float *q, uint32_t d, float *eta, float *etal,
                  uint64_t *cnt) {
  if (d != x->d) return E_SIZE;  /* pq_index.cpp:174-175 */
  const uint32_t m = x->m, k = x->k, dbar = x->dbar, s = x->scales;
  for (uint32_t j = 0; j < m; ++j) {
    for (uint32_t c = 0; c < k; ++c) {
      const float *row = x->codebooks + ((uint64_t)j * k + c) * dbar;
      float acc = 0.0f; /* fixed-order fp32, pq_index.cpp:186-190 */
      for (uint32_t a = 0; a < dbar; ++a) {
        const uint32_t col = j * dbar + a;
        const float qa = col < x->d ? q[col] : 0.0f; /* pad_vector, types.cpp:83-88 */
        const float prod = row[a] * qa;
        acc = acc + prod;
      }
      eta[(uint64_t)j * k + c] = acc;
    }
  }
  if (cnt) cnt[0] += (uint64_t)k * x->padded_d;
  if (s >= 1) {
    if (etal) {
      for (uint32_t j = 0; j < m; ++j)
        for (uint32_t c = 0; c < k; ++c) {
          const float e = eta[(uint64_t)j * k + c];
          for (uint32_t l = 0; l < s; ++l)
            etal[((uint64_t)j * k + c) * s + l] = e * x->scalar_cb[(uint64_t)j * s + l];
        }
    }
    if (cnt) cnt[1] += (uint64_t)s * k * m;
  }
  return E_OK;
}

/* score_all restated over [begin,end) (pq_index.cpp:212-244).  etal may be
 * NULL on the quantized route: eta*lambda is then formed on the fly, which is
 * the same single rounded product the table stores (pq_index.cpp:203). */
int orc_score_range(const orc_index *x, const float *eta, const float *etal, uint64_t begin,
                    uint64_t end, float *scores, uint64_t *cnt) {
  const uint32_t m = x->m, k = x->k, s = x->scales;
  for (uint64_t i = begin; i < end; ++i) {
    const uint32_t *codes = x->center_codes + i * m;
    float acc;
    if (s >= 1) {
      const uint8_t *sc = x->scalar_codes + i * m;
      for (uint32_t j = 0; j < m; ++j) {
        float t;
        if (etal) t = etal[((uint64_t)j * k + codes[j]) * s + sc[j]];
        else t = eta[(uint64_t)j * k + codes[j]] * x->scalar_cb[(uint64_t)j * s + sc[j]];
        acc = (j == 0) ? t : acc + t;
      }
    } else {
      const float *al = x->raw_alphas + i * m;
      for (uint32_t j = 0; j < m; ++j) {
        const float t = al[j] * eta[(uint64_t)j * k + codes[j]];
        acc = (j == 0) ? t : acc + t;
      }
    }
    scores[i - begin] = acc;
  }
  if (cnt) {
    const uint64_t nn = end - begin;
    if (s == 0) cnt[2] += nn * m;
    cnt[3] += nn * m;
    cnt[4] += nn * (m - 1);
  }
  return E_OK;
}

int orc_score_query(const orc_index *x, const float *q, uint32_t d, float *scores, uint64_t *cnt) {
  const uint64_t mk = (uint64_t)x->m * x->k;
  float *eta = malloc(sizeof(float) * mk);
  float *etal = x->scales ? malloc(sizeof(float) * mk * x->scales) : NULL;
  int st = orc_build_lut(x, q, d, eta, etal, cnt);
  if (st == E_OK) st = orc_score_range(x, eta, etal, 0, x->n, scores, cnt);
  free(eta);
  free(etal);
  return st;
}

/* (score desc, id asc): the comparator of proj/tools/main.cpp:235-236 */
static inline int better(float sa, uint32_t ia, float sb, uint32_t ib) {
  if (sa != sb) return sa > sb;
  return ia < ib;
}

/* Bounded heap keeping the best `topn` (worst at the root), then sorted. */
void orc_topn_of_scores(const float *scores, uint64_t n, uint32_t topn, int32_t *ids) {
  if (topn > n) topn = (uint32_t)n;
  if (topn == 0) return;
  uint32_t *h = malloc(sizeof(uint32_t) * topn);
  uint32_t sz = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t id = (uint32_t)i;
    if (sz < topn) {
      uint32_t c = sz++;
      h[c] = id;
      while (c > 0) { /* sift up: parent must be worse than child */
        uint32_t p = (c - 1) / 2;
        if (better(scores[h[p]], h[p], scores[h[c]], h[c])) {
          uint32_t t = h[p]; h[p] = h[c]; h[c] = t; c = p;
        } else break;
      }
    } else if (better(scores[id], id, scores[h[0]], h[0])) {
      h[0] = id;
      uint32_t c = 0;
      for (;;) {
        uint32_t l = 2 * c + 1, r = l + 1, w = c;
        if (l < sz && better(scores[h[w]], h[w], scores[h[l]], h[l])) w = l;
        if (r < sz && better(scores[h[w]], h[w], scores[h[r]], h[r])) w = r;
        if (w == c) break;
        uint32_t t = h[w]; h[w] = h[c]; h[c] = t; c = w;
      }
    }
  }
  /* heap-sort out: repeatedly pop the worst to the end */
  for (uint32_t end = sz; end > 1; --end) {
    uint32_t t = h[0]; h[0] = h[end - 1]; h[end - 1] = t;
    uint32_t c = 0, lim = end - 1;
    for (;;) {
      uint32_t l = 2 * c + 1, r = l + 1, w = c;
      if (l < lim && better(scores[h[w]], h[w], scores[h[l]], h[l])) w = l;
      if (r < lim && better(scores[h[w]], h[w], scores[h[r]], h[r])) w = r;
      if (w == c) break;
      uint32_t u = h[w]; h[w] = h[c]; h[c] = u; c = w;
    }
  }
  for (uint32_t i = 0; i < sz; ++i) ids[i] = (int32_t)h[i];
  free(h);
}

typedef struct {
  const orc_index *x; const float *Q; uint64_t B; uint32_t d, topn_req;
  int32_t *ids; float *scores;
  uint64_t next; pthread_mutex_t mu; int status;
} search_job;

static void *search_worker(void *arg) {
  search_job *J = arg;
  const orc_index *x = J->x;
  const uint32_t topn = J->topn_req < x->n ? J->topn_req : x->n;
  float *sc = malloc(sizeof(float) * x->n);
  int32_t *tmp = malloc(sizeof(int32_t) * (topn ? topn : 1));
  for (;;) {
    pthread_mutex_lock(&J->mu);
    uint64_t qi = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (qi >= J->B) break;
    int st = orc_score_query(x, J->Q + qi * J->d, J->d, sc, NULL);
    if (st) { J->status = st; break; }
    orc_topn_of_scores(sc, x->n, topn, tmp);
    for (uint32_t i = 0; i < J->topn_req; ++i) {
      const int ok = i < topn;
      J->ids[qi * J->topn_req + i] = ok ? tmp[i] : -1;
      if (J->scores) J->scores[qi * J->topn_req + i] = ok ? sc[tmp[i]] : -INFINITY;
    }
  }
  free(sc);
  free(tmp);
  return NULL;
}

int orc_search(const orc_index *x, const float *Q, uint64_t B, uint32_t d, uint32_t topn_req,
               int threads, int32_t *ids, float *scores) {
  if (d != x->d) return E_DATA;
  search_job J = {x, Q, B, d, topn_req, ids, scores, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  if (threads <= 1) {
    search_worker(&J);
  } else {
    pthread_t *th = malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, search_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  return J.status;
}

static uint32_t ceil_log2(uint64_t v) {
  uint32_t b = 0;
  if (v <= 1) return 0;
  v -= 1;
  while (v) { ++b; v >>= 1; }
  return b;
}

uint64_t orc_logical_payload_bits(uint64_t n, uint32_t m, uint32_t k, uint32_t scales) {
  const uint64_t sb = scales == 0 ? 32 : ceil_log2(scales);
  return n * m * (ceil_log2(k) + sb);
}

/* ------------------------------------------------------------- encode */
static double dotf(const float *a, const float *b, uint32_t n) {
  double acc = 0.0;
  for (uint32_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

int orc_assign_projective(const float *x, uint64_t n, uint32_t dbar, const float *centers,
                          uint32_t k, uint32_t *assign, double *alphas, double *ploss) {
  double *c2 = malloc(sizeof(double) * k);
  for (uint32_t j = 0; j < k; ++j) {
    c2[j] = dotf(centers + (uint64_t)j * dbar, centers + (uint64_t)j * dbar, dbar);
    if (c2[j] == 0.0) { free(c2); return E_DATA; }
  }
  for (uint64_t i = 0; i < n; ++i) {
    const float *xi = x + i * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) { assign[i] = 0; alphas[i] = 0.0; if (ploss) ploss[i] = 0.0; continue; }
    double best = INFINITY, bip = 0.0;
    uint32_t bj = 0;
    for (uint32_t j = 0; j < k; ++j) {
      const double ip = dotf(xi, centers + (uint64_t)j * dbar, dbar);
      const double l = nx2 - ip * ip / c2[j];
      if (l < best) { best = l; bj = j; bip = ip; }
    }
    assign[i] = bj;
    alphas[i] = bip / c2[bj];
    if (ploss) ploss[i] = best < 0.0 ? 0.0 : best; /* std::max(best, 0.0) */
  }
  free(c2);
  return E_OK;
}

static double opt_alpha_from(double ip, double nx2, double c2, double hp, double hb) {
  const double denom = (hp - hb) * ip * ip / nx2 + hb * c2;
  if (fabs(denom) <= 1e-30) return 0.0;
  return hp * ip / denom;
}

int orc_assign_anisotropic(const float *x, uint64_t n, uint32_t dbar, const float *centers,
                           uint32_t k, const double *h_par, const double *h_bot,
                           uint32_t *assign, double *alphas, double *ploss) {
  double *c2 = malloc(sizeof(double) * k);
  for (uint32_t j = 0; j < k; ++j) {
    c2[j] = dotf(centers + (uint64_t)j * dbar, centers + (uint64_t)j * dbar, dbar);
    if (c2[j] == 0.0) { free(c2); return E_DATA; }
  }
  for (uint64_t i = 0; i < n; ++i) {
    const float *xi = x + i * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) { assign[i] = 0; alphas[i] = 0.0; if (ploss) ploss[i] = 0.0; continue; }
    const double hp = h_par[i], hb = h_bot[i];
    double bdist = INFINITY, balpha = 1.0;
    uint32_t bj = 0;
    for (uint32_t j = 0; j < k; ++j) {
      const double ip = dotf(xi, centers + (uint64_t)j * dbar, dbar);
      const double beta = opt_alpha_from(ip, nx2, c2[j], hp, hb);
      const double dist = nx2 - 2.0 * beta * ip + beta * beta * c2[j];
      if (dist < bdist) { bdist = dist; bj = j; balpha = beta; }
    }
    const double bip = dotf(xi, centers + (uint64_t)bj * dbar, dbar);
    /* point_quad + quad_at (clustering.cpp:29-34) */
    const double w = (hp - hb) * bip * bip / nx2 + hb * c2[bj];
    const double a = -2.0 * hp * bip, b = hp * nx2;
    const double bloss = (w * balpha + a) * balpha + b;
    assign[i] = bj;
    alphas[i] = balpha;
    if (ploss) ploss[i] = bloss < 0.0 ? 0.0 : bloss;
  }
  free(c2);
  return E_OK;
}

/* Member sums of center_anisotropic (clustering.cpp:382-402) for one cluster:
 * rows in member (id) order; stats = M upper triangle (row-major a <= b),
 * rhs[dbar], diag, accumulated onto the incoming values of `stats`. */
void orc_center_stats(const float *x, const uint32_t *members, uint64_t cnt, uint32_t dbar,
                      const double *alpha, const double *h_par, const double *h_bot,
                      double *stats) {
  const uint32_t r0 = dbar * (dbar + 1) / 2;
  for (uint64_t t = 0; t < cnt; ++t) {
    const uint32_t id = members[t];
    const float *xi = x + (uint64_t)id * dbar;
    double nx2 = 0.0;
    for (uint32_t a = 0; a < dbar; ++a) nx2 += (double)xi[a] * xi[a];
    if (nx2 == 0.0) continue;
    const double a2 = alpha[id] * alpha[id];
    const double coef = a2 * (h_par[id] - h_bot[id]) / nx2;
    uint32_t s = 0;
    for (uint32_t a = 0; a < dbar; ++a) {
      const double xa = xi[a];
      for (uint32_t b = a; b < dbar; ++b) stats[s++] += coef * xa * xi[b];
      stats[r0 + a] += alpha[id] * h_par[id] * xa;
    }
    stats[r0 + dbar] += a2 * h_bot[id];
  }
}

/* center_anisotropic's solve from the sums: symmetric fill, ridge
 * 1e-9*trace/d, solve_spd (clustering.cpp:403-409, numerics.cpp:138-172). */
int orc_center_from_stats(const double *stats, uint32_t d, double *center) {
  double m[256], rhs[16], l[256], y[16];
  if (d > 16) return E_DATA;
  uint32_t s = 0;
  for (uint32_t a = 0; a < d; ++a)
    for (uint32_t b = a; b < d; ++b) m[a * d + b] = stats[s++];
  for (uint32_t a = 0; a < d; ++a) rhs[a] = stats[s + a];
  const double diag = stats[s + d];
  for (uint32_t a = 0; a < d; ++a) {
    m[a * d + a] += diag;
    for (uint32_t b = 0; b < a; ++b) m[a * d + b] = m[b * d + a];
  }
  double trace = 0.0;
  for (uint32_t a = 0; a < d; ++a) trace += m[a * d + a];
  const double ridge = 1e-9 * trace / (double)d;
  for (uint32_t i = 0; i < d * d; ++i) l[i] = m[i];
  for (uint32_t i = 0; i < d; ++i) l[i * d + i] += ridge;
  for (uint32_t j = 0; j < d; ++j) {
    double dg = l[j * d + j];
    for (uint32_t c = 0; c < j; ++c) dg -= l[j * d + c] * l[j * d + c];
    if (!(dg > 0.0)) return E_NUMERIC;
    dg = sqrt(dg);
    l[j * d + j] = dg;
    for (uint32_t i = j + 1; i < d; ++i) {
      double acc = l[i * d + j];
      for (uint32_t c = 0; c < j; ++c) acc -= l[i * d + c] * l[j * d + c];
      l[i * d + j] = acc / dg;
    }
  }
  for (uint32_t i = 0; i < d; ++i) {
    double acc = rhs[i];
    for (uint32_t c = 0; c < i; ++c) acc -= l[i * d + c] * y[c];
    y[i] = acc / l[i * d + i];
  }
  for (uint32_t ii = d; ii-- > 0;) {
    double acc = y[ii];
    for (uint32_t c = ii + 1; c < d; ++c) acc -= l[c * d + ii] * center[c];
    center[ii] = acc / l[ii * d + ii];
  }
  return E_OK;
}

int orc_alpha_codes_aniso(const float *x, uint64_t n, uint32_t dbar, const float *centers,
                          const uint32_t *assign, const double *h_par, const double *h_bot,
                          const float *values, uint32_t s, uint8_t *codes) {
  /* nearest_code(values, 0.0) for excluded points (scalar_quant.cpp:28-39,142-150) */
  uint8_t zero_code = 0;
  double bd = INFINITY;
  for (uint32_t l = 0; l < s; ++l) {
    const double dd = fabs((double)values[l] - 0.0);
    if (dd < bd) { bd = dd; zero_code = (uint8_t)l; }
  }
  for (uint64_t i = 0; i < n; ++i) {
    const float *xi = x + i * dbar;
    const float *c = centers + (uint64_t)assign[i] * dbar;
    const double nx2 = dotf(xi, xi, dbar);
    if (nx2 == 0.0) { codes[i] = zero_code; continue; }
    const double c2 = dotf(c, c, dbar);
    const double ip = dotf(xi, c, dbar);
    const double hp = h_par[i], hb = h_bot[i];
    const double wq = (hp - hb) * ip * ip / nx2 + hb * c2;
    if (!(wq > 0.0)) { codes[i] = zero_code; continue; }
    const double a = -2.0 * hp * ip, b = hp * nx2;
    double best = INFINITY;
    uint8_t bl = 0;
    for (uint32_t l = 0; l < s; ++l) {
      const double lam = values[l];
      const double v = (wq * lam + a) * lam + b;
      if (v < best) { best = v; bl = (uint8_t)l; }
    }
    codes[i] = bl;
  }
  return E_OK;
}

/* ================================================================== IVF
 * PCPQIVF1 container (proj/core/src/ivf.cpp:256-316) and query_ivf
 * (ivf.cpp:89-153), restated. */
void orc_ivf_free(orc_ivf *v) {
  if (!v) return;
  if (v->sub)
    for (uint32_t r = 0; r < v->kbar; ++r) orc_free(v->sub[r]);
  if (v->raw)
    for (uint32_t r = 0; r < v->kbar; ++r) free(v->raw[r]);
  free(v->sub); free(v->raw); free(v->coarse); free(v->member_off); free(v->members);
  free(v->is_raw); free(v->point_cluster); free(v->point_slot);
  free(v);
}

int orc_ivf_parse(const uint8_t *bytes, uint64_t len, orc_ivf **out, char *err, size_t errlen) {
  rd_t r = {bytes, len, 0, 0};
  char magic[8];
  *out = NULL;
  if (!rd_raw(&r, magic, 8)) return set_err(err, errlen, E_TRUNC, "container truncated");
  if (memcmp(magic, "PCPQIVF1", 8) != 0) return set_err(err, errlen, E_MAGIC, "not a container file");
  uint32_t version = rd_u32(&r);
  if (r.bad) return set_err(err, errlen, E_TRUNC, "container truncated");
  if (version != 1) return set_err(err, errlen, E_VERSION, "unsupported container version");
  orc_ivf *v = calloc(1, sizeof(orc_ivf));
  v->n = rd_u32(&r); v->d = rd_u32(&r); v->kbar = rd_u32(&r);
  if (r.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
  if (v->n == 0 || v->d == 0 || v->kbar == 0 || v->kbar > v->n) {
    v->kbar = 0; orc_ivf_free(v); return set_err(err, errlen, E_DATA, "bad container header");
  }
  const uint64_t kd = (uint64_t)v->kbar * v->d;
  v->coarse = malloc(sizeof(float) * kd);
  for (uint64_t i = 0; i < kd; ++i) v->coarse[i] = rd_f32(&r);
  if (r.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
  v->member_off = calloc(v->kbar + 1, sizeof(uint32_t));
  uint64_t total = 0, cap = 16;
  v->members = malloc(sizeof(uint32_t) * cap);
  for (uint32_t c = 0; c < v->kbar; ++c) {
    const uint32_t count = rd_u32(&r);
    if (r.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
    if (count > v->n) { orc_ivf_free(v); return set_err(err, errlen, E_DATA, "member count exceeds n"); }
    if (total + count > cap) {
      while (total + count > cap) cap *= 2;
      v->members = realloc(v->members, sizeof(uint32_t) * cap);
    }
    for (uint32_t i = 0; i < count; ++i) v->members[total + i] = rd_u32(&r);
    if (r.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
    total += count;
    if (total > 0xFFFFFFFFull) { orc_ivf_free(v); return set_err(err, errlen, E_DATA, "member lists too long"); }
    v->member_off[c + 1] = (uint32_t)total;
  }
  v->sub = calloc(v->kbar, sizeof(orc_index *));
  v->raw = calloc(v->kbar, sizeof(float *));
  v->is_raw = calloc(v->kbar, 1);
  for (uint32_t c = 0; c < v->kbar; ++c) {
    const uint64_t lo = rd_u32(&r), hi = rd_u32(&r);
    const uint64_t blen = lo | (hi << 32);
    if (r.bad || blen > r.len - r.pos) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
    const uint8_t *blob = r.p + r.pos;
    r.pos += blen;
    const uint32_t count = v->member_off[c + 1] - v->member_off[c];
    if (blen >= 8 && memcmp(blob, "PCPQRAW1", 8) == 0) {
      rd_t br = {blob, blen, 8, 0};
      const uint32_t bc = rd_u32(&br), dim = rd_u32(&br);
      if (br.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
      if (dim != v->d) { orc_ivf_free(v); return set_err(err, errlen, E_DATA, "raw block dimension mismatch"); }
      if (bc != count) { orc_ivf_free(v); return set_err(err, errlen, E_SIZE, "raw block count mismatch"); }
      v->is_raw[c] = 1;
      v->raw[c] = malloc(sizeof(float) * ((uint64_t)bc * dim + 1));
      for (uint64_t i = 0; i < (uint64_t)bc * dim; ++i) v->raw[c][i] = rd_f32(&br);
      if (br.bad) { orc_ivf_free(v); return set_err(err, errlen, E_TRUNC, "container truncated"); }
      if (br.pos != br.len) { orc_ivf_free(v); return set_err(err, errlen, E_SIZE, "trailing bytes in raw block"); }
    } else {
      int st = orc_parse(blob, blen, &v->sub[c], err, errlen);
      if (st) { orc_ivf_free(v); return st; }
      if (v->sub[c]->n != count) { orc_ivf_free(v); return set_err(err, errlen, E_SIZE, "sub-index size does not match member list"); }
      if (v->sub[c]->d != v->d) { orc_ivf_free(v); return set_err(err, errlen, E_DATA, "sub-index dimension mismatch"); }
    }
  }
  if (r.pos != r.len) { orc_ivf_free(v); return set_err(err, errlen, E_SIZE, "trailing bytes after container"); }
  /* rebuild_point_maps (ivf.cpp:28-43): the member lists must partition [0, n) */
  v->point_cluster = calloc(v->n, sizeof(uint32_t));
  v->point_slot = calloc(v->n, sizeof(uint32_t));
  uint8_t *seen = calloc(v->n, 1);
  for (uint32_t c = 0; c < v->kbar; ++c)
    for (uint32_t pos = v->member_off[c]; pos < v->member_off[c + 1]; ++pos) {
      const uint32_t id = v->members[pos];
      if (id >= v->n || seen[id]) { free(seen); orc_ivf_free(v); return set_err(err, errlen, E_DATA, "member lists do not partition the ids"); }
      seen[id] = 1;
      v->point_cluster[id] = c;
      v->point_slot[id] = pos - v->member_off[c];
    }
  for (uint32_t i = 0; i < v->n; ++i)
    if (!seen[i]) { free(seen); orc_ivf_free(v); return set_err(err, errlen, E_DATA, "member lists do not partition the ids"); }
  free(seen);
  *out = v;
  return E_OK;
}

typedef struct { double s; uint32_t id; } orc_hit;
static const double *g_cs;
static int cmp_coarse(const void *a, const void *b) {  /* stable_sort by coarse desc == ties by r asc */
  const uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  if (g_cs[x] != g_cs[y]) return g_cs[x] > g_cs[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}
static int cmp_hit(const void *a, const void *b) {  /* (score desc, id asc), ivf.cpp:140-143 */
  const orc_hit *x = a, *y = b;
  if (x->s != y->s) return x->s > y->s ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

int orc_ivf_query(const orc_ivf *v, const float *q, uint32_t d, uint32_t k_probe, uint32_t topn,
                  const uint32_t *req, uint32_t R, int32_t *ids, double *scores, uint32_t *count,
                  uint8_t *short_flag, double *req_scores, uint64_t *counters5) {
  if (d != v->d) return E_SIZE;
  if (k_probe < 1 || k_probe > v->kbar) return E_DATA;
  if (topn < 1) return E_DATA;
  for (uint32_t i = 0; i < R; ++i)
    if (req[i] >= v->n) return E_DATA;
  double *cs = malloc(sizeof(double) * v->kbar);
  uint32_t *order = malloc(sizeof(uint32_t) * v->kbar);
  for (uint32_t r = 0; r < v->kbar; ++r) {
    cs[r] = dotf(q, v->coarse + (uint64_t)r * v->d, v->d);  /* ivf.cpp:101-103 */
    order[r] = r;
  }
  g_cs = cs;
  qsort(order, v->kbar, sizeof(uint32_t), cmp_coarse);
  uint64_t pool_n = 0;
  for (uint32_t p = 0; p < k_probe; ++p) {
    const uint32_t r = order[p];
    pool_n += v->member_off[r + 1] - v->member_off[r];
  }
  orc_hit *pool = malloc(sizeof(orc_hit) * (pool_n + 1));
  uint64_t *pool_off = malloc(sizeof(uint64_t) * v->kbar);
  for (uint32_t r = 0; r < v->kbar; ++r) pool_off[r] = UINT64_MAX;
  uint64_t at = 0;
  int st = E_OK;
  for (uint32_t p = 0; p < k_probe && st == E_OK; ++p) {
    const uint32_t r = order[p];
    pool_off[r] = at;
    const uint32_t c0 = v->member_off[r], cnt = v->member_off[r + 1] - c0;
    if (cnt == 0) continue;
    if (v->is_raw[r]) {
      for (uint32_t pos = 0; pos < cnt; ++pos)
        pool[at + pos] = (orc_hit){cs[r] + dotf(q, v->raw[r] + (uint64_t)pos * v->d, v->d), v->members[c0 + pos]};
    } else {
      float *sub = malloc(sizeof(float) * cnt);
      st = orc_score_query(v->sub[r], q, d, sub, counters5);
      for (uint32_t pos = 0; pos < cnt && st == E_OK; ++pos)
        pool[at + pos] = (orc_hit){cs[r] + (double)sub[pos], v->members[c0 + pos]};
      free(sub);
    }
    at += cnt;
  }
  if (st == E_OK) {
    for (uint32_t i = 0; i < R; ++i) {
      const uint32_t r = v->point_cluster[req[i]];
      req_scores[i] = pool_off[r] == UINT64_MAX ? NAN : pool[pool_off[r] + v->point_slot[req[i]]].s;
    }
    const uint64_t keep = pool_n < topn ? pool_n : topn;
    *short_flag = pool_n < topn;
    qsort(pool, pool_n, sizeof(orc_hit), cmp_hit);
    for (uint32_t i = 0; i < topn; ++i) {
      ids[i] = i < keep ? (int32_t)pool[i].id : -1;
      scores[i] = i < keep ? pool[i].s : NAN;
    }
    *count = (uint32_t)keep;
  }
  free(cs); free(order); free(pool); free(pool_off);
  return st;
}

/* ============================================================== eval
 * brute_force_topn (proj/core/src/eval.cpp:36-49): exact dot in double in
 * index order (dot_qx, eval.cpp:18-24), top-n by (score desc, id asc).
 * recall1_single (eval.cpp:57-66). */
static int cmp_hit_desc(const void *a, const void *b) { return cmp_hit(a, b); }

int orc_brute_force_topn(const float *X, uint64_t n, uint32_t d, const float *q, uint32_t topn,
                         int32_t *ids, double *scores) {
  if (topn < 1 || topn > n) return E_DATA;
  orc_hit *all = malloc(sizeof(orc_hit) * n);
  for (uint64_t i = 0; i < n; ++i) all[i] = (orc_hit){dotf(q, X + i * d, d), (uint32_t)i};
  qsort(all, n, sizeof(orc_hit), cmp_hit_desc);
  for (uint32_t i = 0; i < topn; ++i) {
    ids[i] = (int32_t)all[i].id;
    scores[i] = all[i].s;
  }
  free(all);
  return E_OK;
}

int orc_recall1(const float *X, uint64_t n, uint32_t d, const float *q, const uint32_t *retrieved,
                uint32_t R, double exact_top1, int32_t *hit) {
  double best = -INFINITY;
  for (uint32_t i = 0; i < R; ++i) {
    if (retrieved[i] >= n) return E_DATA;
    const double v = dotf(q, X + (uint64_t)retrieved[i] * d, d);
    best = v > best ? v : best;
  }
  *hit = best >= exact_top1 ? 1 : 0;
  return E_OK;
}
