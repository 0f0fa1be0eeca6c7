/*
 * permez_oracle.c -- CPU restatement of the permez PW_REL block compression
 * path.  TEST INFRASTRUCTURE ONLY: this file is the checker the CUDA path is
 * compared against.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it; the product package
 * (paper_2309_09778_b200/) never links or calls it.
 *
 * Every function cites the reference text it restates (paths relative to the
 * reference root):
 *   transform.py = pkg/src/permez/transform.py   (the only reference CODE)
 *   SPEC.md      = behavioural spec of the SPEC-only modules
 * Ambiguities are pinned exactly as DESIGN.md "Decision ledger" (D1..D21).
 *
 * Arithmetic rules (so that results are a pure function of the inputs):
 *  - built with -ffp-contract=off; no FMA contraction anywhere;
 *  - log2 / exp2 are CORRECTLY ROUNDED double results (long double evaluation
 *    with a __float128 fallback near rounding midpoints).  numpy's np.log2 is
 *    within 0.5001 ulp of this; the exhaustive
 *    comparison against the reference's own transform.py is in
 *    tests/test_oracle_pin.py.
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define ORC_API __attribute__((visibility("default")))

enum {
  PMZ_OK = 0,
  PMZ_ERR_CONFIG = -1,
  PMZ_ERR_NONFINITE = -2,
  PMZ_ERR_DEGENERATE = -3,
  PMZ_ERR_SUBNORMAL = -4,
  PMZ_ERR_NONREPRESENTABLE = -5,
  PMZ_ERR_TOO_FEW_BLOCKS = -6,
  PMZ_ERR_BALANCE_FLAG = -7,
  PMZ_ERR_DEGENERATE_ALPHABET = -8,
  PMZ_ERR_UNASSIGNED = -9,
  PMZ_ERR_TRUNCATED = -10,
  PMZ_ERR_INVALID_PREFIX = -11,
  PMZ_ERR_BAD_MAGIC = -12,
  PMZ_ERR_UNSUPPORTED_VERSION = -13,
  PMZ_ERR_CORRUPT = -14,
  PMZ_ERR_BALANCE_UNDERFLOW = -15,
  PMZ_ERR_CAPACITY = -16,
  PMZ_ERR_NOMEM = -20,
};

/* ------------------------------------------------------------------------ */
/* Correctly rounded log2 / exp2 (double in, double out).                    */
/* ------------------------------------------------------------------------ */

/* true when the extended value l is within tol of a rounding midpoint of d */
static int near_mid(long double l, double d, long double tol) {
  double up = nextafter(d, INFINITY), dn = nextafter(d, -INFINITY);
  long double mu = ((long double)d + (long double)up) * 0.5L;
  long double md = ((long double)d + (long double)dn) * 0.5L;
  return fabsl(l - mu) <= tol || fabsl(l - md) <= tol;
}

static int near_mid_q(__float128 l, double d, __float128 tol) {
  double up = nextafter(d, INFINITY), dn = nextafter(d, -INFINITY);
  __float128 mu = ((__float128)d + (__float128)up) * 0.5Q;
  __float128 md = ((__float128)d + (__float128)dn) * 0.5Q;
  return fabsq(l - mu) <= tol || fabsq(l - md) <= tol;
}

/* Counts of slow-path evaluations (diagnostics only). */
static long long g_log2_slow = 0, g_exp2_slow = 0, g_unresolved = 0;

/* np.log2 restated as the correctly rounded log2 (transform.py:95-98,118-123,178). */
ORC_API double orc_log2(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -INFINITY : NAN;
  if (isinf(x)) return INFINITY;
  int e;
  double fr = frexp(x, &e);
  if (fr == 0.5) return (double)(e - 1); /* exact power of two */
  long double l = log2l((long double)x);
  double d = (double)l;
  long double tol = fabsl(l) * 0x1p-60L;
  if (!near_mid(l, d, tol)) return d;
  __atomic_fetch_add(&g_log2_slow, 1, __ATOMIC_RELAXED);
  __float128 q = log2q((__float128)x);
  double dq = (double)q;
  if (near_mid_q(q, dq, fabsq(q) * 0x1p-108Q)) __atomic_fetch_add(&g_unresolved, 1, __ATOMIC_RELAXED);
  return dq;
}

/* np.exp2 restated as the correctly rounded exp2 (transform.py:196-197). */
ORC_API double orc_exp2(double y) {
  if (isnan(y)) return y;
  if (y >= 1024.0) return INFINITY;
  if (y < -1080.0) return 0.0;
  if (y == floor(y)) return ldexp(1.0, (int)y);
  long double l = exp2l((long double)y);
  double d = (double)l;
  if (d != 0.0 && !isinf(d) && fabs(d) >= DBL_MIN) {
    long double tol = fabsl(l) * 0x1p-60L;
    if (!near_mid(l, d, tol)) return d;
  }
  __atomic_fetch_add(&g_exp2_slow, 1, __ATOMIC_RELAXED);
  __float128 q = exp2q((__float128)y);
  return (double)q;
}

ORC_API void orc_slow_counts(long long *out3) {
  out3[0] = g_log2_slow; out3[1] = g_exp2_slow; out3[2] = g_unresolved;
}

/* ------------------------------------------------------------------------ */
/* Configuration / transform parameters                                       */
/* ------------------------------------------------------------------------ */

typedef struct {
  double b_r;        /* user relative bound (0,1)                           */
  double b_a;        /* float(np.log2(1.0 + b_r)), computed by the host     */
  double onepbr2;    /* (1.0 + b_r) ** 2 evaluated by Python on the host     */
  double eps0;       /* float_floor(float32) = 2^-126                        */
  double repair_t;   /* repair_factor * b_r (D8)                              */
  double coverage_target;
  double slope;      /* leaky ReLU slope                                      */
  double w1[8];      /* (S+1) x H row-major                                   */
  double w2[2];
  int32_t block_rows, block_cols, partition_rows;
  int32_t S, H;      /* S in {1,3}; H = 2                                     */
  int32_t m;         /* 0 => select_m                                         */
  int32_t pad;
} orc_cfg;

typedef struct {
  double factor_pos, factor_neg, eps0, b_r, b_a, boundary, zero_code, zero_threshold, lg_pos, lg_neg;
} orc_params;

/* derive_transform_params (transform.py:110-135).  np.log2(epsilon0) of the
 * f32 floor is exactly -126. */
ORC_API void orc_derive_params(double factor_pos, double factor_neg, double b_r, double b_a,
                               double eps0, orc_params *p) {
  p->factor_pos = factor_pos;
  p->factor_neg = factor_neg;
  p->eps0 = eps0;
  p->b_r = b_r;
  p->b_a = b_a;                                       /* :118 */
  p->lg_pos = orc_log2(factor_pos);                   /* :119 */
  p->lg_neg = orc_log2(factor_neg);                   /* :120 */
  p->zero_code = orc_log2(eps0) + p->lg_pos;          /* :121 */
  p->zero_threshold = p->zero_code + b_a;             /* :122 */
  p->boundary = (p->lg_neg + orc_log2(factor_pos - eps0)) - b_a; /* :123 */
}

/* zero_sub_floor_magnitudes (transform.py:205-210) applied to one element. */
static inline double zfloor(float x, double eps0) {
  double d = (double)x;
  return fabs(d) <= eps0 ? 0.0 : d;
}

/* forward_map (transform.py:170-185) for one element. */
static inline double fwd(double x, const orc_params *p) {
  if (x == 0.0) return p->zero_code;
  double lg = orc_log2(fabs(x));
  return x > 0.0 ? lg + p->lg_pos : lg + p->lg_neg;
}

/* inverse_map (transform.py:188-202) for one element, f64 result. */
static inline double inv(double v, const orc_params *p) {
  if (v <= p->zero_threshold) return 0.0;
  if (v > p->boundary) return -orc_exp2(v - p->lg_neg);
  return orc_exp2(v - p->lg_pos);
}

ORC_API void orc_forward_map(const double *x, int64_t n, const orc_params *p, double *out) {
  for (int64_t i = 0; i < n; i++) out[i] = fwd(x[i], p);
}
ORC_API void orc_inverse_map(const double *v, int64_t n, const orc_params *p, double *out) {
  for (int64_t i = 0; i < n; i++) out[i] = inv(v[i], p);
}

/* compute_block_stats + make_transform_params (transform.py:84-107, 138-167)
 * on the zero-floored block.  Returns 1 for a trivial (all-zero) block. */
static int block_params(const float *x, int64_t ld, int64_t r0, int64_t c0, int64_t br, int64_t bc,
                        const orc_cfg *cfg, orc_params *p, int *status) {
  double amin = INFINITY, amax = 0.0;
  int nonfinite = 0;
  for (int64_t i = 0; i < br; i++)
    for (int64_t j = 0; j < bc; j++) {
      float f = x[(r0 + i) * ld + c0 + j];
      if (!isfinite(f)) { nonfinite = 1; continue; }
      double a = fabs(zfloor(f, cfg->eps0));
      if (a > 0.0) { if (a < amin) amin = a; if (a > amax) amax = a; }
    }
  if (nonfinite) { *status = PMZ_ERR_NONFINITE; return 0; }
  if (amax == 0.0) { memset(p, 0, sizeof(*p)); return 1; }
  double fp = amin;
  double fn = (((amax + cfg->eps0) * fp) * cfg->onepbr2) / (amin - cfg->eps0); /* :160-162 */
  if (!isfinite(fn)) { *status = PMZ_ERR_NONREPRESENTABLE; return 0; }
  orc_derive_params(fp, fn, cfg->b_r, cfg->b_a, cfg->eps0, p);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Predictor / quantizer (D3, D5, D6)               */
/* ------------------------------------------------------------------------ */

ORC_API double orc_predict(const orc_cfg *cfg, const double *s) {
  double a[2];
  for (int j = 0; j < cfg->H; j++) {
    double h;
    if (cfg->S == 3)
      h = ((s[0] * cfg->w1[0 * cfg->H + j] + s[1] * cfg->w1[1 * cfg->H + j]) + s[2] * cfg->w1[2 * cfg->H + j]) +
          cfg->w1[3 * cfg->H + j];
    else
      h = s[0] * cfg->w1[0 * cfg->H + j] + cfg->w1[1 * cfg->H + j];
    a[j] = h < 0.0 ? cfg->slope * h : h;
  }
  return a[0] * cfg->w2[0] + a[1] * cfg->w2[1];
}

static inline double round_half_away(double q) { return round(q); }

/* quantize: candidate = center + round(err / (2 b_a)). */
ORC_API int32_t orc_quantize(double err, double b_a, int32_t m) {
  double q = err / (2.0 * b_a);
  double c = (double)(1 << (m - 1)) + round_half_away(q);
  if (c >= 1.0 && c <= (double)((1 << m) - 1)) return (int32_t)c;
  return 0;
}

/* dequantize. */
ORC_API double orc_dequantize(int32_t code, double b_a, int32_t m) {
  return (double)(code - (1 << (m - 1))) * (2.0 * b_a);
}

/* ------------------------------------------------------------------------ */
/* Block geometry (D14)                              */
/* ------------------------------------------------------------------------ */

typedef struct { int64_t r0, c0, br, bc; } geom;

static inline geom block_geom(int64_t rows, int64_t cols, const orc_cfg *cfg, int64_t b) {
  int64_t nbc = (cols + cfg->block_cols - 1) / cfg->block_cols;
  geom g;
  g.r0 = (b / nbc) * cfg->block_rows;
  g.c0 = (b % nbc) * cfg->block_cols;
  g.br = rows - g.r0 < cfg->block_rows ? rows - g.r0 : cfg->block_rows;
  g.bc = cols - g.c0 < cfg->block_cols ? cols - g.c0 : cfg->block_cols;
  return g;
}

ORC_API int64_t orc_num_blocks(int64_t rows, int64_t cols, int32_t block_rows, int32_t block_cols) {
  if (rows == 0 || cols == 0) return 0;
  return ((rows + block_rows - 1) / block_rows) * ((cols + block_cols - 1) / block_cols);
}

/* m required to cover a rounded residual r: smallest m in [4,16] with
 * |r| <= 2^(m-1)-1; 17 = not coverable. */
static inline int m_required(double r) {
  double a = fabs(r);
  for (int m = 4; m <= 16; m++)
    if (a <= (double)((1 << (m - 1)) - 1)) return m;
  return 17;
}

/* ------------------------------------------------------------------------ */
/* Per-block compression: compress_block + verify_and_repair as one streaming */
/* pass (D1, D2, D4, D7, D8, D9)                   */
/* ------------------------------------------------------------------------ */

typedef struct {
  int trivial;
  orc_params p;
  int64_t nparts;
  uint16_t *codes;   /* br*bc, raster within block; anchors hold 0xFFFF      */
  double *anchors;   /* nparts                                              */
  double *bal;       /* balance values (block order)                         */
  int64_t nbal;
  int64_t nrepair;
  uint64_t mreq[18]; /* true-surface coverage histogram (excl. anchors)      */
} blk_out;

/* When m == 0 only the coverage histogram is produced. */
static int compress_block(const float *x, int64_t ld, geom g, const orc_cfg *cfg, int32_t m, blk_out *o) {
  int st = PMZ_OK;
  memset(o->mreq, 0, sizeof(o->mreq));
  o->nbal = 0; o->nrepair = 0;
  o->trivial = block_params(x, ld, g.r0, g.c0, g.br, g.bc, cfg, &o->p, &st);
  if (st) return st;
  o->nparts = (g.br + cfg->partition_rows - 1) / cfg->partition_rows;
  if (o->trivial) return PMZ_OK;
  const orc_params *p = &o->p;
  int64_t n = g.br * g.bc;
  double *v = (double *)malloc(sizeof(double) * n);
  double *vh = (double *)malloc(sizeof(double) * n);
  if (!v || !vh) { free(v); free(vh); return PMZ_ERR_NOMEM; }
  for (int64_t i = 0; i < g.br; i++)
    for (int64_t j = 0; j < g.bc; j++) v[i * g.bc + j] = fwd(zfloor(x[(g.r0 + i) * ld + g.c0 + j], cfg->eps0), p);
  const double two_ba = 2.0 * cfg->b_a;
  for (int64_t pi = 0; pi < o->nparts; pi++) {
    int64_t pr0 = pi * cfg->partition_rows;
    int64_t pr1 = pr0 + cfg->partition_rows < g.br ? pr0 + cfg->partition_rows : g.br;
    for (int64_t i = pr0; i < pr1; i++)
      for (int64_t j = 0; j < g.bc; j++) {
        int64_t e = i * g.bc + j;
        if (i == pr0 && j == 0) { /* forced anchor, D1 */
          if (o->anchors) o->anchors[pi] = v[e];
          vh[e] = v[e];
          if (o->codes) o->codes[e] = 0xFFFF;
          continue;
        }
        double s[3], sh[3];
        int hw = j > 0, hn = i > pr0;
        s[0] = hw ? v[e - 1] : 0.0;
        s[1] = hn ? v[e - g.bc] : 0.0;
        s[2] = (hw && hn) ? v[e - g.bc - 1] : 0.0;
        double err = v[e] - orc_predict(cfg, s); /* D4: true - predicted */
        if (m == 0) {
          o->mreq[m_required(round_half_away(err / two_ba))]++;
          continue;
        }
        int32_t code = orc_quantize(err, cfg->b_a, m);
        if (code != 0) {
          sh[0] = hw ? vh[e - 1] : 0.0;
          sh[1] = hn ? vh[e - g.bc] : 0.0;
          sh[2] = (hw && hn) ? vh[e - g.bc - 1] : 0.0;
          double vhat = orc_predict(cfg, sh) + orc_dequantize(code, cfg->b_a, m);
          float xh = (float)inv(vhat, p);
          double xz = zfloor(x[(g.r0 + i) * ld + g.c0 + j], cfg->eps0);
          int viol;
          if (xz == 0.0) viol = (xh != 0.0f);
          else viol = fabs((double)xh - xz) / fabs(xz) > cfg->repair_t;
          if (viol) { code = 0; o->nrepair++; }
          else vh[e] = vhat;
        }
        if (code == 0) {
          vh[e] = v[e];
          if (o->bal) o->bal[o->nbal] = v[e];
          o->nbal++;
        }
        if (o->codes) o->codes[e] = (uint16_t)code;
      }
  }
  free(v); free(vh);
  return PMZ_OK;
}

/* ------------------------------------------------------------------------ */
/* Canonical Huffman (D10)                                   */
/* ------------------------------------------------------------------------ */

static const uint64_t *g_sort_freq;
static int cmp_leaf(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  if (g_sort_freq[x] != g_sort_freq[y]) return g_sort_freq[x] < g_sort_freq[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

/* build_codebook: two-queue Huffman over leaves sorted by (freq, code); ties
 * prefer the leaf queue; lengths out.  Not thread-safe (qsort context). */
ORC_API int orc_build_codebook(const uint64_t *freq, int32_t n, uint8_t *len) {
  int32_t nz = 0;
  for (int32_t i = 0; i < n; i++) nz += freq[i] > 0;
  if (nz < 2) return PMZ_ERR_DEGENERATE_ALPHABET;
  int32_t *leaf = (int32_t *)malloc(sizeof(int32_t) * nz);
  uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * 2 * nz);
  int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * 2 * nz);
  if (!leaf || !w || !parent) { free(leaf); free(w); free(parent); return PMZ_ERR_NOMEM; }
  int32_t k = 0;
  for (int32_t i = 0; i < n; i++) if (freq[i] > 0) leaf[k++] = i;
  g_sort_freq = freq;
  qsort(leaf, nz, sizeof(int32_t), cmp_leaf);
  /* nodes 0..nz-1 = leaves in sorted order, nz.. = internal in creation order */
  for (int32_t i = 0; i < nz; i++) w[i] = freq[leaf[i]];
  int32_t lq = 0, iq = nz, nn = nz;
  while (nn < 2 * nz - 1) {
    int32_t pick[2];
    for (int t = 0; t < 2; t++) {
      if (lq < nz && (iq >= nn || w[lq] <= w[iq])) pick[t] = lq++;
      else pick[t] = iq++;
    }
    w[nn] = w[pick[0]] + w[pick[1]];
    parent[pick[0]] = nn; parent[pick[1]] = nn;
    nn++;
  }
  int32_t root = nn - 1;
  /* depth of internal nodes: created in increasing order, parents after children */
  int32_t *depth = (int32_t *)calloc(2 * nz, sizeof(int32_t));
  depth[root] = 0;
  for (int32_t i = root - 1; i >= 0; i--) depth[i] = depth[parent[i]] + 1;
  memset(len, 0, n);
  for (int32_t i = 0; i < nz; i++) len[leaf[i]] = (uint8_t)depth[i];
  free(leaf); free(w); free(parent); free(depth);
  return PMZ_OK;
}

/* canonical codewords in (length, code) order. */
ORC_API int orc_canonical_codes(const uint8_t *len, int32_t n, uint32_t *code) {
  uint32_t bl_count[64] = {0}, next[64] = {0};
  int maxl = 0;
  for (int32_t i = 0; i < n; i++) { bl_count[len[i]]++; if (len[i] > maxl) maxl = len[i]; }
  if (maxl > 32) return PMZ_ERR_UNASSIGNED;
  bl_count[0] = 0;
  uint64_t c = 0;
  for (int b = 1; b <= maxl; b++) { c = (c + bl_count[b - 1]) << 1; next[b] = (uint32_t)c; }
  for (int32_t i = 0; i < n; i++) code[i] = len[i] ? next[len[i]]++ : 0;
  return PMZ_OK;
}

/* ------------------------------------------------------------------------ */
/* Byte writer / reader                                                        */
/* ------------------------------------------------------------------------ */

typedef struct { uint8_t *b; int64_t n, cap; int ovf; } wbuf;
static void wput(wbuf *w, const void *src, int64_t k) {
  if (w->n + k > w->cap) { w->ovf = 1; w->n += k; return; }
  if (w->b) memcpy(w->b + w->n, src, k);
  w->n += k;
}
static void w_u8(wbuf *w, uint8_t v) { wput(w, &v, 1); }
static void w_u16(wbuf *w, uint16_t v) { wput(w, &v, 2); }
static void w_u32(wbuf *w, uint32_t v) { wput(w, &v, 4); }
static void w_u64(wbuf *w, uint64_t v) { wput(w, &v, 8); }
static void w_f64(wbuf *w, double v) { wput(w, &v, 8); }

typedef struct { const uint8_t *b; int64_t n, pos; int err; } rbuf;
static int rget(rbuf *r, void *dst, int64_t k) {
  if (r->pos + k > r->n || k < 0) { r->err = 1; return 0; }
  memcpy(dst, r->b + r->pos, k); r->pos += k; return 1;
}
static uint8_t r_u8(rbuf *r) { uint8_t v = 0; rget(r, &v, 1); return v; }
static uint16_t r_u16(rbuf *r) { uint16_t v = 0; rget(r, &v, 2); return v; }
static uint32_t r_u32(rbuf *r) { uint32_t v = 0; rget(r, &v, 4); return v; }
static uint64_t r_u64(rbuf *r) { uint64_t v = 0; rget(r, &v, 8); return v; }
static double r_f64(rbuf *r) { double v = 0; rget(r, &v, 8); return v; }

/* ------------------------------------------------------------------------ */
/* Full compress (cmd_compress flow; container layout :496)      */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t nblocks, ntrivial, nbal, nrepair, ncodes;
  int32_t m;
  int32_t pad;
  uint64_t header_bytes, total_bytes;
  uint64_t mreq[18];
} orc_result;

/* write the container header (D11, D12) */
static void write_header(wbuf *w, int64_t rows, int64_t cols, const orc_cfg *cfg, int32_t m, const uint8_t *lens,
                         int64_t nblocks) {
  wput(w, "PMEZ", 4);
  w_u16(w, 1);
  w_u8(w, 0);
  w_u64(w, (uint64_t)rows);
  w_u64(w, (uint64_t)cols);
  w_u32(w, (uint32_t)cfg->block_rows);
  w_u32(w, (uint32_t)cfg->block_cols);
  w_u32(w, (uint32_t)cfg->partition_rows);
  w_f64(w, cfg->b_r);
  w_f64(w, cfg->coverage_target);
  w_u8(w, (uint8_t)m);
  int nw1 = (cfg->S + 1) * cfg->H;
  w_u64(w, (uint64_t)(4 + 4 + 8 + 8 * nw1 + 8 * cfg->H));
  w_u32(w, (uint32_t)cfg->S);
  w_u32(w, (uint32_t)cfg->H);
  w_f64(w, cfg->slope);
  for (int i = 0; i < nw1; i++) w_f64(w, cfg->w1[i]);
  for (int i = 0; i < cfg->H; i++) w_f64(w, cfg->w2[i]);
  int32_t alpha = 1 << m;
  w_u64(w, (uint64_t)(2 + alpha));
  w_u16(w, (uint16_t)(alpha & 0xFFFF));
  wput(w, lens, alpha);
  w_u64(w, (uint64_t)nblocks);
}

/* Encode one block record into w (D13, D15). */
static void write_record(wbuf *w, const blk_out *o, geom g, const orc_cfg *cfg, const uint8_t *lens,
                         const uint32_t *cw) {
  if (o->trivial) { w_u8(w, 1); return; }
  w_u8(w, 0);
  w_f64(w, o->p.factor_pos);
  w_f64(w, o->p.factor_neg);
  /* bit lengths per partition */
  uint64_t off = 0;
  for (int64_t pi = 0; pi < o->nparts; pi++) {
    int64_t pr0 = pi * cfg->partition_rows;
    int64_t pr1 = pr0 + cfg->partition_rows < g.br ? pr0 + cfg->partition_rows : g.br;
    uint64_t bits = 0;
    for (int64_t e = pr0 * g.bc + 1; e < pr1 * g.bc; e++) bits += lens[o->codes[e]];
    w_u64(w, off);
    w_u64(w, bits);
    w_f64(w, o->anchors[pi]);
    off += (bits + 7) / 8 * 8;
  }
  w_u64(w, (uint64_t)o->nbal);
  for (int64_t i = 0; i < o->nbal; i++) w_f64(w, o->bal[i]);
  for (int64_t pi = 0; pi < o->nparts; pi++) {
    int64_t pr0 = pi * cfg->partition_rows;
    int64_t pr1 = pr0 + cfg->partition_rows < g.br ? pr0 + cfg->partition_rows : g.br;
    uint64_t acc = 0; int nacc = 0; /* MSB-first bit accumulator */
    for (int64_t e = pr0 * g.bc + 1; e < pr1 * g.bc; e++) {
      uint32_t c = o->codes[e];
      int l = lens[c];
      acc = (acc << l) | cw[c];
      nacc += l;
      while (nacc >= 8) { w_u8(w, (uint8_t)(acc >> (nacc - 8))); nacc -= 8; }
    }
    if (nacc > 0) w_u8(w, (uint8_t)(acc << (8 - nacc)));
  }
}

/* Full compress: returns container bytes written (or needed, when out==NULL /
 * too small: PMZ_ERR_CAPACITY and res->total_bytes = required).
 * val_ids: validation block ids (trainer split, computed by the caller). */
ORC_API int64_t orc_compress(const float *x, int64_t rows, int64_t cols, const orc_cfg *cfg_in,
                             const int64_t *val_ids, int64_t n_val, uint8_t *out, int64_t cap, orc_result *res,
                             uint16_t *codes_dbg /* optional rows*cols */, int32_t nthreads) {
  orc_cfg cfg = *cfg_in;
  memset(res, 0, sizeof(*res));
  if (!(cfg.b_r > 0.0 && cfg.b_r < 1.0)) return PMZ_ERR_CONFIG;
  if (cfg.block_rows <= 0 || cfg.block_cols <= 0 || cfg.partition_rows <= 0) return PMZ_ERR_CONFIG;
  int64_t nb = orc_num_blocks(rows, cols, cfg.block_rows, cfg.block_cols);
  res->nblocks = nb;
  (void)nthreads;
  int st = PMZ_OK;
  /* 1. coverage-based m on validation blocks (select_m; D17) */
  int32_t m = cfg.m;
  if (m == 0) {
    uint64_t tot[18] = {0};
    for (int64_t k = 0; k < n_val; k++) {
      blk_out o; memset(&o, 0, sizeof(o));
      int s = compress_block(x, cols, block_geom(rows, cols, &cfg, val_ids[k]), &cfg, 0, &o);
      if (s) return s;
      for (int i = 0; i < 18; i++) tot[i] += o.mreq[i];
    }
    uint64_t total = 0;
    for (int i = 0; i < 18; i++) total += tot[i];
    memcpy(res->mreq, tot, sizeof(tot));
    m = 16;
    if (total == 0) m = 4;
    else {
      uint64_t cov = 0;
      for (int mm = 4; mm <= 16; mm++) {
        cov += tot[mm];
        if ((double)cov / (double)total >= cfg.coverage_target) { m = mm; break; }
      }
    }
  }
  if (m < 4 || m > 16) return PMZ_ERR_CONFIG;
  res->m = m;
  int32_t alpha = 1 << m;
  /* 2. all blocks: codes + repair (parallel over blocks) */
  blk_out *bo = (blk_out *)calloc(nb > 0 ? nb : 1, sizeof(blk_out));
  if (!bo) return PMZ_ERR_NOMEM;
  int64_t maxn = (int64_t)cfg.block_rows * cfg.block_cols;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t b = 0; b < nb; b++) {
    geom g = block_geom(rows, cols, &cfg, b);
    blk_out *o = &bo[b];
    int64_t n = g.br * g.bc;
    o->codes = (uint16_t *)malloc(sizeof(uint16_t) * (n > 0 ? n : 1));
    o->bal = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    o->anchors = (double *)malloc(sizeof(double) * (cfg.block_rows / cfg.partition_rows + 2));
    int s = compress_block(x, cols, g, &cfg, m, o);
    if (s) {
#pragma omp critical
      st = s;
    }
  }
  (void)maxn;
  if (st) goto done;
  /* 3. codebook from validation histograms (estimate_codebook; D10) */
  {
    uint64_t *freq = (uint64_t *)calloc(alpha, sizeof(uint64_t));
    uint8_t *lens = (uint8_t *)malloc(alpha);
    uint32_t *cw = (uint32_t *)malloc(sizeof(uint32_t) * alpha);
    int64_t kval = 0;
    for (int64_t k = 0; k < n_val; k++) {
      blk_out *o = &bo[val_ids[k]];
      if (o->trivial) continue;
      kval++;
      geom g = block_geom(rows, cols, &cfg, val_ids[k]);
      for (int64_t e = 0; e < g.br * g.bc; e++)
        if (o->codes[e] != 0xFFFF) freq[o->codes[e]]++;
    }
    if (kval == 0) kval = 1;
    for (int32_t s = 0; s < alpha; s++) if (freq[s] < (uint64_t)kval) freq[s] = (uint64_t)kval;
    st = orc_build_codebook(freq, alpha, lens);
    if (!st) st = orc_canonical_codes(lens, alpha, cw);
    if (!st) {
      wbuf w = {out, 0, out ? cap : 0, 0};
      write_header(&w, rows, cols, &cfg, m, lens, nb);
      res->header_bytes = (uint64_t)w.n;
      for (int64_t b = 0; b < nb; b++) {
        geom g = block_geom(rows, cols, &cfg, b);
        write_record(&w, &bo[b], g, &cfg, lens, cw);
        res->ntrivial += bo[b].trivial;
        res->nbal += bo[b].nbal;
        res->nrepair += bo[b].nrepair;
        if (!bo[b].trivial) res->ncodes += g.br * g.bc - bo[b].nparts;
        if (codes_dbg)
          for (int64_t i = 0; i < g.br; i++)
            for (int64_t j = 0; j < g.bc; j++)
              codes_dbg[(g.r0 + i) * cols + g.c0 + j] = bo[b].trivial ? 0xFFFE : bo[b].codes[i * g.bc + j];
      }
      res->total_bytes = (uint64_t)w.n;
      st = w.ovf ? PMZ_ERR_CAPACITY : PMZ_OK;
    }
    free(freq); free(lens); free(cw);
  }
done:
  for (int64_t b = 0; b < nb; b++) { free(bo[b].codes); free(bo[b].bal); free(bo[b].anchors); }
  free(bo);
  if (st) return st;
  return (int64_t)res->total_bytes;
}

/* ------------------------------------------------------------------------ */
/* Decompress (cmd_decompress flow; decompress_block :452)   */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t rows, cols;
  int32_t block_rows, block_cols, partition_rows, m;
  int32_t S, H, version, elem;
  double b_r, coverage_target, slope, w1[8], w2[2];
  int64_t nblocks, header_bytes;
} orc_header;

static int parse_header(rbuf *r, orc_header *h, uint8_t *lens /* >= 65536 */) {
  char mg[4];
  if (!rget(r, mg, 4)) return PMZ_ERR_CORRUPT;
  if (memcmp(mg, "PMEZ", 4) != 0) return PMZ_ERR_BAD_MAGIC;
  h->version = r_u16(r);
  if (r->err) return PMZ_ERR_CORRUPT;
  if (h->version != 1) return PMZ_ERR_UNSUPPORTED_VERSION;
  h->elem = r_u8(r);
  h->rows = (int64_t)r_u64(r);
  h->cols = (int64_t)r_u64(r);
  h->block_rows = (int32_t)r_u32(r);
  h->block_cols = (int32_t)r_u32(r);
  h->partition_rows = (int32_t)r_u32(r);
  h->b_r = r_f64(r);
  h->coverage_target = r_f64(r);
  h->m = r_u8(r);
  uint64_t ml = r_u64(r);
  if (r->err) return PMZ_ERR_CORRUPT;
  if (h->elem != 0) return PMZ_ERR_CORRUPT;
  if (h->m < 4 || h->m > 16 || h->block_rows <= 0 || h->block_cols <= 0 || h->partition_rows <= 0)
    return PMZ_ERR_CORRUPT;
  h->S = (int32_t)r_u32(r);
  h->H = (int32_t)r_u32(r);
  h->slope = r_f64(r);
  if (r->err || h->H != 2 || (h->S != 1 && h->S != 3)) return PMZ_ERR_CORRUPT;
  int nw1 = (h->S + 1) * h->H;
  if (ml != (uint64_t)(16 + 8 * nw1 + 8 * h->H)) return PMZ_ERR_CORRUPT;
  for (int i = 0; i < nw1; i++) h->w1[i] = r_f64(r);
  for (int i = 0; i < h->H; i++) h->w2[i] = r_f64(r);
  uint64_t cl = r_u64(r);
  int32_t alpha = 1 << h->m;
  if (r->err || cl != (uint64_t)(2 + alpha)) return PMZ_ERR_CORRUPT;
  uint16_t a16 = r_u16(r);
  if (a16 != (uint16_t)(alpha & 0xFFFF)) return PMZ_ERR_CORRUPT;
  if (!rget(r, lens, alpha)) return PMZ_ERR_CORRUPT;
  h->nblocks = (int64_t)r_u64(r);
  if (r->err) return PMZ_ERR_CORRUPT;
  if (h->nblocks != orc_num_blocks(h->rows, h->cols, h->block_rows, h->block_cols)) return PMZ_ERR_CORRUPT;
  h->header_bytes = r->pos;
  return PMZ_OK;
}

ORC_API int orc_read_header(const uint8_t *buf, int64_t n, orc_header *h) {
  static uint8_t lens[65536];
  rbuf r = {buf, n, 0, 0};
  return parse_header(&r, h, lens);
}

/* canonical decoder tables */
typedef struct {
  uint32_t first[40], count[40], offset[40];
  int32_t *sym;
  int maxl;
} dec_tab;

static int build_dec(const uint8_t *lens, int32_t n, dec_tab *d) {
  memset(d, 0, sizeof(*d));
  d->sym = (int32_t *)malloc(sizeof(int32_t) * n);
  for (int32_t i = 0; i < n; i++) {
    if (lens[i] > 32) return PMZ_ERR_CORRUPT;
    if (lens[i]) d->count[lens[i]]++;
    if (lens[i] > d->maxl) d->maxl = lens[i];
  }
  /* Kraft equality check */
  long double kraft = 0;
  for (int l = 1; l <= d->maxl; l++) kraft += (long double)d->count[l] / (long double)(1ull << l);
  if (kraft != 1.0L) return PMZ_ERR_CORRUPT;
  uint64_t c = 0; uint32_t o = 0;
  for (int l = 1; l <= d->maxl; l++) {
    c = (c + d->count[l - 1]) << 1;
    if (l == 1) c = 0;
    d->first[l] = (uint32_t)c;
    d->offset[l] = o;
    o += d->count[l];
  }
  uint32_t fill[40];
  memcpy(fill, d->offset, sizeof(fill));
  for (int32_t i = 0; i < n; i++) if (lens[i]) d->sym[fill[lens[i]]++] = i;
  return PMZ_OK;
}

/* decode_next: MSB-first canonical decode. */
static int decode_next(const uint8_t *p, uint64_t nbits, uint64_t *pos, const dec_tab *d, int32_t *sym) {
  uint32_t code = 0;
  for (int l = 1; l <= d->maxl; l++) {
    if (*pos >= nbits) return PMZ_ERR_TRUNCATED;
    code = (code << 1) | ((p[*pos >> 3] >> (7 - (*pos & 7))) & 1);
    (*pos)++;
    if (code - d->first[l] < d->count[l]) { *sym = d->sym[d->offset[l] + code - d->first[l]]; return PMZ_OK; }
  }
  return PMZ_ERR_INVALID_PREFIX;
}

ORC_API int orc_decompress(const uint8_t *buf, int64_t n, double b_a_host, float *out, int64_t out_elems,
                           int64_t *consumed) {
  static uint8_t lens[65536];
  rbuf r = {buf, n, 0, 0};
  orc_header h;
  int st = parse_header(&r, &h, lens);
  if (st) return st;
  if (h.rows * h.cols != out_elems) return PMZ_ERR_CONFIG;
  dec_tab d;
  st = build_dec(lens, 1 << h.m, &d);
  if (st) { free(d.sym); return st; }
  orc_cfg cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.block_rows = h.block_rows; cfg.block_cols = h.block_cols; cfg.partition_rows = h.partition_rows;
  cfg.S = h.S; cfg.H = h.H; cfg.slope = h.slope;
  memcpy(cfg.w1, h.w1, sizeof(cfg.w1)); memcpy(cfg.w2, h.w2, sizeof(cfg.w2));
  cfg.b_r = h.b_r;
  /* b_a = float(np.log2(1.0 + b_r)) is evaluated by the host (transform.py:118) */
  double b_a = isnan(b_a_host) ? orc_log2(1.0 + h.b_r) : b_a_host;
  cfg.b_a = b_a;
  double eps0 = 0x1p-126;
  int32_t m = h.m;
  double *vh = NULL, *bal = NULL;
  int64_t maxn = (int64_t)h.block_rows * h.block_cols;
  vh = (double *)malloc(sizeof(double) * maxn);
  int64_t np_max = (h.block_rows + h.partition_rows - 1) / h.partition_rows;
  uint64_t *poff = (uint64_t *)malloc(8 * np_max), *plen = (uint64_t *)malloc(8 * np_max);
  double *panc = (double *)malloc(8 * np_max);
  for (int64_t b = 0; b < h.nblocks && !st; b++) {
    geom g = block_geom(h.rows, h.cols, &cfg, b);
    uint8_t triv = r_u8(&r);
    if (r.err) { st = PMZ_ERR_CORRUPT; break; }
    if (triv == 1) {
      for (int64_t i = 0; i < g.br; i++)
        for (int64_t j = 0; j < g.bc; j++) out[(g.r0 + i) * h.cols + g.c0 + j] = 0.0f;
      continue;
    }
    if (triv != 0) { st = PMZ_ERR_CORRUPT; break; }
    orc_params p;
    double fp = r_f64(&r), fn = r_f64(&r);
    int64_t np = (g.br + h.partition_rows - 1) / h.partition_rows;
    for (int64_t pi = 0; pi < np; pi++) { poff[pi] = r_u64(&r); plen[pi] = r_u64(&r); panc[pi] = r_f64(&r); }
    uint64_t nbal = r_u64(&r);
    if (r.err || nbal > (uint64_t)(g.br * g.bc) || !(fp > 0) || !(fn > 0)) { st = PMZ_ERR_CORRUPT; break; }
    bal = (double *)realloc(bal, 8 * (nbal + 1));
    for (uint64_t i = 0; i < nbal; i++) bal[i] = r_f64(&r);
    uint64_t payload = 0;
    for (int64_t pi = 0; pi < np; pi++) {
      if (poff[pi] != payload * 8) { st = PMZ_ERR_CORRUPT; break; }
      payload += (plen[pi] + 7) / 8;
    }
    if (st) break;
    const uint8_t *pay = r.b + r.pos;
    if (r.err || r.pos + (int64_t)payload > r.n) { st = PMZ_ERR_TRUNCATED; break; }
    r.pos += payload;
    orc_derive_params(fp, fn, h.b_r, b_a, eps0, &p);
    uint64_t bi = 0;
    for (int64_t pi = 0; pi < np && !st; pi++) {
      int64_t pr0 = pi * h.partition_rows;
      int64_t pr1 = pr0 + h.partition_rows < g.br ? pr0 + h.partition_rows : g.br;
      const uint8_t *sp = pay + poff[pi] / 8;
      uint64_t pos = 0;
      for (int64_t i = pr0; i < pr1 && !st; i++)
        for (int64_t j = 0; j < g.bc; j++) {
          int64_t e = i * g.bc + j;
          if (i == pr0 && j == 0) { vh[e] = panc[pi]; continue; }
          int32_t code;
          st = decode_next(sp, plen[pi], &pos, &d, &code);
          if (st) break;
          if (code == 0) {
            if (bi >= nbal) { st = PMZ_ERR_BALANCE_UNDERFLOW; break; }
            vh[e] = bal[bi++];
          } else {
            double s[3];
            int hw = j > 0, hn = i > pr0;
            s[0] = hw ? vh[e - 1] : 0.0;
            s[1] = hn ? vh[e - g.bc] : 0.0;
            s[2] = (hw && hn) ? vh[e - g.bc - 1] : 0.0;
            vh[e] = orc_predict(&cfg, s) + orc_dequantize(code, b_a, m);
          }
        }
      if (!st && pos != plen[pi]) st = PMZ_ERR_CORRUPT;
    }
    if (!st && bi != nbal) st = PMZ_ERR_CORRUPT;
    if (st) break;
    for (int64_t i = 0; i < g.br; i++)
      for (int64_t j = 0; j < g.bc; j++) out[(g.r0 + i) * h.cols + g.c0 + j] = (float)inv(vh[i * g.bc + j], &p);
  }
  if (!st && consumed) *consumed = r.pos;
  free(vh); free(bal); free(poff); free(plen); free(panc); free(d.sym);
  return st;
}
