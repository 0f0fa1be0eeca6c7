/* log2scan.c -- helper of tools/log2_exceptions.py (build-time tool, not
 * product code): compares numpy's np.log2 on float32-derived doubles against
 * the correctly rounded (CR) double, exhaustively.
 *
 * scan(npv, p0, n, ...): npv[i] = np.log2((double)float32_bits(p0 + i)).
 * For every i where npv[i] != CR, record the f32 bit pattern, the direction
 * (+1: numpy is one ulp above CR, -1 below) and where the exact value lies
 * between the two doubles (0.5 = exactly the midpoint).  Also reports, over
 * ALL inputs, the largest |exact - midpoint| (in ulps) of any input whose
 * numpy result differs from CR, and the histogram of CR-vs-midpoint
 * distances (for the GPU certainty band argument).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o log2scan.so log2scan.c -lquadmath -lm */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <string.h>

static double cr_log2_q(double x, __float128 *exact) {
  __float128 q = log2q((__float128)x);
  *exact = q;
  return (double)q;
}

/* CR log2 of a float32-derived double: long double first, __float128 when the
 * long double value is near a midpoint of doubles. */
static double cr_log2(double x, int *slow) {
  long double l = log2l((long double)x);
  double d = (double)l;
  double up = nextafter(d, INFINITY), dn = nextafter(d, -INFINITY);
  long double mu = ((long double)d + (long double)up) * 0.5L;
  long double md = ((long double)d + (long double)dn) * 0.5L;
  long double tol = fabsl(l) * 0x1p-60L;
  if (fabsl(l - mu) > tol && fabsl(l - md) > tol) { *slow = 0; return d; }
  __float128 e;
  *slow = 1;
  return cr_log2_q(x, &e);
}

int64_t scan(const double *npv, uint32_t p0, uint64_t n, uint32_t *out_pat, int8_t *out_dir, double *out_pos,
             int64_t cap, int64_t *nslow) {
  int64_t cnt = 0, slow = 0;
#pragma omp parallel for schedule(static, 65536) reduction(+ : slow)
  for (uint64_t i = 0; i < n; i++) {
    uint32_t pat = p0 + (uint32_t)i;
    float f;
    memcpy(&f, &pat, 4);
    double x = (double)f;
    int s;
    double cr = cr_log2(x, &s);
    slow += s;
    double a = npv[i];
    if (a != cr) {
      __float128 ex;
      cr_log2_q(x, &ex);
      __float128 lo = a < cr ? a : cr, hi = a < cr ? cr : a;
      double pos = (double)((ex - lo) / (hi - lo));
      int64_t k;
#pragma omp atomic capture
      k = cnt++;
      if (k < cap) {
        out_pat[k] = pat;
        out_dir[k] = a > cr ? 1 : -1;
        out_pos[k] = pos;
      }
    }
  }
  *nslow = slow;
  return cnt;
}
