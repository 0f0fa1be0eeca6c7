// cmain.cuh -- throughput-path compression, issue-efficient version:
// forward_map (transform.py:170-185), compress_block,
// verify_and_repair and the per-row entropy coding
// (encode) fused into one anti-diagonal sweep per partition
// (k_c_main), then the block records written from the per-row bitstreams
// (k_c_write, write_container SPEC.md:470-477, layout :496).
//
// k_c_main<PK, MODE>: a WARP per 32-row partition, lane = row, 8 partitions
//   per CTA, two CTAs per SM.  The input streams into a 32 x 64 float ring
//   per warp by cp.async in 8-column chunks, three chunks ahead.  At step t
//   lane r takes column c = t - r.
//
//   Exactness without the exact log2 on the common path.  The codes depend on
//   v = np.log2|x| + lg only through round(err / 2b_a) and through the bound
//   filter; both are decided from an APPROXIMATE v (128-entry table + degree-4
//   series, |v~ - v| < 2^-41) with certified margins:
//     * TRUE-surface residual: |q~ - q| < M (cmain_margins, host) so
//       round(q~) = round_half_away(q) unless frac(q~) is within M of 1/2 (or
//       a leaky-ReLU pre-activation within h_marg of 0): those lanes recompute
//       the four TRUE values exactly;
//     * the recurrence (vhat, the RECONSTRUCTED surface) is exact FP64 with the
//       D3 order; the log-domain filter on d = vhat - v~ keeps its 2^-20
//       margins (the v~ error is ~2^-41);
//     * the exact v (numpy-exact log2: CR + exception table, dmath.cuh) is
//       computed only where it is STORED or becomes the recurrence state: the
//       anchor, balance points (code 0: repairs and out-of-range residuals).
//   Everything rare goes through one warp-voted branch per step.
//
//   Outputs (MODE kCMain): each row's canonical codewords MSB-first into its
//   own word slot (rowbits, g.bc words per row), each row's balance values
//   (TRUE v, D9) into its slot of balrow, {bits, count} per row, the anchor,
//   per-partition bit / balance totals.  kCHist: the final-code histogram of
//   the validation blocks in shared memory (estimate_codebook).
//   kCCov: the select_m coverage of the validation blocks' TRUE residuals.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "wsc.cuh"
#include "tdec.cuh"

namespace pmz {

constexpr int kCW = 8;        // warps (partitions) per CTA
constexpr int kCWW = 4;  // warps (partitions) per CTA of k_c_write
constexpr int kWU = 4;   // k_c_write: balance words per lane per round
constexpr int kQU = 2;   // k_c_write: 16-byte stream chunks per lane per round
constexpr int kCRing = 64;    // ring columns per warp (32 x 64 floats = 8 KB)
constexpr int kCTabMax = 1 << 12;   // packed codeword table in shared memory up to this alphabet
constexpr int kCHistMax = 1 << 13;  // validation histogram in shared memory up to this alphabet
enum { kCMain = 0, kCHist = 1, kCCov = 2 };

// log2 reduction table (tools/gen_cmain_tables.py): entry i for mantissas
// m in [1 + i/256, 1 + (i+1)/256): c_i = 1/(1 + (i+0.5)/256) to 29 bits (m c_i
// is exact), -log2(c_i) as a double-double
struct __align__(32) CL2Ent {
  double c, thi, tlo, pad;
};
__device__ const CL2Ent kCL2Tab[256] = {
#include "cmain_tables.inc"
};
constexpr int kCL2Bytes = 256 * sizeof(CL2Ent);

struct CMainOut {
  unsigned *rowbits;            // row slot = g.bc 32-bit words (MSB-first codewords)
  double *balrow;               // row slot = g.bc doubles
  uint2 *rowinfo;               // {bits, balance count} per row
  double *anchors;
  unsigned long long *part_bits, *part_zeros;
  const uint8_t *lens;
  const unsigned *cw;
  unsigned long long *hist, *cov;
  uint16_t *dump;               // optional: every final code, raster per partition (tcode_base), kAnc at the anchor
};

__host__ __device__ inline size_t cmain_smem_bytes(int mode, int m) {
  size_t b = (size_t)kCW * 32 * kCRing * 4 + kCL2Bytes + PMZ_NP_LOG2_BAND_N * 8;
  if (mode == kCMain && m <= 12) b += ((size_t)8 << m) + 8;
  if (mode == kCHist && m <= 13) b += (size_t)4 << m;
  return b;
}

// shared-memory loads by 32-bit shared-window address (no generic-address conversion per access)
__device__ __forceinline__ unsigned lds_u32(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(unsigned a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_d2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

// log2(1 + r) series: k1 as a double-double, k2..k7 (|r| <= 2^-9: truncation < 2^-74)
constexpr double kE1hi = 0x1.71547652b82fep+0, kE1lo = 0x1.777d0ffda0d24p-56;
constexpr double kE2 = -0x1.71547652b82fep-1, kE3 = 0x1.ec709dc3a03fdp-2, kE4 = -0x1.71547652b82fep-2,
                 kE5 = 0x1.2776c50ef9bfep-2, kE6 = -0x1.ec709dc3a03fdp-3, kE7 = 0x1.a61762a7aded9p-3;

// np.log2 of a positive normal float with bits u (transform.py:178-180):
// double-double evaluation on the shared table (|error| < 2^-69 + 2^-60 |L|),
// accepted when that bound (and numpy's deviation band of the result's
// binade, D22) cannot move the rounding; else the precise CR path with the
// exception table (dmath.cuh, ~0.1%)
__device__ __forceinline__ double c_log2_exact(unsigned u, unsigned l2_s, unsigned band_s, unsigned *amb) {
  const unsigned off = (u >> 10) & 0x1fe0u;
  const double2 T = lds_d2(l2_s + off);  // c, -log2 c (hi)
  const double tlo = lds_f64(l2_s + off + 16);
  const double m = __hiloint2double((int)(0x3ff00000u | ((u & 0x7fffffu) >> 3)), (int)(u << 29));
  const double r = __fma_rn(m, T.x, -1.0);  // exact
  const dd P = two_prod(r, kE1hi);
  double q = __fma_rn(r, kE7, kE6);
  q = __fma_rn(r, q, kE5);
  q = __fma_rn(r, q, kE4);
  q = __fma_rn(r, q, kE3);
  q = __fma_rn(r, q, kE2);
  const double tail = __fma_rn(r, kE1lo, __dmul_rn(__dmul_rn(r, r), q));
  // e + thi exactly as a double-double (|e| >= 1 > |thi|, or e = 0: (thi, 0))
  const double ed = __dsub_rn(__hiloint2double(0x43300000, (int)(((u >> 23) - 127u) ^ 0x80000000u)),
                              4503601774854144.0);
  const dd A = fast_two_sum(ed, T.y);
  const dd B = two_sum(A.hi, P.hi);
  const double lo = __dadd_rn(__dadd_rn(__dadd_rn(A.lo, tlo), __dadd_rn(P.lo, tail)), B.lo);
  const dd R = fast_two_sum(B.hi, lo);
  const int bi = (int)((__double_as_longlong(R.hi) >> 52) & 0x7ff) - 1023 - PMZ_NP_LOG2_BAND_MIN;
  const double band = (unsigned)bi < (unsigned)PMZ_NP_LOG2_BAND_N ? lds_f64(band_s + 8u * (unsigned)bi) : 0.0;
  // |R - log2 x| < 2^-70 (series truncation 2^-74.5, tail rounding 2^-71.5) + 2^-104 |L| (dd sums)
  const double bacc = __fma_rn(fabs(R.hi), 0x1p-98, 0x1p-69);
  // numpy deviates from the CR result only within `band` of a rounding midpoint
  if (__builtin_expect(dd_round_certain(R, __dadd_rn(band, bacc)), 1)) return R.hi;
  if (dd_round_certain(R, bacc)) return np_log2_adjust_bits(u, R.hi);  // CR decided: the exception table
  return pmz_log2_f32((double)__uint_as_float(u), amb);
}

// forward_map (transform.py:170-185) of a zero-floored float given as |x| bits + sign
__device__ __forceinline__ double c_fwd_exact(unsigned u, bool neg, const BlkP &P, unsigned l2_s, unsigned band_s,
                                              unsigned *amb) {
  if (u == 0) return P.zero_code;
  return __dadd_rn(c_log2_exact(u, l2_s, band_s, amb), neg ? P.lg_neg : P.lg_pos);
}
__device__ __forceinline__ double c_fwd_exact_f(float xz, const BlkP &P, unsigned l2_s, unsigned band_s,
                                                unsigned *amb) {
  const unsigned b = __float_as_uint(xz);
  return c_fwd_exact(b & 0x7fffffffu, (int)b < 0, P, l2_s, band_s, amb);
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// log2(1 + r) = r (K1 + r (K2 + r (K3 + r K4))) + O(r^5 / 5 ln 2), |r| <= 2^-8
constexpr double kCK1 = 1.4426950408889634, kCK2 = -0.7213475204444817, kCK3 = 0.48089834696298783,
                 kCK4 = -0.36067376022224085;

// predict of approximate TRUE surfaces; amb when a leaky
// pre-activation is too close to 0 for its sign to be certain
template <int PK>
__device__ __forceinline__ double c_pred_approx(const KParams &k, double w, double n, double nw, bool lane0,
                                                bool &amb) {
  if (PK == 3) {
    double h = __dsub_rn(__dadd_rn(w, n), nw);
    h = lane0 ? w : h;
    amb = fabs(h) < k.h_marg;
    return h < 0.0 ? __dmul_rn(k.slope, h) : h;
  }
  const double s1 = lane0 ? 0.0 : n, s2 = lane0 ? 0.0 : nw;
  const double h0 = __dadd_rn(
      __dadd_rn(__dadd_rn(__dmul_rn(w, k.w1[0]), __dmul_rn(s1, k.w1[2])), __dmul_rn(s2, k.w1[4])), k.w1[6]);
  const double h1 = __dadd_rn(
      __dadd_rn(__dadd_rn(__dmul_rn(w, k.w1[1]), __dmul_rn(s1, k.w1[3])), __dmul_rn(s2, k.w1[5])), k.w1[7]);
  amb = (fabs(h0) < k.h_marg) | (fabs(h1) < k.h_marg);
  const double a0 = h0 < 0.0 ? __dmul_rn(k.slope, h0) : h0;
  const double a1 = h1 < 0.0 ? __dmul_rn(k.slope, h1) : h1;
  return __dadd_rn(__dmul_rn(a0, k.w2[0]), __dmul_rn(a1, k.w2[1]));
}

// partition of (CTA, warp): every partition (kCMain), or the partitions of
// the listed validation blocks (cpb CTAs per block)
__device__ __forceinline__ bool c_part(const Geom &g, int mode, const int64_t *val_ids, int64_t nval, int64_t &p,
                                       int64_t &b, int &pi) {
  const int warp = threadIdx.x >> 5;
  if (mode == kCMain) {
    p = (int64_t)blockIdx.x * kCW + warp;
    if (p >= g.nparts) return false;
    part_of(g, p, b, pi);
    return true;
  }
  const int cpb = (g.np_full + kCW - 1) / kCW;
  const int64_t vb = blockIdx.x / cpb;
  if (vb >= nval) return false;
  b = val_ids[vb];
  if (b < 0 || b >= g.nblocks) return false;
  pi = (int)(blockIdx.x % cpb) * kCW + warp;
  if (pi >= block_box(g, b).np) return false;
  p = first_part(g, b) + pi;
  return true;
}

// chain ch of the kCMain sweep: up to L consecutive partitions of one block,
// swept by one warp as ONE wavefront (the 31-step ramp is paid once per chain)
__host__ __device__ inline int64_t c_nchains(const Geom &g, int L) {
  if (g.nbr <= 0) return 0;
  return (g.nbr - 1) * g.nbc * (int64_t)((g.np_full + L - 1) / L) + g.nbc * (int64_t)((g.np_last + L - 1) / L);
}
__device__ __forceinline__ bool c_chain(const Geom &g, int L, int64_t ch, int64_t &p, int64_t &b, int &pi, int &cnt) {
  const int cf = (g.np_full + L - 1) / L, cl = (g.np_last + L - 1) / L;
  const int64_t nfull = (g.nbr - 1) * g.nbc * (int64_t)cf;
  int np;
  if (ch < nfull) {
    b = ch / cf;
    pi = (int)(ch - b * cf) * L;
    np = g.np_full;
  } else {
    const int64_t q = ch - nfull;
    if (q >= g.nbc * (int64_t)cl) return false;
    b = (g.nbr - 1) * g.nbc + q / cl;
    pi = (int)(q % cl) * L;
    np = g.np_last;
  }
  cnt = min(L, np - pi);
  p = first_part(g, b) + pi;
  return true;
}

// classification of a zero-floored float from its bits (xclass, wsc.cuh):
// 0 zero, 1 / 2 positive / negative inside the filter's range, 3 extreme
constexpr unsigned kClsLo = 0x017fe470u;  // bits of 4.7e-38f
constexpr unsigned kClsHi = 0x7effc99eu;  // bits of 1.7e38f

// The rare lanes of one step: the anchor, a TRUE residual at a rounding tie
// (the IEEE division decides, quantize_rq), a leaky-ReLU output below 2^-1020
// (predict_steady's exact form) or a bound check the log-domain filter cannot
// decide (the exact float32 test, D8).  v is the exact TRUE value; (w, n, nw)
// the exact TRUE surface.  Returns the final code; hnew = the RECONSTRUCTED
// value the recurrence continues from.
template <int PK>
__device__ __noinline__ int c_rare(const KParams &k, const BlkP *Pp, int lane, float xz, double v, double w, double n,
                                   double nw, double hl, double nhl, double pn, bool anchor, int center,
                                   unsigned *amb, double *hnew, bool *repaired) {
  const bool lane0 = lane == 0;
  if (!anchor) {
    const BlkP P = *Pp;
    const int rq = quantize_rq(__dsub_rn(v, predict_steady<PK>(k, w, n, nw, lane0)), k);
    if (rq != kRqOut && abs(rq) < center) {
      const double vh = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0), __dmul_rn((double)rq, k.two_ba));
      const double d2 = __dsub_rn(vh, v);
      const int cls = xclass(xz);
      const bool gz2 = vh > P.zero_threshold, gb2 = vh > P.boundary;
      const bool c1 = cls == 1, c2 = cls == 2, is12 = c1 || c2;
      const bool in2 = c1 ? (gz2 && !gb2) : gb2;
      const bool ac = is12 ? (in2 && d2 < k.dpos_m && d2 > k.dneg_m) : (cls == 0 && !gz2);
      bool vio = is12 && ((k.repair_t < 1.0 && !in2) || (in2 && (d2 > k.dpos_p || d2 < k.dneg_p)));
      if (!ac && !vio) vio = violates(inv_f32(vh, P, amb), xz, k.repair_t);
      if (!vio) {
        *hnew = vh;
        return center + rq;
      }
      *repaired = true;
    }
  }
  *hnew = v;
  return 0;
}

#ifdef PMZ_CSTATS
// rare-path reasons (A/B builds only: tools/cstats.py)
__device__ unsigned long long g_cstats[16];
#define CSTAT(i, cond) do { if (cond) cst[i]++; } while (0)
#else
#define CSTAT(i, cond) do { } while (0)
#endif

template <int PK, int MODE, bool STAB>
__global__ void __launch_bounds__(kCW * 32, 2)
    k_c_main(const float *__restrict__ x, Geom g, const __grid_constant__ KParams k, const BlkP *__restrict__ blkp,
             WsStatus *st, const int64_t *__restrict__ val_ids, int64_t nval, CMainOut o, int chain) {
  extern __shared__ __align__(16) unsigned char smem_c[];
  __shared__ unsigned s_cov[18];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *ring = reinterpret_cast<float *>(smem_c) + warp * 32 * kCRing;
  CL2Ent *s_l2 = reinterpret_cast<CL2Ent *>(smem_c + (size_t)kCW * 32 * kCRing * 4);
  double *s_band = reinterpret_cast<double *>(s_l2 + 256);             // numpy log2 deviation bands (D22)
  uint2 *s_tab = reinterpret_cast<uint2 *>(s_band + PMZ_NP_LOG2_BAND_N);  // {codeword, length} (kCMain, STAB)
  unsigned *s_hist = reinterpret_cast<unsigned *>(s_tab);               // validation histogram (kCHist)
  const int m = MODE == kCCov ? 16 : st->m;
  // the codeword table lives in shared memory for alphabets up to 2^12: the
  // launch whose STAB does not match the selected m has nothing to do
  if (MODE == kCMain && STAB != (m <= 12)) return;
  count_launch(st);
  const int nalpha = 1 << m;
  const bool hist_smem = MODE == kCHist && m <= 13;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_l2[i] = kCL2Tab[i];
  for (int i = threadIdx.x; i < PMZ_NP_LOG2_BAND_N; i += blockDim.x) s_band[i] = pmz_np_log2_band[i];
  if (MODE == kCMain && STAB) {
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) s_tab[i] = make_uint2(o.cw[i], o.lens[i]);
    if (threadIdx.x == 0) s_tab[nalpha] = make_uint2(0u, 0u);  // "no code": inactive lanes encode nothing
  }
  if (hist_smem)
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) s_hist[i] = 0;
  if (MODE == kCCov && threadIdx.x < 18) s_cov[threadIdx.x] = 0;
  __syncthreads();

  // kCMain: a chain of cnt consecutive partitions of one block per warp, swept
  // as one wavefront -- lane r goes from the last column of a partition's row
  // straight to the first column of its row in the next partition, so only
  // the chain's first partition pays the 31-step ramp.  The other modes take
  // one partition of a validation block (cnt = 1).
  int64_t p, b;
  int pi, cnt = 1;
  bool have;
  if (MODE == kCMain) have = c_chain(g, chain, (int64_t)blockIdx.x * kCW + warp, p, b, pi, cnt);
  else have = c_part(g, MODE, val_ids, nval, p, b, pi);
  const BlkP *Pp = blkp + (have ? b : 0);
  const BlkP P = have ? *Pp : BlkP{};
  if (have && !P.trivial) {
    const BlockBox bb = block_box(g, b);
    const int C = bb.bc, Cp = (C + 7) & ~7;       // columns; padded to whole 8-column chunks in the sweep
    const int rows_left = bb.br - pi * g.prow;    // rows of the block from the chain's first partition on
    const int nsteps = cnt * Cp + 31;
    const bool vx = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    // loader (warp-uniform): the next chunk = columns l_c0 .. l_c0 + 7 of partition l_q of the chain
    const float *l_xp = x + (bb.r0 + pi * g.prow) * g.cols + bb.c0;
    int l_c0 = 0, l_q = 0;
    auto load_chunk = [&](int kc) {
      if (l_q < cnt) {
        const int R = min(g.prow, rows_left - l_q * g.prow);
        const int slot = (kc * 8) & (kCRing - 1);
        if (vx && l_c0 + 8 <= C) {
#pragma unroll
          for (int j = 0; j < 2; j++) {  // 16 rows x 32 B per instruction
            const int r = j * 16 + (lane >> 1), h = (lane & 1) * 4;
            if (r < R) cp_async16(ring + r * kCRing + slot + h, l_xp + (int64_t)r * g.cols + l_c0 + h);
          }
        } else {
#pragma unroll 1
          for (int j = 0; j < 8; j++) {
            const int r = j * 4 + (lane >> 3), cc = l_c0 + (lane & 7);
            if (r < R && cc < C) cp_async4(ring + r * kCRing + slot + (lane & 7), l_xp + (int64_t)r * g.cols + cc);
          }
        }
        l_c0 += 8;
        if (l_c0 >= Cp) {
          l_c0 = 0;
          l_q++;
          l_xp += (int64_t)g.prow * g.cols;
        }
      }
      cp_async_commit();
    };
    const int center = 1 << (m - 1);
    const double two_ba = k.two_ba, inv = k.inv_two_ba, slope = k.slope;
    const bool tlt1 = k.repair_t < 1.0;
    const double zthr = P.zero_threshold, bnd = P.boundary;
    const double lgp = P.lg_pos, lgn = P.lg_neg, zcode = P.zero_code;
    unsigned *amb = &st->unresolved;
    const bool lane0 = lane == 0;
    // > 0: the lane has a row in its current partition (lanes >= partition_rows never do)
    int rleft = lane < g.prow ? min(rows_left, cnt * g.prow) - lane : -(1 << 28);
    int cb = -lane;  // column in the lane's current partition = t + cb (< 0: not started)
    double vW = 0.0, pnt = 0.0;  // TRUE: own previous value (W), lane - 1's one column back (NW)
    double hl = 0.0, pn = 0.0;   // RECONSTRUCTED (exact): same
    unsigned long long acc = 0;  // row encoder: pending bits, left-aligned
    int na = 0;
    unsigned nb = 0, repairs = 0, tz = 0;
    int64_t row = p * g.prow + lane;
    unsigned *wp = MODE == kCMain ? o.rowbits + row * (int64_t)g.bc : nullptr;
    double *brow = MODE == kCMain ? o.balrow + row * (int64_t)g.bc : nullptr;
    uint16_t *dump = (MODE == kCMain && o.dump) ? o.dump + tcode_base(g, p) + (int64_t)lane * C : nullptr;
#ifdef PMZ_CSTATS
    unsigned cst[2] = {0, 0};
#endif
    const float *myring = ring + lane * kCRing;
    const unsigned ring_s = smem_u32(myring), l2_s = smem_u32(s_l2), tab_s = smem_u32(s_tab),
                   band_s = smem_u32(s_band);
    load_chunk(0);
    load_chunk(1);
    load_chunk(2);
    for (int t0 = 0; t0 < nsteps; t0 += 8) {
      __syncwarp();
      load_chunk((t0 >> 3) + 3);
      cp_async_wait<3>();
      __syncwarp();
      const int t1 = min(nsteps, t0 + 8);
      // one sweep step; SW: some lane ends its row within these 8 steps (the
      // row-end branch is compiled only into that copy of the body)
      auto step = [&](const int t, auto swc) {
        constexpr bool SW = decltype(swc)::value;
        const int gc = t - lane;  // column of the chain's sweep: the ring slot
        const int c = t + cb;     // column in the lane's current partition
        const bool started = gc >= 0;
        const bool lane_in = rleft > 0;
        // first column of a row (SW copy only: rows start right after a row end): W and NW are
        // 0, partition-local neighbours (D2); the registers still hold the previous row's tail
        const bool first = SW && c == 0;
        const bool active = lane_in & ((unsigned)c < (unsigned)C);
        const bool anchor = lane0 & (c == 0);
        // zero_sub_floor_magnitudes + class from the bits (transform.py:205-210; D8 classes)
        const unsigned u0 = lds_u32(ring_s + ((unsigned)(gc & (kCRing - 1)) << 2));
        const unsigned u = (u0 & 0x7fffffffu) <= 0x00800000u ? 0u : (u0 & 0x7fffffffu);
        const bool neg = (int)u0 < 0;
        const bool normal = (u - (kClsLo + 1u)) < (kClsHi - kClsLo - 1u);
        // approximate forward map (transform.py:170-185): |va - v| < 2^-41 (128-entry
        // pairs of the 256-entry table, degree-4 series); the exact v only where it is
        // stored or becomes the recurrence state (balance points, anchor)
        double va;
        {
          const double2 T = lds_d2(l2_s + ((u >> 10) & 0x1fe0u));
          const double mm = __hiloint2double((int)(0x3ff00000u | ((u & 0x7fffffu) >> 3)), (int)(u << 29));
          const double r = __fma_rn(mm, T.x, -1.0);  // exact
          double q4 = __fma_rn(r, k.lk[3], k.lk[2]);
          q4 = __fma_rn(r, q4, k.lk[1]);
          q4 = __fma_rn(r, q4, k.lk[0]);
          const double ed = __dsub_rn(__hiloint2double(0x43300000, (int)(((u >> 23) - 127u) ^ 0x80000000u)),
                                      k.e_magic);
          va = __dadd_rn(__dadd_rn(__dadd_rn(ed, T.y), neg ? lgn : lgp), __dmul_rn(r, q4));
          va = u == 0 ? zcode : va;
        }
        // TRUE-surface residual from approximate surfaces, certified rounding
        const double nvt = __shfl_up_sync(0xffffffffu, vW, 1);
        bool hamb;
        const double at = c_pred_approx<PK>(k, first ? 0.0 : vW, nvt, first ? 0.0 : pnt, lane0, hamb);
        pnt = nvt;
        vW = started ? va : vW;
        const double q = __dmul_rn(__dsub_rn(va, at), inv);
        const double tq = __dadd_rn(q, k.rnd_magic);
        const double qi = __dsub_rn(tq, k.rnd_magic);
        const bool qamb = (fabs(__dsub_rn(q, qi)) >= k.q_half_m) | hamb;
        const int rq = __double2loint(tq);
        const bool qbig = !(fabs(q) < 1073741824.0);
        // exact TRUE surface of this lane (rare paths): the four values by the numpy-exact forward map
        auto exact4 = [&](double &v, double &w, double &n, double &nw) {
          const float *myring = ring + lane * kCRing;
          v = c_fwd_exact(u, neg, P, l2_s, band_s, amb);
          w = c > 0 ? c_fwd_exact_f(zfloor(myring[(gc - 1) & (kCRing - 1)]), P, l2_s, band_s, amb) : 0.0;
          n = lane0 ? 0.0 : c_fwd_exact_f(zfloor(ring[(lane - 1) * kCRing + (gc & (kCRing - 1))]), P, l2_s, band_s, amb);
          nw = (lane0 || c == 0) ? 0.0
                                 : c_fwd_exact_f(zfloor(ring[(lane - 1) * kCRing + ((gc - 1) & (kCRing - 1))]), P,
                                                 l2_s, band_s, amb);
        };
        if (MODE == kCCov) {
          int rqx = qbig ? (int)kRqOut : (abs(rq) > 32767 ? (int)kRqOut : rq);
          if (__builtin_expect(__any_sync(0xffffffffu, active & qamb), 0)) {
            if (active & qamb) {
              double v, w, n, nw;
              exact4(v, w, n, nw);
              rqx = quantize_rq(__dsub_rn(v, predict_steady<PK>(k, w, n, nw, lane0)), k);
            }
          }
          const bool cnt1 = active & !anchor;
          const int mm = cnt1 ? m_of_rq(rqx) : -1;
          const unsigned grp = __match_any_sync(0xffffffffu, mm);
          if (cnt1 && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&s_cov[mm], (unsigned)__popc(grp));
        } else {
          const bool out = qbig | (abs(rq) >= center);
          // decoder simulation on the RECONSTRUCTED surface (exact FP64, D3 order)
          const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
          const double hW = first ? 0.0 : hl, hNW = first ? 0.0 : pn;
          double ar;
          if (PK == 3) {  // predict_init (D3): a w2_0 + a w2_1 with w2 = 1/2, exactly as written
            double h = __dsub_rn(__dadd_rn(hW, nhl), hNW);
            h = lane0 ? hW : h;
            ar = h < 0.0 ? __dmul_rn(slope, h) : h;
            const double a2 = __dmul_rn(ar, 0.5);
            ar = __dadd_rn(a2, a2);
          } else {
            ar = predict_steady<PK>(k, hW, nhl, hNW, lane0);
          }
          const double dq = __dmul_rn(qi, two_ba);
          const double vhat = __dadd_rn(ar, dq);
          const double d = __dadd_rn(ar, __dsub_rn(dq, va));  // vhat - v to ~2^-40: inside the filter's 2^-20 margin
          const bool gz = vhat > zthr, gb = vhat > bnd;
          const bool in12 = normal & (neg ? gb : (gz & !gb));
          const bool inner = (d < k.dpos_m) & (d > k.dneg_m);
          const bool outer = (d > k.dpos_p) | (d < k.dneg_p);
          const bool sure = !qamb & !anchor;
          const bool accept = sure & !out & ((in12 & inner) | ((u == 0) & !gz));
          // certain violations (D8): out-of-range residual, d outside the bound by more than the
          // margin, a sign flip at t < 1 -> balance point (verify_and_repair)
          const bool vcert = sure & (out | (normal & (in12 ? outer : tlt1)));
          int fin = center + rq;
          double hnew = vhat, vbal = 0.0;
          CSTAT(0, active & !accept & !vcert);
          CSTAT(1, active & vcert);
          if (__builtin_expect(__any_sync(0xffffffffu, active & !accept), 0)) {
            if (active & vcert) {  // balance point: the TRUE value, numpy-exact
              vbal = c_fwd_exact(u, neg, P, l2_s, band_s, amb);
              fin = 0;
              hnew = vbal;
              repairs += out ? 0u : 1u;
              if (MODE == kCMain) brow[nb] = vbal;  // the row's balance list (D9)
              nb++;
            } else if (active & !accept) {  // anchor, ties, the filter's undecided band: all exact
              double v, w, n, nw;
              exact4(v, w, n, nw);
              const float xz = __uint_as_float(u | (neg ? 0x80000000u : 0u));
              bool rep = false;
              double hr;  // (addressed only here: the common path keeps hnew in registers)
              fin = c_rare<PK>(k, Pp, lane, xz, v, w, n, nw, hW, nhl, hNW, anchor, center, amb, &hr, &rep);
              hnew = hr;
              repairs += rep ? 1u : 0u;
              if (MODE == kCMain && anchor) o.anchors[p + (-cb) / Cp] = v;  // forced anchor, D1
              if (fin == 0 && !anchor) {
                if (MODE == kCMain) brow[nb] = v;
                nb++;
              }
            }
          }
          pn = nhl;
          hl = started ? hnew : hl;
          if (MODE == kCHist) {
            const bool cnt1 = active & !anchor;
            const int key = cnt1 ? fin : -1;
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            if (cnt1 && (grp & ((1u << lane) - 1)) == 0) {
              if (hist_smem) atomicAdd(&s_hist[fin], (unsigned)__popc(grp));
              else atomicAdd(&o.hist[fin], (unsigned long long)__popc(grp));
            }
          } else {
            const bool enc = active & !anchor;
            if (dump != nullptr && active) dump[c] = anchor ? kAnc : (uint16_t)fin;
            if (STAB) {  // branch-free: lanes without a code take the empty entry
              const uint2 e = lds_v2(tab_s + ((unsigned)(enc ? fin : nalpha) << 3));
              acc |= (unsigned long long)e.x << ((64 - na - (int)e.y) & 63);
              na += (int)e.y;
            } else if (enc) {
              const unsigned cwv = __ldg(o.cw + fin);
              const int len = __ldg(o.lens + fin);
              acc |= (unsigned long long)cwv << (64 - na - len);
              na += len;
            }
            if (na >= 32) {
              *wp++ = (unsigned)(acc >> 32);
              acc <<= 32;
              na -= 32;
            }
          }
        }
        // end of the lane's row: close it and move to the same row of the chain's next
        // partition (surfaces restart from 0: partition-local neighbours, D2)
        if (SW && c == Cp - 1) {
          if (MODE == kCMain) {
            if (lane_in) {
              const unsigned bits = 32u * (unsigned)(wp - (o.rowbits + row * (int64_t)g.bc)) + (unsigned)na;
              if (na) *wp = (unsigned)(acc >> 32);
              o.rowinfo[row] = make_uint2(bits, nb);  // (partition totals: k_c_part_totals)
              tz += nb;
            }
            row += g.prow;
            wp = o.rowbits + row * (int64_t)g.bc;
            brow = o.balrow + row * (int64_t)g.bc;
            if (dump != nullptr) dump += (int64_t)g.prow * g.bc;  // tcode_base of the next partition
          }
          cb -= Cp;
          rleft -= g.prow;
          acc = 0;
          na = 0;
          nb = 0;
        }
      };
      const int cs = t0 + cb;  // a row ends within these 8 steps, or starts at the first of them
      if (__any_sync(0xffffffffu, ((unsigned)(Cp - 1 - cs) < 8u) | (cs == 0))) {
#pragma unroll 1
        for (int t = t0; t < t1; t++) step(t, std::true_type{});
      } else {
#pragma unroll kUnrC
        for (int t = t0; t < t1; t++) step(t, std::false_type{});
      }
    }
    cp_async_wait<0>();
#ifdef PMZ_CSTATS
    for (int i = 0; i < 2; i++)
      if (cst[i]) atomicAdd(&g_cstats[i], (unsigned long long)cst[i]);
#endif
    if (MODE == kCMain) {
      unsigned tr = repairs;
      for (int s = 16; s; s >>= 1) {
        tz += __shfl_xor_sync(0xffffffffu, tz, s);
        tr += __shfl_xor_sync(0xffffffffu, tr, s);
      }
      if (lane == 0) {
        atomicAdd(&st->nbal, (unsigned long long)tz);
        if (tr) atomicAdd(&st->nrepair, (unsigned long long)tr);
        atomicAdd(&st->ncodes, (unsigned long long)((int64_t)min(cnt * g.prow, rows_left) * C - cnt));
      }
    } else if (MODE == kCHist) {
      if (pi == 0 && lane == 0) atomicAdd(&o.hist[kMaxAlpha], 1ull);  // k for the floor (D10)
    }
  }
  if (MODE == kCCov) {
    __syncthreads();
    if (threadIdx.x < 18 && s_cov[threadIdx.x]) atomicAdd(&o.cov[threadIdx.x], (unsigned long long)s_cov[threadIdx.x]);
  }
  if (hist_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&o.hist[i], (unsigned long long)s_hist[i]);
  }
}

// Per-partition bit and balance-point totals from the rows' {bits, count}
// (a warp per partition; trivial blocks have none).  The sweep closes rows one
// lane at a time, so the sums are taken here in one coalesced pass.
__global__ void __launch_bounds__(256) k_c_part_totals(Geom g, const BlkP *__restrict__ blkp,
                                                       const uint2 *__restrict__ rowinfo,
                                                       unsigned long long *part_bits,
                                                       unsigned long long *part_zeros, WsStatus *st) {
  count_launch(st);
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  unsigned tb = 0, tz = 0;
  if (!blkp[b].trivial) {
    const BlockBox bb = block_box(g, b);
    if (lane < min(g.prow, bb.br - pi * g.prow)) {
      const uint2 ri = rowinfo[p * g.prow + lane];
      tb = ri.x;
      tz = ri.y;
    }
  }
  for (int s = 16; s; s >>= 1) {
    tb += __shfl_xor_sync(0xffffffffu, tb, s);
    tz += __shfl_xor_sync(0xffffffffu, tz, s);
  }
  if (lane == 0) {
    part_bits[p] = tb;
    part_zeros[p] = tz;
  }
}

// ---------------------------------------------------------------------------
// k_c_write: block records (D13-D15) from the per-row streams.
// A warp per partition: partition table entry (+ the block head by the first
// partition), the balance values row by row, and the payload -- the rows'
// bitstreams concatenated at their bit offsets -- as aligned 32-bit words of
// the container (bytes at the two ends of the substream), each assembled from
// at most two rows by funnel shifts.
__device__ __forceinline__ unsigned bswap32(unsigned v) { return __byte_perm(v, 0, 0x0123); }

__global__ void __launch_bounds__(kCWW * 32) k_c_write(Geom g, const BlkP *__restrict__ blkp,
                                                       const unsigned *__restrict__ rowbits,
                                                       const double *__restrict__ balrow,
                                                       const uint2 *__restrict__ rowinfo,
                                                       const double *__restrict__ anchors,
                                                       const unsigned long long *__restrict__ part_bits,
                                                       const unsigned long long *__restrict__ part_zeros,
                                                       const unsigned long long *__restrict__ rec_off, uint8_t *out,
                                                       WsStatus *st) {
  count_launch(st);
  if (st->err_bits) return;  // capacity / codebook errors: nothing is written
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * kCWW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  uint8_t *rec = out + st->header_bytes + rec_off[b];
  if (P.trivial) {
    if (pi == 0 && lane == 0) rec[0] = 1;  // trivial block: the flag alone (D13)
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int np = bb.np, pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const int64_t p0 = first_part(g, b);
  unsigned long long pre_bytes = 0, pre_z = 0, tot_z = 0;
  for (int i0 = 0; i0 < np; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long z = i < np ? part_zeros[p0 + i] : 0ull;
    const unsigned long long by = i < pi ? (part_bits[p0 + i] + 7) / 8 : 0ull;
    unsigned long long a = by, zb = i < pi ? z : 0ull, zt = z;
    for (int s = 16; s; s >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, s);
      zb += __shfl_xor_sync(0xffffffffu, zb, s);
      zt += __shfl_xor_sync(0xffffffffu, zt, s);
    }
    pre_bytes += a;
    pre_z += zb;
    tot_z += zt;
  }
  const unsigned long long head = 25ull + 24ull * (unsigned)np;
  if (pi == 0) {
    if (lane == 0) rec[0] = 0;
    if (lane < 8) {
      rec[1 + lane] = (uint8_t)((unsigned long long)__double_as_longlong(P.factor_pos) >> (8 * lane));
      rec[9 + lane] = (uint8_t)((unsigned long long)__double_as_longlong(P.factor_neg) >> (8 * lane));
      rec[17 + 24 * np + lane] = (uint8_t)(tot_z >> (8 * lane));
    }
  }
  const unsigned long long pbits = part_bits[p];
  if (lane < 24) {
    const unsigned long long f =
        lane < 8 ? 8ull * pre_bytes : (lane < 16 ? pbits : (unsigned long long)__double_as_longlong(anchors[p]));
    rec[17 + 24 * pi + lane] = (uint8_t)(f >> (8 * (lane & 7)));
  }
  const uint2 ri = lane < R ? rowinfo[p * g.prow + lane] : make_uint2(0u, 0u);
  unsigned ib = ri.x, iz = ri.y;  // inclusive prefixes over the rows
  for (int s = 1; s < 32; s <<= 1) {
    const unsigned vb = __shfl_up_sync(0xffffffffu, ib, s), vz = __shfl_up_sync(0xffffffffu, iz, s);
    if (lane >= s) {
      ib += vb;
      iz += vz;
    }
  }
  // balance values (D9): rows in order, as aligned 8-byte words of the
  // container (each from at most two values, the two ends byte by byte)
  const unsigned nz = __shfl_sync(0xffffffffu, iz, 31);
  if (nz) {
    const unsigned zstart = iz - ri.y;  // first value index of this lane's row
    const unsigned long long B0 = (unsigned long long)(rec - out) + head + 8ull * pre_z;  // region start (bytes)
    const unsigned long long w0 = B0 >> 3, w1 = (B0 + 8ull * nz - 1) >> 3;
    const unsigned sh = (unsigned)(B0 & 7) * 8;  // bit shift of the values against the aligned words
    const unsigned nwd = (unsigned)(w1 - w0 + 1);
    const double *bbase = balrow + (p * g.prow) * (int64_t)g.bc;
    // value j of the partition's list (j < nz): row search over the rows' value
    // prefixes; kWU words per lane per round, their loads issued together; the
    // word's low value (jA = jB - 1) is the previous word's high one (a shuffle)
    int rlo = 0;
    unsigned long long carry = 0;  // the high value of the round's last word
    for (unsigned j0 = 0; j0 < nwd; j0 += 32u * kWU) {
      const double *pb[kWU];
#pragma unroll
      for (int u = 0; u < kWU; u++) {
        pb[u] = nullptr;
        if (j0 + 32u * u < nwd) {  // warp-uniform
          const unsigned jw = j0 + 32u * u + lane;
          // the word holds the top sh/8 bytes of value jB - 1 and the low bytes of value jB,
          // jB = ceil(ob / 8) with ob = the word's first byte relative to the list (> -8)
          const long long ob = 8ll * (long long)(w0 + jw) - (long long)B0;
          const unsigned jB = (unsigned)((ob + 7) >> 3);
          const unsigned jlast = __shfl_sync(0xffffffffu, jB, 31);
          int rB = rlo;  // row of value jB (warp-uniform loop: every lane shuffles)
          for (int q = rlo + 1; q < R; q++) {
            const unsigned st_q = __shfl_sync(0xffffffffu, zstart, q);
            if (st_q > jlast) break;
            rB = jB >= st_q ? q : rB;
          }
          const unsigned sB = __shfl_sync(0xffffffffu, zstart, rB);
          if (jw < nwd && jB < nz) pb[u] = bbase + (int64_t)rB * g.bc + (jB - sB);
          rlo = __shfl_sync(0xffffffffu, rB, 31);
        }
      }
      unsigned long long vb[kWU];
#pragma unroll
      for (int u = 0; u < kWU; u++) vb[u] = pb[u] ? (unsigned long long)__double_as_longlong(__ldg(pb[u])) : 0ull;
#pragma unroll
      for (int u = 0; u < kWU; u++) {
        const unsigned jw = j0 + 32u * u + lane;
        const unsigned long long up = __shfl_up_sync(0xffffffffu, vb[u], 1);
        const unsigned long long vA = lane == 0 ? carry : up;
        carry = __shfl_sync(0xffffffffu, vb[u], 31);
        // little-endian: the word = the top bytes of vA, then the low bytes of vB
        const unsigned long long v = sh ? ((vA >> (64 - sh)) | (vb[u] << sh)) : vb[u];
        if (jw < nwd) {
          const unsigned long long A = (w0 + jw) * 8ull;
          if (A >= B0 && A + 8 <= B0 + 8ull * nz) {
            *reinterpret_cast<unsigned long long *>(out + A) = v;
          } else {
#pragma unroll
            for (int qb = 0; qb < 8; qb++) {
              const unsigned long long a = A + qb;
              if (a >= B0 && a < B0 + 8ull * nz) out[a] = (uint8_t)(v >> (8 * qb));
            }
          }
        }
      }
    }
  }
  const unsigned long long pay0 = (unsigned long long)(rec - out) + head + 8ull * tot_z + pre_bytes;
  const unsigned total = __shfl_sync(0xffffffffu, ib, 31);
  const unsigned nbytes = (total + 7) >> 3;
  if (nbytes == 0) return;
  const unsigned rstart = ib - ri.x;  // exclusive prefix: first bit of this lane's row
  const unsigned *rbase = rowbits + (p * g.prow) * (int64_t)g.bc;
  if (C < 129) {
    // rows may be shorter than a 16-byte chunk: one lane assembles the partition byte by byte (narrow blocks)
    if (lane == 0) {
      unsigned long long accb = 0;
      int nacc = 0;
      unsigned long long pos = pay0;
      for (int r = 0; r < R; r++) {
        const unsigned rb = rowinfo[p * g.prow + r].x;
        const unsigned *rp = rbase + (int64_t)r * g.bc;
        for (unsigned s = 0; s < rb; s += 8) {
          const unsigned nbit = min(8u, rb - s);
          const unsigned w = rp[s >> 5];
          const unsigned v = (w << (s & 31)) >> (32 - nbit);
          accb = (accb << nbit) | v;
          nacc += (int)nbit;
          if (nacc >= 8) {
            out[pos++] = (uint8_t)(accb >> (nacc - 8));
            nacc -= 8;
            accb &= (1ull << nacc) - 1;
          }
        }
      }
      if (nacc) out[pos] = (uint8_t)(accb << (8 - nacc));
    }
    return;
  }
  // 16-byte chunks of the container overlapping [pay0, pay0 + nbytes): each
  // lane assembles 128 stream bits from at most two rows (rows hold >= 128
  // bits when C > 128; narrower blocks took the lane-0 path above), the two
  // ends byte by byte; kQU chunks per lane per round, their loads issued together
  const unsigned long long q0 = pay0 >> 4, q1 = (pay0 + nbytes - 1) >> 4;
  const unsigned nq = (unsigned)(q1 - q0 + 1);
  int rlo = 0;  // warp-uniform: the row of the next chunk
  for (unsigned jb = 0; jb < nq; jb += 32u * kQU) {
    unsigned w[kQU][5], nx[kQU][4], offv[kQU], rlv[kQU];
    long long sbv[kQU];
#pragma unroll
    for (int u = 0; u < kQU; u++) {
      const unsigned j = jb + 32u * u + lane;
      const long long sb = 8ll * (long long)((q0 + j) * 16ull) - 8ll * (long long)pay0;  // stream bit of the chunk
      const unsigned s = sb < 0 ? 0u : (unsigned)sb;
      sbv[u] = sb;
      offv[u] = 0u;
      rlv[u] = 0u;
#pragma unroll
      for (int k = 0; k < 5; k++) w[u][k] = 0u;
#pragma unroll
      for (int k = 0; k < 4; k++) nx[u][k] = 0u;
      if (jb + 32u * u < nq) {  // warp-uniform
        const unsigned s_last = __shfl_sync(0xffffffffu, s, 31);
        int r = rlo;
        for (int q = rlo + 1; q < R; q++) {
          const unsigned st_q = __shfl_sync(0xffffffffu, rstart, q);
          if (st_q > s_last) break;
          r = s >= st_q ? q : r;
        }
        rlo = __shfl_sync(0xffffffffu, r, 31);
        const unsigned off = s - __shfl_sync(0xffffffffu, rstart, r & 31);
        const unsigned rl = __shfl_sync(0xffffffffu, ri.x, r & 31);
        offv[u] = off;
        rlv[u] = rl;
        if (j < nq && s < total) {
          const unsigned *rp = rbase + (int64_t)r * g.bc;
          const unsigned nwr = (rl + 31) >> 5, wb = off >> 5;
#pragma unroll
          for (int k = 0; k < 5; k++) w[u][k] = wb + k < nwr ? __ldg(rp + wb + k) : 0u;
          if (rl - off < 128 && r + 1 < R) {
            const unsigned *np_ = rbase + (int64_t)(r + 1) * g.bc;
#pragma unroll
            for (int k = 0; k < 4; k++) nx[u][k] = __ldg(np_ + k);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kQU; u++) {
      const unsigned j = jb + 32u * u + lane;
      if (j >= nq) continue;
      const long long sb = sbv[u];
      const unsigned s = sb < 0 ? 0u : (unsigned)sb;
      unsigned o[4] = {0u, 0u, 0u, 0u};
      if (s < total) {
        const unsigned sh = offv[u] & 31;
        const unsigned left = rlv[u] - offv[u];  // bits of row r from s (the row's words are zero past its end)
#pragma unroll
        for (int k = 0; k < 4; k++) {
          unsigned v = __funnelshift_l(w[u][k + 1], w[u][k], sh);  // row r bits from off + 32 k
          // row r + 1 bits: its bit (32 k - left + i) lands at position i of this word
          const int dpos = 32 * k - (int)left;
          unsigned t = 0;
          if (dpos >= 0) {  // dpos < 128: di <= 3
            const unsigned di = (unsigned)dpos >> 5, ds = (unsigned)dpos & 31;
            const unsigned na = di == 0 ? nx[u][0] : (di == 1 ? nx[u][1] : (di == 2 ? nx[u][2] : nx[u][3]));
            const unsigned nb2 = di == 0 ? nx[u][1] : (di == 1 ? nx[u][2] : (di == 2 ? nx[u][3] : 0u));
            t = __funnelshift_l(nb2, na, ds);
          } else if (dpos > -32) {
            t = nx[u][0] >> (unsigned)(-dpos);
          }
          if (left <= 32u * k) v = 0u;
          else if (left < 32u * (k + 1)) v &= ~(0xffffffffu >> (left - 32u * k));
          o[k] = v | t;
        }
        if (sb < 0) {  // the chunk starts before the stream: shift the 128 bits right by -sb (< 128)
          const unsigned d = (unsigned)(-sb);
          unsigned long long hi = ((unsigned long long)o[0] << 32) | o[1], lo = ((unsigned long long)o[2] << 32) | o[3];
          if (d >= 64) {
            lo = hi >> (d - 64);
            hi = 0ull;
          } else {
            lo = (lo >> d) | (hi << (64 - d));
            hi >>= d;
          }
          o[0] = (unsigned)(hi >> 32);
          o[1] = (unsigned)hi;
          o[2] = (unsigned)(lo >> 32);
          o[3] = (unsigned)lo;
        }
      }
      const unsigned long long A = (q0 + j) * 16ull;
      if (A >= pay0 && A + 16 <= pay0 + nbytes) {
        *reinterpret_cast<uint4 *>(out + A) = make_uint4(bswap32(o[0]), bswap32(o[1]), bswap32(o[2]), bswap32(o[3]));
      } else {
#pragma unroll
        for (int qb = 0; qb < 16; qb++) {
          const unsigned long long aq = A + qb;
          if (aq >= pay0 && aq < pay0 + nbytes) out[aq] = (uint8_t)(o[qb >> 2] >> (24 - 8 * (qb & 3)));
        }
      }
    }
  }
}

}  // namespace pmz
