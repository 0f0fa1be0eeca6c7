// common.cuh -- shared device types: geometry, per-block parameters, predictor,
// quantizer, workspace layout.
#pragma once
#include <cstdint>
#ifndef PMZ_UNR_C
#define PMZ_UNR_C 2
#endif
#ifndef PMZ_DREC_MINB
#define PMZ_DREC_MINB 3
#endif
#ifndef PMZ_UNR_C32
#define PMZ_UNR_C32 4
#endif
#ifndef PMZ_UNR_D
#define PMZ_UNR_D 1
#endif
#include <type_traits>
#include <cuda_runtime.h>
#include "../../include/permez_b200.h"
#include "dmath.cuh"

namespace pmz {
constexpr int kUnrC = PMZ_UNR_C, kUnrC32 = PMZ_UNR_C32, kUnrD = PMZ_UNR_D;  // unroll factors of the sweep bodies (A/B builds)


constexpr int kMaxAlpha = 1 << 16;
constexpr int kWarps = 4;  // warps per CTA for per-partition kernels

// Kernel-parameter copy of pmz_params (passed by value -> constant bank).
struct KParams {
  double b_r, b_a, two_ba, onepbr2, eps0, repair_t, slope, coverage_target;
  double inv_two_ba;       // RN(1 / (2 b_a)) for the filtered quantizer
  double dpos, dneg;       // log2(1 + t), log2(1 - t): violation thresholds in the log domain
  double dpos_m, dneg_m;   // dpos - mu, dneg + mu: inside -> certainly within the bound (mu = 2^-20)
  double dpos_p, dneg_p;   // dpos + mu, dneg - mu: outside -> certainly a violation
  double q_half_m;         // 1/2 - M: |frac(q~)| below it rounds like the exact q (cmain.cuh)
  double h_marg;           // |h~| below it: leaky-ReLU sign not certain from approximate surfaces
  double lk[4];            // log2(1 + r) series k1..k4 of the approximate forward map (cmain.cuh)
  double rnd_magic, e_magic;  // 1.5 2^52 (round to integer), 2^52 + 2^31 (int -> double)
  int init_model;          // weights equal init_model: constant-folded predictor
  int precision;           // 0: FP64 parity (container version 1); 1: FP32 perceptron perf mode (version 2)
  unsigned long long code_dump;  // device address of the optional final-code dump (CMainOut::dump), 0 = none
  double w1[8], w2[2];
  int S, H, block_rows, block_cols, partition_rows, m_fixed;
};

// Shard geometry (derived).
struct Geom {
  int64_t rows, cols;        // shard rows, cols
  int64_t nbr, nbc, nblocks; // block grid of the shard
  int64_t block_row0;        // global block-row of the shard's first block-row
  int br, bc, prow;          // block rows/cols, partition rows
  int np_full, np_last;      // partitions per block (full / last block-row)
  int64_t nparts;
  int br_last;               // rows of the last block-row
  int nct;                   // 32x32 tiles per partition row-strip (ceil(bc / 32))
  int fp32;                  // FP32 perceptron perf mode (container version 2): throughput path only
  int force_tpath;           // a final-code dump was requested (throughput-path kernels write it)
};

// Partition-tiled layout of the per-element compress arrays (v, rq, cls):
// partition p, column chunk kc -> one contiguous 32x32 tile (row-major,
// 1024 elements; rows >= R / columns >= C are padding).  A chunk is then one
// bulk copy.
constexpr int kTile = 1024;
constexpr uint16_t kAnc = 0xFFFF;  // code-tile marker of the partition anchor (raster element 0)
__host__ __device__ __forceinline__ int64_t tile_base(const Geom &g, int64_t p, int kc) {
  return (p * g.nct + kc) * (int64_t)kTile;
}
__host__ __device__ __forceinline__ int64_t tile_elem(const Geom &g, int64_t p, int r, int c) {
  return tile_base(g, p, c >> 5) + r * 32 + (c & 31);
}

// Per-block transform parameters (TransformParams fields, transform.py:61-81).
struct BlkP {
  double factor_pos, factor_neg, lg_pos, lg_neg, zero_code, zero_threshold, boundary;
  int trivial;
  int pad;
};

struct BlockBox { int64_t r0, c0; int br, bc, np; };

__host__ __device__ inline BlockBox block_box(const Geom &g, int64_t b) {
  BlockBox bb;
  int64_t bi = b / g.nbc, bj = b - bi * g.nbc;
  bb.r0 = bi * g.br;
  bb.c0 = bj * g.bc;
  int64_t rr = g.rows - bb.r0, cc = g.cols - bb.c0;
  bb.br = (int)(rr < g.br ? rr : g.br);
  bb.bc = (int)(cc < g.bc ? cc : g.bc);
  bb.np = (bb.br + g.prow - 1) / g.prow;
  return bb;
}

// global partition id -> (block, local partition)
__host__ __device__ inline void part_of(const Geom &g, int64_t p, int64_t &b, int &pi) {
  int64_t nfull = (g.nbr - 1) * g.nbc * g.np_full;
  if (p < nfull) { b = p / g.np_full; pi = (int)(p - b * g.np_full); }
  else { int64_t q = p - nfull; b = (g.nbr - 1) * g.nbc + q / g.np_last; pi = (int)(q % g.np_last); }
}
// first global partition id of block b
__host__ __device__ inline int64_t first_part(const Geom &g, int64_t b) {
  int64_t nfullb = (g.nbr - 1) * g.nbc;
  if (b < nfullb) return b * g.np_full;
  return nfullb * g.np_full + (b - nfullb) * g.np_last;
}

// predict with the D3 evaluation order and no contraction.
__device__ __forceinline__ double predict(const KParams &k, double s0, double s1, double s2) {
  double a0, a1;
  if (k.S == 3) {
    double h0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(s0, k.w1[0]), __dmul_rn(s1, k.w1[2])), __dmul_rn(s2, k.w1[4])),
                          k.w1[6]);
    double h1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(s0, k.w1[1]), __dmul_rn(s1, k.w1[3])), __dmul_rn(s2, k.w1[5])),
                          k.w1[7]);
    a0 = h0 < 0.0 ? __dmul_rn(k.slope, h0) : h0;
    a1 = h1 < 0.0 ? __dmul_rn(k.slope, h1) : h1;
  } else {
    double h0 = __dadd_rn(__dmul_rn(s0, k.w1[0]), k.w1[2]);
    double h1 = __dadd_rn(__dmul_rn(s0, k.w1[1]), k.w1[3]);
    a0 = h0 < 0.0 ? __dmul_rn(k.slope, h0) : h0;
    a1 = h1 < 0.0 ? __dmul_rn(k.slope, h1) : h1;
  }
  return __dadd_rn(__dmul_rn(a0, k.w2[0]), __dmul_rn(a1, k.w2[1]));
}

// predict with compile-time init_model weights: the same D3
// expression with constant weights, which the compiler folds (x*1 -> x,
// x*-1 -> -x; the +0.0 bias is kept, so even the sign of zero is identical).
template <int S>
__device__ __forceinline__ double predict_init(double slope, double s0, double s1, double s2) {
  double h;
  if (S == 3) h = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), -s2), 0.0);
  else h = __dadd_rn(s0, 0.0);
  const double a = h < 0.0 ? __dmul_rn(slope, h) : h;
  const double a2 = __dmul_rn(a, 0.5);
  return __dadd_rn(a2, a2);
}

template <int PK>  // 0: general weights, 3 / 1: init_model with S = 3 / 1
__device__ __forceinline__ double predict_k(const KParams &k, double s0, double s1, double s2) {
  if (PK == 3) return predict_init<3>(k.slope, s0, s1, s2);
  if (PK == 1) return predict_init<1>(k.slope, s0, s1, s2);
  return predict(k, s0, s1, s2);
}

// predict_k with a shorter dependency chain, same value as far as any
// consumer can tell (used by the verify/reconstruct recurrences, whose only
// use of the prediction is vhat = pred + dq):
//  * the "+ 0.0" of the init model only turns -0 into +0, and
//    -0 + dq == +0 + dq for every dq (dq = +0 when code == center);
//  * a2 + a2 with a2 = a * 0.5 equals a whenever |a| >= 2^-1021 (the halving
//    is exact), so the two trailing ops are only evaluated for tiny |a|.
template <int PK>
__device__ __forceinline__ double predict_chain(const KParams &k, double s0, double s1, double s2) {
  if (PK == 3 || PK == 1) {
    const double h = PK == 3 ? __dsub_rn(__dadd_rn(s0, s1), s2) : s0;
    const double a = h < 0.0 ? __dmul_rn(k.slope, h) : h;
    if (__builtin_expect(fabs(a) < 0x1p-1020, 0)) {
      const double a2 = __dmul_rn(a, 0.5);
      return __dadd_rn(a2, a2);
    }
    return a;
  }
  return predict(k, s0, s1, s2);
}

// quantize (D5): center + round_half_away(err / (2 b_a)).
__device__ __forceinline__ int quantize(double err, double two_ba, int m) {
  double q = __ddiv_rn(err, two_ba);
  double c = __dadd_rn((double)(1 << (m - 1)), round(q));
  if (c >= 1.0 && c <= (double)((1 << m) - 1)) return (int)c;
  return 0;
}
// Same result as quantize() without the IEEE division: q' = err * RN(1/(2 b_a))
// differs from RN(err / (2 b_a)) by < 2^-51 |q|, so round(q') is exact unless q'
// sits within 2^-48 |q| of a half-integer, where the division decides.
__device__ __forceinline__ int quantize_fast(double err, const KParams &k, int m) {
  const double q = __dmul_rn(err, k.inv_two_ba);
  const double aq = fabs(q);
  if (aq >= 65536.0) return 0;  // out of range for every m <= 16
  const double f = __dsub_rn(aq, trunc(aq));
  if (__builtin_expect(fabs(__dsub_rn(f, 0.5)) <= aq * 0x1p-48, 0)) return quantize(err, k.two_ba, m);
  const double c = __dadd_rn((double)(1 << (m - 1)), round(q));
  if (c >= 1.0 && c <= (double)((1 << m) - 1)) return (int)c;
  return 0;
}

constexpr int16_t kRqOut = (int16_t)-32768;  // |round(q)| > 32767: code 0 for every m
// round_half_away(err / (2 b_a)) with the same exactness argument as
// quantize_fast (reciprocal multiply, IEEE division only near a tie).
__device__ __forceinline__ int quantize_rq(double err, const KParams &k) {
  const double q = __dmul_rn(err, k.inv_two_ba);
  const double aq = fabs(q);
  if (!(aq < 32768.0)) return kRqOut;
  const double f = __dsub_rn(aq, trunc(aq));
  double r;
  if (__builtin_expect(fabs(__dsub_rn(f, 0.5)) <= aq * 0x1p-48, 0)) r = round(__ddiv_rn(err, k.two_ba));
  else r = round(q);
  return fabs(r) <= 32767.0 ? (int)r : (int)kRqOut;
}

__device__ __forceinline__ int code_of_rq(int rq, int center) {
  return (rq != kRqOut && abs(rq) < center) ? center + rq : 0;
}

__device__ __forceinline__ int m_of_rq(int rq) {
  if (rq == kRqOut) return 17;
  const int bl = 32 - __clz(abs(rq));
  return max(4, bl + 1);
}

// smallest m in [4,16] covering round(q); 17 = none (select_m)
__device__ __forceinline__ int m_required(double err, double two_ba) {
  double a = fabs(round(__ddiv_rn(err, two_ba)));
#pragma unroll 1
  for (int m = 4; m <= 16; m++)
    if (a <= (double)((1 << (m - 1)) - 1)) return m;
  return 17;
}
// dequantize (D6)
__device__ __forceinline__ double dequantize(int code, double two_ba, int m) {
  return __dmul_rn((double)(code - (1 << (m - 1))), two_ba);
}

// zero_sub_floor_magnitudes (transform.py:205-210) on one f32 element.
__device__ __forceinline__ float zfloor(float x) {
  return fabsf(x) <= 1.17549435e-38f ? 0.0f : x;
}

// forward_map (transform.py:170-185) of a zero-floored f32 element.
__device__ __forceinline__ double fwd(float xz, const BlkP &p, unsigned *amb) {
  if (xz == 0.0f) return p.zero_code;
  double lg = pmz_log2_f32_fast((double)fabsf(xz), amb);
  return xz > 0.0f ? __dadd_rn(lg, p.lg_pos) : __dadd_rn(lg, p.lg_neg);
}

// inverse_map (transform.py:188-202) + f32 cast (D20).
__device__ __forceinline__ float inv_f32(double v, const BlkP &p, unsigned *amb) {
  if (v <= p.zero_threshold) return 0.0f;
  if (v > p.boundary) return -pmz_exp2_to_f32(__dsub_rn(v, p.lg_neg), amb);
  return pmz_exp2_to_f32(__dsub_rn(v, p.lg_pos), amb);
}

// D8 violation test on the emitted f32 value.
__device__ __forceinline__ bool violates(float xh, float xz, double t) {
  if (xz == 0.0f) return xh != 0.0f;
  double d = fabs(__dsub_rn((double)xh, (double)xz));
  return __ddiv_rn(d, fabs((double)xz)) > t;
}

// verify_and_repair bound check (D8) without exp2 / division in the common
// case.  With d = vhat - v, log2(xhat/x) = d + e where |e| <= 2^-24/ln2 + 2^-43
// (f32 rounding of xhat plus the rounding of v, vhat and their difference),
// so xhat is within the bound when dneg + mu < d < dpos - mu and out of it when
// d > dpos + mu or d < dneg - mu (mu = 2^-20).  Sign crossings, the zero
// threshold, zeros and f32 range extremes always take the exact path.
// Returns 1 = violation, 0 = fine.
__device__ __forceinline__ int check_filtered(double vhat, double v, float xz, const BlkP &P, const KParams &k,
                                              unsigned *amb) {
  const float ax = fabsf(xz);
  if (__builtin_expect(ax > 0.0f, 1)) {
    const bool pos = xz > 0.0f;
    const bool side_ok = pos ? (vhat <= P.boundary) : (vhat > P.boundary);
    if (side_ok && vhat > P.zero_threshold && ax < 1.7e38f && ax > 4.7e-38f) {
      const double d = __dsub_rn(vhat, v);
      const double mu = 0x1p-20;
      if (d < __dsub_rn(k.dpos, mu) && d > __dadd_rn(k.dneg, mu)) return 0;
      if (d > __dadd_rn(k.dpos, mu) || d < __dsub_rn(k.dneg, mu)) return 1;
    }
  } else if (vhat <= P.zero_threshold) {
    return 0;  // x = 0 decodes to exactly 0
  }
  return violates(inv_f32(vhat, P, amb), xz, k.repair_t) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// workspace layout

struct WsStatus {
  unsigned err_bits;     // PMZ error bitmask (1 << -status)
  unsigned unresolved;   // undecided roundings
  int m;                 // selected code width
  int max_len;           // max codeword length
  int n_val_nontrivial;  // k for the histogram floor (D10)
  unsigned launches;     // kernels of this library that ran (counted on device)
  int err_site, err_part;  // first error's raising site / partition (diagnostics, PMZ_DEBUG)
  unsigned long long nbal, nrepair, ntrivial, ncodes;
  unsigned long long total_bytes, header_bytes, record_bytes;
  unsigned long long nfix;  // blocks whose general-double log2 numpy must decide (pmz_*_np_fixups)
};

struct WsLayout {
  size_t status, cov, hist, lens, cw, cb_keys, cb_w, cb_parent, blkp, part_bits, part_zeros, anchors, rec_size,
      rec_off, cub_tmp, codes, balv, zrow, vflag, bstat, npfix, vbuf, rqbuf, clsbuf, total;
  size_t cub_bytes;
};

// ---------------------------------------------------------------------------
// numpy-exact per-block logarithms of general doubles (DESIGN D22).
//
// lg_neg = np.log2(factor_neg) (transform.py:120) and np.log2(factor_pos -
// eps0) (:123) take doubles that are in general not float32 values, so the
// exhaustive float32 table does not cover them.  The device computes the CR
// double; when the exact log2 lies within 2^-56 of a rounding midpoint (numpy
// is never more than 2^-62.6 beyond one on the exhaustive float32 scan), the
// block goes on a list that the host resolves with np.log2 itself
// (pmz_compress_np_fixups / pmz_compress_np_apply, pipeline.py), after which
// the block's parameters are re-derived on the device.
static_assert(sizeof(pmz_np_fix) == 48, "pmz_np_fix layout");

__device__ __forceinline__ bool np_log2_undecided(double x) {
  const float f = __double2float_rn(x);
  if ((double)f == x && f >= 1.17549435e-38f && f <= 3.40282347e38f) return false;  // exact via the table
  return !dd_round_certain(log2_dd_general(x), 0x1p-56);
}

// append block b to the fixup list when one of its two general logarithms is undecided
__device__ __forceinline__ void np_fix_note(WsStatus *st, pmz_np_fix *fix, int64_t b, double fn, double fpe) {
  const int mask = (np_log2_undecided(fn) ? 1 : 0) | (np_log2_undecided(fpe) ? 2 : 0);
  if (mask) {
    const unsigned long long i = atomicAdd(&st->nfix, 1ull);
    pmz_np_fix e;
    e.block = b;
    e.arg[0] = fn;
    e.arg[1] = fpe;
    e.lg[0] = e.lg[1] = 0.0;
    e.mask = mask;
    e.pad = 0;
    fix[i] = e;
  }
}

// count one executed kernel (first thread of the grid)
__device__ __forceinline__ void count_launch(WsStatus *st) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&st->launches, 1u);
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace pmz
