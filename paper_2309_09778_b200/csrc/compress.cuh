// compress.cuh -- block statistics/parameters, coverage, and the fused
// compress_block + verify_and_repair wavefront.
#pragma once
#include "common.cuh"

namespace pmz {

__device__ __forceinline__ void set_err(WsStatus *st, int status) {
  atomicOr(&st->err_bits, 1u << (-status));
}

// Block-wide min/max reduction helpers (256 threads).
template <int NT>
__device__ __forceinline__ void block_minmax(float &mn, float &mx, int &flag) {
  __shared__ float smn[NT / 32], smx[NT / 32];
  __shared__ int sfl[NT / 32];
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    flag |= __shfl_xor_sync(0xffffffffu, flag, o);
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { smn[w] = mn; smx[w] = mx; sfl[w] = flag; }
  __syncthreads();
  if (w == 0) {
    mn = l < NT / 32 ? smn[l] : INFINITY;
    mx = l < NT / 32 ? smx[l] : 0.0f;
    flag = l < NT / 32 ? sfl[l] : 0;
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      flag |= __shfl_xor_sync(0xffffffffu, flag, o);
    }
  }
}

// derive_transform_params (transform.py:110-135) from the serialized fields.
__device__ inline void derive_params(double fp, double fn, const KParams &k, BlkP &o, unsigned *amb) {
  o.factor_pos = fp;
  o.factor_neg = fn;
  o.lg_pos = pmz_log2_d(fp, amb);                                   // :119
  o.lg_neg = pmz_log2_d(fn, amb);                                   // :120
  o.zero_code = __dadd_rn(-126.0, o.lg_pos);                        // :121 (np.log2(eps0) = -126)
  o.zero_threshold = __dadd_rn(o.zero_code, k.b_a);                 // :122
  o.boundary = __dsub_rn(__dadd_rn(o.lg_neg, pmz_log2_d(__dsub_rn(fp, k.eps0), amb)), k.b_a);  // :123
  o.trivial = 0;
}

// K1: compute_block_stats + make_transform_params per block
// (transform.py:84-107, 138-167) on the zero-floored block.
template <int NT>
__global__ void __launch_bounds__(NT) k_block_params(const float *__restrict__ x, Geom g, KParams k, BlkP *blkp,
                                                     WsStatus *st) {
  count_launch(st);
  int64_t b = blockIdx.x;
  BlockBox bb = block_box(g, b);
  float mn = INFINITY, mx = 0.0f;
  int nonfinite = 0;
  for (int r = 0; r < bb.br; r++) {
    const float *row = x + (bb.r0 + r) * g.cols + bb.c0;
    for (int c = threadIdx.x; c < bb.bc; c += NT) {
      float v = row[c];
      if (!isfinite(v)) { nonfinite = 1; continue; }
      float a = fabsf(zfloor(v));
      if (a > 0.0f) { mn = fminf(mn, a); mx = fmaxf(mx, a); }
    }
  }
  block_minmax<NT>(mn, mx, nonfinite);
  if (threadIdx.x == 0) {
    BlkP o;
    if (nonfinite) set_err(st, PMZ_ERR_NONFINITE);
    if (mx == 0.0f) {
      o = BlkP{};
      o.trivial = 1;
      atomicAdd(&st->ntrivial, 1ull);
    } else {
      double fp = (double)mn, amax = (double)mx;
      // transform.py:160-162: ((abs_max + eps0) * factor_pos * (1 + b_r)**2) / (abs_min - eps0)
      double fn = __ddiv_rn(__dmul_rn(__dmul_rn(__dadd_rn(amax, k.eps0), fp), k.onepbr2), __dsub_rn(fp, k.eps0));
      if (!isfinite(fn)) set_err(st, PMZ_ERR_NONREPRESENTABLE);
      derive_params(fp, fn, k, o, &st->unresolved);
    }
    blkp[b] = o;
  }
}

// K2: select_m residual histogram over validation blocks (true surfaces).
template <int NT>
__global__ void __launch_bounds__(NT) k_coverage(const float *__restrict__ x, Geom g, KParams k, const BlkP *blkp,
                                                 const int64_t *val_ids, unsigned long long *cov, WsStatus *st) {
  count_launch(st);
  __shared__ unsigned int h[18];
  if (threadIdx.x < 18) h[threadIdx.x] = 0;
  __syncthreads();
  int64_t b = val_ids[blockIdx.y];
  BlkP p = blkp[b];
  if (!p.trivial) {
    BlockBox bb = block_box(g, b);
    int64_t n = (int64_t)bb.br * bb.bc;
    for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < n; e += (int64_t)gridDim.x * NT) {
      int r = (int)(e / bb.bc), c = (int)(e - (int64_t)r * bb.bc);
      int pr = r % g.prow;
      if (pr == 0 && c == 0) continue;  // anchors excluded (D17)
      const float *row = x + (bb.r0 + r) * g.cols + bb.c0;
      double v = fwd(zfloor(row[c]), p, &st->unresolved);
      double W = c > 0 ? fwd(zfloor(row[c - 1]), p, &st->unresolved) : 0.0;
      double N = 0.0, NW = 0.0;
      if (k.S == 3 && pr > 0) {
        const float *up = row - g.cols;
        N = fwd(zfloor(up[c]), p, &st->unresolved);
        NW = c > 0 ? fwd(zfloor(up[c - 1]), p, &st->unresolved) : 0.0;
      }
      double err = __dsub_rn(v, predict(k, W, N, NW));
      atomicAdd(&h[m_required(err, k.two_ba)], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < 18 && h[threadIdx.x]) atomicAdd(&cov[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// K3: select_m (D17): smallest m in [4,16] whose coverage
// covered/total (f64) meets the target; 16 when none does, 4 with no residuals.
__global__ void k_select_m(const unsigned long long *cov, KParams k, WsStatus *st) {
  count_launch(st);
  if (threadIdx.x != 0) return;
  int m = k.m_fixed;
  if (m == 0) {
    unsigned long long total = 0;
    for (int i = 0; i < 18; i++) total += cov[i];
    m = 16;
    if (total == 0) {
      m = 4;
    } else {
      unsigned long long c = 0;
      for (int mm = 4; mm <= 16; mm++) {
        c += cov[mm];
        if (__ddiv_rn((double)c, (double)total) >= k.coverage_target) { m = mm; break; }
      }
    }
  }
  st->m = m;
}

// K4: compress_block + verify_and_repair as ONE streaming pass per partition
// (D1, D2, D4, D7, D8, D9).  One warp per partition,
// lane = partition row; step t processes the anti-diagonal c = t - lane, so
// N / NW of both the TRUE surface (codes) and the RECONSTRUCTED surface
// (decoder simulation) arrive from lane-1 by shuffle.  A violation turns the
// element into a balance point immediately, which is exactly "earliest
// violation first, re-simulate" because later elements only see earlier ones.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_wavefront(const float *__restrict__ x, Geom g, KParams k,
                                                       const BlkP *__restrict__ blkp, WsStatus *st,
                                                       uint16_t *__restrict__ codes, double *__restrict__ balv,
                                                       double *__restrict__ anchors,
                                                       unsigned long long *__restrict__ part_zeros) {
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * NW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (lane == 0) part_zeros[p] = 0;
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow;
  const int R = min(g.prow, bb.br - pr0);
  const int C = bb.bc;
  const int m = st->m;
  const int64_t grow = bb.r0 + pr0 + lane;
  const float *xrow = x + grow * g.cols + bb.c0;
  uint16_t *crow = codes + grow * g.cols + bb.c0;
  double *brow = balv + grow * g.cols + bb.c0;
  unsigned *amb = &st->unresolved;
  double vl = 0.0, vp = 0.0, hl = 0.0, hp = 0.0;
  unsigned zeros = 0, repairs = 0;
  for (int t = 0; t < C + R - 1; t++) {
    const double nvl = __shfl_up_sync(0xffffffffu, vl, 1), nvp = __shfl_up_sync(0xffffffffu, vp, 1);
    const double nhl = __shfl_up_sync(0xffffffffu, hl, 1), nhp = __shfl_up_sync(0xffffffffu, hp, 1);
    const int c = t - lane;
    if (lane < R && c >= 0 && c < C) {
      const float xz = zfloor(xrow[c]);
      const double v = fwd(xz, P, amb);
      double vh = v;
      if (lane == 0 && c == 0) {
        anchors[p] = v;  // forced anchor, stored raw in the partition table (D1)
      } else {
        const bool hw = c > 0, hn = lane > 0;
        const double err = __dsub_rn(v, predict(k, hw ? vl : 0.0, hn ? nvl : 0.0, (hw && hn) ? nvp : 0.0));
        int code = quantize(err, k.two_ba, m);
        if (code != 0) {
          const double vhat = __dadd_rn(predict(k, hw ? hl : 0.0, hn ? nhl : 0.0, (hw && hn) ? nhp : 0.0),
                                        dequantize(code, k.two_ba, m));
          if (violates(inv_f32(vhat, P, amb), xz, k.repair_t)) {
            code = 0;
            repairs++;
          } else {
            vh = vhat;
          }
        }
        if (code == 0) {
          brow[c] = v;
          zeros++;
        }
        crow[c] = (uint16_t)code;
      }
      vp = vl; vl = v;
      hp = hl; hl = vh;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
    repairs += __shfl_xor_sync(0xffffffffu, repairs, o);
  }
  if (lane == 0) {
    part_zeros[p] = zeros;
    atomicAdd(&st->nbal, (unsigned long long)zeros);
    atomicAdd(&st->nrepair, (unsigned long long)repairs);
    atomicAdd(&st->ncodes, (unsigned long long)(R * C - 1));
  }
}

}  // namespace pmz
