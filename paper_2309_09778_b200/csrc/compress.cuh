// compress.cuh -- block statistics/parameters, coverage, and the fused
// compress_block + verify_and_repair wavefront.
#pragma once
#include "common.cuh"

namespace pmz {

__device__ __forceinline__ void set_err(WsStatus *st, int status) {
  atomicOr(&st->err_bits, 1u << (-status));
}
// set_err that also records where the first error was raised (site >= 1)
__device__ __forceinline__ void set_err_at(WsStatus *st, int status, int site, long long part) {
  set_err(st, status);
  if (atomicCAS(&st->err_site, 0, site) == 0) st->err_part = (int)part;
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

}  // namespace pmz
