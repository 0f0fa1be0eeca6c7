// blockc.cuh -- compute_block_stats + make_transform_params
// (transform.py:84-167) for one block by one CTA (used by k_stats).
#pragma once
#include "common.cuh"
#include "compress.cuh"

namespace pmz {

constexpr int kBW = 8;          // warps per block CTA


// Per-block stats + params into smem.
__device__ __forceinline__ void block_stats_params(const float *__restrict__ x, const Geom &g, const KParams &k,
                                                   const BlockBox &bb, BlkP &sP, WsStatus *st) {
  float mn = INFINITY, mx = 0.0f;
  int nonfinite = 0;
  auto acc = [&](float v) {
    if (!isfinite(v)) nonfinite = 1;
    const float a = fabsf(v);
    if (a > 1.17549435e-38f && a <= 3.40282347e38f) { mn = fminf(mn, a); mx = fmaxf(mx, a); }
  };
  if ((g.cols & 3) == 0 && (bb.bc & 3) == 0) {
    // float4 path: (rows x bc/4) vectors, 4 independent loads in flight per thread
    const int vpr = bb.bc >> 2;
    const int nv = bb.br * vpr;
    const float *base = x + bb.r0 * g.cols + bb.c0;
    for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * kBW * 32) {
      float4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int i = i0 + u * kBW * 32;
        if (i < nv) {
          const int r = i / vpr, c = (i - r * vpr) << 2;
          q[u] = __ldg(reinterpret_cast<const float4 *>(base + (int64_t)r * g.cols + c));
        } else {
          q[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) { acc(q[u].x); acc(q[u].y); acc(q[u].z); acc(q[u].w); }
    }
  } else {
    const int n = bb.br * bb.bc;
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * kBW * 32) {
      float q[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * kBW * 32;
        if (i < n) {
          const int r = i / bb.bc, c = i - r * bb.bc;
          q[u] = __ldg(x + (bb.r0 + r) * g.cols + bb.c0 + c);
        } else {
          q[u] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; u++) acc(q[u]);
    }
  }
  block_minmax<kBW * 32>(mn, mx, nonfinite);
  __shared__ double s_fn;
  if (threadIdx.x == 0) {
    if (nonfinite) set_err(st, PMZ_ERR_NONFINITE);
    sP = BlkP{};
    if (mx == 0.0f) {
      sP.trivial = 1;
    } else {
      double fp = (double)mn, amax = (double)mx;
      // transform.py:160-162
      s_fn = __ddiv_rn(__dmul_rn(__dmul_rn(__dadd_rn(amax, k.eps0), fp), k.onepbr2), __dsub_rn(fp, k.eps0));
      if (!isfinite(s_fn)) set_err(st, PMZ_ERR_NONREPRESENTABLE);
      sP.factor_pos = fp;
      sP.factor_neg = s_fn;
    }
  }
  __syncthreads();
  if (!sP.trivial) {
    // the three per-block logarithms in parallel (transform.py:119-123)
    double r = 0.0;
    if (threadIdx.x == 0) r = pmz_log2_d(sP.factor_pos, &st->unresolved);
    if (threadIdx.x == 32) r = pmz_log2_d(sP.factor_neg, &st->unresolved);
    if (threadIdx.x == 64) r = pmz_log2_d(__dsub_rn(sP.factor_pos, k.eps0), &st->unresolved);
    __shared__ double s_l[3];
    if ((threadIdx.x & 31) == 0 && threadIdx.x < 96) s_l[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
      sP.lg_pos = s_l[0];
      sP.lg_neg = s_l[1];
      sP.zero_code = __dadd_rn(-126.0, sP.lg_pos);
      sP.zero_threshold = __dadd_rn(sP.zero_code, k.b_a);
      sP.boundary = __dsub_rn(__dadd_rn(sP.lg_neg, s_l[2]), k.b_a);
    }
  }
  __syncthreads();
}

}  // namespace pmz
