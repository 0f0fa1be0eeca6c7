// blockc.cuh -- fused per-block compression kernel: one CTA per compression
// block.
//
//   phase A  compute_block_stats + make_transform_params (transform.py:84-167)
//            over the zero-floored block, all 256 threads;
//   phase B  one warp per 32-row partition.  Columns are processed in chunks
//            of 32: a fully parallel pre-pass (lane = column) forward-maps the
//            chunk and quantizes the TRUE-surface residuals into a 2-slot smem
//            ring; then 32 anti-diagonal steps of the decoder simulation
//            (lane = row) consume the ring, repairing violations on the fly.
//            Only the recurrence (predict from reconstructed neighbours +
//            dequantize + bound check) is on the sequential critical path.
//
// MODE_COVERAGE runs phases A and the pre-pass only and accumulates the
// select_m residual histogram for validation blocks.
#pragma once
#include "common.cuh"
#include "compress.cuh"

namespace pmz {

constexpr int kBW = 8;          // warps per block CTA
constexpr int kCh = 32;         // columns per chunk
constexpr uint16_t kAnchor = 0xFFFF;

enum { MODE_COVERAGE = 0, MODE_CODES = 1 };

struct WarpRing {
  double v[2][32][kCh];          // forward-mapped TRUE values
  uint16_t code[2][32][kCh];     // codes (pre-pass), final codes after the wavefront
};

// Phase A: per-block stats + params into smem (and blkp[b] when requested).
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

// Pre-pass of one chunk (lane = column): forward map every row first (the
// rows are independent, so the compiler overlaps several log2 evaluations),
// then the TRUE-surface codes.  In MODE_COVERAGE accumulates m_required.
template <int MODE, int PK>
__device__ __forceinline__ void prepass_chunk(const float *__restrict__ xp, int64_t ld, int R, int C, int kchunk,
                                              const KParams &k, const BlkP &P, int m, WarpRing &W,
                                              unsigned *cov_s, unsigned *amb) {
  const int lane = threadIdx.x & 31;
  const int slot = kchunk & 1, oslot = slot ^ 1;
  const int c = kchunk * kCh + lane;
  const bool inb = c < C;
#pragma unroll 4
  for (int r = 0; r < R; r++) {
    double v = 0.0;
    if (inb) v = fwd(zfloor(__ldg(xp + r * ld + c)), P, amb);
    W.v[slot][r][lane] = v;
  }
  __syncwarp();
  if (inb) {
#pragma unroll 2
    for (int r = 0; r < R; r++) {
      const double v = W.v[slot][r][lane];
      double w = 0.0, n = 0.0, nw = 0.0;
      if (c > 0) w = lane > 0 ? W.v[slot][r][lane - 1] : W.v[oslot][r][kCh - 1];
      if (r > 0) {
        n = W.v[slot][r - 1][lane];
        if (c > 0) nw = lane > 0 ? W.v[slot][r - 1][lane - 1] : W.v[oslot][r - 1][kCh - 1];
      }
      const bool anchor = (r == 0 && c == 0);
      const double err = __dsub_rn(v, predict_k<PK>(k, w, n, nw));
      if (MODE == MODE_COVERAGE) {
        if (!anchor) atomicAdd(&cov_s[m_required(err, k.two_ba)], 1u);
      } else {
        W.code[slot][r][lane] = anchor ? kAnchor : (uint16_t)quantize_fast(err, k, m);
      }
    }
  }
  __syncwarp();
}

template <int MODE, int PK>
__global__ void __launch_bounds__(kBW * 32, 1) k_compress_blocks(const float *__restrict__ x, Geom g, KParams k,
                                                                 const int64_t *__restrict__ block_ids,
                                                                 BlkP *__restrict__ blkp, WsStatus *st,
                                                                 uint16_t *__restrict__ codes,
                                                                 double *__restrict__ balv,
                                                                 double *__restrict__ anchors,
                                                                 unsigned long long *__restrict__ part_zeros,
                                                                 unsigned long long *__restrict__ cov) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpRing *rings = reinterpret_cast<WarpRing *>(smem_raw);
  __shared__ BlkP sP;
  __shared__ unsigned cov_s[18];
  count_launch(st);
  const int64_t b = block_ids ? block_ids[blockIdx.x] : (int64_t)blockIdx.x;
  const BlockBox bb = block_box(g, b);
  if (MODE == MODE_COVERAGE && threadIdx.x < 18) cov_s[threadIdx.x] = 0;
  block_stats_params(x, g, k, bb, sP, st);
  const BlkP P = sP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = first_part(g, b);
  if (MODE == MODE_CODES && threadIdx.x == 0) {
    blkp[b] = P;
    if (P.trivial) atomicAdd(&st->ntrivial, 1ull);
  }
  if (P.trivial) {
    if (MODE == MODE_CODES)
      for (int pi = threadIdx.x; pi < bb.np; pi += blockDim.x) part_zeros[p0 + pi] = 0;
    return;
  }
  const int m = (MODE == MODE_CODES) ? st->m : 0;
  const int center = (MODE == MODE_CODES) ? (1 << (m - 1)) : 0;
  WarpRing &W = rings[warp];
  unsigned *amb = &st->unresolved;
  for (int pi = warp; pi < bb.np; pi += kBW) {
    const int pr0 = pi * g.prow;
    const int R = min(g.prow, bb.br - pr0);
    const int C = bb.bc;
    const int nch = (C + kCh - 1) / kCh;
    const float *xp = x + (bb.r0 + pr0) * g.cols + bb.c0;
    if (MODE == MODE_COVERAGE) {
      for (int kc = 0; kc < nch; kc++) prepass_chunk<MODE_COVERAGE, PK>(xp, g.cols, R, C, kc, k, P, 0, W, cov_s, amb);
      continue;
    }
    const int64_t grow = bb.r0 + pr0 + lane;
    uint16_t *cpart = codes + (bb.r0 + pr0) * g.cols + bb.c0;
    double *brow = balv + grow * g.cols + bb.c0;
    const int nsteps = C + R - 1;
    const int ngroups = (nsteps + kCh - 1) / kCh;
    double hl = 0.0, hp = 0.0;  // reconstructed W (last) and the one before
    unsigned zeros = 0, repairs = 0;
    for (int kg = 0; kg < ngroups; kg++) {
      if (kg < nch) prepass_chunk<MODE_CODES, PK>(xp, g.cols, R, C, kg, k, P, m, W, nullptr, amb);
      // 32 wavefront steps
      for (int t = kg * kCh; t < min(nsteps, (kg + 1) * kCh); t++) {
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1), nhp = __shfl_up_sync(0xffffffffu, hp, 1);
        const int c = t - lane;
        if (lane < R && c >= 0 && c < C) {
          const int s = (c >> 5) & 1, j = c & (kCh - 1);
          const double v = W.v[s][lane][j];
          int code = W.code[s][lane][j];
          double vh = v;
          if (code == kAnchor) {
            anchors[p0 + pi] = v;  // D1
          } else {
            if (code != 0) {
              const bool hw = c > 0, hn = lane > 0;
              const double vhat = __dadd_rn(predict_k<PK>(k, hw ? hl : 0.0, hn ? nhl : 0.0, (hw && hn) ? nhp : 0.0),
                                            __dmul_rn((double)(code - center), k.two_ba));
              const float xz = zfloor(__ldg(xp + lane * g.cols + c));
              if (check_filtered(vhat, v, xz, P, k, amb)) {
                code = 0;
                repairs++;
                W.code[s][lane][j] = 0;
              } else {
                vh = vhat;
              }
            }
            if (code == 0) {
              brow[c] = v;
              zeros++;
            }
          }
          hp = hl;
          hl = vh;
        }
      }
      __syncwarp();
      // chunk kg-1 is final now: write its codes (lane = column, coalesced)
      if (kg >= 1 && kg - 1 < nch) {
        const int kc = kg - 1, s = kc & 1, c = kc * kCh + lane;
        if (c < C)
          for (int r = 0; r < R; r++) cpart[r * g.cols + c] = W.code[s][r][lane];
      }
      __syncwarp();
    }
    if (ngroups == nch) {  // last chunk not flushed inside the loop
      const int kc = nch - 1, s = kc & 1, c = kc * kCh + lane;
      if (c < C)
        for (int r = 0; r < R; r++) cpart[r * g.cols + c] = W.code[s][r][lane];
      __syncwarp();
    }
    for (int o = 16; o > 0; o >>= 1) {
      zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
      repairs += __shfl_xor_sync(0xffffffffu, repairs, o);
    }
    if (lane == 0) {
      part_zeros[p0 + pi] = zeros;
      atomicAdd(&st->nbal, (unsigned long long)zeros);
      atomicAdd(&st->nrepair, (unsigned long long)repairs);
      atomicAdd(&st->ncodes, (unsigned long long)(R * C - 1));
    }
  }
  if (MODE == MODE_COVERAGE) {
    __syncthreads();
    if (threadIdx.x < 18 && cov_s[threadIdx.x]) atomicAdd(&cov[threadIdx.x], (unsigned long long)cov_s[threadIdx.x]);
  }
}

constexpr size_t kBlockSmem = sizeof(WarpRing) * kBW;

}  // namespace pmz
