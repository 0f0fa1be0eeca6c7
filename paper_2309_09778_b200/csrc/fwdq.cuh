// fwdq.cuh -- the fully parallel half of compress_block:
// forward_map (transform.py:170-185) of every element, its sign/range class,
// and the TRUE-surface residual quantized WITHOUT the m-dependent clamp
// (D5): rq = round_half_away(err / (2 b_a)) when
// |rq| <= 32767, else kRqOut.  code(m) = center + rq when |rq| < center,
// else 0 -- identical to quantize(err, 2 b_a, m) for every m in [4, 16].
//
// The select_m coverage histogram (D17) over validation
// blocks falls out of the same pass: m_required(err) = max(4, bitlen|rq| + 1),
// 17 for kRqOut.
//
// Outputs go to the partition-tiled layout (common.cuh: tile_base).
// One CTA per 32-row partition, swept in 256-column strips: 8 warps forward-map
// a strip (lane = column, 8 interleaved log2 chains per lane) into shared
// memory, then compute the residuals from the shared tile (W / N / NW inside
// the partition; the strip's left neighbour column is kept as a halo).  All
// of it is FP64-throughput work at full occupancy; the sequential
// verify_and_repair recurrence (wsc.cuh) only consumes the results.
#pragma once
#include "common.cuh"
#include "wsc.cuh"

namespace pmz {

constexpr int kFqW = 4;                 // warps per CTA
constexpr int kFqStrip = kFqW * 32;     // columns per strip
constexpr size_t kFqSmem = sizeof(double) * 32 * (kFqStrip + 1);

template <int PK>
__global__ void __launch_bounds__(kFqW * 32, 5) k_fwdq(const float *__restrict__ x, Geom g, KParams k,
                                                   const BlkP *__restrict__ blkp, const uint8_t *__restrict__ vflag,
                                                   WsStatus *st, double *__restrict__ vbuf, int16_t *__restrict__ rqbuf,
                                                   uint8_t *__restrict__ clsbuf, unsigned long long *__restrict__ cov) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double(*sv)[kFqStrip + 1] = reinterpret_cast<double(*)[kFqStrip + 1]>(smem_raw);
  count_launch(st);
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) return;
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const bool val = vflag[b] != 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t off = (bb.r0 + pr0) * g.cols + bb.c0;
  const float *xp = x + off;
  unsigned *amb = &st->unresolved;
  __shared__ unsigned h[18];
  if (threadIdx.x < 18) h[threadIdx.x] = 0;  // first use is after a __syncthreads

  for (int c0 = 0; c0 < C; c0 += kFqStrip) {
    const int j = 1 + warp * 32 + lane;  // smem column (0 = halo)
    const int col = c0 + warp * 32 + lane;
    const bool inb = col < C;
    // ---- forward map of the strip (next batch's loads issued before this
    // batch's log2 chains) ----
    float xn[8];
#pragma unroll
    for (int q = 0; q < 8; q++) xn[q] = (inb && q < R) ? __ldg(xp + (int64_t)q * g.cols + col) : 0.0f;
    for (int rb = 0; rb < R; rb += 8) {
      float xr[8];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        xr[q] = xn[q];
        xn[q] = (inb && rb + 8 + q < R) ? __ldg(xp + (int64_t)(rb + 8 + q) * g.cols + col) : 0.0f;
      }
      double ax[8], lg[8];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const float xz = zfloor(xr[q]);
        ax[q] = xz != 0.0f ? (double)fabsf(xz) : 1.0;
      }
      pmz_log2_f32_fast_n<8>(ax, lg, amb);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (inb && rb + q < R) {
          const float xz = zfloor(xr[q]);
          double v = P.zero_code;
          if (xz > 0.0f) v = __dadd_rn(lg[q], P.lg_pos);
          else if (xz < 0.0f) v = __dadd_rn(lg[q], P.lg_neg);
          sv[rb + q][j] = v;
          const int64_t e = tile_elem(g, p, rb + q, col);
          vbuf[e] = v;
          clsbuf[e] = xclass(xz);
        }
      }
    }
    __syncthreads();
    // ---- TRUE-surface residuals (independent chains, 4 rows per batch) ----
    if (inb) {
      for (int rb = 0; rb < R; rb += 4) {
        int rq[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int r = min(rb + q, R - 1);
          const double v = sv[r][j];
          double w = 0.0, n = 0.0, nw = 0.0;
          if (col > 0) w = sv[r][j - 1];
          if (r > 0) {
            n = sv[r - 1][j];
            if (col > 0) nw = sv[r - 1][j - 1];
          }
          rq[q] = quantize_rq(__dsub_rn(v, predict_k<PK>(k, w, n, nw)), k);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int r = rb + q;
          if (r < R) {
            rqbuf[tile_elem(g, p, r, col)] = (int16_t)rq[q];
            if (val && !(r == 0 && col == 0)) {  // anchors excluded (D17)
              const int mm = m_of_rq(rq[q]);
              const unsigned grp = __match_any_sync(__activemask(), mm);
              if ((grp & ((1u << lane) - 1)) == 0) atomicAdd(&h[mm], (unsigned)__popc(grp));
            }
          }
        }
      }
    }
    __syncthreads();
    if (c0 + kFqStrip < C && threadIdx.x < R) sv[threadIdx.x][0] = sv[threadIdx.x][kFqStrip];
    __syncthreads();
  }
  if (val) {
    __syncthreads();
    if (threadIdx.x < 18 && h[threadIdx.x]) atomicAdd(&cov[threadIdx.x], (unsigned long long)h[threadIdx.x]);
  }
}

// validation flags: vflag[val_ids[i]] = 1
__global__ void k_mark_val(const int64_t *__restrict__ ids, int64_t n, uint8_t *vflag, WsStatus *st) {
  count_launch(st);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) vflag[ids[i]] = 1;
}

}  // namespace pmz
