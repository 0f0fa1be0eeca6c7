// train.cuh -- the objective of train_step (SURVEY.md §8(f)
// row f1) on the device: for every sample (prediction surface s, target t)
// r = predict(s) - t with the perceptron of the parameter block, and the
// gradient of r^2 w.r.t. every weight (backpropagation through the leaky
// ReLU hidden layer).  Sums are deterministic: per-thread strided
// accumulation, a fixed butterfly per warp, warps in order per CTA, CTA
// partials summed in index order by one thread per component -- bit-identical
// for any launch, so a sweep is reproducible (determinism).
//
// Components of a 12-double result: 0..7 d(sum r^2)/d w1 (row-major
// (S+1) x H, bias row last), 8..9 d/d w2, 10 sum r^2, 11 sample count.
#pragma once
#include "common.cuh"
#include "fwdq.cuh"

namespace pmz {

constexpr int kTrC = 12;
constexpr int kTrT = 256;

// predict (D3 evaluation order) and the r^2 gradient terms of one sample
__device__ __forceinline__ void train_term(const KParams &k, const double *s, double t, double (&acc)[kTrC]) {
  const int S = k.S;
  double h[2], a[2];
#pragma unroll
  for (int j = 0; j < 2; j++) {
    double x = __dmul_rn(s[0], k.w1[j]);
    for (int i = 1; i < S; i++) x = __dadd_rn(x, __dmul_rn(s[i], k.w1[i * 2 + j]));
    h[j] = __dadd_rn(x, k.w1[S * 2 + j]);
    a[j] = h[j] < 0.0 ? __dmul_rn(k.slope, h[j]) : h[j];
  }
  const double out = __dadd_rn(__dmul_rn(a[0], k.w2[0]), __dmul_rn(a[1], k.w2[1]));
  const double r = __dsub_rn(out, t), r2 = __dmul_rn(2.0, r);
  acc[10] = __dadd_rn(acc[10], __dmul_rn(r, r));
#pragma unroll
  for (int j = 0; j < 2; j++) {
    acc[8 + j] = __dadd_rn(acc[8 + j], __dmul_rn(r2, a[j]));
    const double dh = __dmul_rn(__dmul_rn(r2, k.w2[j]), h[j] < 0.0 ? k.slope : 1.0);
    for (int i = 0; i < S; i++) acc[i * 2 + j] = __dadd_rn(acc[i * 2 + j], __dmul_rn(dh, s[i]));
    acc[S * 2 + j] = __dadd_rn(acc[S * 2 + j], dh);
  }
  acc[11] = __dadd_rn(acc[11], 1.0);
}

// CTA-wide fixed-order sum of acc into out[kTrC] (thread 0 writes)
__device__ __forceinline__ void train_cta_sum(double (&acc)[kTrC], double *out) {
  __shared__ double s_w[kTrT / 32][kTrC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kTrC; c++)
    for (int o = 16; o > 0; o >>= 1) acc[c] = __dadd_rn(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], o));
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < kTrC; c++) s_w[warp][c] = acc[c];
  __syncthreads();
  if (threadIdx.x < kTrC) {
    double v = 0.0;
    for (int w = 0; w < kTrT / 32; w++) v = __dadd_rn(v, s_w[w][threadIdx.x]);
    out[threadIdx.x] = v;
  }
}

// Samples = every element of the flagged blocks except the partition
// anchors, surfaces from the TRUE forward-mapped values (vbuf tiles, 0
// outside the partition) -- the surfaces compress_block predicts from.
__global__ void __launch_bounds__(kTrT) k_train_tiles(Geom g, KParams k, const BlkP *__restrict__ blkp,
                                                      const uint8_t *__restrict__ tflag,
                                                      const double *__restrict__ vbuf, double *__restrict__ part) {
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  double acc[kTrC];
#pragma unroll
  for (int c = 0; c < kTrC; c++) acc[c] = 0.0;
  if (tflag[b] && !blkp[b].trivial) {
    const BlockBox bb = block_box(g, b);
    const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc;
    const double *vt = vbuf + tile_base(g, p, 0);
    for (int i = threadIdx.x; i < R * C; i += kTrT) {
      const int r = i / C, c = i - r * C;
      if ((r | c) == 0) continue;  // the anchor is stored raw (D1): not a prediction
      const double t = vt[tile_elem(g, p, r, c) - tile_base(g, p, 0)];
      double s[3];
      if (k.S == 1) {
        s[0] = c > 0 ? vt[tile_elem(g, p, r, c - 1) - tile_base(g, p, 0)] : 0.0;
      } else {
        s[0] = c > 0 ? vt[tile_elem(g, p, r, c - 1) - tile_base(g, p, 0)] : 0.0;
        s[1] = r > 0 ? vt[tile_elem(g, p, r - 1, c) - tile_base(g, p, 0)] : 0.0;
        s[2] = (r > 0 && c > 0) ? vt[tile_elem(g, p, r - 1, c - 1) - tile_base(g, p, 0)] : 0.0;
      }
      train_term(k, s, t, acc);
    }
  }
  train_cta_sum(acc, part + p * kTrC);
}

// Samples given explicitly: surfaces n x S (row-major) and targets.
__global__ void __launch_bounds__(kTrT) k_train_batch(KParams k, const double *__restrict__ surf,
                                                      const double *__restrict__ tgt, uint64_t n,
                                                      double *__restrict__ part) {
  double acc[kTrC];
#pragma unroll
  for (int c = 0; c < kTrC; c++) acc[c] = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * kTrT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kTrT) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < k.S; j++) s[j] = surf[i * k.S + j];
    train_term(k, s, tgt[i], acc);
  }
  train_cta_sum(acc, part + (uint64_t)blockIdx.x * kTrC);
}

// partials[np][kTrC] -> out[kTrC], in index order (thread = component)
__global__ void k_train_reduce(const double *__restrict__ part, int64_t np, double *__restrict__ out) {
  if (threadIdx.x >= kTrC) return;
  double v = 0.0;
  for (int64_t i = 0; i < np; i++) v = __dadd_rn(v, part[i * kTrC + threadIdx.x]);
  out[threadIdx.x] = v;
}

}  // namespace pmz
