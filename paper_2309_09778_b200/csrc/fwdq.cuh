// fwdq.cuh -- the fully parallel half of compress_block,
// two kernels over the partition-tiled layout (common.cuh: tile_base):
//
// k_fwd: forward_map (transform.py:170-185) of every element and its
//   sign/range class.  One CTA per partition; a thread takes 4 consecutive
//   columns of one row (a quad: one 16-byte input load, 4 interleaved log2
//   chains, one 32-byte output store); a warp covers 4 rows x 32 columns.
//   Pure FP64-throughput work, no shared memory.
//
// k_quant: the TRUE-surface residual quantized WITHOUT the m-dependent clamp
//   (D5): rq = round_half_away(err / (2 b_a)) when
//   |rq| <= 32767, else kRqOut, so code(m) = center + rq when |rq| < center,
//   else 0 -- identical to quantize(err, 2 b_a, m) for every m in [4, 16].
//   Neighbours W / N / NW come back from L2 (inside the partition; 0 outside).
//   The select_m coverage histogram (D17) over validation
//   blocks falls out of the same pass: m_required = max(4, bitlen|rq| + 1),
//   17 for kRqOut.
#pragma once
#include "common.cuh"
#include "wsc.cuh"

namespace pmz {

constexpr int kFqT = 256;  // threads per CTA (both kernels)

// Quads of a partition: quad i covers row r, columns c0 .. c0 + 3 of chunk
// kc; 8 R quads per 32-column chunk, so short partitions (one-row 1-D
// inputs) keep every thread busy.  nq = the quads, rounded up to whole warps
// (the warp collectives in k_quant need every lane).
struct QuadMap {
  int q8, nq, nqw;
  __device__ QuadMap(int R, int nch) : q8(8 * R), nq(nch * 8 * R), nqw((nch * 8 * R + 31) & ~31) {}
  __device__ void at(int i, int &kc, int &r, int &c0) const {
    kc = q8 == 256 ? i >> 8 : i / q8;  // full 32-row partitions: shifts
    const int rem = i - kc * q8;
    r = rem >> 3;
    c0 = kc * 32 + (rem & 7) * 4;
  }
};

__global__ void __launch_bounds__(kFqT) k_fwd(const float *__restrict__ x, Geom g, const BlkP *__restrict__ blkp,
                                             WsStatus *st, double *__restrict__ vbuf, uint8_t *__restrict__ clsbuf) {
  count_launch(st);
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) return;
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc, nch = (C + 31) >> 5;
  const float *xp = x + (bb.r0 + pr0) * g.cols + bb.c0;
  const bool vec = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  double *vt = vbuf + tile_base(g, p, 0);
  uint8_t *ct = clsbuf + tile_base(g, p, 0);
  unsigned *amb = &st->unresolved;
  // quad i: row (i >> 3) & 31, columns 32 (i >> 8) + 4 (i & 7) .. + 3; the
  // next quad's input is loaded before this quad's log2 chains
  const QuadMap qm(R, nch);
  auto load_quad = [&](int i, float (&xr)[4]) -> bool {
    if (i >= qm.nq) return false;
    int kc, r, c0;
    qm.at(i, kc, r, c0);
    if (c0 >= C) return false;
    const float *src = xp + (int64_t)r * g.cols + c0;
    if (vec && c0 + 3 < C) {
      const float4 q = __ldg(reinterpret_cast<const float4 *>(src));
      xr[0] = q.x; xr[1] = q.y; xr[2] = q.z; xr[3] = q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; u++) xr[u] = c0 + u < C ? __ldg(src + u) : 0.0f;
    }
    return true;
  };
  float xn[4];
  bool hn = load_quad(threadIdx.x, xn);
  for (int i = threadIdx.x; i < qm.nq; i += kFqT) {
    float xr[4] = {xn[0], xn[1], xn[2], xn[3]};
    const bool h = hn;
    hn = load_quad(i + kFqT, xn);
    if (!h) continue;
    int kc, r, c0;
    qm.at(i, kc, r, c0);
    double ax[4], lg[4], v[4];
    unsigned cl = 0;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const float xz = zfloor(xr[u]);
      ax[u] = xz != 0.0f ? (double)fabsf(xz) : 1.0;
    }
    pmz_log2_f32_fast_n<4>(ax, lg, amb);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const float xz = zfloor(xr[u]);
      v[u] = P.zero_code;
      if (xz > 0.0f) v[u] = __dadd_rn(lg[u], P.lg_pos);
      else if (xz < 0.0f) v[u] = __dadd_rn(lg[u], P.lg_neg);
      cl |= (unsigned)xclass(xz) << (8 * u);
    }
    const int o = kc * kTile + r * 32 + (c0 & 31);
    double2 *vo = reinterpret_cast<double2 *>(vt + o);
    vo[0] = make_double2(v[0], v[1]);
    vo[1] = make_double2(v[2], v[3]);
    *reinterpret_cast<unsigned *>(ct + o) = cl;
  }
}

template <int PK>
__global__ void __launch_bounds__(kFqT) k_quant(Geom g, KParams k, const BlkP *__restrict__ blkp,
                                               const uint8_t *__restrict__ vflag, WsStatus *st,
                                               const double *__restrict__ vbuf, int16_t *__restrict__ rqbuf,
                                               unsigned long long *__restrict__ cov) {
  __shared__ unsigned h[18];
  count_launch(st);
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) return;
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc, nch = (C + 31) >> 5;
  const bool val = vflag[b] != 0 && k.m_fixed == 0;  // coverage only when select_m runs
  if (threadIdx.x < 18) h[threadIdx.x] = 0;
  __syncthreads();
  const double *vt = vbuf + tile_base(g, p, 0);
  int16_t *rt = rqbuf + tile_base(g, p, 0);
  const int lane = threadIdx.x & 31;
  const QuadMap qm(R, nch);
  for (int i = threadIdx.x; i < qm.nqw; i += kFqT) {
    int kc, r, c0;
    qm.at(min(i, qm.nq - 1), kc, r, c0);
    const bool ok = i < qm.nq && c0 < C;
    int rq[4] = {0, 0, 0, 0};
    if (ok) {
      const int o = kc * kTile + r * 32 + (c0 & 31);
      // this row and the row above, columns c0 - 1 .. c0 + 3 (0 outside the partition)
      double cur[5], up[5];
      const double2 *q = reinterpret_cast<const double2 *>(vt + o);
      const double2 a0 = __ldg(q), a1 = __ldg(q + 1);
      cur[1] = a0.x; cur[2] = a0.y; cur[3] = a1.x; cur[4] = a1.y;
      const int ol = (c0 & 31) ? o - 1 : o - kTile + 31;  // left neighbour: previous tile's column 31
      cur[0] = c0 > 0 ? __ldg(vt + ol) : 0.0;
      if (r > 0) {
        const double2 *qu = reinterpret_cast<const double2 *>(vt + o - 32);
        const double2 b0 = __ldg(qu), b1 = __ldg(qu + 1);
        up[1] = b0.x; up[2] = b0.y; up[3] = b1.x; up[4] = b1.y;
        up[0] = c0 > 0 ? __ldg(vt + ol - 32) : 0.0;
      } else {
#pragma unroll
        for (int u = 0; u < 5; u++) up[u] = 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int c = c0 + u;
        if (c < C) rq[u] = quantize_rq(__dsub_rn(cur[u + 1], predict_k<PK>(k, cur[u], up[u + 1], up[u])), k);
      }
      const unsigned lo = ((unsigned)(uint16_t)rq[0]) | ((unsigned)(uint16_t)rq[1] << 16);
      const unsigned hi = ((unsigned)(uint16_t)rq[2]) | ((unsigned)(uint16_t)rq[3] << 16);
      *reinterpret_cast<uint2 *>(rt + o) = make_uint2(lo, hi);
    }
    if (val) {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int c = c0 + u;
        const bool cnt = ok && c < C && (r | c);  // anchors excluded (D17)
        const int mm = cnt ? m_of_rq(rq[u]) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, mm);
        if (cnt && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&h[mm], (unsigned)__popc(grp));
      }
    }
  }
  if (val) {
    __syncthreads();
    if (threadIdx.x < 18 && h[threadIdx.x]) atomicAdd(&cov[threadIdx.x], (unsigned long long)h[threadIdx.x]);
  }
}

// validation flags: vflag[val_ids[i]] = 1; an id outside [0, nblocks) is a
// caller error (ConfigError), never a write
__global__ void k_mark_val(const int64_t *__restrict__ ids, int64_t n, int64_t nblocks, uint8_t *vflag,
                           WsStatus *st) {
  count_launch(st);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = ids[i];
  if (b >= 0 && b < nblocks) vflag[b] = 1;
  else set_err(st, PMZ_ERR_CONFIG);
}

}  // namespace pmz
