// dsc.cuh -- warp-specialized decompress_block + inverse_map
// (transform.py:188-202).
//
// One warp PAIR per 32-row partition (same scheme as wsc.cuh):
//   producer (lane = column): stages each 32-column chunk of decoded codes and,
//     for code-0 positions, the next balance values (block-level list, raster
//     order within the partition, D9) into a 3-deep ring; when the consumer has
//     finished a chunk it inverse-maps the reconstructed values to float32 and
//     stores them coalesced (lane = column);
//   consumer (lane = row): the reconstructed-surface recurrence only:
//     vhat = predict(RECONSTRUCTED W, N, NW) + dequantize(code), or the balance
//     value for code 0 (anti-diagonal steps, shuffles for N / NW).
#pragma once
#include "common.cuh"
#include "wsc.cuh"

namespace pmz {

// ---------------------------------------------------------------------------
// k_reconstruct4: the recurrence over the tiles written by k_decode4 (codes +
// per-element addends: balance value at code 0, dequantized residual
// elsewhere).  Warp pair per partition:
//   producer: one elected lane streams the code and addend tile of each
//     32-column chunk into a 3-deep ring with bulk copies on an mbarrier and,
//     when the consumer has finished a chunk, stores its reconstructed tile
//     back with one bulk copy (the inverse map runs in k_inv);
//   consumer (lane = row): vhat = code 0 ? balance value : predict(W, N, NW) +
//     dequantize(code) -- predicated, software-pipelined, one shuffle per step
//     (see k_compress_ws).
struct alignas(128) DRing4 {
  double val[kSlots][kTile];     // addend in; reconstructed value out
  uint16_t code[kSlots][kTile];
  unsigned long long full[kSlots];
};
constexpr size_t kDsc4Smem = sizeof(DRing4) * kPPC;

template <int PK>
__global__ void __launch_bounds__(kPPC * 64) k_reconstruct4(Geom g, KParams k, const BlkP *__restrict__ blkp,
                                                            const uint16_t *__restrict__ codes,
                                                            const double *vtile,
                                                            const double *__restrict__ anchors,
                                                            float *__restrict__ out, double *vh,
                                                            WsStatus *st) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;
  DRing4 &W = reinterpret_cast<DRing4 *>(smem_raw)[pair];
  const int64_t p = (int64_t)blockIdx.x * kPPC + pair;
  if (role == 0 && lane == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&W.full[s], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const int nch = (C + 31) >> 5;
  if (blkp[b].trivial) {
    if (role == 0) {
      float *opart = out + (bb.r0 + pr0) * g.cols + bb.c0;
      for (int r = 0; r < R; r++)
        for (int c = lane; c < C; c += 32) opart[(int64_t)r * g.cols + c] = 0.0f;
    }
    return;
  }
  if (st->err_bits) return;  // the decoder failed: its tiles are incomplete
  const int bar0 = 1 + pair * kSlots;  // empty[s] = bar0 + s (named barriers, 64 threads)
  const int64_t tb = tile_base(g, p, 0);

  if (role == 0) {
    // ------------------------------ producer ------------------------------
    for (int kc = 0; kc < nch; kc++) {
      const int s = kc % kSlots;
      if (kc >= kSlots) {
        bar_sync_n(bar0 + s, 64);  // the consumer is done with chunk kc - kSlots
        if (lane == 0) {
          bulk_s2g(vh + tb + (int64_t)(kc - kSlots) * kTile, W.val[s], kTile * 8);
          bulk_commit();
          bulk_wait_read0();  // the store has read the slot
        }
      }
      if (lane == 0) {
        mbar_expect_tx(&W.full[s], kTile * 10);
        bulk_g2s(W.val[s], vtile + tb + (int64_t)kc * kTile, kTile * 8, &W.full[s]);
        bulk_g2s(W.code[s], codes + tb + (int64_t)kc * kTile, kTile * 2, &W.full[s]);
      }
      __syncwarp();
    }
    for (int kc = max(0, nch - kSlots); kc < nch; kc++) {
      bar_sync_n(bar0 + kc % kSlots, 64);
      if (lane == 0) {
        bulk_s2g(vh + tb + (int64_t)kc * kTile, W.val[kc % kSlots], kTile * 8);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ------------------------------ consumer ------------------------------
    const double anc = anchors[p];
    const int nsteps = C + R - 1;
    const int ngroups = (nsteps + 31) >> 5;
    const bool lane0 = lane == 0, lane_in = lane < R;
    double hl = 0.0, pn = 0.0;
    for (int kg = 0; kg < ngroups; kg++) {
      if (kg < nch) mbar_wait(&W.full[kg % kSlots], (unsigned)(kg / kSlots) & 1u);
      const int t0 = kg * 32, t1 = min(nsteps, t0 + 32);
      const int scur = kg % kSlots, sprev = (kg + kSlots - 1) % kSlots;
      struct In {
        double v;
        int idx;
        bool started, active, bal, anchor;
      };
      auto prep = [&](int t) -> In {
        In q;
        const int c = t - lane;
        q.started = c >= 0;
        q.active = lane_in & q.started & (c < C);
        const int cc = min(max(c, 0), C - 1);
        q.idx = ((cc >> 5) == kg ? scur : sprev) * kTile + lane * 32 + (cc & 31);
        const int code = W.code[0][q.idx];
        q.v = W.val[0][q.idx];
        q.anchor = code == kAnc;
        q.bal = code == 0;
        return q;
      };
      In cur = prep(t0);
#pragma unroll 2
      for (int t = t0; t < t1; t++) {
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
        const In nxt = prep(min(t + 1, t1 - 1));
        const double vhat = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0), cur.v);
        const double vh = cur.anchor ? anc : (cur.bal ? cur.v : vhat);
        if (cur.active) W.val[0][cur.idx] = vh;
        pn = nhl;
        if (cur.started) hl = vh;
        cur = nxt;
      }
      if (kg >= 1 && kg - 1 < nch) {
        fence_proxy_async();  // reconstructed values (generic writes) before the bulk store
        __syncwarp();
        bar_arrive_n(bar0 + (kg - 1) % kSlots, 64);
      }
    }
    if (ngroups == nch) {
      fence_proxy_async();
      __syncwarp();
      bar_arrive_n(bar0 + (nch - 1) % kSlots, 64);
    }
  }
}

// inverse_map (transform.py:188-202) + f32 cast (D20) of the reconstructed
// tiles, one CTA per partition, a thread per 4-column quad (as k_fwd): the
// FP64 exp2 work at full occupancy, coalesced 16-byte output stores.
__global__ void __launch_bounds__(256) k_inv(Geom g, const BlkP *__restrict__ blkp,
                                             const double *__restrict__ vh, float *__restrict__ out,
                                             WsStatus *st) {
  count_launch(st);
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) return;  // written by the reconstruct kernel
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc, nch = (C + 31) >> 5;
  float *op = out + (bb.r0 + pr0) * g.cols + bb.c0;
  const bool vec = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const double *vt = vh + tile_base(g, p, 0);
  unsigned *amb = &st->unresolved;
  // the next quad's values are loaded before this quad's exp2 work
  auto load_quad = [&](int i, double (&v)[4]) -> bool {
    const int kc = i >> 8, r = (i >> 3) & 31, c0 = kc * 32 + (i & 7) * 4;
    if (i >= nch * 256 || r >= R || c0 >= C) return false;
    const double2 *q = reinterpret_cast<const double2 *>(vt + kc * kTile + r * 32 + (c0 & 31));
    const double2 a0 = __ldg(q), a1 = __ldg(q + 1);
    v[0] = a0.x; v[1] = a0.y; v[2] = a1.x; v[3] = a1.y;
    return true;
  };
  double vn[4];
  bool hn = load_quad(threadIdx.x, vn);
  for (int i = threadIdx.x; i < nch * 256; i += 256) {
    const double v[4] = {vn[0], vn[1], vn[2], vn[3]};
    const bool h = hn;
    hn = load_quad(i + 256, vn);
    if (!h) continue;
    const int kc = i >> 8, r = (i >> 3) & 31, c0 = kc * 32 + (i & 7) * 4;
    (void)kc;
    float y[4];
#pragma unroll
    for (int u = 0; u < 4; u++) y[u] = c0 + u < C ? inv_f32(v[u], P, amb) : 0.0f;  // padding columns hold garbage
    float *dst = op + (int64_t)r * g.cols + c0;
    if (vec && c0 + 3 < C) {
      *reinterpret_cast<float4 *>(dst) = make_float4(y[0], y[1], y[2], y[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (c0 + u < C) dst[u] = y[u];
    }
  }
}

}  // namespace pmz

namespace pmz {

// One-row partitions: the W-only recurrence, a lane per partition (no
// shuffles), 32 partitions per warp.  Every 32-column chunk of the warp's
// partitions is staged through shared memory with coalesced loads (lane =
// column), run from there (lane = partition) and written back the same way;
// the reconstructed values replace the addends for k_inv.
template <int PK>
__global__ void __launch_bounds__(32) k_reconstruct_1d(Geom g, KParams k, const BlkP *__restrict__ blkp,
                                                        const uint16_t *__restrict__ codes, double *vtile,
                                                        const double *__restrict__ anchors, float *__restrict__ out,
                                                        WsStatus *st) {
  __shared__ double sv[1][32][33];
  __shared__ uint16_t sc[1][32][34];
  count_launch(st);
  const int lane = threadIdx.x & 31, w = 0;  // one warp per CTA: the CTAs spread over every SM
  const int64_t p0 = (int64_t)blockIdx.x * 32;  // the warp's first partition
  if (p0 >= g.nparts) return;
  const int64_t p = p0 + lane;
  const bool mine = p < g.nparts;
  int C = 0, nch_max = 0;
  bool live = false;
  double hl = 0.0;
  if (mine) {
    int64_t b;
    int pi;
    part_of(g, p, b, pi);
    const BlockBox bb = block_box(g, b);
    C = bb.bc;
    if (blkp[b].trivial) {
      float *o = out + (bb.r0 + pi * g.prow) * g.cols + bb.c0;
      for (int c = 0; c < C; c++) o[c] = 0.0f;
    } else {
      live = true;
      hl = anchors[p];
    }
  }
  if (__any_sync(0xffffffffu, live) && st->err_bits) return;
  int cmax = C;
  for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  nch_max = (cmax + 31) >> 5;
  const unsigned lm = __ballot_sync(0xffffffffu, live);
  for (int kc = 0; kc < nch_max; kc++) {
    // stage: partition i's chunk kc, lane = column
    for (int i = 0; i < 32; i++) {
      if (!((lm >> i) & 1u)) continue;
      const int64_t o = tile_base(g, p0 + i, kc) + lane;
      sv[w][i][lane] = vtile[o];
      sc[w][i][lane] = codes[o];
    }
    __syncwarp();
    if (live) {
      for (int j = 0; j < 32; j++) {
        const int c = kc * 32 + j;
        if (c >= C) break;
        if (c == 0) { sv[w][lane][0] = hl; continue; }  // the anchor (D1)
        const double a = sv[w][lane][j];
        const double vhat = __dadd_rn(predict_steady<PK>(k, hl, 0.0, 0.0, true), a);
        hl = sc[w][lane][j] == 0 ? a : vhat;
        sv[w][lane][j] = hl;
      }
    }
    __syncwarp();
    for (int i = 0; i < 32; i++) {
      if (!((lm >> i) & 1u)) continue;
      vtile[tile_base(g, p0 + i, kc) + lane] = sv[w][i][lane];
    }
    __syncwarp();
  }
}

}  // namespace pmz
