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
// k_reconstruct3: the same recurrence over the partition-tiled codes written
// by k_decode3 (dec3.cuh).  Warp pair per partition:
//   producer (lane = column): per 32-column chunk, loads the code tile, ranks
//     the chunk's balance points per row (row bases from the per-row zero
//     counts of the decoder, ballots within the chunk) and gathers their
//     values from the container into the ring; when the consumer has finished
//     a chunk it inverse-maps it and stores 32 f32 rows coalesced;
//   consumer (lane = row): vhat = code 0 ? balance value : predict(W, N, NW) +
//     dequantize(code) -- predicated, software-pipelined, one shuffle per step
//     (see k_compress_ws).
struct DRing3 {
  double val[kSlots][kTile];     // producer: balance value (code 0); consumer: reconstructed value
  uint16_t code[kSlots][kTile];
};
constexpr size_t kDsc3Smem = sizeof(DRing3) * kPPC;

template <int PK>
__global__ void __launch_bounds__(kPPC * 64) k_reconstruct3(const uint8_t *__restrict__ buf,
                                                            unsigned long long buf_n, Geom g, KParams k, int m,
                                                            const BlkP *__restrict__ blkp,
                                                            const uint16_t *__restrict__ codes,
                                                            const uint16_t *__restrict__ zrow,
                                                            const double *__restrict__ anchors,
                                                            const unsigned long long *__restrict__ part_zeros,
                                                            const unsigned long long *__restrict__ bal_off,
                                                            const unsigned long long *__restrict__ blk_nbal,
                                                            float *__restrict__ out, double *__restrict__ vh,
                                                            WsStatus *st) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;
  DRing3 &W = reinterpret_cast<DRing3 *>(smem_raw)[pair];
  const int64_t p = (int64_t)blockIdx.x * kPPC + pair;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const int nch = (C + 31) >> 5;
  float *opart = out + (bb.r0 + pr0) * g.cols + bb.c0;
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (role == 0)
      for (int r = 0; r < R; r++)
        for (int c = lane; c < C; c += 32) opart[(int64_t)r * g.cols + c] = 0.0f;
    return;
  }
  const int64_t p0 = first_part(g, b);
  unsigned long long zb = 0, ztot = 0;
  for (int i = 0; i < bb.np; i++) {
    const unsigned long long z = part_zeros[p0 + i];
    if (i < pi) zb += z;
    ztot += z;
  }
  if (ztot != blk_nbal[b]) {
    if (role == 0 && lane == 0 && pi == 0) set_err_at(st, ztot > blk_nbal[b] ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 30, b);
    return;
  }
  const int center = 1 << (m - 1);
  const int bar0 = 1 + pair * 2 * kSlots;
  const uint16_t *ct = codes + tile_base(g, p, 0);

  if (role == 0) {
    // ------------------------------ producer ------------------------------
    // balance values: 8-byte little-endian at a block-uniform byte alignment
    // sh -> value i = (word i >> sh) | (word i+1 << (64 - sh)) of the aligned
    // base; word i+1 may lie past the buffer only for the last values (byte
    // path, rare, after the batched loads)
    const uint8_t *bal = buf + bal_off[b], *bend = buf + buf_n;
    const uintptr_t ba = reinterpret_cast<uintptr_t>(bal);
    const unsigned sh = (unsigned)(ba & 7) * 8;
    const unsigned long long *qb = reinterpret_cast<const unsigned long long *>(ba & ~(uintptr_t)7);
    const long long nw = (long long)((reinterpret_cast<uintptr_t>(bend) - (ba & ~(uintptr_t)7)) >> 3);  // whole words
    // balance index of the next code-0 of every row (warp-uniform registers):
    // partition base + zeros of the rows above (the decoder's per-row counts)
    unsigned rb[32];
    {
      const unsigned zr = lane < R ? zrow[p * 32 + lane] : 0u;
      unsigned incl = zr;
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      const unsigned excl = (unsigned)zb + incl - zr;
#pragma unroll
      for (int r = 0; r < 32; r++) rb[r] = __shfl_sync(0xffffffffu, excl, r);
    }
    // a finished chunk: its reconstructed tile goes out with one bulk store
    // (the inverse map runs in k_inv at full occupancy)
    auto flush = [&](int chunk) {
      if (lane == 0) {
        bulk_s2g(vh + tile_base(g, p, chunk), W.val[chunk % kSlots], kTile * 8);
        bulk_commit();
      }
    };
    // codes of a chunk, two rows per register (row 2j low half), padding = 1
    auto load_codes = [&](int kc, unsigned (&c2)[16]) {
      const bool inb = kc * 32 + lane < C;
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const unsigned lo = (inb && 2 * j < R) ? __ldg(&ct[kc * kTile + (2 * j) * 32 + lane]) : 1u;
        const unsigned hi = (inb && 2 * j + 1 < R) ? __ldg(&ct[kc * kTile + (2 * j + 1) * 32 + lane]) : 1u;
        c2[j] = lo | (hi << 16);
      }
    };
    unsigned cn[16];
    load_codes(0, cn);
    for (int kc = 0; kc < nch; kc++) {
      const int s = kc % kSlots;
      unsigned cr2[16];
#pragma unroll
      for (int j = 0; j < 16; j++) cr2[j] = cn[j];
      if (kc + 1 < nch) load_codes(kc + 1, cn);  // next chunk's codes in flight during this gather
      if (kc == 0 && lane == 0) cr2[0] = (cr2[0] & 0xffff0000u) | kAnc;
      if (kc >= kSlots) {
        bar_sync_n(bar0 + kSlots + s, 64);
        flush(kc - kSlots);
        if (lane == 0) bulk_wait_read0();  // the store has read the slot
        __syncwarp();
      }
      // ballots and balance indices of all rows, then the loads in two
      // batches of 16 rows (predicated, no branches between them)
      unsigned zmask = 0;  // bit r: this lane's row r is a balance point
      long long bi[32];
#pragma unroll
      for (int r = 0; r < 32; r++) {
        const unsigned c = (cr2[r >> 1] >> ((r & 1) * 16)) & 0xffffu;
        const bool z = c == 0;
        const unsigned zm = __ballot_sync(0xffffffffu, z);
        bi[r] = (long long)rb[r] + __popc(zm & ((1u << lane) - 1));
        zmask |= (unsigned)z << r;
        rb[r] += __popc(zm);
        if (r < R) W.code[s][r * 32 + lane] = (uint16_t)c;
      }
#pragma unroll
      for (int h = 0; h < 2; h++) {
        unsigned long long lo[16], hi[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int r = h * 16 + j;
          const bool z = (zmask >> r) & 1u;
          lo[j] = z ? __ldg(qb + bi[r]) : 0ull;
          hi[j] = (z && sh) ? __ldg(qb + min(bi[r] + 1, nw - 1)) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int r = h * 16 + j;
          if ((zmask >> r) & 1u) {
            unsigned long long v = sh ? ((lo[j] >> sh) | (hi[j] << (64 - sh))) : lo[j];
            if (sh && bi[r] + 2 > nw) {  // last word partly outside the buffer
              v = 0;
              const uint8_t *pb = bal + 8ll * bi[r];
              for (int i = 7; i >= 0; i--) v = (v << 8) | __ldg(pb + i);
            }
            W.val[s][r * 32 + lane] = __longlong_as_double((long long)v);
          }
        }
      }
      __syncwarp();
      bar_arrive_n(bar0 + s, 64);  // full[s]
    }
    for (int kc = max(0, nch - kSlots); kc < nch; kc++) {
      bar_sync_n(bar0 + kSlots + kc % kSlots, 64);
      flush(kc);
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ------------------------------ consumer ------------------------------
    const double anc = anchors[p];
    const int nsteps = C + R - 1;
    const int ngroups = (nsteps + 31) >> 5;
    const double c_two_ba = pin(k.two_ba);
    const int c_center = pin(center);
    const bool lane0 = lane == 0, lane_in = lane < R;
    double hl = 0.0, pn = 0.0;
    for (int kg = 0; kg < ngroups; kg++) {
      if (kg < nch) bar_sync_n(bar0 + kg % kSlots, 64);
      const int t0 = kg * 32, t1 = min(nsteps, t0 + 32);
      const int scur = kg % kSlots, sprev = (kg + kSlots - 1) % kSlots;
      struct In {
        double v, dq;
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
        q.dq = __dmul_rn((double)(code - c_center), c_two_ba);
        return q;
      };
      In cur = prep(t0);
#pragma unroll 2
      for (int t = t0; t < t1; t++) {
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
        const In nxt = prep(min(t + 1, t1 - 1));
        const double vhat = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0), cur.dq);
        const double vh = cur.anchor ? anc : (cur.bal ? cur.v : vhat);
        if (cur.active) W.val[0][cur.idx] = vh;
        pn = nhl;
        if (cur.started) hl = vh;
        cur = nxt;
      }
      if (kg >= 1 && kg - 1 < nch) {
        fence_proxy_async();  // reconstructed values (generic writes) before the bulk store
        __syncwarp();
        bar_arrive_n(bar0 + kSlots + (kg - 1) % kSlots, 64);
      }
    }
    if (ngroups == nch) {
      fence_proxy_async();
      __syncwarp();
      bar_arrive_n(bar0 + kSlots + (nch - 1) % kSlots, 64);
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
