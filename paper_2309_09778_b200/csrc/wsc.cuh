// wsc.cuh -- compress_block's sequential half: verify_and_repair
// as one streaming pass per 32-row partition.
//
// k_fwdq already produced, per element and in the partition-tiled layout, the
// TRUE value v, its sign/range class and the m-independent quantized residual
// rq (code = center + rq when |rq| < center, else 0).  What remains is the
// decoder simulation, an anti-diagonal recurrence (lane = row): predict from
// RECONSTRUCTED W / N / NW (N, NW by shuffle from lane - 1), dequantize, bound
// check in the log domain, repair (rq := kRqOut, i.e. code 0 / balance point)
// on violation.  Each partition is owned by a warp PAIR:
//   producer warp: one elected lane streams the chunk tiles (v, rq, cls) into
//     a 3-deep shared-memory ring with cp.async.bulk on an mbarrier, and
//     bulk-stores each finished rq tile back in place (final codes);
//   consumer warp: the recurrence; it releases a slot with a named barrier.
// Steady-state steps (all 32 lanes inside the partition) run a guard-free
// variant of the step.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "blockc.cuh"

namespace pmz {

#ifndef PMZ_WS_SLOTS
#define PMZ_WS_SLOTS 3
#endif
constexpr int kPPC = 2;      // partitions (warp pairs) per CTA
constexpr int kSlots = PMZ_WS_SLOTS;    // ring depth

struct alignas(128) PRing {
  double v[kSlots][kTile];         // TRUE values
  int16_t rq[kSlots][kTile];       // quantized residuals; repaired -> kRqOut
  uint8_t cls[kSlots][kTile];      // 0: x == 0, 1: x > 0, 2: x < 0 (normal range), 3: exact path only
  unsigned long long full[kSlots]; // mbarriers: tile bytes landed
};
constexpr size_t kWscSmem = sizeof(PRing) * kPPC;
constexpr unsigned kTileBytes = kTile * (8 + 2 + 1);
#ifndef PMZ_WS_UNROLL
#define PMZ_WS_UNROLL 2
#endif
constexpr int kWsUnroll = PMZ_WS_UNROLL;

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- mbarrier / bulk-copy helpers (sm_90+ PTX) ----
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Keep a loop-invariant value in a register (no rematerialisation from the
// constant bank inside hot loops).
__device__ __forceinline__ double pin(double x) {
  asm volatile("" : "+d"(x));
  return x;
}
__device__ __forceinline__ int pin(int x) {
  asm volatile("" : "+r"(x));
  return x;
}

__device__ __forceinline__ uint8_t xclass(float xz) {
  const float a = fabsf(xz);
  if (a == 0.0f) return 0;
  if (a < 1.7e38f && a > 4.7e-38f) return xz > 0.0f ? 1 : 2;
  return 3;
}

// Prediction for a lane with all of W / N / NW inside the partition except
// that lane 0 has no N / NW (they read 0): predict_chain semantics.
template <int PK>
__device__ __forceinline__ double predict_steady(const KParams &k, double w, double n, double nw, bool lane0) {
  if (PK == 3) {
    double h = __dsub_rn(__dadd_rn(w, n), nw);
    h = lane0 ? w : h;  // (w + 0) - 0 up to the sign of a zero (see predict_chain)
    const double a = h < 0.0 ? __dmul_rn(k.slope, h) : h;
    if (__builtin_expect(fabs(a) < 0x1p-1020, 0)) {
      const double a2 = __dmul_rn(a, 0.5);
      return __dadd_rn(a2, a2);
    }
    return a;
  }
  if (PK == 1) return predict_chain<1>(k, w, 0.0, 0.0);
  return predict(k, w, lane0 ? 0.0 : n, lane0 ? 0.0 : nw);
}

#ifdef PMZ_CMP_PROFILE
__device__ long long g_cmp_prof[65536][2][4];  // [partition][role][start, end, wait, steady]
#endif

template <int PK>
__global__ void __launch_bounds__(kPPC * 64) k_compress_ws(const float *__restrict__ x, Geom g, KParams k,
                                                           const BlkP *__restrict__ blkp, WsStatus *st,
                                                           const double *__restrict__ vbuf, int16_t *rqbuf,
                                                           const uint8_t *__restrict__ clsbuf,
                                                           double *__restrict__ anchors,
                                                           unsigned long long *__restrict__ part_zeros,
                                                           const uint8_t *__restrict__ vflag,
                                                           unsigned long long *__restrict__ hist) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;  // role 0: producer, 1: consumer
  PRing &W = reinterpret_cast<PRing *>(smem_raw)[pair];
  if (role == 0 && lane == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&W.full[s], 1);
    mbar_init_fence();
  }
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * kPPC + pair;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (role == 1 && lane == 0) part_zeros[p] = 0;
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow;
  const int R = min(g.prow, bb.br - pr0);
  const int C = bb.bc;
  const int nch = (C + 31) >> 5;
  const int bar0 = 1 + pair * kSlots;  // empty[s] = bar0 + s (named barriers, 64 threads)
  const int64_t tb = tile_base(g, p, 0);
#ifdef PMZ_CMP_PROFILE
  const long long t_start = clock64();
#endif

  if (role == 0) {
    // ------------------------------ producer ------------------------------
    // validation blocks: the final codes of each finished tile go into the
    // summed code histogram (D10) before the tile is stored (warp-aggregated)
    const bool val = vflag[b] != 0;
    const int center = 1 << (st->m - 1);
    if (val && pi == 0 && lane == 0) atomicAdd(&hist[kMaxAlpha], 1ull);  // k for the floor (D10)
    auto store_rq = [&](int kc) {  // final rq tile of chunk kc back in place
      if (val) {
        const int c = kc * 32 + lane;
        for (int r = 0; r < R; r++) {
          const bool ok = c < C && (r | c);  // the anchor is not coded
          const int code = ok ? code_of_rq(W.rq[kc % kSlots][r * 32 + lane], center) : -1;
          const unsigned peers = __match_any_sync(0xffffffffu, code);
          if (ok && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&hist[code], (unsigned long long)__popc(peers));
        }
      }
      if (lane == 0) {
        bulk_s2g(rqbuf + tb + (int64_t)kc * kTile, W.rq[kc % kSlots], kTile * 2);
        bulk_commit();
      }
    };
    for (int kc = 0; kc < nch; kc++) {
      const int s = kc % kSlots;
      if (kc >= kSlots) {
        bar_sync_n(bar0 + s, 64);  // consumer done with chunk kc - 3
        store_rq(kc - kSlots);
        if (lane == 0) bulk_wait_read0();  // the store has read the slot
      }
      if (lane == 0) {
        const int64_t o = tb + (int64_t)kc * kTile;
        mbar_expect_tx(&W.full[s], kTileBytes);
        bulk_g2s(W.v[s], vbuf + o, kTile * 8, &W.full[s]);
        bulk_g2s(W.rq[s], rqbuf + o, kTile * 2, &W.full[s]);
        bulk_g2s(W.cls[s], clsbuf + o, kTile, &W.full[s]);
      }
      __syncwarp();
    }
    for (int kc = max(0, nch - kSlots); kc < nch; kc++) {
      bar_sync_n(bar0 + kc % kSlots, 64);
      store_rq(kc);
    }
    if (lane == 0) bulk_wait0();
#ifdef PMZ_CMP_PROFILE
    if (lane == 0 && p < 65536) { g_cmp_prof[p][0][0] = t_start; g_cmp_prof[p][0][1] = clock64(); }
#endif
  } else {
    // ------------------------------ consumer ------------------------------
    const float *xp = x + (bb.r0 + pr0) * g.cols + bb.c0;
    unsigned *amb = &st->unresolved;
    const int center = 1 << (st->m - 1);
    const int nsteps = C + R - 1;
    const int ngroups = (nsteps + 31) >> 5;
    const bool tlt1 = k.repair_t < 1.0;
    const double two_ba = k.two_ba, zthr = P.zero_threshold, bnd = P.boundary;
    const bool lane0 = lane == 0;
    double hl = 0.0, hp = 0.0;
    unsigned zeros = 0, repairs = 0;

    // Filtered bound check (check_cls, D8): class 1 lives in (zthr, bnd],
    // class 2 in (bnd, inf).  acc: certainly within the bound, vio: certainly
    // a violation; neither: exact path.
    auto classify = [&](double vhat, double v, int cls, bool &acc, bool &vio) {
      const double d = __dsub_rn(vhat, v);
      const bool gz = vhat > zthr, gb = vhat > bnd;
      const bool in12 = cls == 1 ? (gz && !gb) : gb;
      const bool is12 = cls == 1 || cls == 2;
      acc = is12 ? (in12 && d < k.dpos_m && d > k.dneg_m) : (cls == 0 && !gz);
      vio = is12 && ((tlt1 && !in12) || (in12 && (d > k.dpos_p || d < k.dneg_p)));
    };
    const float *xrow = xp + (int64_t)lane * g.cols;
    auto exact_vio = [&](double vhat, int c) -> bool {
      const float xz = zfloor(__ldg(xrow + c));
      return violates(inv_f32(vhat, P, amb), xz, k.repair_t);
    };
    // one element of the general (guarded) path; returns the reconstructed value
    auto verify = [&](double pred, double v, int rq, int cls, int16_t *rqp, int c, bool anchor) -> double {
      const bool normal = abs(rq) < center && !anchor;
      const double vhat = __dadd_rn(pred, __dmul_rn((double)rq, two_ba));
      bool acc, vio;
      classify(vhat, v, cls, acc, vio);
      if (normal && !acc && !vio) vio = exact_vio(vhat, c);
      const bool keep = normal && !vio;
      if (normal && vio) {
        *rqp = kRqOut;
        repairs++;
      }
      zeros += (!keep && !anchor) ? 1u : 0u;
      return keep ? vhat : v;
    };

#ifdef PMZ_CMP_PROFILE
    long long t_w = 0, t_st = 0, t_m;
#endif
    const double c_two_ba = pin(two_ba), c_zthr = pin(zthr), c_bnd = pin(bnd), c_slope = pin(k.slope);
    const double c_dpm = pin(k.dpos_m), c_dnm = pin(k.dneg_m), c_dpp = pin(k.dpos_p), c_dnp = pin(k.dneg_p);
    const int c_tlt1 = pin((int)tlt1), c_center = pin(center);
    const bool lane_in = lane < R;
    double pn = 0.0;  // lane - 1's value one column back (the NW input)
    for (int kg = 0; kg < ngroups; kg++) {
#ifdef PMZ_CMP_PROFILE
      t_m = clock64();
#endif
      if (kg < nch) mbar_wait(&W.full[kg % kSlots], (unsigned)(kg / kSlots) & 1u);
#ifdef PMZ_CMP_PROFILE
      t_w += clock64() - t_m;
      t_m = clock64();
#endif
      const int t0 = kg * 32, t1 = min(nsteps, t0 + 32);
      const int scur = kg % kSlots, sprev = (kg + kSlots - 1) % kSlots;
      // One predicated step for every lane: a lane that has not started
      // (c < 0) keeps hl = 0, which is exactly the W / NW = 0 boundary; a lane
      // past its row end computes values nobody reads.  Software-pipelined:
      // step t+1's inputs (ring loads, dq, class predicates) are prepared in
      // step t's basic block so they fill the latency gaps of t's chain.
      struct In {
        double v, dq, dqmv;
        int idx;
        bool started, active, anchor, normal, c1, c2, c0;
      };
      auto prep = [&](int t) -> In {
        In q;
        const int c = t - lane;
        q.started = c >= 0;
        q.active = lane_in & q.started & (c < C);
        const int cc = min(max(c, 0), C - 1);
        q.idx = ((cc >> 5) == kg ? scur : sprev) * kTile + lane * 32 + (cc & 31);
        q.v = W.v[0][q.idx];
        const int rq = W.rq[0][q.idx];
        const int cls = W.cls[0][q.idx];
        q.anchor = lane0 & (c == 0);
        q.normal = (abs(rq) < c_center) & !q.anchor;
        q.dq = __dmul_rn((double)rq, c_two_ba);
        q.dqmv = __dsub_rn(q.dq, q.v);  // d = a + (dq - v): off the chain (see below)
        q.c1 = cls == 1;
        q.c2 = cls == 2;
        q.c0 = cls == 0;
        return q;
      };
      In cur = prep(t0);
#pragma unroll kWsUnroll
      for (int t = t0; t < t1; t++) {
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
        const In nxt = prep(min(t + 1, t1 - 1));  // the last step re-reads its own inputs
        double a;
        if (PK == 3) {
          double h = __dsub_rn(__dadd_rn(hl, nhl), pn);
          h = lane0 ? hl : h;  // no N / NW in row 0 (sign of a zero only, see predict_chain)
          a = h < 0.0 ? __dmul_rn(c_slope, h) : h;
        } else {
          a = predict_steady<PK>(k, hl, nhl, pn, lane0);
        }
        double vhat = __dadd_rn(a, cur.dq);
        // classify (check_cls, D8), branch-free
        // log-domain filter on d = (a + dq) - v evaluated as a + (dq - v): the
        // two differ by a few ulp of |vhat| (< 2^-40 here), far inside the
        // filter's 2^-20 margin, so every decision is the one the exact d
        // gives, and d no longer waits for vhat
        const double d = __dadd_rn(a, cur.dqmv);
        const bool gz = vhat > c_zthr, gb = vhat > c_bnd;
        const bool in12 = (cur.c1 & gz & !gb) | (cur.c2 & gb);
        const bool inner = (d < c_dpm) & (d > c_dnm);
        const bool outer = (d > c_dpp) | (d < c_dnp);
        bool acc = (in12 & inner) | (cur.c0 & !gz);
        bool vio = (cur.c1 | cur.c2) & (((c_tlt1 != 0) & !in12) | (in12 & outer));
        const bool rare = cur.active & ((PK == 3 & (fabs(a) < 0x1p-1020)) | (cur.normal & !acc & !vio));
        if (__builtin_expect(rare, 0)) {  // per-lane branch, no warp vote on the dependency chain
          vhat = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0), cur.dq);
          const int cls = W.cls[0][cur.idx];
          classify(vhat, cur.v, cls, acc, vio);
          if (cur.normal && !acc && !vio) vio = exact_vio(vhat, t - lane);
        }
        const bool keep = cur.normal & !vio;
        if (cur.active & cur.normal & vio) {
          W.rq[0][cur.idx] = kRqOut;
          repairs++;
        }
        zeros += (cur.active & !keep & !cur.anchor) ? 1u : 0u;
        if (cur.active & cur.anchor) anchors[p] = cur.v;  // forced anchor, D1
        pn = nhl;
        if (cur.started) {
          hp = hl;
          hl = keep ? vhat : cur.v;
        }
        cur = nxt;
      }
#ifdef PMZ_CMP_PROFILE
      __syncwarp();
      t_st += clock64() - t_m;
#endif
      if (kg >= 1 && kg - 1 < nch) {
        fence_proxy_async();  // repairs (generic writes) before the async-proxy store
        __syncwarp();
        bar_arrive_n(bar0 + (kg - 1) % kSlots, 64);  // empty: chunk kg - 1 final
      }
    }
    if (ngroups == nch) {
      fence_proxy_async();
      __syncwarp();
      bar_arrive_n(bar0 + (nch - 1) % kSlots, 64);
    }
    for (int o = 16; o > 0; o >>= 1) {
      zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
      repairs += __shfl_xor_sync(0xffffffffu, repairs, o);
    }
#ifdef PMZ_CMP_PROFILE
    if (lane == 0 && p < 65536) { g_cmp_prof[p][1][0] = t_start; g_cmp_prof[p][1][1] = clock64();
      g_cmp_prof[p][1][2] = t_w; g_cmp_prof[p][1][3] = t_st; }
#endif
    if (lane == 0) {
      part_zeros[p] = zeros;
      atomicAdd(&st->nbal, (unsigned long long)zeros);
      atomicAdd(&st->nrepair, (unsigned long long)repairs);
      atomicAdd(&st->ncodes, (unsigned long long)(R * C - 1));
    }
  }
}

// verify_and_repair for one-row partitions (1-D inputs,
// block_rows == 1): a thread per partition runs its row's recurrence
// (W-only surface, row-0 semantics of the consumer above: same predict,
// same check_cls filter + exact f32 test, same repair), so 32 partitions
// advance per warp step instead of one active lane per warp pair.
template <int PK>
__global__ void __launch_bounds__(32) k_compress_1d(const float *__restrict__ x, Geom g, KParams k,
                                                    const BlkP *__restrict__ blkp, WsStatus *st,
                                                    const double *__restrict__ vbuf, int16_t *rqbuf,
                                                    const uint8_t *__restrict__ clsbuf,
                                                    double *__restrict__ anchors,
                                                    unsigned long long *__restrict__ part_zeros,
                                                    const uint8_t *__restrict__ vflag,
                                                    unsigned long long *__restrict__ hist) {
  count_launch(st);
  const int64_t p = (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  if (P.trivial) {
    part_zeros[p] = 0;
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, C = bb.bc;
  const int center = 1 << (st->m - 1);
  const bool val = vflag[b] != 0;
  const bool tlt1 = k.repair_t < 1.0;
  const double two_ba = k.two_ba, zthr = P.zero_threshold, bnd = P.boundary;
  const float *xrow = x + (bb.r0 + pr0) * g.cols + bb.c0;
  unsigned *amb = &st->unresolved;
  const int64_t tb = tile_base(g, p, 0);
  if (val && pi == 0) atomicAdd(&hist[kMaxAlpha], 1ull);  // k for the floor (D10)
  double hl = 0.0;
  unsigned zeros = 0, repairs = 0;
  // inputs kPf elements ahead in registers: the loads (one L1 miss per
  // sector) run under the recurrence's dependency chain
  constexpr int kPf = 8;
  auto at_c = [&](int c) -> int64_t { return tb + (int64_t)(c >> 5) * kTile + (c & 31); };  // row 0
  double pv[kPf];
  int prq[kPf], pcls[kPf];
#pragma unroll
  for (int u = 0; u < kPf; u++) {
    const int64_t i = at_c(min(u, C - 1));
    pv[u] = vbuf[i];
    prq[u] = rqbuf[i];
    pcls[u] = clsbuf[i];
  }
  for (int c0 = 0; c0 < C; c0 += kPf)
#pragma unroll
  for (int u = 0; u < kPf; u++) {
    const int c = c0 + u;
    if (c >= C) break;
    const int64_t i = at_c(c);
    const double v = pv[u];
    const int rq = prq[u];
    const int cls = pcls[u];
    {
      const int64_t j = at_c(min(c + kPf, C - 1));
      pv[u] = vbuf[j];
      prq[u] = rqbuf[j];
      pcls[u] = clsbuf[j];
    }
    const bool anchor = c == 0;
    const bool normal = abs(rq) < center && !anchor;
    const double vhat = __dadd_rn(predict_steady<PK>(k, hl, 0.0, 0.0, true), __dmul_rn((double)rq, two_ba));
    // check_cls (D8), as classify() in k_compress_ws
    const double d = __dsub_rn(vhat, v);
    const bool gz = vhat > zthr, gb = vhat > bnd;
    const bool in12 = cls == 1 ? (gz && !gb) : gb;
    const bool is12 = cls == 1 || cls == 2;
    const bool acc = is12 ? (in12 && d < k.dpos_m && d > k.dneg_m) : (cls == 0 && !gz);
    bool vio = is12 && ((tlt1 && !in12) || (in12 && (d > k.dpos_p || d < k.dneg_p)));
    if (normal && !acc && !vio) vio = violates(inv_f32(vhat, P, amb), zfloor(__ldg(xrow + c)), k.repair_t);
    const bool keep = normal && !vio;
    int fin = rq;
    if (normal && vio) {
      fin = kRqOut;
      rqbuf[i] = kRqOut;
      repairs++;
    }
    zeros += (!keep && !anchor) ? 1u : 0u;
    if (anchor) anchors[p] = v;  // forced anchor, D1
    if (val && !anchor) atomicAdd(&hist[code_of_rq(fin, center)], 1ull);
    hl = keep ? vhat : v;
  }
  part_zeros[p] = zeros;
  atomicAdd(&st->nbal, (unsigned long long)zeros);
  if (repairs) atomicAdd(&st->nrepair, (unsigned long long)repairs);
  atomicAdd(&st->ncodes, (unsigned long long)(C - 1));
}

// compute_block_stats + make_transform_params (transform.py:84-167) for
// every block, one CTA per block: the min positive normal magnitude, the max
// magnitude and the non-finite flag from one pass over the block (four rows
// of 16-byte loads in flight per warp), then the block's parameters (its
// three logarithms on three warps in parallel).  BlkStat is the layout of
// the workspace slots the earlier partition-parallel version accumulated in.
struct BlkStat {
  unsigned nmin;   // ~bits of the min |x| (0 = none)
  unsigned max;    // bits of the max |x|
  unsigned flags;  // bit 0: non-finite seen
  unsigned count;  // partitions done
};

constexpr int kST = 512;  // k_stats threads: one CTA per block
__global__ void __launch_bounds__(kST) k_stats(const float *__restrict__ x, Geom g, KParams k,
                                               BlkP *__restrict__ blkp, BlkStat *bst, WsStatus *st,
                                               pmz_np_fix *npfix) {
  __shared__ double s_l[3], s_fn;
  __shared__ unsigned s_mn[kST / 32], s_mx[kST / 32];
  count_launch(st);
  const int64_t b = blockIdx.x;
  const BlockBox bb = block_box(g, b);
  const int R = bb.br, C = bb.bc;
  const float *base = x + bb.r0 * g.cols + bb.c0;
  // on the magnitude bit patterns (ordered like the values): the minimum of
  // (a - 0x00800001) mod 2^32 is the smallest magnitude above the floor
  // (zero_sub_floor: |x| <= 2^-126 is zero, those wrap to the top), the
  // maximum of a is the largest magnitude, >= 0x7f800000 for Inf / NaN
  unsigned umn = 0xffffffffu, umx = 0u;
  auto acc = [&](unsigned bits) {
    const unsigned a = bits & 0x7fffffffu;
    umn = min(umn, a - 0x00800001u);
    umx = max(umx, a);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kST / 32;
  if ((g.cols & 3) == 0 && (C & 3) == 0 && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0)) {
    // warp w takes rows w, w + NW, ...; lanes the row's 16-byte vectors
    const int vpr = C >> 2;
    if (vpr == 64) {  // 256-column blocks: two vectors per lane per row, four rows per pass
      const uint4 *p0 = reinterpret_cast<const uint4 *>(base) + lane;
      const int64_t rs = g.cols >> 2;
      int r = warp;
      for (; r + 3 * NW < R; r += 4 * NW) {
        uint4 q[8];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          q[2 * i] = __ldg(p0 + (int64_t)(r + i * NW) * rs);
          q[2 * i + 1] = __ldg(p0 + (int64_t)(r + i * NW) * rs + 32);
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
          acc(q[i].x);
          acc(q[i].y);
          acc(q[i].z);
          acc(q[i].w);
        }
      }
      for (; r < R; r += NW) {
        const uint4 q0 = __ldg(p0 + (int64_t)r * rs), q1 = __ldg(p0 + (int64_t)r * rs + 32);
        acc(q0.x); acc(q0.y); acc(q0.z); acc(q0.w);
        acc(q1.x); acc(q1.y); acc(q1.z); acc(q1.w);
      }
    } else {
      for (int r = warp; r < R; r += NW) {
        const uint4 *rowp = reinterpret_cast<const uint4 *>(base + (int64_t)r * g.cols);
        for (int v = lane; v < vpr; v += 32) {
          const uint4 q0 = __ldg(rowp + v);
          acc(q0.x); acc(q0.y); acc(q0.z); acc(q0.w);
        }
      }
    }
  } else {
    for (int r = warp; r < R; r += NW)
      for (int c = lane; c < C; c += 32) acc(__float_as_uint(__ldg(base + (int64_t)r * g.cols + c)));
  }
  for (int o = 16; o; o >>= 1) {
    umn = min(umn, __shfl_xor_sync(0xffffffffu, umn, o));
    umx = max(umx, __shfl_xor_sync(0xffffffffu, umx, o));
  }
  if (lane == 0) {
    s_mn[warp] = umn;
    s_mx[warp] = umx;
  }
  __syncthreads();
  umn = s_mn[0];
  umx = s_mx[0];
#pragma unroll
  for (int i = 1; i < NW; i++) {
    umn = min(umn, s_mn[i]);
    umx = max(umx, s_mx[i]);
  }
  (void)bst;
  BlkP P{};
  if (umx >= 0x7f800000u) {  // NaN / Inf: the compress fails; nothing downstream touches the block
    P.trivial = 1;
    if (threadIdx.x == 0) {
      set_err(st, PMZ_ERR_NONFINITE);
      blkp[b] = P;
    }
    return;
  }
  if (umx <= 0x00800000u) {  // every magnitude at or below the floor
    P.trivial = 1;
    if (threadIdx.x == 0) {
      blkp[b] = P;
      atomicAdd(&st->ntrivial, 1ull);
    }
    return;
  }
  const float gmx = __uint_as_float(umx);
  const double fp = (double)__uint_as_float(umn + 0x00800001u), amax = (double)gmx;
  if (threadIdx.x == 0) {
    // transform.py:160-162
    s_fn = __ddiv_rn(__dmul_rn(__dmul_rn(__dadd_rn(amax, k.eps0), fp), k.onepbr2), __dsub_rn(fp, k.eps0));
    if (!isfinite(s_fn)) set_err(st, PMZ_ERR_NONREPRESENTABLE);
  }
  __syncthreads();
  const double fn = s_fn;
  // the three per-block logarithms in parallel (transform.py:119-123)
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < 3) {
    const double arg = w == 0 ? fp : (w == 1 ? fn : __dsub_rn(fp, k.eps0));
    s_l[w] = pmz_log2_d(arg, &st->unresolved);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    P.factor_pos = fp;
    P.factor_neg = fn;
    P.lg_pos = s_l[0];
    P.lg_neg = s_l[1];
    P.zero_code = __dadd_rn(-126.0, P.lg_pos);
    P.zero_threshold = __dadd_rn(P.zero_code, k.b_a);
    P.boundary = __dsub_rn(__dadd_rn(P.lg_neg, s_l[2]), k.b_a);
    blkp[b] = P;
    if (npfix) np_fix_note(st, npfix, b, fn, __dsub_rn(fp, k.eps0));
  }
}

// the host's np.log2 values for the listed blocks -> re-derived parameters
__global__ void k_np_apply(const pmz_np_fix *__restrict__ fix, long long n, double eps0, double b_a, BlkP *blkp,
                           WsStatus *st) {
  count_launch(st);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const pmz_np_fix e = fix[i];
  BlkP P = blkp[e.block];
  if (P.trivial) return;
  if (e.mask & 1) P.lg_neg = e.lg[0];
  const double lpe = (e.mask & 2) ? e.lg[1] : pmz_log2_d(__dsub_rn(P.factor_pos, eps0), &st->unresolved);
  P.boundary = __dsub_rn(__dadd_rn(P.lg_neg, lpe), b_a);  // transform.py:123
  blkp[e.block] = P;
}

}  // namespace pmz
