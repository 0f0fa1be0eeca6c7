// wsc.cuh -- warp-specialized compress_block + verify_and_repair
// (SPEC.md:443-451, 461-469).
//
// Each 32-row partition is owned by a warp PAIR:
//   producer warp (lane = column): for each 32-column chunk, loads the float
//     tile, forward-maps it (transform.py:170-185), classifies the sign/range
//     of every element and quantizes the TRUE-surface residuals
//      into slot k%3 of a 3-deep shared-memory ring; later it
//     flushes the chunk's final codes and balance values to global memory.
//     This is all independent, FP64-throughput work.
//   consumer warp (lane = row): the decoder simulation of verify_and_repair,
//     an anti-diagonal recurrence over the ring: predict from RECONSTRUCTED
//     neighbours (shuffles), dequantize, bound check in the log domain,
//     repair on violation.  Only this chain is sequential.
// Producer and consumer hand slots over with named barriers
// (full[s] / empty[s], 64 threads each), CUTLASS-style.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "blockc.cuh"

namespace pmz {

constexpr int kPPC = 2;      // partitions (warp pairs) per CTA
constexpr int kSlots = 3;    // ring depth
constexpr uint16_t kAnc = 0xFFFF;

struct PRing {
  double v[kSlots][32][32];       // forward-mapped TRUE values
  uint16_t code[kSlots][32][32];  // codes; the consumer zeroes repaired ones
  uint8_t cls[kSlots][32][32];    // 0: x == 0, 1: x > 0, 2: x < 0 (normal range), 3: exact path only
};
constexpr size_t kWscSmem = sizeof(PRing) * kPPC;

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ uint8_t xclass(float xz) {
  const float a = fabsf(xz);
  if (a == 0.0f) return 0;
  if (a < 1.7e38f && a > 4.7e-38f) return xz > 0.0f ? 1 : 2;
  return 3;
}

// D8 bound check with the sign/range class precomputed by the producer.
__device__ __forceinline__ int check_cls(double vhat, double v, int cls, const BlkP &P, const KParams &k) {
  if (cls == 1 || cls == 2) {
    const bool side_ok = cls == 1 ? (vhat <= P.boundary) : (vhat > P.boundary);
    // wrong sign or snapped to zero: relative error >= 1 > t (when t < 1)
    if ((!side_ok || vhat <= P.zero_threshold) && k.repair_t < 1.0) return 1;
    if (side_ok && vhat > P.zero_threshold) {
      const double d = __dsub_rn(vhat, v);
      const double mu = 0x1p-20;
      if (d < __dsub_rn(k.dpos, mu) && d > __dadd_rn(k.dneg, mu)) return 0;
      if (d > __dadd_rn(k.dpos, mu) || d < __dsub_rn(k.dneg, mu)) return 1;
    }
  } else if (cls == 0 && vhat <= P.zero_threshold) {
    return 0;
  }
  return -1;  // undecided: exact path
}

#ifdef PMZ_CMP_PROFILE
__device__ long long g_cmp_prof[65536][2][4];  // [partition][role][start, end, wait cycles, phase cycles]
__device__ long long g_cmp_ph[65536][4];
#endif

template <int PK>
__global__ void __launch_bounds__(kPPC * 64) k_compress_ws(const float *__restrict__ x, Geom g, KParams k,
                                                           const BlkP *__restrict__ blkp, WsStatus *st,
                                                           uint16_t *__restrict__ codes, double *__restrict__ balv,
                                                           double *__restrict__ anchors,
                                                           unsigned long long *__restrict__ part_zeros,
                                                           uint16_t *__restrict__ zrow,
                                                           const double *__restrict__ vbuf,
                                                           const int16_t *__restrict__ rqbuf,
                                                           const uint8_t *__restrict__ clsbuf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;  // role 0: producer, 1: consumer
  PRing &W = reinterpret_cast<PRing *>(smem_raw)[pair];
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
  const int m = st->m;
  const int center = 1 << (m - 1);
  const int bar0 = 1 + pair * 2 * kSlots;  // full[s] = bar0 + s, empty[s] = bar0 + kSlots + s
  const float *xp = x + (bb.r0 + pr0) * g.cols + bb.c0;
  const double *vp = vbuf + (bb.r0 + pr0) * g.cols + bb.c0;
  const int16_t *rqp = rqbuf + (bb.r0 + pr0) * g.cols + bb.c0;
  const uint8_t *clp = clsbuf + (bb.r0 + pr0) * g.cols + bb.c0;
  unsigned *amb = &st->unresolved;

#ifdef PMZ_CMP_PROFILE
  long long t_start = clock64(), t_wait = 0, t_fwd = 0, t_code = 0, t_flush = 0, t_mark;
#define TIMED_SYNC(id) { long long t0_ = clock64(); bar_sync_n(id, 64); t_wait += clock64() - t0_; }
#else
#define TIMED_SYNC(id) bar_sync_n(id, 64);
#endif
  if (role == 0) {
    // ------------------------------ producer ------------------------------
    uint16_t *cpart = codes + (bb.r0 + pr0) * g.cols + bb.c0;
    double *bpart = balv + (bb.r0 + pr0) * g.cols + bb.c0;
    // balance values are appended per row (row-compacted: row r's list starts
    // at column 0 of its block-row segment), counts per row in zrow
    unsigned rowcnt = 0;  // lane r's count for row r (lane = row here)
    auto flush = [&](int chunk) {
      const int s = chunk % kSlots, col = chunk * 32 + lane;
      for (int r = 0; r < R; r++) {
        const uint16_t cd = col < C ? W.code[s][r][lane] : (uint16_t)1;
        if (col < C) cpart[r * g.cols + col] = cd;
        const unsigned zm = __ballot_sync(0xffffffffu, cd == 0);
        const unsigned base = __shfl_sync(0xffffffffu, rowcnt, r);
        if (cd == 0) bpart[r * g.cols + base + __popc(zm & ((1u << lane) - 1))] = W.v[s][r][lane];
        if (lane == r) rowcnt += __popc(zm);
      }
    };
    for (int kc = 0; kc < nch; kc++) {
      const int s = kc % kSlots;
      if (kc >= kSlots) {
        TIMED_SYNC(bar0 + kSlots + s)  // consumer done with chunk kc-3
#ifdef PMZ_CMP_PROFILE
        t_mark = clock64();
#endif
        flush(kc - kSlots);
        __syncwarp();
#ifdef PMZ_CMP_PROFILE
        t_flush += clock64() - t_mark;
#endif
      }
#ifdef PMZ_CMP_PROFILE
      t_mark = clock64();
#endif
      const int col = kc * 32 + lane;
      const bool inb = col < C;
#if defined(PMZ_CMP_ISOLATE) && PMZ_CMP_ISOLATE == 2
      if (kc >= 0) { __syncwarp(); bar_arrive_n(bar0 + s, 64); continue; }
#endif
      // ring fill from the k_fwdq results (L2-resident): TRUE value, class,
      // and the code for this m
      for (int rb = 0; rb < R; rb += 8) {
        double vv[8];
        int rq[8];
        uint8_t cl[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const bool ok = inb && rb + q < R;
          const int64_t e = (int64_t)(rb + q) * g.cols + col;
          vv[q] = ok ? __ldg(vp + e) : 0.0;
          rq[q] = ok ? __ldg(rqp + e) : 0;
          cl[q] = ok ? __ldg(clp + e) : (uint8_t)0;
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if (rb + q < R) {
            W.v[s][rb + q][lane] = vv[q];
            W.cls[s][rb + q][lane] = cl[q];
            W.code[s][rb + q][lane] = (uint16_t)code_of_rq(rq[q], center);
          }
        }
      }
      if (kc == 0 && lane == 0) {
        W.code[s][0][0] = kAnc;
        anchors[p] = W.v[s][0][0];  // forced anchor, D1
      }
      __syncwarp();
#ifdef PMZ_CMP_PROFILE
      t_code += clock64() - t_mark;
#endif
      bar_arrive_n(bar0 + s, 64);  // full[s]
    }
    for (int kc = max(0, nch - kSlots); kc < nch; kc++) {
      TIMED_SYNC(bar0 + kSlots + kc % kSlots)
      flush(kc);
    }
    if (lane < R) zrow[p * 32 + lane] = (uint16_t)rowcnt;
#ifdef PMZ_CMP_PROFILE
    if (lane == 0 && p < 65536) { g_cmp_prof[p][0][0] = t_start; g_cmp_prof[p][0][1] = clock64(); g_cmp_prof[p][0][2] = t_wait;
      g_cmp_ph[p][0] = t_fwd; g_cmp_ph[p][1] = t_code; g_cmp_ph[p][2] = t_flush; }
#endif
  } else {
    // ------------------------------ consumer ------------------------------
    const int nsteps = C + R - 1;
    const int ngroups = (nsteps + 31) >> 5;
    double hl = 0.0, hp = 0.0;
    unsigned zeros = 0, repairs = 0;
    const double mu = 0x1p-20;
    const double dpos_m = __dsub_rn(k.dpos, mu), dneg_m = __dadd_rn(k.dneg, mu);
    const double dpos_p = __dadd_rn(k.dpos, mu), dneg_p = __dsub_rn(k.dneg, mu);
    const bool tlt1 = k.repair_t < 1.0;
    for (int kg = 0; kg < ngroups; kg++) {
      if (kg < nch) TIMED_SYNC(bar0 + kg % kSlots)  // full: chunk kg ready
      const int t1 = min(nsteps, (kg + 1) * 32);
#if defined(PMZ_CMP_ISOLATE) && PMZ_CMP_ISOLATE == 1
      for (int t = t1; t < t1; t++) {
#else
      for (int t = kg * 32; t < t1; t++) {
#endif
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1), nhp = __shfl_up_sync(0xffffffffu, hp, 1);
        const int c = t - lane;
        if (lane < R && c >= 0 && c < C) {
          const int s = (c >> 5) % kSlots, j = c & 31;
          const double v = W.v[s][lane][j];
          const int code = W.code[s][lane][j];
          const int cls = W.cls[s][lane][j];
          const double dq = __dmul_rn((double)(code - center), k.two_ba);  // off the chain
          const bool hw = c > 0, hn = lane > 0;
          const double vhat = __dadd_rn(predict_chain<PK>(k, hw ? hl : 0.0, hn ? nhl : 0.0, (hw && hn) ? nhp : 0.0), dq);
          // check_cls, predicated (D8 log-domain filter)
          const double d = __dsub_rn(vhat, v);
          const bool side_ok = cls == 1 ? (vhat <= P.boundary) : (vhat > P.boundary);
          const bool nz = vhat > P.zero_threshold;
          const bool in12 = side_ok && nz;
          const bool is12 = cls == 1 || cls == 2;
          bool acc = is12 ? (in12 && d < dpos_m && d > dneg_m) : (cls == 0 && !nz);
          bool vio = is12 && ((tlt1 && !in12) || (in12 && (d > dpos_p || d < dneg_p)));
          const bool normal = code != 0 && code != kAnc;
          if (__builtin_expect(normal && !acc && !vio, 0)) {
            const float xz = zfloor(__ldg(xp + lane * g.cols + c));
            vio = violates(inv_f32(vhat, P, amb), xz, k.repair_t);
          }
          const bool keep = normal && !vio;
          if (normal && !keep) {
            W.code[s][lane][j] = 0;
            repairs++;
          }
          zeros += (code == 0 || (normal && !keep)) ? 1u : 0u;
          hp = hl;
          hl = keep ? vhat : v;
        }
      }
      if (kg >= 1 && kg - 1 < nch) {
        __syncwarp();
        bar_arrive_n(bar0 + kSlots + (kg - 1) % kSlots, 64);  // empty: chunk kg-1 final
      }
    }
    if (ngroups == nch) {
      __syncwarp();
      bar_arrive_n(bar0 + kSlots + (nch - 1) % kSlots, 64);
    }
    for (int o = 16; o > 0; o >>= 1) {
      zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
      repairs += __shfl_xor_sync(0xffffffffu, repairs, o);
    }
#ifdef PMZ_CMP_PROFILE
    if (lane == 0 && p < 65536) { g_cmp_prof[p][1][0] = t_start; g_cmp_prof[p][1][1] = clock64(); g_cmp_prof[p][1][2] = t_wait; }
#endif
    if (lane == 0) {
      part_zeros[p] = zeros;
      atomicAdd(&st->nbal, (unsigned long long)zeros);
      atomicAdd(&st->nrepair, (unsigned long long)repairs);
      atomicAdd(&st->ncodes, (unsigned long long)(R * C - 1));
    }
  }
}

// Block statistics + transform parameters for every block (separate, fully
// parallel pass so the main kernel starts from resident parameters).
__global__ void __launch_bounds__(kBW * 32) k_stats(const float *__restrict__ x, Geom g, KParams k,
                                                    BlkP *__restrict__ blkp, WsStatus *st) {
  __shared__ BlkP sP;
  count_launch(st);
  const BlockBox bb = block_box(g, blockIdx.x);
  block_stats_params(x, g, k, bb, sP, st);
  if (threadIdx.x == 0) {
    blkp[blockIdx.x] = sP;
    if (sP.trivial) atomicAdd(&st->ntrivial, 1ull);
  }
}

}  // namespace pmz
