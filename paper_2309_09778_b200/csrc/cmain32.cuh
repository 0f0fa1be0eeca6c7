// cmain32.cuh -- the FP32 perceptron perf mode of the throughput compress
// (BASELINE.json north_star: "the three-layer perceptron is evaluated on FP32
// CUDA cores ... with any perceptron-rounding-induced code mismatch counted
// and reported").  Container version 2 (D12).
//
// Same sweep as k_c_main (cmain.cuh): warp per partition, lane = row,
// anti-diagonal steps, codes appended to per-row streams, balance values to
// per-row lists, k_c_write assembles the records.  What changes is the
// arithmetic of the surfaces, the predictor, the quantizer and the
// recurrence: all float32, D3 order, no contraction:
//   v      = RN32(log2|x|) + RN32(lg)     (MUFU lg2; zero -> RN32(zero_code))
//   pred   = a/2 + a/2, a = leaky((W + N) - NW)         (init model; general
//            weights: the D3 expression in float32)
//   code   = center + round_half_away((v - pred) * RN32(1/2b_a))
//   vhat   = pred(RECONSTRUCTED) + (code - center) * RN32(2 b_a)
// and the bound check of a reconstruction is the exact float32 test on
// inverse_map((double)vhat) (transform.py:188-202, D8), decided in the log
// domain when d = vhat - v is farther from the thresholds than the per-block
// error bound of the float32 v (mu below, ~2^-17.6 at C5).  A balance point
// stores (double)v, so the mirror decoder (k_d_recon32, dmain32.cuh) restarts
// its float32 recurrence from exactly the encoder's value.  Codes and the
// balance list differ from the FP64 reference where float32 rounding moves a
// residual across a quantization boundary or a reconstruction across the
// bound; tools/bench count them (CMainOut::dump, pmz_params::d_code_dump).
#pragma once
#include "cmain.cuh"

namespace pmz {

template <int PK>
__device__ __forceinline__ float c_pred32(const KParams &k, float w, float n, float nw, bool lane0) {
  if (PK == 3) {
    float h = __fsub_rn(__fadd_rn(w, n), nw);
    h = lane0 ? w : h;
    const float a = h < 0.0f ? __fmul_rn((float)k.slope, h) : h;
    const float a2 = __fmul_rn(a, 0.5f);
    return __fadd_rn(a2, a2);
  }
  const float s1 = lane0 ? 0.0f : n, s2 = lane0 ? 0.0f : nw;
  float a[2];
#pragma unroll
  for (int j = 0; j < 2; j++) {
    const float h = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(w, (float)k.w1[j]), __fmul_rn(s1, (float)k.w1[2 + j])),
                                        __fmul_rn(s2, (float)k.w1[4 + j])),
                              (float)k.w1[6 + j]);
    a[j] = h < 0.0f ? __fmul_rn((float)k.slope, h) : h;
  }
  return __fadd_rn(__fmul_rn(a[0], (float)k.w2[0]), __fmul_rn(a[1], (float)k.w2[1]));
}

// round half away from zero of a float32 quotient, as a float (exact integers)
__device__ __forceinline__ float rhaz32(float q) { return copysignf(floorf(__fadd_rn(fabsf(q), 0.5f)), q); }

template <int PK, int MODE, bool STAB>
__global__ void __launch_bounds__(kCW * 32, 2)
    k_c_main32(const float *__restrict__ x, Geom g, const __grid_constant__ KParams k, const BlkP *__restrict__ blkp,
               WsStatus *st, const int64_t *__restrict__ val_ids, int64_t nval, CMainOut o, int chain) {
  extern __shared__ __align__(16) unsigned char smem_c[];
  __shared__ unsigned s_cov[18];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *ring = reinterpret_cast<float *>(smem_c) + warp * 32 * kCRing;
  CL2Ent *s_l2 = reinterpret_cast<CL2Ent *>(smem_c + (size_t)kCW * 32 * kCRing * 4);
  double *s_band = reinterpret_cast<double *>(s_l2 + 256);
  uint2 *s_tab = reinterpret_cast<uint2 *>(s_band + PMZ_NP_LOG2_BAND_N);
  unsigned *s_hist = reinterpret_cast<unsigned *>(s_tab);
  const int m = MODE == kCCov ? 16 : st->m;
  if (MODE == kCMain && STAB != (m <= 12)) return;
  count_launch(st);
  const int nalpha = 1 << m;
  const bool hist_smem = MODE == kCHist && m <= 13;
  if (MODE == kCMain && STAB) {
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) s_tab[i] = make_uint2(o.cw[i], o.lens[i]);
    if (threadIdx.x == 0) s_tab[nalpha] = make_uint2(0u, 0u);
  }
  if (hist_smem)
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) s_hist[i] = 0;
  if (MODE == kCCov && threadIdx.x < 18) s_cov[threadIdx.x] = 0;
  __syncthreads();

  // kCMain: a chain of consecutive partitions per warp, one wavefront (see k_c_main)
  int64_t p, b;
  int pi, cnt = 1;
  bool have;
  if (MODE == kCMain) have = c_chain(g, chain, (int64_t)blockIdx.x * kCW + warp, p, b, pi, cnt);
  else have = c_part(g, MODE, val_ids, nval, p, b, pi);
  const BlkP *Pp = blkp + (have ? b : 0);
  const BlkP P = have ? *Pp : BlkP{};
  if (have && !P.trivial) {
    const BlockBox bb = block_box(g, b);
    const int C = bb.bc, Cp = (C + 7) & ~7;
    const int rows_left = bb.br - pi * g.prow;
    const int nsteps = cnt * Cp + 31;
    const bool vx = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    const float *l_xp = x + (bb.r0 + pi * g.prow) * g.cols + bb.c0;
    int l_c0 = 0, l_q = 0;
    auto load_chunk = [&](int kc) {
      if (l_q < cnt) {
        const int R = min(g.prow, rows_left - l_q * g.prow);
        const int slot = (kc * 8) & (kCRing - 1);
        if (vx && l_c0 + 8 <= C) {
#pragma unroll
          for (int j = 0; j < 2; j++) {
            const int r = j * 16 + (lane >> 1), h = (lane & 1) * 4;
            if (r < R) cp_async16(ring + r * kCRing + slot + h, l_xp + (int64_t)r * g.cols + l_c0 + h);
          }
        } else {
#pragma unroll 1
          for (int j = 0; j < 8; j++) {
            const int r = j * 4 + (lane >> 3), cc = l_c0 + (lane & 7);
            if (r < R && cc < C) cp_async4(ring + r * kCRing + slot + (lane & 7), l_xp + (int64_t)r * g.cols + cc);
          }
        }
        l_c0 += 8;
        if (l_c0 >= Cp) {
          l_c0 = 0;
          l_q++;
          l_xp += (int64_t)g.prow * g.cols;
        }
      }
      cp_async_commit();
    };
    const int center = 1 << (m - 1);
    const float two_ba = (float)k.two_ba, inv = (float)k.inv_two_ba;
    const bool tlt1 = k.repair_t < 1.0;
    const float lgp = (float)P.lg_pos, lgn = (float)P.lg_neg, zc = (float)P.zero_code;
    // float32 images of the double thresholds, rounded outwards, so every
    // float32 comparison below is a certain statement about the double one
    const float zthrU = __double2float_ru(P.zero_threshold), zthrD = __double2float_rd(P.zero_threshold);
    const float bndU = __double2float_ru(P.boundary), bndD = __double2float_rd(P.boundary);
    // |v - (log2|x| + lg)| <= 2^-21 (MUFU lg2) + 2^-24 (|log2 x| + |lg| + |v|) with
    // |log2 x| <= max(|lg_pos|, |lg_neg|) + 1 (amin = factor_pos <= |x| <= amax <= factor_neg):
    // the log-domain filter keeps that, plus the float32 rounding of xhat, away from the bound
    const float lmax = fmaxf(fabsf(lgp), fabsf(lgn)) + 1.0f;
    const float mu = 0x1p-21f + 0x1p-24f * (4.0f * lmax + 4.0f) + 0x1p-22f;
    const float dpm = (float)k.dpos - mu, dnm = (float)k.dneg + mu, dpp = (float)k.dpos + mu, dnp = (float)k.dneg - mu;
    unsigned *amb = &st->unresolved;
    const bool lane0 = lane == 0;
    // > 0: the lane has a row in its current partition (lanes >= partition_rows never do)
    int rleft = lane < g.prow ? min(rows_left, cnt * g.prow) - lane : -(1 << 28);
    int cb = -lane;  // column in the lane's current partition = t + cb
    float vW = 0.0f, pnt = 0.0f, hl = 0.0f, pn = 0.0f;
    unsigned long long acc = 0;
    int na = 0;
    unsigned nb = 0, repairs = 0, tz = 0;
    int64_t row = p * g.prow + lane;
    unsigned *wp = MODE == kCMain ? o.rowbits + row * (int64_t)g.bc : nullptr;
    double *brow = MODE == kCMain ? o.balrow + row * (int64_t)g.bc : nullptr;
    uint16_t *dump = (MODE == kCMain && o.dump) ? o.dump + tcode_base(g, p) + (int64_t)lane * C : nullptr;
    const unsigned ring_s = smem_u32(ring + lane * kCRing), tab_s = smem_u32(s_tab);
    load_chunk(0);
    load_chunk(1);
    load_chunk(2);
    for (int t0 = 0; t0 < nsteps; t0 += 8) {
      __syncwarp();
      load_chunk((t0 >> 3) + 3);
      cp_async_wait<3>();
      __syncwarp();
      const int t1 = min(nsteps, t0 + 8);
      // one sweep step; SW: some lane ends its row within these 8 steps (the
      // row-end branch is compiled only into that copy of the body)
      auto step = [&](const int t, auto swc) {
        constexpr bool SW = decltype(swc)::value;
        const int gc = t - lane;  // column of the chain's sweep: the ring slot
        const int c = t + cb;     // column in the lane's current partition
        const bool started = gc >= 0;
        const bool lane_in = rleft > 0;
        // first column of a row (SW copy only: rows start right after a row end): W and NW are
        // 0, partition-local neighbours (D2); the registers still hold the previous row's tail
        const bool first = SW && c == 0;
        const bool active = lane_in & ((unsigned)c < (unsigned)C);
        const bool anchor = lane0 & (c == 0);
        const unsigned u0 = lds_u32(ring_s + ((unsigned)(gc & (kCRing - 1)) << 2));
        const unsigned u = (u0 & 0x7fffffffu) <= 0x00800000u ? 0u : (u0 & 0x7fffffffu);
        const bool neg = (int)u0 < 0;
        const float xz = __uint_as_float(u | (neg ? 0x80000000u : 0u));
        // forward map in float32
        float v = __fadd_rn(__log2f(__uint_as_float(u | (u == 0 ? 0x3f800000u : 0u))), neg ? lgn : lgp);
        v = u == 0 ? zc : v;
        // TRUE-surface residual and quantization in float32
        const float nvt = __shfl_up_sync(0xffffffffu, vW, 1);
        const float at = c_pred32<PK>(k, first ? 0.0f : vW, nvt, first ? 0.0f : pnt, lane0);
        pnt = nvt;
        vW = started ? v : vW;
        const float qr = rhaz32(__fmul_rn(__fsub_rn(v, at), inv));
        const bool big = !(fabsf(qr) < 32768.0f);
        const int rq = big ? (int)kRqOut : (int)qr;
        if (MODE == kCCov) {
          const bool cnt1 = active & !anchor;
          const int mm = cnt1 ? m_of_rq(rq) : -1;
          const unsigned grp = __match_any_sync(0xffffffffu, mm);
          if (cnt1 && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&s_cov[mm], (unsigned)__popc(grp));
        } else {
          const bool out = big | (abs(rq) >= center);
          // decoder simulation (float32, the mirror of k_d_recon32)
          const float nhl = __shfl_up_sync(0xffffffffu, hl, 1);
          const float ar = c_pred32<PK>(k, first ? 0.0f : hl, nhl, first ? 0.0f : pn, lane0);
          const float vhat = __fadd_rn(ar, __fmul_rn(out ? 0.0f : qr, two_ba));
          const float d = __fsub_rn(vhat, v);
          const bool normal = (u - (kClsLo + 1u)) < (kClsHi - kClsLo - 1u);
          // certainly on the right side of zero_threshold / boundary (D8 classes), certainly flipped
          const bool in12 = normal & (neg ? (vhat > bndU) : ((vhat > zthrU) & (vhat <= bndD)));
          const bool flip = normal & (neg ? (vhat <= bndD) : ((vhat <= zthrD) | (vhat > bndU)));
          const bool inner = (d < dpm) & (d > dnm), outer = (d > dpp) | (d < dnp);
          const bool accept = !anchor & !out & ((in12 & inner) | ((u == 0) & (vhat <= zthrD)));
          const bool vcert = !anchor & (out | (in12 & outer) | (flip & tlt1));
          bool keep = accept;
          if (__builtin_expect(__any_sync(0xffffffffu, active & !accept & !vcert), 0)) {
            if (active & !accept & !vcert) {  // anchor, thresholds, extremes: the exact float32 test (D8)
              if (!anchor && !out) keep = !violates(inv_f32((double)vhat, P, amb), xz, k.repair_t);
            }
          }
          const int fin = keep ? center + rq : 0;
          repairs += (active & !keep & !anchor & !out) ? 1u : 0u;
          pn = nhl;
          hl = started ? (keep ? vhat : v) : hl;
          if (MODE == kCHist) {
            const bool cnt1 = active & !anchor;
            const int key = cnt1 ? fin : -1;
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            if (cnt1 && (grp & ((1u << lane) - 1)) == 0) {
              if (hist_smem) atomicAdd(&s_hist[fin], (unsigned)__popc(grp));
              else atomicAdd(&o.hist[fin], (unsigned long long)__popc(grp));
            }
          } else {
            const bool enc = active & !anchor;
            if (enc & (fin == 0)) {
              brow[nb] = (double)v;  // the row's balance list (D9): the encoder's float32 value, exactly
              nb++;
            }
            if (__builtin_expect(anchor, 0)) {  // forced anchor, D1 (lane 0, once per partition)
              if (active) o.anchors[p + (-cb) / Cp] = (double)v;
            }
            if (dump != nullptr && active) dump[c] = anchor ? kAnc : (uint16_t)fin;
            if (STAB) {
              const uint2 e = lds_v2(tab_s + ((unsigned)(enc ? fin : nalpha) << 3));
              acc |= (unsigned long long)e.x << ((64 - na - (int)e.y) & 63);
              na += (int)e.y;
            } else if (enc) {
              const unsigned cwv = __ldg(o.cw + fin);
              const int len = __ldg(o.lens + fin);
              acc |= (unsigned long long)cwv << (64 - na - len);
              na += len;
            }
            if (na >= 32) {
              *wp++ = (unsigned)(acc >> 32);
              acc <<= 32;
              na -= 32;
            }
          }
        }
        // end of the lane's row: close it, move to the same row of the chain's next partition
        if (SW && c == Cp - 1) {
          if (MODE == kCMain) {
            if (lane_in) {
              const unsigned bits = 32u * (unsigned)(wp - (o.rowbits + row * (int64_t)g.bc)) + (unsigned)na;
              if (na) *wp = (unsigned)(acc >> 32);
              o.rowinfo[row] = make_uint2(bits, nb);  // (partition totals: k_c_part_totals)
              tz += nb;
            }
            row += g.prow;
            wp = o.rowbits + row * (int64_t)g.bc;
            brow = o.balrow + row * (int64_t)g.bc;
            if (dump != nullptr) dump += (int64_t)g.prow * g.bc;  // tcode_base of the next partition
          }
          cb -= Cp;
          rleft -= g.prow;
          acc = 0;
          na = 0;
          nb = 0;
        }
      };
      const int cs = t0 + cb;  // a row ends within these 8 steps, or starts at the first of them
      if (__any_sync(0xffffffffu, ((unsigned)(Cp - 1 - cs) < 8u) | (cs == 0))) {
#pragma unroll 1
        for (int t = t0; t < t1; t++) step(t, std::true_type{});
      } else {
#pragma unroll kUnrC32
        for (int t = t0; t < t1; t++) step(t, std::false_type{});
      }
    }
    cp_async_wait<0>();
    if (MODE == kCMain) {
      unsigned tr = repairs;
      for (int s = 16; s; s >>= 1) {
        tz += __shfl_xor_sync(0xffffffffu, tz, s);
        tr += __shfl_xor_sync(0xffffffffu, tr, s);
      }
      if (lane == 0) {
        atomicAdd(&st->nbal, (unsigned long long)tz);
        if (tr) atomicAdd(&st->nrepair, (unsigned long long)tr);
        atomicAdd(&st->ncodes, (unsigned long long)((int64_t)min(cnt * g.prow, rows_left) * C - cnt));
      }
    } else if (MODE == kCHist) {
      if (pi == 0 && lane == 0) atomicAdd(&o.hist[kMaxAlpha], 1ull);
    }
  }
  if (MODE == kCCov) {
    __syncthreads();
    if (threadIdx.x < 18 && s_cov[threadIdx.x]) atomicAdd(&o.cov[threadIdx.x], (unsigned long long)s_cov[threadIdx.x]);
  }
  if (hist_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&o.hist[i], (unsigned long long)s_hist[i]);
  }
}

}  // namespace pmz
