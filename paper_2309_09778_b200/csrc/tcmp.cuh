// tcmp.cuh -- throughput-path compression (fields with many partitions):
// forward_map (transform.py:170-185), compress_block and
// verify_and_repair fused into one anti-diagonal sweep per
// partition, then encode + write_container.
//
// k_t_main<PK, MODE>: a WARP per 32-row partition, lane = row.  The input
//   arrives in 32 x 32 float tiles by cp.async one column chunk ahead; at
//   step t lane r takes column c = t - r: forward map (numpy-exact log2), the
//   TRUE-surface residual (W from its own previous step, N / NW by shuffle
//   from lane r - 1), quantization, and the decoder simulation on the
//   RECONSTRUCTED surface (one more shuffle) with the log-domain bound filter
//   and the exact float32 test when the filter cannot decide.  Nothing per
//   element goes to HBM but the final 2-byte code (raster layout, tcode_base)
//   and, for code-0 points, the TRUE value appended to the row's balance list.
//   MODE kTCoverage: the select_m coverage of the validation blocks' TRUE
//   residuals only; kTValCodes: the final-code histogram of the validation
//   blocks (estimate_codebook); kTMain: every partition, codes + lists + bits.
// k_t_write: a WARP per partition, lane = row: partition table entry, the
//   row's balance values, and the row's canonical codewords MSB-first at the
//   row's bit offset; bytes shared by two rows are combined by shuffle.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "wsc.cuh"
#include "tdec.cuh"

namespace pmz {

constexpr int kTCW = 4;  // partitions (warps) per CTA
struct TCmpWarp {
  float x[3][32 * 32];        // input tiles, chunk q in slot q % 3
  uint16_t code[2][32 * 32];  // final code tiles, chunk q in slot q & 1
};
constexpr size_t kTCmpSmem = sizeof(TCmpWarp) * kTCW;
enum { kTMain = 0, kTValCodes = 1, kTCoverage = 2 };
constexpr int kTLensSmem = 1 << 12;  // code lengths in shared memory up to this alphabet

// partition of (CTA, warp): every partition, or the partitions of the listed
// validation blocks (cpb CTAs per block)
__device__ __forceinline__ bool t_part(const Geom &g, int mode, const int64_t *val_ids, int64_t nval, int64_t &p,
                                       int64_t &b, int &pi) {
  const int warp = threadIdx.x >> 5;
  if (mode == kTMain) {
    p = (int64_t)blockIdx.x * kTCW + warp;
    if (p >= g.nparts) return false;
    part_of(g, p, b, pi);
    return true;
  }
  const int cpb = (g.np_full + kTCW - 1) / kTCW;
  const int64_t vb = blockIdx.x / cpb;
  if (vb >= nval) return false;
  b = val_ids[vb];
  if (b < 0 || b >= g.nblocks) return false;
  pi = (int)(blockIdx.x % cpb) * kTCW + warp;
  if (pi >= block_box(g, b).np) return false;
  p = first_part(g, b) + pi;
  return true;
}

template <int PK, int MODE>
__global__ void __launch_bounds__(kTCW * 32, 3) k_t_main(const float *__restrict__ x, Geom g, KParams k,
                                                         const BlkP *__restrict__ blkp, WsStatus *st,
                                                         const int64_t *__restrict__ val_ids, int64_t nval,
                                                         uint16_t *__restrict__ codes, double *__restrict__ balrow,
                                                         unsigned *__restrict__ rowinfo,
                                                         double *__restrict__ anchors,
                                                         unsigned long long *__restrict__ part_bits,
                                                         unsigned long long *__restrict__ part_zeros,
                                                         const uint8_t *__restrict__ lens,
                                                         unsigned long long *__restrict__ hist,
                                                         unsigned long long *__restrict__ cov) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint8_t s_lens[kTLensSmem];
  __shared__ unsigned s_cov[18];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TCmpWarp &S = reinterpret_cast<TCmpWarp *>(smem_raw)[warp];
  const int m = MODE == kTCoverage ? 16 : st->m;
  const int nalpha = 1 << m;
  const bool lens_smem = MODE == kTMain && nalpha <= kTLensSmem;
  if (lens_smem)
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) s_lens[i] = lens[i];
  if (MODE == kTCoverage && threadIdx.x < 18) s_cov[threadIdx.x] = 0;
  __syncthreads();
  int64_t p, b;
  int pi;
  const bool have = t_part(g, MODE, val_ids, nval, p, b, pi);
  const BlkP P = have ? blkp[b] : BlkP{};
  if (have && !P.trivial) {
    const BlockBox bb = block_box(g, b);
    const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
    const int nch = (C + 31) >> 5, nsteps = C + R - 1, ngroups = (nsteps + 31) >> 5;
    const float *xp = x + (bb.r0 + pr0) * g.cols + bb.c0;
    const bool vx = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    auto load_x = [&](int q) {
      float *dst = S.x[q % 3];
      const int c0 = q * 32, w = min(32, C - c0);
      if (vx && w == 32) {
#pragma unroll
        for (int j = 0; j < 8; j++) {  // 32 rows x 8 x 16 B, 4 rows per instruction
          const int r = j * 4 + (lane >> 3), pc = lane & 7;
          if (r < R) cp_async16(dst + r * 32 + pc * 4, xp + (int64_t)r * g.cols + c0 + pc * 4);
        }
      } else {
        for (int r = 0; r < R; r++)
          if (lane < w) dst[r * 32 + lane] = __ldg(xp + (int64_t)r * g.cols + c0 + lane);
      }
      cp_async_commit();
    };
    const int center = 1 << (m - 1);
    const bool tlt1 = k.repair_t < 1.0;
    const double two_ba = k.two_ba, zthr = P.zero_threshold, bnd = P.boundary;
    const double lgp = P.lg_pos, lgn = P.lg_neg, zcode = P.zero_code;
    unsigned *amb = &st->unresolved;
    const bool lane0 = lane == 0, lane_in = lane < R;
    double vprev = 0.0, pnt = 0.0;  // TRUE: own previous value (W), lane - 1's value one column back (NW)
    double hl = 0.0, pn = 0.0;      // RECONSTRUCTED: same
    unsigned bits = 0, nb = 0, repairs = 0;
    double *brow = balrow + (p * g.prow + lane) * (int64_t)g.bc;
    uint16_t *cb = codes + tcode_base(g, p);
    const bool vcode = (C & 7) == 0;
    load_x(0);
    for (int kg = 0; kg < ngroups; kg++) {
      if (kg + 1 < nch) {
        load_x(kg + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const int t0 = kg * 32, t1 = min(nsteps, t0 + 32);
      const float *xcur = S.x[kg % 3], *xprv = S.x[(kg + 2) % 3];
#pragma unroll 2
      for (int t = t0; t < t1; t++) {
        const int c = t - lane;
        const bool started = c >= 0;
        const bool active = lane_in & started & (c < C);
        const int cc = min(max(c, 0), C - 1);
        const int sidx = lane * 32 + (cc & 31);
        const float xz = zfloor(((cc >> 5) == kg ? xcur : xprv)[sidx]);
        // forward_map (transform.py:170-185): numpy-exact log2 of |x|
        const double lg = pmz_log2_f32_fast(xz != 0.0f ? (double)fabsf(xz) : 1.0, amb);
        const double v = xz > 0.0f ? __dadd_rn(lg, lgp) : (xz < 0.0f ? __dadd_rn(lg, lgn) : zcode);
        // TRUE-surface residual: W own, N / NW from lane - 1
        const double nvt = __shfl_up_sync(0xffffffffu, vprev, 1);
        const double predt = predict_steady<PK>(k, vprev, nvt, pnt, lane0);
        const int rq = quantize_rq(__dsub_rn(v, predt), k);
        pnt = nvt;
        if (started) vprev = v;
        const bool anchor = lane0 & (c == 0);
        if (MODE == kTCoverage) {
          const bool cnt = active & !anchor;
          const int mm = cnt ? m_of_rq(rq) : -1;
          const unsigned grp = __match_any_sync(0xffffffffu, mm);
          if (cnt && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&s_cov[mm], (unsigned)__popc(grp));
          continue;
        }
        // decoder simulation on the RECONSTRUCTED surface (verify_and_repair)
        const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
        const bool normal = (abs(rq) < center) & !anchor;
        const double dq = __dmul_rn((double)rq, two_ba);
        double a;
        if (PK == 3) {
          double h = __dsub_rn(__dadd_rn(hl, nhl), pn);
          h = lane0 ? hl : h;
          a = h < 0.0 ? __dmul_rn(k.slope, h) : h;
        } else {
          a = predict_steady<PK>(k, hl, nhl, pn, lane0);
        }
        double vhat = __dadd_rn(a, dq);
        const double d = __dadd_rn(a, __dsub_rn(dq, v));  // = vhat - v up to < 2^-40 (see k_compress_ws)
        const int cls = xclass(xz);
        const bool c1 = cls == 1, c2 = cls == 2;
        const bool gz = vhat > zthr, gb = vhat > bnd;
        const bool in12 = (c1 & gz & !gb) | (c2 & gb);
        const bool inner = (d < k.dpos_m) & (d > k.dneg_m);
        const bool outer = (d > k.dpos_p) | (d < k.dneg_p);
        bool acc = (in12 & inner) | ((cls == 0) & !gz);
        bool vio = (c1 | c2) & ((tlt1 & !in12) | (in12 & outer));
        if (__builtin_expect(active & ((PK == 3 & (fabs(a) < 0x1p-1020)) | (normal & !acc & !vio)), 0)) {
          vhat = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0), dq);
          const double d2 = __dsub_rn(vhat, v);
          const bool gz2 = vhat > zthr, gb2 = vhat > bnd;
          const bool in2 = c1 ? (gz2 && !gb2) : gb2;
          const bool is12 = c1 || c2;
          acc = is12 ? (in2 && d2 < k.dpos_m && d2 > k.dneg_m) : (cls == 0 && !gz2);
          vio = is12 && ((tlt1 && !in2) || (in2 && (d2 > k.dpos_p || d2 < k.dneg_p)));
          if (normal && !acc && !vio) vio = violates(inv_f32(vhat, P, amb), xz, k.repair_t);
        }
        const bool keep = normal & !vio;
        repairs += (active & normal & vio) ? 1u : 0u;
        const int fin = keep ? center + rq : 0;
        pn = nhl;
        if (started) hl = keep ? vhat : v;
        if (MODE == kTValCodes) {
          const bool cnt = active & !anchor;
          const int key = cnt ? fin : -1;
          const unsigned grp = __match_any_sync(0xffffffffu, key);
          if (cnt && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&hist[fin], (unsigned long long)__popc(grp));
        } else {
          if (active) {
            S.code[(cc >> 5) & 1][sidx] = anchor ? kAnc : (uint16_t)fin;
            if (anchor) {
              anchors[p] = v;  // forced anchor, D1
            } else {
              bits += lens_smem ? s_lens[fin] : __ldg(lens + fin);
              if (fin == 0) brow[nb++] = v;  // the row's balance list (D9)
            }
          }
        }
      }
      if (MODE == kTMain) {
        __syncwarp();
        const int q = kg - 1;  // complete for every row now
        const bool last = kg == ngroups - 1;
        for (int qq = max(q, 0); qq <= (last ? nch - 1 : q); qq++) {
          if (qq < 0 || qq >= nch) continue;
          const uint16_t *src = S.code[qq & 1];
          const int c0 = qq * 32, w = min(32, C - c0);
          if (vcode && w == 32) {
#pragma unroll
            for (int j = 0; j < 4; j++) {  // 32 rows x 4 x 16 B, 8 rows per instruction
              const int r = j * 8 + (lane >> 2), pc = lane & 3;
              if (r < R)
                *reinterpret_cast<uint4 *>(cb + (int64_t)r * C + c0 + pc * 8) =
                    *reinterpret_cast<const uint4 *>(src + r * 32 + pc * 8);
            }
          } else {
            for (int r = 0; r < R; r++)
              if (lane < w) cb[(int64_t)r * C + c0 + lane] = src[r * 32 + lane];
          }
        }
        __syncwarp();
      }
    }
    cp_async_wait<0>();
    if (MODE == kTMain) {
      if (lane_in) {
        rowinfo[2 * (p * g.prow + lane)] = bits;
        rowinfo[2 * (p * g.prow + lane) + 1] = nb;
      }
      unsigned long long tb = bits, tz = nb;
      unsigned tr = repairs;
      for (int o = 16; o; o >>= 1) {
        tb += __shfl_xor_sync(0xffffffffu, tb, o);
        tz += __shfl_xor_sync(0xffffffffu, tz, o);
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
      }
      if (lane == 0) {
        part_bits[p] = tb;
        part_zeros[p] = tz;
        atomicAdd(&st->nbal, tz);
        if (tr) atomicAdd(&st->nrepair, (unsigned long long)tr);
        atomicAdd(&st->ncodes, (unsigned long long)(R * C - 1));
      }
    } else if (MODE == kTValCodes) {
      if (pi == 0 && lane == 0) atomicAdd(&hist[kMaxAlpha], 1ull);  // k for the floor (D10)
    }
  } else if (have && MODE == kTMain && lane == 0) {
    part_bits[p] = 0;
    part_zeros[p] = 0;
  }
  if (MODE == kTCoverage) {
    __syncthreads();
    if (threadIdx.x < 18 && s_cov[threadIdx.x]) atomicAdd(&cov[threadIdx.x], (unsigned long long)s_cov[threadIdx.x]);
  }
}

// ---------------------------------------------------------------------------
// k_t_write: block records (D13-D15).

__device__ __forceinline__ void st_u8(uint8_t *a, unsigned v) { *a = (uint8_t)v; }

// 8 little-endian bytes of v at any address (one aligned store when possible)
__device__ __forceinline__ void st_u64_any(uint8_t *a, unsigned long long v) {
  if ((reinterpret_cast<uintptr_t>(a) & 7) == 0) {
    *reinterpret_cast<unsigned long long *>(a) = v;
  } else if ((reinterpret_cast<uintptr_t>(a) & 3) == 0) {
    reinterpret_cast<unsigned *>(a)[0] = (unsigned)v;
    reinterpret_cast<unsigned *>(a)[1] = (unsigned)(v >> 32);
  } else {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = (uint8_t)(v >> (8 * i));
  }
}

// MSB-first writer of one row's bits into bytes it owns exclusively:
// [first, last) absolute byte range; bytes are stored one at a time until
// the address is 4-aligned, then as big-endian-packed 32-bit words.
struct TRowWriter {
  uint8_t *out;
  unsigned long long pos;  // next absolute byte to write
  unsigned long long acc;  // pending bits, left-aligned
  int na;                  // pending bit count
  __device__ __forceinline__ void put(unsigned code, int len) {  // len <= 32
    acc |= (unsigned long long)code << (64 - na - len);
    na += len;
    while (na >= 32 || (na >= 8 && (pos & 3))) {
      if ((pos & 3) == 0) {
        const unsigned w = (unsigned)(acc >> 32);
        *reinterpret_cast<unsigned *>(out + pos) = __byte_perm(w, 0, 0x0123);
        acc <<= 32;
        na -= 32;
        pos += 4;
      } else {
        out[pos] = (uint8_t)(acc >> 56);
        acc <<= 8;
        na -= 8;
        pos += 1;
      }
    }
  }
  __device__ __forceinline__ void flush_full_bytes() {
    while (na >= 8) {
      out[pos] = (uint8_t)(acc >> 56);
      acc <<= 8;
      na -= 8;
      pos += 1;
    }
  }
};

__global__ void __launch_bounds__(kTCW * 32) k_t_write(Geom g, const BlkP *__restrict__ blkp,
                                                       const uint16_t *__restrict__ codes,
                                                       const double *__restrict__ balrow,
                                                       const unsigned *__restrict__ rowinfo,
                                                       const double *__restrict__ anchors,
                                                       const unsigned long long *__restrict__ part_bits,
                                                       const unsigned long long *__restrict__ part_zeros,
                                                       const unsigned long long *__restrict__ rec_off,
                                                       const uint8_t *__restrict__ lens,
                                                       const unsigned *__restrict__ cw, uint8_t *out, WsStatus *st) {
  __shared__ unsigned s_cw[kTLensSmem];
  __shared__ uint8_t s_len[kTLensSmem];
  count_launch(st);
  if (st->err_bits) return;  // capacity / codebook errors: nothing is written
  const int m = st->m, nalpha = 1 << m;
  const bool tab_smem = nalpha <= kTLensSmem;
  if (tab_smem)
    for (int i = threadIdx.x; i < nalpha; i += blockDim.x) {
      s_cw[i] = cw[i];
      s_len[i] = lens[i];
    }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * kTCW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlkP P = blkp[b];
  uint8_t *rec = out + st->header_bytes + rec_off[b];
  if (P.trivial) {
    if (pi == 0 && lane == 0) rec[0] = 1;  // trivial block: the flag alone (D13)
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int np = bb.np, pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const int64_t p0 = first_part(g, b);
  // earlier partitions of the block: payload bytes and balance counts; the block's balance count
  unsigned long long pre_bytes = 0, pre_z = 0, tot_z = 0;
  for (int i0 = 0; i0 < np; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long z = i < np ? part_zeros[p0 + i] : 0ull;
    const unsigned long long by = i < pi ? (part_bits[p0 + i] + 7) / 8 : 0ull;
    unsigned long long a = by, zb = i < pi ? z : 0ull, zt = z;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      zb += __shfl_xor_sync(0xffffffffu, zb, o);
      zt += __shfl_xor_sync(0xffffffffu, zt, o);
    }
    pre_bytes += a;
    pre_z += zb;
    tot_z += zt;
  }
  const unsigned long long head = 25ull + 24ull * (unsigned)np;
  // block head (first partition's warp) and this partition's table entry
  if (pi == 0) {
    if (lane == 0) rec[0] = 0;
    if (lane < 8) {
      rec[1 + lane] = (uint8_t)((unsigned long long)__double_as_longlong(P.factor_pos) >> (8 * lane));
      rec[9 + lane] = (uint8_t)((unsigned long long)__double_as_longlong(P.factor_neg) >> (8 * lane));
      rec[17 + 24 * np + lane] = (uint8_t)(tot_z >> (8 * lane));
    }
  }
  if (lane < 24) {
    const unsigned long long f = lane < 8 ? 8ull * pre_bytes
                                 : (lane < 16 ? part_bits[p]
                                              : (unsigned long long)__double_as_longlong(anchors[p]));
    rec[17 + 24 * pi + lane] = (uint8_t)(f >> (8 * (lane & 7)));
  }
  // rows: balance counts / bits -> exclusive prefixes within the partition
  const unsigned rbits = lane < R ? rowinfo[2 * (p * g.prow + lane)] : 0u;
  const unsigned rbal = lane < R ? rowinfo[2 * (p * g.prow + lane) + 1] : 0u;
  unsigned long long ib = rbits;
  unsigned iz = rbal;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long vb = __shfl_up_sync(0xffffffffu, ib, o);
    const unsigned vz = __shfl_up_sync(0xffffffffu, iz, o);
    if (lane >= o) {
      ib += vb;
      iz += vz;
    }
  }
  // balance values of this row, in order (D9)
  {
    uint8_t *dst = rec + head + 8ull * (pre_z + iz - rbal);
    const double *src = balrow + (p * g.prow + lane) * (int64_t)g.bc;
    for (unsigned j = 0; j < rbal; j++)
      st_u64_any(dst + 8ull * j, (unsigned long long)__double_as_longlong(src[j]));
  }
  // payload: this row's codewords from absolute bit A (rows concatenated, D15)
  const unsigned long long pay0 = (unsigned long long)(rec - out) + head + 8ull * tot_z + pre_bytes;
  const uint16_t *crow = codes + tcode_base(g, p) + (int64_t)lane * C;
  auto cwl = [&](unsigned s, unsigned &code) -> int {
    code = tab_smem ? s_cw[s] : __ldg(cw + s);
    return tab_smem ? s_len[s] : __ldg(lens + s);
  };
  if (C < 9) {
    // rows may be shorter than a byte: one lane writes the whole partition
    if (lane == 0) {
      TRowWriter wr{out, pay0, 0ull, 0};
      const uint16_t *cp = codes + tcode_base(g, p);
      for (int i = 1; i < R * C; i++) {
        unsigned code;
        const int l = cwl(cp[i], code);
        wr.put(code, l);
      }
      wr.flush_full_bytes();
      if (wr.na) out[wr.pos] = (uint8_t)(wr.acc >> 56);  // zero-padded last byte
    }
    return;
  }
  const unsigned long long A = 8ull * pay0 + (ib - rbits);  // first bit of this row
  const int s = (int)(A & 7);
  // the first (8 - s) % 8 bits of this row complete the byte row - 1 ends in
  const int hb = (8 - s) & 7;
  unsigned head_bits = 0;  // right-aligned
  int c0 = lane == 0 ? 1 : 0;  // raster 0 is the anchor
  TRowWriter wr{out, (A + 7) >> 3, 0ull, 0};
  if (lane < R) {
    // encode until the head byte is complete, keep the excess in the writer
    unsigned long long acc = 0;
    int na = 0, c = c0;
    while (na < hb) {
      unsigned code;
      const int l = cwl(crow[c++], code);
      acc |= (unsigned long long)code << (64 - na - l);
      na += l;
    }
    head_bits = hb ? (unsigned)(acc >> (64 - hb)) : 0u;
    wr.acc = hb ? (acc << hb) : acc;
    wr.na = na - hb;
    c0 = c;
  }
  const unsigned next_head = __shfl_down_sync(0xffffffffu, head_bits, 1);
  if (lane < R) {
    // flush what the head pass left, then the rest of the row
    {
      int n0 = wr.na;
      unsigned long long a0 = wr.acc;
      wr.acc = 0;
      wr.na = 0;
      if (n0 > 32) {
        wr.put((unsigned)(a0 >> 32), 32);
        a0 <<= 32;
        n0 -= 32;
      }
      if (n0 > 0) wr.put((unsigned)(a0 >> (64 - n0)), n0);
    }
    if (((C - c0) & 7) == 0 && ((reinterpret_cast<uintptr_t>(crow + c0) & 15) == 0)) {
      for (int c = c0; c < C; c += 8) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(crow + c));
        const unsigned q[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; u++) {
          unsigned code;
          int l = cwl(q[u] & 0xffffu, code);
          wr.put(code, l);
          l = cwl(q[u] >> 16, code);
          wr.put(code, l);
        }
      }
    } else {
      for (int c = c0; c < C; c++) {
        unsigned code;
        const int l = cwl(crow[c], code);
        wr.put(code, l);
      }
    }
    wr.flush_full_bytes();
    // the last partial byte: shared with row + 1's head bits (zero padding after the last row)
    if (wr.na) {
      const unsigned hi = (unsigned)(wr.acc >> 56);  // top wr.na bits, rest zero
      const unsigned lo = lane + 1 < R ? next_head : 0u;  // exactly 8 - wr.na bits
      out[wr.pos] = (uint8_t)(hi | lo);
    }
  }
}

}  // namespace pmz
