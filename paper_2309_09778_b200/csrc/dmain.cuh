// dmain.cuh -- throughput-path decompression, issue-efficient version:
// decode_next as k_d_decode, then decompress_block
// + inverse_map (transform.py:188-202) + the float32 cast
// (D20) as k_d_recon.
//
// k_d_decode: a THREAD per partition substream, decoded serially.  The
//   codeword length is the largest l with first_l << (32 - l) <= the next 32
//   stream bits (canonical codes: the left-justified first codewords grow with
//   the length), found by a five-step binary search over the shared table; the
//   symbol is offset_l + the codeword's rank among length-l codewords.  The
//   stream is read from global memory in 16-byte words, one word ahead; codes
//   leave in 16-byte groups of eight (raster per partition, tcode_base),
//   per-row code-0 counts on the side.
// k_d_recon: a WARP per partition, lane = row (the mirror of k_c_main): code
//   tiles stream into a 32 x 64 ring by cp.async three 8-column chunks ahead;
//   at step t lane r reconstructs column t - r: vhat = predict(RECONSTRUCTED
//   W, N, NW) + dequantize(code), or the row's next balance value at code 0
//   (held in a two-deep register queue refilled by plain loads), or the
//   anchor; the inverse map to float32 (256-entry shared table + degree-4
//   series, exact fallback near float32 rounding midpoints) and 8-column
//   output chunks stored from a 32 x 64 float ring once every row finished them.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "decompress.cuh"
#include "wsc.cuh"
#include "tdec.cuh"
#include "cmain.cuh"
#include "cmain32.cuh"

namespace pmz {

#ifndef PMZ_DDT
#define PMZ_DDT 512
#endif
#ifndef PMZ_DRB
#define PMZ_DRB 8
#endif
#ifndef PMZ_DMINB
#define PMZ_DMINB 1
#endif
constexpr int kDDT = PMZ_DDT;      // decoder threads (partitions) per CTA
constexpr int kDRB = PMZ_DRB;      // 16-byte stream blocks in each thread's shared ring

// First-level decode table over the top LB stream bits (built once per
// container by k_d_lut): entry = symbol | length << SB for a codeword of at
// most LB bits.  Alphabets up to 2^11 pack the entry into 16 bits (LB = 14:
// 32 KB; C5 hits 99.4 % of its codes there) and give a longer codeword's
// prefix a second-level table over the next k = clamp(maxl - LB, 1, 4) bits
// (entry length 0, low bits = subtable + 1; L2E entries in all); larger
// alphabets use 32-bit entries over 13 bits.  Entry 0: a binary search over
// the canonical firsts.
template <typename E>
struct DLut;
template <>
struct DLut<uint16_t> {
  static constexpr int LB = 14, SB = 11, L2E = 4096;
};
template <>
struct DLut<unsigned> {
  static constexpr int LB = 13, SB = 16, L2E = 0;
};
template <typename E>
__host__ __device__ constexpr size_t d_lut_bytes() {
  return sizeof(E) * ((1u << DLut<E>::LB) + (size_t)DLut<E>::L2E);
}
constexpr size_t kDLutBytes = d_lut_bytes<uint16_t>() > d_lut_bytes<unsigned>() ? d_lut_bytes<uint16_t>()
                                                                                 : d_lut_bytes<unsigned>();
__host__ __device__ inline bool d_lut16(int m) { return m <= 11; }
template <typename E>
__device__ __forceinline__ int d_l2_bits(int maxl) {
  return min(max(maxl - DLut<E>::LB, 1), 4);
}

__device__ __forceinline__ int d_len_of(unsigned top, const unsigned *lj, int maxl) {
  int l = 1;
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const int c = l + s;
    if (c <= maxl && lj[c] <= top) l = c;
  }
  return l;
}
// lut: [1 << LB] first level, then L2E entries of 2^k-entry subtables;
// lut_n (a device counter, zeroed by the caller) hands out the subtables
template <typename E>
__global__ void k_d_lut(const DecTab *__restrict__ tab, const uint16_t *__restrict__ sym, int nalpha, E *lut,
                        unsigned *lut_n, WsStatus *st) {
  constexpr int LB = DLut<E>::LB, SB = DLut<E>::SB, L2E = DLut<E>::L2E;
  __shared__ unsigned s_lj[34];
  count_launch(st);
  if (threadIdx.x < 34) {
    const unsigned l = threadIdx.x;
    s_lj[l] = (l >= 1 && l <= 32) ? (l == 32 ? tab->first[l] : tab->first[l] << (32 - l)) : 0u;
  }
  __syncthreads();
  const int maxl = tab->maxl;
  const unsigned pfx = blockIdx.x * blockDim.x + threadIdx.x;
  if (pfx >= (1u << LB)) return;
  auto entry = [&](unsigned lo, int lim) -> unsigned {  // the codeword every extension of lo starts with
    const int l0 = d_len_of(lo, s_lj, maxl);
    if (l0 > lim) return 0u;
    unsigned idx = tab->offset[l0] + ((lo - s_lj[l0]) >> (32 - l0));
    idx = idx < (unsigned)nalpha ? idx : (unsigned)nalpha - 1u;
    return (unsigned)sym[idx] | ((unsigned)l0 << SB);
  };
  const unsigned lo = pfx << (32 - LB);
  unsigned e = entry(lo, LB);
  if (e == 0u && L2E > 0) {
    const int k = d_l2_bits<E>(maxl);
    const unsigned j = atomicAdd(lut_n, 1u);
    if (j < (unsigned)(L2E >> k)) {
      E *sub = lut + (1u << LB) + ((size_t)j << k);
      for (unsigned x = 0; x < (1u << k); x++) sub[x] = (E)entry(lo | (x << (32 - LB - k)), LB + k);
      e = j + 1u;
    }
  }
  lut[pfx] = (E)e;
}

// k_d_decode: dynamic shared memory = the tables + the per-thread stream rings
constexpr int kDDTSmall = 128;     // CTA size when the partitions do not fill the GPU at kDDT (spread over all SMs)
template <typename E, int T>
__host__ __device__ constexpr size_t d_dec_smem() {
  return d_lut_bytes<E>() + (size_t)T * kDRB * 16;
}

template <typename E, int T>
__global__ void __launch_bounds__(T, PMZ_DMINB) k_d_decode(const uint8_t *__restrict__ buf, unsigned long long buf_n, Geom g,
                                                   const BlkP *__restrict__ blkp, const DecTab *__restrict__ tab,
                                                   const uint16_t *__restrict__ sym, int nalpha,
                                                   const E *__restrict__ lut1,
                                                   const unsigned long long *__restrict__ part_bits,
                                                   const unsigned long long *__restrict__ part_off,
                                                   const unsigned long long *__restrict__ pay_off,
                                                   uint16_t *__restrict__ codes, unsigned *__restrict__ part_z,
                                                   unsigned *__restrict__ rowz, WsStatus *st) {
  constexpr int LB = DLut<E>::LB, SB = DLut<E>::SB, L2E = DLut<E>::L2E;
  extern __shared__ __align__(16) unsigned char smem_d[];
  E *s_lut = reinterpret_cast<E *>(smem_d);
  const E *s_l2 = s_lut + (1u << LB);
  unsigned *s_ring0 = reinterpret_cast<unsigned *>(smem_d + d_lut_bytes<E>());  // kDRB blocks per thread
  __shared__ unsigned s_lj[34], s_off[34];
  count_launch(st);
  if (threadIdx.x < 34) {
    const unsigned l = threadIdx.x;
    s_lj[l] = (l >= 1 && l <= 32) ? (l == 32 ? tab->first[l] : tab->first[l] << (32 - l)) : 0xffffffffu;
    s_off[l] = tab->offset[l];
  }
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(lut1);
    uint4 *dst = reinterpret_cast<uint4 *>(s_lut);
    for (int i = threadIdx.x; i < (int)(d_lut_bytes<E>() / 16); i += T) dst[i] = src[i];
  }
  const int maxl = tab->maxl;
  const int k2 = d_l2_bits<E>(maxl);
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * T + threadIdx.x;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc;
  unsigned *rz = rowz + p * g.prow;
  if (blkp[b].trivial) {
    part_z[p] = 0;
    for (int r = 0; r < R; r++) rz[r] = 0;
    return;
  }
  const unsigned n = (unsigned)(R * C);
  const unsigned long long L64 = part_bits[p];
  const uint8_t *src = buf + pay_off[b] + part_off[p];
  if (L64 > 32ull * n || pay_off[b] + part_off[p] + (L64 + 7) / 8 > buf_n) {
    set_err_at(st, PMZ_ERR_CORRUPT, 71, p);
    return;
  }
  // reader: the stream's aligned 16-byte blocks stream into a kDRB-block
  // shared ring per thread by cp.async; 32 bits at a time come out of the
  // ring.  The copies are issued and waited for at warp-uniform points (every
  // eight codes, see `ahead`), so each commit group holds the whole warp's
  // copies and a wait covers the lanes' own blocks, not their neighbours'.
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uint4 *qb = reinterpret_cast<const uint4 *>(a & ~(uintptr_t)15);
  const uint4 *qlast = reinterpret_cast<const uint4 *>((reinterpret_cast<uintptr_t>(buf + buf_n) - 1) & ~(uintptr_t)15);
  const unsigned ring_s = smem_u32(s_ring0 + threadIdx.x * (kDRB * 4));
  const unsigned klast = (unsigned)(qlast - qb);  // last readable block (index from qb)
  auto issue = [&](unsigned k) {  // block k -> slot k % kDRB
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring_s + 16u * (k & (kDRB - 1u))),
                 "l"(qb + min(k, klast))
                 : "memory");
  };
#pragma unroll
  for (unsigned k = 0; k < kDRB; k++) issue(k);
  cp_async_commit();
  cp_async_wait<0>();
  unsigned nexti = kDRB;  // next block to copy
  const unsigned wi0 = (unsigned)(a >> 2) & 3u;
  unsigned wi = wi0;  // next 32-bit word (index from qb)
  // before every eight codes: refill the free slots (block k may replace
  // block k - kDRB once word 4 (k - kDRB) + 3 has been read) and wait for the
  // group committed two calls earlier (one when codewords can exceed 24 bits):
  // eight codes and the <= 63 buffered bits read at most 8 (10) words, so the
  // blocks of the next eight codes were issued at least that long ago.
  const bool wide = maxl > 24;
  auto ahead = [&]() {
    const unsigned lim = (wi >> 2) + (kDRB - 1u);
    while (nexti <= lim) issue(nexti++);
    cp_async_commit();
    // (a 4-block ring holds only the blocks of the coming eight codes: wait for this call's copies)
    if (kDRB < 8) cp_async_wait<0>();
    else if (wide) cp_async_wait<1>();
    else cp_async_wait<2>();
  };
  unsigned long long bits = 0;  // left-justified, zeros below the nb valid bits
  int nb = 0;
  auto refill = [&]() {  // nb < 32 -> nb >= 32
    const unsigned w = lds_u32(ring_s + ((wi & (kDRB * 4u - 1u)) << 2));
    wi++;
    bits |= (unsigned long long)__byte_perm(w, 0, 0x0123) << (32 - nb);
    nb += 32;
  };
  refill();
  refill();
  const int sb = (int)(a & 3) * 8;  // bits of the first word before the stream
  bits <<= sb;
  nb -= sb;
  if (nb < 32) refill();
  // a codeword longer than the table: binary search over the canonical
  // firsts; leaves nb >= 32 like every refill
  auto slow = [&]() -> unsigned {
    if (nb < 32) refill();
    const unsigned top = (unsigned)(bits >> 32);
    const int l = d_len_of(top, s_lj, maxl);
    const unsigned idx = s_off[l] + ((top - s_lj[l]) >> (32 - l));  // < nalpha for a complete code
    const unsigned s = __ldg(sym + min(idx, (unsigned)nalpha - 1u));
    bits <<= l;
    nb -= l;
    if (nb < 32) refill();
    return s;
  };
  // longer than the first level: the second-level table, else the search;
  // leaves nb >= LB
  auto dec_long = [&](unsigned e) -> unsigned {
    if (L2E > 0 && e != 0u) {
      if (nb < 32) refill();
      const unsigned e2 = s_l2[((e - 1u) << k2) | (((unsigned)(bits >> 32) << LB) >> (32 - k2))];
      if (e2 != 0u) {
        const unsigned l = e2 >> SB;
        bits <<= l;
        nb -= (int)l;
        return e2 & ((1u << SB) - 1u);
      }
    }
    return slow();
  };
  // one codeword; needs nb >= LB valid bits (a table hit is at most LB bits)
  auto dec = [&]() -> unsigned {
    const unsigned e = s_lut[(unsigned)(bits >> (64 - LB))];
    if (e < (1u << SB)) return dec_long(e);
    const unsigned l = e >> SB;
    bits <<= l;
    nb -= (int)l;
    return e & ((1u << SB) - 1u);
  };
  uint16_t *cp = codes + tcode_base(g, p);
  unsigned zt = 0;
  if ((C & 7) == 0 && ((g.prow * g.bc) & 7) == 0) {
    // groups of eight codes of one row, one 16-byte store; one refill check
    // per pair (nb >= 32 before it, a hit takes <= LB <= 14 bits)
    bool first = true;
    for (int r = 0; r < R; r++) {
      unsigned zr = 0;
      for (int c0 = 0; c0 < C; c0 += 8) {
        ahead();
        unsigned w[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          if (nb < 32) refill();
          unsigned s0;
          if (j == 0 && first) {
            s0 = kAnc;
            first = false;
          } else {
            s0 = dec();
          }
          const unsigned s1 = dec();
          zr += (s0 == 0u) + (s1 == 0u);
          w[j] = s0 | (s1 << 16);
        }
        *reinterpret_cast<uint4 *>(cp) = make_uint4(w[0], w[1], w[2], w[3]);
        cp += 8;
      }
      rz[r] = zr;
      zt += zr;
    }
  } else {
    int col = 0, r = 0;
    unsigned zr = 0;
    for (unsigned i = 0; i < n; i++) {
      if ((i & 7u) == 0) ahead();
      if (nb < 32) refill();
      const unsigned s = i == 0 ? (unsigned)kAnc : dec();
      cp[i] = (uint16_t)s;
      zr += s == 0 ? 1u : 0u;
      if (++col == C) {
        rz[r++] = zr;
        zt += zr;
        zr = 0;
        col = 0;
      }
    }
  }
  part_z[p] = zt;
  const unsigned long long used = 32ull * (wi - wi0) - (unsigned)sb - (unsigned)nb;  // stream bits consumed
  if (used != L64) set_err_at(st, used < L64 ? PMZ_ERR_CORRUPT : PMZ_ERR_TRUNCATED, 72, p);
  cp_async_wait<0>();  // nothing in flight into shared memory at exit
}

// ---------------------------------------------------------------------------
constexpr int kDRW = 8;  // partitions (warps) per reconstruct CTA
__device__ const double kDExp2Tab[257] = {
#include "dmain_tables.inc"
};
struct DRecWarp {
  uint16_t code[32 * kCRing];     // code ring: column c of row r at r * 64 + (c & 63)
  unsigned long long bal[32 * 8]; // per row: the aligned 8-byte words around its next balance values
};
constexpr size_t kDRecSmem = sizeof(DRecWarp) * kDRW + 257 * 8;

__device__ __forceinline__ unsigned long long lds_u64(unsigned a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds_u16(unsigned a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(unsigned a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// (float) of the CR double 2^y for y in (-125, 127) (inverse_map's exp2 + the D20
// cast): 2^(j/256) from the shared table times a degree-4 series in
// t = y - n - j/256 (|t| <= 2^-9, relative error < 2^-50), 2^n through the
// exponent field; when the double lands within 2^-42 of a float32 rounding
// midpoint the exact path decides (pmz_exp2_to_f32)
__device__ __forceinline__ float d_exp2_f32(double y, unsigned tab_s, unsigned *amb) {
  const double tn = __dadd_rn(y, 0x1.8p52);
  const double nn = __dsub_rn(tn, 0x1.8p52);
  const double f = __dsub_rn(y, nn);
  const double tj = __fma_rn(f, 256.0, 0x1.8p52);
  const double jj = __dsub_rn(tj, 0x1.8p52);
  const double t = __fma_rn(jj, -0.00390625, f);  // exact
  double q = __fma_rn(t, 0x1.3b2ab6fba4e77p-7, 0x1.c6b08d704a0c0p-5);
  q = __fma_rn(t, q, 0x1.ebfbdff82c58fp-3);
  q = __fma_rn(t, q, 0x1.62e42fefa39efp-1);
  q = __fma_rn(t, q, 1.0);
  const int j = __double2loint(tj), n = __double2loint(tn);
  const double a0 = __dmul_rn(lds_f64(tab_s + 8u * (unsigned)(j + 128)), q);
  const double a = __hiloint2double(__double2hiint(a0) + (n << 20), __double2loint(a0));
  const unsigned lo29 = (unsigned)__double2loint(a0) & 0x1fffffffu;
  const unsigned dist = (unsigned)abs((int)lo29 - 0x10000000);
  if (__builtin_expect((dist > 1024u) & ((unsigned)(n + 124) < 250u), 1)) return __double2float_rn(a);
  return pmz_exp2_to_f32(y, amb);
}

template <int PK>
__global__ void __launch_bounds__(kDRW * 32, PMZ_DREC_MINB)
    k_d_recon(const uint8_t *__restrict__ buf, unsigned long long buf_n, Geom g, const __grid_constant__ KParams k,
              const BlkP *__restrict__ blkp, const uint16_t *__restrict__ codes, const unsigned *__restrict__ part_z,
              const unsigned *__restrict__ rowz, const double *__restrict__ anchors,
              const unsigned long long *__restrict__ bal_off, const unsigned long long *__restrict__ blk_nbal,
              int center, float *__restrict__ out, WsStatus *st) {
  extern __shared__ __align__(16) unsigned char smem_d[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DRecWarp &S = reinterpret_cast<DRecWarp *>(smem_d)[warp];
  double *s_e2 = reinterpret_cast<double *>(smem_d + sizeof(DRecWarp) * kDRW);
  count_launch(st);
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_e2[i] = kDExp2Tab[i];
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * kDRW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  float *op = out + (bb.r0 + pr0) * g.cols + bb.c0;
  const BlkP P = blkp[b];
  if (P.trivial) {
    for (int r = 0; r < R; r++)
      for (int c = lane; c < C; c += 32) op[(int64_t)r * g.cols + c] = 0.0f;
    return;
  }
  if (st->err_bits) return;  // the decoder failed
  const uint16_t *cb = codes + tcode_base(g, p);
  // balance list of this row (D9): the block's list after the earlier partitions'
  // and the earlier rows' code-0 counts
  unsigned long long bj, bend;
  {
    const int64_t p0 = first_part(g, b);
    unsigned zp = lane < pi ? part_z[p0 + lane] : 0u;
    for (int o = 16; o; o >>= 1) zp += __shfl_xor_sync(0xffffffffu, zp, o);
    const unsigned zr = lane < R ? rowz[p * g.prow + lane] : 0u;
    unsigned incl = zr;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    bj = (unsigned long long)zp + incl - zr;
    bend = (unsigned long long)zp + incl;
    const unsigned long long nbal = blk_nbal[b];
    if (lane == 31 && pi == bb.np - 1 && bend != nbal)
      set_err_at(st, bend > nbal ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 73, p);
    if (__any_sync(0xffffffffu, bend > nbal)) {  // corrupt counts: never read past the list
      if (lane == 0) set_err_at(st, PMZ_ERR_BALANCE_UNDERFLOW, 74, p);
      return;
    }
  }
  // balance values j of this row (bal_off + 8 j, any alignment): value j is
  // bytes of the aligned words j and j + 1 (bq), which stream into an 8-word
  // shared ring per row by cp.async six words ahead of their use
  const uint8_t *bbase = buf + bal_off[b];
  const unsigned bsh = (unsigned)(reinterpret_cast<uintptr_t>(bbase) & 7) * 8;
  const unsigned long long *bq = reinterpret_cast<const unsigned long long *>(reinterpret_cast<uintptr_t>(bbase) & ~(uintptr_t)7);
  const unsigned long long *bqlast =
      reinterpret_cast<const unsigned long long *>((reinterpret_cast<uintptr_t>(buf + buf_n) - 1) & ~(uintptr_t)7);
  const unsigned bal_s = smem_u32(S.bal + lane * 8);
  auto issue_word = [&](unsigned long long w) {  // word w -> slot w & 7 (one cp.async group)
    const unsigned long long *ap = bq + w;
    const bool ok = w <= bend && ap <= bqlast;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(bal_s + 8u * (unsigned)(w & 7)),
                 "l"(ok ? ap : bq), "r"(ok ? 8u : 0u)
                 : "memory");
    cp_async_commit();
  };
  for (unsigned i = 0; i < 7; i++) issue_word(bj + i);
  const double anc = anchors[p];
  unsigned *amb = &st->unresolved;
  const double two_ba = k.two_ba, slope = k.slope;
  const double zthr = P.zero_threshold, bnd = P.boundary, lgp = P.lg_pos, lgn = P.lg_neg;
  const double cmagic = 4503599627370496.0 + (double)center;  // 2^52 + center
  const bool lane0 = lane == 0, lane_in = lane < R;
  const unsigned code_s = smem_u32(S.code + lane * kCRing), tab_s = smem_u32(s_e2);
  const int nsteps = C + R - 1;
  const bool vcode = (C & 7) == 0 && ((g.prow * g.bc) & 7) == 0;
  const bool vout = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  // code chunk kc (columns 8 kc .. 8 kc + 7 of every row): each lane loads its
  // row's 16 bytes one group ahead into registers and stores them into the
  // ring when the group starts (cp.async is left to the balance words)
  auto ld_codes = [&](int kc) -> uint4 {
    const int c0 = kc * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (c0 < C && lane_in) {
      const uint16_t *srcp = cb + (int64_t)lane * C + c0;
      if (vcode) {
        v = __ldg(reinterpret_cast<const uint4 *>(srcp));
      } else {
        unsigned h[8];
        for (int c = 0; c < 8; c++) h[c] = c0 + c < C ? srcp[c] : 0u;
        v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      }
    }
    return v;
  };
  auto st_codes = [&](int kc, uint4 v) {
    *reinterpret_cast<uint4 *>(S.code + lane * kCRing + ((kc * 8) & (kCRing - 1))) = v;
  };
  // outputs: each lane's row, four columns per 16-byte store (the sectors
  // complete in L2 across consecutive stores)
  float4 ob = make_float4(0.f, 0.f, 0.f, 0.f);
  float *orow = op + (int64_t)lane * g.cols;
  double hl = 0.0, pn = 0.0;
  uint4 cnext = ld_codes(0);
  for (int t0 = 0; t0 < nsteps; t0 += 8) {
    __syncwarp();
    st_codes(t0 >> 3, cnext);
    cnext = ld_codes((t0 >> 3) + 1);
    __syncwarp();
    const int t1 = min(nsteps, t0 + 8);
#pragma unroll kUnrD
    for (int t = t0; t < t1; t++) {
      const int c = t - lane;
      const bool started = c >= 0;
      const bool active = lane_in & ((unsigned)c < (unsigned)C);
      const bool anchor = lane0 & (c == 0);
      const unsigned cidx = (unsigned)(c & (kCRing - 1));
      const unsigned code = lds_u16(code_s + (cidx << 1));
      // dequantize: (code - center) exactly via the 2^52 magic, times 2 b_a
      const double dq = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, (int)code), cmagic), two_ba);
      const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
      double a;
      if (PK == 3) {  // predict_init (D3): a w2_0 + a w2_1 with w2 = 1/2, exactly as written
        double h = __dsub_rn(__dadd_rn(hl, nhl), pn);
        h = lane0 ? hl : h;
        a = h < 0.0 ? __dmul_rn(slope, h) : h;
        const double a2 = __dmul_rn(a, 0.5);
        a = __dadd_rn(a2, a2);
      } else {
        a = predict_steady<PK>(k, hl, nhl, pn, lane0);
      }
      const bool isbal = active & (code == 0) & !anchor;
      double qv = 0.0;
      if (isbal) {  // the row's next balance value (words bj, bj + 1 landed: issued 6 groups ago)
        cp_async_wait<5>();
        const unsigned long long lo = lds_u64(bal_s + 8u * (unsigned)(bj & 7));
        const unsigned long long hw = lds_u64(bal_s + 8u * (unsigned)((bj + 1) & 7));
        qv = __longlong_as_double((long long)(bsh ? ((lo >> bsh) | (hw << (64 - bsh))) : lo));
        issue_word(bj + 7);
        bj++;
      }
      const double vh = anchor ? anc : (isbal ? qv : __dadd_rn(a, dq));
      pn = nhl;
      hl = started ? vh : hl;
      // inverse_map (transform.py:188-202) + float32 cast (D20)
      // (lanes outside the partition and zero outputs evaluate 2^0.5 instead)
      const bool negv = vh > bnd, zero = vh <= zthr;
      const float e = d_exp2_f32((active & !zero) ? __dsub_rn(vh, negv ? lgn : lgp) : 0.5, tab_s, amb);
      const float y = zero ? 0.0f : (negv ? -e : e);
      if (active) ob = make_float4(ob.y, ob.z, ob.w, y);
      if (vout) {
        if (active & ((c & 3) == 3)) *reinterpret_cast<float4 *>(orow + (c - 3)) = ob;
      } else if (active) {
        orow[c] = y;
      }
    }
  }
  cp_async_wait<0>();
  // the row's last 1-3 columns when C is not a multiple of 4
  if (vout && lane_in && (C & 3)) {
    const float v4[4] = {ob.x, ob.y, ob.z, ob.w};
    for (int q = 0; q < (C & 3); q++) orow[C - (C & 3) + q] = v4[4 - (C & 3) + q];
  }
}

// FP32 perceptron perf mode (container version 2): the mirror of k_c_main32
// -- the same sweep as k_d_recon with the float32 recurrence; balance values
// and anchors are the encoder's float32 values stored as doubles; the output
// is inverse_map((double)vhat) exactly as the encoder's bound check saw it.
template <int PK>
__global__ void __launch_bounds__(kDRW * 32, PMZ_DREC_MINB)
    k_d_recon32(const uint8_t *__restrict__ buf, unsigned long long buf_n, Geom g, const __grid_constant__ KParams k,
              const BlkP *__restrict__ blkp, const uint16_t *__restrict__ codes, const unsigned *__restrict__ part_z,
              const unsigned *__restrict__ rowz, const double *__restrict__ anchors,
              const unsigned long long *__restrict__ bal_off, const unsigned long long *__restrict__ blk_nbal,
              int center, float *__restrict__ out, WsStatus *st) {
  extern __shared__ __align__(16) unsigned char smem_d[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DRecWarp &S = reinterpret_cast<DRecWarp *>(smem_d)[warp];
  double *s_e2 = reinterpret_cast<double *>(smem_d + sizeof(DRecWarp) * kDRW);
  count_launch(st);
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_e2[i] = kDExp2Tab[i];
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * kDRW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  float *op = out + (bb.r0 + pr0) * g.cols + bb.c0;
  const BlkP P = blkp[b];
  if (P.trivial) {
    for (int r = 0; r < R; r++)
      for (int c = lane; c < C; c += 32) op[(int64_t)r * g.cols + c] = 0.0f;
    return;
  }
  if (st->err_bits) return;  // the decoder failed
  const uint16_t *cb = codes + tcode_base(g, p);
  // balance list of this row (D9): the block's list after the earlier partitions'
  // and the earlier rows' code-0 counts
  unsigned long long bj, bend;
  {
    const int64_t p0 = first_part(g, b);
    unsigned zp = lane < pi ? part_z[p0 + lane] : 0u;
    for (int o = 16; o; o >>= 1) zp += __shfl_xor_sync(0xffffffffu, zp, o);
    const unsigned zr = lane < R ? rowz[p * g.prow + lane] : 0u;
    unsigned incl = zr;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    bj = (unsigned long long)zp + incl - zr;
    bend = (unsigned long long)zp + incl;
    const unsigned long long nbal = blk_nbal[b];
    if (lane == 31 && pi == bb.np - 1 && bend != nbal)
      set_err_at(st, bend > nbal ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 73, p);
    if (__any_sync(0xffffffffu, bend > nbal)) {  // corrupt counts: never read past the list
      if (lane == 0) set_err_at(st, PMZ_ERR_BALANCE_UNDERFLOW, 74, p);
      return;
    }
  }
  // balance values j of this row (bal_off + 8 j, any alignment): value j is
  // bytes of the aligned words j and j + 1 (bq), which stream into an 8-word
  // shared ring per row by cp.async six words ahead of their use
  const uint8_t *bbase = buf + bal_off[b];
  const unsigned bsh = (unsigned)(reinterpret_cast<uintptr_t>(bbase) & 7) * 8;
  const unsigned long long *bq = reinterpret_cast<const unsigned long long *>(reinterpret_cast<uintptr_t>(bbase) & ~(uintptr_t)7);
  const unsigned long long *bqlast =
      reinterpret_cast<const unsigned long long *>((reinterpret_cast<uintptr_t>(buf + buf_n) - 1) & ~(uintptr_t)7);
  const unsigned bal_s = smem_u32(S.bal + lane * 8);
  auto issue_word = [&](unsigned long long w) {  // word w -> slot w & 7 (one cp.async group)
    const unsigned long long *ap = bq + w;
    const bool ok = w <= bend && ap <= bqlast;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(bal_s + 8u * (unsigned)(w & 7)),
                 "l"(ok ? ap : bq), "r"(ok ? 8u : 0u)
                 : "memory");
    cp_async_commit();
  };
  for (unsigned i = 0; i < 7; i++) issue_word(bj + i);
  const double anc = anchors[p];
  unsigned *amb = &st->unresolved;
  const float two_ba32 = (float)k.two_ba;
  const double zthr = P.zero_threshold, bnd = P.boundary, lgp = P.lg_pos, lgn = P.lg_neg;
  const double cmagic = 4503599627370496.0 + (double)center;  // 2^52 + center
  const bool lane0 = lane == 0, lane_in = lane < R;
  const unsigned code_s = smem_u32(S.code + lane * kCRing), tab_s = smem_u32(s_e2);
  const int nsteps = C + R - 1;
  const bool vcode = (C & 7) == 0 && ((g.prow * g.bc) & 7) == 0;
  const bool vout = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  // code chunk kc (columns 8 kc .. 8 kc + 7 of every row): each lane loads its
  // row's 16 bytes one group ahead into registers and stores them into the
  // ring when the group starts (cp.async is left to the balance words)
  auto ld_codes = [&](int kc) -> uint4 {
    const int c0 = kc * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (c0 < C && lane_in) {
      const uint16_t *srcp = cb + (int64_t)lane * C + c0;
      if (vcode) {
        v = __ldg(reinterpret_cast<const uint4 *>(srcp));
      } else {
        unsigned h[8];
        for (int c = 0; c < 8; c++) h[c] = c0 + c < C ? srcp[c] : 0u;
        v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      }
    }
    return v;
  };
  auto st_codes = [&](int kc, uint4 v) {
    *reinterpret_cast<uint4 *>(S.code + lane * kCRing + ((kc * 8) & (kCRing - 1))) = v;
  };
  // outputs: each lane's row, four columns per 16-byte store (the sectors
  // complete in L2 across consecutive stores)
  float4 ob = make_float4(0.f, 0.f, 0.f, 0.f);
  float *orow = op + (int64_t)lane * g.cols;
  float hl = 0.0f, pn = 0.0f;
  uint4 cnext = ld_codes(0);
  for (int t0 = 0; t0 < nsteps; t0 += 8) {
    __syncwarp();
    st_codes(t0 >> 3, cnext);
    cnext = ld_codes((t0 >> 3) + 1);
    __syncwarp();
    const int t1 = min(nsteps, t0 + 8);
#pragma unroll kUnrD
    for (int t = t0; t < t1; t++) {
      const int c = t - lane;
      const bool started = c >= 0;
      const bool active = lane_in & ((unsigned)c < (unsigned)C);
      const bool anchor = lane0 & (c == 0);
      const unsigned cidx = (unsigned)(c & (kCRing - 1));
      const unsigned code = lds_u16(code_s + (cidx << 1));
      // FP32 perceptron perf mode (container version 2, cmain32.cuh): the float32 mirror recurrence
      const float dq = __fmul_rn((float)((int)code - center), two_ba32);
      const float nhl = __shfl_up_sync(0xffffffffu, hl, 1);
      const float a = c_pred32<PK>(k, hl, nhl, pn, lane0);
      const bool isbal = active & (code == 0) & !anchor;
      double qv = 0.0;
      if (isbal) {  // the row's next balance value (words bj, bj + 1 landed: issued 6 groups ago)
        cp_async_wait<5>();
        const unsigned long long lo = lds_u64(bal_s + 8u * (unsigned)(bj & 7));
        const unsigned long long hw = lds_u64(bal_s + 8u * (unsigned)((bj + 1) & 7));
        qv = __longlong_as_double((long long)(bsh ? ((lo >> bsh) | (hw << (64 - bsh))) : lo));
        issue_word(bj + 7);
        bj++;
      }
      const float vh32 = anchor ? (float)anc : (isbal ? (float)qv : __fadd_rn(a, dq));
      const double vh = (double)vh32;
      pn = nhl;
      hl = started ? vh32 : hl;
      // inverse_map (transform.py:188-202) + float32 cast (D20)
      // (lanes outside the partition and zero outputs evaluate 2^0.5 instead)
      const bool negv = vh > bnd, zero = vh <= zthr;
      const float e = d_exp2_f32((active & !zero) ? __dsub_rn(vh, negv ? lgn : lgp) : 0.5, tab_s, amb);
      const float y = zero ? 0.0f : (negv ? -e : e);
      if (active) ob = make_float4(ob.y, ob.z, ob.w, y);
      if (vout) {
        if (active & ((c & 3) == 3)) *reinterpret_cast<float4 *>(orow + (c - 3)) = ob;
      } else if (active) {
        orow[c] = y;
      }
    }
  }
  cp_async_wait<0>();
  // the row's last 1-3 columns when C is not a multiple of 4
  if (vout && lane_in && (C & 3)) {
    const float v4[4] = {ob.x, ob.y, ob.z, ob.w};
    for (int q = 0; q < (C & 3); q++) orow[C - (C & 3) + q] = v4[4 - (C & 3) + q];
  }
}

}  // namespace pmz
