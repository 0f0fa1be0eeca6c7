// tdec.cuh -- throughput-path decompression (fields with many partitions):
// decode_next and decompress_block +
// inverse_map (transform.py:188-202) as two kernels whose work per element is
// minimal, for fields where partition-level parallelism alone fills the GPU.
//
// k_t_decode: a THREAD per partition substream decodes it serially (12-bit
//   first-level table in shared memory, global second level), one codeword per
//   loop iteration, so the 32 threads of a warp advance in lockstep; every 32
//   iterations the warp writes the 32 x 32 codes it buffered in shared memory
//   with coalesced 4-byte stores.  Codes land raster-contiguous per partition
//   (tcode_base); code-0 counts per row and per partition on the side.
// k_t_recon: a WARP per partition (lane = row) runs the anti-diagonal
//   recurrence vhat = predict(RECONSTRUCTED W, N, NW) + dequantize(code) (or
//   the next balance value of the row at code 0, the anchor at raster 0), maps
//   it straight to float32 (inverse_map + D20) and stages the output in shared
//   memory; code tiles arrive by cp.async one 32-column chunk ahead, finished
//   output chunks leave as coalesced 16-byte stores.  No intermediate
//   per-element array ever goes to HBM besides the 2-byte codes.
#pragma once
#include "common.cuh"
#include "compress.cuh"
#include "decompress.cuh"
#include "dec4.cuh"
#include "wsc.cuh"

namespace pmz {

// throughput path from this many partitions on (capi.cu use_tpath): compress / decompress
constexpr int64_t kTputMinPartsC = 5120;
constexpr int64_t kTputMinPartsD = 6144;

// raster-contiguous per-partition code layout (index r * C + c), capacity prow x bc
__host__ __device__ __forceinline__ int64_t tcode_base(const Geom &g, int64_t p) {
  return p * (int64_t)g.prow * (int64_t)g.bc;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// f32 RN of the CR double 2^y (inverse_map's exp2 + the D20 cast) -- same
// value as pmz_exp2_to_f32: degree-6 Taylor on a 64-entry table, 2^n by
// exponent arithmetic, and the rounding-certainty test on the mantissa bits
// below float precision (the approximation is within 2^-60 relative; a result
// within 2^-43 of an f32 rounding midpoint takes the exact path).
__device__ __forceinline__ float t_exp2_to_f32(double y, unsigned *amb) {
  if (__builtin_expect(y > -125.0 && y < 127.0, 1)) {
    const double nn = rint(y);
    const double f = __dsub_rn(y, nn);
    const double jj = rint(__dmul_rn(f, 64.0));
    const double t = __fma_rn(jj, -0.015625, f);  // exact
    double p = pmz_exp2_c_hi[6];
#pragma unroll
    for (int q = 5; q >= 0; --q) p = __fma_rn(p, t, pmz_exp2_c_hi[q]);
    const double a0 = __dmul_rn(__ldg(&pmz_exp2_tab_hi[(int)jj + 32]), p);
    // a0 in [2^-0.5, 2^0.5]: scale by 2^n exactly through the exponent field
    const double a = __dmul_rn(a0, __longlong_as_double((long long)((int)nn + 1023) << 52));
    // bits of a below float precision (29 of the 52 mantissa bits): a
    // rounding midpoint sits at 0x10000000; |a - a~| <= 2^-60 a moves them by < 2^-8
    const unsigned lo29 = (unsigned)__double2loint(a) & 0x1fffffffu;
    const unsigned dist = (unsigned)abs((int)lo29 - 0x10000000);
    if (__builtin_expect(dist > 1024u, 1)) return __double2float_rn(a);
  }
  return __double2float_rn(pmz_exp2_cr(y, amb));
}

// inv_f32 (common.cuh) without divergent branches: one exp2 per element
__device__ __forceinline__ float t_inv_f32(double v, double zthr, double bnd, double lgp, double lgn, unsigned *amb) {
  const bool neg = v > bnd;
  const float e = t_exp2_to_f32(__dsub_rn(v, neg ? lgn : lgp), amb);
  return v <= zthr ? 0.0f : (neg ? -e : e);
}

// ---------------------------------------------------------------------------
constexpr int kTDT = 256;  // decoder threads (partitions) per CTA

__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, unsigned src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void *smem, const void *gmem, unsigned src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
               : "memory");
}

// MSB-first reader over one substream.  The stream's 16-byte aligned blocks
// stream into a 4-block shared-memory ring with cp.async, three blocks ahead
// of use, and a refill takes the next 32-bit word from the ring -- nothing on
// a codeword's dependency chain ever waits for global memory.
struct TReader {
  unsigned long long buf;  // next stream bits, left-aligned
  int nb;                  // valid bits in buf (>= 32 after refill)
  unsigned wi, wi0, skip;  // next word index (from the aligned base); first word; bits skipped in it
  const uint4 *base, *qend;
  unsigned *ring;          // 16 words
  __device__ __forceinline__ void issue(unsigned blk) {
    const uint4 *a = base + blk;
    cp_async16_zfill(ring + 4 * (blk & 3), a < qend ? a : base, a < qend ? 16u : 0u);
    cp_async_commit();
  }
  __device__ __forceinline__ void init(const uint8_t *src, const uint8_t *end, unsigned *r) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    base = reinterpret_cast<const uint4 *>(a & ~(uintptr_t)15);
    qend = reinterpret_cast<const uint4 *>((reinterpret_cast<uintptr_t>(end) + 15) & ~(uintptr_t)15);
    ring = r;
    issue(0);
    issue(1);
    issue(2);
    cp_async_wait<2>();  // block 0
    issue(3);
    const unsigned sk = (unsigned)(a & 15) * 8;
    wi = wi0 = sk >> 5;
    skip = sk & 31;
    buf = 0;
    nb = 0;
    refill();
    refill();
    buf <<= skip;
    nb -= (int)skip;
  }
  __device__ __forceinline__ void refill() {
    const bool need = nb <= 32;
    if (need && (wi & 3u) == 0u && wi != 0u) {  // first word of block k: k landed, k + 3 goes out
      cp_async_wait<2>();
      issue((wi >> 2) + 3u);
    }
    const unsigned w = __byte_perm(ring[wi & 15u], 0, 0x0123);  // big-endian bit order
    buf |= need ? ((unsigned long long)w << (32 - nb)) : 0ull;
    nb += need ? 32 : 0;
    wi += need ? 1u : 0u;
  }
  __device__ __forceinline__ void skip_bits(unsigned l) {
    buf <<= l;
    nb -= (int)l;
  }
  __device__ __forceinline__ unsigned long long consumed() const {
    return 32ull * (wi - wi0) - skip - (unsigned)nb;
  }
};

constexpr int kTDS = 34;   // codes per thread buffer row (32 + 2 pad: conflict-free 2-byte stores)
constexpr int kTDSym = 1 << 11;  // canonical symbol table in shared memory up to this alphabet
struct TDecDyn {
  uint16_t buf[kTDT][kTDS];  // 32 decoded codes per thread between cooperative stores
  unsigned ring[kTDT][16];   // bitstream ring per thread (TReader)
};
constexpr size_t kTDecSmem = sizeof(TDecDyn);

// Codeword longer than the first-level table: canonical search over the
// lengths kLutBits+1 .. maxl (first / count / offset in shared memory), the
// symbol from the shared (or, for alphabets > 2^11, global) canonical table.
__device__ __forceinline__ unsigned td_long(unsigned top, const DecTab &tab, const uint16_t *s_sym, bool sym_smem,
                                            const uint16_t *__restrict__ sym, unsigned &s) {
  for (int l = kLutBits + 1; l <= tab.maxl; l++) {
    const unsigned d = (top >> (32 - l)) - tab.first[l];
    if (d < tab.count[l]) {
      const unsigned i = tab.offset[l] + d;
      s = sym_smem ? s_sym[i] : __ldg(sym + i);
      return (unsigned)l;
    }
  }
  s = 0;
  return 32u;  // no codeword (a corrupt stream): the bit count check reports it
}

__global__ void __launch_bounds__(kTDT, 4) k_t_decode(const uint8_t *__restrict__ buf, unsigned long long buf_n, Geom g,
                                                  const BlkP *__restrict__ blkp, const DecTab *__restrict__ tab,
                                                  const uint16_t *__restrict__ sym, const unsigned *__restrict__ lut,
                                                  const unsigned long long *__restrict__ part_bits,
                                                  const unsigned long long *__restrict__ part_off,
                                                  const unsigned long long *__restrict__ pay_off,
                                                  int nalpha, uint16_t *__restrict__ codes,
                                                  unsigned *__restrict__ part_z, WsStatus *st) {
  __shared__ DecTab s_tab;
  __shared__ unsigned s_t12[1 << kLutBits];  // (length << 16) | symbol; length 0: longer codeword
  __shared__ uint16_t s_sym[kTDSym];         // symbols in canonical order (alphabets up to 2^11)
  extern __shared__ __align__(16) unsigned char tdec_dyn[];
  TDecDyn &D = *reinterpret_cast<TDecDyn *>(tdec_dyn);
  auto &s_buf = D.buf;
  __shared__ unsigned s_n[kTDT];  // codes (raster positions, anchor included) of each thread's partition; 0 = none
  count_launch(st);
  if (threadIdx.x == 0) s_tab = *tab;
  for (int i = threadIdx.x; i < (1 << kLutBits); i += kTDT) {
    const unsigned e = __ldg(lut + i);
    s_t12[i] = (e != 0 && !(e & kLutL2Flag)) ? (e & 0x1fffffu) : 0u;
  }
  const bool sym_smem = nalpha <= kTDSym;
  if (sym_smem)
    for (int i = threadIdx.x; i < nalpha; i += kTDT) s_sym[i] = sym[i];
  const int tid = threadIdx.x, lane = tid & 31, wb = tid & ~31;
  const int64_t p = (int64_t)blockIdx.x * kTDT + tid;
  unsigned n = 0;  // raster positions of this partition (R * C), 0 when nothing to decode
  int C = 1;
  const uint8_t *src = buf;
  unsigned long long L64 = 0;
  if (p < g.nparts) {
    int64_t b;
    int pi;
    part_of(g, p, b, pi);
    if (!blkp[b].trivial) {
      const BlockBox bb = block_box(g, b);
      const int R = min(g.prow, bb.br - pi * g.prow);
      C = bb.bc;
      n = (unsigned)(R * C);
      L64 = part_bits[p];
      if (L64 > 32ull * n) {
        set_err_at(st, PMZ_ERR_CORRUPT, 61, p);
        n = 0;
      } else {
        src = buf + pay_off[b] + part_off[p];
      }
    } else {
      part_z[p] = 0;
    }
  }
  s_n[tid] = n;
  __syncthreads();
  unsigned nmax = n;
  for (int o = 16; o; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
  TReader rd;
  if (n) rd.init(src, buf + buf_n, D.ring[tid]);
  s_buf[tid][0] = kAnc;  // raster 0: the anchor (not a code)
  unsigned zt = 0;
  // cooperative flush of raster chunk q (positions 32 q .. 32 q + 31) of the
  // warp's 32 partitions: two partitions per store instruction, 4-byte pairs
  auto flush = [&](unsigned q) {
    __syncwarp();
#pragma unroll 4
    for (int j = 0; j < 16; j++) {
      const int t = wb + 2 * j + (lane >> 4);  // partition thread
      const unsigned nt = s_n[t];
      const unsigned i0 = 32 * q + 2 * (lane & 15);
      if (i0 < nt) {
        const int64_t pt = (int64_t)blockIdx.x * kTDT + t;
        uint16_t *dst = codes + tcode_base(g, pt) + i0;
        const uint16_t *sp = &s_buf[t][2 * (lane & 15)];
        if (i0 + 1 < nt) *reinterpret_cast<unsigned *>(dst) = *reinterpret_cast<const unsigned *>(sp);
        else dst[0] = sp[0];
      }
    }
    __syncwarp();
  };
  // 32 codewords per thread per round (unrolled: the buffer slot is a
  // constant), then one cooperative store of the warp's 32 x 32 codes
  const unsigned nrounds = (nmax + 31) >> 5;
  unsigned nmin = n;
  for (int o = 16; o; o >>= 1) nmin = min(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
  const unsigned nfast = nmin >> 5;  // rounds 1 .. nfast - 1: every thread decodes all 32
  for (unsigned q = 0; q < nrounds; q++) {
    if (q >= 1 && q < nfast) {
#pragma unroll
      for (int j = 0; j < 32; j++) {
        rd.refill();
        const unsigned top = (unsigned)(rd.buf >> 32);
        const unsigned e = s_t12[top >> (32 - kLutBits)];
        unsigned l = e >> 16, sy = e & 0xffffu;
        if (__builtin_expect(l == 0, 0)) l = td_long(top, s_tab, s_sym, sym_smem, sym, sy);
        rd.skip_bits(l);
        s_buf[tid][j] = (uint16_t)sy;
        zt += sy == 0 ? 1u : 0u;
      }
      flush(q);
      continue;
    }
#pragma unroll
    for (int j = 0; j < 32; j++) {
      const unsigned i = (q << 5) + j;
      if (i != 0 && i < n) {
        rd.refill();
        const unsigned top = (unsigned)(rd.buf >> 32);
        const unsigned e = s_t12[top >> (32 - kLutBits)];
        unsigned l = e >> 16, sy = e & 0xffffu;
        if (__builtin_expect(l == 0, 0)) l = td_long(top, s_tab, s_sym, sym_smem, sym, sy);
        rd.skip_bits(l);
        s_buf[tid][j] = (uint16_t)sy;
        zt += sy == 0 ? 1u : 0u;
      }
    }
    flush(q);
  }
  if (n) {
    part_z[p] = zt;
    const unsigned long long pos = rd.consumed();
    if (pos != L64) set_err_at(st, pos < L64 ? PMZ_ERR_CORRUPT : PMZ_ERR_TRUNCATED, 62, p);
  }
  cp_async_wait<0>();  // nothing in flight into shared memory at exit
}

// ---------------------------------------------------------------------------
constexpr int kTRW = 4;  // partitions (warps) per reconstruct CTA
struct TRecWarp {
  uint16_t code[3][32 * 32];            // code tiles, chunk q in slot q % 3 (cp.async, one chunk ahead)
  float out[2][32 * 32];                // float32 output tiles, chunk q in slot q & 1
  unsigned long long bring[32][16];     // per row: the aligned words around its next balance values
};
constexpr size_t kTRecSmem = sizeof(TRecWarp) * kTRW;

// unaligned little-endian double at byte address a (inside the container;
// never reads at or past `end`)
__device__ __forceinline__ double ld_f64_any(const uint8_t *a, const uint8_t *end) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(a);
  const unsigned sh = (unsigned)(u & 7) * 8;
  const unsigned long long *q = reinterpret_cast<const unsigned long long *>(u & ~(uintptr_t)7);
  unsigned long long v;
  if (!sh) {
    v = __ldg(q);
  } else if (reinterpret_cast<const uint8_t *>(q + 2) <= end) {
    v = (__ldg(q) >> sh) | (__ldg(q + 1) << (64 - sh));
  } else {
    v = 0;
    for (int i = 7; i >= 0; i--) v = (v << 8) | __ldg(a + i);
  }
  return __longlong_as_double((long long)v);
}

template <int PK>
__global__ void __launch_bounds__(kTRW * 32, 3) k_t_recon(const uint8_t *__restrict__ buf, unsigned long long buf_n,
                                                          Geom g, KParams k, const BlkP *__restrict__ blkp,
                                                          const uint16_t *__restrict__ codes,
                                                          const unsigned *__restrict__ part_z,
                                                          const double *__restrict__ anchors,
                                                          const unsigned long long *__restrict__ bal_off,
                                                          const unsigned long long *__restrict__ blk_nbal, int center,
                                                          float *__restrict__ out, WsStatus *st) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TRecWarp &S = reinterpret_cast<TRecWarp *>(smem_raw)[warp];
  const int64_t p = (int64_t)blockIdx.x * kTRW + warp;
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
  const int nch = (C + 31) >> 5, nsteps = C + R - 1, ngroups = (nsteps + 31) >> 5;
  const uint16_t *cb = codes + tcode_base(g, p);
  const bool vcode = (C & 7) == 0;  // rows of 16-byte aligned code runs
  const bool vout = ((g.cols & 3) == 0) && ((bb.c0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  // code tile of chunk q -> slot q % 3 (rows of 32 codes = 64 bytes)
  auto load_codes = [&](int q) {
    uint16_t *dst = S.code[q % 3];
    const int c0 = q * 32, w = min(32, C - c0);
    if (vcode && w == 32) {
#pragma unroll
      for (int j = 0; j < 4; j++) {  // 32 rows x 4 x 16 B: lane -> (row, 16-byte piece)
        const int r = j * 8 + (lane >> 2), pc = lane & 3;
        if (r < R) cp_async16(dst + r * 32 + pc * 8, cb + (int64_t)r * C + c0 + pc * 8);
      }
    } else {
      for (int r = 0; r < R; r++)
        if (lane < w) dst[r * 32 + lane] = cb[(int64_t)r * C + c0 + lane];
    }
    cp_async_commit();
  };
  // balance list of this partition: the block's list (bal_off) from the
  // code-0 counts of the earlier partitions of the block (D9), then row by row
  unsigned long long before = 0;
  {
    const int64_t p0 = first_part(g, b);
    unsigned zp = lane < pi ? part_z[p0 + lane] : 0u;
    for (int o = 16; o; o >>= 1) zp += __shfl_xor_sync(0xffffffffu, zp, o);
    before = zp;
  }
  // this row's code-0 count (the anchor slot holds kAnc, never 0)
  unsigned zrow = 0;
  if (lane < R) {
    const uint16_t *row = cb + (int64_t)lane * C;
    if (vcode) {
      for (int c = 0; c < C; c += 8) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(row + c));
        zrow += (__popc(__vcmpeq2(w.x, 0u)) + __popc(__vcmpeq2(w.y, 0u)) + __popc(__vcmpeq2(w.z, 0u)) +
                 __popc(__vcmpeq2(w.w, 0u))) >> 4;
      }
    } else {
      for (int c = 0; c < C; c++) zrow += row[c] == 0 ? 1u : 0u;
    }
  }
  unsigned incl = zrow;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned long long nbal = blk_nbal[b];
  unsigned long long bj = before + incl - zrow;  // this row's next balance index
  const unsigned long long bend = before + incl;
  if (lane == 31 && pi == bb.np - 1 && before + incl != nbal)
    set_err_at(st, before + incl > nbal ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 63, p);
  if (__any_sync(0xffffffffu, bend > nbal)) {  // corrupt counts: never read past the list
    if (lane == 0) set_err_at(st, PMZ_ERR_BALANCE_UNDERFLOW, 64, p);
    return;
  }
  // this row's balance values (contiguous in the block's list, D9): the
  // aligned 8-byte words around them stream into a 16-word shared ring per
  // row with cp.async, a half (8 words) at a time and one half ahead, so a
  // code 0 reads shared memory, never waits on a global load
  const uintptr_t ba = reinterpret_cast<uintptr_t>(buf + bal_off[b]);
  const unsigned bsh = (unsigned)(ba & 7) * 8;
  const unsigned long long *qb = reinterpret_cast<const unsigned long long *>(ba & ~(uintptr_t)7);
  const unsigned long long *qend = reinterpret_cast<const unsigned long long *>(
      (reinterpret_cast<uintptr_t>(buf + buf_n) + 7) & ~(uintptr_t)7);
  unsigned long long *bring = S.bring[lane];
  auto issue8 = [&](unsigned long long w0) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const unsigned long long *a = qb + w0 + i;
      cp_async8_zfill(bring + ((w0 + i) & 15), a < qend ? a : qb, a < qend ? 8u : 0u);
    }
    cp_async_commit();
  };
  {
    const unsigned long long h = bj & ~7ull;
    issue8(h);
    issue8(h + 8);
    cp_async_wait<1>();
  }
  const double anc = anchors[p];
  unsigned *amb = &st->unresolved;
  const double two_ba = k.two_ba;
  const double zthr = P.zero_threshold, bnd = P.boundary, lgp = P.lg_pos, lgn = P.lg_neg;
  const bool lane0 = lane == 0, lane_in = lane < R;
  double hl = 0.0, pn = 0.0;

  load_codes(0);
  for (int kg = 0; kg < ngroups; kg++) {
    if (kg + 1 < nch) {
      load_codes(kg + 1);
      cp_async_wait<1>();  // chunk kg has landed (kg + 1 may be in flight)
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int t0 = kg * 32, t1 = min(nsteps, t0 + 32);
    const uint16_t *ccur = S.code[kg % 3], *cprev = S.code[(kg + 2) % 3];
    for (int tb = t0; tb < t1; tb += 4) {
      // four recurrence steps, then their four inverse maps (independent
      // exp2 chains off the recurrence's critical path)
      double vq[4];
      int oq[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int t = tb + u;
        oq[u] = -1;
        vq[u] = 0.0;
        if (t < t1) {  // warp-uniform
          const int c = t - lane;
          const bool started = c >= 0;
          const bool active = lane_in & started & (c < C);
          const int cc = min(max(c, 0), C - 1);
          const int sidx = lane * 32 + (cc & 31);
          const int code = ((cc >> 5) == kg ? ccur : cprev)[sidx];
          const double nhl = __shfl_up_sync(0xffffffffu, hl, 1);
          const bool anchor = lane0 & (c == 0);
          const bool isbal = active & (code == 0) & !anchor;
          unsigned long long bw = 0;
          if (isbal) {
            const unsigned long long j = bj++;
            const bool edge = (j & 7) == 7;  // the value's second word opens the next half
            if (edge) cp_async_wait<0>();
            const unsigned long long lo = bring[j & 15], hi = bring[(j + 1) & 15];
            bw = bsh ? ((lo >> bsh) | (hi << (64 - bsh))) : lo;
            if (edge) issue8(j + 9);  // the half just consumed takes words j + 9 .. j + 16
          }
          const double vhat = __dadd_rn(predict_steady<PK>(k, hl, nhl, pn, lane0),
                                        __dmul_rn((double)(code - center), two_ba));
          const double vh = anchor ? anc : (isbal ? __longlong_as_double((long long)bw) : vhat);
          vq[u] = vh;
          oq[u] = active ? ((cc >> 5) & 1) * 1024 + sidx : -1;
          pn = nhl;
          if (started) hl = vh;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const float y = t_inv_f32(vq[u], zthr, bnd, lgp, lgn, amb);
        if (oq[u] >= 0) S.out[0][oq[u]] = y;
      }
    }
    __syncwarp();
    // chunk kg - 1 is complete for every row: store it
    const int q = kg - 1;
    if (q >= 0 && q < nch) {
      const float *src = S.out[q & 1];
      const int c0 = q * 32, w = min(32, C - c0);
      if (vout && w == 32) {
#pragma unroll
        for (int j = 0; j < 8; j++) {  // 32 rows x 8 x 16 B: 4 rows per instruction
          const int r = j * 4 + (lane >> 3), pc = lane & 7;
          if (r < R)
            *reinterpret_cast<float4 *>(op + (int64_t)r * g.cols + c0 + pc * 4) =
                *reinterpret_cast<const float4 *>(src + r * 32 + pc * 4);
        }
      } else {
        for (int r = 0; r < R; r++)
          if (lane < w) op[(int64_t)r * g.cols + c0 + lane] = src[r * 32 + lane];
      }
    }
  }
  // the last chunk (completed by the final group)
  __syncwarp();
  {
    const int q = nch - 1;
    if (ngroups - 1 <= q) {  // not yet stored by the loop above
      const float *src = S.out[q & 1];
      const int c0 = q * 32, w = min(32, C - c0);
      for (int r = 0; r < R; r++)
        if (lane < w) op[(int64_t)r * g.cols + c0 + lane] = src[r * 32 + lane];
    }
  }
}

}  // namespace pmz
