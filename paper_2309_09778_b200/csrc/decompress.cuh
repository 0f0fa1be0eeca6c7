// decompress.cuh -- read_container record parsing, canonical Huffman decode
// (decode_next) and decompress_block as a
// reconstructed-surface wavefront + inverse_map (transform.py:188-202).
#pragma once
#include "common.cuh"
#include "compress.cuh"

namespace pmz {

__device__ __forceinline__ unsigned long long get_u64(const uint8_t *p) {
  unsigned long long v = 0;
#pragma unroll
  for (int i = 7; i >= 0; i--) v = (v << 8) | p[i];
  return v;
}
__device__ __forceinline__ double get_f64(const uint8_t *p) { return __longlong_as_double((long long)get_u64(p)); }

struct DecTab {
  unsigned first[34], count[34], offset[34];
  int maxl;
  int pad;
};

constexpr int kLutBits = 12;

// D1: per-block record heads -> transform parameters and partition tables.
__global__ void k_dec_blocks(const uint8_t *__restrict__ buf, unsigned long long n, Geom g, KParams k,
                             const unsigned long long *__restrict__ boff, BlkP *blkp,
                             unsigned long long *part_bits, unsigned long long *part_off, double *anchors,
                             unsigned long long *bal_off, unsigned long long *pay_off,
                             unsigned long long *blk_nbal, WsStatus *st) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nblocks) return;
  unsigned long long o = boff[b];
  BlockBox bb = block_box(g, b);
  int64_t p0 = first_part(g, b);
  BlkP P{};
  if (o >= n) { set_err(st, PMZ_ERR_CORRUPT); P.trivial = 1; blkp[b] = P; return; }
  uint8_t triv = buf[o];
  if (triv == 1) {
    P.trivial = 1;
    blkp[b] = P;
    for (int i = 0; i < bb.np; i++) { part_bits[p0 + i] = 0; part_off[p0 + i] = 0; }
    blk_nbal[b] = 0;
    return;
  }
  unsigned long long head = 1 + 16 + 24ull * bb.np + 8;
  if (triv != 0 || o + head > n) { set_err(st, PMZ_ERR_CORRUPT); P.trivial = 1; blkp[b] = P; return; }
  double fp = get_f64(buf + o + 1), fn = get_f64(buf + o + 9);
  if (!(fp > 0.0) || !(fn > 0.0) || !isfinite(fp) || !isfinite(fn)) {
    set_err(st, PMZ_ERR_CORRUPT); P.trivial = 1; blkp[b] = P; return;
  }
  derive_params(fp, fn, k, P, &st->unresolved);
  blkp[b] = P;
  unsigned long long pb = 0;
  for (int i = 0; i < bb.np; i++) {
    const uint8_t *e = buf + o + 17 + 24ull * i;
    unsigned long long off = get_u64(e), len = get_u64(e + 8);
    if (off != pb * 8) set_err(st, PMZ_ERR_CORRUPT);
    part_off[p0 + i] = pb;
    part_bits[p0 + i] = len;
    anchors[p0 + i] = get_f64(e + 16);
    pb += (len + 7) / 8;
  }
  unsigned long long nb = get_u64(buf + o + 17 + 24ull * bb.np);
  if (nb > (unsigned long long)bb.br * bb.bc) { set_err(st, PMZ_ERR_CORRUPT); nb = 0; }
  blk_nbal[b] = nb;
  bal_off[b] = o + head;
  pay_off[b] = o + head + 8 * nb;
  if (o + head + 8 * nb + pb > n) set_err(st, PMZ_ERR_TRUNCATED);
}

// D2: canonical decode tables from the header's code lengths.
__global__ void __launch_bounds__(1024) k_dec_tables(const uint8_t *__restrict__ lens, int m, DecTab *tab,
                                                     uint16_t *sym, unsigned *lut, WsStatus *st) {
  __shared__ unsigned cnt[34];
  __shared__ unsigned fill[34];
  const int n = 1 << m;
  if (threadIdx.x < 34) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    int l = lens[s];
    if (l > 32) set_err(st, PMZ_ERR_CORRUPT);
    else if (l) atomicAdd(&cnt[l], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Kraft equality with exact integer arithmetic
    unsigned long long kr = 0;
    int maxl = 0;
    for (int l = 1; l <= 32; l++) if (cnt[l]) maxl = l;
    for (int l = 1; l <= maxl; l++) kr += (unsigned long long)cnt[l] << (maxl - l);
    if (maxl == 0 || kr != (1ull << maxl)) set_err(st, PMZ_ERR_CORRUPT);
    unsigned long long c = 0;
    unsigned o = 0;
    tab->first[0] = 0; tab->count[0] = 0; tab->offset[0] = 0;
    for (int l = 1; l <= 33; l++) {
      c = (c + (l >= 2 ? cnt[l - 1] : 0)) << 1;
      if (l == 1) c = 0;
      tab->first[l] = (unsigned)c;
      tab->count[l] = l <= 32 ? cnt[l] : 0;
      tab->offset[l] = o;
      fill[l] = o;
      o += l <= 32 ? cnt[l] : 0;
    }
    tab->maxl = maxl;
    // symbols in (length, code) order -- sequential, n <= 65536
    for (int s = 0; s < n; s++) { int l = lens[s]; if (l && l <= 32) sym[fill[l]++] = (uint16_t)s; }
  }
  __syncthreads();
  // LUT over the next kLutBits bits: (len << 16) | symbol, or 0 when len > kLutBits
  for (int e = threadIdx.x; e < (1 << kLutBits); e += blockDim.x) {
    unsigned v = 0;
    for (int l = 1; l <= kLutBits && l <= tab->maxl; l++) {
      unsigned code = (unsigned)e >> (kLutBits - l);
      unsigned d = code - tab->first[l];
      if (d < tab->count[l]) { v = ((unsigned)l << 16) | sym[tab->offset[l] + d]; break; }
    }
    lut[e] = v;
  }
}

// MSB-first bit reader over a byte stream with a 64-bit window.
struct BitReader {
  const uint8_t *p;
  unsigned long long nbits, pos;
  __device__ __forceinline__ unsigned peek32() const {
    // 32 bits starting at pos (zero beyond the end of the substream)
    unsigned long long byte = pos >> 3;
    unsigned long long nbytes = (nbits + 7) >> 3;
    unsigned long long w = 0;
#pragma unroll
    for (int i = 0; i < 5; i++) {
      unsigned long long bi = byte + i;
      w = (w << 8) | (bi < nbytes ? p[bi] : 0);
    }
    return (unsigned)(w >> (8 - (pos & 7)));
  }
};

// D3: decode one partition substream per warp (lane 0, sequential), codes to
// the grid, zero counts per partition.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_decode(const uint8_t *__restrict__ buf, Geom g,
                                                    const BlkP *__restrict__ blkp, const DecTab *__restrict__ tab,
                                                    const uint16_t *__restrict__ sym, const unsigned *__restrict__ lut,
                                                    const unsigned long long *__restrict__ part_bits,
                                                    const unsigned long long *__restrict__ part_off,
                                                    const unsigned long long *__restrict__ pay_off,
                                                    uint16_t *codes, unsigned long long *part_zeros, WsStatus *st) {
  __shared__ unsigned s_lut[1 << kLutBits];
  __shared__ DecTab s_tab;
  for (int i = threadIdx.x; i < (1 << kLutBits); i += blockDim.x) s_lut[i] = lut[i];
  if (threadIdx.x == 0) s_tab = *tab;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * NW + warp;
  if (p >= g.nparts || lane != 0) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) { part_zeros[p] = 0; return; }
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  BitReader br{buf + pay_off[b] + part_off[p], part_bits[p], 0};
  unsigned zeros = 0;
  bool bad = false;
  for (int r = 0; r < R && !bad; r++) {
    uint16_t *crow = codes + (bb.r0 + pr0 + r) * g.cols + bb.c0;
    for (int c = (r == 0 ? 1 : 0); c < C; c++) {
      if (br.pos >= br.nbits) { set_err(st, PMZ_ERR_TRUNCATED); bad = true; break; }
      unsigned w = br.peek32();
      unsigned e = s_lut[w >> (32 - kLutBits)];
      int s, l;
      if (e) {
        l = (int)(e >> 16);
        s = (int)(e & 0xffff);
      } else {
        s = -1;
        l = 0;
        for (int ll = kLutBits + 1; ll <= s_tab.maxl; ll++) {
          unsigned code = w >> (32 - ll);
          unsigned d = code - s_tab.first[ll];
          if (d < s_tab.count[ll]) { s = sym[s_tab.offset[ll] + d]; l = ll; break; }
        }
        if (s < 0) { set_err(st, PMZ_ERR_INVALID_PREFIX); bad = true; break; }
      }
      if (br.pos + l > br.nbits) { set_err(st, PMZ_ERR_TRUNCATED); bad = true; break; }
      br.pos += l;
      crow[c] = (uint16_t)s;
      zeros += (s == 0);
    }
  }
  if (!bad && br.pos != br.nbits) set_err(st, PMZ_ERR_CORRUPT);
  part_zeros[p] = zeros;
}

// D4: decompress_block wavefront per partition: code 0 ->
// next balance value, else predict(RECONSTRUCTED surface) + dequantize; then
// inverse_map -> f32 (D20).
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_reconstruct(const uint8_t *__restrict__ buf, Geom g, KParams k, int m,
                                                         const BlkP *__restrict__ blkp,
                                                         const uint16_t *__restrict__ codes,
                                                         const double *__restrict__ anchors,
                                                         const unsigned long long *__restrict__ part_zeros,
                                                         const unsigned long long *__restrict__ bal_off,
                                                         const unsigned long long *__restrict__ blk_nbal,
                                                         float *__restrict__ out, WsStatus *st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * NW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  const BlockBox bb = block_box(g, b);
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const int64_t grow = bb.r0 + pr0 + lane;
  float *orow = out + grow * g.cols + bb.c0;
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (lane < R)
      for (int c = 0; c < C; c++) orow[c] = 0.0f;
    return;
  }
  // balance index base: earlier partitions of the block + earlier rows
  const int64_t p0 = first_part(g, b);
  unsigned long long zb = 0, ztot = 0;
  for (int i = 0; i < bb.np; i++) {
    if (i < pi) zb += part_zeros[p0 + i];
    ztot += part_zeros[p0 + i];
  }
  if (ztot != blk_nbal[b]) {
    if (lane == 0 && pi == 0) set_err(st, ztot > blk_nbal[b] ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT);
    return;
  }
  const uint16_t *crow = codes + grow * g.cols + bb.c0;
  unsigned rz = 0;
  if (lane < R)
    for (int c = (lane == 0 ? 1 : 0); c < C; c++) rz += (crow[c] == 0);
  unsigned incl = rz;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  unsigned long long bidx = zb + (incl - rz);
  const uint8_t *bal = buf + bal_off[b];
  unsigned *amb = &st->unresolved;
  double hl = 0.0, hp = 0.0;
  for (int t = 0; t < C + R - 1; t++) {
    const double nhl = __shfl_up_sync(0xffffffffu, hl, 1), nhp = __shfl_up_sync(0xffffffffu, hp, 1);
    const int c = t - lane;
    if (lane < R && c >= 0 && c < C) {
      double vh;
      if (lane == 0 && c == 0) {
        vh = anchors[p];
      } else {
        int code = crow[c];
        if (code == 0) {
          vh = get_f64(bal + 8 * bidx);
          bidx++;
        } else {
          const bool hw = c > 0, hn = lane > 0;
          vh = __dadd_rn(predict(k, hw ? hl : 0.0, hn ? nhl : 0.0, (hw && hn) ? nhp : 0.0),
                         dequantize(code, k.two_ba, m));
        }
      }
      orow[c] = inv_f32(vh, P, amb);
      hp = hl;
      hl = vh;
    }
  }
}

}  // namespace pmz
