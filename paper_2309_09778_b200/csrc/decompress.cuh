// decompress.cuh -- read_container record parsing and the canonical Huffman
// decode tables (decode_next); the decode itself is in
// dec4.cuh, decompress_block + inverse_map
// (transform.py:188-202) in dsc.cuh.
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
  int l0;     // shortest code length: its first symbol owns the all-zeros codeword
  int zsym;   // that symbol (canonical order)
  int pad;
  unsigned rcp[34];  // ceil(2^32 / l) for l >= 2 (exact floor(n / l) for n < 2^16)
  int sub_bits;      // second-level table: codewords of kLutBits+1 .. kLutBits+sub_bits bits
  int has_l2;        // 1 when every long codeword resolves in the second-level table
};

constexpr int kLutBits = 12;
constexpr unsigned kLut2Max = 1u << 16;  // second-level entries (256 KB of the decode workspace)
constexpr unsigned kLutL2Flag = 0x80000000u;
// Decode table entry: symbol [0,16), length [16,21), run divisor M [21,31)
// (M = ceil(1024 / l) for 2 <= l <= 16: floor(z / l) == (z * M) >> 10 for
// z <= 64; 0 = no run detection), bit 31 = second-level pointer.
__host__ __device__ __forceinline__ unsigned lut_entry(int l, unsigned sym) {
  const unsigned M = (l >= 2 && l <= 16) ? (1024u + (unsigned)l - 1u) / (unsigned)l : 0u;
  return sym | ((unsigned)l << 16) | (M << 21);
}

// D1: per-block record heads -> transform parameters and partition tables,
// one warp per block: the three CR log2 of derive_params on three lanes, the
// partition entries on all lanes with a warp scan of their byte lengths.
__global__ void k_dec_blocks(const uint8_t *__restrict__ buf, unsigned long long n, Geom g, KParams k,
                             const unsigned long long *__restrict__ boff, BlkP *blkp,
                             unsigned long long *part_bits, unsigned long long *part_off, double *anchors,
                             unsigned long long *bal_off, unsigned long long *pay_off,
                             unsigned long long *blk_nbal, WsStatus *st, pmz_np_fix *npfix) {
  count_launch(st);
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= g.nblocks) return;
  const unsigned long long o = boff[b];
  const BlockBox bb = block_box(g, b);
  const int64_t p0 = first_part(g, b);
  BlkP P{};
  P.trivial = 1;
  const unsigned long long head = 1 + 16 + 24ull * bb.np + 8;
  const uint8_t triv = o < n ? buf[o] : (uint8_t)2;
  if (triv == 1) {
    for (int i = lane; i < bb.np; i += 32) { part_bits[p0 + i] = 0; part_off[p0 + i] = 0; }
    if (lane == 0) { blkp[b] = P; blk_nbal[b] = 0; }
    return;
  }
  if (triv != 0 || o + head > n) {
    if (lane == 0) { set_err_at(st, PMZ_ERR_CORRUPT, 41, b); blkp[b] = P; }
    return;
  }
  const double fp = get_f64(buf + o + 1), fn = get_f64(buf + o + 9);
  if (!(fp > 0.0) || !(fn > 0.0) || !isfinite(fp) || !isfinite(fn)) {
    if (lane == 0) { set_err_at(st, PMZ_ERR_CORRUPT, 43, b); blkp[b] = P; }
    return;
  }
  // derive_params (compress.cuh) with its three log2 on lanes 0..2
  const double la = lane < 3 ? pmz_log2_d(lane == 0 ? fp : (lane == 1 ? fn : __dsub_rn(fp, k.eps0)), &st->unresolved)
                             : 0.0;
  const double lg_pos = __shfl_sync(0xffffffffu, la, 0), lg_neg = __shfl_sync(0xffffffffu, la, 1),
               lg_pe = __shfl_sync(0xffffffffu, la, 2);
  P.factor_pos = fp;
  P.factor_neg = fn;
  P.lg_pos = lg_pos;
  P.lg_neg = lg_neg;
  P.zero_code = __dadd_rn(-126.0, lg_pos);            // transform.py:121
  P.zero_threshold = __dadd_rn(P.zero_code, k.b_a);   // :122
  P.boundary = __dsub_rn(__dadd_rn(lg_neg, lg_pe), k.b_a);  // :123
  P.trivial = 0;
  if (lane == 0) {
    blkp[b] = P;
    if (npfix) np_fix_note(st, npfix, b, fn, __dsub_rn(fp, k.eps0));
  }
  unsigned long long pb = 0;  // payload bytes of the partitions before this chunk of 32
  bool bad = false;
  for (int i0 = 0; i0 < bb.np; i0 += 32) {
    const int i = i0 + lane;
    unsigned long long off = 0, len = 0;
    double anc = 0.0;
    if (i < bb.np) {
      const uint8_t *e = buf + o + 17 + 24ull * i;
      off = get_u64(e);
      len = get_u64(e + 8);
      anc = get_f64(e + 16);
    }
    const unsigned long long by = (len + 7) / 8;
    unsigned long long incl = by;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const unsigned long long excl = pb + incl - by;
    if (i < bb.np) {
      bad |= off != excl * 8;
      part_off[p0 + i] = excl;
      part_bits[p0 + i] = len;
      anchors[p0 + i] = anc;
    }
    pb += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) set_err_at(st, PMZ_ERR_CORRUPT, 44, b);
  if (lane == 0) {
    unsigned long long nb = get_u64(buf + o + 17 + 24ull * bb.np);
    if (nb > (unsigned long long)bb.br * bb.bc) { set_err_at(st, PMZ_ERR_CORRUPT, 45, b); nb = 0; }
    blk_nbal[b] = nb;
    bal_off[b] = o + head;
    pay_off[b] = o + head + 8 * nb;
    if (o + head + 8 * nb + pb > n) set_err(st, PMZ_ERR_TRUNCATED);
  }
}

// D2: canonical decode tables from the header's code lengths.
__global__ void __launch_bounds__(1024) k_dec_tables(const uint8_t *__restrict__ lens, int m, DecTab *tab,
                                                     uint16_t *sym, unsigned *lut, WsStatus *st) {
  count_launch(st);
  __shared__ unsigned cnt[34];
  __shared__ unsigned fill[34];
  const int n = 1 << m;
  if (threadIdx.x < 34) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    int l = lens[s];
    if (l > 32) set_err_at(st, PMZ_ERR_CORRUPT, 46, 0);
    else if (l) atomicAdd(&cnt[l], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Kraft equality with exact integer arithmetic
    unsigned long long kr = 0;
    int maxl = 0;
    for (int l = 1; l <= 32; l++) if (cnt[l]) maxl = l;
    for (int l = 1; l <= maxl; l++) kr += (unsigned long long)cnt[l] << (maxl - l);
    if (maxl == 0 || kr != (1ull << maxl)) set_err_at(st, PMZ_ERR_CORRUPT, 47, 0);
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
    int l0 = 0;
    for (int l = maxl; l >= 1; l--) if (cnt[l]) l0 = l;
    tab->l0 = l0;
    tab->rcp[0] = tab->rcp[1] = 0;
    for (int l = 2; l < 34; l++) tab->rcp[l] = (unsigned)(0x100000000ull / (unsigned long long)l) + 1u;
  }
  __syncthreads();
  // symbols in (length, code) order: slot = offset[l] + rank of the symbol
  // among equal-length symbols in index order (match_any ranks within a
  // warp, per-(warp, length) counts scanned across warps, 1024 per round)
  {
    __shared__ unsigned s_wl[32][34];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r0 = 0; r0 < n; r0 += blockDim.x) {
      const int i = r0 + threadIdx.x;
      const int l = i < n ? min((int)lens[i], 33) : 0;
      const unsigned peers = __match_any_sync(0xffffffffu, l);
      const unsigned rank = __popc(peers & ((1u << lane) - 1));
      for (int q = lane; q < 34; q += 32) s_wl[wid][q] = 0;
      __syncwarp();
      if (rank == 0) s_wl[wid][l] = __popc(peers);
      __syncthreads();
      if (threadIdx.x < 34) {
        unsigned acc = fill[threadIdx.x];
        for (int w = 0; w < nw; w++) { const unsigned t = s_wl[w][threadIdx.x]; s_wl[w][threadIdx.x] = acc; acc += t; }
        fill[threadIdx.x] = acc;
      }
      __syncthreads();
      if (i < n && l >= 1 && l <= 32) sym[s_wl[wid][l] + rank] = (uint16_t)i;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) tab->zsym = tab->l0 ? sym[tab->offset[tab->l0]] : 0;
  __syncthreads();
  // LUT over the next kLutBits bits: (len << 16) | symbol; prefixes of longer
  // codewords point into a second-level table over the next sub_bits bits
  // (kLutL2Flag | base), or are 0 (canonical search) when it would not fit.
  __shared__ unsigned s_nlong, s_fit;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  const int maxl = tab->maxl;
  const int sub_bits = maxl > kLutBits ? maxl - kLutBits : 0;
  for (int e = threadIdx.x; e < (1 << kLutBits); e += blockDim.x) {
    unsigned v = 0;
    for (int l = 1; l <= kLutBits && l <= maxl; l++) {
      unsigned code = (unsigned)e >> (kLutBits - l);
      unsigned d = code - tab->first[l];
      if (d < tab->count[l]) { v = lut_entry(l, sym[tab->offset[l] + d]); break; }
    }
    lut[e] = v;
  }
  __syncthreads();
  // long prefixes of a canonical code are the highest prefixes: count them
  for (int e = threadIdx.x; e < (1 << kLutBits); e += blockDim.x)
    if (lut[e] == 0) atomicAdd(&s_nlong, 1u);
  __syncthreads();
  const unsigned nlong = s_nlong;
  if (threadIdx.x == 0) {
    s_fit = sub_bits > 0 && sub_bits <= 16 && ((unsigned long long)nlong << sub_bits) <= kLut2Max;
    tab->sub_bits = sub_bits;
    tab->has_l2 = (int)s_fit;
  }
  __syncthreads();
  if (s_fit) {
    const unsigned p0 = (1u << kLutBits) - nlong;  // first long prefix
    const unsigned per = 1u << sub_bits, total = nlong << sub_bits;
    for (unsigned i = threadIdx.x; i < total; i += blockDim.x) {
      const unsigned pre = p0 + i / per, j = i % per;
      const unsigned long long bits = ((unsigned long long)pre << sub_bits) | j;  // maxl bits
      unsigned v = 0;
      for (int l = kLutBits + 1; l <= maxl; l++) {
        const unsigned code = (unsigned)(bits >> (maxl - l));
        const unsigned d = code - tab->first[l];
        if (d < tab->count[l]) { v = lut_entry(l, sym[tab->offset[l] + d]); break; }
      }
      lut[(1u << kLutBits) + i] = v;
    }
    __syncthreads();
    for (unsigned e = p0 + threadIdx.x; e < (1u << kLutBits); e += blockDim.x)
      lut[e] = kLutL2Flag | ((e - p0) << sub_bits);
  }
}

// MSB-first bit stream over a byte-aligned substream, read as aligned 32-bit
// words (bytes beyond the substream read as zero, never past the buffer end).
struct BitSrc {
  const uint8_t *base;     // 4-byte aligned address <= substream start
  unsigned adj;            // bit offset of the substream start from `base`
  unsigned long long nbits;
  const uint8_t *end;      // one past the last readable byte of the buffer
  __device__ __forceinline__ unsigned word(unsigned long long wi) const {
    const uint8_t *a = base + 4 * wi;
    unsigned v;
    if (a + 4 <= end) v = __ldg(reinterpret_cast<const unsigned *>(a));
    else {
      v = 0;
      for (int i = 0; i < 4; i++) v |= (a + i < end ? (unsigned)__ldg(a + i) : 0u) << (8 * i);
    }
    return __byte_perm(v, 0, 0x0123);  // big-endian bit order
  }
  // 64 bits starting at stream bit `pos`; bits at or beyond nbits are zero
  __device__ __forceinline__ unsigned long long window(unsigned long long pos) const {
    const unsigned long long q = pos + adj;
    const unsigned long long wi = q >> 5;
    const unsigned sh = (unsigned)(q & 31);
    const unsigned long long hi = ((unsigned long long)word(wi) << 32) | word(wi + 1);
    unsigned long long w = sh ? (hi << sh) | (word(wi + 2) >> (32 - sh)) : hi;
    const unsigned long long left = nbits > pos ? nbits - pos : 0;
    if (left < 64) w &= left ? (~0ull << (64 - left)) : 0ull;
    return w;
  }
};

}  // namespace pmz
