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
    int l0 = 0;
    for (int l = maxl; l >= 1; l--) if (cnt[l]) l0 = l;
    tab->l0 = l0;
    // symbols in (length, code) order -- sequential, n <= 65536
    for (int s = 0; s < n; s++) { int l = lens[s]; if (l && l <= 32) sym[fill[l]++] = (uint16_t)s; }
    tab->zsym = l0 ? sym[tab->offset[l0]] : 0;
    tab->rcp[0] = tab->rcp[1] = 0;
    for (int l = 2; l < 34; l++) tab->rcp[l] = (unsigned)(0x100000000ull / (unsigned long long)l) + 1u;
  }
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

// One codeword at `pos` (LUT for <= kLutBits, canonical search beyond).
__device__ __forceinline__ bool decode_sym(unsigned long long win, const unsigned *__restrict__ lut, const DecTab &tab,
                                           const uint16_t *__restrict__ sym, int &s, int &l) {
  const unsigned w32 = (unsigned)(win >> 32);
  const unsigned e = lut[w32 >> (32 - kLutBits)];
  if (e) {
    l = (int)(e >> 16);
    s = (int)(e & 0xffff);
    return true;
  }
  for (int ll = kLutBits + 1; ll <= tab.maxl; ll++) {
    const unsigned code = w32 >> (32 - ll);
    const unsigned d = code - tab.first[ll];
    if (d < tab.count[ll]) {
      s = sym[tab.offset[ll] + d];
      l = ll;
      return true;
    }
  }
  return false;
}

struct DecOut { unsigned long long end; unsigned cnt; unsigned zeros; int err; };

// Big-endian 32-bit words of the substream staged in shared memory (word i =
// stream bytes 4i..4i+3); two extra zero words make every 64-bit window safe.
struct SmemBits {
  const unsigned *w;
  __device__ __forceinline__ unsigned win32(unsigned pos) const {
    const unsigned i = pos >> 5, sh = pos & 31;
    return __funnelshift_l(w[i + 1], w[i], sh);
  }
  __device__ __forceinline__ unsigned long long win64(unsigned pos) const {
    const unsigned i = pos >> 5, sh = pos & 31;
    const unsigned hi = __funnelshift_l(w[i + 1], w[i], sh), lo = __funnelshift_l(w[i + 2], w[i + 1], sh);
    return ((unsigned long long)hi << 32) | lo;
  }
};

// Same interface reading the substream straight from global memory (used for
// substreams larger than the shared-memory staging buffer).
struct GlobBits {
  BitSrc bs;
  __device__ __forceinline__ unsigned win32(unsigned pos) const { return (unsigned)(bs.window(pos) >> 32); }
  __device__ __forceinline__ unsigned long long win64(unsigned pos) const { return bs.window(pos); }
};

// Decode one codeword (+ its back-to-back repetitions) at `cur`.
// Returns false on an invalid prefix.  k = number of identical codewords.
template <class Bits>
__device__ __forceinline__ bool decode_run(const Bits &sb, unsigned cur, unsigned stop, unsigned nbits,
                                           const unsigned *__restrict__ lut, const DecTab &tab,
                                           const uint16_t *__restrict__ sym, int &s, int &l, unsigned &k) {
  const unsigned w = sb.win32(cur);
  const unsigned e = lut[w >> (32 - kLutBits)];
  if (e) {
    l = (int)(e >> 16);
    s = (int)(e & 0xffff);
  } else {
    s = -1;
    for (int ll = kLutBits + 1; ll <= tab.maxl; ll++) {
      const unsigned d = (w >> (32 - ll)) - tab.first[ll];
      if (d < tab.count[ll]) { s = sym[tab.offset[ll] + d]; l = ll; break; }
    }
    if (s < 0) return false;
  }
  k = 1;
  // cheap test on the window already in registers: does the next codeword repeat?
  if (l <= 16 && ((w << l) >> (32 - l)) == (w >> (32 - l))) {
    const unsigned cw = w >> (32 - l);
    const unsigned long long nx = sb.win64(cur);
    unsigned long long pat = (unsigned long long)cw << (64 - l);
    pat |= pat >> l;
    pat |= pat >> (2 * l);
    pat |= pat >> (4 * l);
    if (4 * l < 32) pat |= pat >> (8 * l);
    const unsigned long long x = nx ^ pat;
    const unsigned z = x ? (unsigned)__clzll((long long)x) : 64u;
    const unsigned rl = tab.rcp[l];
    auto divl = [&](unsigned n) { return l == 1 ? n : __umulhi(n, rl); };
    unsigned kk = divl(z);
    if (cur + (kk - 1) * l >= stop) kk = divl(stop - cur + l - 1);  // only codewords starting before stop
    if (cur + kk * l > nbits) kk = divl(nbits - cur);
    k = max(kk, 1u);
  }
  return true;
}

// Phase 3 helper: decode [pos, stop) and store the symbols at raster indices
// idx0+1.. of the partition (the anchor owns raster index 0).
template <class Bits>
__device__ __forceinline__ DecOut write_span(const Bits &sb, unsigned nbits, unsigned pos, unsigned stop,
                                            const unsigned *__restrict__ lut, const DecTab &tab,
                                            const uint16_t *__restrict__ sym, unsigned limit,
                                            uint16_t *__restrict__ dst, unsigned idx0, int C, int64_t ld) {
  DecOut o{pos, 0u, 0u, 0};
  unsigned idx = idx0 + 1;
  int r = (int)(idx / (unsigned)C), c = (int)(idx - (unsigned)r * C);
  unsigned cur = pos;
  while (cur < stop) {
    if (cur >= nbits) { o.err = PMZ_ERR_TRUNCATED; break; }
    int s, l;
    unsigned k;
    if (!decode_run(sb, cur, stop, nbits, lut, tab, sym, s, l, k)) { o.err = PMZ_ERR_INVALID_PREFIX; break; }
    if (cur + l > nbits) { o.err = PMZ_ERR_TRUNCATED; break; }
    if (o.cnt + k > limit) { o.err = PMZ_ERR_CORRUPT; break; }
    for (unsigned j = 0; j < k; j++) {
      dst[r * ld + c] = (uint16_t)s;
      if (++c == C) { c = 0; r++; }
    }
    if (s == 0) o.zeros += k;
    o.cnt += k;
    cur += k * l;
  }
  o.end = cur;
  return o;
}

constexpr int kStageSmall = 2051;  // 8 KB staged substream + slack words (common case)
constexpr int kStageLarge = 8195;  // 32 KB: 8191 codes x 32 bits + slack (second pass)
constexpr int kVisBits = 128;      // merge-detection window after each span start
constexpr int kMaxEntry = 32;      // entry offsets per span (>= max code length)

#ifdef PMZ_DEC_PROFILE
__device__ long long g_dec_prof[65536][6];
#define DEC_STAMP(i) if ((threadIdx.x & 31) == 0 && pid < 65536) g_dec_prof[pid][i] = clock64();
#else
#define DEC_STAMP(i)
#endif

constexpr unsigned kBadExit = 0xffffffffu;

struct DecWarpSmem {
  unsigned exit_[32][kMaxEntry + 1];  // per span, per entry offset: exit boundary (kBadExit: failed)
  uint16_t cnt_[32][kMaxEntry + 2];   // ... and symbol count
  uint16_t vis[32][kVisBits + 2];     // per span: (path+1) << 10 | rank of visited boundaries near the start
  unsigned start[33];                 // true span starts; [32] = final exit
  unsigned tcnt[32];                  // true symbol counts
  int err;
};

__device__ __forceinline__ unsigned bm_rank(const unsigned *bm, unsigned from, unsigned to) {
  // number of set bits in [from, to)
  unsigned r = 0;
  const unsigned w0 = from >> 5, w1 = to >> 5;
  for (unsigned wi = w0; wi <= w1; wi++) {
    unsigned word = bm[wi];
    if (wi == w0) word &= ~0u << (from & 31);
    if (wi == w1) word &= (to & 31) ? ((1u << (to & 31)) - 1) : 0u;
    r += __popc(word);
  }
  return r;
}

// Phases of the partition decode over a bit source (smem or global).
//  1. transfer function: every lane computes, for each entry offset o in
//     [0, maxlen) of its span [i L/32, (i+1) L/32), the exit boundary and the
//     symbol count of the path starting at span_start + o.  Paths merge when
//     they land on a boundary visited by an earlier path (any path near the
//     span start, path 0 anywhere in the span), so typical spans cost about
//     one decode; periodic / fixed-length streams, which never
//     self-synchronize, cost at most one decode per bit of the span.
//  2. lane 0 chains the spans: entry of span i = exit of span i-1 (32 lookups);
//  3. every lane decodes its span from the true entry and stores the symbols.
template <class Bits>
__device__ __forceinline__ void decode_partition(const Bits &sb, unsigned L, unsigned nsym, int C, int64_t ld,
                                                 uint16_t *dst, DecWarpSmem &S, unsigned *bm, unsigned bm_words,
                                                 const unsigned *lut, const DecTab &tab, const uint16_t *sym,
                                                 unsigned &zeros_out, WsStatus *st, int64_t pid) {
  const int lane = threadIdx.x & 31;
  DEC_STAMP(1)
  const unsigned s_i = (unsigned)((unsigned long long)L * lane / 32);
  const unsigned s_n = (lane == 31) ? L : (unsigned)((unsigned long long)L * (lane + 1) / 32);
  const int D = min(tab.maxl, kMaxEntry);
  const bool use_bm = ((L + 31) >> 5) + 1 <= bm_words;
  if (use_bm) {
    for (unsigned w = s_i >> 5; w <= (s_n >> 5); w++) bm[w] = 0;  // overlapping edge words are zeroed twice
    __syncwarp();
    // ---- fast path: speculative path 0 marks its boundaries; every lane then
    // decodes from its assumed entry (the previous lane's path-0 exit) only
    // until it meets path 0.  Valid when every lane meets it.
    unsigned cur = s_i, cnt0 = 0;
    bool bad = false;
    while (cur < s_n) {
      atomicOr(&bm[cur >> 5], 1u << (cur & 31));
      if (cur >= L) { bad = true; break; }
      int s, l;
      unsigned k;
      if (!decode_run(sb, cur, s_n, L, lut, tab, sym, s, l, k) || cur + l > L) { bad = true; break; }
      for (unsigned j = 1; j < k; j++) {
        const unsigned q = cur + j * l;
        atomicOr(&bm[q >> 5], 1u << (q & 31));
      }
      cnt0 += k;
      cur += k * l;
    }
    const unsigned exit0 = bad ? kBadExit : cur;
    __syncwarp();
    unsigned entry = __shfl_up_sync(0xffffffffu, exit0, 1);
    if (lane == 0) entry = 0;
    bool ok = entry != kBadExit && !bad;
    unsigned ex = entry, ct = 0;
    if (ok && entry < s_n) {
      unsigned c2 = entry, n2 = 0;
      bool met = false;
      while (c2 < s_n) {
        if ((bm[c2 >> 5] >> (c2 & 31)) & 1) { met = true; break; }
        int s, l;
        unsigned k;
        if (c2 >= L || !decode_run(sb, c2, s_n, L, lut, tab, sym, s, l, k) || c2 + l > L) break;
        // stop inside a run where it meets path 0
        unsigned kk = k;
        for (unsigned j = 1; j < k; j++) {
          const unsigned q = c2 + j * l;
          if ((bm[q >> 5] >> (q & 31)) & 1) { kk = j; break; }
        }
        n2 += kk;
        c2 += kk * l;
      }
      if (met) {
        ex = exit0;
        ct = n2 + (cnt0 - bm_rank(bm, s_i, c2));
      } else {
        ok = false;
      }
    }
    if (__all_sync(0xffffffffu, ok)) {
      S.start[lane] = entry;
      S.tcnt[lane] = ct;
      if (lane == 31) S.start[32] = ex;
      if (lane == 0) S.err = 0;
      __syncwarp();
      goto place;
    }
  }
  for (int q = 0; q < kVisBits; q++) S.vis[lane][q] = 0;
  if (use_bm)
    for (unsigned w = s_i >> 5; w <= (s_n >> 5); w++) bm[w] = 0;
  __syncwarp();
  for (int o = 0; o < D; o++) {
    unsigned cur = s_i + o, cnt = 0;
    int merged = -1;  // path index merged into, D = path 0 via the bitmap
    unsigned mrank = 0;
    bool bad = false;
    while (cur < s_n) {
      const unsigned off = cur - s_i;
      if (off < (unsigned)kVisBits) {
        const unsigned v = S.vis[lane][off];
        if (v) { merged = (int)(v >> 10) - 1; mrank = v & 1023u; break; }
        S.vis[lane][off] = (uint16_t)(((o + 1) << 10) | min(cnt, 1023u));
      } else if (o > 0 && use_bm && ((bm[cur >> 5] >> (cur & 31)) & 1)) {
        merged = D;  // path 0's boundary: rank by popcount below
        break;
      }
      if (o == 0 && use_bm) atomicOr(&bm[cur >> 5], 1u << (cur & 31));
      if (cur >= L) { bad = true; break; }
      int s, l;
      unsigned k;
      if (!decode_run(sb, cur, s_n, L, lut, tab, sym, s, l, k) || cur + l > L) { bad = true; break; }
      for (unsigned j = 1; j < k; j++) {
        const unsigned q = cur + j * l, qo = q - s_i;
        if (qo < (unsigned)kVisBits) {
          if (!S.vis[lane][qo]) S.vis[lane][qo] = (uint16_t)(((o + 1) << 10) | min(cnt + j, 1023u));
        } else if (o > 0 && use_bm && ((bm[q >> 5] >> (q & 31)) & 1)) {
          cnt += j;
          cur = q;
          merged = D;
          break;
        }
        if (o == 0 && use_bm) atomicOr(&bm[q >> 5], 1u << (q & 31));
      }
      if (merged == D) break;
      cnt += k;
      cur += k * l;
    }
    if (bad) {
      S.exit_[lane][o] = kBadExit;
      S.cnt_[lane][o] = 0;
    } else if (merged == D) {
      const unsigned r0 = bm_rank(bm, s_i, cur);
      S.exit_[lane][o] = S.exit_[lane][0];
      S.cnt_[lane][o] = (uint16_t)(cnt + (S.cnt_[lane][0] - r0));
    } else if (merged >= 0 && mrank < 1023u) {
      S.exit_[lane][o] = S.exit_[lane][merged];
      S.cnt_[lane][o] = (uint16_t)(cnt + (S.cnt_[lane][merged] - mrank));
    } else {
      S.exit_[lane][o] = cur;
      S.cnt_[lane][o] = (uint16_t)cnt;
    }
  }
  __syncwarp();
  DEC_STAMP(2)
  if (lane == 0) {
    unsigned T = 0;
    int e2 = 0;
    for (int i = 0; i < 32; i++) {
      const unsigned si = (unsigned)((unsigned long long)L * i / 32);
      const unsigned sn = (i == 31) ? L : (unsigned)((unsigned long long)L * (i + 1) / 32);
      S.start[i] = T;
      if (T >= sn) { S.tcnt[i] = 0; continue; }  // one codeword covers the whole span
      const unsigned o = T - si;
      if (o >= (unsigned)D || S.exit_[i][o] == kBadExit) { e2 = PMZ_ERR_CORRUPT; T = L + 1; break; }
      S.tcnt[i] = S.cnt_[i][o];
      T = S.exit_[i][o];
    }
    S.start[32] = T;
    S.err = e2;
  }
  __syncwarp();
place:
  DEC_STAMP(3)
  const unsigned start = S.start[lane], cnt = S.tcnt[lane];
  unsigned incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned zeros = 0;
  if (!S.err && total == nsym && S.start[32] == L) {
    DecOut w = write_span(sb, L, start, s_n, lut, tab, sym, cnt, dst, incl - cnt, C, ld);
    zeros = w.zeros;
    if (__any_sync(0xffffffffu, w.err != 0 || w.cnt != cnt) && lane == 0) set_err(st, PMZ_ERR_CORRUPT);
  } else if (lane == 0) {
    set_err(st, S.err ? S.err : (total < nsym ? PMZ_ERR_TRUNCATED : PMZ_ERR_CORRUPT));
  }
  DEC_STAMP(4)
  zeros_out = zeros;
}

template <int NW, bool LARGE>
struct DecCfg {
  static constexpr int kStage = LARGE ? kStageLarge : kStageSmall;
  static constexpr int kBm = kStage;  // one bitmap word per staged word
  static constexpr size_t kPerWarp = sizeof(DecWarpSmem) + 4ull * (kStage + kBm);
  static constexpr size_t kSmem = kPerWarp * NW;
};

// D3: parallel Huffman decode, one warp per partition substream (see
// decode_partition).  The common pass (LARGE = false) stages substreams of up
// to 8 KB; longer ones are appended to a work list served by the LARGE pass.
template <int NW, bool LARGE>
__global__ void __launch_bounds__(NW * 32) k_decode(const uint8_t *__restrict__ buf, Geom g,
                                                    const BlkP *__restrict__ blkp, const DecTab *__restrict__ tab,
                                                    const uint16_t *__restrict__ sym, const unsigned *__restrict__ lut,
                                                    const unsigned long long *__restrict__ part_bits,
                                                    const unsigned long long *__restrict__ part_off,
                                                    const unsigned long long *__restrict__ pay_off,
                                                    uint16_t *codes, unsigned long long *part_zeros,
                                                    unsigned *large_list, WsStatus *st) {
  using Cfg = DecCfg<NW, LARGE>;
  __shared__ unsigned s_lut[1 << kLutBits];
  __shared__ DecTab s_tab;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (LARGE && large_list[0] == 0) return;
  for (int i = threadIdx.x; i < (1 << kLutBits); i += blockDim.x) s_lut[i] = lut[i];
  if (threadIdx.x == 0) s_tab = *tab;
  __syncthreads();
  unsigned char *mine = dyn_raw + Cfg::kPerWarp * warp;
  DecWarpSmem &S = *reinterpret_cast<DecWarpSmem *>(mine);
  unsigned *stg = reinterpret_cast<unsigned *>(mine + sizeof(DecWarpSmem));
  unsigned *bm = stg + Cfg::kStage;
  const int64_t nwork = LARGE ? (int64_t)large_list[0] : g.nparts;
  for (int64_t item = (int64_t)blockIdx.x * NW + warp; item < nwork; item += (int64_t)gridDim.x * NW) {
    const int64_t p = LARGE ? (int64_t)large_list[1 + item] : item;
    int64_t b;
    int pi;
    part_of(g, p, b, pi);
    if (blkp[b].trivial) {
      if (lane == 0) part_zeros[p] = 0;
      continue;
    }
    const BlockBox bb = block_box(g, b);
    const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
    const unsigned nsym = (unsigned)(R * C - 1);
    const unsigned long long L64 = part_bits[p];
    const unsigned long long nw64 = (((L64 + 7) >> 3) + 3) >> 2;
    if (nw64 + 3 > (unsigned long long)Cfg::kStage) {
      if (!LARGE) {
        if (lane == 0) large_list[1 + atomicAdd(&large_list[0], 1u)] = (unsigned)p;
      } else if (lane == 0) {
        set_err(st, PMZ_ERR_CORRUPT);  // longer than any valid substream
      }
      continue;
    }
    const unsigned L = (unsigned)L64;
    const uint8_t *src = buf + pay_off[b] + part_off[p];
    uint16_t *dst = codes + (bb.r0 + pr0) * g.cols + bb.c0;
    if (lane == 0) S.err = 0;
    unsigned zeros = 0;
    const unsigned nbytes = (L + 7) >> 3, nw = (nbytes + 3) >> 2;
    { const int64_t pid = p; DEC_STAMP(0) }
    // stage the substream as big-endian words (+ zero slack words)
    for (unsigned i = lane; i < nw + 3; i += 32) {
      unsigned v = 0;
      if (i < nw) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const unsigned by = 4 * i + q;
          v = (v << 8) | (by < nbytes ? (unsigned)__ldg(src + by) : 0u);
        }
      }
      stg[i] = v;
    }
    __syncwarp();
    SmemBits sb{stg};
    decode_partition(sb, L, nsym, C, g.cols, dst, S, bm, (unsigned)Cfg::kBm, s_lut, s_tab, sym, zeros, st, p);
    for (int d = 16; d > 0; d >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, d);
    if (lane == 0) part_zeros[p] = zeros;
    __syncwarp();
  }
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
