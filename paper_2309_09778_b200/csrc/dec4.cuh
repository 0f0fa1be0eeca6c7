// dec4.cuh -- canonical Huffman decode of the per-partition substreams
// (decode_next; substream layout SPEC.md:496), one CTA per
// partition, writing the codes in the partition-tiled layout (common.cuh).
//
// The decode is exact by construction -- it never relies on a Huffman code
// re-synchronising (the reference's skewed codebooks, e.g. 4-bit codewords
// 0000/0001/0010 for the three commonest codes, keep misaligned parses
// misaligned for thousands of bits, which made speculative decoders
// unbounded):
//   1. word maps: the substream is cut into 32-bit words; for a word, lane q
//      of a warp takes the codeword starting at bit q (one table lookup) and
//      pointer jumping over the lanes resolves, for EVERY entry offset
//      e in [0, 32), the offset at which the parse leaves the word and how
//      many codewords start inside it.  A warp composes the maps of the words
//      of a subsegment (one shuffle pair per word) into the subsegment's map
//      (entry offset -> exit offset, codeword count) -- bounded work: one
//      lookup per bit, no data-dependent iteration;
//   2. chain: from entry 0 the subsegment maps give every subsegment's true
//      entry and codeword count (one short dependent chain in shared memory);
//   3. write pass: thread j decodes its subsegment's codewords from the true
//      entry into a shared-memory copy of the partition's code tiles (runs of
//      a repeated codeword in one step), counting code-0 symbols (balance
//      points) per row; the tiles then go to global memory coalesced.
// Every code is complete (Kraft equality is checked when the tables are
// built, decompress.cuh) and no codeword is longer than 32 bits, so every bit
// position starts a codeword and a parse leaves a word within 32 bits.
#pragma once
#include "common.cuh"
#include "decompress.cuh"

namespace pmz {

#ifndef PMZ_D4_THREADS
#define PMZ_D4_THREADS 256
#endif
constexpr int kD4Threads = PMZ_D4_THREADS;  // threads = subsegments per partition
constexpr int kD4Warps = kD4Threads / 32;
constexpr int kD4Ras = 32 * 256;             // codes staged in shared memory in raster order (R * C <= 8192)
__device__ __forceinline__ unsigned d4_pad(unsigned i) { return i + ((i >> 6) << 1); }  // one bank word per 64 codes

#ifdef PMZ_D3_PROF
// per-partition phase timestamps (experiments only: tools/dec_bench.py)
__device__ unsigned long long g_d3prof[1 << 20];
__device__ __forceinline__ unsigned d3_smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#define D3P(i, v) do { if (threadIdx.x == 0 && p < (1 << 17)) g_d3prof[p * 8 + (i)] = (v); } while (0)
#else
#define D3P(i, v) do { } while (0)
#endif

struct D4Smem {
  union {
    uint16_t map[kD4Threads][32];          // subsegment maps: (count << 5) | exit offset, per entry offset
    uint16_t ras[kD4Ras + kD4Ras / 32];    // the partition's codes, raster order, padded (write pass)
  } u;
  unsigned ent[kD4Threads], cnt[kD4Threads];
  unsigned char on[kD4Threads], hit[kD4Threads];  // chain membership rounds (speculative path)
  unsigned zrow[32];
  unsigned wsum[kD4Warps];
  unsigned long long zb;                   // code-0 symbols of the earlier partitions of the block
  unsigned fin;                            // exit offset after the last word
};
constexpr size_t kD4Smem = sizeof(D4Smem);

// Starts of a run of k codewords of length l beginning at bit pos, OR-ed
// into the bitmap as one periodic mask (k * l <= 64): at most three words.
__device__ __forceinline__ void d4_mark_run(unsigned *bm, const unsigned long long *rep, unsigned pos, unsigned l,
                                            unsigned k) {
  // rep[l]: bits 0, l, 2l, ... below 64; k l <= 64, so (k - 1) l + 1 <= 64
  const unsigned long long m = rep[l] & (k >= 64 ? ~0ull : ((1ull << ((k - 1) * l + 1)) - 1ull));
  const unsigned off = pos & 31, w = pos >> 5;
  bm[w] |= (unsigned)(m << off);
  const unsigned long long hi = off ? (m >> (32 - off)) : (m >> 32);
  if (hi) {
    bm[w + 1] |= (unsigned)hi;
    if (hi >> 32) bm[w + 2] |= (unsigned)(hi >> 32);
  }
}

// ras[d4_pad(idx + j)] = s for j < k: contiguous inside each 64-code row of
// the padded raster; 4-byte stores of code pairs (the padding is even, so a
// pair is aligned iff its raster index is)
__device__ __forceinline__ void d4_fill(uint16_t *ras, unsigned idx, unsigned k, unsigned s) {
  const unsigned pair = s | (s << 16);
  const unsigned end = idx + k;
  while (idx < end) {
    const unsigned n = min(end, (idx | 63u) + 1u) - idx;  // inside this 64-code row
    uint16_t *d = ras + d4_pad(idx);
    unsigned j = 0;
    if (idx & 1u) d[j++] = (uint16_t)s;
    for (; j + 2 <= n; j += 2) *reinterpret_cast<unsigned *>(d + j) = pair;
    if (j < n) d[j] = (uint16_t)s;
    idx += n;
  }
}

// Decoupled look-back flags: code-0 count + 1 once known, kD4Poison when the
// partition failed (reset to 0 before every launch).
constexpr unsigned kD4Poison = 0xffffffffu;
__device__ __forceinline__ void d4_publish(unsigned *f, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

// Register bit reader at an arbitrary bit position of the substream.
struct D4Reader {
  unsigned long long buf;  // next stream bits, left-aligned
  int nb;                  // valid bits in buf (>= 32 after refill)
  unsigned wi;             // index of the prefetched word
  unsigned nxt;            // prefetched next word (off the dependency chain)
  __device__ __forceinline__ void seek(const BitSrc &src, unsigned pos) {
    const unsigned q = pos + src.adj;
    wi = q >> 5;
    const unsigned sh = q & 31;
    buf = (((unsigned long long)src.word(wi) << 32) | src.word(wi + 1)) << sh;
    nb = 64 - (int)sh;
    wi += 2;
    nxt = src.word(wi);
  }
  __device__ __forceinline__ void refill(const BitSrc &src) {
    if (nb < 32) {
      buf |= (unsigned long long)nxt << (32 - nb);
      nb += 32;
      nxt = src.word(++wi);
    }
  }
  __device__ __forceinline__ void skip(unsigned adv) {
    buf <<= adv;
    nb -= (int)adv;
  }
};

// Codeword at the top of `top` through the global tables (codewords longer
// than the shared first level): length, and the symbol through `sym_out`.
__device__ __forceinline__ unsigned d4_slow(unsigned top, const unsigned *__restrict__ lut,
                                         const DecTab &tab, const uint16_t *__restrict__ sym, unsigned &sym_out) {
  unsigned e = __ldg(lut + (top >> (32 - kLutBits)));
  if (e & kLutL2Flag) e = __ldg(lut + (1 << kLutBits) + (e & 0xffffu) + ((top << kLutBits) >> (32 - tab.sub_bits)));
  if (e == 0) {
    for (int ll = kLutBits + 1; ll <= tab.maxl; ll++) {
      const unsigned d = (top >> (32 - ll)) - tab.first[ll];
      if (d < tab.count[ll]) {
        sym_out = sym[tab.offset[ll] + d];
        return (unsigned)ll;
      }
    }
    sym_out = 0;
    return 32u;  // unreachable for a complete code
  }
  sym_out = e & 0xffffu;
  return (e >> 16) & 31u;
}

// Length of the codeword at the top of `top` (32 bits, left-aligned).
__device__ __forceinline__ unsigned d4_len(unsigned top, const uint8_t *__restrict__ len12,
                                           const unsigned *__restrict__ lut, const DecTab &tab,
                                           const uint16_t *__restrict__ sym) {
  const unsigned l = len12[top >> (32 - kLutBits)];
  if (__builtin_expect(l != 0, 1)) return l;
  unsigned sd;
  return d4_slow(top, lut, tab, sym, sd);
}

// Length l of the codeword at the top of the reader (nb >= 32 valid bits)
// and how many back-to-back repeats of it start within the next lim bits
// (k >= 1; a run is periodic with period l, clz(buf ^ (buf << l)) + l bits).
__device__ __forceinline__ unsigned d4_len_run(unsigned long long buf, int nb, unsigned lim,
                                               const uint8_t *len12, const unsigned *__restrict__ lut,
                                               const DecTab &tab, const uint16_t *__restrict__ sym, unsigned &l) {
  const unsigned top = (unsigned)(buf >> 32);
  l = len12[top >> (32 - kLutBits)];
  if (__builtin_expect(l == 0, 0)) {
    unsigned sd;
    l = d4_slow(top, lut, tab, sym, sd);
    return 1;
  }
  const unsigned long long xx = buf ^ (buf << l);
  const unsigned P = (xx ? (unsigned)__clzll((long long)xx) : 64u) + l;
  const unsigned z = min(min(P, (unsigned)nb), lim + l - 1u);  // codewords starting before lim
  return l == 1 ? z : max(__umulhi(z, tab.rcp[l]), 1u);
}

// The codeword at the top of the reader (nb >= 32 valid bits) and how many
// times it repeats back-to-back inside the valid bits (1 <= k <= lim).
__device__ __forceinline__ void d4_run(unsigned long long buf, int nb, unsigned lim, const uint8_t *len12,
                                       const uint16_t *sym12, const unsigned *__restrict__ lut, const DecTab &tab,
                                       const uint16_t *__restrict__ sym, unsigned &s, unsigned &l, unsigned &k) {
  const unsigned top = (unsigned)(buf >> 32);
  const unsigned i = top >> (32 - kLutBits);
  l = len12[i];
  if (__builtin_expect(l == 0, 0)) {
    l = d4_slow(top, lut, tab, sym, s);
    k = 1;
    return;
  }
  s = sym12[i];
  // buf is periodic with period l over its first clz(buf ^ (buf << l)) + l bits
  const unsigned long long x = buf ^ (buf << l);
  const unsigned P = (x ? (unsigned)__clzll((long long)x) : 64u) + l;
  const unsigned z = min(P, (unsigned)nb);
  k = l == 1 ? z : max(__umulhi(z, tab.rcp[l]), 1u);  // floor(z / l)
  k = min(k, lim);
}

__global__ void __launch_bounds__(kD4Threads, 6) k_decode4(const uint8_t *__restrict__ buf, unsigned long long buf_n,
                                                       Geom g, const BlkP *__restrict__ blkp,
                                                       const DecTab *__restrict__ tab,
                                                       const uint16_t *__restrict__ sym,
                                                       const unsigned *__restrict__ lut,
                                                       const unsigned long long *__restrict__ part_bits,
                                                       const unsigned long long *__restrict__ part_off,
                                                       const unsigned long long *__restrict__ pay_off,
                                                       const unsigned long long *__restrict__ bal_off,
                                                       const unsigned long long *__restrict__ blk_nbal,
                                                       int center, double two_ba, unsigned *zflag,
                                                       uint16_t *__restrict__ codes, double *__restrict__ vtile,
                                                       WsStatus *st) {
  constexpr int NS = kD4Threads;
  __shared__ DecTab s_tab;
  // first-level tables as static shared arrays: addressed directly (a
  // pointer into the dynamic block costs a generic-to-shared conversion per
  // lookup): symbol of the codeword on the next 12 bits, and its length (0:
  // longer than 12 bits, global tables)
  __shared__ uint16_t s_sym12[1 << kLutBits];
  __shared__ uint8_t s_len12[1 << kLutBits];
  __shared__ unsigned long long s_rep[33];  // s_rep[l]: bits 0, l, 2l, ... (a run's starts)
  extern __shared__ __align__(16) unsigned char dyn4[];
  D4Smem &W = *reinterpret_cast<D4Smem *>(dyn4);
  count_launch(st);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t p = blockIdx.x;
  if (t == 0) s_tab = *tab;
  if (t < 32) W.zrow[t] = 0;
  if (t <= 32) {
    unsigned long long r = 0;
    if (t >= 1)
      for (int q = 0; q < 64; q += t) r |= 1ull << q;
    s_rep[t] = r;
  }
  for (int i = t; i < (1 << kLutBits); i += NS) {
    const unsigned e = __ldg(lut + i);
    const bool direct = e != 0 && !(e & kLutL2Flag);
    s_len12[i] = direct ? (uint8_t)((e >> 16) & 31u) : (uint8_t)0;
    s_sym12[i] = (uint16_t)(e & 0xffffu);
  }
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) return;
  __syncthreads();
  const BlockBox bb = block_box(g, b);
  const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc;
  const unsigned nsym = (unsigned)(R * C - 1);
  const unsigned long long L64 = part_bits[p];
  if (L64 > 32ull * (nsym + 1ull)) {  // longer than any valid substream (codewords <= 32 bits)
    if (t == 0) {
      set_err_at(st, PMZ_ERR_CORRUPT, 1, p);
      d4_publish(zflag + p, kD4Poison);  // later partitions of the block must not wait forever
    }
    return;
  }
  const unsigned L = (unsigned)L64;
  D3P(0, clock64());
  D3P(7, ((unsigned long long)L64 << 16) | 0);
  BitSrc bs;
  {
    const uint8_t *src = buf + pay_off[b] + part_off[p];
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    bs.base = reinterpret_cast<const uint8_t *>(a & ~(uintptr_t)3);
    bs.adj = (unsigned)(8 * (a & 3));
    bs.nbits = L64;
    bs.end = buf + buf_n;
  }
  const unsigned nw = (L + 31) >> 5;            // 32-bit words of the substream
  const unsigned wps = (nw + NS - 1) / NS;      // words per subsegment

  // ---- 0. speculative decode (the cheap path, ~20x fewer instructions than
  // the word maps).  Thread t parses its subsegment [s_t, s_t+1) from s_t,
  // marking every codeword start in a bitmap; then it continues past its
  // subsegment ("overrun") until it lands on a marked start of a later
  // subsegment -- from there that subsegment's parse IS the continuation --
  // or the end.  The true parse is thread 0's, its overrun, the parse +
  // overrun of the thread it landed in, and so on (chain membership rounds).
  // A parse that has not synchronised within kD4Cap subsegments (the
  // reference's skewed codebooks can keep misaligned parses misaligned for
  // thousands of bits) sends the whole partition to the exact word maps. ----
  constexpr unsigned kBmWords = (unsigned)(sizeof(W.u) / 4);
#ifndef PMZ_D4_CAP
#define PMZ_D4_CAP 16
#endif
  constexpr unsigned kD4Cap = PMZ_D4_CAP;
  bool use_maps = nw + 2 > kBmWords;
  if (!use_maps) {
    unsigned *bm = reinterpret_cast<unsigned *>(&W.u);
    const unsigned seg = 32u * wps;
    const unsigned s_i = min(L, seg * (unsigned)t), s_n = min(L, seg * (unsigned)(t + 1));
    for (unsigned q = min(nw, wps * (unsigned)t); q < min(nw, wps * (unsigned)(t + 1)); q++) bm[q] = 0;
    if (t == 0) bm[nw] = bm[nw + 1] = 0;  // window reads past the last word
    unsigned pos = s_i, nsp = 0;
    if (s_i < s_n) {
      D4Reader rd;
      rd.seek(bs, s_i);
      while (pos < s_n) {
        rd.refill(bs);
        unsigned l;
        const unsigned k = d4_len_run(rd.buf, rd.nb, s_n - pos, s_len12, lut, s_tab, sym, l);
        d4_mark_run(bm, s_rep, pos, l, k);  // own words only: every start < s_n
        rd.skip(k * l);
        pos += k * l;
        nsp += k;
      }
    }
    __syncthreads();  // every subsegment's starts are marked
    unsigned y = pos, nov = 0;
    bool hard = false;
    if (y < L) {
      D4Reader rd;
      rd.seek(bs, y);
      const unsigned cap = s_n + kD4Cap * seg;
      while (y < L) {
        const unsigned wq = y >> 5, off = y & 31;
        unsigned long long win = ((unsigned long long)bm[wq] | ((unsigned long long)bm[wq + 1] << 32)) >> off;
        if (off) win |= (unsigned long long)bm[wq + 2] << (64 - off);
        if (win & 1ull) break;  // landed on a later subsegment's parse
        if (y >= cap) {
          hard = true;
          break;
        }
        rd.refill(bs);
        unsigned l;
        unsigned k = d4_len_run(rd.buf, rd.nb, L - y, s_len12, lut, s_tab, sym, l);
        if (k > 1) {  // a run stops at its first codeword that starts on a marked position
          unsigned long long per = 0;
          const unsigned n = (k - 1) * l + 1;  // <= 64 (k l <= 64)
          per = s_rep[l] & (n >= 64 ? ~0ull : ((1ull << n) - 1ull)) & ~1ull;
          const unsigned long long hm = win & per;
          if (hm) k = ((unsigned)__ffsll((long long)hm) - 1u) / l;
        }
        rd.skip(k * l);
        y += k * l;
        nov += k;
      }
    }
    use_maps = __syncthreads_or(hard);
    if (!use_maps) {
      // chain membership: S_0 = all threads, S_{i+1} = {0} + landing threads
      // of S_i: decreasing supersets of the true chain (usually stable after
      // one round); the round that changes nothing stored the entries
      const unsigned nxt = y >= L ? (unsigned)NS : min(y / seg, (unsigned)NS);
      W.on[t] = 1;
      for (;;) {
        W.hit[t] = t == 0;
        __syncthreads();
        if (W.on[t] && nxt < (unsigned)NS) {
          W.hit[nxt] = 1;
          W.ent[nxt] = y;
        }
        __syncthreads();
        const bool ch = W.hit[t] != W.on[t];
        W.on[t] = W.hit[t];
        if (!__syncthreads_or(ch)) break;
      }
      const bool on = W.on[t];
      const unsigned e = t == 0 ? 0u : W.ent[t];
      unsigned c = 0;
      if (on) {  // spec codewords from the entry on (rank = marked starts before it) + the overrun
        unsigned rk = 0;
        for (unsigned q = s_i >> 5; q < (e >> 5); q++) rk += __popc(bm[q]);
        if (e & 31) rk += __popc(bm[e >> 5] & ((1u << (e & 31)) - 1u));
        c = nsp - rk + nov;
      }
      const bool bad = on && nxt == (unsigned)NS && y != L;
      const bool anybad = __syncthreads_or(bad);
      W.ent[t] = on ? e : L;
      W.cnt[t] = c;
      if (t == 0) W.fin = anybad ? 0xffffffffu : (L & 31u);
      __syncthreads();
    }
  }
  D3P(6, use_maps ? 1ull : 0ull);
  if (use_maps) {
  // ---- 1. subsegment maps (warp w: subsegments 32 w .. 32 w + 31 = the
  // contiguous words [wa, wb)).  Stream words arrive in coalesced batches of
  // 32 (lane i holds word bbase + i, the next batch is in flight) and are
  // broadcast by shuffles; two words per step for instruction-level
  // parallelism.  A parse state is packed as (count << 8) | position, so a
  // pointer-jumping step or a composition is one shuffle; nj =
  // ceil(log2(32 / l0)) jumps resolve a word. ----
  {
    int nj = 0;
    while ((32 >> nj) > s_tab.l0) nj++;
    const unsigned wa = min(nw, (unsigned)(warp * 32) * wps), wb = min(nw, (unsigned)(warp * 32 + 32) * wps);
    unsigned bbase = wa;
    auto sword = [&](unsigned i) -> unsigned { return __funnelshift_l(bs.word(i + 1), bs.word(i), bs.adj); };
    unsigned cur = sword(bbase + lane), nxb = sword(bbase + 32 + lane);
    auto sw = [&](unsigned i) -> unsigned {  // stream word i, i in [bbase, bbase + 64)
      const unsigned d = i - bbase;
      const unsigned v0 = __shfl_sync(0xffffffffu, cur, d & 31), v1 = __shfl_sync(0xffffffffu, nxb, d & 31);
      return d < 32 ? v0 : v1;
    };
    auto advance = [&](unsigned need) {  // keep stream word `need` inside the window
      if (need >= bbase + 64) {
        bbase += 32;
        cur = nxb;
        nxb = sword(bbase + 32 + lane);
      }
    };
    // word w's parse from bit `lane`: (count << 8) | position (>= 32: left the word at position - 32)
    auto word_init = [&](unsigned w, unsigned s0, unsigned s1) -> unsigned {
      const unsigned top = __funnelshift_l(s1, s0, (unsigned)lane);
      const bool in = 32u * w + (unsigned)lane < L;  // past the end: the offset carries over, nothing starts
      const unsigned l = d4_len(top, s_len12, lut, s_tab, sym);  // every lane (branch-free select below)
      return in ? ((unsigned)lane + l) | 0x100u : (unsigned)lane + 32u;
    };
    auto jump = [&](unsigned &pk) {
      const unsigned x = pk & 0xffu;
      const bool open = x < 32u;
      const unsigned v = __shfl_sync(0xffffffffu, pk, open ? x : (unsigned)lane);
      pk = open ? v + (pk & ~0xffu) : pk;
    };
    auto compose = [&](unsigned &F, unsigned pk) {  // entry -> F.pos in this word -> pk(F.pos) - 32 in the next
      const unsigned v = __shfl_sync(0xffffffffu, pk, F & 0xffu);
      F = v - 32u + (F & ~0xffu);
    };
    unsigned s0 = 0, s1 = 0;
    if (wa < wb) {
      s0 = sw(wa);
      s1 = sw(wa + 1);
    }
    unsigned w = wa;
    for (int j = warp * 32; j < warp * 32 + 32; j++) {
      const unsigned w1 = min(nw, (unsigned)(j + 1) * wps);  // end of subsegment j
      unsigned F = (unsigned)lane;  // entry offset lane -> (codewords so far << 8) | offset in word w
      for (; w + 1 < w1; w += 2) {
        advance(w + 3);
        const unsigned s2 = sw(w + 2), s3 = sw(w + 3);
        unsigned pa = word_init(w, s0, s1), pb = word_init(w + 1, s1, s2);
        for (int it = 0; it < nj; it++) {
          jump(pa);
          jump(pb);
        }
        compose(F, pa);
        compose(F, pb);
        s0 = s2;
        s1 = s3;
      }
      if (w < w1) {  // odd word count
        advance(w + 2);
        const unsigned s2 = sw(w + 2);
        unsigned pa = word_init(w, s0, s1);
        for (int it = 0; it < nj; it++) jump(pa);
        compose(F, pa);
        s0 = s1;
        s1 = s2;
        w++;
      }
      W.u.map[j][lane] = (uint16_t)(((F >> 8) << 5) | (F & 0xffu));
    }
  }
  __syncthreads();
  D3P(1, clock64());

  // ---- 2. the chain from entry 0: true entry and count of every subsegment ----
  if (t == 0) {
    unsigned e = 0;
    for (int j = 0; j < NS; j++) {
      W.ent[j] = min(L, 32u * wps * (unsigned)j + e);
      W.cnt[j] = 0;
      if ((unsigned)j * wps >= nw) continue;  // empty subsegment: the offset carries over
      const unsigned v = W.u.map[j][e];
      W.cnt[j] = v >> 5;
      e = v & 31u;
    }
    W.fin = e;  // offset after the last word: (end of the last codeword) mod 32
  }
  __syncthreads();
  }  // use_maps
  D3P(2, clock64());
  const unsigned cnt = W.cnt[t];
  const unsigned entry = W.ent[t];

  // ---- 3. write pass: CTA scan of the counts, then every thread decodes its
  // span into the shared tiles, counting code-0 symbols per row ----
  unsigned incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) W.wsum[warp] = incl;
  __syncthreads();
  unsigned base = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kD4Warps; w++) {
    if (w < warp) base += W.wsum[w];
    total += W.wsum[w];
  }
  // spans of equal bit length start ~64 codes apart: the padding keeps their
  // stores in distinct banks (the tiled layout would put them all in one)
  const bool smem_ras = R * C <= kD4Ras;
  uint16_t *ct = codes + tile_base(g, p, 0);
  if (total != nsym || W.fin != (L & 31u)) {
    if (t == 0) {
      set_err_at(st, total < nsym ? PMZ_ERR_TRUNCATED : PMZ_ERR_CORRUPT,
                 10 + (total > nsym) + 2 * (total < nsym) + 4 * (W.fin != (L & 31u)), p);
      d4_publish(zflag + p, kD4Poison);
    }
    return;
  }
  const unsigned e0 = base + incl - cnt + 1;  // raster index of the first symbol (anchor = 0)
  if (smem_ras) {
    if (cnt) {
      D4Reader rd;
      rd.seek(bs, entry);
      unsigned idx = e0;
      for (unsigned i = 0; i < cnt;) {
        rd.refill(bs);
        unsigned s, l, k;
        d4_run(rd.buf, rd.nb, cnt - i, s_len12, s_sym12, lut, s_tab, sym, s, l, k);
        if (k == 1) W.u.ras[d4_pad(idx)] = (uint16_t)s;
        else d4_fill(W.u.ras, idx, k, s);
        idx += k;
        rd.skip(k * l);
        i += k;
      }
    }
    __syncthreads();
    // code-0 symbols per row (the anchor, raster index 0, is not a code)
    for (int r = warp; r < R; r += kD4Warps) {
      unsigned z = 0;
      for (int c = lane; c < C; c += 32) {
        const unsigned q = (unsigned)(r * C + c);
        z += (q != 0u && W.u.ras[d4_pad(q)] == 0) ? 1u : 0u;
      }
      for (int d = 16; d > 0; d >>= 1) z += __shfl_xor_sync(0xffffffffu, z, d);
      if (lane == 0) W.zrow[r] = z;
    }
  } else if (cnt) {  // wide blocks: codes straight to the global tiles, zeros counted on the way
    D4Reader rd;
    rd.seek(bs, entry);
    int r = (int)(e0 / (unsigned)C), c = (int)(e0 - (unsigned)r * C);
    int zr = r;
    unsigned zc = 0;  // code-0 symbols of row zr not yet added to W.zrow
    for (unsigned i = 0; i < cnt;) {
      rd.refill(bs);
      unsigned s, l, k;
      d4_run(rd.buf, rd.nb, cnt - i, s_len12, s_sym12, lut, s_tab, sym, s, l, k);
      for (unsigned j = 0; j < k; j++) {
        ct[(c >> 5) * kTile + r * 32 + (c & 31)] = (uint16_t)s;
        if (s == 0) {
          if (r != zr) {
            if (zc) atomicAdd(&W.zrow[zr], zc);
            zr = r;
            zc = 0;
          }
          zc++;
        }
        if (++c == C) { c = 0; r++; }
      }
      rd.skip(k * l);
      i += k;
    }
    if (zc) atomicAdd(&W.zrow[zr], zc);
  }
  __syncthreads();
  D3P(3, clock64());
  // ---- 4. balance values (D9: block list, partitions in order, raster order
  // within).  This partition publishes its code-0 count; it adds up the counts
  // of the earlier partitions of its block (decoupled look-back: those are
  // lower-numbered CTAs, already resident or finished) ----
  if (t < 32) {
    const unsigned z = W.zrow[t];
    unsigned incl = z;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    W.zrow[t] = incl - z;  // code-0 symbols of the rows above
    const unsigned zp = __shfl_sync(0xffffffffu, incl, 31);
    if (t == 0) {
      d4_publish(zflag + p, zp + 1u);
      unsigned long long zb = 0;
      bool poisoned = false;
      for (int64_t q = first_part(g, b); q < p; q++) {
        unsigned v;
        long long spins = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(zflag + q) : "memory");
        } while (v == 0u && ++spins < (1ll << 22));
        if (v == 0u) {  // never published (cannot happen): fail instead of hanging
          set_err_at(st, PMZ_ERR_CORRUPT, 31, p);
          v = kD4Poison;
        }
        if (v == kD4Poison) poisoned = true;  // that partition failed and reported its error
        zb += v - 1u;
      }
      const unsigned long long nb = blk_nbal[b];
      const bool last = pi == bb.np - 1;
      if (!poisoned && (zb + zp > nb || (last && zb + zp != nb)))
        set_err_at(st, zb + zp > nb ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 30, p);
      if (poisoned || zb + zp > nb || (last && zb + zp != nb)) zb = ~0ull;
      W.zb = zb;
    }
  }
  __syncthreads();
  const unsigned long long zb = W.zb;
  if (zb == ~0ull) return;
  D3P(5, clock64());
  // codes and per-element addends, tiled for the reconstruction: the balance
  // value at code-0 positions, (code - center) * 2 b_a elsewhere (D6)
  {
    const uint8_t *bal = buf + bal_off[b];
    const uintptr_t ba = reinterpret_cast<uintptr_t>(bal);
    const unsigned sh = (unsigned)(ba & 7) * 8;
    const unsigned long long *qb = reinterpret_cast<const unsigned long long *>(ba & ~(uintptr_t)7);
    const long long nwd = (long long)((reinterpret_cast<uintptr_t>(buf + buf_n) - (ba & ~(uintptr_t)7)) >> 3);
    const int nch = (C + 31) >> 5;
    double *vt = vtile + tile_base(g, p, 0);
    // a warp takes a row, four 32-column chunks at a time: ballots and ranks
    // first, then the (independent) balance loads, then the coalesced stores
    auto ldbal = [&](long long i) -> unsigned long long {
      unsigned long long u = __ldg(qb + i);
      if (sh) {
        if (i + 2 <= nwd) u = (u >> sh) | (__ldg(qb + i + 1) << (64 - sh));
        else {  // the value ends the buffer: byte loads
          u = 0;
          for (int k = 7; k >= 0; k--) u = (u << 8) | __ldg(bal + 8 * i + k);
        }
      }
      return u;
    };
    for (int r = warp; r < R; r += kD4Warps) {
      unsigned long long base = zb + W.zrow[r];
      for (int k0 = 0; k0 < nch; k0 += 4) {
        unsigned code[4];
        long long bi[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int c = (k0 + u) * 32 + lane;
          unsigned cd = 1u;
          if (c < C) cd = smem_ras ? W.u.ras[d4_pad((unsigned)(r * C + c))] : ct[(k0 + u) * kTile + r * 32 + lane];
          if (r == 0 && c == 0) cd = kAnc;
          code[u] = cd;
          const unsigned zm = __ballot_sync(0xffffffffu, cd == 0u);
          bi[u] = cd == 0u ? (long long)(base + __popc(zm & ((1u << lane) - 1u))) : -1ll;
          base += __popc(zm);
        }
        unsigned long long val[4];
#pragma unroll
        for (int u = 0; u < 4; u++) val[u] = bi[u] >= 0 ? ldbal(bi[u]) : 0ull;
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int kc = k0 + u;
          if (kc < nch) {
            const double dq = __dmul_rn((double)((int)code[u] - center), two_ba);
            vt[kc * kTile + r * 32 + lane] = bi[u] >= 0 ? __longlong_as_double((long long)val[u]) : dq;
            ct[kc * kTile + r * 32 + lane] = (uint16_t)code[u];
          }
        }
      }
    }
  }
  D3P(4, clock64());
}

}  // namespace pmz

namespace pmz {

// ---------------------------------------------------------------------------
// One-row partitions (1-D inputs, or block_rows == 1: every block is one
// partition of one row).  A 32-row-tile CTA per partition would idle 31/32 of
// its work; here a THREAD decodes a whole partition substream (lane per
// partition), writing row 0 of the partition's code + addend tiles exactly as
// k_decode4 does, so k_reconstruct_1d / k_inv consume the same layout.  A
// block is one partition: its balance list starts at index 0 (no look-back).
constexpr int kD1T = 32;  // small CTAs: the partitions spread over every SM
__global__ void __launch_bounds__(kD1T) k_decode_1d(const uint8_t *__restrict__ buf, unsigned long long buf_n,
                                                   Geom g, const BlkP *__restrict__ blkp,
                                                   const DecTab *__restrict__ tab,
                                                   const uint16_t *__restrict__ sym,
                                                   const unsigned *__restrict__ lut,
                                                   const unsigned long long *__restrict__ part_bits,
                                                   const unsigned long long *__restrict__ part_off,
                                                   const unsigned long long *__restrict__ pay_off,
                                                   const unsigned long long *__restrict__ bal_off,
                                                   const unsigned long long *__restrict__ blk_nbal, int center,
                                                   double two_ba, uint16_t *__restrict__ codes,
                                                   double *__restrict__ vtile, WsStatus *st) {
  __shared__ DecTab s_tab;
  __shared__ uint16_t s_sym12[1 << kLutBits];
  __shared__ uint8_t s_len12[1 << kLutBits];
  count_launch(st);
  if (threadIdx.x == 0) s_tab = *tab;
  for (int i = threadIdx.x; i < (1 << kLutBits); i += kD1T) {
    const unsigned e = __ldg(lut + i);
    s_len12[i] = (e != 0 && !(e & kLutL2Flag)) ? (uint8_t)((e >> 16) & 31u) : (uint8_t)0;
    s_sym12[i] = (uint16_t)(e & 0xffffu);
  }
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * kD1T + threadIdx.x;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) return;
  const BlockBox bb = block_box(g, b);
  const int C = bb.bc;
  const unsigned nsym = (unsigned)(C - 1);
  const unsigned long long L64 = part_bits[p];
  if (L64 > 32ull * (nsym + 1ull)) {
    set_err_at(st, PMZ_ERR_CORRUPT, 1, p);
    return;
  }
  BitSrc bs;
  {
    const uint8_t *src = buf + pay_off[b] + part_off[p];
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    bs.base = reinterpret_cast<const uint8_t *>(a & ~(uintptr_t)3);
    bs.adj = (unsigned)(8 * (a & 3));
    bs.nbits = L64;
    bs.end = buf + buf_n;
  }
  uint16_t *ct = codes + tile_base(g, p, 0);
  ct[0] = kAnc;
  unsigned pos = 0, c = 1;
  D4Reader rd;
  rd.seek(bs, 0);
  while (c <= nsym) {
    rd.refill(bs);
    unsigned s, l, k;
    d4_run(rd.buf, rd.nb, nsym + 1 - c, s_len12, s_sym12, lut, s_tab, sym, s, l, k);
    for (unsigned j = 0; j < k; j++, c++) ct[(c >> 5) * kTile + (c & 31)] = (uint16_t)s;
    rd.skip(k * l);
    pos += k * l;
  }
  if (pos != (unsigned)L64) set_err_at(st, pos < L64 ? PMZ_ERR_CORRUPT : PMZ_ERR_TRUNCATED, 12, p);
}

// The addends of one-row partitions (a warp per partition, lane = column of
// a 32-column chunk): balance value at code 0 (ranked by ballots, the block's
// list from index 0), (code - center) * 2 b_a elsewhere -- coalesced.
__global__ void __launch_bounds__(128) k_gather_1d(const uint8_t *__restrict__ buf, unsigned long long buf_n,
                                                  Geom g, const BlkP *__restrict__ blkp,
                                                  const unsigned long long *__restrict__ bal_off,
                                                  const unsigned long long *__restrict__ blk_nbal, int center,
                                                  double two_ba, const uint16_t *__restrict__ codes,
                                                  double *__restrict__ vtile, WsStatus *st) {
  count_launch(st);
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial || st->err_bits) return;
  const int C = block_box(g, b).bc, nch = (C + 31) >> 5;
  const uint8_t *bal = buf + bal_off[b];
  const uintptr_t ba = reinterpret_cast<uintptr_t>(bal);
  const unsigned sh = (unsigned)(ba & 7) * 8;
  const unsigned long long *qb = reinterpret_cast<const unsigned long long *>(ba & ~(uintptr_t)7);
  const long long nwd = (long long)((reinterpret_cast<uintptr_t>(buf + buf_n) - (ba & ~(uintptr_t)7)) >> 3);
  const unsigned long long nbal = blk_nbal[b];
  const uint16_t *ct = codes + tile_base(g, p, 0);
  double *vt = vtile + tile_base(g, p, 0);
  unsigned long long base = 0;
  for (int kc = 0; kc < nch; kc++) {
    const int c = kc * 32 + lane;
    const unsigned code = c < C ? ct[kc * kTile + lane] : 1u;  // the anchor reads kAnc: not a code
    const unsigned zm = __ballot_sync(0xffffffffu, code == 0u);
    double v = __dmul_rn((double)((int)code - center), two_ba);
    if (code == 0u) {
      const long long i = (long long)(base + __popc(zm & ((1u << lane) - 1u)));
      if ((unsigned long long)i < nbal) {
        unsigned long long u = __ldg(qb + i);
        if (sh) {
          if (i + 2 <= nwd) u = (u >> sh) | (__ldg(qb + i + 1) << (64 - sh));
          else {
            u = 0;
            for (int q = 7; q >= 0; q--) u = (u << 8) | __ldg(bal + 8 * i + q);
          }
        }
        v = __longlong_as_double((long long)u);
      }
    }
    base += __popc(zm);
    if (c < C) vt[kc * kTile + lane] = v;
  }
  if (lane == 0 && base != nbal)
    set_err_at(st, base > nbal ? PMZ_ERR_BALANCE_UNDERFLOW : PMZ_ERR_CORRUPT, 30, p);
}

}  // namespace pmz
