// dec3.cuh -- canonical Huffman decode of the per-partition substreams
// (decode_next; substream layout SPEC.md:496), one warp per
// partition, writing the codes in the partition-tiled layout (common.cuh).
//
// A decode step keeps the next bits of the stream left-aligned in a 64-bit
// register (refilled one 32-bit word at a time) and resolves a codeword with
// one 12-bit table lookup (codewords longer than 12 bits: canonical
// first/count search).  Parallelism inside a substream of L bits:
//   1. speculative pass: lane t decodes from the 32-bit-aligned segment start
//      s_t = t * seg until it crosses s_{t+1}, marking every codeword boundary
//      of its segment in a bitmap (the lane owns its bitmap words) and
//      recording its exit x_t and symbol count n_t;
//   2. fix-up: lane t re-decodes from its true entry (lane t-1's true exit)
//      until it lands on a marked boundary -- from there its speculative parse
//      is the true parse, so exit = x_t and count = decoded + n_t - rank -- or
//      until it crosses s_{t+1} (then that IS its true exit).  Only a lane
//      whose entry changed redoes; rounds repeat until no entry changes
//      (typically one round: Huffman streams self-synchronise within a few
//      codewords; a stream that never does costs one segment per round);
//   3. write pass: every lane decodes its true span and stores the codes at
//      their tile positions, counting code-0 symbols (balance points) per row.
// Substreams longer than 8 KB (> 8 bits per symbol on average) are served by
// a second launch with a 32 KB stage (work list).
#pragma once
#include "common.cuh"
#include "decompress.cuh"

namespace pmz {

constexpr unsigned kD3Bad = 0xffffffffu;
#ifndef PMZ_D3_WPP
#define PMZ_D3_WPP 8
#endif
constexpr int kD3Wpp = PMZ_D3_WPP;  // warps per partition
constexpr int kD3Nl = 32 * kD3Wpp;  // lane segments per partition
#ifndef PMZ_D3_ROUNDS
#define PMZ_D3_ROUNDS 8
#endif
constexpr int kD3Rounds = PMZ_D3_ROUNDS;        // optimistic re-walk rounds before the transfer function

// One CTA per partition, kD3Nl lanes = segments.  The substream is read
// straight from global memory (the reader prefetches one word ahead, so the
// load is off the dependency chain); the first-level decode table and the
// boundary bitmap live in shared memory, the second-level table is read
// through L1 and the per-lane fallback tables go to a global pool.
// LARGE = false: substreams up to 16 KB; longer ones go to a work list
// served by the LARGE launch (32 KB = the longest valid substream, 8191
// codewords x 32 bits).
template <bool LARGE>
struct D3Cfg {
  static constexpr int kBm = LARGE ? 8192 + 4 : 4096 + 4;  // boundary-bitmap words (substream <= 32 kBm bits)
};
template <bool LARGE>
struct D3Part {
  unsigned lut[1 << kLutBits];          // first-level decode table (second level through L1)
  unsigned bm[D3Cfg<LARGE>::kBm];
  unsigned xs[kD3Nl], ns[kD3Nl];        // speculative exit / symbol count per lane
  unsigned ex[kD3Nl], ent[kD3Nl + 1], cnt[kD3Nl];
  unsigned zrow[32];
  unsigned wsum[kD3Wpp];
};
// Fallback tables of one partition (global scratch, L2-resident; only the
// partitions whose optimistic round fails touch them), from a pool of
// nslots claimed by compare-and-swap: at least as many slots as CTAs can be
// resident at once (d3_fall_slots), so a claim always succeeds and no two
// live CTAs share one.
struct D3Fall {
  uint16_t E[kD3Nl][32];                // exit - s_t per entry offset (0xffff: bad)
  uint16_t Cn[kD3Nl][32];               // symbol count per entry offset
  uint16_t vis[kD3Nl][64];              // (path + 1) << 10 | symbols before s_t + i
};
template <bool LARGE>
constexpr size_t d3_smem() { return sizeof(D3Part<LARGE>); }

// Big-endian words of the substream, straight from the container: word i
// covers stream bits [32 i - adj, 32 i + 32 - adj) of an aligned base.
struct D3Glob {
  BitSrc bs;
  __device__ __forceinline__ unsigned word(unsigned i) const { return bs.word(i); }
};
// Register bit reader at an arbitrary bit position of a word source whose
// word 0 starts at stream bit -adj (adj = 0 for the staged source).
template <class Src>
struct D3Reader {
  unsigned long long buf;  // next stream bits, left-aligned
  int nb;                  // valid bits in buf (>= 32 after refill)
  unsigned wi;             // index of the prefetched word
  unsigned nxt;            // prefetched next word (off the dependency chain)
  __device__ __forceinline__ void seek(const Src &src, unsigned pos, unsigned adj) {
    const unsigned q = pos + adj;
    wi = q >> 5;
    const unsigned sh = q & 31;
    buf = (((unsigned long long)src.word(wi) << 32) | src.word(wi + 1)) << sh;
    nb = 64 - (int)sh;
    wi += 2;
    nxt = src.word(wi);
  }
  __device__ __forceinline__ void refill(const Src &src) {
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

// The codeword at the top of the reader (refilled: nb >= 32 valid bits) and
// how many times it repeats back-to-back inside the valid bits (k >= 1):
// first level over 12 bits, second level for longer codewords (canonical
// search only when the second level did not fit).  A repeat is found with one
// 64-bit compare against the codeword's periodic extension.
__device__ __forceinline__ bool d3_run(unsigned long long buf, int nb, unsigned lim, const unsigned *__restrict__ lut,
                                       const unsigned *__restrict__ lut2, const DecTab &tab,
                                       const uint16_t *__restrict__ sym, int &s, int &l, unsigned &k) {
  const unsigned top = (unsigned)(buf >> 32);
  unsigned e = lut[top >> (32 - kLutBits)];
  if (e & kLutL2Flag) e = lut2[(e & 0xffffu) + ((top << kLutBits) >> (32 - tab.sub_bits))];
  if (__builtin_expect(e == 0, 0)) {
    s = -1;
    for (int ll = kLutBits + 1; ll <= tab.maxl; ll++) {
      const unsigned d = (top >> (32 - ll)) - tab.first[ll];
      if (d < tab.count[ll]) { s = sym[tab.offset[ll] + d]; l = ll; break; }
    }
    if (s < 0) return false;
    k = 1;
    return true;
  }
  l = (int)((e >> 16) & 31u);
  s = (int)(e & 0xffffu);
  // back-to-back repeats: buf is periodic with period l over its first
  // clz(buf ^ (buf << l)) + l bits; count whole codewords inside the valid
  // bits that start before `lim` bits from here
  const unsigned long long x = buf ^ (buf << l);
  const unsigned P = (x ? (unsigned)__clzll((long long)x) : 64u) + (unsigned)l;
  const unsigned z = min(min(P, (unsigned)nb), lim + (unsigned)l - 1u);
  const unsigned M = e >> 21;
  k = l == 1 ? z : max((z * M) >> 10, 1u);
  return true;
}


template <bool LARGE>
__global__ void __launch_bounds__(kD3Nl) k_decode3(const uint8_t *__restrict__ buf, unsigned long long buf_n,
                                                  Geom g, const BlkP *__restrict__ blkp,
                                                  const DecTab *__restrict__ tab,
                                                  const uint16_t *__restrict__ sym,
                                                  const unsigned *__restrict__ lut,
                                                  const unsigned long long *__restrict__ part_bits,
                                                  const unsigned long long *__restrict__ part_off,
                                                  const unsigned long long *__restrict__ pay_off,
                                                  uint16_t *__restrict__ codes,
                                                  unsigned long long *__restrict__ part_zeros,
                                                  uint16_t *__restrict__ zrow_out, unsigned *large_list,
                                                  D3Fall *__restrict__ fall, unsigned *fall_busy, unsigned nslots,
                                                  WsStatus *st) {
  constexpr int NL = kD3Nl, kBm = D3Cfg<LARGE>::kBm;
  __shared__ unsigned long long s_rep[33];
  __shared__ DecTab s_tab;
  __shared__ unsigned s_slot;
  extern __shared__ __align__(16) unsigned char dyn3[];
  D3Part<LARGE> &W = *reinterpret_cast<D3Part<LARGE> *>(dyn3);
  count_launch(st);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t p;
  if (LARGE) {
    if (blockIdx.x >= large_list[0]) return;
    p = large_list[1 + blockIdx.x];
  } else {
    p = blockIdx.x;
  }
  if (t == 0) s_tab = *tab;
  if (t <= 32) {  // s_rep[l]: bits 0, l, 2l, ... (boundaries of a run, LSB first)
    unsigned long long r = 0;
    if (t >= 1)
      for (int q = 0; q < 64; q += t) r |= 1ull << q;
    s_rep[t] = r;
  }
  if (t < 32) W.zrow[t] = 0;
  for (int i = t; i < (1 << kLutBits); i += NL) W.lut[i] = __ldg(lut + i);
  __syncthreads();
  const unsigned *s_lut = W.lut, *lut2 = lut + (1 << kLutBits);  // second level through L1
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) {
    if (t == 0) part_zeros[p] = 0;
    if (t < 32) zrow_out[p * 32 + t] = 0;
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc;
  const unsigned nsym = (unsigned)(R * C - 1);
  const unsigned long long L64 = part_bits[p];
  if (L64 > 0xffffff00ull || ((L64 + 31) >> 5) + 4 > (unsigned long long)kBm) {
    if (t == 0) {
      if (!LARGE && L64 <= 32ull * (nsym + 1)) large_list[1 + atomicAdd(&large_list[0], 1u)] = (unsigned)p;
      else set_err_at(st, PMZ_ERR_CORRUPT, 1, p);  // longer than any valid substream (codewords <= 32 bits)
    }
    return;
  }
  const unsigned L = (unsigned)L64;
  const uint8_t *src = buf + pay_off[b] + part_off[p];
  uint16_t *ct = codes + tile_base(g, p, 0);
  BitSrc bsrc;
  {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    bsrc.base = reinterpret_cast<const uint8_t *>(a & ~(uintptr_t)3);
    bsrc.adj = (unsigned)(8 * (a & 3));
    bsrc.nbits = L64;
    bsrc.end = buf + buf_n;
  }
  const D3Glob ss{bsrc};
  const unsigned adj = bsrc.adj;
  const unsigned segw = (((L + 31) >> 5) + NL - 1) / NL;  // words per lane segment
  const unsigned s_i = min(L, 32 * segw * t), s_n = min(L, 32 * segw * (t + 1));

  // ---- 1. speculative pass: every codeword boundary of the lane's segment
  // goes into the bitmap (a run of k codewords as one periodic mask), the
  // symbol count into ns ----
  {
    // an empty segment (s_i == s_n == L) owns no word: the partial last
    // word belongs to the last non-empty lane
    const unsigned w0 = s_i >> 5, wend = s_n > s_i ? (s_n + 31) >> 5 : w0;
    for (unsigned q = w0; q < wend; q++) W.bm[q] = 0;
    D3Reader<D3Glob> rd;
    rd.seek(ss, s_i, adj);
    unsigned pos = s_i, nsp = 0;
    bool bad = false;
    while (pos < s_n) {
      rd.refill(ss);
      int s, l;
      unsigned k;
      if (!d3_run(rd.buf, rd.nb, s_n - pos, s_lut, lut2, s_tab, sym, s, l, k)) { bad = true; break; }
      const unsigned adv = k * (unsigned)l;  // codewords starting before s_n
      const unsigned long long m = k == 1 ? 1ull : (s_rep[l] & ((1ull << ((k - 1) * l + 1)) - 1ull));
      const unsigned off = pos & 31, wq = pos >> 5;
      W.bm[wq] |= (unsigned)(m << off);
      const unsigned long long hi = off ? (m >> (32 - off)) : (m >> 32);
      if (hi) {
        W.bm[wq + 1] |= (unsigned)hi;
        if (hi >> 32) W.bm[wq + 2] |= (unsigned)(hi >> 32);
      }
      rd.skip(adv);
      pos += adv;
      nsp += k;
    }
    W.xs[t] = bad ? kD3Bad : pos;
    W.ns[t] = nsp;
  }
  __syncthreads();
  // speculative boundaries of [s_i, q): symbols of the speculative path before q
  auto rank = [&](unsigned q) -> unsigned {
    unsigned r = 0;
    const unsigned wa = s_i >> 5, wb = q >> 5;
    for (unsigned w = wa; w < wb; w++) r += __popc(W.bm[w]);
    return r + __popc(W.bm[wb] & ((1u << (q & 31)) - 1u));
  };

  // ---- 2. true exits.  Optimistic rounds: each lane decodes from its
  // assumed entry (first the previous lane's speculative exit) until it lands
  // on a speculative boundary of its own (then its exit is x_t) or crosses
  // s_n; lanes whose entry changed walk again.  Lane 0's entry is exact, so
  // round r fixes lane r; after kD3Rounds the transfer function decides ----
  auto walk = [&](unsigned e0, unsigned &ex, unsigned &cnt) {
    cnt = 0;
    if (e0 == kD3Bad) {
      ex = kD3Bad;
      return;
    }
    if (e0 >= s_n) {  // no codeword starts in this segment
      ex = e0;
      return;
    }
    D3Reader<D3Glob> rd;
    rd.seek(ss, e0, adj);
    unsigned pos = e0, c = 0;
    while (pos < s_n) {
      if ((W.bm[pos >> 5] >> (pos & 31)) & 1u) {
        cnt = c + W.ns[t] - rank(pos);
        ex = W.xs[t];
        return;
      }
      rd.refill(ss);
      int s, l;
      unsigned k;
      if (!d3_run(rd.buf, rd.nb, s_n - pos, s_lut, lut2, s_tab, sym, s, l, k)) {
        ex = kD3Bad;
        return;
      }
      const unsigned adv = k * (unsigned)l;
      rd.skip(adv);
      pos += adv;
      c += k;
    }
    ex = pos;
    cnt = c;
  };
  unsigned entry = t == 0 ? 0u : W.xs[t - 1];
  unsigned ex, cnt;
  walk(entry, ex, cnt);
  bool need_tf;
  int rr = 0;
  for (int r = 0;; r++) {
    rr = r;
    W.ex[t] = ex;
    __syncthreads();
    const unsigned e1 = t == 0 ? 0u : W.ex[t - 1];
    const bool moved = e1 != entry;
    need_tf = __syncthreads_or(moved);
    if (!need_tf || r == kD3Rounds) break;
    if (moved) {
      entry = e1;
      walk(entry, ex, cnt);
    }
  }
  if (need_tf) {
    // ---- fallback: transfer function of every lane over all entry offsets
    // [0, D) (the true entry is the first boundary >= s_t, < s_t + maxl);
    // paths merge into the speculative path (bitmap) or into an earlier
    // offset's path (window of the first 64 bits), then thread 0 chains ----
    const int D = min(s_tab.maxl, 32);
    if (t == 0) {
      unsigned sl = (unsigned)(p % nslots);
      while (atomicCAS(&fall_busy[sl], 0u, 1u) != 0u) sl = (sl + 1) % nslots;
      s_slot = sl;
    }
    __syncthreads();
    D3Fall &F = fall[s_slot];
    unsigned long long vmask = 0;  // offsets of the window with a F.vis entry (no zeroing, no load per step)
    auto rel = [&](unsigned e) -> uint16_t { return e == kD3Bad ? (uint16_t)0xffff : (uint16_t)(e - s_i); };
    F.E[t][0] = rel(W.xs[t]);
    F.Cn[t][0] = (uint16_t)min(W.ns[t], 65535u);
    int o = 1;
    unsigned q = s_i + 1, c = 0;
    D3Reader<D3Glob> rd;
    if (D > 1 && q < s_n) rd.seek(ss, q, adj);
    while (o < D) {
      unsigned e = 0;
      bool fin = false;
      if (q >= s_n) {
        e = q;
        fin = true;
      } else if ((W.bm[q >> 5] >> (q & 31)) & 1u) {
        e = W.xs[t];
        c += W.ns[t] - rank(q);
        fin = true;
      } else {
        const unsigned off = q - s_i;
        if (off < 64u && ((vmask >> off) & 1ull)) {
          const unsigned v = F.vis[t][off];
          const unsigned o2 = (v >> 10) - 1;
          e = F.E[t][o2] == 0xffff ? kD3Bad : s_i + F.E[t][o2];
          c += F.Cn[t][o2] - (v & 1023u);
          fin = true;
        } else {
          rd.refill(ss);
          int s, l;
          unsigned k;
          if (!d3_run(rd.buf, rd.nb, s_n - q, s_lut, lut2, s_tab, sym, s, l, k)) {
            e = kD3Bad;
            fin = true;
          } else {
            // every boundary of this step inside the window belongs to path o
            for (unsigned j = 0; j < k; j++) {
              const unsigned oj = off + j * (unsigned)l;
              if (oj >= 64u) break;
              if (!((vmask >> oj) & 1ull)) {
                vmask |= 1ull << oj;
                F.vis[t][oj] = (uint16_t)(((o + 1) << 10) | min(c + j, 1023u));
              }
            }
            const unsigned adv = k * (unsigned)l;
            rd.skip(adv);
            q += adv;
            c += k;
          }
        }
      }
      if (fin) {
        F.E[t][o] = rel(e);
        F.Cn[t][o] = (uint16_t)min(c, 65535u);
        o++;
        q = s_i + (unsigned)o;
        c = 0;
        if (o < D && q < s_n) rd.seek(ss, q, adj);
      }
    }
    // the bitmap is dead now and the LUT is reloaded below: stage the tables
    // in their (contiguous) space for the serial chain
    static_assert(offsetof(D3Part<LARGE>, bm) == sizeof(unsigned) << kLutBits, "lut, bm contiguous");
    static_assert(NL * 32 <= (1 << kLutBits) + kBm, "staging fits lut + bm");
    __syncthreads();
    uint16_t(*sE)[32] = reinterpret_cast<uint16_t(*)[32]>(W.lut);
    uint16_t(*sC)[32] = reinterpret_cast<uint16_t(*)[32]>(W.lut + NL * 16);
    {
      const uint4 *ge = reinterpret_cast<const uint4 *>(F.E[t]), *gc = reinterpret_cast<const uint4 *>(F.Cn[t]);
      uint4 *se = reinterpret_cast<uint4 *>(sE[t]), *sc = reinterpret_cast<uint4 *>(sC[t]);
      uint4 a[4], c4[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { a[i] = ge[i]; c4[i] = gc[i]; }
#pragma unroll
      for (int i = 0; i < 4; i++) { se[i] = a[i]; sc[i] = c4[i]; }
    }
    __syncthreads();
    if (t == 0) {
      atomicExch(&fall_busy[s_slot], 0u);  // every lane has copied its tables out (barrier above)
      unsigned T = 0;
      for (int u = 0; u < NL; u++) {
        W.ent[u] = T;
        W.cnt[u] = 0;
        const unsigned si = min(L, 32 * segw * u), sn = min(L, 32 * segw * (u + 1));
        if (T == kD3Bad || T >= sn) continue;  // no codeword starts in segment u
        const unsigned oo = T - si;
        if (oo >= (unsigned)D || sE[u][oo] == 0xffff) {
          T = kD3Bad;
          continue;
        }
        W.cnt[u] = sC[u][oo];
        T = si + sE[u][oo];
      }
      W.ent[NL] = T;
    }
    __syncthreads();
    for (int i = t; i < (1 << kLutBits); i += NL) W.lut[i] = __ldg(lut + i);
    __syncthreads();
    entry = W.ent[t];
    ex = W.ent[t + 1];
    cnt = W.cnt[t];
  }

  // ---- 3. write pass: CTA scan of the counts, then every lane decodes its
  // span into the tile layout, counting code-0 symbols per row ----
  unsigned incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) W.wsum[warp] = incl;
  W.ex[t] = ex;
  __syncthreads();
  unsigned base = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kD3Wpp; w++) {
    if (w < warp) base += W.wsum[w];
    total += W.wsum[w];
  }
  const unsigned last = W.ex[NL - 1];
  const bool okall = __syncthreads_and(ex != kD3Bad);
  unsigned zeros = 0;
  if (!okall || total != nsym || last != L) {
    if (t == 0)
      set_err_at(st, !okall ? PMZ_ERR_INVALID_PREFIX : (total < nsym ? PMZ_ERR_TRUNCATED : PMZ_ERR_CORRUPT),
                 10 + (total > nsym) + 2 * (total < nsym) + 4 * (last != L) + 8 * !okall + 100 * rr + 1000 * need_tf, p);
  } else if (cnt) {
    D3Reader<D3Glob> rd;
    rd.seek(ss, entry, adj);
    const unsigned e0 = base + incl - cnt + 1;  // raster index of the first symbol (anchor = 0)
    int r = (int)(e0 / (unsigned)C), c = (int)(e0 - (unsigned)r * C);
    int zr = r;
    unsigned zc = 0;  // code-0 symbols of row zr not yet added to W.zrow
    for (unsigned i = 0; i < cnt;) {
      rd.refill(ss);
      int s, l;
      unsigned k;
      if (!d3_run(rd.buf, rd.nb, 64u, s_lut, lut2, s_tab, sym, s, l, k)) { set_err(st, PMZ_ERR_INVALID_PREFIX); break; }
      k = min(k, cnt - i);
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
      if (s == 0) zeros += k;
      rd.skip(k * (unsigned)l);
      i += k;
    }
    if (zc) atomicAdd(&W.zrow[zr], zc);
  }
  for (int d = 16; d > 0; d >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, d);
  if (lane == 0) W.wsum[warp] = zeros;
  __syncthreads();
  if (t == 0) {
    unsigned z = 0;
    for (int w = 0; w < kD3Wpp; w++) z += W.wsum[w];
    part_zeros[p] = z;
  }
  if (t < 32) zrow_out[p * 32 + t] = (uint16_t)W.zrow[t];
}

}  // namespace pmz
