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
#ifndef PMZ_D3W
#define PMZ_D3W 2
#endif

// The substream is read straight from global memory (the reader prefetches
// one word ahead, so the load is off the dependency chain) and the decode
// tables through L1; the per-partition shared state is the boundary bitmap.
// LARGE = false: substreams up to 16 KB; longer ones go to a work list
// served by the LARGE launch (32 KB = the longest valid substream, 8191
// codewords x 32 bits).
template <bool LARGE>
struct D3Cfg {
  static constexpr int kW = LARGE ? 1 : PMZ_D3W;
  static constexpr int kBm = LARGE ? 8192 + 4 : 4096 + 4;  // boundary-bitmap words (substream <= 32 kBm bits)
};
template <bool LARGE>
struct D3Warp {
  unsigned bm[D3Cfg<LARGE>::kBm];
  unsigned xs[32];               // speculative exit per lane
  unsigned ns[32];               // speculative symbol count per lane
  unsigned ent[33], cnt[32];     // chained true entries / counts (fallback)
  unsigned E[32][32];            // fallback: exit per lane per entry offset
  uint16_t Cn[32][32];           // fallback: symbol count per lane per entry offset
  uint16_t vis[32][64];          // fallback: (path + 1) << 10 | symbols before s_t + i
  unsigned zrow[32];
  int err;
};
template <bool LARGE>
constexpr size_t d3_smem() { return sizeof(D3Warp<LARGE>) * D3Cfg<LARGE>::kW; }

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


#ifdef PMZ_DEC3_PROFILE
__device__ long long g_d3[65536][8];  // t0, t_spec, t_fix, t_write, rounds, L, nsym, large
__device__ long long g_d3n[65536][3];  // max-lane iterations: spec, fix (all rounds), stage-end stamp
#define D3_STAMP(i) if (lane == 0 && p < 65536) g_d3[p][i] = clock64();
#else
#define D3_STAMP(i)
#endif
template <bool LARGE>
__global__ void __launch_bounds__(D3Cfg<LARGE>::kW * 32) k_decode3(const uint8_t *__restrict__ buf, unsigned long long buf_n,
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
                                                      WsStatus *st) {
  constexpr int kW = D3Cfg<LARGE>::kW, kBm = D3Cfg<LARGE>::kBm;
  __shared__ unsigned long long s_rep[33];
  __shared__ DecTab s_tab;
  extern __shared__ __align__(16) unsigned char dyn3[];
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (LARGE && (int64_t)blockIdx.x * kW >= (int64_t)large_list[0]) return;
  if (threadIdx.x == 0) s_tab = *tab;
  if (threadIdx.x <= 32) {  // s_rep[l]: bits 0, l, 2l, ... (boundaries of a run, LSB first)
    unsigned long long r = 0;
    if (threadIdx.x >= 1)
      for (int q = 0; q < 64; q += threadIdx.x) r |= 1ull << q;
    s_rep[threadIdx.x] = r;
  }
  __syncthreads();
  const unsigned *s_lut = lut, *lut2 = lut + (1 << kLutBits);  // through L1
  D3Warp<LARGE> &W = reinterpret_cast<D3Warp<LARGE> *>(dyn3)[warp];
  const int64_t nwork = LARGE ? (int64_t)large_list[0] : g.nparts;
  for (int64_t item = (int64_t)blockIdx.x * kW + warp; item < nwork; item += (int64_t)gridDim.x * kW) {
  const int64_t p = LARGE ? (int64_t)large_list[1 + item] : item;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (blkp[b].trivial) {
    if (lane == 0) part_zeros[p] = 0;
    zrow_out[p * 32 + lane] = 0;
    continue;
  }
  const BlockBox bb = block_box(g, b);
  const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc;
  const unsigned nsym = (unsigned)(R * C - 1);
  const unsigned long long L64 = part_bits[p];
  const uint8_t *src = buf + pay_off[b] + part_off[p];
  uint16_t *ct = codes + tile_base(g, p, 0);
  W.zrow[lane] = 0;
  if (lane == 0) W.err = 0;
  unsigned zeros = 0;
  if (L64 > 0xffffff00ull || ((L64 + 31) >> 5) + 4 > (unsigned long long)kBm) {
    if (!LARGE && L64 <= 32ull * (nsym + 1)) {
      if (lane == 0) large_list[1 + atomicAdd(&large_list[0], 1u)] = (unsigned)p;
      continue;
    }
    // longer than any valid substream (codewords <= 32 bits)
    if (lane == 0) set_err(st, PMZ_ERR_CORRUPT);
    continue;
  } else {
    const unsigned L = (unsigned)L64;
    D3_STAMP(0)
#ifdef PMZ_DEC3_PROFILE
    if (lane == 0 && p < 65536) { g_d3[p][5] = L; g_d3[p][6] = nsym; g_d3[p][7] = LARGE; g_d3n[p][2] = clock64(); }
#endif
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
    const unsigned segw = (((L + 31) >> 5) + 31) >> 5;  // words per lane segment
    const unsigned s_i = min(L, 32 * segw * lane), s_n = min(L, 32 * segw * (lane + 1));
    // ---- 1. speculative pass: every codeword boundary of the lane's
    // segment goes into the bitmap (a run of k codewords as one periodic
    // mask), the symbol count into ns ----
    unsigned xs = s_i, nsp = 0;
    {
      const unsigned w0 = s_i >> 5, wend = (s_n + 31) >> 5;
      for (unsigned q = w0; q < wend; q++) W.bm[q] = 0;
      D3Reader<D3Glob> rd;
      rd.seek(ss, s_i, adj);
      unsigned pos = s_i;
      bool bad = false;
#ifdef PMZ_DEC3_PROFILE
      unsigned it_spec = 0;
#endif
      while (pos < s_n) {
#ifdef PMZ_DEC3_PROFILE
        it_spec++;
#endif
        rd.refill(ss);
        int s, l;
        unsigned k;
        if (!d3_run(rd.buf, rd.nb, s_n - pos, s_lut, lut2, s_tab, sym, s, l, k)) { bad = true; break; }
        const unsigned adv = k * (unsigned)l;  // codewords starting before s_n
        // boundaries pos + j l, j < k: LSB-first mask shifted to pos's word
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
      xs = bad ? kD3Bad : pos;
#ifdef PMZ_DEC3_PROFILE
      unsigned mx = it_spec;
      for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      if (lane == 0 && p < 65536) g_d3n[p][0] = mx;
#endif
    }
    W.xs[lane] = xs;
    W.ns[lane] = nsp;
    __syncwarp();
    // speculative boundaries of [s_i, q): symbols of the speculative path before q
    auto rank = [&](unsigned q) -> unsigned {
      unsigned r = 0;
      const unsigned wa = s_i >> 5, wb = q >> 5;
      for (unsigned w = wa; w < wb; w++) r += __popc(W.bm[w]);
      return r + __popc(W.bm[wb] & ((1u << (q & 31)) - 1u));
    };
    D3_STAMP(1)
    // ---- 2. true exits.  Optimistic round: each lane re-decodes from its
    // assumed entry (the previous lane's speculative exit) until it lands on
    // its own speculative path (then its exit is x_t) or crosses s_n. ----
    unsigned entry = lane == 0 ? 0u : W.xs[lane - 1];
    // decode from `from` until landing on a speculative boundary (then the
    // rest is the speculative parse) or crossing s_n; returns the exit and
    // the symbol count of [from, exit)
    auto walk = [&](unsigned from, unsigned &cnt) -> unsigned {
      D3Reader<D3Glob> rd;
      rd.seek(ss, from, adj);
      unsigned pos = from, c = 0;
      while (pos < s_n) {
        if ((W.bm[pos >> 5] >> (pos & 31)) & 1u) {
          cnt = c + W.ns[lane] - rank(pos);
          return W.xs[lane];
        }
        rd.refill(ss);
        int s, l;
        unsigned k;
        if (!d3_run(rd.buf, rd.nb, s_n - pos, s_lut, lut2, s_tab, sym, s, l, k)) return kD3Bad;
        const unsigned adv = k * (unsigned)l;
        rd.skip(adv);
        pos += adv;
        c += k;
      }
      cnt = c;
      return pos;
    };
    unsigned ex, cnt = 0;
    ex = entry == kD3Bad ? kD3Bad : (entry >= s_n ? entry : walk(entry, cnt));
    const unsigned nent = __shfl_up_sync(0xffffffffu, ex, 1);
    if (__any_sync(0xffffffffu, lane > 0 && nent != entry)) {
      // ---- fallback: transfer function of every lane over all entry offsets
      // [0, D) (the true entry is the first boundary >= s_t, < s_t + maxl);
      // paths merge into the speculative path (bitmap) or into an earlier
      // offset's path (window of the first 64 bits), then lane 0 chains. ----
      const int D = min(s_tab.maxl, 32);
      for (int i = 0; i < 64; i++) W.vis[lane][i] = 0;
#ifdef PMZ_DEC3_PROFILE
      unsigned it_tf = 0, n_new = 0;
#endif
      W.E[lane][0] = W.xs[lane];
      W.Cn[lane][0] = (uint16_t)min(W.ns[lane], 65535u);
      // one flat work loop per lane (lanes progress independently): advance
      // the current path one step, or finish it and start the next offset
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
#ifdef PMZ_DEC3_PROFILE
          n_new++;
#endif
        } else if ((W.bm[q >> 5] >> (q & 31)) & 1u) {
          e = W.xs[lane];
          c += W.ns[lane] - rank(q);
          fin = true;
        } else {
          const unsigned off = q - s_i;
          const unsigned v = off < 64u ? W.vis[lane][off] : 0u;
          if (v) {
            const unsigned o2 = (v >> 10) - 1;
            e = W.E[lane][o2];
            c += W.Cn[lane][o2] - (v & 1023u);
            fin = true;
          } else {
            rd.refill(ss);
            int s, l;
            unsigned k;
            if (!d3_run(rd.buf, rd.nb, s_n - q, s_lut, lut2, s_tab, sym, s, l, k)) {
              e = kD3Bad;
              fin = true;
            } else {
#ifdef PMZ_DEC3_PROFILE
              it_tf++;
#endif
              // every boundary of this step inside the window belongs to path o
              for (unsigned j = 0; j < k; j++) {
                const unsigned oj = off + j * (unsigned)l;
                if (oj >= 64u) break;
                if (!W.vis[lane][oj]) W.vis[lane][oj] = (uint16_t)(((o + 1) << 10) | min(c + j, 1023u));
              }
              const unsigned adv = k * (unsigned)l;
              rd.skip(adv);
              q += adv;
              c += k;
            }
          }
        }
        if (fin) {
          W.E[lane][o] = e;
          W.Cn[lane][o] = (uint16_t)min(c, 65535u);
          o++;
          q = s_i + (unsigned)o;
          c = 0;
          if (o < D && q < s_n) rd.seek(ss, q, adj);
        }
      }
#ifdef PMZ_DEC3_PROFILE
      {
        unsigned mx = it_tf, mn = n_new;
        for (int d = 16; d > 0; d >>= 1) { mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d)); mn = max(mn, __shfl_xor_sync(0xffffffffu, mn, d)); }
        if (lane == 0 && p < 65536) { g_d3n[p][1] = mx; g_d3[p][4] = 100 + mn; }
      }
#endif
      __syncwarp();
      if (lane == 0) {
        const unsigned segw2 = 32 * segw;
        unsigned T = 0;
        for (int t = 0; t < 32; t++) {
          W.ent[t] = T;
          W.cnt[t] = 0;
          const unsigned si = min(L, segw2 * t), sn = min(L, segw2 * (t + 1));
          if (T == kD3Bad || T >= sn) continue;  // no codeword starts in segment t
          const unsigned o = T - si;
          W.cnt[t] = o < (unsigned)D ? W.Cn[t][o] : 0u;
          T = o < (unsigned)D ? W.E[t][o] : kD3Bad;
        }
        W.ent[32] = T;
      }
      __syncwarp();
      entry = W.ent[lane];
      ex = W.ent[lane + 1];
      cnt = W.cnt[lane];
    }
    D3_STAMP(2)
    // ---- 3. write pass ----
    unsigned incl = cnt;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    const unsigned last = __shfl_sync(0xffffffffu, ex, 31);
    const bool okall = __all_sync(0xffffffffu, ex != kD3Bad);
    if (!okall || total != nsym || last != L) {
      if (lane == 0) set_err(st, !okall ? PMZ_ERR_INVALID_PREFIX : (total < nsym ? PMZ_ERR_TRUNCATED : PMZ_ERR_CORRUPT));
    } else if (cnt) {
      D3Reader<D3Glob> rd;
      rd.seek(ss, entry, adj);
      const unsigned e0 = incl - cnt + 1;  // raster index of the first symbol (anchor = 0)
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
    __syncwarp();
    D3_STAMP(3)
  }
  for (int d = 16; d > 0; d >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, d);
  if (lane == 0) part_zeros[p] = zeros;
  zrow_out[p * 32 + lane] = (uint16_t)W.zrow[lane];
  __syncwarp();
  }
}

}  // namespace pmz
