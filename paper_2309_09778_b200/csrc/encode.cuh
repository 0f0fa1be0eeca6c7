// encode.cuh -- validation histogram, canonical Huffman codebook, bit packing
// and container records (layout :496).
#pragma once
#include "common.cuh"

namespace pmz {

// K5: per-block code histograms of the validation blocks, summed (D10).
// Warp-aggregated: lanes holding the same code elect one leader (match_any).
template <int NT>
__global__ void __launch_bounds__(NT) k_val_hist(Geom g, const BlkP *__restrict__ blkp, const int64_t *val_ids,
                                                 const uint16_t *__restrict__ codes, unsigned long long *hist,
                                                 WsStatus *st) {
  count_launch(st);
  int64_t b = val_ids[blockIdx.y];
  if (blkp[b].trivial) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&hist[kMaxAlpha], 1ull);  // k for the floor (D10)
  BlockBox bb = block_box(g, b);
  int64_t n = (int64_t)bb.br * bb.bc;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * NT; base < n; base += (int64_t)gridDim.x * NT) {
    int64_t e = base + threadIdx.x;
    int code = -1;
    if (e < n) {
      int r = (int)(e / bb.bc), c = (int)(e - (int64_t)r * bb.bc);
      if (!((r % g.prow) == 0 && c == 0)) code = codes[(bb.r0 + r) * g.cols + bb.c0 + c];
    }
    unsigned peers = __match_any_sync(0xffffffffu, code);
    int leader = __ffs(peers) - 1;
    if (code >= 0 && lane == leader) atomicAdd(&hist[code], (unsigned long long)__popc(peers));
  }
}

// Bitonic sort of n (power of two) u64 keys, ascending, by one CTA.
__device__ void bitonic_sort(unsigned long long *a, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          unsigned long long x = a[i], y = a[l];
          bool up = (i & k) == 0;
          if ((x > y) == up) { a[i] = y; a[l] = x; }
        }
      }
      __syncthreads();
    }
  }
}

// K6: build_codebook (D10).  Frequencies = summed validation
// histograms floored at k (= number of non-trivial validation blocks), leaves
// sorted by (frequency, code); two-queue Huffman with ties preferring the leaf
// (Moffat-Katajainen in-place form, same tree); canonical codewords in
// (length, code) order.  One CTA; smem when 2^m <= 8192, else global scratch.
__global__ void __launch_bounds__(1024) k_codebook(const unsigned long long *hist, WsStatus *st,
                                                   unsigned long long *g_keys, unsigned *g_A, uint8_t *lens,
                                                   unsigned *cw) {
  extern __shared__ unsigned long long sm[];
  count_launch(st);
  const int m = st->m;
  const int n = 1 << m;
  const bool in_smem = n <= 8192;
  unsigned long long *keys = in_smem ? sm : g_keys;
  unsigned *A = in_smem ? (unsigned *)(sm + n) : g_A;
  unsigned long long kval = hist[kMaxAlpha] > 0 ? hist[kMaxAlpha] : 1ull;
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    unsigned long long f = hist[s];
    if (f < kval) f = kval;
    keys[s] = (f << 17) | (unsigned long long)s;
  }
  __syncthreads();
  bitonic_sort(keys, n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) A[i] = (unsigned)(keys[i] >> 17);
  __syncthreads();
  if (threadIdx.x == 0) {
    // phase 1: pair up (internal node weights / parent pointers in place)
    A[0] += A[1];
    int root = 0, leaf = 2;
    for (int nxt = 1; nxt < n - 1; nxt++) {
      if (leaf >= n || A[root] < A[leaf]) { A[nxt] = A[root]; A[root++] = nxt; }
      else A[nxt] = A[leaf++];
      if (leaf >= n || (root < nxt && A[root] < A[leaf])) { A[nxt] += A[root]; A[root++] = nxt; }
      else A[nxt] += A[leaf++];
    }
    // phase 2: internal node depths
    A[n - 2] = 0;
    for (int nxt = n - 3; nxt >= 0; nxt--) A[nxt] = A[A[nxt]] + 1;
    // phase 3: leaf depths
    int avail = 1, used = 0, depth = 0, r = n - 2, nxt = n - 1;
    while (avail > 0) {
      while (r >= 0 && (int)A[r] == depth) { used++; r--; }
      while (avail > used) { A[nxt--] = depth; avail--; }
      avail = 2 * used; depth++; used = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) lens[keys[i] & 0x1ffff] = (uint8_t)A[i];
  __syncthreads();
  __shared__ unsigned s_cnt[64], s_next[64];
  __shared__ int s_maxl;
  if (threadIdx.x < 64) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_maxl = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    atomicAdd(&s_cnt[lens[i]], 1u);
    atomicMax(&s_maxl, (int)lens[i]);
  }
  __syncthreads();
  const int maxl = s_maxl;
  if (threadIdx.x == 0) {
    st->max_len = maxl;
    unsigned long long c = 0;
    s_cnt[0] = 0;
    for (int l = 1; l <= maxl && l < 64; l++) { c = (c + s_cnt[l - 1]) << 1; s_next[l] = (unsigned)c; }
  }
  __syncthreads();
  if (maxl > 32) {
    if (threadIdx.x == 0) atomicOr(&st->err_bits, 1u << (-PMZ_ERR_UNASSIGNED));
    return;
  }
  // canonical codewords in (length, code) order: code = first[len] + rank of the
  // symbol among equal-length symbols; ranks via the sorted order (keys hold the
  // symbol; the leaf order by (freq, sym) is not the code order, so count
  // per length with a block-wide scan over symbols in index order).
  __shared__ unsigned s_wsum[32][33];
  const int nt = blockDim.x, tid = threadIdx.x;
  const int per = (n + nt - 1) / nt;
  const int lo = tid * per, hi = min(n, lo + per);
  // each thread counts lengths in its contiguous symbol range (lengths <= 32)
  unsigned myc[33];
#pragma unroll
  for (int l = 0; l <= 32; l++) myc[l] = 0;
  for (int i = lo; i < hi; i++) myc[lens[i]]++;
  // exclusive prefix over threads, per length: warp scans then warp totals
  const int wid = tid >> 5, ln = tid & 31;
  unsigned mypre[33];
#pragma unroll
  for (int l = 1; l <= 32; l++) {
    unsigned v = myc[l], incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
      if (ln >= d) incl += t;
    }
    mypre[l] = incl - v;
    if (ln == 31) s_wsum[wid][l] = incl;
  }
  __syncthreads();
  if (tid < 33 && tid >= 1) {
    unsigned acc = 0;
    for (int w = 0; w < nt / 32; w++) { const unsigned t = s_wsum[w][tid]; s_wsum[w][tid] = acc; acc += t; }
  }
  __syncthreads();
  unsigned nxt[33];
#pragma unroll
  for (int l = 1; l <= 32; l++) nxt[l] = s_next[l] + s_wsum[wid][l] + mypre[l];
  for (int i = lo; i < hi; i++) {
    const int l = lens[i];
    cw[i] = l ? nxt[l]++ : 0;
  }
}

// K7: per-partition payload bits and balance counts.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_part_bits(Geom g, const BlkP *__restrict__ blkp,
                                                       const uint16_t *__restrict__ codes,
                                                       const uint8_t *__restrict__ lens,
                                                       unsigned long long *part_bits, WsStatus *st) {
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * NW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  unsigned long long bits = 0;
  if (!blkp[b].trivial) {
    BlockBox bb = block_box(g, b);
    int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
    const uint16_t *cp = codes + (bb.r0 + pr0) * g.cols + bb.c0;
    if ((g.cols & 7) == 0 && (C & 7) == 0) {
      const int vpr = C >> 3, nv = R * vpr;  // 8 codes per 16-byte vector
      for (int i0 = lane; i0 < nv; i0 += 128) {
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = i0 + 32 * u;
          if (i < nv) {
            const int r = i / vpr, c = (i - r * vpr) << 3;
            q[u] = __ldg(reinterpret_cast<const uint4 *>(cp + (int64_t)r * g.cols + c));
          } else {
            q[u] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);  // anchor marker -> len 0 below
          }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
          for (int h = 0; h < 4; h++) {
            const unsigned a = w[h] & 0xffff, c2 = w[h] >> 16;
            if (a != 0xffff) bits += __ldg(&lens[a]);
            if (c2 != 0xffff) bits += __ldg(&lens[c2]);
          }
        }
      }
    } else {
      for (int r = 0; r < R; r++) {
        const uint16_t *crow = cp + (int64_t)r * g.cols;
        for (int c = lane; c < C; c += 32)
          if (r | c) bits += __ldg(&lens[crow[c]]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o);
  }
  if (lane == 0) part_bits[p] = bits;
}

__host__ __device__ inline uint64_t model_blob_bytes(int S, int H) { return 16 + 8ull * (S + 1) * H + 8ull * H; }
__host__ __device__ inline uint64_t header_bytes(int m, int S, int H) {
  return 52 + 8 + model_blob_bytes(S, H) + 8 + 2 + (1ull << m) + 8;
}

// K8: record size per block (D13, D15).
__global__ void k_block_sizes(Geom g, const BlkP *__restrict__ blkp, const unsigned long long *part_bits,
                              const unsigned long long *part_zeros, unsigned long long *rec_size,
                              WsStatus *st) {
  count_launch(st);
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > g.nblocks) return;
  if (b == g.nblocks) { rec_size[b] = 0; return; }
  if (blkp[b].trivial) { rec_size[b] = 1; return; }
  BlockBox bb = block_box(g, b);
  int64_t p0 = first_part(g, b);
  unsigned long long sz = 1 + 16 + 24ull * bb.np + 8;
  for (int i = 0; i < bb.np; i++) sz += 8ull * part_zeros[p0 + i] + (part_bits[p0 + i] + 7) / 8;
  rec_size[b] = sz;
}

__device__ __forceinline__ void put_bytes(uint8_t *p, const void *v, int n) {
  const uint8_t *s = (const uint8_t *)v;
  for (int i = 0; i < n; i++) p[i] = s[i];
}
__device__ __forceinline__ void put_u64(uint8_t *p, unsigned long long v) { put_bytes(p, &v, 8); }
__device__ __forceinline__ void put_f64(uint8_t *p, double v) { put_bytes(p, &v, 8); }

// K9: container header (D11, D12).
__global__ void k_write_header(uint8_t *out, Geom g, KParams k, uint64_t global_rows, const uint8_t *lens,
                               WsStatus *st) {
  count_launch(st);
  const int m = st->m;
  const int n = 1 << m;
  const uint64_t mb = model_blob_bytes(k.S, k.H);
  if (threadIdx.x == 0) {
    uint8_t *p = out;
    p[0] = 'P'; p[1] = 'M'; p[2] = 'E'; p[3] = 'Z';
    unsigned short ver = 1;
    put_bytes(p + 4, &ver, 2);
    p[6] = 0;
    unsigned long long rows = global_rows, cols = (unsigned long long)g.cols;
    put_u64(p + 7, rows);
    put_u64(p + 15, cols);
    unsigned br = k.block_rows, bcl = k.block_cols, pr = k.partition_rows;
    put_bytes(p + 23, &br, 4);
    put_bytes(p + 27, &bcl, 4);
    put_bytes(p + 31, &pr, 4);
    put_f64(p + 35, k.b_r);
    put_f64(p + 43, k.coverage_target);
    p[51] = (uint8_t)m;
    put_u64(p + 52, mb);
    uint8_t *q = p + 60;
    unsigned S = k.S, H = k.H;
    put_bytes(q, &S, 4);
    put_bytes(q + 4, &H, 4);
    put_f64(q + 8, k.slope);
    int nw1 = (k.S + 1) * k.H;
    for (int i = 0; i < nw1; i++) put_f64(q + 16 + 8 * i, k.w1[i]);
    for (int i = 0; i < k.H; i++) put_f64(q + 16 + 8 * nw1 + 8 * i, k.w2[i]);
    q += mb;
    put_u64(q, 2ull + n);
    unsigned short a16 = (unsigned short)(n & 0xffff);
    put_bytes(q + 8, &a16, 2);
    unsigned long long gnb = ((global_rows + k.block_rows - 1) / k.block_rows) * (unsigned long long)g.nbc;
    put_u64(q + 10 + n, gnb);
  }
  uint8_t *L = out + 60 + mb + 10;
  for (int i = threadIdx.x; i < n; i += blockDim.x) L[i] = lens[i];
}

// MSB-first OR of a codeword (len <= 32) into a little-endian u32 smem window
// at window bit position `bit` (bit i of the stream = bit 7 - i%8 of byte i/8).
__device__ __forceinline__ void or_bits_smem(unsigned *win, unsigned bit, unsigned code, int len) {
  if (len == 0) return;
  const unsigned o = bit & 7;
  const unsigned long long w = ((unsigned long long)code) << (64 - len - o);  // big-endian window
  const int nbytes = (int)((o + len + 7) >> 3);
  const unsigned byte0 = bit >> 3;
#pragma unroll
  for (int i = 0; i < 5; i++) {
    if (i < nbytes) {
      const unsigned by = (unsigned)((w >> (56 - 8 * i)) & 0xff);
      if (by) {
        const unsigned bi = byte0 + i;
        atomicOr(&win[bi >> 2], by << (8 * (bi & 3)));
      }
    }
  }
}

constexpr int kWinWords = 1024;  // 4 KB bit-packing window per warp

// K10: write one block record per CTA (D9, D13, D15).  Each warp
// packs a partition's codewords into a shared-memory window (warp prefix sum
// of code lengths -> bit offsets, smem atomics) and flushes finished bytes to
// the (byte-aligned, unaligned-to-word) output with coalesced byte stores.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_write_records(Geom g, const BlkP *__restrict__ blkp,
                                                           const uint16_t *__restrict__ codes,
                                                           const double *__restrict__ balv,
                                                           const double *__restrict__ anchors,
                                                           const unsigned long long *__restrict__ part_bits,
                                                           const unsigned long long *__restrict__ part_zeros,
                                                           const unsigned long long *__restrict__ rec_off,
                                                           const uint8_t *__restrict__ lens,
                                                           const unsigned *__restrict__ cw, uint8_t *out,
                                                           unsigned long long rec_base, WsStatus *st) {
  __shared__ unsigned s_win[NW][kWinWords];
  __shared__ unsigned long long s_zb[64], s_pb[64];
  __shared__ unsigned long long s_nbal;
  count_launch(st);
  const int64_t b = blockIdx.x;
  uint8_t *base = out + rec_base + rec_off[b];
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (threadIdx.x == 0) base[0] = 1;
    return;
  }
  const BlockBox bb = block_box(g, b);
  const int64_t p0 = first_part(g, b);
  if (threadIdx.x == 0) {
    unsigned long long zb = 0, pb = 0;
    for (int i = 0; i < bb.np; i++) {
      s_zb[i] = zb;
      s_pb[i] = pb;
      zb += part_zeros[p0 + i];
      pb += (part_bits[p0 + i] + 7) / 8;
    }
    s_nbal = zb;
  }
  __syncthreads();
  // fixed head: trivial flag, factors, partition table, balance count (coalesced bytes)
  const unsigned head = 25 + 24u * bb.np;
  for (unsigned i = threadIdx.x; i < head; i += blockDim.x) {
    unsigned long long word;
    unsigned byte;
    if (i == 0) { base[0] = 0; continue; }
    if (i < 17) {
      word = __double_as_longlong(i < 9 ? P.factor_pos : P.factor_neg);
      byte = (i - 1) & 7;
    } else if (i < 17 + 24u * bb.np) {
      const unsigned q = i - 17, pi = q / 24, f = (q % 24) / 8;
      word = f == 0 ? s_pb[pi] * 8 : (f == 1 ? part_bits[p0 + pi] : __double_as_longlong(anchors[p0 + pi]));
      byte = q & 7;
    } else {
      word = s_nbal;
      byte = (i - 17 - 24u * bb.np) & 7;
    }
    base[i] = (uint8_t)(word >> (8 * byte));
  }
  uint8_t *bal0 = base + head;
  uint8_t *pay0 = bal0 + 8ull * s_nbal;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned *win = s_win[warp];
  for (int pi = warp; pi < bb.np; pi += NW) {
    const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
    uint8_t *pay = pay0 + s_pb[pi];
    for (int i = lane; i < kWinWords; i += 32) win[i] = 0;
    __syncwarp();
    unsigned long long zb = s_zb[pi];
    unsigned long long bit = 0, wbase = 0;  // partition bit position, window base (bits, multiple of 32)
    const int n = R * C;
    const uint16_t *cbase = codes + (bb.r0 + pr0) * g.cols + bb.c0;
    const double *bbase = balv + (bb.r0 + pr0) * g.cols + bb.c0;
    auto load_code = [&](int e, int &r, int &c) -> int {
      r = 0;
      c = 0;
      if (e < n && e > 0) {
        r = (int)((unsigned)e / (unsigned)C);
        c = e - r * C;
        return __ldg(&cbase[(int64_t)r * g.cols + c]);
      }
      return -1;
    };
    int nr, nc;
    int ncode = load_code(lane, nr, nc);
    for (int e0 = 0; e0 < n; e0 += 32) {
      const int code = ncode, r = nr, c = nc;
      ncode = load_code(e0 + 32 + lane, nr, nc);  // prefetch the next 32 codes
      const unsigned zmask = __ballot_sync(0xffffffffu, code == 0);
      if (code == 0) {
        const unsigned idx = __popc(zmask & ((1u << lane) - 1));
        const unsigned long long v = __double_as_longlong(bbase[(int64_t)r * g.cols + c]);
        uint8_t *d = bal0 + 8ull * (zb + idx);
#pragma unroll
        for (int q = 0; q < 8; q++) d[q] = (uint8_t)(v >> (8 * q));
      }
      zb += __popc(zmask);
      const int len = code >= 0 ? __ldg(&lens[code]) : 0;
      unsigned s = len;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
      }
      if (code >= 0) or_bits_smem(win, (unsigned)(bit + (s - len) - wbase), __ldg(&cw[code]), len);
      bit += __shfl_sync(0xffffffffu, s, 31);
      __syncwarp();
      if (bit - wbase > (unsigned long long)(kWinWords - 64) * 32) {
        // flush the whole words below the current position
        const unsigned nw = (unsigned)((bit - wbase) >> 5);
        uint8_t *dst = pay + (wbase >> 3);
        const uint8_t *wb = reinterpret_cast<const uint8_t *>(win);
        for (unsigned i = lane; i < nw * 4; i += 32) dst[i] = wb[i];
        __syncwarp();
        const unsigned keep = win[nw];
        __syncwarp();
        for (int i = lane; i < kWinWords; i += 32) win[i] = 0;
        __syncwarp();
        if (lane == 0) win[0] = keep;
        __syncwarp();
        wbase += (unsigned long long)nw * 32;
      }
    }
    // final flush, zero-padded to the byte boundary (D15)
    const unsigned nbytes = (unsigned)(((bit + 7) >> 3) - (wbase >> 3));
    uint8_t *dst = pay + (wbase >> 3);
    const uint8_t *wb = reinterpret_cast<const uint8_t *>(win);
    for (unsigned i = lane; i < nbytes; i += 32) dst[i] = wb[i];
    __syncwarp();
  }
}

// Store 8 little-endian bytes at an arbitrary byte address with at most four
// naturally aligned stores.
__device__ __forceinline__ void put8_unaligned(uint8_t *p, unsigned long long v) {
  const unsigned a = (unsigned)(reinterpret_cast<uintptr_t>(p) & 7);
  if (a == 0) { *reinterpret_cast<unsigned long long *>(p) = v; return; }
  if ((a & 3) == 0) {
    reinterpret_cast<unsigned *>(p)[0] = (unsigned)v;
    reinterpret_cast<unsigned *>(p)[1] = (unsigned)(v >> 32);
    return;
  }
  if ((a & 1) == 0) {  // a = 2 or 6
    *reinterpret_cast<uint16_t *>(p) = (uint16_t)v;
    *reinterpret_cast<unsigned *>(p + 2) = (unsigned)(v >> 16);
    *reinterpret_cast<uint16_t *>(p + 6) = (uint16_t)(v >> 48);
    return;
  }
  if ((a & 3) == 1) {  // a = 1 or 5
    p[0] = (uint8_t)v;
    *reinterpret_cast<uint16_t *>(p + 1) = (uint16_t)(v >> 8);
    *reinterpret_cast<unsigned *>(p + 3) = (unsigned)(v >> 24);
    p[7] = (uint8_t)(v >> 56);
    return;
  }
  // a = 3 or 7
  p[0] = (uint8_t)v;
  *reinterpret_cast<unsigned *>(p + 1) = (unsigned)(v >> 8);
  *reinterpret_cast<uint16_t *>(p + 5) = (uint16_t)(v >> 40);
  p[7] = (uint8_t)(v >> 56);
}

// OR one byte into global memory (the containing aligned word, atomically).
__device__ __forceinline__ void or_byte(uint8_t *p, unsigned v) {
  if (!v) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  atomicOr(reinterpret_cast<unsigned *>(a & ~(uintptr_t)3), v << (8 * (unsigned)(a & 3)));
}

// K10 (v2): one warp per partition.  The partition's codes are staged in
// shared memory (coalesced), lane j owns a contiguous run of them in raster
// order (the anchor excluded, D1): pass 1 sums code lengths, a warp scan gives
// each lane its bit offset, pass 2 packs the codewords MSB-first in a 64-bit
// register and stores whole bytes (the <= 2 bytes a lane shares with its
// neighbours are zeroed first and OR-ed atomically).  The balance list is
// written by a lane-parallel ballot pass.  The warp of partition 0 also writes
// the block's record head (D9, D13, D15).
#ifdef PMZ_CMP_PROFILE
__device__ long long g_wr_prof[65536][6];
#define WR_STAMP(i) if (lane == 0 && p < 65536) g_wr_prof[p][i] = clock64();
#else
#define WR_STAMP(i)
#endif
constexpr unsigned kPackWords = 2048;  // 8 KB packed payload per warp in smem (else direct global path)

template <int NW>
__global__ void __launch_bounds__(NW * 32) k_write_records2(Geom g, const BlkP *__restrict__ blkp,
                                                            const uint16_t *__restrict__ codes,
                                                            const double *__restrict__ balv,
                                                            const double *__restrict__ anchors,
                                                            const unsigned long long *__restrict__ part_bits,
                                                            const unsigned long long *__restrict__ part_zeros,
                                                            const unsigned long long *__restrict__ rec_off,
                                                            const uint8_t *__restrict__ lens,
                                                            const unsigned *__restrict__ cw, int m, uint8_t *out,
                                                            unsigned long long rec_base,
                                                            const uint16_t *__restrict__ zrow, WsStatus *st) {
  __shared__ uint8_t s_len[4096];
  __shared__ unsigned s_cw[4096];
  extern __shared__ __align__(16) uint16_t s_codes_all[];
  count_launch(st);
  const bool small_tab = m <= 12;
  if (small_tab) {
    for (int i = threadIdx.x; i < (1 << m); i += blockDim.x) {
      s_len[i] = lens[i];
      s_cw[i] = cw[i];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * NW + warp;
  if (p >= g.nparts) return;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  uint8_t *base = out + rec_base + rec_off[b];
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (pi == 0 && lane == 0) base[0] = 1;
    return;
  }
  WR_STAMP(0)
  const BlockBox bb = block_box(g, b);
  const int64_t p0 = first_part(g, b);
  unsigned long long zb = 0, pb = 0, nbal = 0;
  for (int i = 0; i < bb.np; i++) {
    const unsigned long long z = part_zeros[p0 + i], by = (part_bits[p0 + i] + 7) / 8;
    if (i < pi) { zb += z; pb += by; }
    nbal += z;
  }
  const unsigned head = 25 + 24u * bb.np;
  if (pi == 0) {
    // record head: trivial flag, factors, partition table, balance count
    for (unsigned i = lane; i < head; i += 32) {
      unsigned long long word;
      unsigned byte;
      if (i == 0) { base[0] = 0; continue; }
      if (i < 17) {
        word = __double_as_longlong(i < 9 ? P.factor_pos : P.factor_neg);
        byte = (i - 1) & 7;
      } else if (i < 17 + 24u * bb.np) {
        const unsigned q = i - 17, pq = q / 24, f = (q % 24) / 8;
        if (f == 0) {
          unsigned long long off = 0;
          for (unsigned t = 0; t < pq; t++) off += (part_bits[p0 + t] + 7) / 8;
          word = off * 8;
        } else {
          word = f == 1 ? part_bits[p0 + pq] : __double_as_longlong(anchors[p0 + pq]);
        }
        byte = q & 7;
      } else {
        word = nbal;
        byte = (i - 17 - 24u * bb.np) & 7;
      }
      base[i] = (uint8_t)(word >> (8 * byte));
    }
  }
  uint8_t *bal = base + head + 8ull * zb;
  uint8_t *pay = base + head + 8ull * nbal + pb;
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const uint16_t *cp = codes + (bb.r0 + pr0) * g.cols + bb.c0;
  uint16_t *sc = s_codes_all + (size_t)warp * ((size_t)g.prow * g.bc + 160 + 2 * kPackWords + 4);
  const unsigned n = (unsigned)(R * C - 1);  // codes at raster indices 1..n
  // lane j packs codes [1 + j RUN, 1 + (j+1) RUN); they are staged at
  // sc[j STRIDE + i] with STRIDE/2 odd so the 32 lanes hit 32 different banks
  const unsigned RUN = (n + 31) / 32;
  unsigned STRIDE = RUN + 1;
  while ((STRIDE & 1) || !((STRIDE >> 1) & 1)) STRIDE++;
  const unsigned rrun = RUN > 1 ? (unsigned)(0x100000000ull / RUN) + 1u : 0u;  // floor(x/RUN) = umulhi(x, rrun)
  auto spos = [&](unsigned e) -> unsigned {  // e >= 1
    const unsigned x = e - 1, j = RUN > 1 ? __umulhi(x, rrun) : x;
    return j * STRIDE + (x - j * RUN);
  };
  // stage the partition's codes (coalesced global reads)
  for (int r = 0; r < R; r++)
    for (int c = lane; c < C; c += 32) {
      const unsigned e = (unsigned)(r * C + c);
      if (e) sc[spos(e)] = __ldg(&cp[(int64_t)r * g.cols + c]);
    }
  __syncwarp();
  WR_STAMP(1)
  // balance list: the compress kernel left each row's balance values
  // compacted at the start of the row segment (zrow = counts): contiguous,
  // coalesced copies at row offsets from a warp scan of the counts
  {
    const double *bp = balv + (bb.r0 + pr0) * g.cols + bb.c0;
    const unsigned zc = lane < R ? zrow[p * 32 + lane] : 0u;
    unsigned zi = zc;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, zi, d);
      if (lane >= d) zi += t;
    }
    zi -= zc;  // exclusive
    // flattened over the partition's whole list: element i belongs to the
    // last row whose exclusive prefix is <= i (5-step search over the lanes'
    // prefixes); 4 independent loads in flight per lane
    const unsigned T = __shfl_sync(0xffffffffu, zi + zc, 31);
    for (unsigned i0 = 0; i0 < T; i0 += 128) {
      unsigned long long v[4];
      unsigned ii[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const unsigned i = i0 + u * 32 + lane;
        int r = 0;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
          const unsigned zr = __shfl_sync(0xffffffffu, zi, r + d);
          if (r + d < R && zr <= i) r += d;
        }
        const unsigned rb = __shfl_sync(0xffffffffu, zi, r);
        ii[u] = i;
        v[u] = i < T ? __double_as_longlong(__ldg(&bp[(int64_t)r * g.cols + (i - rb)])) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (ii[u] < T) put8_unaligned(bal + 8ull * ii[u], v[u]);
    }
  }
  WR_STAMP(2)
  auto len_of = [&](unsigned c) -> unsigned { return small_tab ? s_len[c] : __ldg(&lens[c]); };
  auto cw_of = [&](unsigned c) -> unsigned { return small_tab ? s_cw[c] : __ldg(&cw[c]); };
  const unsigned e0 = min(n + 1, 1 + lane * RUN), e1 = min(n + 1, 1 + (lane + 1) * RUN);
  const uint16_t *myc = sc + lane * STRIDE;
  unsigned bits = 0;
#pragma unroll 8
  for (unsigned e = e0; e < e1; e++) bits += len_of(myc[e - e0]);
  unsigned ib = bits;
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, ib, d);
    if (lane >= d) ib += t;
  }
  const unsigned B = ib - bits;
  const unsigned total_bits = __shfl_sync(0xffffffffu, ib, 31);
  const unsigned nwords = (total_bits + 31) >> 5;
  unsigned *sw = reinterpret_cast<unsigned *>(sc + 32 * STRIDE + 2);  // payload words after the codes
  if (nwords <= kPackWords) {
    // MSB-first words in shared memory: interior words stored, the two words a
    // lane may share with its neighbours OR-ed (zeroed first)
    sw = reinterpret_cast<unsigned *>((reinterpret_cast<uintptr_t>(sw) + 3) & ~(uintptr_t)3);
    const unsigned fw = B >> 5, lw = bits ? (B + bits - 1) >> 5 : fw;
    if (bits) { sw[fw] = 0; sw[lw] = 0; }
    __syncwarp();
    WR_STAMP(3)
    unsigned long long acc = 0;
    int nacc = (int)(B & 31);
    unsigned ow = fw;
#pragma unroll 4
    for (unsigned e = e0; e < e1; e++) {
      const unsigned cd = myc[e - e0];
      const int l = (int)len_of(cd);
      acc = (acc << l) | cw_of(cd);
      nacc += l;
      if (nacc >= 32) {
        const unsigned w = (unsigned)(acc >> (nacc - 32));
        if (ow == fw || ow == lw) atomicOr(&sw[ow], w);
        else sw[ow] = w;
        ow++;
        nacc -= 32;
      }
    }
    if (nacc > 0) atomicOr(&sw[ow], (unsigned)(acc << (32 - nacc)));
    __syncwarp();
    // coalesced byte copy to the (byte-aligned) payload
    const unsigned nbytes = (total_bits + 7) >> 3;
    for (unsigned i = lane; i < nbytes; i += 32) pay[i] = (uint8_t)(sw[i >> 2] >> (24 - 8 * (i & 3)));
  } else {
    const unsigned fbyte = B >> 3, lbyte = bits ? (B + bits - 1) >> 3 : fbyte;
    if (bits) {
      pay[fbyte] = 0;
      pay[lbyte] = 0;
    }
    __syncwarp();
    unsigned long long acc = 0;
    int nacc = (int)(B & 7);  // leading bits owned by the previous lane
    unsigned outb = fbyte;
    for (unsigned e = e0; e < e1; e++) {
      const unsigned cd = myc[e - e0];
      const int l = (int)len_of(cd);
      acc = (acc << l) | cw_of(cd);
      nacc += l;
      while (nacc >= 8) {
        const unsigned byte = (unsigned)(acc >> (nacc - 8)) & 0xffu;
        if (outb == fbyte || outb == lbyte) or_byte(pay + outb, byte);
        else pay[outb] = (uint8_t)byte;
        outb++;
        nacc -= 8;
      }
    }
    if (nacc > 0) or_byte(pay + outb, (unsigned)(acc << (8 - nacc)) & 0xffu);
  }
  __syncwarp();
  WR_STAMP(4)
}

// One block record's share written by ONE CTA per partition (kWT threads):
// the record head (partition 0 only), the partition's slice of the block
// balance list, and its Huffman substream.  Thread t
// encodes the raster run [t RUN, (t+1) RUN) of the partition (raster index 0
// = the anchor, not coded, D1); bit offsets come from a CTA-wide scan of the
// runs' bit counts; words are assembled MSB-first in shared memory and copied
// out coalesced.
constexpr int kWT = 256;
constexpr unsigned kPartWords = 4096;  // 16 KB payload staging (else direct byte writes)

__global__ void __launch_bounds__(kWT) k_write_part(Geom g, const BlkP *__restrict__ blkp,
                                                    const uint16_t *__restrict__ codes,
                                                    const double *__restrict__ balv,
                                                    const double *__restrict__ anchors,
                                                    const unsigned long long *__restrict__ part_bits,
                                                    const unsigned long long *__restrict__ part_zeros,
                                                    const unsigned long long *__restrict__ rec_off,
                                                    const uint8_t *__restrict__ lens,
                                                    const unsigned *__restrict__ cw, int m, uint8_t *out,
                                                    unsigned long long rec_base,
                                                    const uint16_t *__restrict__ zrow, WsStatus *st) {
  __shared__ uint8_t s_len[4096];
  __shared__ unsigned s_cw[4096];
  __shared__ unsigned sw[kPartWords];
  __shared__ unsigned s_wsum[kWT / 32], s_zi[33];
  count_launch(st);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  uint8_t *base = out + rec_base + rec_off[b];
  const BlkP P = blkp[b];
  if (P.trivial) {
    if (pi == 0 && tid == 0) base[0] = 1;
    return;
  }
  const bool small_tab = m <= 12;
  if (small_tab) {
    for (int i = tid; i < (1 << m); i += kWT) {
      s_len[i] = lens[i];
      s_cw[i] = cw[i];
    }
  }
  const BlockBox bb = block_box(g, b);
  const int64_t p0 = first_part(g, b);
  unsigned long long zb = 0, pb = 0, nbal = 0;
  for (int i = 0; i < bb.np; i++) {
    const unsigned long long z = part_zeros[p0 + i], by = (part_bits[p0 + i] + 7) / 8;
    if (i < pi) { zb += z; pb += by; }
    nbal += z;
  }
  const unsigned head = 25 + 24u * bb.np;
  if (pi == 0) {
    // record head: trivial flag, factors, partition table, balance count
    for (unsigned i = tid; i < head; i += kWT) {
      unsigned long long word;
      unsigned byte;
      if (i == 0) { base[0] = 0; continue; }
      if (i < 17) {
        word = __double_as_longlong(i < 9 ? P.factor_pos : P.factor_neg);
        byte = (i - 1) & 7;
      } else if (i < 17 + 24u * bb.np) {
        const unsigned q = i - 17, pq = q / 24, f = (q % 24) / 8;
        if (f == 0) {
          unsigned long long off = 0;
          for (unsigned t = 0; t < pq; t++) off += (part_bits[p0 + t] + 7) / 8;
          word = off * 8;
        } else {
          word = f == 1 ? part_bits[p0 + pq] : __double_as_longlong(anchors[p0 + pq]);
        }
        byte = q & 7;
      } else {
        word = nbal;
        byte = (i - 17 - 24u * bb.np) & 7;
      }
      base[i] = (uint8_t)(word >> (8 * byte));
    }
  }
  uint8_t *bal = base + head + 8ull * zb;
  uint8_t *pay = base + head + 8ull * nbal + pb;
  const int pr0 = pi * g.prow, R = min(g.prow, bb.br - pr0), C = bb.bc;
  const uint16_t *cp = codes + (bb.r0 + pr0) * g.cols + bb.c0;

  // ---- balance list: row-compacted by the compress kernel (zrow = counts) ----
  if (warp == 0) {
    const unsigned zc = lane < R ? zrow[p * 32 + lane] : 0u;
    unsigned zi = zc;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, zi, d);
      if (lane >= d) zi += t;
    }
    s_zi[lane] = zi - zc;
    if (lane == 31) s_zi[32] = zi;
  }
  __syncthreads();  // also publishes s_len / s_cw
  {
    const double *bp = balv + (bb.r0 + pr0) * g.cols + bb.c0;
    const unsigned T = s_zi[32];
    for (unsigned i = tid; i < T; i += kWT) {
      int r = 0;
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1)
        if (r + d < R && s_zi[r + d] <= i) r += d;
      put8_unaligned(bal + 8ull * i, __double_as_longlong(__ldg(&bp[(int64_t)r * g.cols + (i - s_zi[r])])));
    }
  }

  // ---- Huffman substream ----
  auto len_of = [&](unsigned c) -> unsigned { return small_tab ? s_len[c] : __ldg(&lens[c]); };
  auto cw_of = [&](unsigned c) -> unsigned { return small_tab ? s_cw[c] : __ldg(&cw[c]); };
  const unsigned ne = (unsigned)(R * C);
  const unsigned RUN = (ne + kWT - 1) / kWT;
  const unsigned e0 = min(ne, tid * RUN), e1 = min(ne, e0 + RUN);
  // element e -> (e / C, e % C): walk the run with a (row, col) cursor
  const int r0 = (int)(e0 / (unsigned)C), c0 = (int)(e0 - (unsigned)r0 * C);
  unsigned bits = 0;
  {
    int r = r0, c = c0;
#pragma unroll 8
    for (unsigned e = e0; e < e1; e++) {
      if (e) bits += len_of(__ldg(&cp[(int64_t)r * g.cols + c]));
      if (++c == C) { c = 0; r++; }
    }
  }
  // CTA exclusive scan of the runs' bit counts
  unsigned ib = bits;
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, ib, d);
    if (lane >= d) ib += t;
  }
  if (lane == 31) s_wsum[warp] = ib;
  __syncthreads();
  unsigned wofs = 0, total_bits = 0;
#pragma unroll
  for (int w = 0; w < kWT / 32; w++) {
    const unsigned v = s_wsum[w];
    if (w < warp) wofs += v;
    total_bits += v;
  }
  const unsigned B = wofs + ib - bits;
  const unsigned nwords = (total_bits + 31) >> 5;
  if (nwords <= kPartWords) {
    for (unsigned i = tid; i < nwords; i += kWT) sw[i] = 0;
    __syncthreads();
    const unsigned fw = B >> 5, lw = bits ? (B + bits - 1) >> 5 : fw;
    unsigned long long acc = 0;
    int nacc = (int)(B & 31);
    unsigned ow = fw;
    int r = r0, c = c0;
#pragma unroll 4
    for (unsigned e = e0; e < e1; e++) {
      if (e) {
        const unsigned cd = __ldg(&cp[(int64_t)r * g.cols + c]);
        const int l = (int)len_of(cd);
        acc = (acc << l) | cw_of(cd);
        nacc += l;
        if (nacc >= 32) {
          const unsigned w = (unsigned)(acc >> (nacc - 32));
          if (ow == fw || ow == lw) atomicOr(&sw[ow], w);
          else sw[ow] = w;
          ow++;
          nacc -= 32;
        }
      }
      if (++c == C) { c = 0; r++; }
    }
    if (nacc > 0) atomicOr(&sw[ow], (unsigned)(acc << (32 - nacc)));
    __syncthreads();
    const unsigned nbytes = (total_bits + 7) >> 3;
    for (unsigned i = tid; i < nbytes; i += kWT) pay[i] = (uint8_t)(sw[i >> 2] >> (24 - 8 * (i & 3)));
  } else {
    // oversized substream: bytes straight to global, boundary bytes OR-ed
    const unsigned fbyte = B >> 3, lbyte = bits ? (B + bits - 1) >> 3 : fbyte;
    if (bits) {
      pay[fbyte] = 0;
      pay[lbyte] = 0;
    }
    __syncthreads();
    unsigned long long acc = 0;
    int nacc = (int)(B & 7);
    unsigned outb = fbyte;
    int r = r0, c = c0;
    for (unsigned e = e0; e < e1; e++) {
      if (e) {
        const unsigned cd = __ldg(&cp[(int64_t)r * g.cols + c]);
        const int l = (int)len_of(cd);
        acc = (acc << l) | cw_of(cd);
        nacc += l;
        while (nacc >= 8) {
          const unsigned byte = (unsigned)(acc >> (nacc - 8)) & 0xffu;
          if (outb == fbyte || outb == lbyte) or_byte(pay + outb, byte);
          else pay[outb] = (uint8_t)byte;
          outb++;
          nacc -= 8;
        }
      }
      if (++c == C) { c = 0; r++; }
    }
    if (nacc > 0) or_byte(pay + outb, (unsigned)(acc << (8 - nacc)) & 0xffu);
  }
}

}  // namespace pmz
