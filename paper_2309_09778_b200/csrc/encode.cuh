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
// sorted by (frequency, code); two-queue Huffman with ties preferring the leaf;
// canonical codewords in (length, code) order.  One CTA:
//   1. bitonic sort of (freq << 17 | sym) keys;
//   2. two-queue merge by ONE thread with the four queue heads cached in
//      registers (the only sequential part; internal weights u64, parent of
//      every internal node recorded);
//   3. internal-node depths by pointer jumping (parallel);
//   4. leaf depths from the per-depth internal counts (leaves at depth d =
//      2 I(d-1) - I(d), shallowest to the heaviest leaves -- the
//      Moffat-Katajainen leaf-depth assignment), parallel;
//   5. canonical codes: rank among equal-length symbols by match_any within
//      a warp + a per-(warp, length) scan, 1024 symbols per round.
// Scratch in smem when 2^m <= 8192 (20 B / symbol), else in the workspace.
#ifdef PMZ_CMP_PROFILE
__device__ long long g_cb_prof[8];
#define CB_STAMP(i) if (threadIdx.x == 0) g_cb_prof[i] = clock64();
#else
#define CB_STAMP(i)
#endif
// Two-queue Huffman merge over sorted leaves keys[0..n) (weight = key >> 17):
// internal node k gets weight I[k]; P[c] = parent of internal node c.  The
// queue heads live in registers, refilled 3-4 picks ahead of their use.
__device__ __forceinline__ void huff_merge(const unsigned long long *__restrict__ keys,
                                           unsigned long long *__restrict__ I, unsigned *__restrict__ P, int n) {
  const unsigned long long INF = ~0ull;
  auto leafw = [&](int i) -> unsigned long long { return i < n ? keys[i] >> 17 : INF; };
  int li = 0, ii = 0;
  unsigned long long l0 = leafw(0), l1 = leafw(1), l2 = leafw(2), l3 = leafw(3);
  unsigned long long i0 = INF, i1 = INF, i2 = INF;
  for (int k = 0; k < n - 1; k++) {
    unsigned long long w = 0;
#pragma unroll
    for (int pick = 0; pick < 2; pick++) {
      // internal only when strictly lighter (ties prefer the leaf); an
      // exhausted internal queue reads INF
      if (l0 <= i0) {
        w += l0;
        l0 = l1; l1 = l2; l2 = l3; l3 = leafw(li + 4); li++;
      } else {
        w += i0;
        P[ii] = k;
        i0 = i1; i1 = i2; i2 = (ii + 3 < k) ? I[ii + 3] : INF; ii++;
      }
    }
    I[k] = w;
    if (ii == k) i0 = w;
    else if (ii + 1 == k) i1 = w;
    else if (ii + 2 == k) i2 = w;
  }
  P[n - 2] = n - 2;  // root
}

constexpr int kCbSmemSyms = 8192;
constexpr size_t kCbSmem = (size_t)kCbSmemSyms * 20;

__global__ void __launch_bounds__(1024) k_codebook(const unsigned long long *hist, WsStatus *st,
                                                   unsigned long long *g_keys, unsigned long long *g_I,
                                                   unsigned *g_P, uint8_t *lens, unsigned *cw) {
  extern __shared__ unsigned long long sm[];
  __shared__ unsigned s_cntI[64], s_first[64], s_lcum[65];
  __shared__ unsigned s_wl[32][33];
  __shared__ int s_maxl;
  count_launch(st);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int m = st->m;
  const int n = 1 << m;
  const bool in_smem = n <= kCbSmemSyms;
  unsigned long long *keys = in_smem ? sm : g_keys;
  unsigned long long *I = in_smem ? sm + n : g_I;
  unsigned *P = in_smem ? reinterpret_cast<unsigned *>(sm + 2 * n) : g_P;
  CB_STAMP(0)
  const unsigned long long kval = hist[kMaxAlpha] > 0 ? hist[kMaxAlpha] : 1ull;
  for (int s = tid; s < n; s += nt) {
    unsigned long long f = hist[s];
    if (f < kval) f = kval;
    keys[s] = (f << 17) | (unsigned long long)s;
  }
  if (tid < 64) s_cntI[tid] = 0;
  __syncthreads();
  CB_STAMP(1)
  bitonic_sort(keys, n);
  CB_STAMP(2)
  // ---- 2. two-queue merge (thread 0) ----
  if (tid == 0) {
    if (in_smem) huff_merge(sm, sm + n, reinterpret_cast<unsigned *>(sm + 2 * n), n);
    else huff_merge(g_keys, g_I, g_P, n);
  }
  __syncthreads();
  CB_STAMP(3)
  // ---- 3. depths of the n-1 internal nodes: pointer jumping ----
  // D, Q overlay I (no longer needed): D[k] = distance to the root so far
  unsigned *D = reinterpret_cast<unsigned *>(I), *Q = D + n;
  const int ni = n - 1;
  for (int k = tid; k < ni; k += nt) {
    D[k] = k == ni - 1 ? 0u : 1u;
    Q[k] = P[k];
  }
  __syncthreads();
  for (int span = 1; span < ni; span <<= 1) {
    unsigned dn[8], qn[8];
    // ni <= 65535, nt = 1024: <= 64 nodes per thread, 8 per batch
    for (int k0 = 0; k0 < ni; k0 += 8 * nt) {
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int k = k0 + u * nt + tid;
        if (k < ni) {
          const unsigned q = Q[k];
          dn[u] = D[k] + D[q];
          qn[u] = Q[q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int k = k0 + u * nt + tid;
        if (k < ni) { D[k] = dn[u]; Q[k] = qn[u]; }
      }
      __syncthreads();
    }
  }
  for (int k = tid; k < ni; k += nt) atomicAdd(&s_cntI[min(D[k], 63u)], 1u);
  __syncthreads();
  // ---- 4. leaf depths ----
  if (tid == 0) {
    // leaves at depth d: 2 I(d-1) - I(d) (I(-1) = 1/2: the root level holds
    // no leaf when n >= 2); cumulative from the shallowest level
    unsigned cum = 0, prev = 0;
    int maxl = 0;
    s_lcum[0] = 0;
    for (int d = 1; d < 64; d++) {
      prev = s_cntI[d - 1];
      const unsigned leaves = 2 * prev - s_cntI[d];
      cum += leaves;
      s_lcum[d] = cum;
      if (leaves) maxl = d;
    }
    s_lcum[64] = cum;
    s_maxl = maxl;
  }
  __syncthreads();
  const int maxl = s_maxl;
  for (int j = tid; j < n; j += nt) {
    // the t-th heaviest leaf (t = n-1-j) sits at the first depth d with t < lcum[d]
    const unsigned t = (unsigned)(n - 1 - j);
    int d = 1;
    while (d < 64 && t >= s_lcum[d]) d++;
    lens[keys[j] & 0x1ffff] = (uint8_t)d;
  }
  __syncthreads();
  CB_STAMP(4)
  if (tid == 0) st->max_len = maxl;
  if (maxl > 32) {
    if (tid == 0) atomicOr(&st->err_bits, 1u << (-PMZ_ERR_UNASSIGNED));
    return;
  }
  // ---- 5. canonical codes: first code per length ----
  if (tid == 0) {
    unsigned cnt[34];
    for (int l = 0; l <= 33; l++) cnt[l] = 0;
    for (int d = 1; d <= maxl; d++) cnt[d] = s_lcum[d] - s_lcum[d - 1];
    unsigned long long c = 0;
    s_first[0] = 0;
    for (int l = 1; l <= 32; l++) { c = (c + cnt[l - 1]) << 1; s_first[l] = (unsigned)c; }
  }
  __syncthreads();
  // running per-length base: ranks handed out in earlier rounds
  __shared__ unsigned s_base[33];
  if (tid < 33) s_base[tid] = 0;
  __syncthreads();
  for (int r0 = 0; r0 < n; r0 += nt) {
    const int i = r0 + tid;
    const int l = i < n ? lens[i] : 0;
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const unsigned rank = __popc(peers & ((1u << lane) - 1));
    // per-warp counts per length
    for (int q = lane; q < 33; q += 32) s_wl[wid][q] = 0;
    __syncwarp();
    if (i < n && rank == 0) s_wl[wid][l] = __popc(peers);
    __syncthreads();
    // exclusive scan over warps, per length (thread = length)
    if (tid < 33) {
      unsigned acc = s_base[tid];
      for (int w = 0; w < nt / 32; w++) { const unsigned t = s_wl[w][tid]; s_wl[w][tid] = acc; acc += t; }
      s_base[tid] = acc;
    }
    __syncthreads();
    if (i < n) cw[i] = l ? s_first[l] + s_wl[wid][l] + rank : 0u;
    __syncthreads();
  }
  CB_STAMP(5)
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
