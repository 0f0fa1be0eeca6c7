// encode.cuh -- validation histogram, canonical Huffman codebook, bit packing
// and container records (layout :496).
#pragma once
#include "common.cuh"

namespace pmz {

// K5: per-block code histograms of the validation blocks, summed (D10).
// Reads the final rq tiles (a block's partitions are consecutive, so its
// tiles are one contiguous range); code = code_of_rq(rq, center).
// Warp-aggregated: lanes holding the same code elect one leader (match_any).
template <int NT>
__global__ void __launch_bounds__(NT) k_val_hist(Geom g, const BlkP *__restrict__ blkp, const int64_t *val_ids,
                                                 const int16_t *__restrict__ rqbuf, unsigned long long *hist,
                                                 WsStatus *st) {
  count_launch(st);
  const int64_t b = val_ids[blockIdx.y];
  if (blkp[b].trivial) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&hist[kMaxAlpha], 1ull);  // k for the floor (D10)
  const int center = 1 << (st->m - 1);
  const BlockBox bb = block_box(g, b);
  const int64_t p0 = first_part(g, b);
  const int64_t n = (int64_t)bb.np * g.nct * kTile;
  const int16_t *rp = rqbuf + tile_base(g, p0, 0);
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * NT; base < n; base += (int64_t)gridDim.x * NT) {
    const int64_t i = base + threadIdx.x;
    int code = -1;
    if (i < n) {
      const int t = (int)(i >> 10), off = (int)(i & (kTile - 1));
      const int pi = t / g.nct, kc = t - pi * g.nct;
      const int r = off >> 5, c = kc * 32 + (off & 31);
      const int R = min(g.prow, bb.br - pi * g.prow);
      if (r < R && c < bb.bc && (r | c)) code = code_of_rq(__ldg(rp + i), center);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, code);
    if (code >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[code], (unsigned long long)__popc(peers));
  }
}

// Bitonic sort of n (power of two) u64 keys, ascending, by the first nt
// threads of a CTA (the others have exited).
__device__ void bitonic_sort(unsigned long long *a, int n, int nt) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += nt) {
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
// queue heads live in registers.  Two bulk steps reproduce runs of identical
// single steps in one go (large alphabets are mostly leaves floored at the
// same weight):
//   A. a run of r equal leaves not heavier than the internal head pairs off:
//      floor(r/2) leaf+leaf merges (the new nodes are heavier, so the head and
//      the tie rule stay the same throughout);
//   B. a run of equal internal nodes strictly lighter than the next leaf
//      pairs off (parents recorded).
// Runs are found by binary search (both queues are nondecreasing).
template <class Wt>
__device__ __forceinline__ void huff_merge(const unsigned long long *__restrict__ keys,
                                           unsigned long long *__restrict__ I, unsigned *__restrict__ P, int n) {
  const Wt INF = (Wt)~0ull;
  auto leafw = [&](int i) -> Wt { return i < n ? (Wt)(keys[i] >> 17) : INF; };
  auto intw = [&](int i) -> Wt { return (Wt)I[i]; };
  int li = 0, ii = 0, k = 0;
  Wt l0, l1, l2, l3, i0, i1, i2;
  auto refresh = [&]() {
    l0 = leafw(li); l1 = leafw(li + 1); l2 = leafw(li + 2); l3 = leafw(li + 3);
    i0 = ii < k ? intw(ii) : INF; i1 = ii + 1 < k ? intw(ii + 1) : INF; i2 = ii + 2 < k ? intw(ii + 2) : INF;
  };
  refresh();
  while (k < n - 1) {
    if (l0 == l1 && l1 != INF && l1 <= i0 && l3 == l0) {  // bulk A (runs >= 4)
      int lo = li + 3, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (leafw(mid) == l0) lo = mid; else hi = mid - 1;
      }
      const int nb = (lo - li + 1) >> 1;
      const unsigned long long w = 2ull * l0;
      for (int j = 0; j < nb; j++) I[k + j] = w;
      li += 2 * nb;
      k += nb;
      refresh();
      continue;
    }
    if (i0 == i1 && i1 != INF && i1 < l0 && i2 == i0 && ii + 3 < k && intw(ii + 3) == i0) {  // bulk B (runs >= 4)
      int lo = ii + 3, hi = k - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (intw(mid) == i0) lo = mid; else hi = mid - 1;
      }
      const int nb = (lo - ii + 1) >> 1;
      const unsigned long long w = 2ull * i0;
      for (int j = 0; j < nb; j++) {
        P[ii + 2 * j] = k + j;
        P[ii + 2 * j + 1] = k + j;
        I[k + j] = w;
      }
      ii += 2 * nb;
      k += nb;
      refresh();
      continue;
    }
    Wt w = 0;
#pragma unroll
    for (int pick = 0; pick < 2; pick++) {
      // internal only when strictly lighter (ties prefer the leaf); an
      // exhausted internal queue reads INF.  Branch-free: both refill loads
      // are unconditional (clamped in-bounds addresses, INF selected past
      // the end), a leaf pick writes its parent slot to the unused P[n-1].
      const bool tl = l0 <= i0;
      const Wt lk = (Wt)(keys[min(li + 4, n - 1)] >> 17);
      const Wt ik = intw(min(ii + 3, n - 1));
      const Wt nl3 = li + 4 < n ? lk : INF;
      const Wt ni2 = ii + 3 < k ? ik : INF;
      w += tl ? l0 : i0;
      P[tl ? n - 1 : ii] = (unsigned)k;
      l0 = tl ? l1 : l0; l1 = tl ? l2 : l1; l2 = tl ? l3 : l2; l3 = tl ? nl3 : l3;
      i0 = tl ? i0 : i1; i1 = tl ? i1 : i2; i2 = tl ? i2 : ni2;
      li += tl ? 1 : 0;
      ii += tl ? 0 : 1;
    }
    I[k] = (unsigned long long)w;
    if (ii == k) i0 = w;
    else if (ii + 1 == k) i1 = w;
    else if (ii + 2 == k) i2 = w;
    k++;
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
  const int m = st->m;
  const int n = 1 << m;
  // small alphabets: fewer threads, cheaper barriers (the rest exit now)
  const int nt = min((int)blockDim.x, max(128, n));
  if ((int)threadIdx.x >= nt) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool in_smem = n <= kCbSmemSyms;
  unsigned long long *keys = in_smem ? sm : g_keys;
  unsigned long long *I = in_smem ? sm + n : g_I;
  unsigned *P = in_smem ? reinterpret_cast<unsigned *>(sm + 2 * n) : g_P;
  CB_STAMP(0)
  const unsigned long long kval = hist[kMaxAlpha] > 0 ? hist[kMaxAlpha] : 1ull;
  if (tid < 64) s_cntI[tid] = 0;
  // ---- 1. leaves in (frequency, symbol) order: every symbol at or below the
  // floor k has weight k, the minimum, so those come first in index order;
  // only the symbols above the floor need sorting ----
  __shared__ unsigned s_wr[32][2], s_rb[2];
  if (tid < 2) s_rb[tid] = 0;
  // the real (above-floor) symbols are collected in a scratch array: the I
  // region (free until the merge), or the shared buffer for large alphabets
  unsigned long long *rk = in_smem ? I : sm;
  const bool rk_fits = in_smem || n <= 2 * kCbSmemSyms;  // 160 KB of shared memory = 20480 keys
  if (!rk_fits) rk = I;
  __syncthreads();
  for (int r0 = 0; r0 < n; r0 += nt) {
    const int s = r0 + tid;
    const unsigned long long f = s < n ? hist[s] : 0ull;
    const bool real = s < n && f > kval;
    const unsigned br = __ballot_sync(0xffffffffu, real), bf = __ballot_sync(0xffffffffu, s < n && !real);
    if (lane == 0) { s_wr[wid][0] = __popc(br); s_wr[wid][1] = __popc(bf); }
    __syncthreads();
    if (tid < 2) {
      unsigned acc = s_rb[tid];
      for (int w = 0; w < nt / 32; w++) { const unsigned t = s_wr[w][tid]; s_wr[w][tid] = acc; acc += t; }
      s_rb[tid] = acc;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1;
    if (real) rk[s_wr[wid][0] + __popc(br & lt)] = (f << 17) | (unsigned long long)s;
    else if (s < n) keys[s_wr[wid][1] + __popc(bf & lt)] = (kval << 17) | (unsigned long long)s;
    __syncthreads();
  }
  const int nr = (int)s_rb[0], nf = n - nr;
  int np2 = 1;
  while (np2 < nr) np2 <<= 1;
  for (int i = nr + tid; i < np2; i += nt) rk[i] = ~0ull;
  __syncthreads();
  CB_STAMP(1)
  if (nr > 1) bitonic_sort(rk, np2, nt);
  for (int i = tid; i < nr; i += nt) keys[nf + i] = rk[i];
  __syncthreads();
  CB_STAMP(2)
  // ---- 2. two-queue merge (thread 0) ----
  // 32-bit weights when the total (the root weight) fits: every node weight
  // is at most the total
  __shared__ unsigned long long s_total;
  if (tid == 0) s_total = 0;
  __syncthreads();
  {
    unsigned long long part = 0;
    for (int s2 = tid; s2 < n; s2 += nt) part += keys[s2] >> 17;
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) atomicAdd(&s_total, part);
  }
  __syncthreads();
  const bool w32 = s_total < 0xffffffffull;
  if (tid == 0) {
    if (in_smem) {
      if (w32) huff_merge<unsigned>(sm, sm + n, reinterpret_cast<unsigned *>(sm + 2 * n), n);
      else huff_merge<unsigned long long>(sm, sm + n, reinterpret_cast<unsigned *>(sm + 2 * n), n);
    } else {
      if (w32) huff_merge<unsigned>(g_keys, g_I, g_P, n);
      else huff_merge<unsigned long long>(g_keys, g_I, g_P, n);
    }
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

// K7: per-partition payload bits from the final rq tiles: one CTA per
// partition, warp w sums chunks w, w + 8, ... (8 residuals per 16-byte load,
// the anchor excluded).
constexpr int kPbW = 8;
__global__ void __launch_bounds__(kPbW * 32) k_part_bits(Geom g, const BlkP *__restrict__ blkp,
                                                        const int16_t *__restrict__ rqbuf,
                                                        const uint8_t *__restrict__ lens,
                                                        unsigned long long *part_bits, WsStatus *st) {
  __shared__ unsigned long long s_bits;
  count_launch(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = blockIdx.x;
  int64_t b;
  int pi;
  part_of(g, p, b, pi);
  if (threadIdx.x == 0) s_bits = 0;
  __syncthreads();
  if (!blkp[b].trivial) {
    const int center = 1 << (st->m - 1);
    const BlockBox bb = block_box(g, b);
    const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc, nch = (C + 31) >> 5;
    const uint4 *tp = reinterpret_cast<const uint4 *>(rqbuf + tile_base(g, p, 0));
    unsigned bits = 0;
    // vector v of a tile: row v >> 2, columns 8 (v & 3) .. + 7
    for (int kc = warp; kc < nch; kc += kPbW) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = __ldg(tp + kc * (kTile / 8) + lane + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int vi = lane + 32 * u, r = vi >> 2, c0 = kc * 32 + (vi & 3) * 8;
        if (r >= R) continue;
        const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int h = 0; h < 8; h++) {
          const int c = c0 + h;
          const int rq = (int)(int16_t)(w[h >> 1] >> (16 * (h & 1)));
          if (c < C && (r | c)) bits += __ldg(&lens[code_of_rq(rq, center)]);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o);
    if (lane == 0 && bits) atomicAdd(&s_bits, (unsigned long long)bits);
  }
  __syncthreads();
  if (threadIdx.x == 0) part_bits[p] = s_bits;
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
  if (st->err_bits) return;  // capacity / codebook errors: nothing is written
  const int m = st->m;
  const int n = 1 << m;
  const uint64_t mb = model_blob_bytes(k.S, k.H);
  if (threadIdx.x == 0) {
    uint8_t *p = out;
    p[0] = 'P'; p[1] = 'M'; p[2] = 'E'; p[3] = 'Z';
    unsigned short ver = k.precision ? 2 : 1;  // D12: 2 = FP32 perceptron perf mode
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

// Copy n bytes from shared memory (word-aligned source) to an arbitrary
// global byte address with aligned 32-bit stores (funnel-shifted source
// words; at most 3 + 3 bytes at the ends go out as single bytes).  CTA-wide.
__device__ __forceinline__ void copy_s2g_bytes(uint8_t *dst, const unsigned *src, unsigned n, int tid, int nt) {
  if (n == 0) return;
  const uint8_t *sb = reinterpret_cast<const uint8_t *>(src);
  const unsigned head = (unsigned)((4 - ((uintptr_t)dst & 3)) & 3);
  const unsigned hb = min(head, n);
  for (unsigned i = tid; i < hb; i += nt) dst[i] = sb[i];
  if (n <= hb) return;
  const unsigned nw = (n - hb) >> 2, tail = (n - hb) & 3;
  unsigned *dw = reinterpret_cast<unsigned *>(dst + hb);
  // output word j = source bytes [hb + 4j, hb + 4j + 4): little-endian words
  const unsigned sh = 8 * (hb & 3), wq = hb >> 2;
  for (unsigned j = tid; j < nw; j += nt) {
    const unsigned lo = src[wq + j];
    dw[j] = sh ? __funnelshift_r(lo, src[wq + j + 1], sh) : lo;
  }
  for (unsigned i = tid; i < tail; i += nt) dst[hb + 4 * nw + i] = sb[hb + 4 * nw + i];
}

// One block record's share written by ONE CTA per partition (kWT threads):
// the record head (partition 0 only), the partition's slice of the block
// balance list, and its Huffman substream (D9).
// A run is one 32-column tile-row segment of the partition (run q = row *
// nch + chunk: raster order); thread t owns runs t, t + kWT, ...  Per round of
// kWT runs: the 32 residuals come in four 16-byte loads, pass 1 counts bits
// and balance points (code 0; raster index 0 = the anchor is neither, D1), a
// CTA scan gives both offsets; balance values (TRUE surface, D9) are staged in
// shared memory and copied out with aligned word stores; codewords are
// assembled MSB-first into shared-memory words, copied out at the end.
constexpr int kWT = 256;
constexpr unsigned kPartWords = 4096;  // 16 KB payload staging (else direct byte writes)
#ifndef PMZ_BAL_STAGE
#define PMZ_BAL_STAGE 2048
#endif
constexpr unsigned kBalStage = PMZ_BAL_STAGE;   // balance values per staging sub-round
#ifndef PMZ_BAL_ILP
#define PMZ_BAL_ILP 4
#endif
constexpr int kWpTabM = 10;            // codebook tables in shared memory up to this m
constexpr size_t kWpSmem = (size_t)(1u << kWpTabM) * 5;

// The partition's runs (see k_write_part), with the codebook tables in shared
// memory (SMALL) or read through L1: a uniform branch per CTA instead of a
// predicated pair of loads per symbol.
template <bool SMALL>
__device__ __forceinline__ void wp_runs(const Geom &g, const BlkP &P, int64_t b, int64_t p, int pi,
                                        unsigned long long nbal, unsigned long long zb, unsigned long long pb,
                                        uint8_t *base, unsigned head, int m, const int16_t *__restrict__ rqbuf,
                                        const double *__restrict__ vbuf,
                                        const unsigned long long *__restrict__ part_bits,
                                        const uint8_t *__restrict__ lens, const unsigned *__restrict__ cw,
                                        const uint8_t *s_len, const unsigned *s_cw, unsigned *sw,
                                        unsigned long long *sbal, unsigned *s_bidx, unsigned (*s_wsum)[2],
                                        unsigned *s_carry) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const BlockBox bb = block_box(g, b);
  uint8_t *bal = base + head + 8ull * zb;
  uint8_t *pay = base + head + 8ull * nbal + pb;
  const int R = min(g.prow, bb.br - pi * g.prow), C = bb.bc, nch = (C + 31) >> 5;
  const int center = 1 << (m - 1);
  const int16_t *rp = rqbuf + tile_base(g, p, 0);
  const double *vp = vbuf + tile_base(g, p, 0);
  const unsigned total_bits = (unsigned)part_bits[p];
  const unsigned nwords = (total_bits + 31) >> 5;
  const bool staged = nwords <= kPartWords;
  auto len_of = [&](unsigned c) -> unsigned { return SMALL ? (unsigned)s_len[c] : (unsigned)__ldg(&lens[c]); };
  auto cw_of = [&](unsigned c) -> unsigned { return SMALL ? s_cw[c] : __ldg(&cw[c]); };
  const int nrun = R * nch;
  for (int q0 = 0; q0 < nrun; q0 += kWT) {
    const int q = q0 + tid;
    const bool valid = q < nrun;
    const int r = valid ? q / nch : 0, kc = valid ? q - r * nch : 0;
    const int ncol = valid ? min(32, C - 32 * kc) : 0;
    // the run's 32 residuals (16-byte aligned tile row)
    unsigned w[16];
    if (valid) {
      const uint4 *src = reinterpret_cast<const uint4 *>(rp + (int64_t)kc * kTile + r * 32);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint4 x4 = __ldg(src + u);
        w[4 * u] = x4.x; w[4 * u + 1] = x4.y; w[4 * u + 2] = x4.z; w[4 * u + 3] = x4.w;
      }
    }
    // codes of the run, two per register (computed once for both passes)
    const int i0 = (r == 0 && kc == 0) ? 1 : 0;  // the anchor
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const unsigned lo = (unsigned)code_of_rq((int)(int16_t)(w[u] & 0xffffu), center);
      const unsigned hi = (unsigned)code_of_rq((int)(int16_t)(w[u] >> 16), center);
      w[u] = lo | (hi << 16);
    }
    auto code_at = [&](int i) -> unsigned { return (w[i >> 1] >> (16 * (i & 1))) & 0xffffu; };
    unsigned bits = 0, zmask = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) {
      if (i >= i0 && i < ncol) {
        const unsigned cd = code_at(i);
        bits += len_of(cd);
        zmask |= (cd == 0 ? 1u : 0u) << i;
      }
    }
    const unsigned nz = __popc(zmask);
    // CTA scan of (bits, nz) over this round's runs, plus the carry
    unsigned ib = bits, iz = nz;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, ib, d), u = __shfl_up_sync(0xffffffffu, iz, d);
      if (lane >= d) { ib += t; iz += u; }
    }
    if (lane == 31) { s_wsum[warp][0] = ib; s_wsum[warp][1] = iz; }
    __syncthreads();
    unsigned wofs = s_carry[0], zofs = s_carry[1], rb = 0, rz = 0;
#pragma unroll
    for (int w2 = 0; w2 < kWT / 32; w2++) {
      const unsigned a = s_wsum[w2][0], z = s_wsum[w2][1];
      if (w2 < warp) { wofs += a; zofs += z; }
      rb += a;
      rz += z;
    }
    const unsigned B = wofs + ib - bits, Z = zofs + iz - nz;
    const unsigned zr0 = s_carry[1];  // first balance index of the round
    __syncthreads();
    if (tid == 0) { s_carry[0] += rb; s_carry[1] += rz; }

    // ---- balance values: staged sub-rounds of kBalStage values.  Runs list
    // their balance points' tile offsets, then the whole CTA gathers the
    // values (4 loads in flight per thread) and copies them out. ----
    for (unsigned s0 = zr0; s0 < zr0 + rz; s0 += kBalStage) {
      const unsigned s1 = min(zr0 + rz, s0 + kBalStage);
      if (nz && Z < s1 && Z + nz > s0) {
        unsigned zm = zmask, k = Z;
        const int tofs = kc * kTile + r * 32;
        while (zm) {
          const int i = __ffs(zm) - 1;
          zm &= zm - 1;
          if (k >= s0 && k < s1) s_bidx[k - s0] = tofs + i;
          k++;
        }
      }
      __syncthreads();
      const unsigned nv = s1 - s0;
      for (unsigned j0 = 0; j0 < nv; j0 += PMZ_BAL_ILP * kWT) {
        unsigned long long vv[PMZ_BAL_ILP];
#pragma unroll
        for (int u = 0; u < PMZ_BAL_ILP; u++) {
          const unsigned j = j0 + u * kWT + tid;
          vv[u] = j < nv ? __double_as_longlong(__ldg(vp + s_bidx[j])) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < PMZ_BAL_ILP; u++) {
          const unsigned j = j0 + u * kWT + tid;
          if (j < nv) sbal[j] = vv[u];
        }
      }
      __syncthreads();
      copy_s2g_bytes(bal + 8ull * s0, reinterpret_cast<const unsigned *>(sbal), 8 * nv, tid, kWT);
      __syncthreads();
    }

    // ---- codewords of the run ----
    if (staged) {
      const unsigned fw = B >> 5, lw = bits ? (B + bits - 1) >> 5 : fw;
      unsigned long long acc = 0;
      int nacc = (int)(B & 31);
      unsigned ow = fw;
#pragma unroll
      for (int i = 0; i < 32; i++) {
        if (i >= i0 && i < ncol) {
          const unsigned cd = code_at(i);
          const int l = (int)len_of(cd);
          acc = (acc << l) | cw_of(cd);
          nacc += l;
          if (nacc >= 32) {
            const unsigned wv = (unsigned)(acc >> (nacc - 32));
            if (ow == fw || ow == lw) atomicOr(&sw[ow], wv);
            else sw[ow] = wv;
            ow++;
            nacc -= 32;
          }
        }
      }
      if (nacc > 0) atomicOr(&sw[ow], (unsigned)(acc << (32 - nacc)));
    } else {
      // oversized substream: bytes straight to global, boundary bytes OR-ed
      const unsigned fbyte = B >> 3, lbyte = bits ? (B + bits - 1) >> 3 : fbyte;
      if (bits) {
        // a round's first run may share its first byte with the previous round
        if ((B & 7) == 0 || q != q0) pay[fbyte] = 0;
        pay[lbyte] = 0;
      }
      __syncthreads();
      unsigned long long acc = 0;
      int nacc = (int)(B & 7);
      unsigned outb = fbyte;
#pragma unroll
      for (int i = 0; i < 32; i++) {
        if (i < i0 || i >= ncol) continue;
        const unsigned cd = code_at(i);
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
      __syncthreads();
    }
  }
  if (staged) {  // MSB-first words -> byte order, then aligned word stores
    __syncthreads();
    for (unsigned i = tid; i < nwords; i += kWT) sw[i] = __byte_perm(sw[i], 0, 0x0123);
    __syncthreads();
    copy_s2g_bytes(pay, sw, (total_bits + 7) >> 3, tid, kWT);
  }
}

__global__ void __launch_bounds__(kWT) k_write_part(Geom g, const BlkP *__restrict__ blkp,
                                                    const int16_t *__restrict__ rqbuf,
                                                    const double *__restrict__ vbuf,
                                                    const double *__restrict__ anchors,
                                                    const unsigned long long *__restrict__ part_bits,
                                                    const unsigned long long *__restrict__ part_zeros,
                                                    const unsigned long long *__restrict__ rec_off,
                                                    const uint8_t *__restrict__ lens,
                                                    const unsigned *__restrict__ cw, uint8_t *out,
                                                    WsStatus *st) {
  extern __shared__ __align__(16) unsigned char wp_dyn[];
  __shared__ unsigned sw[kPartWords];
  __shared__ unsigned long long sbal[kBalStage + 1];
  __shared__ unsigned s_bidx[kBalStage];
  __shared__ unsigned s_wsum[kWT / 32][2];
  __shared__ unsigned s_carry[2];
  count_launch(st);
  // m, the header size and the capacity check come from the device status:
  // no host round trip between the codebook and the writers
  if (st->err_bits) return;
  const int m = st->m;
  const unsigned long long rec_base = st->header_bytes;
  const int tid = threadIdx.x;
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
  const bool small_tab = m <= kWpTabM;
  unsigned *s_cw = reinterpret_cast<unsigned *>(wp_dyn);
  uint8_t *s_len = wp_dyn + (4u << kWpTabM);
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
  for (unsigned i = tid; i < (((unsigned)part_bits[p] + 31) >> 5 <= kPartWords ? ((unsigned)part_bits[p] + 31) >> 5 : 0u);
       i += kWT)
    sw[i] = 0;
  if (tid < 2) s_carry[tid] = 0;
  __syncthreads();  // tables, sw, carry

  if (small_tab) wp_runs<true>(g, P, b, p, pi, nbal, zb, pb, base, head, m, rqbuf, vbuf, part_bits, lens, cw, s_len, s_cw, sw, sbal, s_bidx, s_wsum, s_carry);
  else wp_runs<false>(g, P, b, p, pi, nbal, zb, pb, base, head, m, rqbuf, vbuf, part_bits, lens, cw, s_len, s_cw, sw, sbal, s_bidx, s_wsum, s_carry);
}

}  // namespace pmz
