// Isolated decode-loop micro-benchmark: one warp per "partition", every lane
// decodes a span of a synthetic canonical-Huffman stream from smem.
#include "../../paper_2309_09778_b200/csrc/capi.cu"
#include <vector>
#include <random>
#include <algorithm>
__global__ void bench(const unsigned *words, unsigned L, const unsigned *lut_g, const DecTab *tab_g, const uint16_t *sym,
                      uint16_t *dst, long long *cyc, unsigned *cnts, int mode) {
  __shared__ unsigned s_lut[1 << kLutBits];
  __shared__ DecTab s_tab;
  __shared__ unsigned stg[2051];
  for (int i = threadIdx.x; i < (1 << kLutBits); i += blockDim.x) s_lut[i] = lut_g[i];
  for (int i = threadIdx.x; i < 2051; i += blockDim.x) stg[i] = words[i];
  if (threadIdx.x == 0) s_tab = *tab_g;
  __syncthreads();
  SmemBits sb{stg};
  const int lane = threadIdx.x & 31;
  const unsigned s_i = L * lane / 32, s_n = lane == 31 ? L : L * (lane + 1) / 32;
  long long t0 = clock64();
  unsigned cnt = 0;
  if (mode == 0) {
    // bare loop: lut decode only
    unsigned cur = s_i;
    while (cur < s_n) {
      const unsigned w = sb.win32(cur);
      const unsigned e = s_lut[w >> (32 - kLutBits)];
      cur += e >> 16;
      cnt++;
    }
  } else if (mode == 1) {
    unsigned cur = s_i;
    while (cur < s_n) {
      int s, l; unsigned k;
      decode_run(sb, cur, s_n, L, s_lut, s_tab, sym, s, l, k);
      cur += k * l; cnt += k;
    }
  } else {
    DecOut o = write_span(sb, L, s_i, s_n, s_lut, s_tab, sym, 100000, dst + blockIdx.x * 8192, 0, 256, 256);
    cnt = o.cnt;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  cnts[blockIdx.x * 32 + lane] = cnt;
}
int main() {
  // code: m=8, lengths from a geometric-ish distribution around center
  const int m = 8, n = 1 << m;
  std::vector<uint64_t> f(n);
  for (int i = 0; i < n; i++) { int d = abs(i - 128); f[i] = d < 8 ? (1000 >> d) + 1 : 1; }
  std::vector<uint8_t> lens(n);
  // simple Huffman via repeated merging (not canonical tie-exact; fine for a benchmark)
  std::vector<std::pair<uint64_t, std::vector<int>>> nodes;
  for (int i = 0; i < n; i++) nodes.push_back({f[i], {i}});
  while (nodes.size() > 1) {
    std::sort(nodes.begin(), nodes.end(), [](auto &a, auto &b) { return a.first > b.first; });
    auto a = nodes.back(); nodes.pop_back(); auto b = nodes.back(); nodes.pop_back();
    for (int s : a.second) lens[s]++;
    for (int s : b.second) lens[s]++;
    a.second.insert(a.second.end(), b.second.begin(), b.second.end());
    nodes.push_back({a.first + b.first, a.second});
  }
  // canonical codes
  unsigned cntl[40] = {0}, next[40] = {0}; int maxl = 0;
  for (int i = 0; i < n; i++) { cntl[lens[i]]++; maxl = std::max(maxl, (int)lens[i]); }
  cntl[0] = 0; unsigned long long c = 0;
  for (int l = 1; l <= maxl; l++) { c = (c + cntl[l - 1]) << 1; next[l] = (unsigned)c; }
  std::vector<unsigned> cw(n);
  for (int i = 0; i < n; i++) cw[i] = next[lens[i]]++;
  // stream of 8191 symbols
  std::mt19937 rng(1);
  std::vector<unsigned> words(2051, 0);
  unsigned long long bit = 0;
  std::discrete_distribution<int> dist(f.begin(), f.end());
  for (int i = 0; i < 8191 && bit < 2040 * 32; i++) {
    int s = dist(rng);
    for (int b = lens[s] - 1; b >= 0; b--) { if ((cw[s] >> b) & 1) words[bit >> 5] |= 1u << (31 - (bit & 31)); bit++; }
  }
  unsigned L = (unsigned)bit;
  printf("stream bits %u, maxl %d\n", L, maxl);
  uint8_t *d_lens; unsigned *d_words, *d_lut, *d_cnts; DecTab *d_tab; uint16_t *d_sym, *d_dst; long long *d_cyc;
  cudaMalloc(&d_lens, n); cudaMemcpy(d_lens, lens.data(), n, cudaMemcpyHostToDevice);
  cudaMalloc(&d_words, 2051 * 4); cudaMemcpy(d_words, words.data(), 2051 * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&d_lut, 4 << kLutBits); cudaMalloc(&d_tab, sizeof(DecTab)); cudaMalloc(&d_sym, 2 * 65536);
  WsStatus *d_st; cudaMalloc(&d_st, sizeof(WsStatus)); cudaMemset(d_st, 0, sizeof(WsStatus));
  k_dec_tables<<<1, 1024>>>(d_lens, m, d_tab, d_sym, d_lut, d_st);
  cudaMalloc(&d_dst, 2 * 8192 * 256); cudaMalloc(&d_cyc, 8 * 256); cudaMalloc(&d_cnts, 4 * 32 * 256);
  for (int mode = 0; mode < 3; mode++) {
    for (int grid : {1}) {
      bench<<<grid, 32>>>(d_words, L, d_lut, d_tab, d_sym, d_dst, d_cyc, d_cnts, mode);
      cudaDeviceSynchronize();
      std::vector<long long> cyc(grid); std::vector<unsigned> cn(32 * grid);
      cudaMemcpy(cyc.data(), d_cyc, 8 * grid, cudaMemcpyDeviceToHost);
      cudaMemcpy(cn.data(), d_cnts, 4 * 32 * grid, cudaMemcpyDeviceToHost);
      unsigned mx = 0; for (int i = 0; i < 32; i++) mx = std::max(mx, cn[i]);
      printf("mode %d grid %d: %lld cycles, max lane symbols %u -> %.1f cycles/symbol-step\n", mode, grid, cyc[0], mx,
             (double)cyc[0] / mx);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
