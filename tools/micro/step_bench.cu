// Decode-step latency micro-benchmark: one warp, lanes decode their segment of
// a staged substream (partition P of a container) with variants of the step.
#include "../../paper_2309_09778_b200/csrc/capi.cu"
#include <vector>
#include <cmath>
using namespace pmz;

template <int V>
__global__ void k_step(const unsigned *words, unsigned L, const unsigned *lut, DecTab tab, const uint16_t *sym,
                       long long *out) {
  __shared__ unsigned stage[2052], bm[2052], s_lut[4096], s_lut2[2048];
  for (int i = threadIdx.x; i < 2052; i += 32) stage[i] = words[i];
  for (int i = threadIdx.x; i < 4096; i += 32) s_lut[i] = lut[i];
  for (int i = threadIdx.x; i < 2048; i += 32) s_lut2[i] = lut[4096 + i];
  __syncwarp();
  const int lane = threadIdx.x;
  const unsigned segw = (((L + 31) >> 5) + 31) >> 5;
  const unsigned s_i = min(L, 32 * segw * lane), s_n = min(L, 32 * segw * (lane + 1));
  D3Smem ss{stage};
  long long t0 = clock64();
  unsigned steps = 0, syms = 0;
  D3Reader<D3Smem> rd;
  rd.seek(ss, s_i, 0);
  unsigned pos = s_i, accw = s_i >> 5, acc = 0;
  while (pos < s_n) {
    steps++;
    if (V == 0) {  // full: mark + run
      if ((pos >> 5) != accw) { bm[accw] = acc; accw = pos >> 5; acc = 0; }
      acc |= 1u << (pos & 31);
    }
    rd.refill(ss);
    int s, l;
    unsigned k;
    if (V <= 1) {
      if (!d3_run(rd.buf, rd.nb, s_n - pos, s_lut, s_lut2, tab, sym, s, l, k)) break;
    } else {  // LUT only, k = 1
      const unsigned top = (unsigned)(rd.buf >> 32);
      unsigned e = s_lut[top >> 20];
      if (e & kLutL2Flag) e = s_lut2[(e & 0xffffu) + ((top << 12) >> (32 - tab.sub_bits))];
      l = (int)((e >> 16) & 31u);
      k = 1;
    }
    const unsigned adv = k * (unsigned)l;
    rd.skip(adv);
    pos += adv;
    syms += k;
  }
  long long t1 = clock64();
  bm[0] = acc;
  unsigned mx = steps, ms = syms;
  for (int d = 16; d > 0; d >>= 1) { mx = max(mx, __shfl_xor_sync(~0u, mx, d)); ms = max(ms, __shfl_xor_sync(~0u, ms, d)); }
  if (lane == 0) { out[0] = t1 - t0; out[1] = mx; out[2] = ms; }
}

int main(int argc, char **argv) {
  FILE *f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
  std::vector<uint8_t> h(n); fread(h.data(), 1, n, f); fclose(f);
  pmz_header hd; pmz_parse_header(h.data(), n, &hd);
  std::vector<uint64_t> offs(hd.nblocks + 1); pmz_index_blocks(h.data(), n, &hd, offs.data());
  uint8_t *d_buf; cudaMalloc(&d_buf, n); cudaMemcpy(d_buf, h.data(), n, cudaMemcpyHostToDevice);
  uint64_t *d_off; cudaMalloc(&d_off, 8 * offs.size()); cudaMemcpy(d_off, offs.data(), 8 * offs.size(), cudaMemcpyHostToDevice);
  float *d_out; cudaMalloc(&d_out, 4 * hd.rows * hd.cols);
  uint64_t wsb; pmz_decompress_workspace_size(&hd, &wsb); void *ws; cudaMalloc(&ws, wsb);
  pmz_decompress(d_buf, n, &hd, std::log2(1.0 + hd.b_r), d_off, d_out, ws, wsb, 0);
  Geom G = hdr_geom(&hd);
  DecLayout L = dec_layout(G);
  DecTab tab; cudaMemcpy(&tab, at<DecTab>(ws, L.tab), sizeof(DecTab), cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> pb(G.nparts), po(G.nparts), pay(G.nblocks);
  cudaMemcpy(pb.data(), at<unsigned long long>(ws, L.part_bits), 8 * G.nparts, cudaMemcpyDeviceToHost);
  cudaMemcpy(po.data(), at<unsigned long long>(ws, L.part_off), 8 * G.nparts, cudaMemcpyDeviceToHost);
  cudaMemcpy(pay.data(), at<unsigned long long>(ws, L.pay_off), 8 * G.nblocks, cudaMemcpyDeviceToHost);
  long long *d_r; cudaMalloc(&d_r, 64);
  unsigned *d_w; cudaMalloc(&d_w, 4 * 2052);
  for (int ai = 2; ai < argc; ai++) {
    int P = atoi(argv[ai]);
    int64_t b = P / G.np_full; // full blocks only
    unsigned Lb = (unsigned)pb[P];
    const uint8_t *src = h.data() + offs[b] + 0;  // unused
    (void)src;
    // substream bytes: container offset = block record + pay_off(b, relative) + part_off
    uint64_t base = pay[b] + po[P];
    std::vector<unsigned> w(2052, 0);
    unsigned nbytes = (Lb + 7) / 8;
    for (unsigned i = 0; i < std::min(nbytes, 2048u * 4); i++) w[i / 4] |= (unsigned)h[base + i] << (24 - 8 * (i % 4));
    cudaMemcpy(d_w, w.data(), 4 * 2052, cudaMemcpyHostToDevice);
    long long r[3];
    const char *nm[3] = {"full", "no-mark", "lut-only"};
    for (int v = 0; v < 3; v++) {
      if (v == 0) k_step<0><<<1, 32>>>(d_w, Lb, at<unsigned>(ws, L.lut), tab, at<uint16_t>(ws, L.sym), d_r);
      if (v == 1) k_step<1><<<1, 32>>>(d_w, Lb, at<unsigned>(ws, L.lut), tab, at<uint16_t>(ws, L.sym), d_r);
      if (v == 2) k_step<2><<<1, 32>>>(d_w, Lb, at<unsigned>(ws, L.lut), tab, at<uint16_t>(ws, L.sym), d_r);
      cudaMemcpy(r, d_r, 24, cudaMemcpyDeviceToHost);
      printf("P%d L %u %-9s cycles %lld  max-lane steps %lld  -> %.0f cycles/step (syms %lld)\n", P, Lb, nm[v], r[0], r[1], (double)r[0] / r[1], r[2]);
    }
  }
  return 0;
}
