// k_decode3 phase profiler: decompress a container file with clock64 stamps.
#define PMZ_DEC3_PROFILE 1
#include "../../paper_2309_09778_b200/csrc/capi.cu"
#include <vector>
#include <algorithm>
int main(int argc, char **argv) {
  FILE *f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
  std::vector<uint8_t> h(n); fread(h.data(), 1, n, f); fclose(f);
  pmz_header hd; printf("parse %d\n", pmz_parse_header(h.data(), n, &hd));
  std::vector<uint64_t> offs(hd.nblocks + 1);
  printf("index %d\n", pmz_index_blocks(h.data(), n, &hd, offs.data()));
  uint8_t *d_buf; cudaMalloc(&d_buf, n); cudaMemcpy(d_buf, h.data(), n, cudaMemcpyHostToDevice);
  uint64_t *d_off; cudaMalloc(&d_off, 8 * offs.size()); cudaMemcpy(d_off, offs.data(), 8 * offs.size(), cudaMemcpyHostToDevice);
  float *d_out; cudaMalloc(&d_out, 4 * hd.rows * hd.cols);
  uint64_t wsb; pmz_decompress_workspace_size(&hd, &wsb); void *ws; cudaMalloc(&ws, wsb);
  double b_a = std::log2(1.0 + hd.b_r);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; it++) {
    cudaEventRecord(e0);
    int st = pmz_decompress(d_buf, n, &hd, b_a, d_off, d_out, ws, wsb, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("decompress %d  %.3f ms\n", st, ms);
  }
  Geom G = hdr_geom(&hd);
  std::vector<long long> q(65536 * 8), qn(65536 * 3);
  cudaMemcpyFromSymbol(qn.data(), g_d3n, 8 * 65536 * 3);
  cudaMemcpyFromSymbol(q.data(), g_d3, 8 * 65536 * 8);
  double sp = 0, fx = 0, wr = 0, rounds = 0, stg = 0; long long mx = 0; int nl = 0, np = 0;
  std::vector<std::pair<long long, int>> tot;
  for (int i = 0; i < G.nparts; i++) {
    long long *r = &q[i * 8];
    if (r[5] == 0) continue;
    np++;
    stg += qn[i * 3 + 2] - r[0];
    sp += r[1] - r[0]; fx += r[2] - r[1]; wr += r[3] - r[2]; rounds += r[4]; nl += r[7] != 0;
    tot.push_back({r[3] - r[0], i});
  }
  std::sort(tot.begin(), tot.end());
  {
    int b1 = 0, b2 = 0, b3 = 0;
    for (auto &t : tot) { if (t.first > 250000) b1++; if (t.first > 500000) b2++; if (t.first > 1000000) b3++; }
    printf("partitions > 250k cycles: %d, > 500k: %d, > 1M: %d; median %lld\n", b1, b2, b3, tot[tot.size() / 2].first);
  }
  printf("stage avg %.0f\n", stg / np);
  printf("partitions %d (large %d): spec %.0f  fix %.0f  write %.0f  rounds %.2f (avg cycles)\n", np, nl, sp / np, fx / np, wr / np, rounds / np);
  for (int k = 0; k < 8 && k < (int)tot.size(); k++) {
    int i = tot[tot.size() - 1 - k].second; long long *r = &q[i * 8];
    printf("  slow p%d: %lld cycles spec %lld fix %lld write %lld rounds %lld L %lld nsym %lld large %lld | iters spec %lld fix %lld | stage %lld\n", i, tot[tot.size()-1-k].first, r[1]-r[0], r[2]-r[1], r[3]-r[2], r[4], r[5], r[6], r[7], qn[i*3], qn[i*3+1], qn[i*3+2]-r[0]);
  }
  return 0;
}
