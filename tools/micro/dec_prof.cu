// Decode-phase profiler: decompress a container file with clock64 stamps.
#define PMZ_DEC_PROFILE 1
#include "../../paper_2309_09778_b200/csrc/capi.cu"
#include <vector>
#include <cmath>
#include <algorithm>
int main(int argc, char **argv) {
  FILE *f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
  std::vector<uint8_t> h(n); fread(h.data(), 1, n, f); fclose(f);
  pmz_header hd; printf("parse %d\n", pmz_parse_header(h.data(), n, &hd));
  std::vector<uint64_t> offs(hd.nblocks + 1);
  printf("index %d\n", pmz_index_blocks(h.data(), n, &hd, offs.data()));
  uint8_t *d_buf; uint64_t *d_off; float *d_out; void *ws; uint64_t wsb;
  cudaMalloc(&d_buf, n + 64); cudaMemcpy(d_buf, h.data(), n, cudaMemcpyHostToDevice);
  cudaMalloc(&d_off, 8 * offs.size()); cudaMemcpy(d_off, offs.data(), 8 * offs.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&d_out, 4 * hd.rows * hd.cols);
  pmz_decompress_workspace_size(&hd, &wsb); cudaMalloc(&ws, wsb);
  double b_a = std::log2(1.0 + hd.b_r);
  for (int it = 0; it < 3; it++) printf("decompress %d\n", pmz_decompress(d_buf, n, &hd, b_a, d_off, d_out, ws, wsb, 0));
  Geom G = hdr_geom(&hd);
  std::vector<long long> prof(65536 * 6);
  cudaMemcpyFromSymbol(prof.data(), g_dec_prof, sizeof(long long) * 65536 * 6);
  double ph[4] = {0}, mx[4] = {0}; long long tmax = 0, tmin = prof[0];
  int np = (int)G.nparts;
  for (int p = 0; p < np; p++) {
    long long *q = &prof[p * 6];
    for (int i = 0; i < 4; i++) { double d = (double)(q[i + 1] - q[i]); ph[i] += d; if (d > mx[i]) mx[i] = d; }
  }
  const char *nm[4] = {"stage", "speculate", "walk", "write"};
  for (int i = 0; i < 4; i++) printf("%-10s avg %9.0f cycles  max %9.0f\n", nm[i], ph[i] / np, mx[i]);
  double tot = 0, tmx = 0;
  for (int p = 0; p < np; p++) { double d = (double)(prof[p*6+4] - prof[p*6]); tot += d; tmx = std::max(tmx, d); }
  printf("total      avg %9.0f cycles  max %9.0f\n", tot / np, tmx);
  std::vector<std::pair<long long,int>> w;
  for (int p = 0; p < np; p++) w.push_back({prof[p*6+3]-prof[p*6+2], p});
  std::sort(w.begin(), w.end());
  printf("slowest walks:");
  for (int i = 0; i < 8; i++) printf(" p%d:%lld", w[np-1-i].second, w[np-1-i].first);
  printf("\n");
  return 0;
}
