// Compress profiler: runs pmz_compress on a raw f32 file with producer/consumer stamps.
#define PMZ_CMP_PROFILE 1
#include "../../paper_2309_09778_b200/csrc/capi.cu"
#include <vector>
#include <cmath>
#include <algorithm>
int main(int argc, char **argv) {
  long rows = atol(argv[2]), cols = atol(argv[3]);
  std::vector<float> h(rows * cols);
  FILE *f = fopen(argv[1], "rb"); fread(h.data(), 4, h.size(), f); fclose(f);
  float *d_in; cudaMalloc(&d_in, 4 * h.size()); cudaMemcpy(d_in, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
  pmz_params p{}; p.b_r = 1e-2; p.b_a = std::log2(1.01); p.onepbr2 = 1.01 * 1.01; p.eps0 = 0x1p-126; p.repair_t = 1e-2;
  p.coverage_target = 0.99; p.slope = 0.01; double w1[8] = {1, 1, 1, 1, -1, -1, 0, 0}; for (int i = 0; i < 8; i++) p.w1[i] = w1[i];
  p.w2[0] = p.w2[1] = 0.5; p.block_rows = p.block_cols = 256; p.partition_rows = 32; p.S = 3; p.H = 2; p.m = 8;
  pmz_geom g{(uint64_t)rows, (uint64_t)cols, 0, (uint64_t)rows};
  uint64_t wsb, cap; pmz_workspace_size(&p, &g, &wsb); pmz_max_container_size(&p, &g, &cap);
  void *ws; uint8_t *out; cudaMalloc(&ws, wsb); cudaMalloc(&out, cap);
  // validation = every block (a realistic code histogram for the codebook)
  const int64_t nb = ((rows + 255) / 256) * ((cols + 255) / 256);
  std::vector<int64_t> hv(nb);
  for (int64_t i = 0; i < nb; i++) hv[i] = i;
  int64_t *d_val; cudaMalloc(&d_val, 8 * nb); cudaMemcpy(d_val, hv.data(), 8 * nb, cudaMemcpyHostToDevice);
  p.m = 0;
  pmz_result res;
  for (int it = 0; it < 3; it++) printf("compress %d\n", pmz_compress(d_in, &g, &p, d_val, nb, out, cap, nullptr, ws, wsb, 0, &res));
  printf("m %d\n", res.m);
  Geom G = geom_of(&p, &g);
  std::vector<long long> pr(65536 * 8);
  cudaMemcpyFromSymbol(pr.data(), g_cmp_prof, 8 * 65536 * 8);
  long long tmin = 1LL << 62, tmax = 0; double pw = 0, cw = 0, pd = 0, cd = 0, cst = 0;
  for (int i = 0; i < G.nparts; i++) {
    long long *q = &pr[i * 8];
    tmin = std::min(tmin, std::min(q[0], q[4])); tmax = std::max(tmax, std::max(q[1], q[5]));
    pd += q[1] - q[0]; pw += q[2]; cd += q[5] - q[4]; cw += q[6]; cst += q[7];
  }
  int n = (int)G.nparts;
  printf("partitions %d  kernel span %lld cycles\n", n, tmax - tmin);
  {
    long long cb[8];
    cudaMemcpyFromSymbol(cb, g_cb_prof, 64);
    printf("codebook: init %lld sort %lld mk %lld lens+cnt %lld canon %lld\n", cb[1] - cb[0], cb[2] - cb[1], cb[3] - cb[2], cb[4] - cb[3], cb[5] - cb[4]);
  }
  printf("producer: avg %.0f cycles, waiting %.0f\nconsumer: avg %.0f cycles, mbar wait %.0f, steady groups %.0f\n", pd / n, pw / n, cd / n, cw / n, cst / n);
  return 0;
}
