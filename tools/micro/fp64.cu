// FP64 throughput / latency microbenchmark + log2 variants throughput.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include "../../paper_2309_09778_b200/csrc/dmath.cuh"
using namespace pmz;

__global__ void dfma_tput(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) {
      a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
      a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dfma_lat(double *out, int iters, long long *cyc) {
  double a = threadIdx.x * 1e-3;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) a = __fma_rn(a, b, c);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void ffma_tput(float *out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) {
      a0 = __fmaf_rn(a0, b, c); a1 = __fmaf_rn(a1, b, c); a2 = __fmaf_rn(a2, b, c); a3 = __fmaf_rn(a3, b, c);
      a4 = __fmaf_rn(a4, b, c); a5 = __fmaf_rn(a5, b, c); a6 = __fmaf_rn(a6, b, c); a7 = __fmaf_rn(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void log2_kern(const float *x, double *out, long long n, int variant, unsigned *amb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = (double)x[i];
    out[i] = variant == 0 ? pmz_log2_f32_fast(a, amb) : pmz_log2_f32(a, amb);
  }
}
__global__ void ddiv_tput(double *out, int iters) {
  double a = threadIdx.x * 1e-3 + 1.0, s = 0;
  for (int i = 0; i < iters; i++) { s += __ddiv_rn(a, 1.0 + i * 1e-9); a += 1e-12; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main1();
int main2();
int main() { main2(); return main1(); }
int main1() {
  double *d; float *f; long long *cyc;
  cudaMalloc(&d, 1 << 28); cudaMalloc(&f, 1 << 28); cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 2000;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    dfma_tput<<<148 * 8, 256>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  double flops = 2.0 * 148 * 8 * 256 * (double)iters * 16 * 8;
  printf("DFMA throughput: %.2f TFLOP/s (%.1f DFMA/clk/SM @1.965GHz)\n", flops / ms / 1e9, flops / 2 / (ms * 1e-3) / 148 / 1.965e9);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    ffma_tput<<<148 * 8, 256>>>(f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("FFMA throughput: %.2f TFLOP/s\n", flops / ms / 1e9);
  dfma_lat<<<1, 32>>>(d, iters, cyc);
  long long hc; cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA latency: %.2f cycles\n", (double)hc / (iters * 16));
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    ddiv_tput<<<148 * 8, 256>>>(d, 200);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("DDIV: %.2f Gdiv/s\n", 148.0 * 8 * 256 * 200 / ms / 1e6);
  long long n = 1 << 25;
  float *hx = (float *)malloc(n * 4);
  for (long long i = 0; i < n; i++) { unsigned u = 0x00800000u + (unsigned)((i * 2654435761ull) % 0x7e800000u); memcpy(&hx[i], &u, 4); }
  cudaMemcpy(f, hx, n * 4, cudaMemcpyHostToDevice);
  unsigned *amb; cudaMalloc(&amb, 4); cudaMemset(amb, 0, 4);
  for (int v = 0; v < 2; v++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      log2_kern<<<148 * 8, 256>>>(f, d, n, v, amb);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("log2 variant %d: %.2f G/s  (%.1f cycles/elem/SM)\n", v, n / ms / 1e6, 148 * 1.965e9 / (n / (ms * 1e-3)));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
// ---- single-warp latency of the batched log2
__global__ void lat_log2n(const float *x, double *out, long long *cyc, int iters) {
  unsigned amb = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    double ax[8], lg[8];
#pragma unroll
    for (int q = 0; q < 8; q++) ax[q] = (double)x[(it * 8 + q) * 32 + threadIdx.x];
    pmz_log2_f32_fast_n<8>(ax, lg, &amb);
#pragma unroll
    for (int q = 0; q < 8; q++) acc += lg[q];
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_log2_1(const float *x, double *out, long long *cyc, int iters) {
  unsigned amb = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters * 8; it++) acc += pmz_log2_f32_fast((double)x[it * 32 + threadIdx.x], &amb);
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main2() {
  int iters = 64;
  float *x; double *o; long long *c;
  cudaMalloc(&x, 4 * 32 * 8 * iters); cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 8);
  std::vector<float> h(32 * 8 * iters);
  for (size_t i = 0; i < h.size(); i++) h[i] = 1.0f + 0.37f * (float)i;
  cudaMemcpy(x, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
  long long hc;
  for (int r = 0; r < 2; r++) { lat_log2n<<<1, 32>>>(x, o, c, iters); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); }
  printf("log2 x8 interleaved: %.1f cycles per batch of 8 (%.1f per value)\n", (double)hc / iters, (double)hc / iters / 8);
  for (int r = 0; r < 2; r++) { lat_log2_1<<<1, 32>>>(x, o, c, iters); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); }
  printf("log2 scalar: %.1f cycles per value\n", (double)hc / iters / 8);
  return 0;
}
