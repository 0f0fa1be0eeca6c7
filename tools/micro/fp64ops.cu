#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void tput(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) {
      if (OP == 0) { a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c); a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c); }
      if (OP == 1) { a0 = __dadd_rn(a0, c); a1 = __dadd_rn(a1, c); a2 = __dadd_rn(a2, c); a3 = __dadd_rn(a3, c); a4 = __dadd_rn(a4, c); a5 = __dadd_rn(a5, c); a6 = __dadd_rn(a6, c); a7 = __dadd_rn(a7, c); }
      if (OP == 2) { a0 = __dmul_rn(a0, b); a1 = __dmul_rn(a1, b); a2 = __dmul_rn(a2, b); a3 = __dmul_rn(a3, b); a4 = __dmul_rn(a4, b); a5 = __dmul_rn(a5, b); a6 = __dmul_rn(a6, b); a7 = __dmul_rn(a7, b); }
      if (OP == 3) { a0 = a0 < c ? a1 : a0; a1 = a1 < c ? a2 : a1; a2 = a2 < c ? a3 : a2; a3 = a3 < c ? a4 : a3; a4 = a4 < c ? a5 : a4; a5 = a5 < c ? a6 : a5; a6 = a6 < c ? a7 : a6; a7 = a7 < c ? a0 : a7; a0 += 1e-300; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double *d; cudaMalloc(&d, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const char *nm[4] = {"DFMA", "DADD", "DMUL", "DSETP+sel"};
  for (int op = 0; op < 4; op++) {
    for (int r = 0; r < 2; r++) {
      cudaEventRecord(e0);
      if (op == 0) tput<0><<<148 * 8, 256>>>(d, 1000);
      if (op == 1) tput<1><<<148 * 8, 256>>>(d, 1000);
      if (op == 2) tput<2><<<148 * 8, 256>>>(d, 1000);
      if (op == 3) tput<3><<<148 * 8, 256>>>(d, 1000);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double ops = 148.0 * 8 * 256 * 1000 * 16 * 8;
    printf("%-10s %.1f G/s  = %.1f per clk per SM @1.965\n", nm[op], ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
  }
}
