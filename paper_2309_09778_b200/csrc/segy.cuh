// segy.cuh -- SEG-Y trace samples -> IEEE float32 rows (read_segy,
// SPEC.md:519-526): one thread per sample of the
// trace records (240-byte trace header + ns big-endian 32-bit samples each)
// resident in device memory, traces as rows.  Format code 1 (IBM hex float:
// sign, 7-bit excess-64 base-16 exponent, 24-bit fraction) is evaluated
// exactly in double (fraction * 2^(4 (e - 64) - 24)) and rounded once to
// float32 (overflow -> inf, tiny -> subnormal / zero); format code 5 is a
// byte swap.
#pragma once
#include <cstdint>

namespace pmz {

__device__ __forceinline__ float ibm_to_ieee(unsigned w) {
  const unsigned frac = w & 0xffffffu;
  const int e = (int)((w >> 24) & 0x7fu);
  const double v = ldexp((double)frac, 4 * (e - 64) - 24);  // exact: 24-bit integer times a power of two
  const float f = (float)v;
  return (w >> 31) ? -f : f;
}

__global__ void k_segy_samples(const uint8_t *__restrict__ traces, uint64_t ntr, unsigned ns, int fmt,
                               float *__restrict__ out) {
  const uint64_t n = ntr * ns;
  const uint64_t rec = 240ull + 4ull * ns;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / ns, s = i - t * ns;
    const uint8_t *q = traces + t * rec + 240 + 4 * s;
    const unsigned w = ((unsigned)q[0] << 24) | ((unsigned)q[1] << 16) | ((unsigned)q[2] << 8) | (unsigned)q[3];
    out[i] = fmt == 1 ? ibm_to_ieee(w) : __uint_as_float(w);
  }
}

}  // namespace pmz
