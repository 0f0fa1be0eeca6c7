// capi.cu -- extern "C" boundary (include/permez_b200.h): workspace layout,
// stage launches, container header parsing and block indexing.
// Single translation unit: all kernels are included here.
#include <cub/device/device_scan.cuh>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"
#include "compress.cuh"
#include "blockc.cuh"
#include "wsc.cuh"
#include "dsc.cuh"
#include "decompress.cuh"
#include "encode.cuh"
#include "fwdq.cuh"
#include "dec4.cuh"
#include "train.cuh"
#include "segy.cuh"
#include "tdec.cuh"
#include "cmain.cuh"
#include "cmain32.cuh"
#include "dmain.cuh"

using namespace pmz;

static int cuda_fail(cudaError_t e) {
  if (getenv("PMZ_DEBUG")) fprintf(stderr, "permez: CUDA error: %s\n", cudaGetErrorString(e));
  return PMZ_ERR_CUDA;
}
#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

namespace {

int check_params(const pmz_params *p) {
  if (!p) return PMZ_ERR_CONFIG;
  if (!(p->b_r > 0.0 && p->b_r < 1.0)) return PMZ_ERR_CONFIG;  // transform.py:146-147
  if (p->block_rows <= 0 || p->block_cols <= 0 || p->partition_rows <= 0) return PMZ_ERR_CONFIG;
  if (p->partition_rows > 32) return PMZ_ERR_CONFIG;  // one warp lane per partition row
  if (p->block_rows / p->partition_rows > 64) return PMZ_ERR_CONFIG;
  if (p->S != 1 && p->S != 3) return PMZ_ERR_CONFIG;
  if (p->H != 2) return PMZ_ERR_CONFIG;
  if (p->m != 0 && (p->m < 4 || p->m > 16)) return PMZ_ERR_CONFIG;
  if (!(p->b_a > 0.0) || !(p->repair_t > 0.0)) return PMZ_ERR_CONFIG;
  if (p->precision != 0 && p->precision != 1) return PMZ_ERR_CONFIG;
  if ((p->precision == 1 || p->d_code_dump) && (p->S != 3 || p->block_rows == 1))
    return PMZ_ERR_CONFIG;  // FP32 mode and code dumps: 2-D fields (throughput path)
  return PMZ_OK;
}

Geom make_geom(int64_t rows, int64_t cols, int br, int bc, int prow, int64_t block_row0) {
  Geom g{};
  g.rows = rows;
  g.cols = cols;
  g.br = br;
  g.bc = bc;
  g.prow = prow;
  g.block_row0 = block_row0;
  g.nbr = rows > 0 ? (rows + br - 1) / br : 0;
  g.nbc = cols > 0 ? (cols + bc - 1) / bc : 0;
  g.nblocks = g.nbr * g.nbc;
  g.np_full = (br + prow - 1) / prow;
  g.br_last = g.nbr > 0 ? (int)(rows - (g.nbr - 1) * br) : 0;
  g.np_last = g.nbr > 0 ? (g.br_last + prow - 1) / prow : 0;
  g.nparts = g.nbr > 0 ? (g.nbr - 1) * g.nbc * g.np_full + g.nbc * g.np_last : 0;
  g.nct = (bc + 31) / 32;
  return g;
}

Geom geom_of(const pmz_params *p, const pmz_geom *g) {
  Geom G = make_geom((int64_t)g->rows, (int64_t)g->cols, p->block_rows, p->block_cols, p->partition_rows,
                     (int64_t)g->block_row0);
  G.fp32 = p->precision == 1;
  G.force_tpath = p->d_code_dump != 0;
  return G;
}

// weights equal init_model(S) -> constant-folded predictor
int is_init_model(int S, const double *w1, const double *w2) {
  if (w2[0] != 0.5 || w2[1] != 0.5) return 0;
  static const double i3[8] = {1, 1, 1, 1, -1, -1, 0, 0}, i1[4] = {1, 1, 0, 0};
  const double *ref = S == 3 ? i3 : i1;
  int n = S == 3 ? 8 : 4;
  for (int i = 0; i < n; i++)
    if (w1[i] != ref[i] || std::signbit(w1[i]) != std::signbit(ref[i])) return 0;
  return S;
}

KParams kparams(const pmz_params *p) {
  KParams k{};
  k.b_r = p->b_r;
  k.b_a = p->b_a;
  k.two_ba = 2.0 * p->b_a;
  k.onepbr2 = p->onepbr2;
  k.eps0 = p->eps0;
  k.repair_t = p->repair_t;
  k.slope = p->slope;
  k.coverage_target = p->coverage_target;
  for (int i = 0; i < 8; i++) k.w1[i] = p->w1[i];
  for (int i = 0; i < 2; i++) k.w2[i] = p->w2[i];
  k.S = p->S;
  k.H = p->H;
  k.block_rows = p->block_rows;
  k.block_cols = p->block_cols;
  k.partition_rows = p->partition_rows;
  k.m_fixed = p->m;
  k.inv_two_ba = 1.0 / (2.0 * p->b_a);
  k.dpos = std::log2(1.0 + p->repair_t);
  k.dneg = std::log2(1.0 - p->repair_t);
  k.dpos_m = k.dpos - 0x1p-20;
  k.dneg_m = k.dneg + 0x1p-20;
  k.dpos_p = k.dpos + 0x1p-20;
  k.dneg_p = k.dneg - 0x1p-20;
  k.init_model = is_init_model(p->S, p->w1, p->w2);
  k.precision = p->precision;
  k.code_dump = p->d_code_dump;
  // certified-rounding margins of the approximate TRUE residual (cmain.cuh):
  // |v~ - v| < 2^-41 per surface value moves a hidden pre-activation by at most
  // sum_k |w1_kj| 2^-41 (+ roundings) and the residual by amp 2^-41; 2^-37
  // leaves 16x headroom over the rounding terms for |v| < 2^9
  double amp = 1.0, hsum = 1.0;
  for (int j = 0; j < p->H && j < 2; j++) {
    double sj = 0.0;
    for (int q = 0; q < p->S; q++) sj += std::fabs(p->w1[q * p->H + j]);
    amp += std::fabs(p->w2[j]) * sj;
    hsum = std::max(hsum, sj + 1.0);
  }
  k.q_half_m = 0.5 - std::max(0x1p-20, k.inv_two_ba * amp * 0x1p-37);
  k.h_marg = hsum * 0x1p-36;
  k.lk[0] = 1.4426950408889634;   // 1 / ln 2
  k.lk[1] = -0.7213475204444817;  // -1 / (2 ln 2)
  k.lk[2] = 0.48089834696298783;  // 1 / (3 ln 2)
  k.lk[3] = -0.36067376022224085; // -1 / (4 ln 2)
  k.rnd_magic = 0x1.8p52;
  k.e_magic = 4503601774854144.0;
  return k;
}

size_t cub_scan_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                (int)(n > 0 ? n : 1));
  return bytes;
}

// every block is one partition of one row (1-D inputs, block_rows == 1)
bool one_row_parts(const Geom &G) { return G.br == 1 || G.rows == 1; }

// Throughput path (tdec.cuh / tcmp.cuh) or latency path (dec4/dsc, fwdq/wsc):
// the throughput kernels need partition-level parallelism only, the latency
// kernels also split each partition's work across a CTA.  PMZ_PATH=latency |
// throughput overrides the size rule (tests exercise both on small fields).
// The size rule is per direction (tools/path_cross.py, C2-like fields of 1024
// columns; profiles/r2_configs.txt): the throughput compress wins from ~5 K
// partitions on (with chains sized to the partition count), the
// thread-per-substream throughput decoder from ~6 K (C4, 3136 partitions:
// decompress 4.84 ms on the throughput path, 1.72 ms on the latency path).
bool use_tpath(const Geom &G, bool decomp = false) {
  if (G.fp32 || G.force_tpath) return true;  // the FP32 perf mode and the code dump: throughput path only
  if (one_row_parts(G)) return false;
  const char *e = getenv("PMZ_PATH");
  if (e && e[0] == 'l') return false;
  if (e && e[0] == 't') return true;
  return G.nparts >= (decomp ? kTputMinPartsD : kTputMinPartsC);
}

WsLayout compress_layout(const Geom &g) {
  WsLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.status = take(sizeof(WsStatus));
  L.cov = take(18 * 8);
  L.hist = take((kMaxAlpha + 1) * 8);
  L.vflag = take((size_t)g.nblocks + 1);  // zeroed with status / cov / hist
  L.bstat = take(16 * ((size_t)g.nblocks + 1));  // BlkStat per block, zeroed too
  L.npfix = take(sizeof(pmz_np_fix) * ((size_t)g.nblocks + 1));
  L.lens = take(kMaxAlpha);
  L.cw = take(kMaxAlpha * 4);
  L.cb_keys = take(kMaxAlpha * 8);
  L.cb_w = take(kMaxAlpha * 8);       // internal weights (u64), reused as depth / jump arrays
  L.cb_parent = take(kMaxAlpha * 4);  // parent of every internal node
  L.blkp = take(sizeof(BlkP) * (size_t)(g.nblocks + 1));
  L.part_bits = take(8 * (size_t)(g.nparts + 1));
  L.part_zeros = take(8 * (size_t)(g.nparts + 1));
  L.anchors = take(8 * (size_t)(g.nparts + 1));
  L.rec_size = take(8 * (size_t)(g.nblocks + 1));
  L.rec_off = take(8 * (size_t)(g.nblocks + 1));
  L.cub_bytes = cub_scan_bytes(g.nblocks + 1);
  L.cub_tmp = take(L.cub_bytes);
  const size_t ntile = (size_t)g.nparts * (size_t)g.nct * kTile;  // partition-tiled elements
  L.vbuf = take(8 * ntile);
  L.rqbuf = take((use_tpath(g) ? 4 : 2) * ntile);  // throughput path: per-row bitstreams (32 bits per code max)
  L.clsbuf = take(ntile);
  L.total = o;
  return L;
}

template <class T>
T *at(void *ws, size_t off) {
  return reinterpret_cast<T *>(reinterpret_cast<uint8_t *>(ws) + off);
}

int err_from_bits(unsigned bits) {
  for (int i = 1; i < 32; i++)
    if (bits & (1u << i)) return -i;
  return PMZ_OK;
}

int launch_check() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && getenv("PMZ_DEBUG")) fprintf(stderr, "permez: CUDA error: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? PMZ_OK : PMZ_ERR_CUDA;
}

constexpr int kNT = 256;


// the throughput-path views of the compress workspace: per-row balance
// lists in vbuf, per-row bitstreams in rqbuf, per-row {bits, count} in clsbuf
CMainOut cmain_out(void *d_ws, const WsLayout &L) {
  CMainOut o;
  o.rowbits = at<unsigned>(d_ws, L.rqbuf);
  o.balrow = at<double>(d_ws, L.vbuf);
  o.rowinfo = at<uint2>(d_ws, L.clsbuf);
  o.anchors = at<double>(d_ws, L.anchors);
  o.part_bits = at<unsigned long long>(d_ws, L.part_bits);
  o.part_zeros = at<unsigned long long>(d_ws, L.part_zeros);
  o.lens = at<uint8_t>(d_ws, L.lens);
  o.cw = at<unsigned>(d_ws, L.cw);
  o.hist = at<unsigned long long>(d_ws, L.hist);
  o.cov = at<unsigned long long>(d_ws, L.cov);
  o.dump = nullptr;
  return o;
}
template <int PK, int MODE>
void launch_cmain(const float *x, const Geom &G, const KParams &k, const int64_t *d_val, int64_t n_val, void *d_ws,
                  const WsLayout &L, cudaStream_t st) {
  // kCMain: a warp sweeps a chain of up to `chain` consecutive partitions of a
  // block as one wavefront (PMZ_CHAIN overrides the default for experiments)
  // Longer chains save more ramps but leave fewer, longer work items: keep at
  // least ~6 rounds of chains over the GPU's resident warps (2 CTAs of kCW
  // warps per SM), so a shard of a multi-GPU run (1/8 of C5: 32768 partitions)
  // still balances.
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sm_count <= 0)
      sm_count = 148;
  }
  int chain = (int)std::min<int64_t>(8, std::max<int64_t>(1, G.nparts / ((int64_t)sm_count * 2 * kCW * 6)));
  if (const char *e = getenv("PMZ_CHAIN")) chain = atoi(e) > 0 ? atoi(e) : chain;
  unsigned grid;
  if (MODE == kCMain) grid = (unsigned)((c_nchains(G, chain) + kCW - 1) / kCW);
  else grid = (unsigned)(n_val * ((G.np_full + kCW - 1) / kCW));
  if (grid == 0) return;
  CMainOut o = cmain_out(d_ws, L);
  if (MODE == kCMain) {
    o.dump = reinterpret_cast<uint16_t *>(k.code_dump);
  }
  // m is selected on the device: size for the largest shared-memory table;
  // alphabets above 2^12 take the launch whose codewords come from global memory
  const int smem = (int)cmain_smem_bytes(MODE, MODE == kCHist ? 13 : 12);
  const int smem2 = (int)cmain_smem_bytes(MODE, 16);
  auto *fa = k.precision ? k_c_main32<PK, MODE, true> : k_c_main<PK, MODE, true>;
  auto *fb = k.precision ? k_c_main32<PK, MODE, false> : k_c_main<PK, MODE, false>;
  cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  fa<<<grid, kCW * 32, smem, st>>>(x, G, k, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status), d_val, n_val, o,
                                   chain);
  if (getenv("PMZ_DEBUG")) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) fprintf(stderr, "permez: k_c_main%s<%d,%d,1>: %s\n", k.precision ? "32" : "", PK, MODE,
                                  cudaGetErrorString(e));
  }
  if (MODE == kCMain) {
    cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    fb<<<grid, kCW * 32, smem2, st>>>(x, G, k, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status), d_val, n_val,
                                      o, chain);
    k_c_part_totals<<<(unsigned)((G.nparts + 7) / 8), 256, 0, st>>>(G, at<BlkP>(d_ws, L.blkp), o.rowinfo, o.part_bits,
                                                                    o.part_zeros, at<WsStatus>(d_ws, L.status));
  }
}
template <int MODE>
void launch_tmain_pk(const float *x, const Geom &G, const KParams &k, const int64_t *d_val, int64_t n_val,
                     void *d_ws, const WsLayout &L, cudaStream_t st) {
  if (k.init_model == 3) launch_cmain<3, MODE>(x, G, k, d_val, n_val, d_ws, L, st);
  else launch_cmain<0, MODE>(x, G, k, d_val, n_val, d_ws, L, st);
}

template <int PK>
int launch_ws(const KParams &k, unsigned grid, cudaStream_t st, const float *x, const Geom &G, void *d_ws,
              const WsLayout &L) {
  if (G.br == 1 || G.rows == 1) {  // one-row partitions: a thread per partition
    k_compress_1d<PK><<<(unsigned)((G.nparts + 31) / 32), 32, 0, st>>>(
        x, G, k, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status), at<double>(d_ws, L.vbuf),
        at<int16_t>(d_ws, L.rqbuf), at<uint8_t>(d_ws, L.clsbuf), at<double>(d_ws, L.anchors),
        at<unsigned long long>(d_ws, L.part_zeros), at<uint8_t>(d_ws, L.vflag), at<unsigned long long>(d_ws, L.hist));
    return PMZ_OK;
  }
  CK(cudaFuncSetAttribute(k_compress_ws<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWscSmem));
  k_compress_ws<PK><<<grid, kPPC * 64, kWscSmem, st>>>(x, G, k, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status),
                                                       at<double>(d_ws, L.vbuf), at<int16_t>(d_ws, L.rqbuf),
                                                       at<uint8_t>(d_ws, L.clsbuf), at<double>(d_ws, L.anchors),
                                                       at<unsigned long long>(d_ws, L.part_zeros),
                                                       at<uint8_t>(d_ws, L.vflag), at<unsigned long long>(d_ws, L.hist));
  return PMZ_OK;
}

template <int PK>
void launch_quant(const KParams &k, cudaStream_t st, const Geom &G, void *d_ws, const WsLayout &L) {
  k_quant<PK><<<(unsigned)G.nparts, kFqT, 0, st>>>(G, k, at<BlkP>(d_ws, L.blkp), at<uint8_t>(d_ws, L.vflag),
                                                   at<WsStatus>(d_ws, L.status), at<double>(d_ws, L.vbuf),
                                                   at<int16_t>(d_ws, L.rqbuf), at<unsigned long long>(d_ws, L.cov));
}


}  // namespace

// C linkage comes from the declarations in permez_b200.h.

int pmz_abi_version(void) { return PMZ_ABI_VERSION; }

int pmz_code_dump_elems(const pmz_params *p, const pmz_geom *g, uint64_t *elems) {
  int s = check_params(p);
  if (s) return s;
  const Geom G = geom_of(p, g);
  *elems = (uint64_t)G.nparts * (uint64_t)G.prow * (uint64_t)G.bc;
  return PMZ_OK;
}

const char *pmz_status_string(int s) {
  switch (s) {
    case PMZ_OK: return "ok";
    case PMZ_ERR_CONFIG: return "ConfigError";
    case PMZ_ERR_NONFINITE: return "NonFiniteInput";
    case PMZ_ERR_DEGENERATE: return "DegenerateBlock";
    case PMZ_ERR_SUBNORMAL: return "SubnormalMinimum";
    case PMZ_ERR_NONREPRESENTABLE: return "NonRepresentableFactor";
    case PMZ_ERR_TOO_FEW_BLOCKS: return "TooFewBlocks";
    case PMZ_ERR_BALANCE_FLAG: return "BalanceFlagNotDequantizable";
    case PMZ_ERR_DEGENERATE_ALPHABET: return "DegenerateAlphabet";
    case PMZ_ERR_UNASSIGNED: return "UnassignedCode";
    case PMZ_ERR_TRUNCATED: return "TruncatedStream";
    case PMZ_ERR_INVALID_PREFIX: return "InvalidPrefix";
    case PMZ_ERR_BAD_MAGIC: return "BadMagic";
    case PMZ_ERR_UNSUPPORTED_VERSION: return "UnsupportedVersion";
    case PMZ_ERR_CORRUPT: return "Corrupt";
    case PMZ_ERR_BALANCE_UNDERFLOW: return "BalanceUnderflow";
    case PMZ_ERR_CAPACITY: return "CapacityExceeded";
    case PMZ_ERR_CUDA: return "CudaError";
    case PMZ_ERR_WORKSPACE: return "WorkspaceTooSmall";
    case PMZ_ERR_UNRESOLVED_ROUNDING: return "UnresolvedRounding";
    default: return "unknown";
  }
}

int pmz_workspace_size(const pmz_params *p, const pmz_geom *g, uint64_t *bytes) {
  int s = check_params(p);
  if (s) return s;
  *bytes = compress_layout(geom_of(p, g)).total;
  return PMZ_OK;
}

int pmz_max_container_size(const pmz_params *p, const pmz_geom *g, uint64_t *bytes) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  // header at m = 16 + per block fixed part + every element a balance value +
  // every code at the 32-bit maximum length.
  uint64_t b = header_bytes(16, p->S, p->H);
  b += (uint64_t)G.nblocks * 25 + (uint64_t)G.nparts * 24;
  b += (uint64_t)(G.rows * G.cols) * 12 + (uint64_t)G.nparts;
  *bytes = b;
  return PMZ_OK;
}

uint64_t *pmz_ws_coverage(void *d_ws, const pmz_params *p, const pmz_geom *g) {
  return at<uint64_t>(d_ws, compress_layout(geom_of(p, g)).cov);
}

uint64_t *pmz_ws_histogram(void *d_ws, const pmz_params *p, const pmz_geom *g) {
  return at<uint64_t>(d_ws, compress_layout(geom_of(p, g)).hist);
}

int pmz_compress_stats(const float *d_in, const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes,
                       void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  // zero status, coverage, histogram, flags and block stats (contiguous at the front)
  CK(cudaMemsetAsync(d_ws, 0, L.lens, st));
  if (G.nblocks == 0) return PMZ_OK;
  k_stats<<<(unsigned)G.nblocks, kST, 0, st>>>(d_in, G, k, at<BlkP>(d_ws, L.blkp), at<BlkStat>(d_ws, L.bstat),
                                               at<WsStatus>(d_ws, L.status), at<pmz_np_fix>(d_ws, L.npfix));
  return launch_check();
}

int pmz_compress_transform(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val,
                           int64_t n_val, void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  if (G.nblocks == 0) return PMZ_OK;
  if (n_val > 0)
    k_mark_val<<<(unsigned)((n_val + 255) / 256), 256, 0, st>>>(d_val, n_val, G.nblocks, at<uint8_t>(d_ws, L.vflag),
                                                               at<WsStatus>(d_ws, L.status));
  if (use_tpath(G)) {
    // throughput path: only the coverage of the validation blocks' TRUE
    // residuals here (select_m); the forward map runs fused in k_c_main
    if (k.m_fixed == 0 && n_val > 0) launch_tmain_pk<kCCov>(d_in, G, k, d_val, n_val, d_ws, L, st);
    return launch_check();
  }
  // forward map + m-independent TRUE-surface quantization of every element,
  // coverage of the validation blocks in the same pass
  if (G.nparts > 0) {
    k_fwd<<<(unsigned)G.nparts, kFqT, 0, st>>>(d_in, G, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status),
                                               at<double>(d_ws, L.vbuf), at<uint8_t>(d_ws, L.clsbuf));
    if (k.init_model == 3) launch_quant<3>(k, st, G, d_ws, L);
    else if (k.init_model == 1) launch_quant<1>(k, st, G, d_ws, L);
    else launch_quant<0>(k, st, G, d_ws, L);
  }
  return launch_check();
}

int pmz_compress_analyze(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val,
                         int64_t n_val, void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = pmz_compress_stats(d_in, g, p, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_compress_transform(d_in, g, p, d_val, n_val, d_ws, ws_bytes, stream);
}

namespace {
// Small stream-ordered device -> host read (status words, fix-up lists) that
// does not queue behind bulk copies on the DMA engines: a one-CTA kernel stores
// into mapped pinned memory, the stream is synchronised, the bytes are copied
// out.  (A cudaMemcpyAsync of a few bytes waits for every device->host slab
// copy already queued on the copy engine: the slab pipeline of hostpipe.py
// synchronises per slab and would serialise on that.)
__global__ void k_read_small(const unsigned char *src, unsigned char *dst, int n) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {  // 16-byte words, then the tail
    const int nq = n >> 4;
    for (int i = tid; i < nq; i += nt) reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    for (int i = (nq << 4) + tid; i < n; i += nt) dst[i] = src[i];
  } else {
    for (int i = tid; i < n; i += nt) dst[i] = src[i];
  }
  __threadfence_system();
}
__host__ inline unsigned small_grid(size_t bytes) { return (unsigned)std::min<size_t>(32, (bytes + 4095) / 4096 + 0); }
// (a full fix-up list: 4096 entries of 40 bytes)
constexpr size_t kBounceBytes = 192 * 1024;
void *small_bounce(void **dptr) {
  thread_local void *bounce = nullptr;
  if (!bounce && cudaHostAlloc(&bounce, kBounceBytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    bounce = nullptr;
    cudaGetLastError();
  }
  if (bounce && cudaHostGetDevicePointer(dptr, bounce, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return bounce;
}
int read_small(void *h_dst, const void *d_src, size_t bytes, cudaStream_t st) {
  void *dptr = nullptr;
  void *bounce = bytes <= kBounceBytes ? small_bounce(&dptr) : nullptr;
  if (bounce) {
    k_read_small<<<std::max(1u, small_grid(bytes)), 256, 0, st>>>(static_cast<const unsigned char *>(d_src),
                                                                  static_cast<unsigned char *>(dptr), (int)bytes);
    if (cudaStreamSynchronize(st) != cudaSuccess) return PMZ_ERR_CUDA;
    memcpy(h_dst, bounce, bytes);
    return PMZ_OK;
  }
  if (cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) return PMZ_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PMZ_ERR_CUDA;
  return PMZ_OK;
}
// The mirror: a small stream-ordered host -> device write that does not queue
// behind the slab uploads (the kernel reads the mapped bounce buffer).
// Synchronises the stream (the bounce buffer is reused by the next call).
int write_small(void *d_dst, const void *h_src, size_t bytes, cudaStream_t st) {
  void *dptr = nullptr;
  void *bounce = bytes <= kBounceBytes ? small_bounce(&dptr) : nullptr;
  if (bounce) {
    memcpy(bounce, h_src, bytes);
    k_read_small<<<std::max(1u, small_grid(bytes)), 256, 0, st>>>(static_cast<const unsigned char *>(dptr),
                                                                  static_cast<unsigned char *>(d_dst), (int)bytes);
    if (cudaStreamSynchronize(st) != cudaSuccess) return PMZ_ERR_CUDA;
    return PMZ_OK;
  }
  if (cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return PMZ_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PMZ_ERR_CUDA;
  return PMZ_OK;
}
int64_t read_np_fixups(WsStatus *d_status, const pmz_np_fix *d_fix, cudaStream_t st, pmz_np_fix *h, int64_t cap) {
  unsigned long long n = 0;
  if (read_small(&n, &d_status->nfix, sizeof(n), st) != PMZ_OK) return PMZ_ERR_CUDA;
  const int64_t k = (int64_t)n < cap ? (int64_t)n : cap;
  if (k > 0 && h) {
    if (read_small(h, d_fix, sizeof(pmz_np_fix) * (size_t)k, st) != PMZ_OK) return PMZ_ERR_CUDA;
  }
  return (int64_t)n;
}
int apply_np_fixups(pmz_np_fix *d_fix, BlkP *d_blkp, WsStatus *d_status, int64_t nmax, double eps0, double b_a,
                    cudaStream_t st, const pmz_np_fix *h, int64_t n) {
  if (n <= 0) return PMZ_OK;
  if (n > nmax) return PMZ_ERR_CONFIG;
  for (int64_t i = 0; i < n; i++)
    if (h[i].block < 0 || h[i].block >= nmax) return PMZ_ERR_CONFIG;
  if (write_small(d_fix, h, sizeof(pmz_np_fix) * (size_t)n, st) != PMZ_OK) return PMZ_ERR_CUDA;
  k_np_apply<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(d_fix, n, eps0, b_a, d_blkp, d_status);
  CK(cudaStreamSynchronize(st));  // h may be released by the caller
  return launch_check();
}
}  // namespace

int64_t pmz_compress_np_fixups(const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes, void *stream,
                               pmz_np_fix *h_fix, int64_t cap) {
  int s = check_params(p);
  if (s) return s;
  WsLayout L = compress_layout(geom_of(p, g));
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  return read_np_fixups(at<WsStatus>(d_ws, L.status), at<pmz_np_fix>(d_ws, L.npfix), (cudaStream_t)stream, h_fix,
                        cap);
}

int pmz_compress_np_apply(const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes, void *stream,
                          const pmz_np_fix *h_fix, int64_t n) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  return apply_np_fixups(at<pmz_np_fix>(d_ws, L.npfix), at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status),
                         G.nblocks, p->eps0, p->b_a, (cudaStream_t)stream, h_fix, n);
}

int pmz_compress_codes(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val,
                       int64_t n_val, void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  k_select_m<<<1, 32, 0, st>>>(at<unsigned long long>(d_ws, L.cov), k, at<WsStatus>(d_ws, L.status));
  if (use_tpath(G)) {
    // throughput path: the validation blocks' final codes -> histogram
    // (estimate_codebook); every block is coded after the codebook
    if (n_val > 0) launch_tmain_pk<kCHist>(d_in, G, k, d_val, n_val, d_ws, L, st);
    return launch_check();
  }
  if (G.nparts > 0) {
    const unsigned grid = (unsigned)((G.nparts + kPPC - 1) / kPPC);
    if (k.init_model == 3) s = launch_ws<3>(k, grid, st, d_in, G, d_ws, L);
    else if (k.init_model == 1) s = launch_ws<1>(k, grid, st, d_in, G, d_ws, L);
    else s = launch_ws<0>(k, grid, st, d_in, G, d_ws, L);
    if (s) return s;
  }
  return launch_check();
}

__global__ void k_block_offsets(Geom g, KParams k, int write_header, const unsigned long long *rec_off,
                                WsStatus *st, unsigned long long *boff) {
  count_launch(st);
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > g.nblocks) return;
  unsigned long long base = write_header ? header_bytes(st->m, k.S, k.H) : 0;
  boff[b] = base + rec_off[b];
}

__global__ void k_finish_status(Geom g, KParams k, int write_header, const unsigned long long *rec_off,
                                unsigned long long cap, WsStatus *st) {
  count_launch(st);
  unsigned long long hb = write_header ? header_bytes(st->m, k.S, k.H) : 0;
  st->header_bytes = hb;
  st->record_bytes = rec_off[g.nblocks];
  st->total_bytes = hb + rec_off[g.nblocks];
  if (st->total_bytes > cap) atomicOr(&st->err_bits, 1u << (-PMZ_ERR_CAPACITY));
}

int pmz_compress_encode(const float *d_in, const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes,
                        void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  WsStatus *S = at<WsStatus>(d_ws, L.status);
  CK(cudaFuncSetAttribute(k_codebook, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCbSmem));
  k_codebook<<<1, 1024, kCbSmem, st>>>(at<unsigned long long>(d_ws, L.hist), S,
                                       at<unsigned long long>(d_ws, L.cb_keys), at<unsigned long long>(d_ws, L.cb_w),
                                       at<unsigned>(d_ws, L.cb_parent), at<uint8_t>(d_ws, L.lens),
                                       at<unsigned>(d_ws, L.cw));
  if (G.nparts > 0) {
    if (use_tpath(G)) {
      launch_tmain_pk<kCMain>(d_in, G, k, nullptr, 0, d_ws, L, st);
    } else {
      k_part_bits<<<(unsigned)G.nparts, kPbW * 32, 0, st>>>(G, at<BlkP>(d_ws, L.blkp), at<int16_t>(d_ws, L.rqbuf),
                                                           at<uint8_t>(d_ws, L.lens),
                                                           at<unsigned long long>(d_ws, L.part_bits), S);
    }
  }
  return launch_check();
}

int pmz_compress_write_async(const pmz_geom *g, const pmz_params *p, int write_header, uint8_t *d_out,
                             uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes,
                             void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  WsStatus *S = at<WsStatus>(d_ws, L.status);
  k_block_sizes<<<(unsigned)((G.nblocks + 1 + 255) / 256), 256, 0, st>>>(
      G, at<BlkP>(d_ws, L.blkp), at<unsigned long long>(d_ws, L.part_bits),
      at<unsigned long long>(d_ws, L.part_zeros), at<unsigned long long>(d_ws, L.rec_size), S);
  size_t cb = L.cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(at<void>(d_ws, L.cub_tmp), cb, at<unsigned long long>(d_ws, L.rec_size),
                                   at<unsigned long long>(d_ws, L.rec_off), (int)(G.nblocks + 1), st));
  k_finish_status<<<1, 1, 0, st>>>(G, k, write_header, at<unsigned long long>(d_ws, L.rec_off), out_cap, S);
  // the writers read m, the header size and the capacity verdict from the
  // device status: one host synchronisation, at the end
  if (d_out != nullptr) {
    if (write_header)
      k_write_header<<<1, 256, 0, st>>>(d_out, G, k, g->global_rows, at<uint8_t>(d_ws, L.lens), S);
    if (G.nparts > 0 && use_tpath(G)) {
      k_c_write<<<(unsigned)((G.nparts + kCWW - 1) / kCWW), kCWW * 32, 0, st>>>(
          G, at<BlkP>(d_ws, L.blkp), at<unsigned>(d_ws, L.rqbuf), at<double>(d_ws, L.vbuf),
          at<uint2>(d_ws, L.clsbuf), at<double>(d_ws, L.anchors), at<unsigned long long>(d_ws, L.part_bits),
          at<unsigned long long>(d_ws, L.part_zeros), at<unsigned long long>(d_ws, L.rec_off), d_out, S);
    } else if (G.nparts > 0) {
      k_write_part<<<(unsigned)G.nparts, kWT, kWpSmem, st>>>(
          G, at<BlkP>(d_ws, L.blkp), at<int16_t>(d_ws, L.rqbuf), at<double>(d_ws, L.vbuf),
          at<double>(d_ws, L.anchors), at<unsigned long long>(d_ws, L.part_bits),
          at<unsigned long long>(d_ws, L.part_zeros), at<unsigned long long>(d_ws, L.rec_off),
          at<uint8_t>(d_ws, L.lens), at<unsigned>(d_ws, L.cw), d_out, S);
    }
    if (d_block_offsets)
      k_block_offsets<<<(unsigned)((G.nblocks + 1 + 255) / 256), 256, 0, st>>>(
          G, k, write_header, at<unsigned long long>(d_ws, L.rec_off), S, (unsigned long long *)d_block_offsets);
  }
  return launch_check();
}

int pmz_compress_finish_async(const float *d_in, const pmz_geom *g, const pmz_params *p, int write_header,
                              uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws,
                              uint64_t ws_bytes, void *stream) {
  const int s = pmz_compress_encode(d_in, g, p, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_compress_write_async(g, p, write_header, d_out, out_cap, d_block_offsets, d_ws, ws_bytes, stream);
}

int pmz_compress_result(const pmz_geom *g, const pmz_params *p, int wrote_output, void *d_ws, uint64_t ws_bytes,
                        void *stream, pmz_result *res) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  // status and coverage are adjacent at the front of the workspace: one copy
  static_assert(sizeof(WsStatus) <= 256, "status slot");
  alignas(8) uint8_t front[256 + 18 * 8];
  if (read_small(front, d_ws, L.cov + 18 * 8, st) != PMZ_OK) return PMZ_ERR_CUDA;
  WsStatus hs;
  memcpy(&hs, front, sizeof(WsStatus));
  if (res) {
    memset(res, 0, sizeof(*res));
    res->header_bytes = hs.header_bytes;
    res->record_bytes = hs.record_bytes;
    res->nblocks = (uint64_t)G.nblocks;
    res->ntrivial = hs.ntrivial;
    res->nbal = hs.nbal;
    res->nrepair = hs.nrepair;
    res->ncodes = hs.ncodes;
    res->m = hs.m;
    res->max_code_len = hs.max_len;
    res->unresolved = hs.unresolved;
    res->launches = hs.launches;
    memcpy(res->coverage, front + L.cov, 18 * 8);
  }
  int err = err_from_bits(hs.err_bits);
  if (err) return err;
  if (hs.unresolved) return PMZ_ERR_UNRESOLVED_ROUNDING;
  if (!wrote_output) return PMZ_ERR_CAPACITY;
  return PMZ_OK;
}

int pmz_compress_finish(const float *d_in, const pmz_geom *g, const pmz_params *p, int write_header, uint8_t *d_out,
                        uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes, void *stream,
                        pmz_result *res) {
  int s = pmz_compress_finish_async(d_in, g, p, write_header, d_out, out_cap, d_block_offsets, d_ws, ws_bytes,
                                    stream);
  if (s) return s;
  return pmz_compress_result(g, p, d_out != nullptr, d_ws, ws_bytes, stream, res);
}

int pmz_compress_enqueue(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val,
                         int64_t n_val, int write_header, uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets,
                         void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = pmz_compress_analyze(d_in, g, p, d_val, n_val, d_ws, ws_bytes, stream);
  if (s) return s;
  s = pmz_compress_codes(d_in, g, p, d_val, n_val, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_compress_finish_async(d_in, g, p, write_header, d_out, out_cap, d_block_offsets, d_ws, ws_bytes,
                                   stream);
}

int pmz_compress(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val, int64_t n_val,
                 uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes,
                 void *stream, pmz_result *res) {
  int s = pmz_compress_analyze(d_in, g, p, d_val, n_val, d_ws, ws_bytes, stream);
  if (s) return s;
  s = pmz_compress_codes(d_in, g, p, d_val, n_val, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_compress_finish(d_in, g, p, 1, d_out, out_cap, d_block_offsets, d_ws, ws_bytes, stream, res);
}

// ---------------------------------------------------------------------------
// container header / index (host)

namespace {
struct HReader {
  const uint8_t *b;
  uint64_t n, pos;
  bool err;
  bool get(void *d, uint64_t k) {
    if (err || pos + k > n) { err = true; return false; }
    memcpy(d, b + pos, k);
    pos += k;
    return true;
  }
  template <class T>
  T v() {
    T x{};
    get(&x, sizeof(T));
    return x;
  }
};
}  // namespace

int pmz_parse_header(const uint8_t *h, uint64_t n, pmz_header *hd) {
  memset(hd, 0, sizeof(*hd));
  HReader r{h, n, 0, false};
  char mg[4];
  if (!r.get(mg, 4)) return PMZ_ERR_CORRUPT;
  if (memcmp(mg, "PMEZ", 4) != 0) return PMZ_ERR_BAD_MAGIC;
  hd->version = r.v<uint16_t>();
  if (r.err) return PMZ_ERR_CORRUPT;
  if (hd->version != 1 && hd->version != 2) return PMZ_ERR_UNSUPPORTED_VERSION;  // 2: FP32 perf mode
  hd->elem = r.v<uint8_t>();
  hd->rows = r.v<uint64_t>();
  hd->cols = r.v<uint64_t>();
  hd->block_rows = r.v<uint32_t>();
  hd->block_cols = r.v<uint32_t>();
  hd->partition_rows = r.v<uint32_t>();
  hd->b_r = r.v<double>();
  hd->coverage_target = r.v<double>();
  hd->m = r.v<uint8_t>();
  uint64_t ml = r.v<uint64_t>();
  if (r.err) return PMZ_ERR_CORRUPT;
  if (hd->elem != 0) return PMZ_ERR_CORRUPT;
  if (hd->m < 4 || hd->m > 16 || hd->block_rows == 0 || hd->block_cols == 0 || hd->partition_rows == 0 ||
      hd->partition_rows > 32 || hd->block_rows / hd->partition_rows > 64)
    return PMZ_ERR_CORRUPT;
  if (!(hd->b_r > 0.0 && hd->b_r < 1.0)) return PMZ_ERR_CORRUPT;
  hd->S = r.v<uint32_t>();
  hd->H = r.v<uint32_t>();
  hd->slope = r.v<double>();
  if (r.err || hd->H != 2 || (hd->S != 1 && hd->S != 3)) return PMZ_ERR_CORRUPT;
  uint32_t nw1 = (hd->S + 1) * hd->H;
  if (ml != model_blob_bytes(hd->S, hd->H)) return PMZ_ERR_CORRUPT;
  for (uint32_t i = 0; i < nw1; i++) hd->w1[i] = r.v<double>();
  for (uint32_t i = 0; i < hd->H; i++) hd->w2[i] = r.v<double>();
  uint64_t cl = r.v<uint64_t>();
  uint64_t alpha = 1ull << hd->m;
  if (r.err || cl != 2 + alpha) return PMZ_ERR_CORRUPT;
  uint16_t a16 = r.v<uint16_t>();
  if (a16 != (uint16_t)(alpha & 0xffff)) return PMZ_ERR_CORRUPT;
  hd->lens_offset = r.pos;
  r.pos += alpha;
  hd->nblocks = r.v<uint64_t>();
  if (r.err) return PMZ_ERR_CORRUPT;
  uint64_t nb = (hd->rows && hd->cols)
                    ? ((hd->rows + hd->block_rows - 1) / hd->block_rows) * ((hd->cols + hd->block_cols - 1) / hd->block_cols)
                    : 0;
  if (hd->nblocks != nb) return PMZ_ERR_CORRUPT;
  hd->header_bytes = r.pos;
  return PMZ_OK;
}

int pmz_index_blocks_range(const uint8_t *h, uint64_t n, const pmz_header *hd, uint64_t b0, uint64_t b1,
                           uint64_t pos0, uint64_t *offs) {
  Geom G = make_geom((int64_t)hd->rows, (int64_t)hd->cols, (int)hd->block_rows, (int)hd->block_cols,
                     (int)hd->partition_rows, 0);
  if (b0 > b1 || b1 > (uint64_t)G.nblocks || !offs) return PMZ_ERR_CONFIG;
  uint64_t pos = pos0;
  for (int64_t b = (int64_t)b0; b < (int64_t)b1; b++) {
    if (pos >= n) return PMZ_ERR_TRUNCATED;
    offs[b - (int64_t)b0] = pos;
    uint8_t t = h[pos];
    if (t == 1) { pos += 1; continue; }
    if (t != 0) return PMZ_ERR_CORRUPT;
    BlockBox bb = block_box(G, b);
    uint64_t head = 25 + 24ull * bb.np;
    if (pos + head > n) return PMZ_ERR_TRUNCATED;
    uint64_t pay = 0;
    for (int i = 0; i < bb.np; i++) {
      uint64_t off, len;
      memcpy(&off, h + pos + 17 + 24ull * i, 8);
      memcpy(&len, h + pos + 25 + 24ull * i, 8);
      if (off != pay * 8) return PMZ_ERR_CORRUPT;
      if (len > 40ull * bb.br * bb.bc) return PMZ_ERR_CORRUPT;
      pay += (len + 7) / 8;
    }
    uint64_t nb;
    memcpy(&nb, h + pos + 17 + 24ull * bb.np, 8);
    if (nb > (uint64_t)bb.br * bb.bc) return PMZ_ERR_CORRUPT;
    pos += head + 8 * nb + pay;
    if (pos > n) return PMZ_ERR_TRUNCATED;
  }
  if (b1 == (uint64_t)G.nblocks && pos != n) return PMZ_ERR_CORRUPT;  // the last record ends the container
  offs[b1 - b0] = pos;
  return PMZ_OK;
}

int pmz_index_blocks(const uint8_t *h, uint64_t n, const pmz_header *hd, uint64_t *offs) {
  Geom G = make_geom((int64_t)hd->rows, (int64_t)hd->cols, (int)hd->block_rows, (int)hd->block_cols,
                     (int)hd->partition_rows, 0);
  return pmz_index_blocks_range(h, n, hd, 0, (uint64_t)G.nblocks, hd->header_bytes, offs);
}

// ---------------------------------------------------------------------------
// decompression

namespace {
struct DecLayout {
  size_t status, blkp, part_bits, part_off, zflag, anchors, bal_off, pay_off, blk_nbal, tab, sym, lut, lut1, npfix,
      codes, vtile, rowz, total;
  bool tpath;
};
DecLayout dec_layout(const Geom &g) {
  DecLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t a = o;
    o = align_up(o + bytes, 256);
    return a;
  };
  L.status = take(sizeof(WsStatus));
  L.blkp = take(sizeof(BlkP) * (size_t)(g.nblocks + 1));
  L.part_bits = take(8 * (size_t)(g.nparts + 1));
  L.part_off = take(8 * (size_t)(g.nparts + 1));
  L.zflag = take(4 * (size_t)(g.nparts + 1));                     // decoder look-back flags
  L.anchors = take(8 * (size_t)(g.nparts + 1));
  L.bal_off = take(8 * (size_t)(g.nblocks + 1));
  L.pay_off = take(8 * (size_t)(g.nblocks + 1));
  L.blk_nbal = take(8 * (size_t)(g.nblocks + 1));
  L.tab = take(sizeof(DecTab));
  L.sym = take(2 * kMaxAlpha);
  L.lut = take(4ull * ((1u << kLutBits) + kLut2Max));            // first + second level
  L.lut1 = take(kDLutBytes + 16);                                 // k_d_decode's tables + subtable counter
  L.npfix = take(sizeof(pmz_np_fix) * (size_t)(g.nblocks + 1));
  L.tpath = use_tpath(g, true);
  if (L.tpath) {
    L.codes = take(2 * (size_t)g.nparts * (size_t)g.prow * (size_t)g.bc);  // raster per partition (tcode_base)
    L.rowz = take(4 * (size_t)g.nparts * (size_t)g.prow + 4);  // code-0 count per row
    L.vtile = o;
  } else {
    L.codes = take(2 * (size_t)g.nparts * (size_t)g.nct * kTile);  // partition-tiled
    L.vtile = take(8 * (size_t)g.nparts * (size_t)g.nct * kTile);   // per-element addends, then reconstructed values
    L.rowz = o;
  }
  L.total = o;
  return L;
}
template <int PK>
int launch_recon(const KParams &k, unsigned grid, cudaStream_t st, const Geom &G, void *d_ws, const DecLayout &L,
                 float *d_out) {
  if (one_row_parts(G)) {
    k_reconstruct_1d<PK><<<(unsigned)((G.nparts + 31) / 32), 32, 0, st>>>(
        G, k, at<BlkP>(d_ws, L.blkp), at<uint16_t>(d_ws, L.codes), at<double>(d_ws, L.vtile),
        at<double>(d_ws, L.anchors), d_out, at<WsStatus>(d_ws, L.status));
    k_inv<<<(unsigned)G.nparts, 256, 0, st>>>(G, at<BlkP>(d_ws, L.blkp), at<double>(d_ws, L.vtile), d_out,
                                              at<WsStatus>(d_ws, L.status));
    return PMZ_OK;
  }
  CK(cudaFuncSetAttribute(k_reconstruct4<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDsc4Smem));
  k_reconstruct4<PK><<<grid, kPPC * 64, kDsc4Smem, st>>>(
      G, k, at<BlkP>(d_ws, L.blkp), at<uint16_t>(d_ws, L.codes), at<double>(d_ws, L.vtile),
      at<double>(d_ws, L.anchors), d_out, at<double>(d_ws, L.vtile), at<WsStatus>(d_ws, L.status));
  k_inv<<<(unsigned)G.nparts, 256, 0, st>>>(G, at<BlkP>(d_ws, L.blkp), at<double>(d_ws, L.vtile), d_out,
                                            at<WsStatus>(d_ws, L.status));
  return PMZ_OK;
}

Geom hdr_geom(const pmz_header *h) {
  Geom G = make_geom((int64_t)h->rows, (int64_t)h->cols, (int)h->block_rows, (int)h->block_cols,
                     (int)h->partition_rows, 0);
  G.fp32 = h->version == 2;
  return G;
}
KParams hdr_kparams(const pmz_header *h, double b_a) {
  KParams k{};
  k.b_r = h->b_r;
  k.b_a = b_a;
  k.two_ba = 2.0 * b_a;
  k.eps0 = 0x1p-126;
  k.slope = h->slope;
  for (int i = 0; i < 8; i++) k.w1[i] = h->w1[i];
  for (int i = 0; i < 2; i++) k.w2[i] = h->w2[i];
  k.S = (int)h->S;
  k.H = (int)h->H;
  k.block_rows = (int)h->block_rows;
  k.block_cols = (int)h->block_cols;
  k.partition_rows = (int)h->partition_rows;
  k.m_fixed = (int)h->m;
  k.inv_two_ba = 1.0 / (2.0 * b_a);
  k.init_model = is_init_model(k.S, k.w1, k.w2);
  k.precision = h->version == 2 ? 1 : 0;
  return k;
}
}  // namespace

int pmz_decompress_workspace_size(const pmz_header *hdr, uint64_t *bytes) {
  *bytes = dec_layout(hdr_geom(hdr)).total;
  return PMZ_OK;
}

int pmz_decompress_prepare(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                           const uint64_t *d_boff, void *d_ws, uint64_t ws_bytes, void *stream) {
  Geom G = hdr_geom(hdr);
  DecLayout L = dec_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  if (!(b_a > 0.0)) return PMZ_ERR_CONFIG;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = hdr_kparams(hdr, b_a);
  WsStatus *S = at<WsStatus>(d_ws, L.status);
  CK(cudaMemsetAsync(S, 0, sizeof(WsStatus), st));
  if (G.nblocks > 0) {
    k_dec_blocks<<<(unsigned)((G.nblocks + 3) / 4), 128, 0, st>>>(
        d_buf, n, G, k, (const unsigned long long *)d_boff, at<BlkP>(d_ws, L.blkp),
        at<unsigned long long>(d_ws, L.part_bits), at<unsigned long long>(d_ws, L.part_off),
        at<double>(d_ws, L.anchors), at<unsigned long long>(d_ws, L.bal_off),
        at<unsigned long long>(d_ws, L.pay_off), at<unsigned long long>(d_ws, L.blk_nbal), S,
        at<pmz_np_fix>(d_ws, L.npfix));
    k_dec_tables<<<1, 1024, 0, st>>>(d_buf + hdr->lens_offset, (int)hdr->m, at<DecTab>(d_ws, L.tab),
                                     at<uint16_t>(d_ws, L.sym), at<unsigned>(d_ws, L.lut), S);
    if (L.tpath) {
      unsigned *lut_n = at<unsigned>(d_ws, L.lut1 + kDLutBytes);
      CK(cudaMemsetAsync(lut_n, 0, 4, st));
      if (d_lut16((int)hdr->m))
        k_d_lut<uint16_t><<<(1u << DLut<uint16_t>::LB) / 256, 256, 0, st>>>(
            at<DecTab>(d_ws, L.tab), at<uint16_t>(d_ws, L.sym), 1 << (int)hdr->m, at<uint16_t>(d_ws, L.lut1), lut_n,
            S);
      else
        k_d_lut<unsigned><<<(1u << DLut<unsigned>::LB) / 256, 256, 0, st>>>(
            at<DecTab>(d_ws, L.tab), at<uint16_t>(d_ws, L.sym), 1 << (int)hdr->m, at<unsigned>(d_ws, L.lut1), lut_n,
            S);
    }
  }
  return launch_check();
}

int64_t pmz_decompress_np_fixups(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream, pmz_np_fix *h_fix,
                                 int64_t cap) {
  DecLayout L = dec_layout(hdr_geom(hdr));
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  return read_np_fixups(at<WsStatus>(d_ws, L.status), at<pmz_np_fix>(d_ws, L.npfix), (cudaStream_t)stream, h_fix,
                        cap);
}

int pmz_decompress_np_apply(const pmz_header *hdr, double b_a, void *d_ws, uint64_t ws_bytes, void *stream,
                            const pmz_np_fix *h_fix, int64_t n) {
  Geom G = hdr_geom(hdr);
  DecLayout L = dec_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  return apply_np_fixups(at<pmz_np_fix>(d_ws, L.npfix), at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status),
                         G.nblocks, 0x1p-126, b_a, (cudaStream_t)stream, h_fix, n);
}

int pmz_decompress_run(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a, const uint64_t *d_boff,
                       float *d_out, void *d_ws, uint64_t ws_bytes, void *stream) {
  Geom G = hdr_geom(hdr);
  DecLayout L = dec_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  if (!(b_a > 0.0)) return PMZ_ERR_CONFIG;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = hdr_kparams(hdr, b_a);
  WsStatus *S = at<WsStatus>(d_ws, L.status);
  if (G.nblocks > 0 && L.tpath) {
    const int center = 1 << ((int)hdr->m - 1);
    // a thread per partition substream: big CTAs when the partitions fill every SM
    // twice over, small ones otherwise so that they spread over all SMs (C3: 16384
    // partitions are 32 CTAs of 512 threads, or 128 CTAs of 128)
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    bool big = G.nparts >= (int64_t)sms * 2 * kDDT;
    if (const char *e = getenv("PMZ_DEC_CTA")) big = e[0] == 'b' ? true : (e[0] == 's' ? false : big);  // tests
#define PMZ_T_DECODE(E, T)                                                                                          \
  do {                                                                                                              \
    CK(cudaFuncSetAttribute(k_d_decode<E, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,                          \
                            (int)d_dec_smem<E, T>()));                                                              \
    k_d_decode<E, T><<<(unsigned)((G.nparts + T - 1) / T), T, d_dec_smem<E, T>(), st>>>(                            \
        d_buf, n, G, at<BlkP>(d_ws, L.blkp), at<DecTab>(d_ws, L.tab), at<uint16_t>(d_ws, L.sym), 1 << (int)hdr->m, \
        at<E>(d_ws, L.lut1), at<unsigned long long>(d_ws, L.part_bits), at<unsigned long long>(d_ws, L.part_off),  \
        at<unsigned long long>(d_ws, L.pay_off), at<uint16_t>(d_ws, L.codes), at<unsigned>(d_ws, L.zflag),         \
        at<unsigned>(d_ws, L.rowz), S);                                                                             \
  } while (0)
    if (d_lut16((int)hdr->m)) {
      if (big) PMZ_T_DECODE(uint16_t, kDDT);
      else PMZ_T_DECODE(uint16_t, kDDTSmall);
    } else {
      if (big) PMZ_T_DECODE(unsigned, kDDT);
      else PMZ_T_DECODE(unsigned, kDDTSmall);
    }
#undef PMZ_T_DECODE
    const unsigned grid = (unsigned)((G.nparts + kDRW - 1) / kDRW);
#define PMZ_T_RECON(PKV)                                                                                            \
  do {                                                                                                              \
    auto *fr = k.precision ? k_d_recon32<PKV> : k_d_recon<PKV>;                                                    \
    CK(cudaFuncSetAttribute(fr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDRecSmem));                      \
    fr<<<grid, kDRW * 32, kDRecSmem, st>>>(                                                                         \
        d_buf, n, G, k, at<BlkP>(d_ws, L.blkp), at<uint16_t>(d_ws, L.codes), at<unsigned>(d_ws, L.zflag),           \
        at<unsigned>(d_ws, L.rowz), at<double>(d_ws, L.anchors), at<unsigned long long>(d_ws, L.bal_off),           \
        at<unsigned long long>(d_ws, L.blk_nbal), center, d_out, S);                                                \
  } while (0)
    if (k.init_model == 3) PMZ_T_RECON(3);
    else if (k.init_model == 1) PMZ_T_RECON(1);
    else PMZ_T_RECON(0);
#undef PMZ_T_RECON
    return launch_check();
  }
  if (G.nblocks > 0) {
    if (one_row_parts(G)) {
      k_decode_1d<<<(unsigned)((G.nparts + kD1T - 1) / kD1T), kD1T, 0, st>>>(
          d_buf, n, G, at<BlkP>(d_ws, L.blkp), at<DecTab>(d_ws, L.tab), at<uint16_t>(d_ws, L.sym),
          at<unsigned>(d_ws, L.lut), at<unsigned long long>(d_ws, L.part_bits),
          at<unsigned long long>(d_ws, L.part_off), at<unsigned long long>(d_ws, L.pay_off),
          at<unsigned long long>(d_ws, L.bal_off), at<unsigned long long>(d_ws, L.blk_nbal), 1 << ((int)hdr->m - 1),
          k.two_ba, at<uint16_t>(d_ws, L.codes), at<double>(d_ws, L.vtile), S);
      k_gather_1d<<<(unsigned)((G.nparts + 3) / 4), 128, 0, st>>>(
          d_buf, n, G, at<BlkP>(d_ws, L.blkp), at<unsigned long long>(d_ws, L.bal_off),
          at<unsigned long long>(d_ws, L.blk_nbal), 1 << ((int)hdr->m - 1), k.two_ba, at<uint16_t>(d_ws, L.codes),
          at<double>(d_ws, L.vtile), S);
    } else {
    CK(cudaMemsetAsync(at<unsigned>(d_ws, L.zflag), 0, 4 * (size_t)G.nparts, st));
    CK(cudaFuncSetAttribute(k_decode4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kD4Smem));
    k_decode4<<<(unsigned)G.nparts, kD4Threads, kD4Smem, st>>>(
        d_buf, n, G, at<BlkP>(d_ws, L.blkp), at<DecTab>(d_ws, L.tab), at<uint16_t>(d_ws, L.sym),
        at<unsigned>(d_ws, L.lut), at<unsigned long long>(d_ws, L.part_bits),
        at<unsigned long long>(d_ws, L.part_off), at<unsigned long long>(d_ws, L.pay_off),
        at<unsigned long long>(d_ws, L.bal_off), at<unsigned long long>(d_ws, L.blk_nbal), 1 << ((int)hdr->m - 1),
        k.two_ba, at<unsigned>(d_ws, L.zflag), at<uint16_t>(d_ws, L.codes), at<double>(d_ws, L.vtile), S);
    }
    const unsigned rgrid = (unsigned)((G.nparts + kPPC - 1) / kPPC);
    int s2;
    if (k.init_model == 3) s2 = launch_recon<3>(k, rgrid, st, G, d_ws, L, d_out);
    else if (k.init_model == 1) s2 = launch_recon<1>(k, rgrid, st, G, d_ws, L, d_out);
    else s2 = launch_recon<0>(k, rgrid, st, G, d_ws, L, d_out);
    if (s2) return s2;
  }
  return launch_check();
}

int pmz_decompress_enqueue(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                           const uint64_t *d_boff, float *d_out, void *d_ws, uint64_t ws_bytes, void *stream) {
  const int s = pmz_decompress_prepare(d_buf, n, hdr, b_a, d_boff, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_decompress_run(d_buf, n, hdr, b_a, d_boff, d_out, d_ws, ws_bytes, stream);
}

int pmz_decompress_result(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream) {
  Geom G = hdr_geom(hdr);
  DecLayout L = dec_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  WsStatus hs;
  if (read_small(&hs, at<WsStatus>(d_ws, L.status), sizeof(WsStatus), st) != PMZ_OK) return PMZ_ERR_CUDA;
  const int s = err_from_bits(hs.err_bits);
  if (s && getenv("PMZ_DEBUG"))
    fprintf(stderr, "pmz_decompress: status %d bits 0x%x first site %d part %d\n", s, hs.err_bits, hs.err_site,
            hs.err_part);
  if (s) return s;
  if (hs.unresolved) return PMZ_ERR_UNRESOLVED_ROUNDING;
  return PMZ_OK;
}

int pmz_decompress_status(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream, pmz_result *res) {
  Geom G = hdr_geom(hdr);
  DecLayout L = dec_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  WsStatus hs;
  if (read_small(&hs, at<WsStatus>(d_ws, L.status), sizeof(WsStatus), st) != PMZ_OK) return PMZ_ERR_CUDA;
  if (res) {
    memset(res, 0, sizeof(*res));
    res->nblocks = (uint64_t)G.nblocks;
    res->m = (int32_t)hdr->m;
    res->unresolved = hs.unresolved;
    res->launches = hs.launches;
  }
  const int s = err_from_bits(hs.err_bits);
  if (s) return s;
  if (hs.unresolved) return PMZ_ERR_UNRESOLVED_ROUNDING;
  return PMZ_OK;
}

int pmz_decompress(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a, const uint64_t *d_boff,
                   float *d_out, void *d_ws, uint64_t ws_bytes, void *stream) {
  const int s = pmz_decompress_enqueue(d_buf, n, hdr, b_a, d_boff, d_out, d_ws, ws_bytes, stream);
  if (s) return s;
  return pmz_decompress_result(hdr, d_ws, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// transform module entry points

__global__ void k_params10(Geom g, const BlkP *blkp, KParams k, double *out, uint8_t *triv) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nblocks) return;
  BlkP P = blkp[b];
  double *o = out + 10 * b;
  o[0] = P.factor_pos; o[1] = P.factor_neg; o[2] = k.eps0; o[3] = k.b_r; o[4] = k.b_a;
  o[5] = P.boundary; o[6] = P.zero_code; o[7] = P.zero_threshold; o[8] = P.lg_pos; o[9] = P.lg_neg;
  triv[b] = (uint8_t)P.trivial;
}

int pmz_transform_params(const float *d_in, const pmz_geom *g, const pmz_params *p, double *d_params10,
                         uint8_t *d_trivial, void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  CK(cudaMemsetAsync(d_ws, 0, L.lens, st));
  if (G.nblocks == 0) return PMZ_OK;
  k_block_params<kNT><<<(unsigned)G.nblocks, kNT, 0, st>>>(d_in, G, k, at<BlkP>(d_ws, L.blkp),
                                                            at<WsStatus>(d_ws, L.status));
  k_params10<<<(unsigned)((G.nblocks + 127) / 128), 128, 0, st>>>(G, at<BlkP>(d_ws, L.blkp), k, d_params10,
                                                                  d_trivial);
  s = launch_check();
  if (s) return s;
  WsStatus hs;
  if (read_small(&hs, at<WsStatus>(d_ws, L.status), sizeof(WsStatus), st) != PMZ_OK) return PMZ_ERR_CUDA;
  return err_from_bits(hs.err_bits);
}

struct P10 { double v[10]; };

__global__ void k_forward(const double *x, uint64_t n, P10 q, double *v, unsigned *amb) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xi = x[i];
  if (xi == 0.0) { v[i] = q.v[6]; return; }
  double a = fabs(xi), lg;
  float af = (float)a;
  if ((double)af == a && af >= 1.17549435e-38f && isfinite(af)) lg = pmz_log2_f32_fast(a, amb);
  else if (a >= 0x1p-1022 && isfinite(a)) lg = pmz_log2_d(a, amb);
  else lg = log2(a);  // subnormal doubles / inf: outside the path's domain
  v[i] = xi > 0.0 ? __dadd_rn(lg, q.v[8]) : __dadd_rn(lg, q.v[9]);
}

__global__ void k_inverse(const double *v, uint64_t n, P10 q, double *x64, float *x32, unsigned *amb) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double vi = v[i], r;
  if (vi <= q.v[7]) r = 0.0;
  else if (vi > q.v[5]) r = -pmz_exp2_cr(__dsub_rn(vi, q.v[9]), amb);
  else r = pmz_exp2_cr(__dsub_rn(vi, q.v[8]), amb);
  if (x64) x64[i] = r;
  if (x32) x32[i] = __double2float_rn(r);
}

int pmz_forward_map(const double *d_x, uint64_t n, const double *params10, double *d_v, void *stream) {
  P10 q;
  memcpy(q.v, params10, sizeof(q.v));
  if (n == 0) return PMZ_OK;
  k_forward<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_x, n, q, d_v, nullptr);
  return launch_check();
}

int pmz_inverse_map(const double *d_v, uint64_t n, const double *params10, double *d_x64, float *d_x32,
                    void *stream) {
  P10 q;
  memcpy(q.v, params10, sizeof(q.v));
  if (n == 0) return PMZ_OK;
  k_inverse<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_v, n, q, d_x64, d_x32, nullptr);
  return launch_check();
}

// compute_block_stats (transform.py:84-107) over n doubles: one CTA per 8192
// elements, warp/CTA reductions, atomics on order-preserving bit patterns.
// out[0..5] = abs_min (nonzero), abs_max, has_zero, has_negative, nonfinite, count.
__global__ void k_block_stats_f64(const double *__restrict__ x, uint64_t n, unsigned long long *acc) {
  unsigned long long mn = ~0ull, mx = 0ull;  // bit patterns of non-negative doubles order like the values
  int zero = 0, neg = 0, nonfin = 0;
  const uint64_t base = (uint64_t)blockIdx.x * 8192;
  for (uint64_t i = base + threadIdx.x; i < n && i < base + 8192; i += blockDim.x) {
    const double v = x[i];
    if (!isfinite(v)) { nonfin = 1; continue; }
    const double a = fabs(v);
    if (a > 0.0) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(a);
      mn = min(mn, b);
      mx = max(mx, b);
    } else {
      zero = 1;
    }
    if (v < 0.0) neg = 1;
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  zero = __any_sync(0xffffffffu, zero);
  neg = __any_sync(0xffffffffu, neg);
  nonfin = __any_sync(0xffffffffu, nonfin);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&acc[0], mn);
    atomicMax(&acc[1], mx);
    if (zero) atomicOr(&acc[2], 1ull);
    if (neg) atomicOr(&acc[3], 1ull);
    if (nonfin) atomicOr(&acc[4], 1ull);
  }
}
__global__ void k_block_stats_init(unsigned long long *acc) {
  acc[0] = ~0ull;
  acc[1] = acc[2] = acc[3] = acc[4] = 0ull;
}
__global__ void k_block_stats_out(const unsigned long long *acc, uint64_t n, double *out) {
  const bool any = acc[0] != ~0ull;
  out[0] = any ? __longlong_as_double((long long)acc[0]) : 0.0;
  out[1] = any ? __longlong_as_double((long long)acc[1]) : 0.0;
  out[2] = (double)acc[2];
  out[3] = (double)acc[3];
  out[4] = (double)acc[4];
  out[5] = (double)n;
}

int pmz_block_stats(const double *d_x, uint64_t n, double *d_out6, void *d_scratch, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(d_scratch);
  k_block_stats_init<<<1, 1, 0, st>>>(acc);
  if (n > 0) k_block_stats_f64<<<(unsigned)((n + 8191) / 8192), 256, 0, st>>>(d_x, n, acc);
  k_block_stats_out<<<1, 1, 0, st>>>(acc, n, d_out6);
  return launch_check();
}

// derive_transform_params (transform.py:110-135) on the device: in4 = factor_pos,
// factor_neg, b_r, epsilon0; out10 in TransformParams field order; mask bit i
// set when np.log2 of (factor_neg, factor_pos - epsilon0, factor_pos,
// epsilon0)[i] must be decided by the host (numpy), see pmz_np_fix.
__global__ void k_derive_params(const double *in4, double b_a, double *out10, int *mask) {
  const int lane = threadIdx.x;
  const double fp = in4[0], fn = in4[1], b_r = in4[2], e0 = in4[3];
  const double arg = lane == 0 ? fn : (lane == 1 ? __dsub_rn(fp, e0) : (lane == 2 ? fp : e0));
  double l = 0.0;
  int und = 0;
  if (lane < 4) {
    l = pmz_log2_d(arg, nullptr);
    und = np_log2_undecided(arg) ? 1 : 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, und);
  const double lg_neg = __shfl_sync(0xffffffffu, l, 0), lpe = __shfl_sync(0xffffffffu, l, 1),
               lg_pos = __shfl_sync(0xffffffffu, l, 2), l0 = __shfl_sync(0xffffffffu, l, 3);
  if (lane == 0) {
    const double zc = __dadd_rn(l0, lg_pos);
    out10[0] = fp; out10[1] = fn; out10[2] = e0; out10[3] = b_r; out10[4] = b_a;
    out10[5] = __dsub_rn(__dadd_rn(lg_neg, lpe), b_a);  // boundary, :123
    out10[6] = zc;                                        // zero_code_value, :121
    out10[7] = __dadd_rn(zc, b_a);                        // zero_threshold, :122
    out10[8] = lg_pos; out10[9] = lg_neg;
    *mask = (int)(bal & 15u);
  }
}

int pmz_derive_params(const double *d_in4, double b_a, double *d_out10, int32_t *d_mask, void *stream) {
  k_derive_params<<<1, 32, 0, (cudaStream_t)stream>>>(d_in4, b_a, d_out10, d_mask);
  return launch_check();
}

// zero_sub_floor_magnitudes (transform.py:205-210) elementwise on doubles
__global__ void k_zero_sub_floor(const double *__restrict__ x, uint64_t n, double eps0, double *out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    out[i] = fabs(v) <= eps0 ? 0.0 : v;
  }
}

int pmz_zero_sub_floor(const double *d_x, uint64_t n, double eps0, double *d_out, void *stream) {
  if (n == 0) return PMZ_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  k_zero_sub_floor<<<grid, 256, 0, (cudaStream_t)stream>>>(d_x, n, eps0, d_out);
  return launch_check();
}

__global__ void k_log2_batch(const float *x, uint64_t n, double *out, unsigned *amb, int variant) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double a = (double)x[i];
    out[i] = variant == 0 ? pmz_log2_f32_fast(a, amb) : (variant == 1 ? pmz_log2_f32(a, amb) : pmz_log2_d(a, amb));
  }
}

int pmz_log2_f32_batch(const float *d_x, uint64_t n, double *d_out, uint32_t *d_amb, int variant, void *stream) {
  if (n == 0) return PMZ_OK;
  k_log2_batch<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(d_x, n, d_out, d_amb, variant);
  return launch_check();
}


// Host pipeline helper (hostpipe.py): pack n blocks of br x bc floats out of a
// row-major host field (row length `cols`) into a dense host array, block i at
// h_dst + i * br * bc, on `nthreads` host threads.  (Strided DMA copies of the
// same blocks run at ~22 GB/s: 1 KiB rows; packed, the blocks upload as one
// contiguous copy while the CPU packing overlaps the first slab uploads.)
extern "C" PMZ_API int pmz_pack_blocks_host(const float *h_field, int64_t cols, int32_t br, int32_t bc,
                                            const int64_t *h_r0, const int64_t *h_c0, int64_t n, float *h_dst,
                                            int32_t nthreads) {
  if (!h_field || !h_dst || !h_r0 || !h_c0 || cols <= 0 || br <= 0 || bc <= 0 || n < 0) return PMZ_ERR_CONFIG;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads > 0 ? nthreads : 1, n));
  auto work = [&](int tid) {
    for (int64_t i = tid; i < n; i += T) {
      const float *src = h_field + h_r0[i] * cols + h_c0[i];
      float *dst = h_dst + i * (int64_t)br * bc;
      for (int r = 0; r < br; r++) memcpy(dst + (int64_t)r * bc, src + (int64_t)r * cols, (size_t)bc * 4);
    }
  };
  if (T == 1) {
    work(0);
    return PMZ_OK;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int t = 0; t < T; t++) th.emplace_back(work, t);
  for (auto &t : th) t.join();
  return PMZ_OK;
}

#ifdef PMZ_CSTATS
extern "C" PMZ_API int pmz_cstats_read(void *host) {
  return cudaMemcpyFromSymbol(host, pmz::g_cstats, sizeof(pmz::g_cstats)) == cudaSuccess ? 0 : -1;
}
#endif
#ifdef PMZ_D3_PROF
// experiments only (tools/dec_bench.py): the decoder's per-partition phase timestamps
extern "C" PMZ_API int pmz_d3prof_read(void *host, uint64_t bytes) {
  return cudaMemcpyFromSymbol(host, pmz::g_d3prof, bytes) == cudaSuccess ? 0 : -1;
}
#endif

#ifdef PMZ_CMP_PROFILE
// experiments only: the codebook kernel's phase timestamps
extern "C" PMZ_API int pmz_cbprof_read(void *host) {
  return cudaMemcpyFromSymbol(host, pmz::g_cb_prof, 8 * sizeof(long long)) == cudaSuccess ? 0 : -1;
}
#endif

// ---------------------------------------------------------------------------
// trainer objective

int pmz_train_gradient(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_blocks,
                       int64_t n_blocks, double *d_out12, void *d_ws, uint64_t ws_bytes, void *stream) {
  int s = check_params(p);
  if (s) return s;
  Geom G = geom_of(p, g);
  WsLayout L = compress_layout(G);
  if (ws_bytes < L.total) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  CK(cudaMemsetAsync(d_ws, 0, L.lens, st));  // status, flags, block stats
  CK(cudaMemsetAsync(d_out12, 0, sizeof(double) * kTrC, st));
  if (G.nblocks == 0 || n_blocks <= 0) return launch_check();
  // (the training objective keeps the device's CR per-block logarithms: no host fixup)
  k_stats<<<(unsigned)G.nblocks, kST, 0, st>>>(d_in, G, k, at<BlkP>(d_ws, L.blkp), at<BlkStat>(d_ws, L.bstat),
                                               at<WsStatus>(d_ws, L.status), nullptr);
  // the training blocks are flagged in the validation-flag slots (no quantization runs here)
  k_mark_val<<<(unsigned)((n_blocks + 255) / 256), 256, 0, st>>>(d_blocks, n_blocks, G.nblocks,
                                                                   at<uint8_t>(d_ws, L.vflag),
                                                                   at<WsStatus>(d_ws, L.status));
  k_fwd<<<(unsigned)G.nparts, kFqT, 0, st>>>(d_in, G, at<BlkP>(d_ws, L.blkp), at<WsStatus>(d_ws, L.status),
                                             at<double>(d_ws, L.vbuf), at<uint8_t>(d_ws, L.clsbuf));
  // per-partition partials in the (unused here) rq tiles: >= 2 KB per partition
  double *part = at<double>(d_ws, L.rqbuf);
  k_train_tiles<<<(unsigned)G.nparts, kTrT, 0, st>>>(G, k, at<BlkP>(d_ws, L.blkp), at<uint8_t>(d_ws, L.vflag),
                                                    at<double>(d_ws, L.vbuf), part);
  k_train_reduce<<<1, 32, 0, st>>>(part, G.nparts, d_out12);
  s = launch_check();
  if (s) return s;
  WsStatus hs;
  if (read_small(&hs, at<WsStatus>(d_ws, L.status), sizeof(WsStatus), st) != PMZ_OK) return PMZ_ERR_CUDA;
  return err_from_bits(hs.err_bits);
}

int pmz_train_gradient_batch(const double *d_surf, const double *d_tgt, uint64_t n, const pmz_params *p,
                             double *d_out12, void *d_ws, uint64_t ws_bytes, void *stream) {
  if (!p || (p->S != 1 && p->S != 3) || p->H != 2) return PMZ_ERR_CONFIG;
  if (ws_bytes < (uint64_t)PMZ_TRAIN_BATCH_WS) return PMZ_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  KParams k = kparams(p);
  const unsigned grid = PMZ_TRAIN_BATCH_WS / (kTrC * 8);
  k_train_batch<<<grid, kTrT, 0, st>>>(k, d_surf, d_tgt, n, reinterpret_cast<double *>(d_ws));
  k_train_reduce<<<1, 32, 0, st>>>(reinterpret_cast<const double *>(d_ws), grid, d_out12);
  return launch_check();
}

// ---------------------------------------------------------------------------
// SEG-Y ingest

int pmz_segy_samples(const uint8_t *d_traces, uint64_t n_traces, uint32_t ns, int format_code, float *d_out,
                     void *stream) {
  if (format_code != 1 && format_code != 5) return PMZ_ERR_CONFIG;
  if (n_traces == 0 || ns == 0) return PMZ_OK;
  const uint64_t n = n_traces * ns;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  k_segy_samples<<<grid, 256, 0, (cudaStream_t)stream>>>(d_traces, n_traces, ns, format_code, d_out);
  return launch_check();
}
