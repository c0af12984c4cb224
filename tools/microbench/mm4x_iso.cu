// The product fp4 operand-copy scan kernel (fps_mma4x.cuh) run in isolation
// on synthetic operands, to compare its per-tile cost with the stripped-down
// pipeline of mm_pipe.cu (B200, sm_100a):
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1906_06170_b200/csrc \
//        -o mm4x_iso tools/microbench/mm4x_iso.cu -lcuda && ./mm4x_iso
//
// Random operand tiles and B columns, tests off (FPS_SCAN_FLAGS 4096: no
// candidate lists needed), 5 query chunks per library range as in C4.
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "fps_mma4x.cuh"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

using namespace fps;

template <int EPI, int N = 208>
void run(u64 n_tiles, u32 nchunks, u32 parts, unsigned flags, unsigned char* op, const CUtensorMap& tmap,
         unsigned char* bop, u32* qcol, const char* what) {
  MmArgs a{};
  a.n = n_tiles * MM_M;
  a.n_tiles = n_tiles;
  a.Q = nchunks * N;
  a.nchunks = nchunks;
  a.parts = parts;
  a.bop = bop;
  a.qcol = qcol;
  a.mode = 0;
  a.flags = flags;
  const size_t smem = mm4x_smem(N);
  CK(cudaFuncSetAttribute(mma4x_scan_kernel<N, EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  mma4x_scan_kernel<N, EPI, 2><<<nchunks * parts, mm4x_threads(EPI), smem>>>(a, op, tmap);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma4x_scan_kernel<N, EPI, 2><<<nchunks * parts, mm4x_threads(EPI), smem>>>(a, op, tmap);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int mhz = 0;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  const double tiles_per_cta = (double)n_tiles / parts;
  printf("N=%3d EPI=%2d chunks=%u parts=%u flags=%8u %-36s %.3f ms  %.1f ns/tile\n", N, EPI, nchunks, parts, flags,
         what, ms, ms * 1e6 / tiles_per_cta);
}

int main(int argc, char** argv) {
  const u64 n_tiles = 745447;  // 95,417,114 entries / 128
  unsigned char* op;
  CK(cudaMalloc(&op, n_tiles * MM4X_TILE));
  {
    std::vector<u32> h(n_tiles * MM4X_TILE / 4 / 16);
    u32 x = 7;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; v = x & 0x77777777u; }  // nibbles 0..7 (positive e2m1)
    for (int r = 0; r < 16; ++r) CK(cudaMemcpy(op + (size_t)r * h.size() * 4, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  }
  unsigned char* bop;
  u32* qcol;
  CK(cudaMalloc(&bop, 8 * mm4_b_bytes(208)));
  CK(cudaMalloc(&qcol, 8 * 208 * 4));
  CK(cudaMemset(bop, 0x22, 8 * mm4_b_bytes(208)));
  CK(cudaMemset(qcol, 0, 8 * 208 * 4));
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  alignas(64) CUtensorMap tmap;
  const cuuint64_t gdim[2] = {MM4X_ROW, (cuuint64_t)n_tiles * MM4X_BOX_ROWS};
  const cuuint64_t gstride[1] = {MM4X_ROW};
  const cuuint32_t box[2] = {MM4X_ROW, MM4X_BOX_ROWS};
  const cuuint32_t es[2] = {1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, op, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  // (the test epilogue stays off: this harness sets up no candidate lists)
  const unsigned OFF = 4096, NO_LOADS = 8192, NO_MMA = 1u << 23;
  if (argc > 1) {  // one variant (for ncu): extra flags
    run<8>(n_tiles / 4, 5, 29, OFF | (unsigned)strtoul(argv[1], nullptr, 0), op, tmap, bop, qcol, "single variant");
    return 0;
  }
  run<8>(n_tiles, 5, 29, OFF, op, tmap, bop, qcol, "C4 shape, tests off");
  run<8>(n_tiles, 5, 29, OFF | NO_LOADS, op, tmap, bop, qcol, "no operand loads");
  run<8>(n_tiles, 5, 29, OFF | NO_MMA, op, tmap, bop, qcol, "no MMAs");
  run<8>(n_tiles, 5, 29, OFF | NO_LOADS | NO_MMA, op, tmap, bop, qcol, "no operand loads, no MMAs");
  run<8>(n_tiles / 6, 5, 29, OFF, op, tmap, bop, qcol, "1/6 of the tiles");
  run<8>(n_tiles, 1, 148, OFF, op, tmap, bop, qcol, "1 chunk (C5-like, N = 208)");
  run<16>(n_tiles, 5, 29, OFF, op, tmap, bop, qcol, "16 epilogue warps");
  return 0;
}
