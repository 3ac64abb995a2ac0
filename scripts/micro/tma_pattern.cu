// Microbenchmark: HBM read bandwidth of TMA box patterns (diagnosis only, not part of the product).
// A: y-solve pattern, element-major layout: box {16 deg, 8 el (1 KB apart), 1, 16 rows}
// B: same bytes, degree-block-major layout: box {16 deg, 8 el (128 B apart), 1, 1, 16 rows}
// C: x-solve pattern: box {256 cols, 1, 8 rows}
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../../paper_2402_11299_b200/csrc/ptx.cuh"
using namespace hpfem;

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (EncFn)p;
}
constexpr int NST = 6, STAGE = 16384;

template <int PAT>
__global__ void __launch_bounds__(32) k(const __grid_constant__ CUtensorMap m, int ntiles, int spt, unsigned long long* sink, int kwn) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * STAGE);
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int my = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int total = my * spt;
  auto issue = [&](int g) {
    const int tl = g / spt, s = g % spt, tile = blockIdx.x + tl * gridDim.x, slot = g % NST;
    mbar_expect_tx(&full[slot], STAGE);
    if (PAT == 0) {  // tile = (g8 16, e_x 128, kw 4)
      const int gg = tile % 16, ex = (tile / 16) % 128, kw = (tile / 2048) % kwn;
      tma_load_4d(sm + slot * STAGE, &m, &full[slot], 16 * s, 8 * gg, ex, 16 * kw);
    } else if (PAT == 1) {
      const int gg = tile % 16, ex = (tile / 16) % 128, kw = (tile / 2048) % kwn;
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(su32(sm + slot * STAGE)), "l"(&m), "r"(0), "r"(8 * gg), "r"(s), "r"(ex), "r"(16 * kw), "r"(su32(&full[slot])) : "memory");
    } else {  // x: tile = (e_x 128, group 64 of 256 cols, kh-block 8 of 8 rows): stage = 8 rows
      const int ex = tile % 128, gg = (tile / 128) % 64;
      tma_load_3d(sm + slot * STAGE, &m, &full[slot], 256 * gg, ex, (8 * s) % (8 * kwn));
    }
  };
  for (int g = 0; g < NST && g < total; ++g) issue(g);
  unsigned long long acc = 0;
  for (int g = 0; g < total; ++g) {
    mbar_wait(&full[g % NST], (g / NST) & 1);
    acc += reinterpret_cast<const unsigned long long*>(sm + (g % NST) * STAGE)[g & 1023];
    if (g + NST < total) issue(g + NST);
  }
  if (acc == 0x12345) *sink = acc;
}

int main(int argc, char** argv) {
  const uint64_t ld = 16512, rows = argc > 1 ? 16384 / atoi(argv[1]) : 16384;  // ~2.16 GB (argv[1] = divisor: L2-resident runs)
  double* a; cudaMalloc(&a, ld * rows * 8); cudaMemset(a, 0, ld * rows * 8);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  EncFn f = enc();
  CUtensorMap mA, mB, mC;
  cuuint32_t e5[5] = {1, 1, 1, 1, 1};
  {  // A: {Q=128, n=128 (1 KB), e_x 128 (ld), kh 64 (2*128*ld)}
    cuuint64_t d[4] = {128, 128, 128, 64 * rows / 16384}; cuuint64_t s[3] = {1024, ld * 8, 2 * 128 * ld * 8}; cuuint32_t b[4] = {16, 8, 1, 16};
    printf("encA %d\n", (int)f(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a, d, s, b, e5, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {  // B: {16, n=128 (128 B), 8 blocks (16 KB), e_x 128, kh 64}
    cuuint64_t d[5] = {16, 128, 8, 128, 64 * rows / 16384}; cuuint64_t s[4] = {128, 16384, ld * 8, 2 * 128 * ld * 8}; cuuint32_t b[5] = {16, 8, 1, 1, 16};
    printf("encB %d\n", (int)f(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a, d, s, b, e5, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {  // C: {ld, e_x 128, kh 64}
    cuuint64_t d[3] = {16384, 128, 64 * rows / 16384}; cuuint64_t s[2] = {ld * 8, 2 * 128 * ld * 8}; cuuint32_t b[3] = {256, 1, 8};
    printf("encC %d\n", (int)f(&mC, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, d, s, b, e5, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  const int smem = NST * STAGE + 1024;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ctas : {148, 296}) for (int pat = 0; pat < 3; ++pat) {
    const int ntiles = pat < 2 ? 16 * 128 * 4 : 128 * 64 * 1, spt = 8;  // A/B: 8192 tiles x 8 x 16 KB; C: 8192 x 8 x 16 KB
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (pat == 0) k<0><<<ctas, 32, smem>>>(mA, ntiles, spt, sink, (int)(4 * rows / 16384));
      else if (pat == 1) k<1><<<ctas, 32, smem>>>(mB, ntiles, spt, sink, (int)(4 * rows / 16384));
      else k<2><<<ctas, 32, smem>>>(mC, ntiles, spt, sink, (int)(8 * rows / 16384));
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double bytes = (double)ntiles * spt * STAGE;
    printf("ctas %d pattern %c: %.3f ms  %.1f GB/s  (err %s)\n", ctas, "ABC"[pat], best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
