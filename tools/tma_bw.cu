// TMA streaming microbenchmark (diagnostic): how fast can one CTA per SM pull
// 32 KB tiles from random 16 KB "pages" of a large HBM buffer into a smem ring?
//   mode 0: tensor TMA, boxes of 64 rows x 128 B (4 boxes / tile), one issuing thread
//   mode 1: 1-D bulk copies (cp.async.bulk), 2 x 16 KB per tile, one issuing thread
//   mode 2: tensor TMA, two issuing threads (alternate tiles)
//   mode 3: 1-D bulk copies, 4 x 8 KB per tile, one issuing thread
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_24832_b200/csrc/ptx.cuh"
using namespace optimus;

#ifndef STAGES
#define STAGES 6
#endif
#ifndef HOLD
#define HOLD 0
#endif
constexpr int TILE = 32768;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* buf,
                                                        const int* pages, int n_tiles, int mode, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + STAGES * TILE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_fence_init();
  }
  __syncthreads();
  const int* pg = pages + (int64_t)blockIdx.x * n_tiles * 2;
  const int n_prod = mode == 2 ? 2 : 1;
  if (warp < n_prod && lane == 0) {
    for (int t = warp; t < n_tiles; t += n_prod) {
      const int st = t % STAGES;
      mbar_wait(&empty[st], ((t / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[st], TILE);
      uint8_t* dst = sm + st * TILE;
      const int p0 = pg[2 * t], p1 = pg[2 * t + 1];
      if (mode == 0 || mode == 2) {
        // two 16 KB pages, each [64 rows][256 B] -> 2 boxes of 64 x 128 B per page
        for (int k = 0; k < 2; ++k) {
          const int page = k ? p1 : p0;
          tma_load_4d(dst + k * 16384, &tm, &full[st], 0, 0, 0, page);
          tma_load_4d(dst + k * 16384 + 8192, &tm, &full[st], 64, 0, 0, page);
        }
      } else if (mode == 1) {
        bulk_g2s(dst, buf + (int64_t)p0 * 16384, 16384, &full[st]);
        bulk_g2s(dst + 16384, buf + (int64_t)p1 * 16384, 16384, &full[st]);
      } else {
        for (int k = 0; k < 4; ++k) {
          const int page = (k < 2) ? p0 : p1;
          bulk_g2s(dst + k * 8192, buf + (int64_t)page * 16384 + (k & 1) * 8192, 8192, &full[st]);
        }
      }
    }
  } else if (warp == 3) {
    float acc = 0.f;
    for (int t = 0; t < n_tiles; ++t) {
      const int st = t % STAGES;
      mbar_wait(&full[st], (t / STAGES) & 1);
      acc += *(volatile float*)(sm + st * TILE + lane * 4);
      if (HOLD) { const long long t0 = clock64(); while (clock64() - t0 < HOLD) {} }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (lane == 0) sink[blockIdx.x] = acc;
  }
}

int main(int argc, char** argv) {
  const int n_pages = 1 << 17;  // 2 GB of 16 KB pages
  const int n_tiles = 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  cudaMalloc(&buf, (size_t)n_pages * 16384);
  cudaMemset(buf, 1, (size_t)n_pages * 16384);
  std::vector<int> hp((size_t)sms * n_tiles * 2);
  srand(1);
  for (auto& x : hp) x = rand() % n_pages;
  int* pages;
  cudaMalloc(&pages, hp.size() * 4);
  cudaMemcpy(pages, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
  float* sink;
  cudaMalloc(&sink, sms * 4);
  // tensor view: [pages][64 rows][128 elems bf16]
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t gd[4] = {128, 64, 1, (cuuint64_t)n_pages};
  cuuint64_t gs[3] = {256, 16384, 16384};
  cuuint32_t bd[4] = {64, 64, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, gd, gs, bd, es,
                                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
  const int smem = STAGES * TILE + 1024 + 2048;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"tensor 4x(64x128B) 1 thread", "bulk 2x16KB 1 thread", "tensor 2 threads", "bulk 4x8KB 1 thread"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      stream_kernel<<<sms, 128, smem>>>(tm, buf, pages, n_tiles, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      if (rep == 2) printf("mode %d %-30s %8.1f GB/s  (%s)\n", mode, names[mode],
                           (double)sms * n_tiles * TILE / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    }
  }
  return 0;
}
