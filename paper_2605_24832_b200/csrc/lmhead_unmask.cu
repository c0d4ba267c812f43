// f3: LM-head GEMM with the unmask statistics in its epilogue.
//
// logits[r, v] = sum_k H[r, k] * W[v, k] is never written to memory.  Each CTA owns a
// 128-row x 256-vocab tile: TMA streams 64-wide k-blocks of H and W into a 4-stage
// shared-memory ring (SWIZZLE_128B, K-major), one elected thread issues
// tcgen05.mma (M=128, N=256, fp32 accumulate in TMEM), and after the last k-block the
// four warps read their rows back with tcgen05.ld and reduce the 256 logits to the
// unmask partial of K3 (unmask.cu `Part`: max, sum exp(x - max), lowest argmax).
// optimus_unmask_finalize then merges the vocab tiles exactly as it merges K3's
// vocab splits, so the commit rule (commit.py:86-112 replaced by the confidence
// threshold) is unchanged.
//
// The logits traffic K3 removes: rows x V x 2 bytes written by the GEMM and read
// by K3 (340 MB at 1,121 rows x 151,936 for SDAR-8B).  What remains is the weight
// stream (V x K x 2 = 1.24 GB) and the tensor-core work.
#include "ptx.cuh"

#include <cudaTypedefs.h>

namespace optimus {

constexpr int kLmM = 128;      // rows per tile (TMEM lanes)
constexpr int kLmN = 256;      // vocab columns per tile (TMEM columns per accumulator)
constexpr int kLmK = 64;       // k per stage: one 128-byte swizzle row
constexpr int kLmStages = 4;
constexpr int kLmABytes = kLmM * kLmK * 2;
constexpr int kLmBBytes = kLmN * kLmK * 2;
constexpr int kLmThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kLmSmem = kLmStages * (kLmABytes + kLmBBytes) + 1024 /*align*/ + 256 /*barriers*/;

struct LmPart {
  float m;
  float s;
  int idx;
};

// Persistent: one CTA per SM walks the (row tile, vocab tile) grid with stride
// gridDim.x (row tiles fastest, so CTAs running together share W tiles in L2).  Two
// TMEM accumulators (2 x 256 columns): the epilogue warps reduce tile i while the
// MMA warp accumulates tile i + 1.
__global__ void __launch_bounds__(kLmThreads, 1) lmhead_unmask_kernel(const __grid_constant__ CUtensorMap tm_h,
                                                                      const __grid_constant__ CUtensorMap tm_w,
                                                                      int n_rows, int vocab, int k_dim,
                                                                      int vocab_offset, int n_rt, int n_vt,
                                                                      LmPart* __restrict__ part) {
  extern __shared__ uint8_t lm_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lm_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kLmStages * kLmABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kLmStages * kLmBBytes);
  uint64_t* empty = full + kLmStages;
  uint64_t* acc_full = empty + kLmStages;   // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;       // [2] epilogue -> MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (k_dim + kLmK - 1) / kLmK;
  const int n_tiles = n_rt * n_vt;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kLmStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    mbar_fence_init();
    prefetch_tmap(&tm_h);
    prefetch_tmap(&tm_w);
  }
  if (warp == 0) tmem_alloc<2 * kLmN>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---- TMA producer: one continuous stage stream over this CTA's tiles
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int rt = t % n_rt, vt = t / n_rt;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int st = it % kLmStages;
        mbar_wait(&empty[st], ((it / kLmStages) & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[st], kLmABytes + kLmBBytes);
          tma_load_4d(sA + st * kLmABytes, &tm_h, &full[st], kb * kLmK, rt * kLmM, 0, 0);
          tma_load_4d(sB + st * kLmBBytes, &tm_w, &full[st], kb * kLmK, vt * kLmN, 0, 0);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: 4 k-steps of 16 per stage (+32 bytes inside the swizzle row)
    constexpr uint32_t idesc = umma_idesc_bf16(kLmM, kLmN, false, false);
    const uint32_t sA_a = smem_u32(sA), sB_a = smem_u32(sB);
    int it = 0, i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int buf = i & 1;
      mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);  // the epilogue drained this accumulator
      tc_fence_after();
      const uint32_t d = tmem + buf * kLmN;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int st = it % kLmStages;
        mbar_wait(&full[st], (it / kLmStages) & 1);
        tc_fence_after();
        const uint64_t ad = umma_sdesc_sw128(sA_a + st * kLmABytes, 16, 1024);
        const uint64_t bd = umma_sdesc_sw128(sB_a + st * kLmBBytes, 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kLmK / 16; ++ks)
            umma_bf16_ss(d, ad + ((ks * 32) >> 4), bd + ((ks * 32) >> 4), idesc, (kb | ks) ? 1u : 0u);
          umma_commit(&empty[st]);
          if (kb == nk - 1) umma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue (warps 2-5; TMEM lane quarter = warp % 4): thread = row; online
    // (max, sum exp, argmax) over the tile's 256 columns, vocabulary tail masked
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    constexpr float kLog2e = 1.4426950408889634f;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int rt = t % n_rt, vt = t / n_rt;
      const int buf = i & 1;
      mbar_wait(&acc_full[buf], (i >> 1) & 1);
      tc_fence_after();
      const int row = rt * kLmM + q * 32 + lane;
      const int v0 = vt * kLmN;
      const int n_valid = min(kLmN, vocab - v0);
      float m = -INFINITY, s = 0.f;
      int idx = 0x7FFFFFFF;
#pragma unroll 1
      for (int c0 = 0; c0 < kLmN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + buf * kLmN + lane_off + c0, r);
        tmem_wait_ld();
        if (c0 >= n_valid) continue;
        const int nv = min(32, n_valid - c0);
        float cm = -INFINITY;
        int ci = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x = __uint_as_float(r[c]);
          if (c < nv && x > cm) {  // ascending columns: first maximum
            cm = x;
            ci = c;
          }
        }
        if (cm > m) {
          s = (m == -INFINITY) ? 0.f : s * fast_exp2((m - cm) * kLog2e);
          m = cm;
          idx = v0 + c0 + ci;
        }
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nv) acc += fast_exp2((__uint_as_float(r[c]) - m) * kLog2e);
        s += acc;
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (row < n_rows) part[static_cast<int64_t>(row) * n_vt + vt] = LmPart{m, s, idx + vocab_offset};
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<2 * kLmN>(tmem);
}

// Merge each row's n_split partials into one record (one warp per row: every lane
// folds splits lane, lane + 32, ... in order, then a fixed xor-tree across lanes), so
// the finalize step sees n_vsplit = 1 instead of hundreds of vocab tiles.
__device__ __forceinline__ void lm_merge(float& m, float& s, int& idx, float m2, float s2, int i2) {
  constexpr float kLog2e = 1.4426950408889634f;
  if (i2 < 0) return;
  if (idx < 0 || m2 > m || (m2 == m && i2 < idx)) {
    s = (idx < 0 || m == -INFINITY) ? s2 : s * fast_exp2((m - m2) * kLog2e) + s2;
    m = m2;
    idx = i2;
  } else {
    s += (m2 == -INFINITY) ? 0.f : s2 * fast_exp2((m2 - m) * kLog2e);
  }
}

__global__ void __launch_bounds__(256) merge_splits_kernel(const LmPart* __restrict__ part, int n_rows,
                                                           int n_split, LmPart* __restrict__ out) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  float m = -INFINITY, s = 0.f;
  int idx = -1;
  const LmPart* pr = part + static_cast<int64_t>(row) * n_split;
  for (int k = lane; k < n_split; k += 32) {
    const LmPart q = pr[k];
    lm_merge(m, s, idx, q.m, q.s, q.idx);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float m2 = __shfl_xor_sync(0xFFFFFFFFu, m, o);
    const float s2 = __shfl_xor_sync(0xFFFFFFFFu, s, o);
    const int i2 = __shfl_xor_sync(0xFFFFFFFFu, idx, o);
    lm_merge(m, s, idx, m2, s2, i2);
  }
  if (lane == 0) out[row] = LmPart{m, s, idx};
}

int launch_merge_splits(const float* part, int n_rows, int n_split, float* out, cudaStream_t stream) {
  if (n_rows <= 0) return 0;
  merge_splits_kernel<<<(n_rows * 32 + 255) / 256, 256, 0, stream>>>(
      reinterpret_cast<const LmPart*>(part), n_rows, n_split, reinterpret_cast<LmPart*>(out));
  return static_cast<int>(cudaGetLastError());
}

int lmhead_unmask_smem() { return kLmSmem; }

int launch_lmhead_unmask(const CUtensorMap& tm_h, const CUtensorMap& tm_w, int n_rows, int vocab, int k_dim,
                         int vocab_offset, float* part, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(lmhead_unmask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLmSmem);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  const int n_rt = (n_rows + kLmM - 1) / kLmM, n_vt = (vocab + kLmN - 1) / kLmN;
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = n_rt * n_vt < n_sm ? n_rt * n_vt : n_sm;
  lmhead_unmask_kernel<<<grid, kLmThreads, kLmSmem, stream>>>(tm_h, tm_w, n_rows, vocab, k_dim, vocab_offset,
                                                               n_rt, n_vt, reinterpret_cast<LmPart*>(part));
  return static_cast<int>(cudaGetLastError());
}

}  // namespace optimus
