// K2 — variable-length paged attention for streaming chunked block decoding.
//
// What it computes (SURVEY §8c rule V): every query token of
// request r (its kv-recompute rows and its MASK window rows, ChunkPlan order,
// engine.py:28-37,67) attends to the keys it may see — the whole prompt, every
// output position that is DECODED_CACHED or recomputed in this step, block-causal
// (bidirectional inside a block, nothing from later blocks).  The visible set
// arrives as a per-request bitmap anchored at vis_base plus a per-query limit.
//
// How (sm_100a, one persistent CTA per SM, warp-specialised):
//   warp 0   TMA producer: per work item, one Q tile (all G heads of a KV head
//            folded into 128 MMA rows, row = token*G + head) and a ring of
//            64-key K/V tiles gathered page by page through the block table
//            (4-D tensor maps, SWIZZLE_128B boxes of 64 columns).
//   warp 1   MMA issuer (one thread): S = Q K^T into TMEM (double buffered),
//            O += P V into TMEM (double buffered across work items).
//   warp 2   TMEM allocator.
//   warps 4-7  softmax + epilogue: thread i owns query row i (= TMEM lane i), so
//            the row max/sum need no shuffles; online softmax in the exp2 domain
//            with a lazy rescale (O in TMEM is only rescaled when the running max
//            grows by more than 2^8); P goes to shared memory as the A operand of
//            the PV MMA, split into two bf16 planes P = hi + lo so the PV product
//            carries ~16 mantissa bits of P (the tensor pipe has the headroom:
//            this kernel is HBM-bound).  Epilogue normalises O and stores bf16,
//            or writes fp32 split-KV partials for the combine kernel.
// Work items are planned on the host (optimus_attn_plan): long contexts are split
// into key ranges and items are distributed longest-first over the CTAs.
#include "attn.cuh"

namespace optimus {

constexpr int kTileN = 64;     // keys per pipeline stage
constexpr int kBlockM = 128;   // MMA rows (query token x head-in-group)
constexpr int kThreads = 256;  // 8 warps
constexpr int kTraceSlots = 512;  // per CTA: [role*128 + i]

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(const AttnParams& p, int role, int i) {
  if (p.trace != nullptr && i < 128)
    p.trace[static_cast<int64_t>(blockIdx.x) * kTraceSlots + role * 128 + i] = gtimer();
}



template <int HD, int STAGES>
struct AttnSmem {
  static constexpr int KB = HD / 64;
  static constexpr uint32_t Q_BYTES = KB * kBlockM * 128;
  static constexpr uint32_t KT_BYTES = KB * kTileN * 128;
  static constexpr uint32_t P_HALF = kBlockM * 128;       // one bf16 [128][64] plane
  static constexpr uint32_t P_BYTES = 2 * P_HALF;          // hi + lo planes
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * KT_BYTES;
  static constexpr uint32_t OFF_P = OFF_V + STAGES * KT_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 2 * 7;
  static constexpr uint32_t BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr uint32_t ALLOC = BYTES + 1024;  // slack for 1024-byte alignment
  static constexpr uint32_t TMEM_COLS = (128 + 2 * HD) <= 256 ? 256 : 512;
};

template <int HD, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    paged_attn_kernel(const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using L = AttnSmem<HD, STAGES>;
  constexpr int KB = L::KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = kv_full + STAGES;
  uint64_t* q_full = kv_empty + STAGES;
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_empty + 2;
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 2;
  uint64_t* o_full = pv_done + 2;
  uint64_t* o_empty = o_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace(p, 3, 127);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  // Zero the operand buffers once: rows a partial tile never loads must hold finite
  // values (their probabilities are 0, and 0 * NaN would poison O).
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (uint32_t i = threadIdx.x; i < L::OFF_BAR / 16; i += kThreads) z[i] = zero;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace(p, 3, 126);
  const uint32_t tm_s0 = tmem_base;           // S buffers: columns [0,64) and [64,128)
  const uint32_t tm_o0 = tmem_base + 128;     // O buffers: [128,128+HD) and [128+HD,128+2HD)

  const int w_begin = p.cta_off[blockIdx.x];
  const int w_end = p.cta_off[blockIdx.x + 1];

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t q_tx = KB * 64 * p.group * p.tok_per_tile * 2;
      const uint32_t chunk_tx = p.box_rows * 128 * KB * 2;  // K + V for one box row group
      const int chunks_per_tile = kTileN / p.box_rows;
      int tile_ctr = 0;
      int unit = 0;
      for (int w = w_begin; w < w_end; ++w, ++unit) {
        const int* wk = p.work + 8 * w;
        const int req = wk[0], head = wk[1], tok_begin = wk[2];
        const int key_begin = wk[4], key_end = wk[5];
        const int qb = unit & 1;
        mbar_wait(&q_empty[qb], ((unit >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], q_tx);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_4d(sQ + qb * L::Q_BYTES + kb * (kBlockM * 128), &tm_q, &q_full[qb], kb * 64, 0,
                      head, tok_begin);
        const int32_t* bt = p.block_tables + static_cast<int64_t>(req) * p.max_pages;
        for (int kt = key_begin; kt < key_end; kt += kTileN, ++tile_ctr) {
          const int st = tile_ctr % STAGES;
          mbar_wait(&kv_empty[st], ((tile_ctr / STAGES) & 1) ^ 1);
          trace(p, 0, tile_ctr);
          int n_chunks = (min(kTileN, key_end - kt) + p.box_rows - 1) / p.box_rows;
          if (n_chunks > chunks_per_tile) n_chunks = chunks_per_tile;
          mbar_arrive_expect_tx(&kv_full[st], n_chunks * chunk_tx);
          for (int c = 0; c < n_chunks; ++c) {
            const int s0 = kt + c * p.box_rows;
            const int page = bt[s0 / p.page_size];
            const int row0 = s0 % p.page_size;
            for (int kb = 0; kb < KB; ++kb) {
              const uint32_t off = st * L::KT_BYTES + kb * (kTileN * 128) + c * p.box_rows * 128;
              tma_load_4d(sK + off, &tm_k, &kv_full[st], kb * 64, row0, head, page);
              tma_load_4d(sV + off, &tm_v, &kv_full[st], kb * 64, row0, head, page);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(kBlockM, kTileN, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kBlockM, HD, false, true);
      const uint32_t sQ_a = smem_u32(sQ), sK_a = smem_u32(sK), sV_a = smem_u32(sV),
                     sP_a = smem_u32(sP);
      int tile_ctr = 0;
      int unit = 0;
      for (int w = w_begin; w < w_end; ++w, ++unit) {
        const int* wk = p.work + 8 * w;
        const int n_tiles = (wk[5] - wk[4] + kTileN - 1) / kTileN;
        const int qb = unit & 1;
        const int ob = unit & 1;
        mbar_wait(&q_full[qb], (unit >> 1) & 1);
        tc_fence_after();
        auto issue_s = [&](int t) {
          const int st = t % STAGES;
          mbar_wait(&kv_full[st], (t / STAGES) & 1);
          tc_fence_after();
          trace(p, 1, t);
          const uint32_t d = tm_s0 + (t & 1) * kTileN;
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const int kb = ks >> 2;
            const uint32_t koff = (ks & 3) * 32;
            const uint64_t a = umma_sdesc_sw128(
                sQ_a + qb * L::Q_BYTES + kb * (kBlockM * 128) + koff, 16, 1024);
            const uint64_t b = umma_sdesc_sw128(
                sK_a + st * L::KT_BYTES + kb * (kTileN * 128) + koff, 16, 1024);
            umma_bf16_ss(d, a, b, idesc_s, ks > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[t & 1]);
        };
        issue_s(tile_ctr);
        mbar_wait(&o_empty[ob], ((unit >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int j = 0; j < n_tiles; ++j) {
          const int t = tile_ctr + j;
          if (j + 1 < n_tiles) issue_s(t + 1);
          mbar_wait(&p_full[t & 1], (t >> 1) & 1);
          tc_fence_after();
          const int st = t % STAGES;
          const uint32_t d = tm_o0 + ob * HD;
#pragma unroll
          for (int ks = 0; ks < kTileN / 16; ++ks) {
            const uint32_t pa = sP_a + (t & 1) * L::P_BYTES + ks * 32;
            const uint64_t b =
                umma_sdesc_sw128(sV_a + st * L::KT_BYTES + ks * 16 * 128, kTileN * 128, 1024);
            umma_bf16_ss(d, umma_sdesc_sw128(pa, 16, 1024), b, idesc_o, (j > 0 || ks > 0) ? 1u : 0u);
            umma_bf16_ss(d, umma_sdesc_sw128(pa + L::P_HALF, 16, 1024), b, idesc_o, 1u);
          }
          umma_commit(&pv_done[t & 1]);
          umma_commit(&kv_empty[st]);
        }
        umma_commit(&q_empty[qb]);
        umma_commit(&o_full[ob]);
        tile_ctr += n_tiles;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int row = threadIdx.x - 128;          // query row == TMEM lane
    const int wq = warp - 4;                    // TMEM lane quarter
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const int G = p.group;
    const int t_in = row / G;
    const int g_in = row - t_in * G;
    const bool row_exists = t_in < p.tok_per_tile;
    const uint32_t p_row_addr = smem_u32(sP) + row * 128;
    const int sw = row & 7;
    int tile_ctr = 0;
    int unit = 0;
    for (int w = w_begin; w < w_end; ++w, ++unit) {
      const int* wk = p.work + 8 * w;
      const int req = wk[0], head = wk[1], tok_begin = wk[2], n_tok = wk[3];
      const int key_begin = wk[4], key_end = wk[5], slot = wk[6];
      const int n_tiles = (key_end - key_begin + kTileN - 1) / kTileN;
      const int ob = unit & 1;
      const bool valid = row_exists && t_in < n_tok;
      const bool warp_valid = (wq * 32) / G < n_tok;  // first row of this warp is a real token
      const int prompt = p.prompt_len[req];
      const int vb = p.vis_base[req];
      const uint32_t* words = p.vis_words + p.vis_off[req];
      int lim = 0;
      if (valid) {
        const int qp = p.q_pos[tok_begin + t_in];
        lim = prompt + (qp / p.block_size + 1) * p.block_size;
        if (lim > key_end) lim = key_end;
      }
      float m = -INFINITY;
      float l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int t = tile_ctr + j;
        const int sb = t & 1;
        mbar_wait(&s_full[sb], (t >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 128) trace(p, 2, t);
        if (warp_valid) {
          uint32_t sr[2][32];
          tmem_ld32(tm_s0 + lane_off + sb * kTileN, sr[0]);
          tmem_ld32(tm_s0 + lane_off + sb * kTileN + 32, sr[1]);
          tmem_wait_ld();
          const int kt = key_begin + j * kTileN;
          // visibility of the 64 keys of this tile for this row
          uint64_t vis = ~0ull;
          if (kt + kTileN > lim || kt + kTileN > vb) {
            uint32_t lo = 0xFFFFFFFFu, hi = 0xFFFFFFFFu;
            if (kt + 32 > vb && kt < lim) lo = words[(kt - vb) >> 5];
            if (kt + 64 > vb && kt + 32 < lim) hi = words[(kt + 32 - vb) >> 5];
            vis = (static_cast<uint64_t>(hi) << 32) | lo;
            const int n = lim - kt;
            const uint64_t lm = n >= 64 ? ~0ull : (n <= 0 ? 0ull : ((1ull << n) - 1));
            vis &= lm;
          }
          float x[64];
          float tmax = -INFINITY;
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const float s = __uint_as_float(sr[c >> 5][c & 31]) * p.scale_log2;
            x[c] = ((vis >> c) & 1ull) ? s : -INFINITY;
            tmax = fmaxf(tmax, x[c]);
          }
          const bool need = tmax > m + 8.0f;
          const float m_new = need ? tmax : m;
          if (j > 0 && __any_sync(0xFFFFFFFFu, need)) {
            // O holds sum_{u<t} P_u V_u once PV_{t-1} retires; rescale it in TMEM.
            mbar_wait(&pv_done[(t - 1) & 1], ((t - 1) >> 1) & 1);
            tc_fence_after();
            const float alpha = need ? fast_exp2(m - m_new) : 1.0f;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
              uint32_t o[32];
              const uint32_t ta = tm_o0 + lane_off + ob * HD + c0;
              tmem_ld32(ta, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              tmem_st32(ta, o);
            }
            tmem_wait_st();
          }
          if (need) {
            l = (m == -INFINITY) ? 0.f : l * fast_exp2(m - m_new);
            m = m_new;
          }
          const float m_use = (m == -INFINITY) ? 0.f : m;
          // P buffer sb was last read by PV_{t-2}.
          if (t >= 2) mbar_wait(&pv_done[sb], ((t - 2) >> 1) & 1);
          float rs = 0.f;
          const uint32_t pbase = p_row_addr + sb * L::P_BYTES;
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            float e[8];
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              e[k] = fast_exp2(x[c8 * 8 + k] - m_use);
              rs += e[k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              hi[k] = pack_bf16x2(e[2 * k], e[2 * k + 1]);
              lo[k] = pack_bf16x2(e[2 * k] - __uint_as_float(hi[k] << 16),
                                  e[2 * k + 1] - __uint_as_float(hi[k] & 0xFFFF0000u));
            }
            const uint32_t cofs = (c8 ^ sw) << 4;
            st_shared_v4(pbase + cofs, hi[0], hi[1], hi[2], hi[3]);
            st_shared_v4(pbase + L::P_HALF + cofs, lo[0], lo[1], lo[2], lo[3]);
          }
          l += rs;
          fence_proxy_async_smem();
        }
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        if (threadIdx.x == 128) trace(p, 3, t);
      }
      tile_ctr += n_tiles;
      // ---------------------------------------------------------- epilogue
      mbar_wait(&o_full[ob], (unit >> 1) & 1);
      tc_fence_after();
      if (warp_valid) {
        const float inv_l = (l > 0.f) ? 1.0f / l : 0.f;
        const int tok = tok_begin + t_in;
        const int qh = head * G + g_in;
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(tm_o0 + lane_off + ob * HD + c0, o);
          tmem_wait_ld();
          if (valid) {
            if (slot < 0) {
              uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<int64_t>(tok) * p.out_stride_tok +
                                                    static_cast<int64_t>(qh) * HD + c0);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const int c = v * 8;
                dst[v] = make_uint4(
                    pack_bf16x2(__uint_as_float(o[c + 0]) * inv_l, __uint_as_float(o[c + 1]) * inv_l),
                    pack_bf16x2(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l),
                    pack_bf16x2(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l),
                    pack_bf16x2(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l));
              }
            } else {
              float4* dst = reinterpret_cast<float4*>(
                  p.ws_o + (static_cast<int64_t>(slot) * kBlockM + row) * HD + c0);
#pragma unroll
              for (int v = 0; v < 8; ++v)
                dst[v] = make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]),
                                     __uint_as_float(o[4 * v + 2]), __uint_as_float(o[4 * v + 3]));
            }
          }
        }
        if (valid && slot >= 0) {
          reinterpret_cast<float2*>(p.ws_ml)[static_cast<int64_t>(slot) * kBlockM + row] =
              make_float2(m, l);
        }
      }
      tc_fence_before();
      mbar_arrive(&o_empty[ob]);
    }
  }
  if (threadIdx.x == 0) trace(p, 2, 127);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<L::TMEM_COLS>(tmem_base);
  if (threadIdx.x == 64) trace(p, 2, 126);
}

// Split-KV combine: merge the (m, l, O) partials of every split query tile.
// One warp per output row (grid.x = group, grid.y = 8-row slab): lane s reads the
// (m, l) of split s, the warp reduces the merged max / denominator with shuffles,
// then every lane accumulates a 4-column float4 slice over the splits.
template <int HD>
__global__ void __launch_bounds__(256) attn_combine_kernel(const int32_t* __restrict__ groups,
                                                           const float* __restrict__ ws_o,
                                                           const float* __restrict__ ws_ml,
                                                           __nv_bfloat16* __restrict__ out,
                                                           int64_t out_stride_tok, int group_sz) {
  const int* gr = groups + 8 * blockIdx.x;
  const int head = gr[1], tok_begin = gr[2], n_tok = gr[3], slot0 = gr[4], n_split = gr[5];
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n_tok * group_sz) return;
  const float2* ml = reinterpret_cast<const float2*>(ws_ml);
  float mx = -INFINITY;
  for (int s = lane; s < n_split; s += 32) {
    const float2 v = ml[static_cast<int64_t>(slot0 + s) * kBlockM + r];
    if (v.y > 0.f) mx = fmaxf(mx, v.x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  float den = 0.f;
  for (int s = lane; s < n_split; s += 32) {
    const float2 v = ml[static_cast<int64_t>(slot0 + s) * kBlockM + r];
    if (v.y > 0.f) den += exp2f(v.x - mx) * v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xFFFFFFFFu, den, o);
  constexpr int PER = HD / 32;  // columns per lane (4 for HD=128, 2 for HD=64)
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  for (int s = 0; s < n_split; ++s) {
    const float2 v = ml[static_cast<int64_t>(slot0 + s) * kBlockM + r];
    if (!(v.y > 0.f)) continue;
    const float wgt = exp2f(v.x - mx);
    const float* src = ws_o + (static_cast<int64_t>(slot0 + s) * kBlockM + r) * HD + lane * PER;
    if constexpr (PER == 4) {
      const float4 o = *reinterpret_cast<const float4*>(src);
      acc[0] += wgt * o.x; acc[1] += wgt * o.y; acc[2] += wgt * o.z; acc[3] += wgt * o.w;
    } else {
      const float2 o = *reinterpret_cast<const float2*>(src);
      acc[0] += wgt * o.x; acc[1] += wgt * o.y;
    }
  }
  const float inv = den > 0.f ? 1.f / den : 0.f;
  const int t = r / group_sz, g = r - t * group_sz;
  __nv_bfloat16* dst = out + static_cast<int64_t>(tok_begin + t) * out_stride_tok +
                       static_cast<int64_t>(head * group_sz + g) * HD + lane * PER;
  if constexpr (PER == 4) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(acc[0] * inv, acc[1] * inv),
                                                pack_bf16x2(acc[2] * inv, acc[3] * inv));
  } else {
    *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(acc[0] * inv, acc[1] * inv);
  }
}

template <int HD, int STAGES>
static int launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const AttnParams& prm, int grid, const int32_t* groups, int n_groups,
                         cudaStream_t stream) {
  using L = AttnSmem<HD, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(paged_attn_kernel<HD, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  if (grid > 0) {
    paged_attn_kernel<HD, STAGES><<<grid, kThreads, L::ALLOC, stream>>>(tq, tk, tv, prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  if (n_groups > 0) {
    attn_combine_kernel<HD><<<dim3(n_groups, kBlockM / 8), 256, 0, stream>>>(
        groups, prm.ws_o, prm.ws_ml, prm.out, prm.out_stride_tok, prm.group);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

int launch_paged_attn(int head_dim, const CUtensorMap& tq, const CUtensorMap& tk,
                      const CUtensorMap& tv, const AttnParams& prm, int grid,
                      const int32_t* groups, int n_groups, cudaStream_t stream) {
  if (head_dim == 128) return launch_attn_t<128, 3>(tq, tk, tv, prm, grid, groups, n_groups, stream);
  if (head_dim == 64) return launch_attn_t<64, 4>(tq, tk, tv, prm, grid, groups, n_groups, stream);
  return -1;
}

}  // namespace optimus
