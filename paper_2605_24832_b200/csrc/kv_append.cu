// K1 — KV append: scatter each step's new K/V rows into the paged cache.
//
// Replaces the KV write that the reference charges through
// `cost_model.latency(total_computed)` (pkg/src/dllmsim/sim.py:293) and that
// the paper describes as "maps per-chunk KV states into the paged KV cache"
// (PAPER.md:9).  Slot rule (SURVEY §8c rule S): absolute position
// s = prompt_len[r] + p, slot = block_table[r][s / P] * P + s % P.
//
// Every token of the plan is appended (rule K): kv_positions produce final KV,
// window rows produce provisional KV that the visibility rule of K2 hides
// until the position is recomputed with its committed token.
//
// Pure streaming: one warp per token; each lane moves 16-byte vectors, so a
// token's Hkv*head_dim*2 bytes of K (and of V) are read and written once.
#include "ptx.cuh"

namespace optimus {

__global__ void __launch_bounds__(256) kv_append_kernel(
    const uint4* __restrict__ k_new, const uint4* __restrict__ v_new, int64_t new_stride_vec,
    const int32_t* __restrict__ tok_req, const int32_t* __restrict__ tok_pos,
    const int32_t* __restrict__ prompt_len, const int32_t* __restrict__ block_tables,
    int max_pages, int n_tok, int hkv, int vec_per_head, int page_size, uint4* __restrict__ k_cache,
    uint4* __restrict__ v_cache, int64_t* __restrict__ slot_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_tok) return;
  const int r = tok_req[warp];
  const int s = prompt_len[r] + tok_pos[warp];
  const int page = block_tables[static_cast<int64_t>(r) * max_pages + s / page_size];
  const int off = s % page_size;
  if (lane == 0 && slot_out != nullptr)
    slot_out[warp] = static_cast<int64_t>(page) * page_size + off;
  const int total = hkv * vec_per_head;
  const uint4* ksrc = k_new + static_cast<int64_t>(warp) * new_stride_vec;
  const uint4* vsrc = v_new + static_cast<int64_t>(warp) * new_stride_vec;
  // (page, head, off) row base in 16-byte vectors.
  const int64_t page_base = static_cast<int64_t>(page) * hkv * page_size;
#pragma unroll 4
  for (int i = lane; i < total; i += 32) {
    const int h = i / vec_per_head;
    const int c = i - h * vec_per_head;
    const int64_t dst = ((page_base + static_cast<int64_t>(h) * page_size + off) * vec_per_head) + c;
    const uint4 kv = __ldg(ksrc + i);
    const uint4 vv = __ldg(vsrc + i);
    k_cache[dst] = kv;
    v_cache[dst] = vv;
  }
}

int launch_kv_append(const void* k_new, const void* v_new, int64_t new_stride_tok,
                     const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                     const int32_t* block_tables, int max_pages, int n_tok, int hkv, int head_dim,
                     int page_size, void* k_cache, void* v_cache, int64_t* slot_out,
                     cudaStream_t stream) {
  if (n_tok == 0) return 0;
  const int vec_per_head = head_dim / 8;  // 8 bf16 per 16-byte vector
  const int threads = 256;
  const int blocks = (n_tok * 32 + threads - 1) / threads;
  kv_append_kernel<<<blocks, threads, 0, stream>>>(
      static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), new_stride_tok / 8,
      tok_req, tok_pos, prompt_len, block_tables, max_pages, n_tok, hkv, vec_per_head, page_size,
      static_cast<uint4*>(k_cache), static_cast<uint4*>(v_cache), slot_out);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace optimus
