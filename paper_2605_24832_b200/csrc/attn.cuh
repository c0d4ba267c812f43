// attn.cuh — parameter block shared by the K2 kernel (paged_attn.cu) and the
// C-ABI launcher (capi.cu).
#pragma once
#include "ptx.cuh"

namespace optimus {

struct AttnParams {
  const int32_t* q_pos;
  const int32_t* prompt_len;
  const int32_t* vis_base;
  const int32_t* vis_off;
  const uint32_t* vis_words;
  const int32_t* block_tables;
  const int32_t* work;     // [n][8]
  const int32_t* cta_off;  // [grid+1]
  __nv_bfloat16* out;
  int64_t out_stride_tok;
  float* ws_o;
  float* ws_ml;
  int max_pages;
  int block_size;
  int num_q_heads;
  int group;       // G = Hq / Hkv
  int tok_per_tile;  // 128 / G
  int page_size;
  int page_shift;  // log2(page_size)
  int box_rows;    // min(page_size, 64)
  float scale_log2;
  // fused KV append (K1 folded into K2): the new K/V rows of every query token are
  // scattered into the pages by the CTA whose work item covers their position
  // (valid when each (request, KV head) is a single query tile); nullptr = off
  const void* k_new;
  const void* v_new;
  int64_t new_stride_tok;  // elements between tokens in k_new / v_new
  int64_t* slot_out;       // optional slot mapping output (rule S)
  const int32_t* slot_abs; // optional per-step {abs pos, slot} per token (else computed)
  void* k_cache_w;         // the caches the append writes (the K2 inputs k_cache / v_cache)
  void* v_cache_w;
  int num_kv_heads;
  int v_fp16;              // V cache is fp16: convert on the way
  unsigned long long* trace;
  int dbg;  // diagnostics: bit0 skip lo-plane PV, bit1 skip S MMA, bit2 skip softmax math, bit3 skip PV  // optional per-CTA timeline (diagnostics), nullptr in production
};

int launch_attn_combine_dev(int head_dim, const AttnParams& prm, const int32_t* groups, int max_groups,
                            const int32_t* n_groups_dev, cudaStream_t stream);
int launch_paged_attn(int head_dim, bool v_fp16, const CUtensorMap& tq, const CUtensorMap& tk,
                      const CUtensorMap& tv, const AttnParams& prm, int grid,
                      const int32_t* groups, int n_groups, cudaStream_t stream);

}  // namespace optimus
