/*
 * optimus_b200.h — C-ABI of the B200 (sm_100a) streaming chunked block-decode path.
 *
 * The reference (arxiv 2605.24832, package `dllmsim`) has no native code: its
 * decode step is the Python call chain
 *     _Loop.run_decode (pkg/src/dllmsim/sim.py:269-305)
 *       -> plan_chunk (engine.py:45-67)
 *       -> oracle.commits(request, window) (sim.py:278; commit.py:279-280)
 *       -> apply_chunk (engine.py:79-95)
 * and the model forward it stands in for (KV append into pages, varlen paged
 * attention, confidence-threshold unmask) is specified in
 * prose only.  Each entry point below is the native replacement for one piece of
 * that forward; the Python host layer (paper_2605_24832_b200/) binds them with
 * ctypes the same way a reference-side binding would.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless its name ends in `_host`;
 *  - tensors are bf16 ("uint16_t" storage) unless stated; strides are in elements;
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *  - return value: 0 on success, OPTIMUS_EINVAL (-1) for a bad argument / shape,
 *    OPTIMUS_ENOSYS (-2) when the device is not sm_100, or a positive cudaError_t;
 *  - the library never allocates device memory: workspaces are caller-owned.
 *
 * KV cache layout (per layer, one allocation for K and one for V):
 *     cache[num_pages][Hkv][page_size][head_dim]   bf16
 * so each (page, head) is a contiguous page_size x head_dim tile that the
 * attention kernel stages with TMA (SWIZZLE_128B boxes of 64 columns).
 * Absolute sequence position of output position p of request r is
 * prompt_len[r] + p; its slot is block_table[r][s / P] * P + s % P
 * (SURVEY.md §8c rule S).
 */
#ifndef OPTIMUS_B200_H
#define OPTIMUS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPTIMUS_EINVAL (-1)
#define OPTIMUS_ENOSYS (-2)

/* Attention work item / combine group records (8 x int32 each). */
#define OPTIMUS_WORK_INTS 8

/* Library version, e.g. 100 for 0.1.0. */
int optimus_version(void);

/* Human-readable description of the last error raised on this thread. */
const char* optimus_last_error(void);

/* Diagnostics: record a per-CTA globaltimer timeline of K2 into `buf`
 * (device, uint64[grid][512]); NULL disables (the default). */
void optimus_set_attn_trace(unsigned long long* buf);

/* Number of SMs of the current device (0 if no device). */
int optimus_device_sm_count(void);

/*
 * K1 — KV append (replaces the KV write of the forward that the reference models
 * with `cost_model.latency`, sim.py:293; rule S/K of SURVEY §8c).
 *
 * For token i (0 <= i < n_tok) of request tok_req[i] at output position
 * tok_pos[i]:  s = prompt_len[req] + tok_pos[i],
 *              slot = block_tables[req * max_pages + s / page_size] * page_size + s % page_size,
 * and K/V rows k_new[i*new_stride + h*head_dim + :] are written to
 * k_cache[((page*Hkv + h)*page_size + off)*head_dim + :] for every head h.
 * slot_mapping_out (optional, int64[n_tok]) receives the slots.
 * v_dtype: 0 = the V cache is bf16 (copied), 1 = fp16 (bf16 rows converted, exact for
 * |v| < 65504, saturating beyond).  K is always bf16.
 */
int optimus_kv_append(const void* k_new, const void* v_new, int64_t new_stride_tok,
                      const int32_t* tok_req, const int32_t* tok_pos,
                      const int32_t* prompt_len, const int32_t* block_tables,
                      int max_pages, int n_tok, int num_kv_heads, int head_dim,
                      int page_size, void* k_cache, void* v_cache, int64_t num_pages,
                      int64_t* slot_mapping_out, int v_dtype, void* stream);

/*
 * Host-side work planner for K2 (the length-aware persistent tile scheduler).
 * Inputs are HOST arrays describing the step:
 *   cu_seqlens_q_host[n_req+1]  query tokens of each request (kv rows then window rows)
 *   key_end_host[n_req]         absolute end of the keys any query of the request may see
 * It splits every (request, kv head, 128-row query tile) into key ranges of whole
 * 64-key tiles, assigns them to `grid` persistent CTAs by longest-processing-time
 * first, and writes:
 *   work_host[max_work][8]      {req, kv_head, tok_begin, n_tok, key_begin, key_end, partial_slot, 0}
 *                               ordered CTA by CTA
 *   cta_off_host[grid+1]        CSR offsets of each CTA's items in work_host
 *   groups_host[max_groups][8]  {req, kv_head, tok_begin, n_tok, slot0, n_splits, 0, 0}
 *                               (query tiles that were split and need the combine)
 * Returns the number of work items (>= 0) or OPTIMUS_EINVAL; *n_groups and
 * *n_partials receive the combine-group count and the partial-slot count.
 * `min_split_tiles` bounds how finely a long context is split (64-key tiles);
 * an item never spans more than 255 pages of `page_size` keys.
 */
int optimus_attn_plan(int n_req, const int32_t* cu_seqlens_q_host, const int32_t* key_end_host,
                      int num_q_heads, int num_kv_heads, int grid, int min_split_tiles,
                      int page_size, int32_t* work_host, int max_work, int32_t* cta_off_host,
                      int32_t* groups_host, int max_groups, int* n_groups, int* n_partials);

/* Upper bounds for the planner's output buffers. */
int optimus_attn_plan_bounds(int n_req, const int32_t* cu_seqlens_q_host,
                             const int32_t* key_end_host, int num_q_heads, int num_kv_heads,
                             int min_split_tiles, int page_size, int* max_work, int* max_groups);

/*
 * K2 — variable-length paged attention with the diffusion visibility rule
 * (SURVEY §8c rule V).  Query token i belongs to request r (via the work items);
 * q_pos[i] is its output position.  Key at absolute position s is visible to it iff
 *     s < prompt_len[r] + (q_pos[i] / block_size + 1) * block_size   (block-causal)
 * and (s < vis_base[r] or bit (s - vis_base[r]) of vis_words[vis_off[r]...] is set)
 * and s < the work item's key_end.
 * q:   [n_tok][Hq][head_dim] (row stride q_stride_tok); out: same shape (out_stride_tok).
 * ws_o / ws_ml: split-KV partials, float[n_partials][128][head_dim] and
 * float[n_partials][128][2] (may be NULL when n_partials == 0).
 * work/cta_off/groups are the planner's outputs copied to the device; `grid` must
 * equal the grid used for planning.  v_dtype as for optimus_kv_append: with an fp16
 * V cache P.V runs with an fp16 P (11-bit), with a bf16 V cache P is split into two
 * bf16 planes (hi + lo) so both forms stay far inside the 2e-3 tolerance.
 */
int optimus_paged_attn(const void* q, int64_t q_stride_tok, int n_tok_total,
                       const void* k_cache, const void* v_cache, int64_t num_pages,
                       const int32_t* q_pos, const int32_t* prompt_len,
                       const int32_t* vis_base, const int32_t* vis_off, const uint32_t* vis_words,
                       const int32_t* block_tables, int max_pages,
                       const int32_t* work, const int32_t* cta_off, int grid,
                       const int32_t* groups, int n_groups,
                       int block_size, int num_q_heads, int num_kv_heads, int head_dim,
                       int page_size, float sm_scale,
                       void* out, int64_t out_stride_tok,
                       float* ws_o, float* ws_ml, int v_dtype, void* stream);

/*
 * K1 folded into K2: the same attention, with the step's new K/V rows (k_new /
 * v_new [n_tok][Hkv][head_dim] bf16, token stride new_stride_tok elements) scattered
 * into the pages by rule S inside the attention kernel (no separate append launch).
 * Requires every (request, KV head) to be a single query tile (max chunk tokens x
 * Hq/Hkv <= 128), so that the CTA covering a key position is the only reader of the
 * row it writes.  slot_mapping_out (optional, int64 [n_tok]) as optimus_kv_append.
 * slot_abs (optional): the step's optimus_slot_mapping output; without it every
 * launch re-derives positions and slots from q_pos / prompt_len / block_tables.
 */
int optimus_paged_attn_append(const void* q, int64_t q_stride_tok, int n_tok_total,
                              const void* k_new, const void* v_new, int64_t new_stride_tok,
                              void* k_cache, void* v_cache, int64_t num_pages,
                              const int32_t* q_pos, const int32_t* prompt_len,
                              const int32_t* vis_base, const int32_t* vis_off,
                              const uint32_t* vis_words, const int32_t* block_tables,
                              int max_pages, const int32_t* work, const int32_t* cta_off, int grid,
                              const int32_t* groups, int n_groups,
                              int block_size, int num_q_heads, int num_kv_heads, int head_dim,
                              int page_size, float sm_scale, void* out, int64_t out_stride_tok,
                              float* ws_o, float* ws_ml, int v_dtype, int64_t* slot_mapping_out,
                              const int32_t* slot_abs, void* stream);

/*
 * The step's slot map for the fused append, computed once per step (rule S):
 * int32 [n_tok][2]: slot_abs_out[2t] = s = prompt_len[tok_req[t]] + tok_pos[t]
 * (absolute position), slot_abs_out[2t + 1] = block_tables[r][s / P] * P + s % P.
 */
int optimus_slot_mapping(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                         const int32_t* block_tables, int max_pages, int n_tok, int page_size,
                         int32_t* slot_abs_out, void* stream);

/*
 * K1 over the step's slot map (optimus_slot_mapping output slot_abs): the same page
 * writes as optimus_kv_append with one round trip per row (the slot is read, not
 * derived through tok_req -> prompt_len -> block_tables).  Requires a power-of-two
 * page_size.
 */
int optimus_kv_append_slots(const void* k_new, const void* v_new, int64_t new_stride_tok,
                            const int32_t* slot_abs, int n_tok, int num_kv_heads, int head_dim,
                            int page_size, void* k_cache, void* v_cache, int64_t num_pages,
                            int v_dtype, void* stream);

/*
 * Executor: K1 + K2 for n_layers layers in one call (per-layer device pointers in
 * HOST arrays q[l], k_new[l], v_new[l], k_cache[l], v_cache[l], out[l]; metadata and
 * work list shared).  Enqueues everything on `stream` and returns; used when the
 * per-layer activations are already resident (no model work between the layers).
 * append_mode: 0 = optimus_kv_append + optimus_paged_attn per layer; 1 = the step's
 * optimus_slot_mapping once into slot_ws (int32 [n_tok][2], 8-byte aligned), then per
 * layer an append over that slot map + optimus_paged_attn;
 * 2 = slot map once, then one optimus_paged_attn_append launch per layer (K1 folded
 * into K2; same precondition as that call).
 */
int optimus_attn_layers(int n_layers, const void* const* q, const void* const* k_new,
                        const void* const* v_new, int64_t q_stride_tok, int64_t new_stride_tok,
                        int n_tok_total, int n_tok, void* const* k_cache, void* const* v_cache,
                        int64_t num_pages, const int32_t* tok_req, const int32_t* q_pos,
                        const int32_t* prompt_len, const int32_t* vis_base,
                        const int32_t* vis_off, const uint32_t* vis_words,
                        const int32_t* block_tables, int max_pages, const int32_t* work,
                        const int32_t* cta_off, int grid, const int32_t* groups, int n_groups,
                        int block_size, int num_q_heads, int num_kv_heads, int head_dim,
                        int page_size, float sm_scale, void* const* out, int64_t out_stride_tok,
                        float* ws_o, float* ws_ml, int v_dtype, int append_mode, int32_t* slot_ws,
                        void* stream);

/*
 * K3 — fused confidence-threshold unmask (replaces StochasticOracle.commits,
 * commit.py:279-280 -> commit_step commit.py:86-112, with the model rule
 * "commit tokens whose confidence exceeds the threshold"; tau=0.9
 * PAPER.md:49).  Two phases so the vocabulary may be sharded across ranks:
 *
 * (a) partials: for window row i (0 <= i < n_rows) read logits row
 *     (row_src ? row_src[i] : i), columns [0, vocab) of this shard, and write
 *     part[i][j] = {max, sum exp(x - max), argmax + vocab_offset} for vocab split j
 *     (n_vsplit splits; record = 3 x 32-bit: float, float, int32).
 *     logits_dtype: 0 = bf16, 1 = fp32.
 */
int optimus_unmask_partials(const void* logits, int logits_dtype, int64_t row_stride,
                            const int32_t* row_src, int n_rows, int vocab, int vocab_offset,
                            int n_vsplit, float* part, void* stream);

/*
 * (b) finalize: part is [n_outer][n_rows][n_vsplit] records (n_outer = number of
 *     vocab shards gathered, 1 on a single GPU), merged in a fixed order.
 *     conf = max softmax probability, tok = argmax (lowest index on ties).
 *     Rows of request r are cu_rows[r] .. cu_rows[r+1]-1 in window order.
 *     commit iff conf >= tau; progress rule per request:
 *       fallback_mode 0 ("earliest"): the first window row always commits
 *                       (exactly commit.py:103);
 *       fallback_mode 1 ("top1"): if no row passes, the highest-confidence row
 *                       commits (ties -> earliest);
 *       fallback_mode 2 ("none"): threshold only (a step may commit nothing,
 *                       as a ReplayOracle step can, commit.py:254-267).
 *     Optional state mirror / token update (pass NULL to skip either): for
 *     committed row i of request r at output position row_pos[i]:
 *       state[r*state_stride + pos] = 1 (DECODED_UNCACHED), token_buf[same] = tok.
 */
int optimus_unmask_finalize(const float* part, int n_outer, int n_rows, int n_vsplit,
                            const int32_t* cu_rows, int n_req, float tau, int fallback_mode,
                            uint8_t* commit_mask, int32_t* tok, float* conf,
                            const int32_t* row_pos, uint8_t* state, int32_t* token_buf,
                            int64_t state_stride, void* stream);

/*
 * Native host side of the batched step (host memory only; see csrc/host_step.cu).
 * optimus_host_plan mirrors plan_chunk (engine.py:45-67) for every slot of the batch
 * over packed per-slot state and emits the kernels' step metadata;
 * chunk_per_req (optional, [n]) gives each request its own chunk size (mixed chunks).
 * optimus_host_apply mirrors apply_chunk + advance_blocks (engine.py:79-95,
 * core.py:109-116) from the D2H commit mask.
 */
int optimus_host_plan(int n, const int32_t* slots, int chunk, const int32_t* chunk_per_req,
                      int block, int window_rule,
                      int8_t* states, int64_t state_stride, int32_t* queue, int qcap,
                      int32_t* q_head, int32_t* q_len, int32_t* block_index,
                      int32_t* cached_prefix, const int32_t* prompt, const int32_t* out_len,
                      const int32_t* block_tables, int max_pages, int32_t* cu_seqlens,
                      int32_t* tok_req, int32_t* tok_pos, int cap_tok, int32_t* prompt_len,
                      int32_t* key_end, int32_t* vis_base, int32_t* vis_off,
                      uint32_t* vis_words, int cap_words, int32_t* cu_rows, int32_t* row_tok,
                      int32_t* row_pos, int32_t* row_req, int cap_rows,
                      int32_t* block_tables_out, int32_t* counts_out);
int optimus_host_apply(int n, const int32_t* slots, int block, const int32_t* cu_seqlens,
                       const int32_t* tok_pos, const int32_t* cu_rows, const int32_t* row_pos,
                       const uint8_t* commit_mask, int8_t* states, int64_t state_stride,
                       int32_t* queue, int qcap, int32_t* q_head, int32_t* q_len,
                       int32_t* block_index, int32_t* committed, int32_t* steps_taken,
                       int32_t* cached_prefix, const int32_t* out_len, int32_t* commits_out);

/*
 * fp16 V-cache range gate.  With an fp16 V cache, K1 (and the fused append) store
 * each bf16 V value as fp16 with cvt.rn.satfinite: |v| > 65504 is clamped to
 * +-65504.  Every kernel that clamps sets a device flag; this copies the flags
 * (out[0]: K1, out[1]: fused append; pinned host memory, stream-ordered: read them
 * after synchronizing `stream`) and, with reset != 0, clears them.  A set flag means
 * the model's V range needs a bf16 V cache.
 */
int optimus_v_saturated(int32_t* out, int reset, void* stream);

/* Recommended vocab split count for n_rows x vocab on the current device. */
int optimus_unmask_splits(int n_rows, int vocab);

/*
 * K3 in ONE launch on a single vocab shard: (a) and (b) above fused.  Each
 * (row, split) CTA writes its record to part [n_rows][n_vsplit]; the CTA that
 * completes a request's records (arrival counter counters[row_req[row]]) runs (b)
 * for that request.  counters: int32 [n_req], zero before the first call; every
 * call leaves them zero.  row_req[i] = request of window row i (rows of a request
 * are contiguous, cu_rows as in (b)).  n_rows_dev (optional): the row count of a
 * device-planned step, read on the device; n_rows then only bounds it (and the grid).
 * Results, commit rule and state update are exactly those of (a) + (b).
 */
int optimus_unmask_commit(const void* logits, int logits_dtype, int64_t row_stride, const int32_t* row_src,
                          int n_rows, const int32_t* n_rows_dev, int vocab, int n_vsplit, float* part,
                          const int32_t* cu_rows, const int32_t* row_req, int n_req, int32_t* counters, float tau,
                          int fallback_mode, uint8_t* commit_mask, int32_t* tok, float* conf,
                          const int32_t* row_pos, uint8_t* state, int32_t* token_buf, int64_t state_stride,
                          void* stream);

/*
 * f3: LM-head GEMM with the unmask partials in its epilogue; the
 * logits are never written.  hidden: bf16 [n_rows][hidden_stride] (first k_dim used),
 * weight: bf16 [vocab][weight_stride] (the LM head, row v = token v).  Writes
 * part[n_rows][optimus_lmhead_splits(vocab)] records in the layout of
 * optimus_unmask_partials (max logit, sum exp(x - max), lowest argmax + vocab_offset);
 * finish with optimus_unmask_finalize(part, 1, n_rows, optimus_lmhead_splits(vocab), ...).
 * tcgen05 (M=128, N=256) with a 4-stage TMA ring; k_dim and strides multiples of 8.
 */
int optimus_lmhead_splits(int vocab);
/* Merge part[n_rows][n_split] unmask records into out[n_rows][1] (same record layout;
 * a fixed per-row merge order), e.g. the hundreds of LM-head vocab tiles before
 * optimus_unmask_finalize(out, 1, n_rows, 1, ...). */
int optimus_unmask_merge_splits(const float* part, int n_rows, int n_split, float* out, void* stream);
int optimus_lmhead_unmask_partials(const void* hidden, int64_t hidden_stride, int n_rows, const void* weight,
                                   int64_t weight_stride, int vocab, int k_dim, int vocab_offset, float* part,
                                   void* stream);

/*
 * Device twins of optimus_host_plan / optimus_host_apply (device half):
 * the same packed per-slot state and step metadata, all pointers DEVICE pointers,
 * enqueued on `stream`, bit-identical results (tests/test_device_step_gpu.py).
 * n <= 256 requests, out_len <= 4096 positions, chunk <= 128.  counts[0..4) =
 * {n_tok, n_rows, n_words, status}; *status (apply) is set to OPTIMUS_EINVAL on an
 * illegal plan / commit (caller zeroes it).
 */
int optimus_device_plan(int n, const int32_t* slots, int chunk, const int32_t* chunk_per_req, int block,
                        int window_rule, const int8_t* states, int64_t state_stride, const int32_t* queue,
                        int qcap, const int32_t* q_head, const int32_t* q_len, const int32_t* block_index,
                        const int32_t* cached_prefix, const int32_t* prompt, const int32_t* out_len,
                        const int32_t* block_tables, int max_pages, int32_t* cu_seqlens, int32_t* tok_req,
                        int32_t* tok_pos, int cap_tok, int32_t* prompt_len, int32_t* key_end,
                        int32_t* vis_base, int32_t* vis_off, uint32_t* vis_words, int cap_words,
                        int32_t* cu_rows, int32_t* row_tok, int32_t* row_pos, int32_t* row_req, int cap_rows,
                        int32_t* block_tables_out, int32_t* counts, void* stream);
int optimus_device_apply(int n, const int32_t* slots, int block, const int32_t* cu_seqlens,
                         const int32_t* tok_pos, const int32_t* cu_rows, const int32_t* row_pos,
                         const uint8_t* commit_mask, int8_t* states, int64_t state_stride, int32_t* queue,
                         int qcap, int32_t* q_head, int32_t* q_len, int32_t* block_index, int32_t* committed,
                         int32_t* steps_taken, int32_t* cached_prefix, const int32_t* out_len,
                         int32_t* commits_out, int32_t* status, void* stream);

/*
 * Continuous batching on the device state (DeviceLoop.replace): copy n_adm admitted
 * requests' packed rows into their batch slots with ONE launch.  `records` (device)
 * holds n_adm records of optimus_admit_record_ints(state_stride, qcap, max_pages) int32:
 * {slot, q_head, q_len, block_index, committed, steps_taken, cached_prefix, prompt,
 * out_len, states row (state_stride bytes; state_stride % 4 == 0), queue row (qcap),
 * block-table row (max_pages)}.
 */
int optimus_admit_record_ints(int64_t state_stride, int qcap, int max_pages);
int optimus_device_admit(int n_adm, const int32_t* records, int8_t* states, int64_t state_stride, int32_t* queue,
                         int qcap, int32_t* q_head, int32_t* q_len, int32_t* block_index, int32_t* committed,
                         int32_t* steps_taken, int32_t* cached_prefix, int32_t* prompt, int32_t* out_len,
                         int32_t* block_tables, int max_pages, void* stream);

/*
 * Device twin of optimus_attn_plan (capi.cu) from device-resident cu_seqlens /
 * key_end (n_req <= 256, <= 4096 units and pieces, grid <= 1024).  allow_cut = 0:
 * its whole-unit placement (candidate A), output identical to the host planner under
 * OPTIMUS_PLAN_FORCE=whole.  allow_cut = 1: units costlier than the per-CTA budget are
 * cut into equal pieces when the longest unit would otherwise set the makespan (the
 * host's candidate-B rule), merged by optimus_paged_attn_combine_dev.
 * counts[0..4) = {n_work, n_groups, n_partials, status}.
 */
int optimus_device_attn_plan(int n_req, const int32_t* cu_seqlens, const int32_t* key_end, int num_q_heads,
                             int num_kv_heads, int grid, int page_size, int allow_cut, int32_t* work, int max_work,
                             int32_t* cta_off, int32_t* groups, int max_groups, int32_t* counts, void* stream);

/*
 * Split-KV combine of a device-planned step: merges the partials of the groups
 * optimus_device_attn_plan wrote (their count read from n_groups_dev = &counts[1];
 * max_groups = the groups buffer capacity).  Launch right after the layer's
 * optimus_paged_attn, with the same ws_o / ws_ml workspace.
 */
int optimus_paged_attn_combine_dev(const int32_t* groups, const int32_t* n_groups_dev, int max_groups,
                                   const float* ws_o, const float* ws_ml, int num_q_heads, int num_kv_heads,
                                   int head_dim, void* out, int64_t out_stride_tok, void* stream);

/*
 * Device-planned steps (counts produced on the device by optimus_device_plan):
 * K1 and the K3 partials with their token / row count read from device memory and
 * grids sized for the capacity (graph-capturable), and the slot-indexed logits-row
 * map of the synthetic forward (counts = optimus_device_plan's counts).
 */
int optimus_kv_append_dev(const void* k_new, const void* v_new, int64_t new_stride_tok, const int32_t* tok_req,
                          const int32_t* tok_pos, const int32_t* prompt_len, const int32_t* block_tables,
                          int max_pages, int n_tok_cap, const int32_t* n_tok_dev, int num_kv_heads, int head_dim,
                          int page_size, void* k_cache, void* v_cache, int v_dtype, void* stream);
/*
 * Device-count twins of optimus_slot_mapping / optimus_kv_append_slots (the loop's
 * "slots" K1: the step's slot map once, then one round trip per row in every layer).
 * optimus_slot_mapping_dev is a plain launch; optimus_kv_append_slots_dev launches with
 * programmatic stream serialization and reads n_tok_dev / slot_abs before its PDL wait,
 * so the slot map must come from an earlier, non-PDL launch of the same step.
 */
int optimus_slot_mapping_dev(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                             const int32_t* block_tables, int max_pages, int n_tok_cap, const int32_t* n_tok_dev,
                             int page_size, int32_t* slot_abs_out, void* stream);
int optimus_kv_append_slots_dev(const void* k_new, const void* v_new, int64_t new_stride_tok,
                                const int32_t* slot_abs, int n_tok_cap, const int32_t* n_tok_dev, int num_kv_heads,
                                int head_dim, int page_size, void* k_cache, void* v_cache, int v_dtype,
                                void* stream);
int optimus_unmask_partials_dev(const void* logits, int logits_dtype, int64_t row_stride, const int32_t* row_src,
                                int n_rows_cap, const int32_t* n_rows_dev, int vocab, int vocab_offset,
                                int n_vsplit, float* part, void* stream);
int optimus_device_row_src(const int32_t* counts, const int32_t* slots, const int32_t* cu_rows,
                           const int32_t* row_req, int cap_rows, int rows_per_slot, int base, int32_t* row_src,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OPTIMUS_B200_H */
