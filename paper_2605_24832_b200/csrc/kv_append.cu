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
// Pure streaming: each K/V byte is read once and written once.  With an fp16 V
// cache (v_fp16) the bf16 V rows are converted on the way (exact for |v| < 65504,
// saturating beyond), which lets the attention kernel form P.V in fp16 with an
// 11-bit P in one MMA instead of two bf16 planes.
#include "ptx.cuh"

namespace optimus {

// Set when a bf16 V value beyond the fp16 range (|v| > 65504) was clamped on its way
// into an fp16 V cache (cvt.rn.satfinite); read and cleared by optimus_v_saturated.
__device__ int g_v_saturated_k1;

// Store 8 bf16 V values (one 16-byte vector) as fp16; flag values fp16 clamps.
__device__ __forceinline__ uint4 v_to_fp16(uint4 vv) {
  const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
  uint32_t h[4];
  bool sat = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
    sat |= fabsf(lo) > 65504.f || fabsf(hi) > 65504.f;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(hi), "f"(lo));
  }
  if (__builtin_expect(sat, 0)) atomicOr(&g_v_saturated_k1, 1);
  return make_uint4(h[0], h[1], h[2], h[3]);
}

// One thread per 16-byte vector of a (token, head) row: n_tok*Hkv*head_dim/8
// independent load/store pairs for K and for V, so the scatter runs at full
// memory-level parallelism instead of one serial loop per token.
__global__ void __launch_bounds__(256) kv_append_kernel(
    const uint4* __restrict__ k_new, const uint4* __restrict__ v_new, int64_t new_stride_vec,
    const int32_t* __restrict__ tok_req, const int32_t* __restrict__ tok_pos,
    const int32_t* __restrict__ prompt_len, const int32_t* __restrict__ block_tables,
    int max_pages, int n_tok, int hkv, int vec_per_head, int page_size, uint4* __restrict__ k_cache,
    uint4* __restrict__ v_cache, int64_t* __restrict__ slot_out, int v_fp16,
    const int32_t* __restrict__ n_tok_dev) {
  // let a PDL-launched dependent (the attention kernel) start its prologue now; it
  // waits for this grid's completion before reading the cache.
  grid_dep_launch();
  if (n_tok_dev != nullptr) n_tok = *n_tok_dev;  // device-planned step (grid sized for capacity)
  const int per_tok = hkv * vec_per_head;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= static_cast<int64_t>(n_tok) * per_tok) return;
  const int t = static_cast<int>(gid / per_tok);
  const int i = static_cast<int>(gid - static_cast<int64_t>(t) * per_tok);
  const int h = i / vec_per_head;
  const int c = i - h * vec_per_head;
  const int r = __ldg(tok_req + t);
  const int s = __ldg(prompt_len + r) + __ldg(tok_pos + t);
  const int page = __ldg(block_tables + static_cast<int64_t>(r) * max_pages + s / page_size);
  const int off = s % page_size;
  const int64_t src = static_cast<int64_t>(t) * new_stride_vec + i;
  // PDL: the slot computation above overlapped the preceding grid's tail; the rows
  // (its outputs in a model) and the pages (a preceding attention grid may still read
  // them) are touched only after it completed
  grid_dep_wait();
  const uint4 kv = __ldg(k_new + src);
  const uint4 vv = __ldg(v_new + src);
  const int64_t dst =
      ((static_cast<int64_t>(page) * hkv + h) * page_size + off) * vec_per_head + c;
  k_cache[dst] = kv;
  if (v_fp16) {
    v_cache[dst] = v_to_fp16(vv);
  } else {
    v_cache[dst] = vv;
  }
  if (i == 0 && slot_out != nullptr) slot_out[t] = static_cast<int64_t>(page) * page_size + off;
}

// K1 launches with programmatic stream serialization: its blocks start on the SMs the
// preceding grid (the previous layer's attention) releases, and wait in-kernel.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int blocks, int threads, cudaStream_t stream,
                              Args... args) {
  static const bool pdl = [] {
    const char* e = getenv("OPTIMUS_K1_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int launch_kv_append(const void* k_new, const void* v_new, int64_t new_stride_tok,
                     const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                     const int32_t* block_tables, int max_pages, int n_tok, int hkv, int head_dim,
                     int page_size, void* k_cache, void* v_cache, int64_t* slot_out,
                     int v_fp16, cudaStream_t stream) {
  if (n_tok == 0) return 0;
  const int vec_per_head = head_dim / 8;  // 8 bf16 per 16-byte vector
  const int64_t total = static_cast<int64_t>(n_tok) * hkv * vec_per_head;
  const int threads = 256;
  const int blocks = static_cast<int>((total + threads - 1) / threads);
  return static_cast<int>(launch_pdl(
      kv_append_kernel, blocks, threads, stream, static_cast<const uint4*>(k_new),
      static_cast<const uint4*>(v_new), new_stride_tok / 8, tok_req, tok_pos, prompt_len, block_tables,
      max_pages, n_tok, hkv, vec_per_head, page_size, static_cast<uint4*>(k_cache),
      static_cast<uint4*>(v_cache), slot_out, v_fp16, static_cast<const int32_t*>(nullptr)));
}

// Same, with the token count read from device memory (n_tok_cap sizes the grid).
int launch_kv_append_dev(const void* k_new, const void* v_new, int64_t new_stride_tok,
                         const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                         const int32_t* block_tables, int max_pages, int n_tok_cap, const int32_t* n_tok_dev,
                         int hkv, int head_dim, int page_size, void* k_cache, void* v_cache, int v_fp16,
                         cudaStream_t stream) {
  if (n_tok_cap == 0) return 0;
  const int vec_per_head = head_dim / 8;
  const int64_t total = static_cast<int64_t>(n_tok_cap) * hkv * vec_per_head;
  const int blocks = static_cast<int>((total + 255) / 256);
  return static_cast<int>(launch_pdl(
      kv_append_kernel, blocks, 256, stream, static_cast<const uint4*>(k_new),
      static_cast<const uint4*>(v_new), new_stride_tok / 8, tok_req, tok_pos, prompt_len, block_tables,
      max_pages, n_tok_cap, hkv, vec_per_head, page_size, static_cast<uint4*>(k_cache),
      static_cast<uint4*>(v_cache), static_cast<int64_t*>(nullptr), v_fp16, n_tok_dev));
}

// K1 over a precomputed per-step slot map (optimus_slot_mapping): one round trip
// (slot + row loads in parallel) instead of the tok_req -> prompt -> block-table chain.
__global__ void __launch_bounds__(256) kv_append_slots_kernel(
    const uint4* __restrict__ k_new, const uint4* __restrict__ v_new, int64_t new_stride_vec,
    const int2* __restrict__ slot_abs, int n_tok, int hkv, int vec_per_head, int page_size,
    int page_shift, uint4* __restrict__ k_cache, uint4* __restrict__ v_cache, int v_fp16,
    const int32_t* __restrict__ n_tok_dev) {
  grid_dep_launch();
  // device-planned step: the count (and slot_abs, from the non-PDL slot-map launch
  // earlier in the step) are complete before this grid starts
  if (n_tok_dev != nullptr) n_tok = *n_tok_dev;
  const int per_tok = hkv * vec_per_head;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= static_cast<int64_t>(n_tok) * per_tok) return;
  const int t = static_cast<int>(gid / per_tok);
  const int i = static_cast<int>(gid - static_cast<int64_t>(t) * per_tok);
  const int h = i / vec_per_head;
  const int c = i - h * vec_per_head;
  const int slot = __ldg(slot_abs + t).y;
  const int64_t src = static_cast<int64_t>(t) * new_stride_vec + i;
  grid_dep_wait();
  const uint4 kv = __ldg(k_new + src);
  const uint4 vv = __ldg(v_new + src);
  const int64_t dst = ((static_cast<int64_t>(slot >> page_shift) * hkv + h) * page_size +
                       (slot & (page_size - 1))) * vec_per_head + c;
  k_cache[dst] = kv;
  if (v_fp16) {
    v_cache[dst] = v_to_fp16(vv);
  } else {
    v_cache[dst] = vv;
  }
}

int launch_kv_append_slots(const void* k_new, const void* v_new, int64_t new_stride_tok,
                           const int32_t* slot_abs, int n_tok, int hkv, int head_dim, int page_size,
                           void* k_cache, void* v_cache, int v_fp16, cudaStream_t stream) {
  if (n_tok == 0) return 0;
  const int vec_per_head = head_dim / 8;
  const int64_t total = static_cast<int64_t>(n_tok) * hkv * vec_per_head;
  const int blocks = static_cast<int>((total + 255) / 256);
  return static_cast<int>(launch_pdl(
      kv_append_slots_kernel, blocks, 256, stream, static_cast<const uint4*>(k_new),
      static_cast<const uint4*>(v_new), new_stride_tok / 8, reinterpret_cast<const int2*>(slot_abs), n_tok,
      hkv, vec_per_head, page_size, __builtin_ctz(static_cast<unsigned>(page_size)),
      static_cast<uint4*>(k_cache), static_cast<uint4*>(v_cache), v_fp16, static_cast<const int32_t*>(nullptr)));
}

// Same, with the token count read from device memory (n_tok_cap sizes the grid).
int launch_kv_append_slots_dev(const void* k_new, const void* v_new, int64_t new_stride_tok,
                               const int32_t* slot_abs, int n_tok_cap, const int32_t* n_tok_dev, int hkv,
                               int head_dim, int page_size, void* k_cache, void* v_cache, int v_fp16,
                               cudaStream_t stream) {
  if (n_tok_cap == 0) return 0;
  const int vec_per_head = head_dim / 8;
  const int64_t total = static_cast<int64_t>(n_tok_cap) * hkv * vec_per_head;
  const int blocks = static_cast<int>((total + 255) / 256);
  return static_cast<int>(launch_pdl(
      kv_append_slots_kernel, blocks, 256, stream, static_cast<const uint4*>(k_new),
      static_cast<const uint4*>(v_new), new_stride_tok / 8, reinterpret_cast<const int2*>(slot_abs), n_tok_cap,
      hkv, vec_per_head, page_size, __builtin_ctz(static_cast<unsigned>(page_size)),
      static_cast<uint4*>(k_cache), static_cast<uint4*>(v_cache), v_fp16, n_tok_dev));
}

// Per-step slot map for the fused append (K2 with k_new): out[t] = {prompt + pos,
// slot} (rule S), computed once per step instead of in every layer's kernel.
__global__ void __launch_bounds__(256) slot_map_kernel(
    const int32_t* __restrict__ tok_req, const int32_t* __restrict__ tok_pos,
    const int32_t* __restrict__ prompt_len, const int32_t* __restrict__ block_tables, int max_pages,
    int n_tok, int page_size, int32_t* __restrict__ out, const int32_t* __restrict__ n_tok_dev) {
  if (n_tok_dev != nullptr) n_tok = *n_tok_dev;  // device-planned step (grid sized for capacity)
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tok) return;
  const int r = __ldg(tok_req + t);
  const int s = __ldg(prompt_len + r) + __ldg(tok_pos + t);
  const int page = __ldg(block_tables + static_cast<int64_t>(r) * max_pages + s / page_size);
  reinterpret_cast<int2*>(out)[t] = make_int2(s, page * page_size + s % page_size);
}

int launch_slot_map(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                    const int32_t* block_tables, int max_pages, int n_tok, int page_size,
                    int32_t* out, cudaStream_t stream) {
  if (n_tok == 0) return 0;
  slot_map_kernel<<<(n_tok + 255) / 256, 256, 0, stream>>>(tok_req, tok_pos, prompt_len, block_tables,
                                                           max_pages, n_tok, page_size, out, nullptr);
  return static_cast<int>(cudaGetLastError());
}

// Same, with the token count read from device memory (a plain launch: the per-layer K1
// of the step, PDL-launched behind it, reads its output before their PDL wait).
int launch_slot_map_dev(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                        const int32_t* block_tables, int max_pages, int n_tok_cap, const int32_t* n_tok_dev,
                        int page_size, int32_t* out, cudaStream_t stream) {
  if (n_tok_cap == 0) return 0;
  slot_map_kernel<<<(n_tok_cap + 255) / 256, 256, 0, stream>>>(tok_req, tok_pos, prompt_len, block_tables,
                                                               max_pages, n_tok_cap, page_size, out, n_tok_dev);
  return static_cast<int>(cudaGetLastError());
}

// Copy the saturation flag into *out (stream-ordered) and optionally clear it.
int v_saturated_k1(int32_t* out, int reset, cudaStream_t stream) {
  cudaError_t e = cudaMemcpyFromSymbolAsync(out, g_v_saturated_k1, sizeof(int), 0, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess && reset) {
    void* a = nullptr;
    e = cudaGetSymbolAddress(&a, g_v_saturated_k1);
    if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, sizeof(int), stream);
  }
  return static_cast<int>(e);
}

}  // namespace optimus
