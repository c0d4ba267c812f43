// capi.cu — the extern "C" boundary (include/optimus_b200.h): argument
// validation, TMA descriptor encoding (cached), the host-side split-KV /
// persistent-CTA work planner, and kernel launches.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "../../include/optimus_b200.h"
#include "attn.cuh"

namespace optimus {

int launch_kv_append_slots(const void*, const void*, int64_t, const int32_t*, int, int, int, int,
                           void*, void*, int, cudaStream_t);
int launch_kv_append_dev(const void*, const void*, int64_t, const int32_t*, const int32_t*, const int32_t*,
                         const int32_t*, int, int, const int32_t*, int, int, int, void*, void*, int, cudaStream_t);
int launch_unmask_partials_dev(const void*, int, int64_t, const int32_t*, int, const int32_t*, int, int, int,
                               float*, cudaStream_t);
int launch_slot_map(const int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int,
                    int32_t*, cudaStream_t);
int launch_slot_map_dev(const int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, const int32_t*,
                        int, int32_t*, cudaStream_t);
int launch_kv_append_slots_dev(const void*, const void*, int64_t, const int32_t*, int, const int32_t*, int, int,
                               int, void*, void*, int, cudaStream_t);
int launch_kv_append(const void*, const void*, int64_t, const int32_t*, const int32_t*,
                     const int32_t*, const int32_t*, int, int, int, int, int, void*, void*,
                     int64_t*, int, cudaStream_t);
int launch_unmask_partials(const void*, int, int64_t, const int32_t*, int, int, int, int, float*,
                           cudaStream_t);
int launch_unmask_finalize(const float*, int, int, int, const int32_t*, int, float, int, uint8_t*,
                           int32_t*, float*, const int32_t*, uint8_t*, int32_t*, int64_t,
                           cudaStream_t);
int launch_unmask_commit(const void*, int, int64_t, const int32_t*, int, const int32_t*, int, int, float*,
                         const int32_t*, const int32_t*, int32_t*, float, int, uint8_t*, int32_t*, float*,
                         const int32_t*, uint8_t*, int32_t*, int64_t, cudaStream_t);
int v_saturated_k1(int32_t*, int, cudaStream_t);
int v_saturated_k2(int32_t*, int, cudaStream_t);
int launch_lmhead_unmask(const CUtensorMap&, const CUtensorMap&, int, int, int, int, float*, cudaStream_t);
int launch_merge_splits(const float*, int, int, float*, cudaStream_t);

}  // namespace optimus



using namespace optimus;

namespace {

thread_local std::string g_last_error;
unsigned long long* g_trace = nullptr;  // optimus_set_attn_trace (diagnostics)

int fail(const char* what) {
  g_last_error = what;
  return OPTIMUS_EINVAL;
}
int cuda_status(int st, const char* where) {
  if (st != 0) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(static_cast<cudaError_t>(st));
  }
  return st;
}

// -1 unknown, 0 not sm_100, 1 ok
int g_arch_ok = -1;
int g_sm_count = 0;
std::mutex g_mu;

int check_device() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_arch_ok < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      g_arch_ok = 0;
    } else {
      cudaDeviceProp prop;
      if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
        g_arch_ok = 0;
      } else {
        g_arch_ok = (prop.major == 10 && prop.minor == 0) ? 1 : 0;
        g_sm_count = prop.multiProcessorCount;
      }
    }
  }
  if (g_arch_ok != 1) {
    g_last_error = "device is not an sm_100 (B200) GPU";
    return OPTIMUS_ENOSYS;
  }
  return 0;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

struct MapKey {
  const void* ptr;
  uint64_t dims[4];
  uint64_t strides[3];
  uint32_t box[4];
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && !memcmp(dims, o.dims, sizeof(dims)) &&
           !memcmp(strides, o.strides, sizeof(strides)) && !memcmp(box, o.box, sizeof(box));
  }
};
struct MapEntry {
  MapKey key;
  CUtensorMap map;
};
thread_local std::vector<MapEntry> g_maps;

// 4-D bf16 tensor map with SWIZZLE_128B (boxes are 64 columns = 128 bytes wide).
int get_map(const void* ptr, const uint64_t dims[4], const uint64_t strides[3],
            const uint32_t box[4], CUtensorMap* out, bool fp16 = false) {
  MapKey key;
  key.ptr = static_cast<const char*>(ptr) + (fp16 ? 1 : 0) * 0;  // dtype folded into box[2] below
  memcpy(key.dims, dims, sizeof(key.dims));
  memcpy(key.strides, strides, sizeof(key.strides));
  memcpy(key.box, box, sizeof(key.box));
  if (fp16) key.box[2] |= 0x80000000u;
  for (size_t i = 0; i < g_maps.size(); ++i)
    if (g_maps[i].key == key) {
      *out = g_maps[i].map;
      return 0;
    }
  auto fn = encode_fn();
  if (!fn) return fail("cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t gs[3] = {strides[0], strides[1], strides[2]};
  cuuint32_t bd[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(&m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                  const_cast<void*>(ptr), gd, gs, bd, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return fail(buf);
  }
  if (g_maps.size() >= 256) g_maps.erase(g_maps.begin());
  g_maps.push_back({key, m});
  *out = m;
  return 0;
}

// Page sizes: powers of two from 8 to 1024 keys (a 64-key tile covers whole pages,
// or whole tiles fit in one page).
bool page_ok(int P) { return P >= 8 && P <= 1024 && (P & (P - 1)) == 0; }

}  // namespace

extern "C" {

int optimus_version(void) { return 100; }

void optimus_set_attn_trace(unsigned long long* buf) { g_trace = buf; }

const char* optimus_last_error(void) { return g_last_error.c_str(); }

int optimus_device_sm_count(void) {
  if (check_device() != 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      return n;
    return 0;
  }
  return g_sm_count;
}

int optimus_kv_append(const void* k_new, const void* v_new, int64_t new_stride_tok,
                      const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                      const int32_t* block_tables, int max_pages, int n_tok, int num_kv_heads,
                      int head_dim, int page_size, void* k_cache, void* v_cache,
                      int64_t num_pages, int64_t* slot_mapping_out, int v_dtype, void* stream) {
  if (v_dtype != 0 && v_dtype != 1) return fail("kv_append: v_dtype must be 0 (bf16) or 1 (fp16)");
  if (n_tok < 0 || num_kv_heads < 1 || max_pages < 1 || num_pages < 1)
    return fail("kv_append: bad sizes");
  if (head_dim % 8 || head_dim < 8) return fail("kv_append: head_dim must be a multiple of 8");
  if (new_stride_tok < static_cast<int64_t>(num_kv_heads) * head_dim || new_stride_tok % 8)
    return fail("kv_append: new_stride_tok must be >= Hkv*head_dim and a multiple of 8");
  if (page_size < 1) return fail("kv_append: page_size must be >= 1");
  if (n_tok == 0) return 0;
  if (!k_new || !v_new || !tok_req || !tok_pos || !prompt_len || !block_tables || !k_cache ||
      !v_cache)
    return fail("kv_append: null pointer");
  if (int st = check_device()) return st;
  return cuda_status(
      launch_kv_append(k_new, v_new, new_stride_tok, tok_req, tok_pos, prompt_len, block_tables,
                       max_pages, n_tok, num_kv_heads, head_dim, page_size, k_cache, v_cache,
                       slot_mapping_out, v_dtype, static_cast<cudaStream_t>(stream)),
      "kv_append");
}

int optimus_kv_append_slots(const void* k_new, const void* v_new, int64_t new_stride_tok,
                            const int32_t* slot_abs, int n_tok, int num_kv_heads, int head_dim,
                            int page_size, void* k_cache, void* v_cache, int64_t num_pages,
                            int v_dtype, void* stream) {
  if (v_dtype != 0 && v_dtype != 1) return fail("kv_append_slots: v_dtype must be 0 (bf16) or 1 (fp16)");
  if (n_tok < 0 || num_kv_heads < 1 || num_pages < 1) return fail("kv_append_slots: bad sizes");
  if (head_dim % 8 || head_dim < 8) return fail("kv_append_slots: head_dim must be a multiple of 8");
  if (new_stride_tok < static_cast<int64_t>(num_kv_heads) * head_dim || new_stride_tok % 8)
    return fail("kv_append_slots: new_stride_tok must be >= Hkv*head_dim and a multiple of 8");
  if (!page_ok(page_size)) return fail("kv_append_slots: page_size must be a power of two in [8, 1024]");
  if (n_tok == 0) return 0;
  if (!k_new || !v_new || !slot_abs || !k_cache || !v_cache) return fail("kv_append_slots: null pointer");
  if (reinterpret_cast<uintptr_t>(slot_abs) % 8) return fail("kv_append_slots: slot_abs must be 8-byte aligned");
  if (int st = check_device()) return st;
  return cuda_status(launch_kv_append_slots(k_new, v_new, new_stride_tok, slot_abs, n_tok, num_kv_heads,
                                            head_dim, page_size, k_cache, v_cache, v_dtype,
                                            static_cast<cudaStream_t>(stream)),
                     "kv_append_slots");
}

int optimus_kv_append_dev(const void* k_new, const void* v_new, int64_t new_stride_tok, const int32_t* tok_req,
                          const int32_t* tok_pos, const int32_t* prompt_len, const int32_t* block_tables,
                          int max_pages, int n_tok_cap, const int32_t* n_tok_dev, int num_kv_heads, int head_dim,
                          int page_size, void* k_cache, void* v_cache, int v_dtype, void* stream) {
  if (v_dtype != 0 && v_dtype != 1) return fail("kv_append_dev: v_dtype must be 0 or 1");
  if (n_tok_cap < 0 || num_kv_heads < 1 || head_dim % 8 || page_size < 1) return fail("kv_append_dev: bad sizes");
  if (new_stride_tok < static_cast<int64_t>(num_kv_heads) * head_dim || new_stride_tok % 8)
    return fail("kv_append_dev: bad new_stride_tok");
  if (!n_tok_dev || !k_new || !v_new || !tok_req || !tok_pos || !prompt_len || !block_tables || !k_cache ||
      !v_cache)
    return fail("kv_append_dev: null pointer");
  if (int st = check_device()) return st;
  return cuda_status(launch_kv_append_dev(k_new, v_new, new_stride_tok, tok_req, tok_pos, prompt_len, block_tables,
                                          max_pages, n_tok_cap, n_tok_dev, num_kv_heads, head_dim, page_size,
                                          k_cache, v_cache, v_dtype, static_cast<cudaStream_t>(stream)),
                     "kv_append_dev");
}

int optimus_unmask_partials_dev(const void* logits, int logits_dtype, int64_t row_stride, const int32_t* row_src,
                                int n_rows_cap, const int32_t* n_rows_dev, int vocab, int vocab_offset,
                                int n_vsplit, float* part, void* stream) {
  if (logits_dtype != 0 && logits_dtype != 1) return fail("unmask_dev: logits_dtype must be 0 or 1");
  const int vec = logits_dtype == 0 ? 8 : 4;
  if (vocab < 1 || vocab % vec || row_stride % vec || row_stride < vocab) return fail("unmask_dev: bad vocab");
  if (n_rows_cap < 0 || n_vsplit < 1 || !n_rows_dev || !logits || !part) return fail("unmask_dev: bad args");
  if (int st = check_device()) return st;
  return cuda_status(launch_unmask_partials_dev(logits, logits_dtype, row_stride, row_src, n_rows_cap, n_rows_dev,
                                                vocab, vocab_offset, n_vsplit, part,
                                                static_cast<cudaStream_t>(stream)),
                     "unmask_partials_dev");
}

// f3: LM-head GEMM with the unmask partials in its epilogue (lmhead_unmask.cu).
int optimus_lmhead_splits(int vocab) { return vocab < 1 ? 0 : (vocab + 255) / 256; }

int optimus_lmhead_unmask_partials(const void* hidden, int64_t hidden_stride, int n_rows, const void* weight,
                                   int64_t weight_stride, int vocab, int k_dim, int vocab_offset, float* part,
                                   void* stream) {
  if (n_rows < 0 || vocab < 1 || k_dim < 8 || k_dim % 8) return fail("lmhead: bad sizes (k_dim % 8 == 0)");
  if (hidden_stride < k_dim || weight_stride < k_dim || hidden_stride % 8 || weight_stride % 8)
    return fail("lmhead: row strides must be >= k_dim and multiples of 8 elements");
  if (!hidden || !weight || !part) return fail("lmhead: null pointer");
  if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(weight)) & 15)
    return fail("lmhead: hidden / weight must be 16-byte aligned");
  if (n_rows == 0) return 0;
  if (int st = check_device()) return st;
  CUtensorMap th, tw;
  const uint64_t dh[4] = {static_cast<uint64_t>(k_dim), static_cast<uint64_t>(n_rows), 1, 1};
  const uint64_t sh[3] = {static_cast<uint64_t>(hidden_stride) * 2, static_cast<uint64_t>(hidden_stride) * 2 * n_rows,
                          static_cast<uint64_t>(hidden_stride) * 2 * n_rows};
  const uint32_t bh[4] = {64, 128, 1, 1};
  if (int st = get_map(hidden, dh, sh, bh, &th)) return st;
  const uint64_t dw[4] = {static_cast<uint64_t>(k_dim), static_cast<uint64_t>(vocab), 1, 1};
  const uint64_t sw[3] = {static_cast<uint64_t>(weight_stride) * 2, static_cast<uint64_t>(weight_stride) * 2 * vocab,
                          static_cast<uint64_t>(weight_stride) * 2 * vocab};
  const uint32_t bw[4] = {64, 256, 1, 1};
  if (int st = get_map(weight, dw, sw, bw, &tw)) return st;
  return cuda_status(launch_lmhead_unmask(th, tw, n_rows, vocab, k_dim, vocab_offset, part,
                                          static_cast<cudaStream_t>(stream)),
                     "lmhead_unmask");
}

int optimus_slot_mapping_dev(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                             const int32_t* block_tables, int max_pages, int n_tok_cap, const int32_t* n_tok_dev,
                             int page_size, int32_t* slot_abs_out, void* stream) {
  if (n_tok_cap < 0 || max_pages < 1 || page_size < 1) return fail("slot_mapping_dev: bad sizes");
  if (n_tok_cap == 0) return 0;
  if (!n_tok_dev || !tok_req || !tok_pos || !prompt_len || !block_tables || !slot_abs_out)
    return fail("slot_mapping_dev: null pointer");
  if (reinterpret_cast<uintptr_t>(slot_abs_out) % 8) return fail("slot_mapping_dev: slot_abs must be 8-byte aligned");
  if (int st = check_device()) return st;
  return cuda_status(launch_slot_map_dev(tok_req, tok_pos, prompt_len, block_tables, max_pages, n_tok_cap,
                                         n_tok_dev, page_size, slot_abs_out, static_cast<cudaStream_t>(stream)),
                     "slot_mapping_dev");
}

int optimus_kv_append_slots_dev(const void* k_new, const void* v_new, int64_t new_stride_tok,
                                const int32_t* slot_abs, int n_tok_cap, const int32_t* n_tok_dev, int num_kv_heads,
                                int head_dim, int page_size, void* k_cache, void* v_cache, int v_dtype,
                                void* stream) {
  if (v_dtype != 0 && v_dtype != 1) return fail("kv_append_slots_dev: v_dtype must be 0 or 1");
  if (n_tok_cap < 0 || num_kv_heads < 1 || head_dim % 8 || head_dim < 8)
    return fail("kv_append_slots_dev: bad sizes");
  if (new_stride_tok < static_cast<int64_t>(num_kv_heads) * head_dim || new_stride_tok % 8)
    return fail("kv_append_slots_dev: bad new_stride_tok");
  if (!page_ok(page_size)) return fail("kv_append_slots_dev: page_size must be a power of two in [8, 1024]");
  if (n_tok_cap == 0) return 0;
  if (!n_tok_dev || !k_new || !v_new || !slot_abs || !k_cache || !v_cache)
    return fail("kv_append_slots_dev: null pointer");
  if (reinterpret_cast<uintptr_t>(slot_abs) % 8) return fail("kv_append_slots_dev: slot_abs must be 8-byte aligned");
  if (int st = check_device()) return st;
  return cuda_status(launch_kv_append_slots_dev(k_new, v_new, new_stride_tok, slot_abs, n_tok_cap, n_tok_dev,
                                                num_kv_heads, head_dim, page_size, k_cache, v_cache, v_dtype,
                                                static_cast<cudaStream_t>(stream)),
                     "kv_append_slots_dev");
}

int optimus_unmask_merge_splits(const float* part, int n_rows, int n_split, float* out, void* stream) {
  if (n_rows < 0 || n_split < 1 || (n_rows > 0 && (!part || !out))) return fail("merge_splits: bad args");
  if (n_rows == 0) return 0;
  if (int st = check_device()) return st;
  return cuda_status(launch_merge_splits(part, n_rows, n_split, out, static_cast<cudaStream_t>(stream)),
                     "merge_splits");
}

int optimus_slot_mapping(const int32_t* tok_req, const int32_t* tok_pos, const int32_t* prompt_len,
                         const int32_t* block_tables, int max_pages, int n_tok, int page_size,
                         int32_t* slot_abs_out, void* stream) {
  if (n_tok < 0 || max_pages < 1 || page_size < 1) return fail("slot_mapping: bad sizes");
  if (n_tok == 0) return 0;
  if (!tok_req || !tok_pos || !prompt_len || !block_tables || !slot_abs_out)
    return fail("slot_mapping: null pointer");
  if (int st = check_device()) return st;
  return cuda_status(launch_slot_map(tok_req, tok_pos, prompt_len, block_tables, max_pages, n_tok,
                                     page_size, slot_abs_out, static_cast<cudaStream_t>(stream)),
                     "slot_mapping");
}

namespace {
// An item's key range must span at most 255 pages (the kernel stages an item's page
// ids in shared memory, kMaxUnitPages = 256).
int item_tile_cap(int page_size) {
  const long long cap = (255LL * std::max(page_size, 1)) / 64;
  return static_cast<int>(std::max(1LL, std::min(cap, 1LL << 20)));
}
}  // namespace

int optimus_attn_plan_bounds(int n_req, const int32_t* cu, const int32_t* key_end, int hq,
                             int hkv, int min_split_tiles, int page_size, int* max_work,
                             int* max_groups) {
  if (n_req < 0 || hkv < 1 || hq % hkv) return fail("attn_plan_bounds: bad heads");
  const int G = hq / hkv;
  if (G > 128) return fail("attn_plan_bounds: group size > 128");
  const int T = 128 / G;
  if (min_split_tiles < 1) min_split_tiles = 1;
  long long w = 0, g = 0;
  for (int r = 0; r < n_req; ++r) {
    const int nq = cu[r + 1] - cu[r];
    if (nq <= 0) continue;
    const int mt = (nq + T - 1) / T;
    const int nt = (key_end[r] + 63) / 64;
    const int cap = item_tile_cap(page_size);
    const int maxs = std::max(std::max(1, nt / min_split_tiles), (nt + cap - 1) / cap);
    w += static_cast<long long>(hkv) * mt * maxs;
    g += static_cast<long long>(hkv) * mt;
  }
  *max_work = static_cast<int>(w);
  *max_groups = static_cast<int>(g);
  return 0;
}

int optimus_attn_plan(int n_req, const int32_t* cu, const int32_t* key_end, int hq, int hkv,
                      int grid, int min_split_tiles, int page_size, int32_t* work, int max_work,
                      int32_t* cta_off, int32_t* groups, int max_groups, int* n_groups_out,
                      int* n_partials_out) {
  if (n_req < 0 || hkv < 1 || hq % hkv || grid < 1) return fail("attn_plan: bad arguments");
  const int G = hq / hkv;
  if (G > 128) return fail("attn_plan: group size > 128");
  const int T = 128 / G;
  if (min_split_tiles < 1) min_split_tiles = 1;
  struct Unit {
    int req, head, tok_begin, n_tok, tiles;
  };
  std::vector<Unit> units;
  units.reserve(static_cast<size_t>(n_req) * hkv * 2);
  for (int r = 0; r < n_req; ++r) {
    const int nq = cu[r + 1] - cu[r];
    if (nq <= 0) continue;
    if (key_end[r] < 1) return fail("attn_plan: key_end must be >= 1 for a request with queries");
    const int nt = (key_end[r] + 63) / 64;
    for (int h = 0; h < hkv; ++h)
      for (int t0 = 0; t0 < nq; t0 += T) {
        units.push_back({r, h, cu[r] + t0, std::min(T, nq - t0), nt});
      }
  }
  // Cost model (in 64-key tile units; a tile is ~1100 SM cycles in the steady
  // state): every item pays a fixed prologue/epilogue (Q load, O drain, pipeline
  // refill: ~1.9 tiles in a per-CTA fit since the epilogue warpgroup drains O beside
  // the softmax, 0.57 us/tile + 1.08 us/item; 1.5 picks the faster plans across the
  // bench workloads, profiles/r2ce_kitem.md) and a cut item also pays its partial write
  // and the combine read.
  double kItem = 1.5;
  const double kSplit = 1.5;
  if (const char* e = std::getenv("OPTIMUS_PLAN_KITEM")) kItem = std::atof(e);  // diagnostics
  const int hard_cap = item_tile_cap(page_size);
  const int nu = static_cast<int>(units.size());
  std::vector<int> order(nu);
  for (int i = 0; i < nu; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return units[a].tiles > units[b].tiles; });
  struct Piece {
    int unit, t0, nt, cta;
  };

  // ---- candidate A: whole units (cut only at the per-item page cap), placed
  // longest-first on the least-loaded CTA.
  std::vector<Piece> pa;
  pa.reserve(nu + 16);
  double span_a = 0;
  {
    typedef std::pair<double, int> LoadCta;
    std::vector<LoadCta> heap;
    heap.reserve(grid);
    for (int c = 0; c < grid; ++c) heap.push_back(LoadCta(0.0, c));
    auto cmp = [](const LoadCta& a, const LoadCta& b) { return a > b; };  // min-heap
    for (int ui : order) {
      const int tiles = units[ui].tiles;
      const int sc = (tiles + hard_cap - 1) / hard_cap;
      const int base = tiles / sc, rem = tiles % sc;
      int t0 = 0;
      for (int k = 0; k < sc; ++k) {
        const int nt = base + (k < rem ? 1 : 0);
        std::pop_heap(heap.begin(), heap.end(), cmp);
        LoadCta& lc = heap.back();
        pa.push_back({ui, t0, nt, lc.second});
        lc.first += nt + kItem + (sc > 1 ? kSplit : 0.0);
        span_a = std::max(span_a, lc.first);
        std::push_heap(heap.begin(), heap.end(), cmp);
        t0 += nt;
      }
    }
  }

  // Cutting can only win if even a perfectly balanced cut plan (the mean CTA load)
  // plus the combine launch beats whole units by > 3% (the rule below): otherwise
  // keep candidate A and skip B.
  // ~12 tiles: measured on the tp30b batch (G = 8), where the cut plan the old 7-tile
  // figure picked ran 30.5 us against 28.2 us whole; the other workloads keep their plans
  double kCombine = 12.0;
  if (const char* e = std::getenv("OPTIMUS_PLAN_KCOMBINE")) kCombine = std::atof(e);  // diagnostics
  double lb = 0;
  for (const Unit& u : units) lb += u.tiles + kItem;
  lb /= grid;
  const bool a_good = lb + kCombine >= 0.97 * span_a && std::getenv("OPTIMUS_PLAN_FORCE") == nullptr;

  // ---- candidate B: LPT with cutting.  Pieces are placed largest first on the
  // least-loaded CTA; a piece that would push that CTA past the balanced budget
  // (mean load + one item) is cut to fit and its remainder re-queued, so only the
  // units that do not pack are split, and each only as far as needed.
  std::vector<Piece> pb;
  double span_b = 1e300;
  if (!a_good) {
    pb.reserve(nu + 2 * grid + 16);
    span_b = 0;
    double total_cost = 0;
    for (const Unit& u : units) total_cost += u.tiles + kItem;
    const double budget = total_cost / grid + kItem;
    typedef std::pair<double, int> LoadCta;
    std::vector<LoadCta> heap;
    heap.reserve(grid);
    for (int c = 0; c < grid; ++c) heap.push_back(LoadCta(0.0, c));
    auto cmin = [](const LoadCta& a, const LoadCta& b) { return a > b; };
    struct Pend {
      int tiles, unit, t0;
      bool operator<(const Pend& o) const {  // max-heap on size, then unit order
        return tiles != o.tiles ? tiles < o.tiles : (unit != o.unit ? unit > o.unit : t0 > o.t0);
      }
    };
    std::vector<Pend> pend;
    pend.reserve(nu + grid);
    for (int ui = 0; ui < nu; ++ui) pend.push_back({units[ui].tiles, ui, 0});
    std::make_heap(pend.begin(), pend.end());
    std::vector<char> cut(nu, 0);
    while (!pend.empty()) {
      std::pop_heap(pend.begin(), pend.end());
      Pend pc = pend.back();
      pend.pop_back();
      std::pop_heap(heap.begin(), heap.end(), cmin);
      LoadCta& lc = heap.back();
      int take = std::min(pc.tiles, hard_cap);
      if (lc.first + take + kItem + (cut[pc.unit] ? kSplit : 0.0) > budget) {
        const int fit = static_cast<int>(budget - lc.first - kItem - kSplit);
        if (fit >= min_split_tiles && pc.tiles - fit >= min_split_tiles) take = std::min(fit, take);
      }
      if (take < pc.tiles) cut[pc.unit] = 1;
      pb.push_back({pc.unit, pc.t0, take, lc.second});
      lc.first += take + kItem + (cut[pc.unit] ? kSplit : 0.0);
      std::push_heap(heap.begin(), heap.end(), cmin);
      if (take < pc.tiles) {
        pend.push_back({pc.tiles - take, pc.unit, pc.t0 + take});
        std::push_heap(pend.begin(), pend.end());
      }
    }
    // a unit's first piece was charged before it was known to be cut
    std::vector<double> loads(grid, 0.0);
    for (const Piece& pc : pb) loads[pc.cta] += pc.nt + kItem + (cut[pc.unit] ? kSplit : 0.0);
    for (double l : loads) span_b = std::max(span_b, l);
  }

  // ---- candidate C: one flat stream.  The units' tiles, in unit order, are cut into
  // grid equal contiguous ranges (one per CTA), so every CTA streams the same number
  // of tiles and a unit is cut only where a range ends (few units split, each at most
  // into ceil(tiles / range) + 1 pieces).  A boundary that would leave a piece under
  // min_split_tiles moves to the unit's end.
  std::vector<Piece> pc_;
  double span_c = 1e300;
  if (!a_good) {
    long long total = 0;
    for (const Unit& u : units) total += u.tiles;
    const long long E = std::max<long long>(1, (total + grid - 1) / grid);
    pc_.reserve(nu + 2 * grid + 16);
    std::vector<double> loads(grid, 0.0);
    std::vector<char> cutc(nu, 0);
    int cta = 0;
    long long room = E;  // tiles left in the current CTA's range
    for (int ui = 0; ui < nu; ++ui) {
      int t0 = 0, left = units[ui].tiles;
      while (left > 0) {
        if (room <= 0 && cta + 1 < grid) {
          ++cta;
          room = E;
        }
        const long long here = cta == grid - 1 ? static_cast<long long>(left) : std::max<long long>(room, 1);
        int take = static_cast<int>(std::min<long long>(left, here));
        take = std::min(take, hard_cap);
        if (left - take > 0 && left - take < min_split_tiles) take = std::min(left, hard_cap);  // no sliver
        if (take < min_split_tiles && left > take && cta + 1 < grid) {  // sliver at the range end: next CTA
          ++cta;
          room = E;
          continue;
        }
        if (take < units[ui].tiles) cutc[ui] = 1;
        pc_.push_back({ui, t0, take, cta});
        t0 += take;
        left -= take;
        room -= take;
      }
    }
    for (const Piece& x : pc_) loads[x.cta] += x.nt + kItem + (cutc[x.unit] ? kSplit : 0.0);
    span_c = 0;
    for (double l : loads) span_c = std::max(span_c, l);
  }

  // ---- candidate D: halve the giants.  Only the units costlier than the mean CTA load
  // are cut, into the fewest equal pieces that fit it; then LPT over pieces and whole
  // units alike.  (B cuts whatever overflows as it places, which scatters small pieces
  // over many CTAs; D leaves every other unit whole.)
  std::vector<Piece> pd;
  double span_d = 1e300;
  if (!a_good) {
    struct Job {
      double cost;
      int unit, t0, nt;
      bool cut;
    };
    std::vector<Job> jobs;
    jobs.reserve(nu + 2 * grid);
    for (int ui : order) {
      const int tiles = units[ui].tiles;
      int k = std::max(1, (tiles + hard_cap - 1) / hard_cap);
      if (tiles + kItem > lb && tiles >= 2 * min_split_tiles)
        k = std::max(k, std::min(tiles / min_split_tiles, static_cast<int>(std::ceil((tiles + kItem) / lb))));
      const int base = tiles / k, rem = tiles % k;
      int t0 = 0;
      for (int q = 0; q < k; ++q) {
        const int nt = base + (q < rem ? 1 : 0);
        jobs.push_back({nt + kItem + (k > 1 ? kSplit : 0.0), ui, t0, nt, k > 1});
        t0 += nt;
      }
    }
    std::stable_sort(jobs.begin(), jobs.end(), [](const Job& a, const Job& b) { return a.cost > b.cost; });
    typedef std::pair<double, int> LoadCta;
    std::vector<LoadCta> heap;
    heap.reserve(grid);
    for (int c = 0; c < grid; ++c) heap.push_back(LoadCta(0.0, c));
    auto cmp = [](const LoadCta& a, const LoadCta& b) { return a > b; };
    pd.reserve(jobs.size());
    span_d = 0;
    for (const Job& j : jobs) {
      std::pop_heap(heap.begin(), heap.end(), cmp);
      LoadCta& lc = heap.back();
      pd.push_back({j.unit, j.t0, j.nt, lc.second});
      lc.first += j.cost;
      span_d = std::max(span_d, lc.first);
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
  }

  // Prefer whole units unless cutting buys >3% of the makespan, net of the split
  // combine launch and partial traffic it brings (kCombine, measured).
  int which = 0;  // 0 whole, 1 LPT-cut, 2 flat, 3 giants halved
  double span_cut = span_b;
  which = 1;
  if (span_c < span_cut) span_cut = span_c, which = 2;
  if (span_d < span_cut) span_cut = span_d, which = 3;
  const std::vector<Piece>* cand[4] = {&pa, &pb, &pc_, &pd};
  if (!(span_cut + kCombine < 0.97 * span_a) || static_cast<int>(cand[which]->size()) > max_work) which = 0;
  if (const char* f = std::getenv("OPTIMUS_PLAN_FORCE")) {  // diagnostics: whole | cut | flat | giants
    which = std::strcmp(f, "cut") == 0 ? 1 : std::strcmp(f, "flat") == 0 ? 2 : std::strcmp(f, "giants") == 0 ? 3 : 0;
    if (cand[which]->empty() || static_cast<int>(cand[which]->size()) > max_work) which = 0;
  }
  const std::vector<Piece>& P = *cand[which];
  if (static_cast<int>(P.size()) > max_work) return fail("attn_plan: work buffer too small");
  if (std::getenv("OPTIMUS_PLAN_DEBUG"))
    std::fprintf(stderr, "attn_plan: whole-unit LPT span %.1f (%zu items), cutting LPT %.1f (%zu items), "
                 "flat %.1f (%zu items), giants %.1f (%zu items) -> %d\n", span_a, pa.size(), span_b, pb.size(),
                 span_c, pc_.size(), span_d, pd.size(), which);
  // Split groups: the pieces of a unit, in key order, get consecutive partial slots.
  std::vector<int> byu(P.size());
  for (size_t x = 0; x < P.size(); ++x) byu[x] = static_cast<int>(x);
  std::sort(byu.begin(), byu.end(), [&](int a, int b) {
    return P[a].unit != P[b].unit ? P[a].unit < P[b].unit : P[a].t0 < P[b].t0;
  });
  std::vector<int> slot(P.size(), -1);
  int n_groups = 0, n_partials = 0;
  for (size_t i = 0; i < byu.size();) {
    size_t k = i + 1;
    while (k < byu.size() && P[byu[k]].unit == P[byu[i]].unit) ++k;
    if (k - i > 1) {
      if (n_groups >= max_groups) return fail("attn_plan: groups buffer too small");
      const Unit& u = units[P[byu[i]].unit];
      int32_t* g = groups + 8 * n_groups++;
      g[0] = u.req;
      g[1] = u.head;
      g[2] = u.tok_begin;
      g[3] = u.n_tok;
      g[4] = n_partials;
      g[5] = static_cast<int>(k - i);
      g[6] = 0;
      g[7] = 0;
      for (size_t x = i; x < k; ++x) slot[byu[x]] = n_partials++;
    }
    i = k;
  }
  // Work list in CTA order (stable: a CTA runs its pieces in placement order).
  std::vector<int> cnt(grid + 1, 0);
  for (const Piece& pc : P) ++cnt[pc.cta + 1];
  for (int c = 0; c < grid; ++c) cnt[c + 1] += cnt[c];
  for (int c = 0; c <= grid; ++c) cta_off[c] = cnt[c];
  for (size_t x = 0; x < P.size(); ++x) {
    const Piece& pc = P[x];
    const Unit& u = units[pc.unit];
    int32_t* w = work + 8 * cnt[pc.cta]++;
    w[0] = u.req;
    w[1] = u.head;
    w[2] = u.tok_begin;
    w[3] = u.n_tok;
    w[4] = pc.t0 * 64;
    w[5] = std::min(key_end[u.req], (pc.t0 + pc.nt) * 64);
    w[6] = slot[x];
    w[7] = 0;
  }
  *n_groups_out = n_groups;
  *n_partials_out = n_partials;
  return static_cast<int>(P.size());
}

}  // extern "C"

// Shared body of optimus_paged_attn and optimus_paged_attn_append (k_new == nullptr:
// attention only).
static int paged_attn_impl(const void* q, int64_t q_stride_tok, int n_tok_total, const void* k_cache,
                           const void* v_cache, int64_t num_pages, const int32_t* q_pos,
                           const int32_t* prompt_len, const int32_t* vis_base, const int32_t* vis_off,
                           const uint32_t* vis_words, const int32_t* block_tables, int max_pages,
                           const int32_t* work, const int32_t* cta_off, int grid,
                           const int32_t* groups, int n_groups, int block_size, int hq, int hkv,
                           int head_dim, int page_size, float sm_scale, void* out,
                           int64_t out_stride_tok, float* ws_o, float* ws_ml, int v_dtype,
                           const void* k_new, const void* v_new, int64_t new_stride_tok,
                           int64_t* slot_out, const int32_t* slot_abs, void* stream) {
  if (v_dtype != 0 && v_dtype != 1) return fail("paged_attn: v_dtype must be 0 (bf16) or 1 (fp16)");
  if (head_dim != 64 && head_dim != 128) return fail("paged_attn: head_dim must be 64 or 128");
  if (hkv < 1 || hq % hkv) return fail("paged_attn: Hq must be a multiple of Hkv");
  const int G = hq / hkv;
  if (G > 128) return fail("paged_attn: group size > 128");
  if (!page_ok(page_size))
    return fail("paged_attn: page_size must be a power of two in [8, 1024]");
  if (block_size < 1) return fail("paged_attn: block_size must be >= 1");
  if (q_stride_tok % 8 || q_stride_tok < static_cast<int64_t>(hq) * head_dim)
    return fail("paged_attn: q_stride_tok must be >= Hq*head_dim and a multiple of 8");
  if (out_stride_tok % 8 || out_stride_tok < static_cast<int64_t>(hq) * head_dim)
    return fail("paged_attn: out_stride_tok must be >= Hq*head_dim and a multiple of 8");
  if (grid < 0 || n_groups < 0 || num_pages < 1 || max_pages < 1)
    return fail("paged_attn: bad sizes");
  if (n_tok_total == 0 || grid == 0) return 0;
  if (n_groups > 0 && (!ws_o || !ws_ml)) return fail("paged_attn: split-KV needs a workspace");
  if (reinterpret_cast<uintptr_t>(q) % 16 || reinterpret_cast<uintptr_t>(k_cache) % 16 ||
      reinterpret_cast<uintptr_t>(v_cache) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
    return fail("paged_attn: tensors must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(work) % 16) return fail("paged_attn: work list must be 16-byte aligned");
  if (int st = check_device()) return st;
  const int T = 128 / G;
  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[4] = {static_cast<uint64_t>(head_dim), static_cast<uint64_t>(G),
                              static_cast<uint64_t>(hkv), static_cast<uint64_t>(n_tok_total)};
    const uint64_t strides[3] = {static_cast<uint64_t>(head_dim) * 2,
                                 static_cast<uint64_t>(G) * head_dim * 2,
                                 static_cast<uint64_t>(q_stride_tok) * 2};
    const uint32_t box[4] = {64, static_cast<uint32_t>(G), 1, static_cast<uint32_t>(T)};
    if (int st = get_map(q, dims, strides, box, &tq)) return st;
  }
  const int box_rows = std::min(page_size, 64);
  {
    const uint64_t dims[4] = {static_cast<uint64_t>(head_dim), static_cast<uint64_t>(page_size),
                              static_cast<uint64_t>(hkv), static_cast<uint64_t>(num_pages)};
    const uint64_t strides[3] = {static_cast<uint64_t>(head_dim) * 2,
                                 static_cast<uint64_t>(page_size) * head_dim * 2,
                                 static_cast<uint64_t>(hkv) * page_size * head_dim * 2};
    const uint32_t box[4] = {64, static_cast<uint32_t>(box_rows), 1, 1};
    if (int st = get_map(k_cache, dims, strides, box, &tk)) return st;
    if (int st = get_map(v_cache, dims, strides, box, &tv, v_dtype == 1)) return st;
  }
  if (k_new != nullptr) {
    if (!v_new) return fail("paged_attn_append: v_new is null");
    if (new_stride_tok % 8 || new_stride_tok < static_cast<int64_t>(hkv) * head_dim)
      return fail("paged_attn_append: new_stride_tok must be >= Hkv*head_dim and a multiple of 8");
    if (reinterpret_cast<uintptr_t>(k_new) % 16 || reinterpret_cast<uintptr_t>(v_new) % 16)
      return fail("paged_attn_append: k_new / v_new must be 16-byte aligned");
  }
  AttnParams prm{};
  prm.k_new = k_new;
  prm.v_new = v_new;
  prm.new_stride_tok = new_stride_tok;
  prm.slot_out = slot_out;
  prm.slot_abs = slot_abs;
  prm.num_kv_heads = hkv;
  prm.v_fp16 = v_dtype == 1;
  prm.k_cache_w = const_cast<void*>(k_cache);
  prm.v_cache_w = const_cast<void*>(v_cache);
  prm.q_pos = q_pos;
  prm.prompt_len = prompt_len;
  prm.vis_base = vis_base;
  prm.vis_off = vis_off;
  prm.vis_words = vis_words;
  prm.block_tables = block_tables;
  prm.work = work;
  prm.cta_off = cta_off;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.out_stride_tok = out_stride_tok;
  prm.ws_o = ws_o;
  prm.ws_ml = ws_ml;
  prm.max_pages = max_pages;
  prm.block_size = block_size;
  prm.num_q_heads = hq;
  prm.group = G;
  prm.tok_per_tile = T;
  prm.page_size = page_size;
  prm.page_shift = __builtin_ctz(static_cast<unsigned>(page_size));
  prm.box_rows = box_rows;
  prm.scale_log2 = sm_scale * 1.4426950408889634f;
  prm.trace = g_trace;
  {
    const char* e = getenv("OPTIMUS_DBG");
    prm.dbg = e ? atoi(e) : 0;
  }
  return cuda_status(launch_paged_attn(head_dim, v_dtype == 1, tq, tk, tv, prm, grid, groups,
                                       n_groups, static_cast<cudaStream_t>(stream)),
                     "paged_attn");
}

extern "C" {

int optimus_paged_attn(const void* q, int64_t q_stride_tok, int n_tok_total, const void* k_cache,
                       const void* v_cache, int64_t num_pages, const int32_t* q_pos,
                       const int32_t* prompt_len, const int32_t* vis_base, const int32_t* vis_off,
                       const uint32_t* vis_words, const int32_t* block_tables, int max_pages,
                       const int32_t* work, const int32_t* cta_off, int grid,
                       const int32_t* groups, int n_groups, int block_size, int hq, int hkv,
                       int head_dim, int page_size, float sm_scale, void* out,
                       int64_t out_stride_tok, float* ws_o, float* ws_ml, int v_dtype,
                       void* stream) {
  return paged_attn_impl(q, q_stride_tok, n_tok_total, k_cache, v_cache, num_pages, q_pos, prompt_len,
                         vis_base, vis_off, vis_words, block_tables, max_pages, work, cta_off, grid,
                         groups, n_groups, block_size, hq, hkv, head_dim, page_size, sm_scale, out,
                         out_stride_tok, ws_o, ws_ml, v_dtype, nullptr, nullptr, 0, nullptr, nullptr,
                         stream);
}

// Split-KV combine for a device-planned step: the group count is read from
// n_groups_dev (optimus_device_attn_plan's counts[1]); max_groups bounds the grid.
int optimus_paged_attn_combine_dev(const int32_t* groups, const int32_t* n_groups_dev, int max_groups,
                                   const float* ws_o, const float* ws_ml, int hq, int hkv, int head_dim,
                                   void* out, int64_t out_stride_tok, void* stream) {
  if (head_dim != 64 && head_dim != 128) return fail("paged_attn_combine_dev: head_dim must be 64 or 128");
  if (hkv < 1 || hq % hkv || hq / hkv > 128) return fail("paged_attn_combine_dev: bad head counts");
  if (max_groups < 0 || !n_groups_dev) return fail("paged_attn_combine_dev: bad group capacity");
  if (max_groups == 0) return 0;
  if (!ws_o || !ws_ml) return fail("paged_attn_combine_dev: split-KV needs a workspace");
  optimus::AttnParams prm = {};
  prm.ws_o = const_cast<float*>(ws_o);
  prm.ws_ml = const_cast<float*>(ws_ml);
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.out_stride_tok = out_stride_tok;
  prm.group = hq / hkv;
  return cuda_status(optimus::launch_attn_combine_dev(head_dim, prm, groups, max_groups, n_groups_dev,
                                                      static_cast<cudaStream_t>(stream)),
                     "paged_attn_combine_dev");
}

int optimus_paged_attn_append(const void* q, int64_t q_stride_tok, int n_tok_total,
                              const void* k_new, const void* v_new, int64_t new_stride_tok,
                              void* k_cache, void* v_cache, int64_t num_pages,
                              const int32_t* q_pos, const int32_t* prompt_len,
                              const int32_t* vis_base, const int32_t* vis_off,
                              const uint32_t* vis_words, const int32_t* block_tables,
                              int max_pages, const int32_t* work, const int32_t* cta_off, int grid,
                              const int32_t* groups, int n_groups, int block_size, int hq, int hkv,
                              int head_dim, int page_size, float sm_scale, void* out,
                              int64_t out_stride_tok, float* ws_o, float* ws_ml, int v_dtype,
                              int64_t* slot_mapping_out, const int32_t* slot_abs, void* stream) {
  if (!k_new) return fail("paged_attn_append: k_new is null");
  return paged_attn_impl(q, q_stride_tok, n_tok_total, k_cache, v_cache, num_pages, q_pos, prompt_len,
                         vis_base, vis_off, vis_words, block_tables, max_pages, work, cta_off, grid,
                         groups, n_groups, block_size, hq, hkv, head_dim, page_size, sm_scale, out,
                         out_stride_tok, ws_o, ws_ml, v_dtype, k_new, v_new, new_stride_tok,
                         slot_mapping_out, slot_abs, stream);
}

int optimus_attn_layers(int n_layers, const void* const* q, const void* const* k_new,
                        const void* const* v_new, int64_t q_stride_tok, int64_t new_stride_tok,
                        int n_tok_total, int n_tok, void* const* k_cache, void* const* v_cache,
                        int64_t num_pages, const int32_t* tok_req, const int32_t* q_pos,
                        const int32_t* prompt_len, const int32_t* vis_base,
                        const int32_t* vis_off, const uint32_t* vis_words,
                        const int32_t* block_tables, int max_pages, const int32_t* work,
                        const int32_t* cta_off, int grid, const int32_t* groups, int n_groups,
                        int block_size, int hq, int hkv, int head_dim, int page_size,
                        float sm_scale, void* const* out, int64_t out_stride_tok, float* ws_o,
                        float* ws_ml, int v_dtype, int append_mode, int32_t* slot_ws,
                        void* stream) {
  if (n_layers < 0 || !q || !k_new || !v_new || !k_cache || !v_cache || !out)
    return fail("attn_layers: bad layer arrays");
  if (append_mode < 0 || append_mode > 2) return fail("attn_layers: append_mode must be 0, 1 or 2");
  if (append_mode != 0 && slot_ws == nullptr) return fail("attn_layers: append_mode 1/2 needs slot_ws");
  if (append_mode != 0 && n_tok > 0) {
    // the step's slot map once (rule S), shared by every layer's append
    const int st = optimus_slot_mapping(tok_req, q_pos, prompt_len, block_tables, max_pages, n_tok,
                                        page_size, slot_ws, stream);
    if (st) return st;
  }
  for (int l = 0; l < n_layers; ++l) {
    if (append_mode == 1) {
      int st = cuda_status(launch_kv_append_slots(k_new[l], v_new[l], new_stride_tok, slot_ws, n_tok,
                                                  hkv, head_dim, page_size, k_cache[l], v_cache[l],
                                                  v_dtype == 1, static_cast<cudaStream_t>(stream)),
                           "kv_append_slots");
      if (st) return st;
      st = optimus_paged_attn(q[l], q_stride_tok, n_tok_total, k_cache[l], v_cache[l], num_pages, q_pos,
                              prompt_len, vis_base, vis_off, vis_words, block_tables, max_pages, work,
                              cta_off, grid, groups, n_groups, block_size, hq, hkv, head_dim,
                              page_size, sm_scale, out[l], out_stride_tok, ws_o, ws_ml, v_dtype, stream);
      if (st) return st;
      continue;
    }
    if (append_mode == 2) {
      // K1 folded into K2 (caller guarantees one query tile per (request, KV head))
      const int st = optimus_paged_attn_append(
          q[l], q_stride_tok, n_tok_total, k_new[l], v_new[l], new_stride_tok, k_cache[l], v_cache[l],
          num_pages, q_pos, prompt_len, vis_base, vis_off, vis_words, block_tables, max_pages, work,
          cta_off, grid, groups, n_groups, block_size, hq, hkv, head_dim, page_size, sm_scale, out[l],
          out_stride_tok, ws_o, ws_ml, v_dtype, nullptr, slot_ws, stream);
      if (st) return st;
      continue;
    }
    int st = optimus_kv_append(k_new[l], v_new[l], new_stride_tok, tok_req, q_pos, prompt_len,
                               block_tables, max_pages, n_tok, hkv, head_dim, page_size,
                               k_cache[l], v_cache[l], num_pages, nullptr, v_dtype, stream);
    if (st) return st;
    st = optimus_paged_attn(q[l], q_stride_tok, n_tok_total, k_cache[l], v_cache[l], num_pages, q_pos,
                            prompt_len, vis_base, vis_off, vis_words, block_tables, max_pages, work,
                            cta_off, grid, groups, n_groups, block_size, hq, hkv, head_dim,
                            page_size, sm_scale, out[l], out_stride_tok, ws_o, ws_ml, v_dtype, stream);
    if (st) return st;
  }
  return 0;
}

int optimus_unmask_splits(int n_rows, int vocab) {
  if (n_rows <= 0 || vocab <= 0) return 1;
  // Measured table (tools/k3_sweep.py --splits, profiles/r2h_k3_splits*.txt: fused K3 on
  // B200 over 32..2,100 rows x 151,936 bf16, every split count timed in one process; the
  // 2-split band re-measured up to 1,550 rows, profiles/r2d2_k3_splits_pipes.txt, "pipe 0":
  // 1,300 / 1,400 / 1,500 rows 72.7 / 76.0 / 82.0 us with 2 splits against 77.3 / 79.7 /
  // 83.3 with 1).  Rows are scaled to that vocabulary so the table is in CTA bytes.  Few
  // large CTAs win once the grid fills the machine; small batches need slices to reach
  // every SM.
  const double eq = static_cast<double>(n_rows) * vocab / 151936.0;
  int s = eq < 64 ? 8 : eq < 256 ? 4 : eq < 400 ? 2 : eq < 650 ? 3 : eq < 1550 ? 2 : 1;
  s = std::min(s, std::max(1, vocab / 8192));
  return s;
}

int optimus_v_saturated(int32_t* out, int reset, void* stream) {
  if (!out) return fail("v_saturated: null pointer");
  if (int st = check_device()) return st;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  int st = cuda_status(v_saturated_k1(out, reset, s), "v_saturated");
  if (st) return st;
  return cuda_status(v_saturated_k2(out + 1, reset, s), "v_saturated");
}

int optimus_unmask_commit(const void* logits, int logits_dtype, int64_t row_stride, const int32_t* row_src,
                          int n_rows, const int32_t* n_rows_dev, int vocab, int n_vsplit, float* part,
                          const int32_t* cu_rows, const int32_t* row_req, int n_req, int32_t* counters, float tau,
                          int fallback_mode, uint8_t* commit_mask, int32_t* tok, float* conf,
                          const int32_t* row_pos, uint8_t* state, int32_t* token_buf, int64_t state_stride,
                          void* stream) {
  if (logits_dtype != 0 && logits_dtype != 1) return fail("unmask_commit: logits_dtype must be 0 or 1");
  const int vec = logits_dtype == 0 ? 8 : 4;
  if (vocab < 1 || vocab % vec) return fail("unmask_commit: vocab must be a multiple of 8 (bf16) / 4 (fp32)");
  if (row_stride % vec || row_stride < vocab) return fail("unmask_commit: bad row_stride");
  if (n_rows < 0 || n_vsplit < 1 || n_req < 0) return fail("unmask_commit: bad sizes");
  if (fallback_mode < 0 || fallback_mode > 2) return fail("unmask_commit: fallback_mode must be 0, 1 or 2");
  if (n_rows == 0) return 0;
  if (!logits || !part || !cu_rows || !row_req || !counters || !commit_mask || !tok || !conf)
    return fail("unmask_commit: null pointer");
  if ((state || token_buf) && !row_pos) return fail("unmask_commit: state / token update needs row_pos");
  if (reinterpret_cast<uintptr_t>(logits) % 16) return fail("unmask_commit: logits must be 16-byte aligned");
  if (int st = check_device()) return st;
  return cuda_status(launch_unmask_commit(logits, logits_dtype, row_stride, row_src, n_rows, n_rows_dev, vocab,
                                          n_vsplit, part, cu_rows, row_req, counters, tau, fallback_mode,
                                          commit_mask, tok, conf, row_pos, state, token_buf, state_stride,
                                          static_cast<cudaStream_t>(stream)),
                     "unmask_commit");
}

int optimus_unmask_partials(const void* logits, int logits_dtype, int64_t row_stride,
                            const int32_t* row_src, int n_rows, int vocab, int vocab_offset,
                            int n_vsplit, float* part, void* stream) {
  if (logits_dtype != 0 && logits_dtype != 1) return fail("unmask: logits_dtype must be 0 or 1");
  const int vec = logits_dtype == 0 ? 8 : 4;
  if (vocab < 1 || vocab % vec) return fail("unmask: vocab must be a multiple of 8 (bf16) / 4 (fp32)");
  if (row_stride % vec || row_stride < vocab) return fail("unmask: bad row_stride");
  if (n_rows < 0 || n_vsplit < 1) return fail("unmask: bad sizes");
  if (n_rows == 0) return 0;
  if (!logits || !part) return fail("unmask: null pointer");
  if (reinterpret_cast<uintptr_t>(logits) % 16) return fail("unmask: logits must be 16-byte aligned");
  if (int st = check_device()) return st;
  return cuda_status(launch_unmask_partials(logits, logits_dtype, row_stride, row_src, n_rows,
                                            vocab, vocab_offset, n_vsplit, part,
                                            static_cast<cudaStream_t>(stream)),
                     "unmask_partials");
}

int optimus_unmask_finalize(const float* part, int n_outer, int n_rows, int n_vsplit,
                            const int32_t* cu_rows, int n_req, float tau, int fallback_mode,
                            uint8_t* commit_mask, int32_t* tok, float* conf,
                            const int32_t* row_pos, uint8_t* state, int32_t* token_buf,
                            int64_t state_stride, void* stream) {
  if (n_outer < 1 || n_rows < 0 || n_vsplit < 1 || n_req < 0) return fail("unmask: bad sizes");
  if (fallback_mode < 0 || fallback_mode > 2) return fail("unmask: fallback_mode must be 0, 1 or 2");
  if (n_req == 0) return 0;
  if (!part || !cu_rows || !commit_mask || !tok || !conf) return fail("unmask: null pointer");
  if ((state || token_buf) && !row_pos) return fail("unmask: state / token update needs row_pos");
  if (int st = check_device()) return st;
  return cuda_status(
      launch_unmask_finalize(part, n_outer, n_rows, n_vsplit, cu_rows, n_req, tau, fallback_mode,
                             commit_mask, tok, conf, row_pos, state, token_buf, state_stride,
                             static_cast<cudaStream_t>(stream)),
      "unmask_finalize");
}

}  // extern "C"
