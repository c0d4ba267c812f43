// device_step.cu — the control half of the streaming decode step on the device
// (device half).
//
// optimus_device_plan / optimus_device_apply are the device twins of
// optimus_host_plan / optimus_host_apply (host_step.cu), which mirror the
// reference's plan_chunk (engine.py:45-67) and apply_chunk + advance_blocks
// (engine.py:79-95, core.py:109-116) batch-wide.  Same packed per-slot state (now
// device-resident), same step metadata out, bit for bit
// (tests/test_device_step_gpu.py): with them the plan -> K1/K2 -> K3 -> apply loop
// needs no host round trip, which is what a graph-captured step requires.
//
// Plan: one CTA of 32 warps; warp w plans requests w, w+32, ...  Pass 1 selects each
// request's kv positions (FIFO front of the uncached ring) and window (earliest
// MASKED of the current block, or anywhere capped at the block for OUT_BLOCK) with
// warp ballots in position order, and derives key_end / vis_base from a per-warp
// "planned" bitmap in shared memory; a block scan turns the counts into offsets;
// pass 2 writes the query / row layouts, the rule-V visibility words and the
// gathered block-table rows.
// Apply: one warp per request.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "ptx.cuh"
#include "../../include/optimus_b200.h"

namespace optimus {
namespace dstep {

constexpr int8_t MASKED = 0, UNCACHED = 1, CACHED = 2;
constexpr int kWarps = 32;
constexpr int kMaxOut = 4096;          // planned bitmap capacity per warp (positions)
constexpr int kMaxReq = 256;           // requests per step (the reference's max_batch, sim.py:62)

// Exclusive prefix sum over a 1024-thread block's values (warp shuffles, then one
// warp over the 32 warp totals); *total = the sum.  All threads must call it.
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* ws, unsigned* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  const unsigned pre = (warp ? ws[warp - 1] : 0u) + x - v;
  *total = ws[31];
  __syncthreads();  // ws is reused by the next call
  return pre;
}
constexpr int kMaxChunk = 128;

struct PlanArgs {
  int n;
  const int32_t* slots;
  int chunk;
  const int32_t* chunk_per_req;
  int block, window_rule;
  const int8_t* states;
  int64_t stride;
  const int32_t* queue;
  int qcap;
  const int32_t* q_head;
  const int32_t* q_len;
  const int32_t* block_index;
  const int32_t* cached_prefix;
  const int32_t* prompt;
  const int32_t* out_len;
  const int32_t* block_tables;
  int max_pages;
  int32_t* cu_seqlens;
  int32_t* tok_req;
  int32_t* tok_pos;
  int cap_tok;
  int32_t* prompt_len;
  int32_t* key_end;
  int32_t* vis_base;
  int32_t* vis_off;
  uint32_t* vis_words;
  int cap_words;
  int32_t* cu_rows;
  int32_t* row_tok;
  int32_t* row_pos;
  int32_t* row_req;
  int cap_rows;
  int32_t* block_tables_out;
  int32_t* counts;  // {n_tok, n_rows, n_words, status}
};

__device__ __forceinline__ bool planned_bit(const uint32_t* bm, int p) { return (bm[p >> 5] >> (p & 31)) & 1u; }

// Copy a request's state row (out positions, int8) into the warp's shared-memory slot:
// one round trip of independent 16-byte loads (rows padded to 16 bytes, BatchState)
// instead of a dependent global load per 32 positions in every scan below.
__device__ __forceinline__ const int8_t* stage_row(int8_t* dst, const int8_t* src, int64_t stride, int out,
                                                   int lane) {
  if ((stride & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int nv = (out + 15) >> 4;  // <= stride / 16: the tail bytes are the row's padding
    for (int i = lane; i < nv; i += 32) reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  } else {
    for (int i = lane; i < out; i += 32) dst[i] = src[i];
  }
  __syncwarp();
  return dst;
}

__global__ void __launch_bounds__(kWarps * 32, 1) plan_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) int8_t stage_sm[];  // [kWarps][kMaxOut]: the warp's staged state row
  __shared__ uint32_t bitmap[kWarps][kMaxOut / 32];
  __shared__ int ntok_s[kMaxReq], nrow_s[kMaxReq], nword_s[kMaxReq], nkv_s[kMaxReq];
  __shared__ int ke_s[kMaxReq], vb_s[kMaxReq];
  __shared__ int bad;
  __shared__ unsigned scan_ws[32];
  // per-request scalars, loaded once for the whole batch (two parallel round trips)
  // instead of a dependent chain of global loads inside each warp's request loop
  __shared__ int sl_s[kMaxReq], out_s[kMaxReq], ch_s[kMaxReq], bi_s[kMaxReq], qh_s[kMaxReq], ql_s[kMaxReq];
  __shared__ int cp_s[kMaxReq], pr_s[kMaxReq], t0_s[kMaxReq], r0_s[kMaxReq], vo_s[kMaxReq];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) bad = 0;
  if (threadIdx.x < a.n) {
    const int r = threadIdx.x;
    const int s = a.slots[r];
    sl_s[r] = s;
    ch_s[r] = a.chunk_per_req ? a.chunk_per_req[r] : a.chunk;
    out_s[r] = a.out_len[s];
    bi_s[r] = a.block_index[s];
    qh_s[r] = a.q_head[s];
    ql_s[r] = a.q_len[s];
    cp_s[r] = a.cached_prefix[s];
    pr_s[r] = a.prompt[s];
  }
  __syncthreads();
  uint32_t* bm = bitmap[warp];
  // ---- pass 1: counts, key_end, vis_base
  for (int r = warp; r < a.n; r += kWarps) {
    const int s = sl_s[r];
    const int out = out_s[r];
    const int chunk_r = ch_s[r];
    if (chunk_r < 2 || chunk_r > kMaxChunk || out > kMaxOut) {
      if (lane == 0) bad = 1;
      continue;
    }
    const int8_t* st = stage_row(stage_sm + warp * kMaxOut, a.states + static_cast<int64_t>(s) * a.stride, a.stride,
                                 out, lane);
    // finished (no MASKED left in the current block, advance_blocks' invariant): nothing
    bool done;
    {
      const int b0 = bi_s[r] * a.block, b1 = min(b0 + a.block, out);
      bool any = false;
      for (int base = b0; base < b1; base += 32)
        any = any || __any_sync(0xFFFFFFFFu, base + lane < b1 && st[base + lane] == MASKED);
      done = !any;
    }
    const int nkv = done ? 0 : min(ql_s[r], chunk_r);
    int room = done ? 0 : chunk_r - nkv;
    int lo = bi_s[r] * a.block;
    int hi = min(lo + a.block, out);
    if (a.window_rule == 1) {
      hi = out;
      room = min(room, a.block);
    }
    for (int w = lane; w < (out + 31) / 32; w += 32) bm[w] = 0;
    __syncwarp();
    // kv positions: the FIFO front of the uncached ring
    int maxq = -1;
    for (int i = lane; i < nkv; i += 32) {
      const int p = a.queue[static_cast<int64_t>(s) * a.qcap + (qh_s[r] + i) % a.qcap];
      atomicOr(&bm[p >> 5], 1u << (p & 31));
      maxq = max(maxq, p);
    }
    // window: earliest MASKED in [lo, hi), up to `room`, in position order
    int nwin = 0;
    for (int base = lo; base < hi && nwin < room; base += 32) {
      const int p = base + lane;
      const bool m = p < hi && st[p] == MASKED;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
      const int rank = __popc(bal & ((1u << lane) - 1u));
      if (m && nwin + rank < room) {
        atomicOr(&bm[p >> 5], 1u << (p & 31));
        maxq = max(maxq, p);
      }
      nwin = min(room, nwin + __popc(bal));
    }
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxq = max(maxq, __shfl_xor_sync(0xFFFFFFFFu, maxq, o));
    if (lane == 0) {
      ntok_s[r] = nkv + nwin;
      nrow_s[r] = nwin;
      nkv_s[r] = nkv;
    }
    if (nkv + nwin == 0) {
      if (lane == 0) {
        ke_s[r] = 0;
        vb_s[r] = 0;
        nword_s[r] = 0;
      }
      continue;
    }
    // rule V: visible = CACHED before the step, or planned now
    // cp: first position from cached_prefix on that is not visible
    int cp = min(cp_s[r], out);
    while (true) {
      const int p = cp + lane;
      const bool v = p < out && (st[p] == CACHED || planned_bit(bm, p));
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v);
      if (bal == 0xFFFFFFFFu) {
        cp += 32;
        continue;
      }
      cp += __ffs(~bal) - 1;
      break;
    }
    cp = min(cp, out);
    const int cap_end = (maxq / a.block + 1) * a.block;
    // last: the largest visible position = max(largest planned (maxq), largest CACHED);
    // the CACHED one by a backward scan of the staged row, 16 positions per lane
    int last = maxq;
    {
      const uint4* st4 = reinterpret_cast<const uint4*>(st);
      const int nvec = (out + 15) >> 4;
      for (int top = nvec - 1; top >= 0; top -= 32) {
        const int j = top - lane;
        int c = -1;
        if (j >= 0) {
          const uint4 v = st4[j];
          uint32_t m[4] = {__vcmpeq4(v.x, 0x02020202u), __vcmpeq4(v.y, 0x02020202u), __vcmpeq4(v.z, 0x02020202u),
                           __vcmpeq4(v.w, 0x02020202u)};  // CACHED == 2
          const int lim = out - 16 * j;  // positions of this vector inside the row
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int nb = lim - 4 * q;
            m[q] &= nb >= 4 ? 0xFFFFFFFFu : nb <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - nb)));
          }
#pragma unroll
          for (int q = 3; q >= 0; --q)
            if (c < 0 && m[q]) c = 16 * j + 4 * q + (31 - __clz(m[q])) / 8;
        }
        const int best = __reduce_max_sync(0xFFFFFFFFu, c);
        if (best >= 0) {
          last = max(last, best);
          break;
        }
      }
    }
    const int pr = pr_s[r];
    const int ke = pr + min(last + 1, cap_end);
    int vb = ((pr + cp) / 32) * 32;
    if (vb > ke) vb = (ke / 32) * 32;
    if (lane == 0) {
      ke_s[r] = ke;
      vb_s[r] = vb;
      nword_s[r] = ke > vb ? (ke - vb + 31) / 32 : 0;
    }
  }
  __syncthreads();
  // ---- offsets: block scans over the requests (thread r = request r, n <= 256)
  {
    const int r = threadIdx.x;
    const bool live = r < a.n;
    unsigned tt, tr, tw;
    const unsigned t_pre = block_exclusive_scan(live ? static_cast<unsigned>(ntok_s[r]) : 0u, scan_ws, &tt);
    const unsigned r_pre = block_exclusive_scan(live ? static_cast<unsigned>(nrow_s[r]) : 0u, scan_ws, &tr);
    const unsigned w_pre = block_exclusive_scan(live ? static_cast<unsigned>(nword_s[r]) : 0u, scan_ws, &tw);
    if (live) {
      a.vis_off[r] = static_cast<int>(w_pre);
      a.cu_seqlens[r + 1] = static_cast<int>(t_pre) + ntok_s[r];
      a.cu_rows[r + 1] = static_cast<int>(r_pre) + nrow_s[r];
      a.prompt_len[r] = pr_s[r];
      t0_s[r] = static_cast<int>(t_pre);
      r0_s[r] = static_cast<int>(r_pre);
      vo_s[r] = static_cast<int>(w_pre);
      a.key_end[r] = ke_s[r];
      a.vis_base[r] = vb_s[r];
    }
    if (r == 0) {
      a.cu_seqlens[0] = 0;
      a.cu_rows[0] = 0;
      a.vis_off[a.n] = static_cast<int>(tw);
      if (static_cast<int>(tt) > a.cap_tok || static_cast<int>(tr) > a.cap_rows || static_cast<int>(tw) > a.cap_words)
        bad = 1;
      a.counts[0] = static_cast<int>(tt);
      a.counts[1] = static_cast<int>(tr);
      a.counts[2] = static_cast<int>(tw);
      a.counts[3] = bad ? OPTIMUS_EINVAL : 0;
    }
  }
  __syncthreads();
  if (bad) {
    // rejected: an empty step for every consumer that reads the counts / offsets
    // (K1, K3, the work planner, apply), so a captured graph that keeps running
    // cannot act on half-written metadata; counts[3] tells the host
    for (int i = threadIdx.x; i <= a.n; i += blockDim.x) {
      a.cu_seqlens[i] = 0;
      a.cu_rows[i] = 0;
      a.vis_off[i] = 0;
    }
    if (threadIdx.x == 0) {
      a.counts[0] = 0;
      a.counts[1] = 0;
      a.counts[2] = 0;
    }
    return;
  }
  // ---- pass 2: layouts, visibility words, block tables
  for (int r = warp; r < a.n; r += kWarps) {
    const int s = sl_s[r];
    const int out = out_s[r];
    const int8_t* st = stage_row(stage_sm + warp * kMaxOut, a.states + static_cast<int64_t>(s) * a.stride, a.stride,
                                 out, lane);
    const int t0 = t0_s[r], r0 = r0_s[r];
    const int nkv = nkv_s[r], nwin = nrow_s[r];
    // rebuild the planned bitmap and window of this request (pass 1's were per warp
    // and reused by later requests of the same warp)
    for (int w = lane; w < (out + 31) / 32; w += 32) bm[w] = 0;
    __syncwarp();
    for (int i = lane; i < nkv; i += 32) {
      const int p = a.queue[static_cast<int64_t>(s) * a.qcap + (qh_s[r] + i) % a.qcap];
      a.tok_req[t0 + i] = r;
      a.tok_pos[t0 + i] = p;
      atomicOr(&bm[p >> 5], 1u << (p & 31));
    }
    {
      int room = nwin;  // pass 1's window size (0 for a finished request)
      int lo = bi_s[r] * a.block;
      int hi = min(lo + a.block, out);
      if (a.window_rule == 1) {
        hi = out;
        room = min(room, a.block);
      }
      int got = 0;
      for (int base = lo; base < hi && got < room; base += 32) {
        const int p = base + lane;
        const bool m = p < hi && st[p] == MASKED;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
        const int rank = __popc(bal & ((1u << lane) - 1u));
        if (m && got + rank < room) {
          const int k = got + rank;
          a.row_tok[r0 + k] = t0 + nkv + k;
          a.row_pos[r0 + k] = p;
          a.row_req[r0 + k] = r;
          a.tok_req[t0 + nkv + k] = r;
          a.tok_pos[t0 + nkv + k] = p;
          atomicOr(&bm[p >> 5], 1u << (p & 31));
        }
        got = min(room, got + __popc(bal));
      }
    }
    __syncwarp();
    const int pr = pr_s[r];
    const int ke = ke_s[r], vb = vb_s[r];
    const int words = nword_s[r];
    uint32_t* vw = a.vis_words + vo_s[r];
    for (int w = 0; w < words; ++w) {
      const int abs = vb + w * 32 + lane;
      const int p = abs - pr;
      const bool v = abs < ke && (p < 0 || (p < out && (st[p] == CACHED || planned_bit(bm, p))));
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v);
      if (lane == 0) vw[w] = bal;
    }
    const int32_t* src = a.block_tables + static_cast<int64_t>(s) * a.max_pages;
    int32_t* dst = a.block_tables_out + static_cast<int64_t>(r) * a.max_pages;
    for (int i = lane; i < a.max_pages; i += 32) dst[i] = src[i];
  }
}

struct ApplyArgs {
  int n;
  const int32_t* slots;
  int block;
  const int32_t* cu_seqlens;
  const int32_t* tok_pos;
  const int32_t* cu_rows;
  const int32_t* row_pos;
  const uint8_t* commit_mask;
  int8_t* states;
  int64_t stride;
  int32_t* queue;
  int qcap;
  int32_t* q_head;
  int32_t* q_len;
  int32_t* block_index;
  int32_t* committed;
  int32_t* steps;
  int32_t* cached_prefix;
  const int32_t* out_len;
  int32_t* commits_out;
  int32_t* status;
};

// Validation pass (one thread per request, no writes but *status): the KV plan pops
// the FIFO in order and every committed row is MASKED (engine.py:70-76,85-88).  The
// apply kernel runs after it on the same stream and does nothing when *status is
// set, so an illegal step leaves the whole batch unchanged (the reference checks
// before it mutates, engine.py:83).  *status is sticky: the caller zeroes it (the
// device loop shares it with the plan's counts[3], so a rejected plan skips apply).
__global__ void __launch_bounds__(128) apply_validate_kernel(const ApplyArgs a) {
  // one warp per request: the lanes check the FIFO front and the committed rows in
  // parallel (no dependent load chain per entry)
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= a.n) return;
  const int s = a.slots[r];
  const int out = a.out_len[s];
  if (a.committed[s] >= out) return;
  const int8_t* st = a.states + static_cast<int64_t>(s) * a.stride;
  const int32_t* q = a.queue + static_cast<int64_t>(s) * a.qcap;
  const int t0 = a.cu_seqlens[r], r0 = a.cu_rows[r], r1 = a.cu_rows[r + 1];
  const int nkv = (a.cu_seqlens[r + 1] - t0) - (r1 - r0);
  const int head = a.q_head[s], len = a.q_len[s];
  bool ok = nkv >= 0 && nkv <= len;
  if (ok)
    for (int i = lane; i < nkv; i += 32) ok = ok && q[(head + i) % a.qcap] == a.tok_pos[t0 + i];
  int k = 0;
  for (int i = r0 + lane; i < r1; i += 32) {
    if (!a.commit_mask[i]) continue;
    const int p = a.row_pos[i];
    ok = ok && p >= 0 && p < out && st[p] == MASKED;
    ++k;
  }
  ok = __all_sync(0xFFFFFFFFu, ok);
  k = __reduce_add_sync(0xFFFFFFFFu, k);
  if (lane == 0 && (!ok || len - nkv + k > a.qcap)) *a.status = OPTIMUS_EINVAL;
}

// One warp per request: the KV plan's positions become CACHED and the commits (in
// row order) are pushed onto the FIFO by all lanes at once; lane 0 updates the scalars.
__global__ void __launch_bounds__(128) apply_kernel(const ApplyArgs a) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= a.n || *a.status != 0) return;
  const int s = a.slots[r];
  int8_t* st = a.states + static_cast<int64_t>(s) * a.stride;
  int32_t* q = a.queue + static_cast<int64_t>(s) * a.qcap;
  const int out = a.out_len[s];
  if (a.committed[s] >= out) {  // finished: not stepped (sim.py:307-313)
    if (lane == 0) a.commits_out[r] = 0;
    return;
  }
  {  // validated: pop the KV plan, push the commits
    const int t0 = a.cu_seqlens[r], r0 = a.cu_rows[r], r1 = a.cu_rows[r + 1];
    const int nkv = (a.cu_seqlens[r + 1] - t0) - (r1 - r0);
    for (int i = lane; i < nkv; i += 32) st[a.tok_pos[t0 + i]] = CACHED;
    const int head = (a.q_head[s] + nkv) % a.qcap;
    const int len = a.q_len[s] - nkv;
    int k = 0;
    for (int base = r0; base < r1; base += 32) {
      const int i = base + lane;
      const bool m = i < r1 && a.commit_mask[i];
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
      if (m) {
        const int p = a.row_pos[i];
        st[p] = UNCACHED;
        q[(head + len + k + __popc(bal & ((1u << lane) - 1u))) % a.qcap] = p;
      }
      k += __popc(bal);
    }
    if (lane == 0) {
      a.q_head[s] = head;
      a.q_len[s] = len + k;
      a.commits_out[r] = k;
      a.committed[s] += k;
      a.steps[s] += 1;
    }
  }
  __syncwarp();
  // advance_blocks: skip blocks without MASKED positions
  int bi = a.block_index[s];
  const int committed = a.committed[s];
  while (committed < out) {
    const int lo = bi * a.block, hi = min(lo + a.block, out);
    bool any = false;
    for (int base = lo; base < hi; base += 32) {
      const int p = base + lane;
      if (__any_sync(0xFFFFFFFFu, p < hi && st[p] == MASKED)) {
        any = true;
        break;
      }
    }
    if (any) break;
    ++bi;
  }
  // cached_prefix: first non-CACHED position
  int cp = a.cached_prefix[s];
  while (cp < out) {
    const int p = cp + lane;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, p < out && st[p] == CACHED);
    if (bal == 0xFFFFFFFFu) {
      cp += 32;
      continue;
    }
    cp += __ffs(~bal) - 1;
    break;
  }
  if (lane == 0) {
    a.block_index[s] = bi;
    a.cached_prefix[s] = min(cp, out);
  }
}

// Admissions: one block per admitted request copies its record into the slot's rows.
__global__ void __launch_bounds__(256) admit_kernel(int n_adm, const int32_t* __restrict__ rec, int rec_ints,
                                                    int8_t* states, int64_t stride, int32_t* queue, int qcap,
                                                    int32_t* q_head, int32_t* q_len, int32_t* block_index,
                                                    int32_t* committed, int32_t* steps, int32_t* cached_prefix,
                                                    int32_t* prompt, int32_t* out_len, int32_t* tables,
                                                    int max_pages) {
  if (blockIdx.x >= n_adm) return;
  const int32_t* r = rec + static_cast<int64_t>(blockIdx.x) * rec_ints;
  const int s = r[0];
  if (threadIdx.x == 0) {
    q_head[s] = r[1];
    q_len[s] = r[2];
    block_index[s] = r[3];
    committed[s] = r[4];
    steps[s] = r[5];
    cached_prefix[s] = r[6];
    prompt[s] = r[7];
    out_len[s] = r[8];
  }
  const int sw = static_cast<int>(stride / 4);
  const int32_t* src = r + 9;
  int32_t* st = reinterpret_cast<int32_t*>(states + static_cast<int64_t>(s) * stride);
  for (int i = threadIdx.x; i < sw; i += blockDim.x) st[i] = src[i];
  src += sw;
  for (int i = threadIdx.x; i < qcap; i += blockDim.x) queue[static_cast<int64_t>(s) * qcap + i] = src[i];
  src += qcap;
  for (int i = threadIdx.x; i < max_pages; i += blockDim.x) tables[static_cast<int64_t>(s) * max_pages + i] = src[i];
}

}  // namespace dstep
}  // namespace optimus

extern "C" {

int optimus_admit_record_ints(int64_t state_stride, int qcap, int max_pages) {
  if (state_stride < 0 || state_stride % 4 || qcap < 0 || max_pages < 0) return OPTIMUS_EINVAL;
  return static_cast<int>(9 + state_stride / 4 + qcap + max_pages);
}

int optimus_device_admit(int n_adm, const int32_t* records, int8_t* states, int64_t state_stride, int32_t* queue,
                         int qcap, int32_t* q_head, int32_t* q_len, int32_t* block_index, int32_t* committed,
                         int32_t* steps_taken, int32_t* cached_prefix, int32_t* prompt, int32_t* out_len,
                         int32_t* block_tables, int max_pages, void* stream) {
  using namespace optimus::dstep;
  const int rec_ints = optimus_admit_record_ints(state_stride, qcap, max_pages);
  if (n_adm < 0 || rec_ints < 0) return OPTIMUS_EINVAL;
  if (n_adm == 0) return 0;
  if (!records || !states || !queue || !q_head || !q_len || !block_index || !committed || !steps_taken ||
      !cached_prefix || !prompt || !out_len || !block_tables)
    return OPTIMUS_EINVAL;
  admit_kernel<<<n_adm, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n_adm, records, rec_ints, states, state_stride, queue, qcap, q_head, q_len, block_index, committed,
      steps_taken, cached_prefix, prompt, out_len, block_tables, max_pages);
  return static_cast<int>(cudaGetLastError());
}

int optimus_device_plan(int n, const int32_t* slots, int chunk, const int32_t* chunk_per_req, int block,
                        int window_rule, const int8_t* states, int64_t state_stride, const int32_t* queue,
                        int qcap, const int32_t* q_head, const int32_t* q_len, const int32_t* block_index,
                        const int32_t* cached_prefix, const int32_t* prompt, const int32_t* out_len,
                        const int32_t* block_tables, int max_pages, int32_t* cu_seqlens, int32_t* tok_req,
                        int32_t* tok_pos, int cap_tok, int32_t* prompt_len, int32_t* key_end,
                        int32_t* vis_base, int32_t* vis_off, uint32_t* vis_words, int cap_words,
                        int32_t* cu_rows, int32_t* row_tok, int32_t* row_pos, int32_t* row_req, int cap_rows,
                        int32_t* block_tables_out, int32_t* counts, void* stream) {
  using namespace optimus::dstep;
  if (n < 0 || n > kMaxReq || block < 1 || (window_rule != 0 && window_rule != 1)) return OPTIMUS_EINVAL;
  if (n == 0) return 0;
  PlanArgs a{n, slots, chunk, chunk_per_req, block, window_rule, states, state_stride, queue, qcap,
             q_head, q_len, block_index, cached_prefix, prompt, out_len, block_tables, max_pages,
             cu_seqlens, tok_req, tok_pos, cap_tok, prompt_len, key_end, vis_base, vis_off, vis_words,
             cap_words, cu_rows, row_tok, row_pos, row_req, cap_rows, block_tables_out, counts};
  constexpr int kStageSmem = kWarps * kMaxOut;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageSmem);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  plan_kernel<<<1, kWarps * 32, kStageSmem, static_cast<cudaStream_t>(stream)>>>(a);
  return static_cast<int>(cudaGetLastError());
}

int optimus_device_apply(int n, const int32_t* slots, int block, const int32_t* cu_seqlens,
                         const int32_t* tok_pos, const int32_t* cu_rows, const int32_t* row_pos,
                         const uint8_t* commit_mask, int8_t* states, int64_t state_stride, int32_t* queue,
                         int qcap, int32_t* q_head, int32_t* q_len, int32_t* block_index, int32_t* committed,
                         int32_t* steps_taken, int32_t* cached_prefix, const int32_t* out_len,
                         int32_t* commits_out, int32_t* status, void* stream) {
  using namespace optimus::dstep;
  if (n < 0 || block < 1) return OPTIMUS_EINVAL;
  if (n == 0) return 0;
  ApplyArgs a{n, slots, block, cu_seqlens, tok_pos, cu_rows, row_pos, commit_mask, states, state_stride, queue,
              qcap, q_head, q_len, block_index, committed, steps_taken, cached_prefix, out_len, commits_out,
              status};
  apply_validate_kernel<<<(n * 32 + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  apply_kernel<<<(n * 32 + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // extern "C"

// ----------------------------------------------------------------------------
// Device twin of the attention work planner's whole-unit candidate
// (optimus_attn_plan, capi.cu, candidate A): units (request, KV head, query tile)
// sorted longest first (stable), each cut only at the per-item page cap, placed
// piece by piece on the least-loaded CTA (ties: lowest CTA), costs in half-tiles
// (2 * tiles + 3 per item, + 3 for a cut piece: the host's 1.5 / 1.5 exactly);
// work list in CTA order, split groups / partial slots in unit order.  Same output
// as the host planner whenever it keeps whole units (OPTIMUS_PLAN_FORCE=whole);
// one CTA, ~10 us for 512 units.
namespace optimus {
namespace dstep {

constexpr int kPlanThreads = 1024;
constexpr int kMaxUnits = 4096;


template <int KPER>  // CTAs per lane: grid <= 32 * KPER
__global__ void __launch_bounds__(kPlanThreads, 1) work_plan_kernel(
    int n_req, const int32_t* __restrict__ cu, const int32_t* __restrict__ key_end, int hkv, int T, int grid,
    int hard_cap, int allow_cut, int32_t* __restrict__ work, int max_work, int32_t* __restrict__ cta_off,
    int32_t* __restrict__ groups, int max_groups, int32_t* __restrict__ counts) {
  extern __shared__ uint8_t sm_raw[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm_raw);  // [kMaxUnits]
  int* u_req = reinterpret_cast<int*>(keys + kMaxUnits);
  int* u_head = u_req + kMaxUnits;
  int* u_tok = u_head + kMaxUnits;
  int* u_ntok = u_tok + kMaxUnits;
  int* u_tiles = u_ntok + kMaxUnits;
  int* u_first = u_tiles + kMaxUnits;  // first piece of the unit
  int* p_unit = u_first + kMaxUnits;   // pieces in placement order
  int* p_t0 = p_unit + kMaxUnits;
  int* p_nt = p_t0 + kMaxUnits;
  int* p_cta = p_nt + kMaxUnits;
  int* p_slot = p_cta + kMaxUnits;
  int* u_sc = p_slot + kMaxUnits;  // pieces per unit
  __shared__ int req_off[257];
  __shared__ int n_units_s, n_pieces_s, bad;
  __shared__ unsigned scan_ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad = 0;
  __syncthreads();
  // 1. units: per request hkv * ceil(nq / T), request-major then head then token group
  unsigned n_units_req = 0;
  if (tid < n_req) {
    const int nq = cu[tid + 1] - cu[tid];
    n_units_req = nq > 0 ? hkv * ((nq + T - 1) / T) : 0;
    if (nq > 0 && key_end[tid] < 1) bad = 1;
  }
  {
    unsigned total;
    const unsigned pre = block_exclusive_scan(n_units_req, scan_ws, &total);
    if (tid < n_req) req_off[tid] = static_cast<int>(pre);
    if (tid == 0) {
      req_off[n_req] = static_cast<int>(total);
      n_units_s = static_cast<int>(total);
      if (total > static_cast<unsigned>(kMaxUnits)) bad = 1;
    }
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) counts[3] = OPTIMUS_EINVAL;
    return;
  }
  const int nu = n_units_s;
  if (tid < n_req) {
    const int nq = cu[tid + 1] - cu[tid];
    if (nq > 0) {
      const int nt = (key_end[tid] + 63) / 64;
      int u = req_off[tid];
      for (int h = 0; h < hkv; ++h)
        for (int t0 = 0; t0 < nq; t0 += T, ++u) {
          u_req[u] = tid;
          u_head[u] = h;
          u_tok[u] = cu[tid] + t0;
          u_ntok[u] = min(T, nq - t0);
          u_tiles[u] = nt;
        }
    }
  }
  __syncthreads();
  // 2. stable sort of the units by tiles, descending.  A request's units are
  // contiguous and share its tile count, so sorting the requests (stable, by rank
  // counting: tpr threads per request each compare a stripe of the others) and laying
  // each request's units out in index order gives the stable unit order.
  {
    int* rank_cnt = p_slot;  // [257] units of the request of each rank, then their offsets
    int* rank_of = p_t0;     // [256] (both arrays are written only from step 3 on)
    // threads per request: a power of two <= 32 (a request's threads share a warp)
    const int tpr = 1 << (31 - __clz(min(32, max(1, kPlanThreads / max(n_req, 1)))));
    const int r = tid / tpr, sub = tid - r * tpr;
    int tiles_r = 0, cnt_r = 0, rank = 0;
    if (r < n_req) {
      cnt_r = req_off[r + 1] - req_off[r];
      tiles_r = (key_end[r] + 63) / 64;
      if (cnt_r > 0)
        for (int q = sub; q < n_req; q += tpr) {
          if (req_off[q + 1] == req_off[q]) continue;
          const int tq = (key_end[q] + 63) / 64;
          rank += (tq > tiles_r || (tq == tiles_r && q < r)) ? 1 : 0;
        }
    }
    for (int o = 1; o < tpr; o <<= 1) rank += __shfl_xor_sync(0xFFFFFFFFu, rank, o);
    if (tid < 257) rank_cnt[tid] = 0;
    __syncthreads();
    if (r < n_req && sub == 0 && cnt_r > 0) {
      rank_cnt[rank] = cnt_r;
      rank_of[r] = rank;
    }
    __syncthreads();
    unsigned total;
    const unsigned pre = block_exclusive_scan(tid < n_req ? static_cast<unsigned>(rank_cnt[tid]) : 0u, scan_ws, &total);
    __syncthreads();
    if (tid < n_req) rank_cnt[tid] = static_cast<int>(pre);
    __syncthreads();
    if (r < n_req && cnt_r > 0) {
      const int base = rank_cnt[rank_of[r]];
      const unsigned long long hi = static_cast<unsigned long long>(0x7FFFFFFF - tiles_r) << 32;
      for (int j = sub; j < cnt_r; j += tpr) keys[base + j] = hi | static_cast<unsigned>(req_off[r] + j);
    }
    __syncthreads();
  }
  // 3. placement (loads in half-tiles)
  if (warp == 0) {
    // 3a. pieces per unit: the page cap, and with allow_cut a balanced cut of every
    // unit costlier than the per-CTA budget (mean load + one item) when the longest
    // unit exceeds the budget plus the combine (12 tiles) by more than 12%: the host
    // planner's candidate-B rule with the margin measured for the loop graph, where a
    // cut layer also pays the combine's pass over the partials behind K2 (ShareGPT
    // closed-loop batches, tools/loop_parts.py --ab-cut: longest / (budget + combine)
    // = 1.07 cut 3.2 and 1.4 us per layer slower than whole; 1.17 / 1.21 / 1.37 cut 3.8 /
    // 5.9 / 7.5 us faster; profiles/r2az_device_cut_rule.md), capacity permitting.
    long long total = 0;
    for (int u = lane; u < nu; u += 32) total += 2LL * u_tiles[u] + 3;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(0xFFFFFFFFu, total, off);
    const long long budget = (total + grid - 1) / grid + 3;
    const long long longest = nu > 0 ? 2LL * u_tiles[static_cast<int>(keys[0] & 0xFFFFFFFFu)] + 3 : 0;
    const int nt_max = static_cast<int>(max(4LL, (budget - 6) / 2));
    bool cut = allow_cut && 100 * (budget + 24) < 89 * longest;  // + the combine (12 tiles)
    for (int pass = 0; pass < 2; ++pass) {
      int pieces = 0, cut_units = 0;
      for (int u = lane; u < nu; u += 32) {
        const int tiles = u_tiles[u];
        int sc = (tiles + hard_cap - 1) / hard_cap;
        if (cut && 2LL * tiles + 3 > budget) sc = max(sc, (tiles + nt_max - 1) / nt_max);
        u_sc[u] = sc;
        pieces += sc;
        cut_units += sc > 1;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        pieces += __shfl_xor_sync(0xFFFFFFFFu, pieces, off);
        cut_units += __shfl_xor_sync(0xFFFFFFFFu, cut_units, off);
      }
      if (!cut || (pieces <= min(max_work, kMaxUnits) && cut_units <= max_groups)) break;
      cut = false;  // over capacity: whole units
    }
  }
  __syncthreads();
  // 3b. the flat piece list in placement order (units longest first, each unit's
  // pieces in key order) with each piece's cost: a block scan of the piece counts
  {
    constexpr int kPT = kMaxUnits / kPlanThreads;
    const int o0 = tid * kPT;
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < kPT; ++k)
      if (o0 + k < nu) v += static_cast<unsigned>(u_sc[static_cast<int>(keys[o0 + k] & 0xFFFFFFFFu)]);
    unsigned total;
    unsigned pre = block_exclusive_scan(v, scan_ws, &total);
    if (tid == 0) n_pieces_s = static_cast<int>(total);
    if (total <= static_cast<unsigned>(kMaxUnits)) {
#pragma unroll
      for (int k = 0; k < kPT; ++k) {
        const int o = o0 + k;
        if (o >= nu) break;
        const int u = static_cast<int>(keys[o] & 0xFFFFFFFFu);
        const int tiles = u_tiles[u], sc = u_sc[u];
        const int base = tiles / sc, rem = tiles % sc;
        u_first[u] = static_cast<int>(pre);
        int t0 = 0;
        for (int q = 0; q < sc; ++q) {
          const int x = static_cast<int>(pre) + q, nt = base + (q < rem ? 1 : 0);
          p_unit[x] = u;
          p_t0[x] = t0;
          p_nt[x] = nt;
          p_cta[x] = 2 * nt + 3 + (sc > 1 ? 3 : 0);  // cost in half-tiles, replaced by the placement
          t0 += nt;
        }
        pre += static_cast<unsigned>(sc);
      }
    }
  }
  __syncthreads();
  const int npc = n_pieces_s;
  if (npc > kMaxUnits || npc > max_work) {
    if (tid == 0) counts[3] = OPTIMUS_EINVAL;
    return;
  }
  // 3c. LPT placement by warp 0.  CTA loads live in registers (lane l holds CTAs
  // l, l + 32, ...; static indexing only, so nothing spills to local memory); the
  // argmin is two warp reductions (min load, then min CTA among the lanes holding it:
  // the host heap's tie order).  p_cta[x] becomes cta | rank-in-CTA << 10.
  if (warp == 0) {
    unsigned load[KPER];
    int cnt[KPER];  // pieces booked per CTA
#pragma unroll
    for (int i = 0; i < KPER; ++i) {
      load[i] = lane + 32 * i < grid ? 0u : 0xFFFFFFFFu;
      cnt[i] = 0;
    }
    // the first `grid` pieces land on CTAs 0, 1, ... in order (every load is still
    // zero when each is placed, ties go to the lowest CTA): place them in parallel
    const int first = min(npc, grid);
#pragma unroll
    for (int i = 0; i < KPER; ++i) {
      const int c = lane + 32 * i;
      if (c < first) {
        load[i] = static_cast<unsigned>(p_cta[c]);
        cnt[i] = 1;
        p_cta[c] = c;
      }
    }
    __syncwarp();
    // when every load fits 22 bits, one reduction of (load << 10 | cta) gives the
    // least-loaded CTA with the lowest index on ties
    unsigned sum = 0;
    for (int x = first + lane; x < npc; x += 32) sum += static_cast<unsigned>(p_cta[x]);
#pragma unroll
    for (int i = 0; i < KPER; ++i) sum += lane + 32 * i < first ? load[i] : 0u;
    sum = __reduce_add_sync(0xFFFFFFFFu, sum);
    const bool packed = sum < (1u << 22);
    if (packed) {
      unsigned key[KPER];
#pragma unroll
      for (int i = 0; i < KPER; ++i) {
        const int c = lane + 32 * i;
        key[i] = c < grid ? ((load[i] << 10) | static_cast<unsigned>(c)) : 0xFFFFFFFFu;
      }
#pragma unroll 4
      for (int x = first; x < npc; ++x) {
        const unsigned cost = static_cast<unsigned>(p_cta[x]) << 10;
        unsigned lm = key[0];
#pragma unroll
        for (int i = 1; i < KPER; ++i) lm = min(lm, key[i]);
        const int bc = static_cast<int>(__reduce_min_sync(0xFFFFFFFFu, lm) & 1023u);
        const int sel = (bc & 31) == lane ? (bc >> 5) : -1;
        int rank = 0;
#pragma unroll
        for (int i = 0; i < KPER; ++i) {
          const bool hit = i == sel;
          rank = hit ? cnt[i] : rank;
          key[i] += hit ? cost : 0u;
          cnt[i] += hit ? 1 : 0;
        }
        if (sel >= 0) p_cta[x] = bc | (rank << 10);
      }
    }
#pragma unroll 4
    for (int x = packed ? npc : first; x < npc; ++x) {
      const unsigned cost = static_cast<unsigned>(p_cta[x]);
      unsigned best = 0xFFFFFFFFu;
      int bi = 0;
#pragma unroll
      for (int i = 0; i < KPER; ++i)
        if (load[i] < best) {  // increasing CTA per lane: first minimum
          best = load[i];
          bi = i;
        }
      const unsigned m = __reduce_min_sync(0xFFFFFFFFu, best);
      const int bc = static_cast<int>(
          __reduce_min_sync(0xFFFFFFFFu, best == m ? static_cast<unsigned>(lane + 32 * bi) : 0xFFFFFFFFu));
      const int sel = (bc & 31) == lane ? (bc >> 5) : -1;  // the owning lane books the piece
      int rank = 0;
#pragma unroll
      for (int i = 0; i < KPER; ++i) {  // selects, not an indexed store: the arrays stay in registers
        const bool hit = i == sel;
        rank = hit ? cnt[i] : rank;
        load[i] += hit ? cost : 0u;
        cnt[i] += hit ? 1 : 0;
      }
      if (sel >= 0) p_cta[x] = bc | (rank << 10);
    }
    __syncwarp();
    int* cc = reinterpret_cast<int*>(keys);  // per-CTA piece counts (the keys are dead)
#pragma unroll
    for (int i = 0; i < KPER; ++i)
      if (lane + 32 * i < grid) cc[lane + 32 * i] = cnt[i];
  }
  __syncthreads();
  int* cta_cnt = reinterpret_cast<int*>(keys);  // the sort keys are dead now (written by warp 0 above)
  // 4. split groups and partial slots, in unit order: one block scan of
  // (cut units << 16 | their pieces) over 4 consecutive units per thread
  {
    constexpr int kPerThread = kMaxUnits / kPlanThreads;
    const int u0 = tid * kPerThread;
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)
      if (u0 + k < nu && u_sc[u0 + k] > 1) v += (1u << 16) | static_cast<unsigned>(u_sc[u0 + k]);
    unsigned total;
    unsigned pre = block_exclusive_scan(v, scan_ws, &total);
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
      const int u = u0 + k;
      if (u >= nu) break;
      const int sc = u_sc[u], f = u_first[u];
      if (sc > 1) {
        const int gi = static_cast<int>(pre >> 16), part = static_cast<int>(pre & 0xFFFFu);
        if (gi < max_groups) {
          int32_t* g = groups + 8 * gi;
          g[0] = u_req[u];
          g[1] = u_head[u];
          g[2] = u_tok[u];
          g[3] = u_ntok[u];
          g[4] = part;
          g[5] = sc;
          g[6] = 0;
          g[7] = 0;
        }
        for (int q = 0; q < sc; ++q) p_slot[f + q] = part + q;
        pre += (1u << 16) | static_cast<unsigned>(sc);
      } else {
        p_slot[f] = -1;
      }
    }
    if (tid == 0) {
      const int ng = static_cast<int>(total >> 16);
      counts[0] = npc;
      counts[1] = ng;
      counts[2] = static_cast<int>(total & 0xFFFFu);
      counts[3] = ng > max_groups ? OPTIMUS_EINVAL : 0;
    }
  }
  // 5. work list in CTA order (each CTA's pieces in placement order): scan of the
  // per-CTA counts, then every piece written at cta_off[cta] + rank
  {
    unsigned total;
    const unsigned pre =
        block_exclusive_scan(tid < grid ? static_cast<unsigned>(cta_cnt[tid]) : 0u, scan_ws, &total);
    if (tid < grid) {
      cta_off[tid] = static_cast<int>(pre);
      cta_cnt[tid] = static_cast<int>(pre);
    }
    if (tid == 0) cta_off[grid] = npc;
    __syncthreads();
    for (int x = tid; x < npc; x += kPlanThreads) {
      const int c = p_cta[x] & 1023, rank = p_cta[x] >> 10;
      const int u = p_unit[x];
      int32_t* w = work + 8 * (cta_cnt[c] + rank);
      w[0] = u_req[u];
      w[1] = u_head[u];
      w[2] = u_tok[u];
      w[3] = u_ntok[u];
      w[4] = p_t0[x] * 64;
      w[5] = min(key_end[u_req[u]], (p_t0[x] + p_nt[x]) * 64);
      w[6] = p_slot[x];
      w[7] = 0;
    }
  }
}

}  // namespace dstep
}  // namespace optimus

extern "C" int optimus_device_attn_plan(int n_req, const int32_t* cu_seqlens, const int32_t* key_end, int hq,
                                        int hkv, int grid, int page_size, int allow_cut, int32_t* work, int max_work,
                                        int32_t* cta_off, int32_t* groups, int max_groups, int32_t* counts,
                                        void* stream) {
  using namespace optimus::dstep;
  if (n_req < 0 || n_req > 256 || hkv < 1 || hq % hkv || grid < 1 || grid > 1024) return OPTIMUS_EINVAL;
  const int G = hq / hkv;
  if (G > 128) return OPTIMUS_EINVAL;
  const int hard_cap = static_cast<int>(std::max(1LL, std::min((255LL * std::max(page_size, 1)) / 64, 1LL << 20)));
  const size_t smem = kMaxUnits * (8 + 12 * 4);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(work_plan_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(work_plan_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(work_plan_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  // CTA loads per lane: 5 covers one B200 (148 SMs); fewer registers to reduce per placed piece
  auto kern = grid <= 160 ? work_plan_kernel<5> : grid <= 256 ? work_plan_kernel<8> : work_plan_kernel<32>;
  kern<<<1, kPlanThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      n_req, cu_seqlens, key_end, hkv, 128 / G, grid, hard_cap, allow_cut, work, max_work, cta_off, groups, max_groups,
      counts);
  return static_cast<int>(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// Window row -> logits row of a slot-indexed logits table (the synthetic forward's
// layout: rows_per_slot rows per batch slot, version block `base`), for device-planned
// steps: row_src[i] = base + slot(row i) * rows_per_slot + min(rank in request, rows_per_slot - 1).
namespace optimus {
namespace dstep {
__global__ void row_src_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ slots,
                               const int32_t* __restrict__ cu_rows, const int32_t* __restrict__ row_req,
                               int rows_per_slot, int base, int32_t* __restrict__ row_src) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= counts[1]) return;
  const int r = row_req[i];
  row_src[i] = base + slots[r] * rows_per_slot + min(i - cu_rows[r], rows_per_slot - 1);
}
}  // namespace dstep
}  // namespace optimus

extern "C" int optimus_device_row_src(const int32_t* counts, const int32_t* slots, const int32_t* cu_rows,
                                      const int32_t* row_req, int cap_rows, int rows_per_slot, int base,
                                      int32_t* row_src, void* stream) {
  if (cap_rows <= 0 || rows_per_slot < 1) return OPTIMUS_EINVAL;
  optimus::dstep::row_src_kernel<<<(cap_rows + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, slots, cu_rows, row_req, rows_per_slot, base, row_src);
  return static_cast<int>(cudaGetLastError());
}
