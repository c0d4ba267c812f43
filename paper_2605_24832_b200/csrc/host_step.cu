// host_step.cu — native host side of the batched decode step (host code only).
//
// The reference runs the control half of every decode iteration in Python, one
// request at a time (sim.py:276-291): plan_chunk (engine.py:45-67), then
// apply_chunk (engine.py:79-95) with advance_blocks (core.py:109-116).  Here the
// whole batch is planned and applied in one call over packed per-slot state, and
// the plan is emitted directly as the kernels' step metadata (rule V bitmaps,
// query/window layouts) into a caller-provided (pinned) buffer.  Semantics are
// those of the reference functions; tests/test_host_step.py checks plans, metadata
// and state transitions against the Python mirror request by request.
//
// Packed state (caller-owned, indexed by slot):
//   states   int8  [slots][state_stride]   TokenState per output position
//   queue    int32 [slots][qcap]           FIFO ring of decoded-but-uncached positions
//   q_head, q_len, block_index, committed, steps_taken, cached_prefix,
//   prompt, out_len                        int32 [slots]
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/optimus_b200.h"

namespace {

constexpr int8_t MASKED = 0, UNCACHED = 1, CACHED = 2;

struct Packed {
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
  const int32_t* prompt;
  const int32_t* out_len;
};

inline int qget(const Packed& P, int slot, int i) {
  return P.queue[static_cast<int64_t>(slot) * P.qcap + (P.q_head[slot] + i) % P.qcap];
}

}  // namespace

extern "C" {

// Plan one step for the batch `slots[0..n)` and write the step metadata.
// Output arrays (capacities in elements; all int32 except vis_words):
//   cu_seqlens[n+1], tok_req[cap_tok], tok_pos[cap_tok], prompt_len[n], key_end[n],
//   vis_base[n], vis_off[n+1], vis_words[cap_words], cu_rows[n+1], row_tok[cap_rows],
//   row_pos[cap_rows], row_req[cap_rows], block_tables_out[n][max_pages]
//   (gathered from block_tables[slot][max_pages]).
// counts_out[0..3) = {n_tok, n_rows, n_words}.  Returns 0 or OPTIMUS_EINVAL.
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
                      int32_t* block_tables_out, int32_t* counts_out) {
  if (block < 1 || n < 0 || (window_rule != 0 && window_rule != 1)) return OPTIMUS_EINVAL;
  Packed P{states, state_stride, queue, qcap, q_head, q_len, block_index,
           nullptr, nullptr, cached_prefix, prompt, out_len};
  int nt = 0, nr = 0, nw = 0;
  cu_seqlens[0] = 0;
  cu_rows[0] = 0;
  std::vector<uint8_t> planned;
  for (int r = 0; r < n; ++r) {
    const int s = slots[r];
    const int out = out_len[s];
    const int8_t* st = states + static_cast<int64_t>(s) * state_stride;
    const int chunk_r = chunk_per_req ? chunk_per_req[r] : chunk;  // mixed chunks (elastic)
    if (chunk_r < 2) return OPTIMUS_EINVAL;                        // ChunkTooSmall, engine.py:56
    // A finished request plans nothing (the reference's loop drops it, sim.py:307-313).
    // advance_blocks keeps an unfinished request's current block holding a MASKED
    // position, so "finished" == no MASKED position in the current block.
    bool done = true;
    for (int p = block_index[s] * block, e = std::min(p + block, out); p < e; ++p)
      if (st[p] == MASKED) {
        done = false;
        break;
      }
    const int nkv = done ? 0 : std::min(q_len[s], chunk_r);
    if (nt + chunk_r > cap_tok) return OPTIMUS_EINVAL;
    const int t0 = nt;
    for (int i = 0; i < nkv; ++i) {
      tok_req[nt] = r;
      tok_pos[nt++] = qget(P, s, i);
    }
    int room = done ? 0 : chunk_r - nkv;
    const int r0 = nr;
    int lo = block_index[s] * block;
    int hi = std::min(lo + block, out);
    if (window_rule == 1) {  // OUT_BLOCK: earliest masked anywhere, capped at block
      hi = out;
      room = std::min(room, block);
    }
    for (int p = lo; p < hi && room > 0; ++p) {
      if (st[p] == MASKED) {
        if (nr >= cap_rows) return OPTIMUS_EINVAL;
        row_tok[nr] = nt;
        row_pos[nr] = p;
        row_req[nr++] = r;
        tok_req[nt] = r;
        tok_pos[nt++] = p;
        --room;
      }
    }
    cu_seqlens[r + 1] = nt;
    cu_rows[r + 1] = nr;
    const int pr = prompt[s];
    prompt_len[r] = pr;
    vis_off[r] = nw;
    if (nt == t0) {
      key_end[r] = 0;
      vis_base[r] = 0;
      continue;
    }
    // rule V: visible = CACHED before the step, or planned now
    planned.assign(out, 0);
    int max_q = -1;
    for (int i = t0; i < nt; ++i) {
      planned[tok_pos[i]] = 1;
      max_q = std::max(max_q, tok_pos[i]);
    }
    auto vis = [&](int p) { return st[p] == CACHED || planned[p]; };
    int cp = std::min(cached_prefix[s], out);
    while (cp < out && vis(cp)) ++cp;
    const int cap_end = (max_q / block + 1) * block;  // block-causal cap of the latest query
    int last = out - 1;
    while (last >= 0 && !vis(last)) --last;
    const int ke = pr + std::min(last + 1, cap_end);
    key_end[r] = ke;
    int vb = ((pr + cp) / 32) * 32;
    if (vb > ke) vb = (ke / 32) * 32;
    vis_base[r] = vb;
    if (ke > vb) {
      const int words = (ke - vb + 31) / 32;
      if (nw + words > cap_words) return OPTIMUS_EINVAL;
      for (int w = 0; w < words; ++w) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
          const int a = vb + w * 32 + b;  // absolute key position
          if (a >= ke) break;
          const int p = a - pr;
          if (p < 0 || vis(p)) bits |= 1u << b;
        }
        vis_words[nw + w] = bits;
      }
      nw += words;
    }
  }
  vis_off[n] = nw;
  for (int r = 0; r < n; ++r)
    std::memcpy(block_tables_out + static_cast<int64_t>(r) * max_pages,
                block_tables + static_cast<int64_t>(slots[r]) * max_pages, sizeof(int32_t) * max_pages);
  counts_out[0] = nt;
  counts_out[1] = nr;
  counts_out[2] = nw;
  return 0;
}

// Apply one step: kv positions -> DECODED_CACHED (FIFO pops), committed window rows
// (commit_mask in row order) -> DECODED_UNCACHED appended to the ring, counters,
// advance_blocks.  commits_out[r] receives the number of commits of batch row r.
// Like the reference (_check_commits before any state change, engine.py:70-83),
// every request of the batch is validated first; on OPTIMUS_EINVAL no state has
// changed.
int optimus_host_apply(int n, const int32_t* slots, int block, const int32_t* cu_seqlens,
                       const int32_t* tok_pos, const int32_t* cu_rows, const int32_t* row_pos,
                       const uint8_t* commit_mask, int8_t* states, int64_t state_stride,
                       int32_t* queue, int qcap, int32_t* q_head, int32_t* q_len,
                       int32_t* block_index, int32_t* committed, int32_t* steps_taken,
                       int32_t* cached_prefix, const int32_t* out_len, int32_t* commits_out) {
  if (n < 0 || block < 1) return OPTIMUS_EINVAL;
  // pass 1: validate (no writes)
  for (int r = 0; r < n; ++r) {
    const int s = slots[r];
    if (committed[s] >= out_len[s]) continue;
    const int8_t* st = states + static_cast<int64_t>(s) * state_stride;
    const int32_t* q = queue + static_cast<int64_t>(s) * qcap;
    const int nkv = (cu_seqlens[r + 1] - cu_seqlens[r]) - (cu_rows[r + 1] - cu_rows[r]);
    if (nkv < 0 || nkv > q_len[s]) return OPTIMUS_EINVAL;
    for (int i = 0; i < nkv; ++i)  // KV plan must pop the FIFO in order (engine.py:85-88)
      if (q[(q_head[s] + i) % qcap] != tok_pos[cu_seqlens[r] + i]) return OPTIMUS_EINVAL;
    int k = 0;
    for (int i = cu_rows[r]; i < cu_rows[r + 1]; ++i) {
      if (!commit_mask[i]) continue;
      const int p = row_pos[i];
      if (p < 0 || p >= out_len[s] || st[p] != MASKED) return OPTIMUS_EINVAL;  // IllegalCommit
      ++k;
    }
    if (q_len[s] - nkv + k > qcap) return OPTIMUS_EINVAL;
  }
  // pass 2: apply
  for (int r = 0; r < n; ++r) {
    const int s = slots[r];
    if (committed[s] >= out_len[s]) {  // finished: not stepped (sim.py:307-313)
      commits_out[r] = 0;
      continue;
    }
    int8_t* st = states + static_cast<int64_t>(s) * state_stride;
    int32_t* q = queue + static_cast<int64_t>(s) * qcap;
    const int nkv = (cu_seqlens[r + 1] - cu_seqlens[r]) - (cu_rows[r + 1] - cu_rows[r]);
    for (int i = 0; i < nkv; ++i) {
      st[tok_pos[cu_seqlens[r] + i]] = CACHED;
      q_head[s] = (q_head[s] + 1) % qcap;
      --q_len[s];
    }
    int k = 0;
    for (int i = cu_rows[r]; i < cu_rows[r + 1]; ++i) {
      if (!commit_mask[i]) continue;
      const int p = row_pos[i];
      st[p] = UNCACHED;
      q[(q_head[s] + q_len[s]) % qcap] = p;
      ++q_len[s];
      ++k;
    }
    commits_out[r] = k;
    committed[s] += k;
    steps_taken[s] += 1;
    const int out = out_len[s];
    while (committed[s] < out) {
      const int lo = block_index[s] * block;
      const int hi = std::min(lo + block, out);
      bool any = false;
      for (int p = lo; p < hi; ++p)
        if (st[p] == MASKED) {
          any = true;
          break;
        }
      if (any) break;
      ++block_index[s];
    }
    int cp = cached_prefix[s];
    while (cp < out && st[cp] == CACHED) ++cp;
    cached_prefix[s] = cp;
  }
  return 0;
}

}  // extern "C"
