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
//   warp 8   TMA producer: per work item one Q tile (the G query heads of a KV head
//            folded into 128 MMA rows, row = token*G + head) and the K ring of
//            64-key tiles gathered page by page through the block table (4-D tensor
//            maps, SWIZZLE_128B boxes of 64 columns).  warp 10: TMEM allocator,
//            then the V ring.  K and V slots have separate full/empty barriers: a K
//            slot is refilled as soon as its S = Q K^T retires.
//   warp 9   MMA issuer: one stream of tiles across the CTA's work items.  The
//            item's Q tile is copied smem -> TMEM (tcgen05.cp) and is the A operand
//            of S = Q K^T (only K is read from shared memory); S goes to one of three
//            rotating S/P buffers in TMEM, three tiles ahead of PV and across item
//            boundaries; O += P V with P read from TMEM (TS-MMA).
//   warp 11  metadata: stages the next work item's page ids / limits in smem.
//   warps 0-7  softmax + epilogue, two warpgroups ping-ponging over the tiles of
//            a work item: thread i owns query row i (= TMEM lane i), so the row
//            max/sum need no shuffles; each warpgroup keeps its own (m, l, O) and
//            the epilogue merges them.  Online softmax in the exp2 domain with a
//            lazy rescale (O in TMEM is only rescaled when the running max grows by
//            more than 2^8).  P overwrites S in TMEM: one fp16 plane with the fp16 V
//            cache, or two bf16 planes P = hi + lo with a bf16 V cache.  An item's
//            epilogue (normalise O, store bf16 or fp32 split-KV partials) runs
//            after the warpgroup's first tile of the next item.
//   Control roles issue from a converged warp with one elected lane, so their
//   operands sit in uniform registers (no per-instruction R2UR loop).
// Work items are planned on the host (optimus_attn_plan): whole (request, KV head,
// token group) units placed longest-first, cut at tile boundaries when that balances
// the CTAs; cut pieces are merged by the split-KV combine kernel below.
#include "attn.cuh"

namespace optimus {

// Set when the fused append clamps a bf16 V value beyond the fp16 range (see K1).
__device__ int g_v_saturated_k2;

int v_saturated_k2(int32_t* out, int reset, cudaStream_t stream) {
  cudaError_t e = cudaMemcpyFromSymbolAsync(out, g_v_saturated_k2, sizeof(int), 0, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess && reset) {
    void* a = nullptr;
    e = cudaGetSymbolAddress(&a, g_v_saturated_k2);
    if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, sizeof(int), stream);
  }
  return static_cast<int>(e);
}

constexpr int kTileN = 64;     // keys per pipeline stage
constexpr int kBlockM = 128;   // MMA rows (query token x head-in-group)
constexpr int kThreads = 512;  // 16 warps: 8 softmax, 4 control, 4 epilogue
// registers per thread after the setmaxnreg split (launch: 512 x 128):
// 128 x 56 (control) + 128 x 80 (epilogue) + 256 x 184 (softmax) = 64,512 <= 65,536
constexpr int kCtrlRegs = 56;
constexpr int kEpiRegs = 80;
constexpr int kMathRegs = 184;
static_assert(128 * kCtrlRegs + 128 * kEpiRegs + 256 * kMathRegs <= 65536, "setmaxnreg split exceeds the SM");
constexpr int kSBuf = 3;       // S/P buffers in TMEM, rotating over the CTA's tile stream
constexpr int kInfo = 4;       // staged work-item records: the metadata warp runs 3 items ahead
constexpr int kEpiRing = 16;   // per-item epilogue records (outlive the staged record)
static_assert(kEpiRing > kInfo + 1, "epilogue records must outlive the staging ring");
constexpr int kTraceSlots = 4096;
constexpr int kAppItems = 64;  // work records per fused-append batch  // per CTA: [role*256 + i], 16 roles

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// roles: 0 producer top, 1 MMA S issue, 2 softmax S ready, 3 softmax P done,
// 4 producer slot free, 5 producer K issued, 6 misc (0 entry [globaltimer], 1 setup,
// 2 producer done, 3 CTA done, 4 CTA done [globaltimer], 5.. metadata item staged),
// 7 PV issued, 8 MMA reaches PV (v_full wait), 9 V landed (p_full wait), 10 V producer
// slot free, 11 V producer issued, 12 MMA reaches S, 13/14/15 epilogue of item i
// entered / O complete / O released (warpgroup 0).  Tile-indexed roles count the
// CTA's tile stream.
__device__ __forceinline__ void trace(const AttnParams& p, int role, int i) {
  if (p.trace != nullptr && i < 256)
    p.trace[static_cast<int64_t>(blockIdx.x) * kTraceSlots + role * 256 + i] =
        (role == 6 && (i == 0 || i == 4)) ? gtimer() : static_cast<unsigned long long>(clock64());
}

// Per-work-item record staged in shared memory by the metadata warp up to kInfo items
// ahead (scalars by plain stores, page ids / query positions / visibility words by
// 4-byte cp.async), so no other role touches global memory on its critical path and
// the stager itself never waits on a load.
constexpr int kMaxUnitPages = 256;  // the planner caps an item at 255 pages of keys
constexpr int kMaxUnitWords = 16;   // visibility words held in smem (more: read from global)
struct UnitInfo {
  int req, head, tok_begin, n_tok, key_begin, key_end, slot, vb;
  int n_words, vis_off, prompt, pad0;
  int qpos[kBlockM];                // query positions of the item's tokens
  uint32_t words[kMaxUnitWords];
  int pages[kMaxUnitPages];
};
// epilogue record of item u at [u % kEpiRing]: {head, tok_begin, n_tok, slot, n_tiles}
constexpr int kEpiInts = 8;

template <int HD, int KST, int VST>
struct AttnSmem {
  static constexpr int KB = HD / 64;
  static constexpr uint32_t Q_BYTES = KB * kBlockM * 128;
  static constexpr uint32_t KT_BYTES = KB * kTileN * 128;
  static constexpr uint32_t OFF_Q = 0;  // one Q tile: copied into TMEM per item
  static constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
  static constexpr uint32_t OFF_V = OFF_K + KST * KT_BYTES;
  static constexpr uint32_t OFF_INFO = OFF_V + VST * KT_BYTES;
  static constexpr uint32_t OFF_RED = OFF_INFO + kInfo * sizeof(UnitInfo);  // float[item&1][{m,l}][wg][128]
  static constexpr uint32_t OFF_EPI = OFF_RED + 2 * 2 * 2 * kBlockM * 4;
  static constexpr uint32_t OFF_APP = OFF_EPI + kEpiRing * kEpiInts * 4;  // fused-append scratch
  static constexpr uint32_t OFF_BAR = (OFF_APP + (kAppItems * 9 + 1) * 4 + 15) / 16 * 16;
  static constexpr int NUM_BARS = 2 * KST + 2 * VST + 2 + 3 * kSBuf + 6 + 3 * kInfo + 2;
  static constexpr uint32_t BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr uint32_t ALLOC = BYTES + 1024;  // slack for 1024-byte alignment
  static_assert(ALLOC <= 232448, "exceeds the 227 KB per-CTA shared memory of sm_100");
  // TMEM columns: three S/P buffers [0,192), the item's Q tile (A operand of
  // S = Q K^T) [192, 192+HD/2), then the warpgroups' O accumulators
  // O_0 = [256,256+HD), O_1 = [256+HD,256+2HD).
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t TM_Q = kSBuf * kTileN;
  static constexpr uint32_t TM_O = 256;
  static_assert(TM_Q + HD / 2 <= TM_O && TM_O + 2 * HD <= TMEM_COLS, "TMEM budget");
};

template <int HD, int KST, int VST, bool VF16>
__global__ void __launch_bounds__(kThreads, 1)
    paged_attn_kernel(const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using L = AttnSmem<HD, KST, VST>;
  constexpr int KB = L::KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* q_full = v_empty + VST;  // Q tile landed in smem
  uint64_t* q_empty = q_full + 1;    // Q tile copied into TMEM (smem free)
  uint64_t* s_full = q_empty + 1;    // [buffer]
  uint64_t* p_full = s_full + kSBuf;   // [buffer]
  uint64_t* pv_done = p_full + kSBuf;  // [buffer]
  uint64_t* o_full = pv_done + kSBuf;
  uint64_t* o_empty = o_full + 1;
  uint64_t* red_full = o_empty + 1;   // [item & 1]: both softmax warpgroups' (m, l) are in `red`
  uint64_t* red_empty = red_full + 2; // [item & 1]: the epilogue warpgroup has read them
  uint64_t* info_full = red_empty + 2;
  uint64_t* info_empty = info_full + kInfo;
  uint64_t* pg_full = info_empty + kInfo;      // [kInfo]: the record's key range, page ids, query positions
  uint64_t* append_done = pg_full + kInfo;     // fused KV append of this CTA's items landed
  uint64_t* append_issued = append_done + 1;   // ... and its first loads are in flight
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(append_issued + 1);
  UnitInfo* info = reinterpret_cast<UnitInfo*>(smem + L::OFF_INFO);
  float* red = reinterpret_cast<float*>(smem + L::OFF_RED);  // epilogue (m, l) exchange
  int* epi = reinterpret_cast<int*>(smem + L::OFF_EPI);

  const int warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0);  // provably warp-uniform
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace(p, 6, 0);

  if (warp == 8 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 9 && lane == 0) {
    for (int i = 0; i < KST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < kInfo; ++i) {
      mbar_init(&info_full[i], 33);  // 32 cp.async arrivals + lane 0's store arrival
      mbar_init(&pg_full[i], 33);    // the same, for the part the TMA producers need
      mbar_init(&info_empty[i], 256 + 2);  // softmax threads + K and V producers
    }
    for (int i = 0; i < kSBuf; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);  // the epilogue warpgroup
    for (int i = 0; i < 2; ++i) {
      mbar_init(&red_full[i], 256);
      mbar_init(&red_empty[i], 128);
    }
    mbar_init(append_done, 256);
    mbar_init(append_issued, 256);
    mbar_fence_init();
  }
  if (warp == 10) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  // Zero the K/V rings once: rows a partial tile never loads must hold finite values
  // (their probabilities are 0, and 0 * NaN would poison O).  With 64-row boxes (pages
  // of >= 64 keys) every tile is one full box, so no row is left unloaded.
  if (p.box_rows < kTileN) {
    uint4* z = reinterpret_cast<uint4*>(sK);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (uint32_t i = threadIdx.x; i < (KST + VST) * L::KT_BYTES / 16; i += kThreads) z[i] = zero;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace(p, 6, 1);
  // Every CTA of this grid is resident (one per SM, grid <= #SM): let the next
  // PDL-launched kernel take each SM as soon as this CTA leaves it, so its prologue
  // (and a K1's index math) fills this grid's tail.  Dependents read nothing this grid
  // writes before their griddepcontrol.wait, which waits for this grid's completion.
  if (!(p.dbg & 128)) grid_dep_launch();
  const uint32_t tm_s0 = tmem_base;           // S/P buffers
  const uint32_t tm_qt = tmem_base + L::TM_Q; // Q tile (MMA A operand)
  const uint32_t tm_o0 = tmem_base + L::TM_O; // O accumulators

  const int w_begin = p.cta_off[blockIdx.x];
  const int w_end = p.cta_off[blockIdx.x + 1];

  // Register split (setmaxnreg, per warpgroup): the control warpgroup (warps 8-11: TMA
  // producers, MMA issuer, metadata) runs in kCtrlRegs registers and the epilogue
  // warpgroup (12-15) in kEpiRegs, handing the rest to the two softmax warpgroups.
  // Each side's code is reachable only after its own setmaxnreg, so the allocator
  // budgets the sides separately.
  if (warp >= 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kEpiRegs));
    // ------------------------------------------------------------ epilogue warpgroup
    // Per item, in order: merge the two softmax warpgroups' (m_0, l_0, O_0) and
    // (m_1, l_1, O_1) like two key splits, hand O back to the MMA warp as soon as it is
    // read, and write the output rows (bf16, or fp32 split-KV partials).  Warp w reads
    // TMEM lanes 32 (w % 4) .. +31, so the four warps cover the tile's 128 rows.  The
    // softmax warpgroups never stop for an epilogue: the next item's tiles flow while
    // this warpgroup drains the last one.
    const int ew = warp & 3;
    const int row = ew * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const int G = p.group;
    const int t_in = row / G;
    const int g_in = row - t_in * G;
    const bool row_exists = t_in < p.tok_per_tile;
    const int n_units = w_end - w_begin;
    {
      // zero O_0 / O_1 once: an accumulator a warpgroup does not touch in an item (no
      // tile of its parity) then holds finite values, and the merge below can weight it
      // by 0 with one FMA instead of a select (first phase of o_empty: the MMA's first
      // PV waits for it)
      uint32_t z[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) z[c] = 0u;
#pragma unroll
      for (int c0 = 0; c0 < 2 * HD; c0 += 16) tmem_st16(tm_o0 + lane_off + c0, z);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(o_empty);
    }
    for (int e = 0; e < n_units; ++e) {
      mbar_wait(&red_full[e & 1], (e >> 1) & 1);
      // (the item's epilogue record was published before its staged record, which the
      // softmax warpgroups acquired before arriving on red_full)
      const int* er = epi + (e % kEpiRing) * kEpiInts;
      const int head = er[0], tok_begin = er[1], n_tok = er[2], slot = er[3];
      const bool valid = row_exists && t_in < n_tok;
      const bool warp_valid = (ew * 32) / G < n_tok;
      if (threadIdx.x == 384) trace(p, 13, e);
      const float* rd = red + (e & 1) * 4 * kBlockM;
      const float m0 = rd[0 * kBlockM + row], m1 = rd[1 * kBlockM + row];
      const float l0 = rd[2 * kBlockM + row], l1 = rd[3 * kBlockM + row];
      mbar_arrive(&red_empty[e & 1]);
      const float mx = fmaxf(m0, m1);
      const float w0 = l0 > 0.f ? fast_exp2(m0 - mx) : 0.f;
      const float w1 = l1 > 0.f ? fast_exp2(m1 - mx) : 0.f;
      const float l_tot = w0 * l0 + w1 * l1;
      const float inv_l = (l_tot > 0.f) ? 1.0f / l_tot : 0.f;
      const float f0 = w0 * (slot < 0 ? inv_l : 1.f), f1 = w1 * (slot < 0 ? inv_l : 1.f);
      mbar_wait(o_full, e & 1);
      tc_fence_after();
      if (threadIdx.x == 384) trace(p, 14, e);
      const int tok = tok_begin + t_in;
      const int qh = head * G + g_in;
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 16) {
        uint32_t o0[16], o1[16];
        if (warp_valid) {
          tmem_ld16(tm_o0 + lane_off + c0, o0);
          tmem_ld16(tm_o0 + lane_off + HD + c0, o1);
          tmem_wait_ld();
        }
        if (c0 + 16 >= HD) {  // all of O_0 / O_1 read: back to the MMA warp
          tc_fence_before();
          mbar_arrive(o_empty);
          if (threadIdx.x == 384) trace(p, 15, e);
        }
        if (valid) {
          // f0 / f1 are 0 for a warpgroup without keys (w = 0), whose O is finite
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            float a0, a1, b0, b1;
            ffma2(a0, a1, __uint_as_float(o0[c]), __uint_as_float(o0[c + 1]), f0, f0, 0.f, 0.f);
            ffma2(b0, b1, __uint_as_float(o1[c]), __uint_as_float(o1[c + 1]), f1, f1, a0, a1);
            o0[c] = __float_as_uint(b0);
            o0[c + 1] = __float_as_uint(b1);
          }
          const float* o = reinterpret_cast<const float*>(o0);
          if (slot < 0) {
            uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<int64_t>(tok) * p.out_stride_tok +
                                                  static_cast<int64_t>(qh) * HD + c0);
#pragma unroll
            for (int v = 0; v < 2; ++v)
              dst[v] = make_uint4(pack_bf16x2(o[8 * v], o[8 * v + 1]), pack_bf16x2(o[8 * v + 2], o[8 * v + 3]),
                                  pack_bf16x2(o[8 * v + 4], o[8 * v + 5]), pack_bf16x2(o[8 * v + 6], o[8 * v + 7]));
          } else {
            float4* dst = reinterpret_cast<float4*>(p.ws_o + (static_cast<int64_t>(slot) * kBlockM + row) * HD + c0);
#pragma unroll
            for (int v = 0; v < 4; ++v) dst[v] = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
          }
        }
      }
      if (valid && slot >= 0)
        reinterpret_cast<float2*>(p.ws_ml)[static_cast<int64_t>(slot) * kBlockM + row] = make_float2(mx, l_tot);
    }
  } else if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kCtrlRegs));
  if (warp == 8 || warp == 10) {
      // ------------------------------------------------------------ TMA producers
      // Warp 8 loads Q and the K ring, warp 10 the V ring.  The whole warp runs the
      // loop (operands warp-uniform, in uniform registers); one elected lane issues.
      const bool is_k = warp == 8;
      const int NST = is_k ? KST : VST;
      const uint32_t q_tx = KB * 64 * p.group * p.tok_per_tile * 2;
      const uint32_t chunk_tx = p.box_rows * 128 * KB;  // one tensor, one box-row group
      const int chunks_per_tile = kTileN / p.box_rows;
      const int shift = p.page_shift;
      const int pmask = p.page_size - 1;
      const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
      uint8_t* ring = is_k ? sK : sV;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      // K/V pages are read once per step: stream them through L2 with evict_first so
      // the step metadata and Q stay resident
      const uint64_t pol_stream = l2_policy_evict_first();
      int tile_ctr = 0;
      int unit = 0;
      bool need_append = p.k_new != nullptr;  // output-region tiles wait for the fused append
      if (need_append) {
        // the append's loads go first; (diagnostics, dbg 64: no load before it landed)
        mbar_wait((p.dbg & 64) ? append_done : append_issued, 0);
        if (p.dbg & 64) need_append = false;
      }
      for (int w = w_begin; w < w_end; ++w, ++unit) {
        const int ib = unit % kInfo;
        // the key range and page ids land one round trip before the visibility words
        // (which need the request's scalars): the first loads of a launch go out on them
        mbar_wait(need_append ? &info_full[ib] : &pg_full[ib], (unit / kInfo) & 1);
        // Q/K/V are written by the preceding kernels (QKV producer, K1 append):
        // everything above overlapped their tail under PDL; the loads may not.
        if (unit == 0) grid_dep_wait();
        const UnitInfo& u = info[ib];
        const int head = __shfl_sync(0xFFFFFFFFu, u.head, 0);
        const int key_begin = __shfl_sync(0xFFFFFFFFu, u.key_begin, 0);
        const int key_end = __shfl_sync(0xFFFFFFFFu, u.key_end, 0);
        const int pg0 = key_begin >> shift;
        // first key this step appends in this item's range: tiles below it never wait
        // for the fused append (new rows are the recomputed kv positions + the window)
        int first_new = 0x7FFFFFFF;
        if (need_append) {
          const int n_tok_u = __shfl_sync(0xFFFFFFFFu, u.n_tok, 0);
          for (int i = lane; i < n_tok_u; i += 32) first_new = min(first_new, u.qpos[i]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) first_new = min(first_new, __shfl_xor_sync(0xFFFFFFFFu, first_new, o));
          first_new += __shfl_sync(0xFFFFFFFFu, u.prompt, 0);
        }
        if (is_k) {
          const int tok_begin = __shfl_sync(0xFFFFFFFFu, u.tok_begin, 0);
          mbar_wait(q_empty, (unit & 1) ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(q_full, q_tx);
            for (int kb = 0; kb < KB; ++kb)
              tma_load_4d(sQ + kb * (kBlockM * 128), &tm_q, q_full, kb * 64, 0, head, tok_begin);
          }
          __syncwarp();
        }
        for (int kt = key_begin; kt < key_end; kt += kTileN, ++tile_ctr) {
          const int st = tile_ctr % NST;
          int n_chunks = (min(kTileN, key_end - kt) + p.box_rows - 1) / p.box_rows;
          if (n_chunks > chunks_per_tile) n_chunks = chunks_per_tile;
          if (is_k && lane == 0) trace(p, 0, tile_ctr);
          if (need_append && kt + kTileN > first_new) {
            // this tile holds rows appended in this step: wait for the append once
            mbar_wait(append_done, 0);
            need_append = false;
          }
          mbar_wait(&empty[st], ((tile_ctr / NST) & 1) ^ 1);
          if (lane == 0) trace(p, is_k ? 4 : 10, tile_ctr);
          uint8_t* dst = ring + st * L::KT_BYTES;
          const int pg_lane = lane < n_chunks ? u.pages[((kt + lane * p.box_rows) >> shift) - pg0] : 0;
          if (elect_one()) mbar_arrive_expect_tx(&full[st], n_chunks * chunk_tx);
          for (int c = 0; c < n_chunks; ++c) {
            const int s0 = kt + c * p.box_rows;
            const int page = __shfl_sync(0xFFFFFFFFu, pg_lane, c);
            if (elect_one()) {
              for (int kb = 0; kb < KB; ++kb) {
                if (p.dbg & 32)
                  tma_load_4d(dst + kb * (kTileN * 128) + c * p.box_rows * 128, tm, &full[st], kb * 64,
                              s0 & pmask, head, page);
                else
                  tma_load_4d_hint(dst + kb * (kTileN * 128) + c * p.box_rows * 128, tm, &full[st],
                                   kb * 64, s0 & pmask, head, page, pol_stream);
              }
            }
          }
          __syncwarp();
          if (lane == 0) trace(p, is_k ? 5 : 11, tile_ctr);
        }
        if (elect_one()) mbar_arrive(&info_empty[ib]);
        __syncwarp();
      }
    } else if (warp == 9) {
      // ------------------------------------------------------------ MMA issuer
      // One stream of tiles over the CTA's work items.  S(t) = Q K^T goes to S/P buffer
      // t % 3 with A = the item's Q tile in TMEM (copied from smem by tcgen05.cp when
      // the S stream enters the item) and B = the K tile; PV(t) accumulates
      // P(t) (TMEM, TS-MMA) x V into O_{j&1} of its item.  S runs three tiles ahead
      // of PV, across item boundaries: the in-order tensor pipe retires PV(t) before
      // S(t+3) overwrites the buffer holding P(t), and the last S of an item before the
      // next item's Q copy overwrites the Q columns.  The whole warp runs the loop
      // (warp-uniform operands in uniform registers); one elected lane issues.
      constexpr uint32_t idesc_s = umma_idesc_bf16(kBlockM, kTileN, false, false);
      // PV: A = P from TMEM, B = V (MN-major).  fp16 V cache: one fp16 P plane;
      // bf16 V cache: P = hi + lo bf16 planes, two MMAs per k-step.
      constexpr uint32_t idesc_o = VF16 ? umma_idesc_f16(kBlockM, HD, false, true, 0u, 0u)
                                        : umma_idesc_bf16(kBlockM, HD, false, true);
      const uint32_t sQ_a = smem_u32(sQ), sK_a = smem_u32(sK), sV_a = smem_u32(sV);
      const int n_units = w_end - w_begin;
      int s_unit = -1, s_j = 0, s_n = 0, s_cnt = 0;  // S stream cursor
      auto s_more = [&]() { return s_j < s_n || s_unit + 1 < n_units; };
      auto issue_s = [&]() {
        if (s_j == s_n) {
          // enter the next item: its record gives the tile count, its Q tile goes to TMEM
          ++s_unit;
          s_j = 0;
          mbar_wait(&info_full[s_unit % kInfo], (s_unit / kInfo) & 1);
          s_n = __shfl_sync(0xFFFFFFFFu, epi[(s_unit % kEpiRing) * kEpiInts + 4], 0);
          mbar_wait(q_full, s_unit & 1);
          tc_fence_after();
          const uint64_t q0 = umma_sdesc_sw128(sQ_a, 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks)
              tmem_cp_128x256b(tm_qt + ks * 8, q0 + (((ks >> 2) * (kBlockM * 128) + (ks & 3) * 32) >> 4));
            umma_commit(q_empty);  // the smem tile is free once the copies land
          }
          __syncwarp();
        }
        const int t = s_cnt;
        const int b = t % kSBuf;
        const int st = t % KST;
        if (lane == 0) trace(p, 12, t);
        mbar_wait(&k_full[st], (t / KST) & 1);
        tc_fence_after();
        if (lane == 0) trace(p, 1, t);
        const uint32_t d = tm_s0 + b * kTileN;
        const uint64_t b0 = umma_sdesc_sw128(sK_a + st * L::KT_BYTES, 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            if (p.dbg & 2) break;
            // +32 B per k-step inside a 128 B swizzle row, +one 64-column box per 4
            const uint64_t db = ((ks >> 2) * (kTileN * 128) + (ks & 3) * 32) >> 4;
            umma_bf16_ts(d, tm_qt + ks * 8, b0 + db, idesc_s, ks > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[b]);
          umma_commit(&k_empty[st]);
        }
        __syncwarp();
        ++s_cnt;
        ++s_j;
      };
      for (int i = 0; i < kSBuf && s_more(); ++i) issue_s();
      int t = 0;  // PV stream position
      for (int u = 0; u < n_units; ++u) {
        const int n_tiles = __shfl_sync(0xFFFFFFFFu, epi[(u % kEpiRing) * kEpiInts + 4], 0);
        mbar_wait(o_empty, u & 1);  // O zeroed (u = 0) / the previous item's epilogue has read O_0/O_1
        tc_fence_after();
        for (int j = 0; j < n_tiles; ++j, ++t) {
          const int h = j & 1;
          const int b = t % kSBuf;
          const int st = t % VST;
          if (lane == 0) trace(p, 8, t);
          mbar_wait(&v_full[st], (t / VST) & 1);
          if (lane == 0) trace(p, 9, t);
          mbar_wait(&p_full[b], (t / kSBuf) & 1);
          tc_fence_after();
          if (lane == 0) trace(p, 7, t);
          const uint32_t d = tm_o0 + h * HD;
          const uint32_t pa = tm_s0 + b * kTileN;  // P (hi) at +0..31, bf16 lo plane at +32..63
          const uint64_t b0 = umma_sdesc_sw128(sV_a + st * L::KT_BYTES, kTileN * 128, 1024);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < kTileN / 16; ++ks) {
              if (p.dbg & 8) break;
              const uint64_t bd = b0 + ((ks * 16 * 128) >> 4);  // 16 keys = 16 rows of 128 B
              umma_bf16_ts(d, pa + ks * 8, bd, idesc_o, (j > 1 || ks > 0) ? 1u : 0u);
              if (!VF16 && !(p.dbg & 1)) umma_bf16_ts(d, pa + 32 + ks * 8, bd, idesc_o, 1u);
            }
            umma_commit(&pv_done[b]);
            umma_commit(&v_empty[st]);
            // the item's accumulator is complete after its last PV
            if (j == n_tiles - 1) umma_commit(o_full);
          }
          __syncwarp();
          if (s_more()) issue_s();
        }
      }
    } else if (warp == 11) {
      // ------------------------------------------------------------ metadata warp
      // Stages work items into the kInfo-deep record ring.  The work records and the
      // per-request scalars of up to 32 items are fetched once per batch (lane k holds
      // item k); per item the warp then only issues asynchronous 4-byte copies of the
      // page ids, query positions and visibility words, so several items' copies are
      // in flight at once and the ring fills at the memory system's throughput, not
      // one dependent round trip chain per item.
      for (int base = w_begin; base < w_end; base += 32) {
        const int nb = min(32, w_end - base);
        int f[8];
        if (lane < nb) {
          const int4* wp = reinterpret_cast<const int4*>(p.work + 8 * (base + lane));
          const int4 a = __ldg(wp), b = __ldg(wp + 1);
          f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = 0;
        }
        int prompt_l = 0, vb_l = 0, voff_l = 0;
        if (lane < nb) {
          prompt_l = __ldg(p.prompt_len + f[0]);
          vb_l = __ldg(p.vis_base + f[0]);
          voff_l = __ldg(p.vis_off + f[0]);
        }
        for (int k = 0; k < nb; ++k) {
          const int unit = base - w_begin + k;
          const int ib = unit % kInfo;
          const int req = __shfl_sync(0xFFFFFFFFu, f[0], k);
          const int head = __shfl_sync(0xFFFFFFFFu, f[1], k);
          const int tok_begin = __shfl_sync(0xFFFFFFFFu, f[2], k);
          const int n_tok = __shfl_sync(0xFFFFFFFFu, f[3], k);
          const int key_begin = __shfl_sync(0xFFFFFFFFu, f[4], k);
          const int key_end = __shfl_sync(0xFFFFFFFFu, f[5], k);
          const int slot = __shfl_sync(0xFFFFFFFFu, f[6], k);
          mbar_wait(&info_empty[ib], ((unit / kInfo) & 1) ^ 1);
          UnitInfo& u = info[ib];
          const int pg0 = key_begin >> p.page_shift;
          const int npg = min(((key_end - 1) >> p.page_shift) - pg0 + 1, kMaxUnitPages);
          const int32_t* bt = p.block_tables + static_cast<int64_t>(req) * p.max_pages + pg0;
          for (int i = lane; i < npg; i += 32) cp_async_4(&u.pages[i], bt + i);
          for (int i = lane; i < n_tok; i += 32) cp_async_4(&u.qpos[i], p.q_pos + tok_begin + i);
          cp_async_arrive_noinc(&pg_full[ib]);
          if (lane < 7) {
            const int v = lane == 0 ? req : lane == 1 ? head : lane == 2 ? tok_begin : lane == 3 ? n_tok
                        : lane == 4 ? key_begin : lane == 5 ? key_end : slot;
            (&u.req)[lane] = v;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&pg_full[ib]);
          // the request's scalars (loaded for the batch, in flight beside the copies above)
          const int prompt = __shfl_sync(0xFFFFFFFFu, prompt_l, k);
          const int vb = __shfl_sync(0xFFFFFFFFu, vb_l, k);
          const int voff = __shfl_sync(0xFFFFFFFFu, voff_l, k);
          const int nw = key_end > vb ? (key_end - vb + 31) / 32 : 0;
          if (nw <= kMaxUnitWords && lane < nw) cp_async_4(&u.words[lane], p.vis_words + voff + lane);
          cp_async_arrive_noinc(&info_full[ib]);
          if (lane < kEpiInts) {
            const int n_tiles = (key_end - key_begin + kTileN - 1) / kTileN;
            const int v = lane == 0 ? head : lane == 1 ? tok_begin : lane == 2 ? n_tok
                        : lane == 3 ? slot : lane == 4 ? n_tiles : 0;
            epi[(unit % kEpiRing) * kEpiInts + lane] = v;
          }
          if (lane >= 7 && lane < 11) {
            const int v = lane == 7 ? vb : lane == 8 ? nw : lane == 9 ? voff : prompt;
            (&u.req)[lane] = v;
          }
          __syncwarp();
          if (lane == 0) {
            trace(p, 6, 5 + unit);
            mbar_arrive(&info_full[ib]);
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kMathRegs));
    // ------------------------------------------------------------ softmax + epilogue
    // Two warpgroups ping-pong over the tiles of a work item (h = tile & 1), each
    // with its own running max m_h, sum l_h and TMEM accumulator O_h; the epilogue
    // merges (m_0, l_0, O_0) and (m_1, l_1, O_1) like two key splits.
    const int wg = warp >> 2;                   // this warpgroup
    const int wq = warp & 3;                    // TMEM lane quarter
    const int row = wq * 32 + lane;             // query row == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const int G = p.group;
    const int t_in = row / G;
    const int g_in = row - t_in * G;
    const bool row_exists = t_in < p.tok_per_tile;
    const float sc = p.scale_log2;
    if (p.k_new != nullptr) {
      // Fused KV append (K1): while the first tiles are in flight, the softmax
      // threads scatter the new K/V rows of this CTA's items into the pages.  Item i
      // appends token t for its head iff s = prompt + q_pos[t] lies in its key
      // range: the pieces of a (request, head) partition its keys, so every appended
      // row is read only by the CTA that wrote it.  One warp per (item, token) pair,
      // lanes [0, HD/8) copy K and [HD/8, HD/4) copy V in 16-byte vectors.
      grid_dep_wait();  // k_new / v_new are written by the preceding kernel
      if (threadIdx.x == 0) trace(p, 6, 250);
      int* app = reinterpret_cast<int*>(smem + L::OFF_APP);  // [kAppItems][8] + prefix
      int* pre = app + kAppItems * 8;
      constexpr int VPH = HD / 8;
      const int hkv = p.num_kv_heads;
      bool issued = false;
      for (int base = w_begin; base < w_end; base += kAppItems) {
        const int nb = min(kAppItems, w_end - base);
        if (threadIdx.x < nb) {
          const int4* wp = reinterpret_cast<const int4*>(p.work + 8 * (base + threadIdx.x));
          const int4 a = __ldg(wp), b = __ldg(wp + 1);
          int* r = app + 8 * threadIdx.x;
          r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y;
          r[6] = p.slot_abs != nullptr ? 0 : __ldg(p.prompt_len + a.x);
        }
        named_bar_sync(1, 256);
        if (threadIdx.x == 0) {
          int acc = 0;
          for (int i = 0; i < nb; ++i) {
            pre[i] = acc;
            acc += app[8 * i + 3];
          }
          pre[nb] = acc;
        }
        named_bar_sync(1, 256);
        const int total = pre[nb];
        const int kind = lane / VPH;  // 0: K row, 1: V row, else idle
        const int c = lane - kind * VPH;
        // B pairs per warp per pass: all of a pass's loads are issued before any
        // store, and the first pass's issue releases the TMA producers (so these
        // loads sit ahead of the page stream in the DRAM queues)
        constexpr int B = 12;
        for (int q0 = warp; q0 < total; q0 += 8 * B) {
          uint4 val[B];
          int2 sa[B];  // {absolute position, slot}; x = -1: nothing to write
#pragma unroll
          for (int k = 0; k < B; ++k) {
            const int q = q0 + 8 * k;
            sa[k] = make_int2(-1, 0);
            if (q < total && kind < 2) {
              int it = 0;
              while (it + 1 < nb && pre[it + 1] <= q) ++it;
              const int* r = app + 8 * it;
              const int tok = r[2] + (q - pre[it]);
              const void* src = kind == 0 ? p.k_new : p.v_new;
              val[k] = __ldg(reinterpret_cast<const uint4*>(src) +
                             (static_cast<int64_t>(tok) * p.new_stride_tok + r[1] * HD) / 8 + c);
              if (p.slot_abs != nullptr) {
                // per-step slot map: one round trip, in parallel with the row load
                sa[k] = __ldg(reinterpret_cast<const int2*>(p.slot_abs) + tok);
              } else {
                const int s_abs = r[6] + __ldg(p.q_pos + tok);
                const int page = __ldg(p.block_tables + static_cast<int64_t>(r[0]) * p.max_pages +
                                       (s_abs >> p.page_shift));
                sa[k] = make_int2(s_abs, page * p.page_size + (s_abs & (p.page_size - 1)));
              }
            }
          }
          if (!issued) {
            mbar_arrive(append_issued);
            issued = true;
          }
#pragma unroll
          for (int k = 0; k < B; ++k) {
            const int q = q0 + 8 * k;
            if (sa[k].x < 0) continue;
            int it = 0;
            while (it + 1 < nb && pre[it + 1] <= q) ++it;
            const int* r = app + 8 * it;
            if (sa[k].x < r[4] || sa[k].x >= r[5]) continue;  // another piece's key range
            const int tok = r[2] + (q - pre[it]);
            const int head = r[1];
            const int slot = sa[k].y;
            const int64_t page = slot >> p.page_shift;
            const int off = slot & (p.page_size - 1);
            const int64_t dst = ((page * hkv + head) * p.page_size + off) * VPH + c;
            if (kind == 0) {
              reinterpret_cast<uint4*>(p.k_cache_w)[dst] = val[k];
              if (head == 0 && c == 0 && p.slot_out != nullptr) p.slot_out[tok] = slot;
            } else if (p.v_fp16) {
              const uint32_t w4[4] = {val[k].x, val[k].y, val[k].z, val[k].w};
              uint32_t hv[4];
              bool sat = false;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float lo = __uint_as_float(w4[i] << 16), hi = __uint_as_float(w4[i] & 0xFFFF0000u);
                sat |= fabsf(lo) > 65504.f || fabsf(hi) > 65504.f;
                asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(hv[i]) : "f"(hi), "f"(lo));
              }
              if (__builtin_expect(sat, 0)) atomicOr(&g_v_saturated_k2, 1);
              reinterpret_cast<uint4*>(p.v_cache_w)[dst] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
            } else {
              reinterpret_cast<uint4*>(p.v_cache_w)[dst] = val[k];
            }
          }
        }
        named_bar_sync(1, 256);  // scratch reused by the next batch
      }
      if (!issued) mbar_arrive(append_issued);
      fence_proxy_async_global();
      mbar_arrive(append_done);
      if (threadIdx.x == 0) trace(p, 6, 251);
    }
    int cw = 0;     // tiles processed by this warpgroup (trace index)
    int tbase = 0;  // stream index of the current item's first tile
    int unit = 0;
    for (int w = w_begin; w < w_end; ++w, ++unit) {
      const int ib = unit % kInfo;
      mbar_wait(&info_full[ib], (unit / kInfo) & 1);
      const UnitInfo& u = info[ib];
      const int n_tok = u.n_tok;
      const int key_begin = u.key_begin, key_end = u.key_end;
      const int n_tiles = (key_end - key_begin + kTileN - 1) / kTileN;
      const bool valid = row_exists && t_in < n_tok;
      const bool warp_valid = (wq * 32) / G < n_tok;  // first row of this warp is a real token
      const int vb = u.vb;
      const bool words_smem = u.n_words <= kMaxUnitWords;
      const uint32_t* words = words_smem ? u.words : p.vis_words + u.vis_off;
      const int lim = valid ? min(u.prompt + (u.qpos[t_in] / p.block_size + 1) * p.block_size, key_end) : 0;
      float m = -INFINITY;
      float l = 0.f;
      for (int j = wg; j < n_tiles; j += 2, ++cw) {
        const int t = tbase + j;
        const int b = t % kSBuf;
        const uint32_t tsp = tm_s0 + lane_off + b * kTileN;  // this tile's S/P
        mbar_wait(&s_full[b], (t / kSBuf) & 1);
        tc_fence_after();
        if (threadIdx.x == 0) trace(p, 2, cw);
        if (warp_valid && !(p.dbg & 4)) {
          uint32_t sr[2][32];
          tmem_ld32(tsp, sr[0]);
          tmem_ld32(tsp + 32, sr[1]);
          const int kt = key_begin + j * kTileN;
          // visibility of the 64 keys of this tile for this row
          uint64_t vis = ~0ull;
          if (kt + kTileN > lim || kt + kTileN > vb) {
            uint32_t lo = 0xFFFFFFFFu, hi = 0xFFFFFFFFu;
            if (kt + 32 > vb && kt < lim) lo = words[(kt - vb) >> 5];
            if (kt + 64 > vb && kt + 32 < lim) hi = words[(kt + 32 - vb) >> 5];
            vis = (static_cast<uint64_t>(hi) << 32) | lo;
            const int n = lim - kt;
            vis &= n >= 64 ? ~0ull : (n <= 0 ? 0ull : ((1ull << n) - 1));
          }
          tmem_wait_ld();
          float sv[64];
#pragma unroll
          for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(sr[c >> 5][c & 31]);
          if (vis != ~0ull) {
#pragma unroll
            for (int c = 0; c < 64; ++c) sv[c] = ((vis >> c) & 1ull) ? sv[c] : -INFINITY;
          }
          float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
            a0 = fmax3(a0, sv[c], sv[c + 1]);
            a1 = fmax3(a1, sv[c + 2], sv[c + 3]);
            a2 = fmax3(a2, sv[c + 4], sv[c + 5]);
            a3 = fmax3(a3, sv[c + 6], sv[c + 7]);
          }
          const float tmax = fmax3(a0, a1, fmaxf(a2, a3)) * sc;  // scale > 0
          const bool need = tmax > m + 8.0f;
          const float m_new = need ? tmax : m;
          if (j >= 2 && __any_sync(0xFFFFFFFFu, need)) {
            // O_wg holds this warpgroup's earlier tiles once its previous PV retires
            const int tp = t - 2;
            mbar_wait(&pv_done[tp % kSBuf], (tp / kSBuf) & 1);
            tc_fence_after();
            const float alpha = need ? fast_exp2(m - m_new) : 1.0f;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
              uint32_t o[32];
              const uint32_t ta = tm_o0 + lane_off + wg * HD + c0;
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
          const float neg_m = (m == -INFINITY) ? 0.f : -m;
          float r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t phi[16], plo[16];
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8) {
              const int c = half * 32 + c8 * 8;
              float e[8];
#pragma unroll
              for (int q = 0; q < 8; q += 2)
                ffma2(e[q], e[q + 1], sv[c + q], sv[c + q + 1], sc, sc, neg_m, neg_m);
#pragma unroll
              for (int q = 0; q < 8; ++q) e[q] = fast_exp2(e[q]);
              fadd2(r0, r1, r0, r1, e[0], e[1]);
              fadd2(r2, r3, r2, r3, e[2], e[3]);
              fadd2(r0, r1, r0, r1, e[4], e[5]);
              fadd2(r2, r3, r2, r3, e[6], e[7]);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if constexpr (VF16) {
                  phi[c8 * 4 + q] = pack_f16x2(e[2 * q], e[2 * q + 1]);
                } else {
                  const uint32_t hb = pack_bf16x2(e[2 * q], e[2 * q + 1]);
                  float d0, d1;
                  fadd2(d0, d1, e[2 * q], e[2 * q + 1], -__uint_as_float(hb << 16),
                        -__uint_as_float(hb & 0xFFFF0000u));
                  phi[c8 * 4 + q] = hb;
                  plo[c8 * 4 + q] = pack_bf16x2(d0, d1);
                }
              }
            }
            // P overwrites this tile's S columns: plane [0,32) (and the bf16 lo
            // plane [32,64)); 64 keys are 32 packed 16-bit pairs per plane.
            tmem_st16(tsp + half * 16, phi);
            if constexpr (!VF16) tmem_st16(tsp + 32 + half * 16, plo);
          }
          l += (r0 + r1) + (r2 + r3);
          tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(&p_full[b]);
        if (threadIdx.x == 0) trace(p, 3, cw);
      }
      mbar_arrive(&info_empty[ib]);
      {  // this warpgroup's (m, l) of the item, for the epilogue warpgroup (two slots by
         // item parity; slot reuse waits until the item two back was read)
        if (unit >= 2) mbar_wait(&red_empty[unit & 1], ((unit >> 1) - 1) & 1);
        float* rw = red + (unit & 1) * 4 * kBlockM;
        rw[(0 * 2 + wg) * kBlockM + row] = m;
        rw[(1 * 2 + wg) * kBlockM + row] = l;
        mbar_arrive(&red_full[unit & 1]);
      }
      tbase += n_tiles;
    }
  }
  grid_dep_launch();
  if (threadIdx.x == 256) trace(p, 6, 2);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 10) tmem_dealloc<L::TMEM_COLS>(tmem_base);
  if (threadIdx.x == 320) {
    trace(p, 6, 3);
    trace(p, 6, 4);  // globaltimer at the end: cycles / ns = the SM clock under load
  }
}

// Split-KV combine: merge the (m, l, O) partials of every split query tile.
// One warp per output row (one block per (group, 8-row slab) pair): lane s reads the
// (m, l) of split s, the warp reduces the merged max / denominator with shuffles,
// then every lane accumulates a 4-column float4 slice over the splits.
template <int HD>
__global__ void __launch_bounds__(256) attn_combine_kernel(const int32_t* __restrict__ groups,
                                                           const float* __restrict__ ws_o,
                                                           const float* __restrict__ ws_ml,
                                                           __nv_bfloat16* __restrict__ out,
                                                           int64_t out_stride_tok, int group_sz,
                                                           int n_groups,
                                                           const int32_t* __restrict__ n_groups_dev) {
  // device-planned steps: the group count is read from device memory and the grid,
  // sized for capacity, strides over the groups
  if (n_groups_dev != nullptr) n_groups = *n_groups_dev;
  constexpr int kSlabs = kBlockM / 8;  // 8-row slabs per group (one warp per row)
  const int lane = threadIdx.x & 31;
  for (int idx = blockIdx.x; idx < n_groups * kSlabs; idx += gridDim.x) {
    const int gi = idx / kSlabs;
    const int r = (idx - gi * kSlabs) * 8 + (threadIdx.x >> 5);
    const int* gr = groups + 8 * gi;
    const int head = gr[1], tok_begin = gr[2], n_tok = gr[3], slot0 = gr[4], n_split = gr[5];
    if (r >= n_tok * group_sz) continue;
    grid_dep_wait();  // partials of the preceding attention grid are visible after this
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
}

// Launch the combine with PDL after the attention grid: one block per (group, 8-row
// slab).  n_groups_dev != nullptr: the count is on the device and a grid of at most
// 128 blocks strides over the (group, slab) pairs (cheap when there are none).
template <int HD>
static int launch_combine_t(const AttnParams& prm, const int32_t* groups, int n_groups,
                            const int32_t* n_groups_dev, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  const int pairs = n_groups * (kBlockM / 8);
  cfg.gridDim = dim3(n_groups_dev ? (pairs < 128 ? pairs : 128) : pairs);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, attn_combine_kernel<HD>, groups,
                                             static_cast<const float*>(prm.ws_o),
                                             static_cast<const float*>(prm.ws_ml), prm.out,
                                             prm.out_stride_tok, prm.group, n_groups, n_groups_dev));
}

int launch_attn_combine_dev(int head_dim, const AttnParams& prm, const int32_t* groups, int max_groups,
                            const int32_t* n_groups_dev, cudaStream_t stream) {
  if (max_groups <= 0) return 0;
  return head_dim == 128 ? launch_combine_t<128>(prm, groups, max_groups, n_groups_dev, stream)
                         : launch_combine_t<64>(prm, groups, max_groups, n_groups_dev, stream);
}

template <int HD, int KST, int VST, bool VF16>
static int launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const AttnParams& prm, int grid, const int32_t* groups, int n_groups,
                         cudaStream_t stream) {
  using L = AttnSmem<HD, KST, VST>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(paged_attn_kernel<HD, KST, VST, VF16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  if (grid > 0) {
    // Launched with programmatic stream serialization: the prologue (barriers, TMEM,
    // work-item staging) overlaps the previous kernel; the TMA producers execute
    // griddepcontrol.wait before their first load.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L::ALLOC;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, paged_attn_kernel<HD, KST, VST, VF16>, tq, tk, tv, prm);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  if (n_groups > 0) {
    // PDL: the combine's CTAs are resident before K2 drains; they wait on
    // griddepcontrol.wait before reading the partials.
    cudaError_t e = static_cast<cudaError_t>(launch_combine_t<HD>(prm, groups, n_groups, nullptr, stream));
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

int launch_paged_attn(int head_dim, bool v_fp16, const CUtensorMap& tq, const CUtensorMap& tk,
                      const CUtensorMap& tv, const AttnParams& prm, int grid,
                      const int32_t* groups, int n_groups, cudaStream_t stream) {
  // 227 KB of shared memory: one Q tile + the K ring + a deeper V ring (a V slot is
  // held until its PV retires, a K slot only until its S does).
  if (head_dim == 128) {
    // Shallow rings measured fastest (3/3 vs 5/6: -10% on the ShareGPT batch, -4% at
    // 4K): every CTA keeps ~96-128 KB in flight, enough to cover the unloaded HBM
    // latency at its bandwidth share, while deeper rings only lengthen the DRAM queues
    // that every dependent step (item start, first tile, tail) waits behind.  With the
    // epilogue warpgroup 4/4 edges out 3/3 (ShareGPT K2 29.7 -> 29.3 us, 4K and
    // LongBench -1%, LLaDA +1%: profiles/r2ck_rings.md).
    const char* e = getenv("OPTIMUS_K2_RINGS");  // diagnostics: ring-depth variants
    const int rings = e ? atoi(e) : 44;
    if (rings == 44)
      return v_fp16 ? launch_attn_t<128, 4, 4, true>(tq, tk, tv, prm, grid, groups, n_groups, stream)
                    : launch_attn_t<128, 4, 4, false>(tq, tk, tv, prm, grid, groups, n_groups, stream);
    if (rings == 56)
      return v_fp16 ? launch_attn_t<128, 5, 6, true>(tq, tk, tv, prm, grid, groups, n_groups, stream)
                    : launch_attn_t<128, 5, 6, false>(tq, tk, tv, prm, grid, groups, n_groups, stream);
    return v_fp16 ? launch_attn_t<128, 3, 3, true>(tq, tk, tv, prm, grid, groups, n_groups, stream)
                  : launch_attn_t<128, 3, 3, false>(tq, tk, tv, prm, grid, groups, n_groups, stream);
  }
  if (head_dim == 64)
    return v_fp16 ? launch_attn_t<64, 6, 6, true>(tq, tk, tv, prm, grid, groups, n_groups, stream)
                  : launch_attn_t<64, 6, 6, false>(tq, tk, tv, prm, grid, groups, n_groups, stream);
  return -1;
}

}  // namespace optimus
