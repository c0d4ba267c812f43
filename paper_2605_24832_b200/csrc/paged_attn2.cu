// K2, dual-slot form — two independent attention pipelines per SM.
//
// Same computation, inputs and outputs as paged_attn_kernel (paged_attn.cu; SURVEY
// §8c rule V).  What differs is the shape of the persistent CTA: instead of one item
// stream whose two softmax warpgroups ping-pong over the tiles of an item (and must
// merge two O accumulators at every item end, stalling the item's PV stream), the
// CTA runs TWO slots, each a complete pipeline over its own work list (the host
// planner places items on 2 x #SM virtual CTAs):
//
//   slot s: warp 8+2s   stager + TMA producer: stages its items' page ids / query
//                       positions / visibility words (cp.async, one item ahead), then
//                       issues Q (SW128, into the slot's Q buffer) and its K/V tiles
//                       into the slot's own 2-stage K and V rings
//           warp 9+2s   MMA issuer: S = Q K^T (both operands from shared memory) into
//                       one of two S/P buffers, O += P V (P from TMEM) into the slot's
//                       single O accumulator; order S(t), PV(t-1)
//           warps 4s..4s+3  softmax + epilogue: thread i owns row i; online softmax with
//                       the lazy rescale; at an item end the warpgroup drains O (no
//                       merge) while the OTHER slot keeps the tensor pipe and HBM busy
//
// TMEM: per slot 2 S/P buffers (128 columns) + O (128 columns) = 256; two slots = 512.
// Shared memory per slot: Q 32 KB + K 2x16 KB + V 2x16 KB + staging ring.
#include "attn.cuh"

namespace optimus {
namespace dual {

constexpr int kTileN = 64;
constexpr int kBlockM = 128;
constexpr int kThreads = 384;
constexpr int kStg = 2;        // K and V ring stages per slot
constexpr int kInfo = 3;       // staged work-item records per slot
constexpr int kMaxUnitPages = 256;
constexpr int kMaxUnitWords = 16;

struct UnitInfo {
  int req, head, tok_begin, n_tok, key_begin, key_end, slot, vb;
  int n_words, vis_off, prompt, pad0;
  int qpos[kBlockM];
  uint32_t words[kMaxUnitWords];
  int pages[kMaxUnitPages];
};

template <int HD>
struct Smem {
  static constexpr int KB = HD / 64;
  static constexpr uint32_t Q_BYTES = KB * kBlockM * 128;
  static constexpr uint32_t KT_BYTES = KB * kTileN * 128;
  static constexpr uint32_t SLOT_BYTES = Q_BYTES + 2 * kStg * KT_BYTES;  // Q, K ring, V ring
  static constexpr uint32_t OFF_INFO = 2 * SLOT_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_INFO + 2 * kInfo * sizeof(UnitInfo);
  // per slot: k_full/empty, v_full/empty [kStg], q_full, q_empty, s_full[2], p_full[2],
  // pv_done[2], o_full, o_empty, info_full/empty [kInfo]
  static constexpr int BARS_PER_SLOT = 4 * kStg + 2 + 6 + 2 + 2 * kInfo;
  static constexpr uint32_t BYTES = OFF_BAR + 2 * BARS_PER_SLOT * 8 + 16;
  static constexpr uint32_t ALLOC = BYTES + 1024;
  static_assert(ALLOC <= 232448, "exceeds the 227 KB per-CTA shared memory of sm_100");
};

template <int HD, bool VF16>
__global__ void __launch_bounds__(kThreads, 1)
    paged_attn_dual_kernel(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using L = Smem<HD>;
  constexpr int KB = L::KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::BYTES - 16);

  const int warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0);
  const int lane = threadIdx.x & 31;
  // slot of this warp: softmax warps 0-3 -> 0, 4-7 -> 1; control warps 8,9 -> 0, 10,11 -> 1
  const int s = warp < 8 ? (warp >> 2) : ((warp - 8) >> 1);
  uint8_t* sQ = smem + s * L::SLOT_BYTES;
  uint8_t* sK = sQ + L::Q_BYTES;
  uint8_t* sV = sK + kStg * L::KT_BYTES;
  UnitInfo* info = reinterpret_cast<UnitInfo*>(smem + L::OFF_INFO) + s * kInfo;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR) + s * L::BARS_PER_SLOT;
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + kStg;
  uint64_t* v_full = k_empty + kStg;
  uint64_t* v_empty = v_full + kStg;
  uint64_t* q_full = v_empty + kStg;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_empty + 1;   // [2]
  uint64_t* p_full = s_full + 2;    // [2]
  uint64_t* pv_done = p_full + 2;   // [2]
  uint64_t* o_full = pv_done + 2;
  uint64_t* o_empty = o_full + 1;
  uint64_t* info_full = o_empty + 1;       // [kInfo]
  uint64_t* info_empty = info_full + kInfo;  // [kInfo]

  if (warp == 8 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if ((warp == 9 || warp == 11) && lane == 0) {
    for (int i = 0; i < kStg; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    for (int i = 0; i < kInfo; ++i) {
      mbar_init(&info_full[i], 33);       // 32 cp.async arrivals + lane 0's store arrival
      mbar_init(&info_empty[i], 128 + 1);  // softmax warpgroup + MMA warp
    }
    mbar_fence_init();
  }
  if (warp == 10) tmem_alloc<512>(tmem_slot);
  {
    // rows a partial tile never loads must hold finite values (P = 0 there)
    uint4* z = reinterpret_cast<uint4*>(smem);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (uint32_t i = threadIdx.x; i < 2 * L::SLOT_BYTES / 16; i += kThreads) z[i] = zero;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot + s * 256;  // this slot's 256 columns
  const uint32_t tm_sp = tmem_base;                 // two S/P buffers of 64 columns
  const uint32_t tm_o = tmem_base + 128;            // O accumulator (HD columns)

  const int vslot = 2 * blockIdx.x + s;  // virtual CTA of the planner
  const int w_begin = p.cta_off[vslot];
  const int w_end = p.cta_off[vslot + 1];
  const int n_units = w_end - w_begin;

  if (warp == 8 || warp == 10) {
    // ------------------------------------------------- stager + TMA producer (slot s)
    const int shift = p.page_shift;
    const int pmask = p.page_size - 1;
    const uint32_t q_tx = KB * 64 * p.group * p.tok_per_tile * 2;
    const uint32_t chunk_tx = p.box_rows * 128 * KB;
    const int chunks_per_tile = kTileN / p.box_rows;
    const uint64_t pol = l2_policy_evict_first();
    // work records + per-request scalars of up to 32 items, lane k holds item k
    int f[8];
    int prompt_l = 0, vb_l = 0, voff_l = 0;
    auto load_batch = [&](int base) {
      const int nb = min(32, w_end - base);
      if (lane < nb) {
        const int4* wp = reinterpret_cast<const int4*>(p.work + 8 * (base + lane));
        const int4 a = __ldg(wp), b = __ldg(wp + 1);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
        prompt_l = __ldg(p.prompt_len + f[0]);
        vb_l = __ldg(p.vis_base + f[0]);
        voff_l = __ldg(p.vis_off + f[0]);
      }
    };
    int batch_base = -1;
    auto stage = [&](int unit) {  // stage item `unit` (0-based in this slot's list)
      const int w = w_begin + unit;
      const int base = w_begin + (unit / 32) * 32;
      if (base != batch_base) {
        load_batch(base);
        batch_base = base;
      }
      const int k = w - base;
      const int ib = unit % kInfo;
      const int req = __shfl_sync(0xFFFFFFFFu, f[0], k);
      const int head = __shfl_sync(0xFFFFFFFFu, f[1], k);
      const int tok_begin = __shfl_sync(0xFFFFFFFFu, f[2], k);
      const int n_tok = __shfl_sync(0xFFFFFFFFu, f[3], k);
      const int key_begin = __shfl_sync(0xFFFFFFFFu, f[4], k);
      const int key_end = __shfl_sync(0xFFFFFFFFu, f[5], k);
      const int pslot = __shfl_sync(0xFFFFFFFFu, f[6], k);
      const int prompt = __shfl_sync(0xFFFFFFFFu, prompt_l, k);
      const int vb = __shfl_sync(0xFFFFFFFFu, vb_l, k);
      const int voff = __shfl_sync(0xFFFFFFFFu, voff_l, k);
      mbar_wait(&info_empty[ib], ((unit / kInfo) & 1) ^ 1);
      UnitInfo& u = info[ib];
      const int pg0 = key_begin >> shift;
      const int npg = min(((key_end - 1) >> shift) - pg0 + 1, kMaxUnitPages);
      const int32_t* bt = p.block_tables + static_cast<int64_t>(req) * p.max_pages + pg0;
      for (int i = lane; i < npg; i += 32) cp_async_4(&u.pages[i], bt + i);
      for (int i = lane; i < n_tok; i += 32) cp_async_4(&u.qpos[i], p.q_pos + tok_begin + i);
      const int nw = key_end > vb ? (key_end - vb + 31) / 32 : 0;
      if (nw <= kMaxUnitWords && lane < nw) cp_async_4(&u.words[lane], p.vis_words + voff + lane);
      cp_async_arrive_noinc(&info_full[ib]);
      if (lane < 11) {
        const int v = lane == 0 ? req : lane == 1 ? head : lane == 2 ? tok_begin : lane == 3 ? n_tok
                    : lane == 4 ? key_begin : lane == 5 ? key_end : lane == 6 ? pslot : lane == 7 ? vb
                    : lane == 8 ? nw : lane == 9 ? voff : prompt;
        (&u.req)[lane] = v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_full[ib]);
    };
    if (n_units > 0) stage(0);
    int tile = 0;
    for (int unit = 0; unit < n_units; ++unit) {
      if (unit + 1 < n_units) stage(unit + 1);  // one item ahead
      const int ib = unit % kInfo;
      mbar_wait(&info_full[ib], (unit / kInfo) & 1);
      if (unit == 0) grid_dep_wait();  // Q / K / V come from the preceding kernels
      const UnitInfo& u = info[ib];
      const int head = __shfl_sync(0xFFFFFFFFu, u.head, 0);
      const int tok_begin = __shfl_sync(0xFFFFFFFFu, u.tok_begin, 0);
      const int key_begin = __shfl_sync(0xFFFFFFFFu, u.key_begin, 0);
      const int key_end = __shfl_sync(0xFFFFFFFFu, u.key_end, 0);
      const int pg0 = key_begin >> shift;
      mbar_wait(q_empty, (unit & 1) ^ 1);  // the previous item's S MMAs have read Q
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, q_tx);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_4d(sQ + kb * (kBlockM * 128), &tm_q, q_full, kb * 64, 0, head, tok_begin);
      }
      __syncwarp();
      for (int kt = key_begin; kt < key_end; kt += kTileN, ++tile) {
        const int st = tile % kStg;
        int n_chunks = (min(kTileN, key_end - kt) + p.box_rows - 1) / p.box_rows;
        if (n_chunks > chunks_per_tile) n_chunks = chunks_per_tile;
        const int pg_lane = lane < n_chunks ? u.pages[((kt + lane * p.box_rows) >> shift) - pg0] : 0;
        for (int kv = 0; kv < 2; ++kv) {
          const CUtensorMap* tm = kv ? &tm_v : &tm_k;
          uint64_t* full = kv ? v_full : k_full;
          uint64_t* empty = kv ? v_empty : k_empty;
          uint8_t* dst = (kv ? sV : sK) + st * L::KT_BYTES;
          mbar_wait(&empty[st], ((tile / kStg) & 1) ^ 1);
          if (elect_one()) mbar_arrive_expect_tx(&full[st], n_chunks * chunk_tx);
          for (int c = 0; c < n_chunks; ++c) {
            const int s0 = kt + c * p.box_rows;
            const int page = __shfl_sync(0xFFFFFFFFu, pg_lane, c);
            if (elect_one()) {
              for (int kb = 0; kb < KB; ++kb)
                tma_load_4d_hint(dst + kb * (kTileN * 128) + c * p.box_rows * 128, tm, &full[st], kb * 64,
                                 s0 & pmask, head, page, pol);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 9 || warp == 11) {
    // ------------------------------------------------------------- MMA issuer (slot s)
    constexpr uint32_t idesc_s = umma_idesc_bf16(kBlockM, kTileN, false, false);
    constexpr uint32_t idesc_o = VF16 ? umma_idesc_f16(kBlockM, HD, false, true, 0u, 0u)
                                      : umma_idesc_bf16(kBlockM, HD, false, true);
    const uint32_t sQ_a = smem_u32(sQ), sK_a = smem_u32(sK), sV_a = smem_u32(sV);
    int t = 0;  // slot-local tile stream
    for (int unit = 0; unit < n_units; ++unit) {
      const int ib = unit % kInfo;
      mbar_wait(&info_full[ib], (unit / kInfo) & 1);
      const int n_tiles = __shfl_sync(0xFFFFFFFFu, (info[ib].key_end - info[ib].key_begin + kTileN - 1) / kTileN, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_empty[ib]);  // the record was read (n_tiles)
      mbar_wait(q_full, unit & 1);
      tc_fence_after();
      for (int j = 0; j <= n_tiles; ++j) {
        if (j < n_tiles) {
          // S(t+j) = Q K^T into S/P buffer (t+j) & 1; that buffer's P(t+j-2) was consumed
          // by PV(t+j-2), issued earlier in this in-order stream
          const int tt = t + j;
          const int st = tt % kStg;
          mbar_wait(&k_full[st], (tt / kStg) & 1);
          tc_fence_after();
          const uint32_t d = tm_sp + (tt & 1) * kTileN;
          const uint64_t a0 = umma_sdesc_sw128(sQ_a, 16, 1024);
          const uint64_t b0 = umma_sdesc_sw128(sK_a + st * L::KT_BYTES, 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks) {
              const uint64_t da = ((ks >> 2) * (kBlockM * 128) + (ks & 3) * 32) >> 4;
              const uint64_t db = ((ks >> 2) * (kTileN * 128) + (ks & 3) * 32) >> 4;
              umma_bf16_ss(d, a0 + da, b0 + db, idesc_s, ks > 0 ? 1u : 0u);
            }
            umma_commit(&s_full[tt & 1]);
            umma_commit(&k_empty[st]);
            if (j == n_tiles - 1) umma_commit(q_empty);  // Q read by the item's last S
          }
          __syncwarp();
        }
        if (j >= 1) {
          // O += P V for tile t+j-1
          const int tt = t + j - 1;
          const int st = tt % kStg;
          if (j == 1) {
            mbar_wait(o_empty, (unit & 1) ^ 1);  // the previous item's epilogue drained O
            tc_fence_after();
          }
          mbar_wait(&v_full[st], (tt / kStg) & 1);
          mbar_wait(&p_full[tt & 1], (tt >> 1) & 1);
          tc_fence_after();
          const uint32_t pa = tm_sp + (tt & 1) * kTileN;
          const uint64_t b0 = umma_sdesc_sw128(sV_a + st * L::KT_BYTES, kTileN * 128, 1024);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < kTileN / 16; ++ks) {
              const uint64_t bd = b0 + ((ks * 16 * 128) >> 4);
              umma_bf16_ts(tm_o, pa + ks * 8, bd, idesc_o, (j > 1 || ks > 0) ? 1u : 0u);
              if (!VF16) umma_bf16_ts(tm_o, pa + 32 + ks * 8, bd, idesc_o, 1u);
            }
            umma_commit(&pv_done[tt & 1]);
            umma_commit(&v_empty[st]);
            if (j == n_tiles) umma_commit(o_full);
          }
          __syncwarp();
        }
      }
      t += n_tiles;
    }
  } else {
    // ------------------------------------------------- softmax + epilogue (slot s)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const int G = p.group;
    const int t_in = row / G;
    const int g_in = row - t_in * G;
    const bool row_exists = t_in < p.tok_per_tile;
    const float sc = p.scale_log2;
    int t = 0;
    for (int unit = 0; unit < n_units; ++unit) {
      const int ib = unit % kInfo;
      mbar_wait(&info_full[ib], (unit / kInfo) & 1);
      const UnitInfo& u = info[ib];
      const int n_tok = u.n_tok;
      const int key_begin = u.key_begin, key_end = u.key_end;
      const int n_tiles = (key_end - key_begin + kTileN - 1) / kTileN;
      const bool valid = row_exists && t_in < n_tok;
      const bool warp_valid = (wq * 32) / G < n_tok;
      const int vb = u.vb;
      const bool words_smem = u.n_words <= kMaxUnitWords;
      const uint32_t* words = words_smem ? u.words : p.vis_words + u.vis_off;
      const int lim = valid ? min(u.prompt + (u.qpos[t_in] / p.block_size + 1) * p.block_size, key_end) : 0;
      const int head = u.head, tok_begin = u.tok_begin, pslot = u.slot;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int tt = t + j;
        const uint32_t tsp = tm_sp + lane_off + (tt & 1) * kTileN;
        mbar_wait(&s_full[tt & 1], (tt >> 1) & 1);
        tc_fence_after();
        if (warp_valid) {
          uint32_t sr[2][32];
          tmem_ld32(tsp, sr[0]);
          tmem_ld32(tsp + 32, sr[1]);
          const int kt = key_begin + j * kTileN;
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
          const float tmax = fmax3(a0, a1, fmaxf(a2, a3)) * sc;
          const bool need = tmax > m + 8.0f;
          const float m_new = need ? tmax : m;
          if (j >= 1 && __any_sync(0xFFFFFFFFu, need)) {
            // O holds tiles < j once PV(tt-1) retired
            mbar_wait(&pv_done[(tt - 1) & 1], ((tt - 1) >> 1) & 1);
            tc_fence_after();
            const float alpha = need ? fast_exp2(m - m_new) : 1.0f;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 32) {
              uint32_t o[32];
              tmem_ld32(tm_o + lane_off + c0, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              tmem_st32(tm_o + lane_off + c0, o);
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
            tmem_st16(tsp + half * 16, phi);
            if constexpr (!VF16) tmem_st16(tsp + 32 + half * 16, plo);
          }
          l += (r0 + r1) + (r2 + r3);
          tmem_wait_st();
        }
        tc_fence_before();
        mbar_arrive(&p_full[tt & 1]);
      }
      mbar_arrive(&info_empty[ib]);
      // epilogue: this warpgroup owns the whole O of the item (no merge)
      mbar_wait(o_full, unit & 1);
      tc_fence_after();
      const float inv_l = (pslot < 0) ? (l > 0.f ? 1.0f / l : 0.f) : 1.f;
      const int tok = tok_begin + t_in;
      const int qh = head * G + g_in;
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t o[32];
        if (warp_valid) {
          tmem_ld32(tm_o + lane_off + c0, o);
          tmem_wait_ld();
        }
        if (valid) {
          if (pslot < 0) {
            uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<int64_t>(tok) * p.out_stride_tok +
                                                  static_cast<int64_t>(qh) * HD + c0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int c = v * 8;
              dst[v] = make_uint4(
                  pack_bf16x2(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l),
                  pack_bf16x2(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l),
                  pack_bf16x2(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l),
                  pack_bf16x2(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l));
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(
                p.ws_o + (static_cast<int64_t>(pslot) * kBlockM + row) * HD + c0);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              dst[v] = make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]),
                                   __uint_as_float(o[4 * v + 2]), __uint_as_float(o[4 * v + 3]));
          }
        }
      }
      if (valid && pslot >= 0)
        reinterpret_cast<float2*>(p.ws_ml)[static_cast<int64_t>(pslot) * kBlockM + row] = make_float2(m, l);
      tc_fence_before();
      mbar_arrive(o_empty);
      t += n_tiles;
    }
  }
  grid_dep_launch();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 10) tmem_dealloc<512>(*tmem_slot);
}

}  // namespace dual

template <int HD, bool VF16>
static int launch_dual_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const AttnParams& prm, int grid, cudaStream_t stream) {
  using L = dual::Smem<HD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(dual::paged_attn_dual_kernel<HD, VF16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dual::kThreads);
  cfg.dynamicSmemBytes = L::ALLOC;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dual::paged_attn_dual_kernel<HD, VF16>, tq, tk, tv, prm));
}

// grid = CTAs (each runs virtual CTAs 2c and 2c+1 of the work list).
int launch_paged_attn_dual(int head_dim, bool v_fp16, const CUtensorMap& tq, const CUtensorMap& tk,
                           const CUtensorMap& tv, const AttnParams& prm, int grid, cudaStream_t stream) {
  if (head_dim != 128) return -1;
  return v_fp16 ? launch_dual_t<128, true>(tq, tk, tv, prm, grid, stream)
                : launch_dual_t<128, false>(tq, tk, tv, prm, grid, stream);
}

}  // namespace optimus
