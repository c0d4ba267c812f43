// K3 — fused confidence-threshold unmask / commit.
//
// Replaces the commit decision of the reference's oracle
// (StochasticOracle.commits, pkg/src/dllmsim/commit.py:279-280 -> commit_step
// commit.py:86-112) with the model rule it stands for: a window position
// commits when its max softmax probability reaches tau (
// tau = 0.9), and every request commits at least one position per
// step (the progress rule, commit.py:103).
//
// Phase (a) streams the logits once: each CTA reduces one vocab slice of one
// window row to {max, sum exp(x - max), argmax} (12 bytes) with 16-byte vector
// loads and exp2 on the MUFU pipe.  Phase (b) merges the slices of each row in
// a fixed order (bitwise identical on every rank), forms conf = 1 / sum, and
// applies threshold + progress rule per request (one warp per request).
#include "ptx.cuh"

namespace optimus {

constexpr float kLog2e = 1.4426950408889634f;

struct Part {
  float m;    // max logit (natural units)
  float s;    // sum exp(x - m)
  int idx;    // argmax (global vocab index), lowest on ties
};

__device__ __forceinline__ void part_merge(float& m, float& s, int& idx, float m2, float s2, int i2) {
  if (m2 > m || (m2 == m && i2 < idx)) {
    // take the other side's max; rescale our sum
    const float sc = (m == -INFINITY) ? 0.f : fast_exp2((m - m2) * kLog2e);
    s = s * sc + s2;
    if (m2 > m) {
      m = m2;
    }
    idx = i2;
  } else {
    const float sc = (m2 == -INFINITY) ? 0.f : fast_exp2((m2 - m) * kLog2e);
    s += s2 * sc;
  }
}

template <typename T>
struct VecLoad;

template <>
struct VecLoad<__nv_bfloat16> {
  static constexpr int N = 8;  // elements per 16-byte vector
  __device__ static void load(const __nv_bfloat16* base, int64_t i, float (&v)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(base) + i);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = __uint_as_float(w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  }
};

template <>
struct VecLoad<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* base, int64_t i, float (&v)[4]) {
    const float4 u = __ldg(reinterpret_cast<const float4*>(base) + i);
    v[0] = u.x;
    v[1] = u.y;
    v[2] = u.z;
    v[3] = u.w;
  }
};

// Phase (b) for one request, run by one warp: merge the request's row partials in a
// fixed order, threshold, progress rule, optional state-mirror update.
__device__ __forceinline__ void finalize_request(
    int req, int lane, const Part* __restrict__ part, int n_outer, int n_rows, int n_vsplit,
    const int32_t* __restrict__ cu_rows, float tau, int fallback_mode, uint8_t* __restrict__ commit_mask,
    int32_t* __restrict__ tok_out, float* __restrict__ conf_out, const int32_t* __restrict__ row_pos,
    uint8_t* __restrict__ state, int32_t* __restrict__ token_buf, int64_t state_stride) {
  const int r0 = cu_rows[req], r1 = cu_rows[req + 1];
  bool any = false;
  float best_conf = -1.f;
  int best_row = 0x7FFFFFFF;
  for (int base = r0; base < r1; base += 32) {
    const int r = base + lane;
    bool commit = false;
    float conf = 0.f;
    int tok = -1;
    if (r < r1) {
      float M = -INFINITY, S = 0.f;
      int I = 0x7FFFFFFF;
      for (int o = 0; o < n_outer; ++o)
        for (int k = 0; k < n_vsplit; ++k) {
          const Part q = part[(static_cast<int64_t>(o) * n_rows + r) * n_vsplit + k];
          if (q.idx < 0) continue;
          part_merge(M, S, I, q.m, q.s, q.idx);
        }
      conf = S > 0.f ? 1.0f / S : 0.f;
      tok = I;
      commit = conf >= tau;
      if (fallback_mode == 0 && r == r0) commit = true;
      conf_out[r] = conf;
      tok_out[r] = tok;
      if (conf > best_conf || (conf == best_conf && r < best_row)) {
        best_conf = conf;
        best_row = r;
      }
    }
    any = any || __any_sync(0xFFFFFFFFu, commit);
    if (r < r1) commit_mask[r] = commit ? 1 : 0;
  }
  if (fallback_mode == 1 && !any && r1 > r0) {
    // highest confidence row (ties -> earliest) commits
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float c2 = __shfl_xor_sync(0xFFFFFFFFu, best_conf, o);
      const int b2 = __shfl_xor_sync(0xFFFFFFFFu, best_row, o);
      if (c2 > best_conf || (c2 == best_conf && b2 < best_row)) {
        best_conf = c2;
        best_row = b2;
      }
    }
    if (lane == 0) commit_mask[best_row] = 1;
  }
  if (state != nullptr || token_buf != nullptr) {
    __syncwarp();
    for (int r = r0 + lane; r < r1; r += 32) {
      if (commit_mask[r]) {
        const int64_t at = static_cast<int64_t>(req) * state_stride + row_pos[r];
        if (state) state[at] = 1;
        if (token_buf) token_buf[at] = tok_out[r];
      }
    }
  }
}

// One warp per request.
__global__ void __launch_bounds__(128) unmask_finalize_kernel(
    const Part* __restrict__ part, int n_outer, int n_rows, int n_vsplit,
    const int32_t* __restrict__ cu_rows, int n_req, float tau, int fallback_mode,
    uint8_t* __restrict__ commit_mask, int32_t* __restrict__ tok_out, float* __restrict__ conf_out,
    const int32_t* __restrict__ row_pos, uint8_t* __restrict__ state,
    int32_t* __restrict__ token_buf, int64_t state_stride) {
  const int req = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (req >= n_req) return;
  finalize_request(req, threadIdx.x & 31, part, n_outer, n_rows, n_vsplit, cu_rows, tau, fallback_mode,
                   commit_mask, tok_out, conf_out, row_pos, state, token_buf, state_stride);
}

// Fused phase (b) (single vocab shard): the CTA that writes a request's last partial
// (per-request arrival counter) finalizes that request, so the whole unmask is one launch.
struct FuseArgs {
  const int32_t* cu_rows;
  const int32_t* row_req;
  int32_t* counters;  // [n_req], zero between launches (the finalizing CTA resets its entry)
  int n_rows_cap;     // stride of part (rows)
  float tau;
  int fallback_mode;
  uint8_t* commit_mask;
  int32_t* tok;
  float* conf;
  const int32_t* row_pos;
  uint8_t* state;
  int32_t* token_buf;
  int64_t state_stride;
};

template <typename T, int THREADS>
__global__ void __launch_bounds__(THREADS) unmask_partial_kernel(
    const T* __restrict__ logits, int64_t row_stride, const int32_t* __restrict__ row_src,
    int vocab, int vocab_offset, int n_vsplit, Part* __restrict__ part,
    const int32_t* __restrict__ n_rows_dev, const FuseArgs fuse) {
  constexpr int N = VecLoad<T>::N;
  const int row = blockIdx.x;
  const int split = blockIdx.y;
  if (n_rows_dev != nullptr && row >= *n_rows_dev) return;  // device-planned step
  const int64_t src = row_src ? row_src[row] : row;
  const T* base = logits + src * row_stride;
  // vocab slice of this split, in whole vectors (vocab is a multiple of N here)
  const int nvec = vocab / N;
  const int per = (nvec + n_vsplit - 1) / n_vsplit;
  const int v0 = split * per;
  const int v1 = min(nvec, v0 + per);
  float m = -INFINITY, s = 0.f;
  int idx = 0x7FFFFFFF;
  // Each thread walks its vectors in increasing index order; within the thread the
  // first maximum wins (strict >), so the kept index is the lowest among equals.
  int i = v0 + threadIdx.x;
  constexpr int U = 4;
  for (; i + (U - 1) * THREADS < v1; i += U * THREADS) {
    float v[U][N];
#pragma unroll
    for (int u = 0; u < U; ++u) VecLoad<T>::load(base, i + u * THREADS, v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // vector max by a 3-input FMNMX tree; the position of the max is searched only
      // when it beats the running max (rare after the first vectors)
      float cm = v[u][0];
#pragma unroll
      for (int k = 1; k + 1 < N; k += 2) cm = fmax3(cm, v[u][k], v[u][k + 1]);
      if constexpr (N % 2 == 0) cm = fmaxf(cm, v[u][N - 1]);
      if (__builtin_expect(cm > m, 0)) {
        int ci = N - 1;
#pragma unroll
        for (int k = N - 2; k >= 0; --k) ci = (v[u][k] == cm) ? k : ci;
        s = (m == -INFINITY) ? 0.f : s * fast_exp2((m - cm) * kLog2e);
        m = cm;
        idx = (i + u * THREADS) * N + ci;
      }
      const float mb = -m * kLog2e;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int k = 0; k + 1 < N; k += 2) {
        float e0, e1;
        ffma2(e0, e1, v[u][k], v[u][k + 1], kLog2e, kLog2e, mb, mb);
        fadd2(s0, s1, s0, s1, fast_exp2(e0), fast_exp2(e1));
      }
      s += s0 + s1;
    }
  }
  for (; i < v1; i += THREADS) {
    float v[N];
    VecLoad<T>::load(base, i, v);
    float cm = v[0];
    int ci = 0;
#pragma unroll
    for (int k = 1; k < N; ++k)
      if (v[k] > cm) {
        cm = v[k];
        ci = k;
      }
    if (cm > m) {
      s = (m == -INFINITY) ? 0.f : s * fast_exp2((m - cm) * kLog2e);
      m = cm;
      idx = i * N + ci;
    }
    const float mb = m * kLog2e;
#pragma unroll
    for (int k = 0; k < N; ++k) s += fast_exp2(fmaf(v[k], kLog2e, -mb));
  }
  // warp reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xFFFFFFFFu, m, o);
    const float s2 = __shfl_xor_sync(0xFFFFFFFFu, s, o);
    const int i2 = __shfl_xor_sync(0xFFFFFFFFu, idx, o);
    part_merge(m, s, idx, m2, s2, i2);
  }
  __shared__ float sm[THREADS / 32], ss[THREADS / 32];
  __shared__ int si[THREADS / 32];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[warp] = m;
    ss[warp] = s;
    si[warp] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    int I = si[0];
    for (int k = 1; k < THREADS / 32; ++k) part_merge(M, S, I, sm[k], ss[k], si[k]);
    Part out;
    out.m = M;
    out.s = S;
    out.idx = (I == 0x7FFFFFFF) ? -1 : I + vocab_offset;
    part[static_cast<int64_t>(row) * n_vsplit + split] = out;
  }
  if (fuse.counters != nullptr) {
    const FuseArgs& f = fuse;
    __shared__ int last;
    if (threadIdx.x == 0) {
      const int req = f.row_req[row];
      const int parts = (f.cu_rows[req + 1] - f.cu_rows[req]) * n_vsplit;
      __threadfence();  // release this CTA's record before counting it
      last = (atomicAdd(&f.counters[req], 1) == parts - 1) ? req : -1;
    }
    __syncthreads();
    if (last >= 0 && threadIdx.x < 32) {
      __threadfence();  // acquire the other CTAs' records
      finalize_request(last, threadIdx.x, part, 1, f.n_rows_cap, n_vsplit, f.cu_rows, f.tau, f.fallback_mode,
                       f.commit_mask, f.tok, f.conf, f.row_pos, f.state, f.token_buf, f.state_stride);
      if (threadIdx.x == 0) f.counters[last] = 0;  // ready for the next launch (stream order)
    }
  }
}

int launch_unmask_partials(const void* logits, int dtype, int64_t row_stride,
                           const int32_t* row_src, int n_rows, int vocab, int vocab_offset,
                           int n_vsplit, float* part, cudaStream_t stream) {
  if (n_rows == 0) return 0;
  dim3 grid(n_rows, n_vsplit);
  if (dtype == 0) {
    unmask_partial_kernel<__nv_bfloat16, 256><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(logits), row_stride, row_src, vocab, vocab_offset,
        n_vsplit, reinterpret_cast<Part*>(part), nullptr, FuseArgs{});
  } else {
    unmask_partial_kernel<float, 256><<<grid, 256, 0, stream>>>(
        static_cast<const float*>(logits), row_stride, row_src, vocab, vocab_offset, n_vsplit,
        reinterpret_cast<Part*>(part), nullptr, FuseArgs{});
  }
  return static_cast<int>(cudaGetLastError());
}

// Phase (a) with the row count read from device memory (grid sized for n_rows_cap).
int launch_unmask_partials_dev(const void* logits, int dtype, int64_t row_stride, const int32_t* row_src,
                               int n_rows_cap, const int32_t* n_rows_dev, int vocab, int vocab_offset,
                               int n_vsplit, float* part, cudaStream_t stream) {
  if (n_rows_cap == 0) return 0;
  dim3 grid(n_rows_cap, n_vsplit);
  if (dtype == 0) {
    unmask_partial_kernel<__nv_bfloat16, 256><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(logits), row_stride, row_src, vocab, vocab_offset, n_vsplit,
        reinterpret_cast<Part*>(part), n_rows_dev, FuseArgs{});
  } else {
    unmask_partial_kernel<float, 256><<<grid, 256, 0, stream>>>(
        static_cast<const float*>(logits), row_stride, row_src, vocab, vocab_offset, n_vsplit,
        reinterpret_cast<Part*>(part), n_rows_dev, FuseArgs{});
  }
  return static_cast<int>(cudaGetLastError());
}

// Both phases in one launch (single vocab shard): partials, and the CTA completing a
// request's partials finalizes it.  n_rows_dev (optional) holds the row count of a
// device-planned step; n_rows then bounds it and strides part.
int launch_unmask_commit(const void* logits, int dtype, int64_t row_stride, const int32_t* row_src, int n_rows,
                         const int32_t* n_rows_dev, int vocab, int n_vsplit, float* part, const int32_t* cu_rows,
                         const int32_t* row_req, int32_t* counters, float tau, int fallback_mode,
                         uint8_t* commit_mask, int32_t* tok, float* conf, const int32_t* row_pos, uint8_t* state,
                         int32_t* token_buf, int64_t state_stride, cudaStream_t stream) {
  if (n_rows == 0) return 0;
  const FuseArgs f{cu_rows, row_req, counters, n_rows, tau, fallback_mode, commit_mask, tok, conf, row_pos,
                   state, token_buf, state_stride};
  dim3 grid(n_rows, n_vsplit);
  if (dtype == 0) {
    unmask_partial_kernel<__nv_bfloat16, 256><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(logits), row_stride, row_src, vocab, 0, n_vsplit,
        reinterpret_cast<Part*>(part), n_rows_dev, f);
  } else {
    unmask_partial_kernel<float, 256><<<grid, 256, 0, stream>>>(
        static_cast<const float*>(logits), row_stride, row_src, vocab, 0, n_vsplit, reinterpret_cast<Part*>(part),
        n_rows_dev, f);
  }
  return static_cast<int>(cudaGetLastError());
}

int launch_unmask_finalize(const float* part, int n_outer, int n_rows, int n_vsplit,
                           const int32_t* cu_rows, int n_req, float tau, int fallback_mode,
                           uint8_t* commit_mask, int32_t* tok, float* conf, const int32_t* row_pos,
                           uint8_t* state, int32_t* token_buf, int64_t state_stride,
                           cudaStream_t stream) {
  if (n_req == 0) return 0;
  const int blocks = (n_req * 32 + 127) / 128;
  unmask_finalize_kernel<<<blocks, 128, 0, stream>>>(
      reinterpret_cast<const Part*>(part), n_outer, n_rows, n_vsplit, cu_rows, n_req, tau,
      fallback_mode, commit_mask, tok, conf, row_pos, state, token_buf, state_stride);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace optimus
