// kernels.cuh — PROBE hot-path kernels other than the tensor-core GEMM.
// Citations: PAPER.md line numbers (P:n) and SURVEY.md §8(c) readings (Rn).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "gemm_sm100.cuh"

namespace probe {

constexpr int kMaxRb = 3;          // "at most three redundant experts per rank"
constexpr int kChunk = 128;        // tokens per top-k CTA (one bit per token in 4 × 32-bit masks)
constexpr int kMaxE = 256;
constexpr int kMaxK = 16;
constexpr int kMaxG = 64;

enum : int { ERR_RECV_OVERFLOW = 1, ERR_PLAN = 2, ERR_SHAPE = 4, ERR_Y_RANGE = kErrYRange };

// Symmetric buffer table: sym[buf * G + r] = address of rank r's buffer `buf`.
struct Sym {
  const uint64_t* ptr;
  __device__ __forceinline__ uint8_t* at(int buf, int G, int r) const {
    return reinterpret_cast<uint8_t*>(ptr[buf * G + r]);
  }
};

struct Dims {
  int G, R0, GL, E, EL, k, H, F, h, T, cap, Rb;
};

// board layout per rank: int32 [2 parity][2 kind][G][E]
__device__ __forceinline__ int board_off(const Dims& d, int parity, int kind) {
  return ((parity * 2 + kind) * d.G) * d.E;
}

// =============================================================================
// a1/a2 top-k: per token, first k experts by (logit ↓, id ↑) (R3, R4); gate mode
// also writes softmax weights over the selected logits (R1), and per-chunk
// expert bitmasks → per-chunk histograms and the intra-chunk rank of every pair
// (deterministic dispatch positions, R23/R24).
// grid (ceil(T/128), GL), block 128 (4 warps × 32 tokens).
// =============================================================================
template <int VPL, bool PRED>
__global__ void __launch_bounds__(128) k_topk(Dims d, int T, const float* __restrict__ logits,
                                              const float* __restrict__ logits2, const float* __restrict__ bias,
                                              int32_t* __restrict__ ids, float* __restrict__ gw,
                                              int32_t* __restrict__ pos, int32_t* __restrict__ hist,
                                              int32_t* __restrict__ pred_counts, float* __restrict__ logits_out) {
  __shared__ uint32_t mask[kMaxE * 4];
  __shared__ int32_t scount[kMaxE];
  const int E = d.E, k = d.k;
  const int chunk = blockIdx.x, gl = blockIdx.y;
  const int nchunks = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E * 4; i += blockDim.x) mask[i] = 0u;
  for (int i = threadIdx.x; i < E; i += blockDim.x) scount[i] = 0;
  __syncthreads();
  for (int i = 0; i < 32; ++i) {
    const int tl = warp * 32 + i;
    const int t = chunk * kChunk + tl;
    if (t >= T) break;
    const size_t rowoff = (static_cast<size_t>(gl) * T + t) * E;
    float v[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int e = lane + 32 * q;
      float x = -INFINITY;
      if (e < E) {
        x = logits[rowoff + e];
        if (PRED && logits2) x += logits2[rowoff + e];
        if (bias) x += bias[e];
        if (PRED && logits_out) logits_out[rowoff + e] = x;
      }
      v[q] = x;
    }
    float selv[kMaxK];
    int sele[kMaxK];
    uint32_t taken = 0u;   // bit q: expert lane+32q already selected
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int be = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int e = lane + 32 * q;
        if (e < E && !((taken >> q) & 1u) && (v[q] > bv || (v[q] == bv && e < be))) { bv = v[q]; be = e; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      selv[j] = bv;
      sele[j] = be;
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
    }
    if (!PRED) {
      // softmax over the selected logits (R1), max = selv[0]
      float sum = 0.f;
      for (int j = 0; j < k; ++j) sum += expf(selv[j] - selv[0]);
      if (lane < k) {
        float sv = selv[0];
        int se = sele[0];
        for (int j = 1; j < k; ++j)
          if (lane == j) { sv = selv[j]; se = sele[j]; }
        const size_t o = (static_cast<size_t>(gl) * T + t) * k + lane;
        ids[o] = se;
        gw[o] = expf(sv - selv[0]) / sum;
        mask[se * 4 + warp] |= (1u << i);   // only this warp writes word `warp`
      }
    } else {
      if (lane < k) {
        int se = sele[0];
        for (int j = 1; j < k; ++j)
          if (lane == j) se = sele[j];
        atomicAdd(&scount[se], 1);
        if (ids) ids[(static_cast<size_t>(gl) * T + t) * k + lane] = se;
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (PRED) {
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      if (scount[e]) atomicAdd(&pred_counts[gl * E + e], scount[e]);
    return;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const uint32_t* m = &mask[e * 4];
    hist[(static_cast<size_t>(gl) * nchunks + chunk) * E + e] =
        __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
  }
  {
    const int tl = threadIdx.x;
    const int t = chunk * kChunk + tl;
    if (t < T) {
      const int w = tl >> 5, b = tl & 31;
      for (int j = 0; j < k; ++j) {
        const size_t o = (static_cast<size_t>(gl) * T + t) * k + j;
        const int e = ids[o];
        const uint32_t* m = &mask[e * 4];
        int p = __popc(m[w] & ((1u << b) - 1u));
        for (int ww = 0; ww < w; ++ww) p += __popc(m[ww]);
        pos[o] = p;
      }
    }
  }
}

// =============================================================================
// a1/a2 top-k, thread per token (high occupancy): each thread streams its logit row
// with 16-byte loads, 32 values at a time in registers (L1 absorbs the line reuse), and
// keeps a register list sorted by (value ↓, id ↑) (R3, R4; KK compile-time, no local
// memory).  Gate mode also writes the softmax over the selected logits (R1) and the
// per-chunk dispatch ranks (expert bitmasks as in k_rank); predictor mode accumulates
// n̂[rank][e] (R9).  grid (ceil(T/128), GL), block 128 (thread = token).  E % 32 == 0
// or E < 32 handled by masking.
// =============================================================================
// Top-k by sorting networks: topk_sort8 / topk_merge8 (gemm_sm100.cuh, shared with the GEMM-epilogue top-k).

// The predictor instance (PRED) is capped at 64 registers (8 CTAs of 128 threads per SM) and
// streams 16 logits per step: it must fit beside a persistent expert-GEMM CTA (224 × 256
// registers) when the aux track still runs after the expert GEMMs started (C3 on one GPU:
// the 4-TFLOP predictor outlasts the dispatch; a 95-register select then waited for the
// GEMMs to end, the plan came after the combine and split-phase part 1 pushed nothing).
template <int KK, bool PRED>
__global__ void __launch_bounds__(128, PRED ? 8 : 1) k_select(Dims d, int T, const float* __restrict__ logits,
                                                const float* __restrict__ bias, int32_t* __restrict__ ids,
                                                float* __restrict__ gw, int32_t* __restrict__ pos,
                                                int32_t* __restrict__ hist, int32_t* __restrict__ counts,
                                                float* __restrict__ logits_out = nullptr,
                                                int32_t* __restrict__ pred_ids = nullptr,
                                                const float* __restrict__ logits2 = nullptr) {
  __shared__ uint32_t mask[kMaxE * 4];
  __shared__ int32_t scount[kMaxE];
  const int E = d.E;
  const int chunk = blockIdx.x, gl = blockIdx.y, nchunks = gridDim.x;
  const int tl = threadIdx.x, t = chunk * kChunk + tl;
  for (int i = tl; i < E * 4; i += blockDim.x) mask[i] = 0u;
  for (int i = tl; i < E; i += blockDim.x) scount[i] = 0;
  __syncthreads();
  int te[8];
  if (t < T) {
    float tv[8];   // running top 8, sorted by (value ↓, id ↑); the first KK are the selection
#pragma unroll
    for (int j = 0; j < 8; ++j) { tv[j] = -INFINITY; te[j] = 0x7fffffff; }
    const float* row = logits + (static_cast<size_t>(gl) * T + t) * E;
    constexpr int CW = PRED ? 8 : 32;      // logits per step (8-wide groups)
#pragma unroll 1
    for (int c = 0; c < E; c += CW) {
      float v[CW];
#pragma unroll
      for (int q = 0; q < CW / 4; ++q) {
        if (c + 4 * q + 3 < E) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(row + c) + q);
          v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) v[4 * q + u] = (c + 4 * q + u < E) ? row[c + 4 * q + u] : -INFINITY;
        }
      }
      if (PRED && logits2) {   // fused predictor (D10): l̂ = prior + residual, both fp32 GEMM outputs
        const float* row2 = logits2 + (static_cast<size_t>(gl) * T + t) * E;
#pragma unroll
        for (int q = 0; q < CW / 4; ++q) {
          if (c + 4 * q + 3 < E) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(row2 + c) + q);
            v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c + 4 * q + u < E) v[4 * q + u] += row2[c + 4 * q + u];
          }
        }
      }
      if (bias) {
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (c + i < E) v[i] += __ldg(bias + c + i);
      }
      if (PRED && logits_out) {   // l̂ = prior + residual + b, exactly the values the selection ranks
        float* lo = logits_out + (static_cast<size_t>(gl) * T + t) * E + c;
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (c + i < E) lo[i] = v[i];
      }
#pragma unroll
      for (int g = 0; g < CW / 8; ++g) {
        float gv[8];
        int ge[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { gv[i] = v[8 * g + i]; ge[i] = c + 8 * g + i; }
        topk_sort8(gv, ge);
        topk_merge8(tv, te, gv, ge);
      }
    }
    const size_t o = (static_cast<size_t>(gl) * T + t) * KK;
    if (!PRED) {
      float w[KK], sum = 0.f;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        w[j] = expf(tv[j] - tv[0]);
        sum += w[j];
      }
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        ids[o + j] = te[j];
        gw[o + j] = w[j] / sum;
        atomicOr(&mask[te[j] * 4 + (tl >> 5)], 1u << (tl & 31));
      }
    } else {
#pragma unroll
      for (int j = 0; j < KK; ++j) atomicAdd(&scount[te[j]], 1);
      if (pred_ids) {            // predicted sets per token (NEXT-4 pre-dispatch reads them)
#pragma unroll
        for (int j = 0; j < KK; ++j) pred_ids[o + j] = te[j];
      }
    }
  }
  __syncthreads();
  if (PRED) {
    for (int e = tl; e < E; e += blockDim.x)
      if (scount[e]) atomicAdd(&counts[gl * E + e], scount[e]);
    return;
  }
  for (int e = tl; e < E; e += blockDim.x) {
    const uint32_t* m = &mask[e * 4];
    hist[(static_cast<size_t>(gl) * nchunks + chunk) * E + e] = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
  }
  if (t < T) {
    const int w = tl >> 5, b = tl & 31;
    const size_t o = (static_cast<size_t>(gl) * T + t) * KK;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      const uint32_t* m = &mask[te[j] * 4];
      int p = __popc(m[w] & ((1u << b) - 1u));
      for (int ww = 0; ww < w; ++ww) p += __popc(m[ww]);
      pos[o + j] = p;
    }
  }
}

// =============================================================================
// a5/a6 helper after the fused gate: per 128-token chunk, expert bitmasks built
// from the routing ids (order-independent atomicOr) → per-chunk histograms and
// the rank of every (token, slot) among the chunk's tokens of its expert (token
// order), i.e. deterministic dispatch positions (R23/R24).
// grid (ceil(T/128), GL), block 128 (thread = token).
// =============================================================================
__global__ void __launch_bounds__(128) k_rank(Dims d, int T, const int32_t* __restrict__ ids,
                                              int32_t* __restrict__ pos, int32_t* __restrict__ hist) {
  __shared__ uint32_t mask[kMaxE * 4];
  const int E = d.E, k = d.k;
  const int chunk = blockIdx.x, gl = blockIdx.y, nchunks = gridDim.x;
  const int tl = threadIdx.x, t = chunk * kChunk + tl;
  for (int i = tl; i < E * 4; i += blockDim.x) mask[i] = 0u;
  __syncthreads();
  const size_t base = (static_cast<size_t>(gl) * T + t) * k;
  int e_loc[kMaxK];
  if (t < T)
    for (int j = 0; j < k; ++j) {
      e_loc[j] = ids[base + j];
      atomicOr(&mask[e_loc[j] * 4 + (tl >> 5)], 1u << (tl & 31));
    }
  __syncthreads();
  for (int e = tl; e < E; e += blockDim.x) {
    const uint32_t* m = &mask[e * 4];
    hist[(static_cast<size_t>(gl) * nchunks + chunk) * E + e] = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
  }
  if (t < T) {
    const int w = tl >> 5, b = tl & 31;
    for (int j = 0; j < k; ++j) {
      const uint32_t* m = &mask[e_loc[j] * 4];
      int p = __popc(m[w] & ((1u << b) - 1u));
      for (int ww = 0; ww < w; ++ww) p += __popc(m[ww]);
      pos[base + j] = p;
    }
  }
}

// =============================================================================
// a3: per-(rank, expert) exclusive scan over chunks → chunk bases and actual
// counts n[r][e]; all-gather the counts into every rank's board (M2).
// grid GL, block 256.
// =============================================================================
__global__ void k_count_scan(Dims d, int nchunks, const int32_t* __restrict__ hist, int32_t* __restrict__ cbase,
                             Sym sym, int buf_board, int parity) {
  const int gl = blockIdx.x;
  for (int e = threadIdx.x; e < d.E; e += blockDim.x) {
    int run = 0;
    // 8 chunk histograms in flight per step (the scan is a serial chain of L2 round trips otherwise)
    for (int c0 = 0; c0 < nchunks; c0 += 8) {
      int h[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        h[u] = c0 + u < nchunks ? hist[(static_cast<size_t>(gl) * nchunks + c0 + u) * d.E + e] : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + u < nchunks) cbase[(static_cast<size_t>(gl) * nchunks + c0 + u) * d.E + e] = run;
        run += h[u];
      }
    }
    const int off = board_off(d, parity, 0) + (d.R0 + gl) * d.E + e;
    for (int r = 0; r < d.G; ++r) reinterpret_cast<int32_t*>(sym.at(buf_board, d.G, r))[off] = run;
  }
}

// predicted counts [GL][E] → every rank's board (kind 1); optional copy-out of the full [G,E].
__global__ void k_pred_publish(Dims d, const int32_t* __restrict__ pred_local, Sym sym, int buf_board,
                               int parity) {
  const int gl = blockIdx.x;
  for (int e = threadIdx.x; e < d.E; e += blockDim.x) {
    const int off = board_off(d, parity, 1) + (d.R0 + gl) * d.E + e;
    const int v = pred_local[gl * d.E + e];
    for (int r = 0; r < d.G; ++r) reinterpret_cast<int32_t*>(sym.at(buf_board, d.G, r))[off] = v;
  }
}

// R26 measured hiding window: the expert-GEMM phase of this process's ranks is stamped with
// %globaltimer (phase 0: start, before GEMM1; phase 1: end, after GEMM2) and stored for every
// local rank into EVERY rank's count board (int64 slot after the [2][2][G][E] counts), so every
// rank plans from the same all-gathered windows (R10).  One process per GPU (one local rank):
// the window is the measured GEMM time.  Several logical ranks sharing one GPU run their
// tiles in one grouped GEMM, so the measured time covers all of them; rank r's window is then
// its share of it by the planner's own compute cost (R11), T_GEMM · C_r / Σ C with
// C_r = Σ_{slots j of r with rows} max(rows_j, n_sat) — the time its GEMMs take on a GPU of its
// own: rows for prefill-sized groups, weight streaming (n_sat per active expert) for decode.
__device__ __forceinline__ int64_t* window_board(const Dims& d, uint8_t* board) {
  return reinterpret_cast<int64_t*>(board + static_cast<size_t>(4) * d.G * d.E * 4);
}
__device__ __forceinline__ int64_t rank_gemm_cost(const Dims& d, const int32_t* group_rows, int r, int n_sat) {
  const int S = d.EL + kMaxRb;
  int64_t c = 0;
  for (int j = 0; j < S; ++j) {
    const int m = group_rows[r * S + j];
    if (m > 0) c += m > n_sat ? m : n_sat;
  }
  return c;
}
__global__ void k_window_stamp(Dims d, int64_t* t0, int phase, Sym sym, int buf_board,
                               const int32_t* __restrict__ group_rows, int n_sat) {
  // phase 0: one thread stamps; phase 1: thread gl (< GL ≤ 64) handles local rank gl
  __shared__ int64_t cost[kMaxG];
  __shared__ int64_t s_w, s_tot;
  const int gl = threadIdx.x;
  if (phase == 0) {
    if (gl == 0) *t0 = static_cast<int64_t>(ptx::globaltimer_ns());
    return;
  }
  if (gl == 0) s_w = static_cast<int64_t>(ptx::globaltimer_ns()) - *t0;
  if (gl < d.GL) cost[gl] = rank_gemm_cost(d, group_rows, d.R0 + gl, n_sat);
  __syncthreads();
  if (gl == 0) {
    int64_t tot = 0;
    for (int i = 0; i < d.GL; ++i) tot += cost[i];
    s_tot = tot;
  }
  __syncthreads();
  if (gl < d.GL) {
    const int64_t w = s_w, tot = s_tot;
    const int64_t wr = (d.GL == 1 || tot == 0) ? w : w * cost[gl] / tot;
    for (int r = 0; r < d.G; ++r) window_board(d, sym.at(buf_board, d.G, r))[d.R0 + gl] = wr > 0 ? wr : 1;
  }
}
// window_ns[r] = measured[r] (or fallback_ns where nothing was measured yet) + attention_ns
__global__ void k_window_read(Dims d, const uint8_t* board, int64_t attention_ns, int64_t fallback_ns,
                              int64_t* window_ns) {
  const int64_t* wb = window_board(d, const_cast<uint8_t*>(board));
  for (int r = threadIdx.x; r < d.G; r += blockDim.x) {
    const int64_t m = wb[r];
    window_ns[r] = (m > 0 ? m : fallback_ns) + attention_ns;
  }
}

// history[g][e] = (reset ? 0 : history[g][e]) + n[g][e]  (statistics-based baseline policy)
__global__ void k_history(int n_elems, const int32_t* __restrict__ counts, int32_t* __restrict__ hist, int reset) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_elems; i += gridDim.x * blockDim.x)
    hist[i] = (reset ? 0 : hist[i]) + counts[i];
}

__global__ void k_copy_i32(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// =============================================================================
// a4: Greedy Balance-Optimal Planning (Algorithm 1) on ONE CTA,
// integer costs (R11), readings R13-R22.  Every rank runs it on the same n̂ (R10).
// Incremental cost updates (only r_src and r_dst change).  The split [G][E][G] lives in the
// quota output itself (global memory, L1/L2-resident): with ≤ 6 KB of shared memory and 64
// threads the planner CTA fits beside a persistent expert-GEMM CTA (≈ 214 KB smem), so the
// plan for L+1 completes during layer L's GEMM instead of waiting for a free SM.
// =============================================================================
struct PlanParams {
  int64_t alpha, beta, bw, wbytes;
  int n_sat, kmax, Rb;
};

__device__ __forceinline__ int64_t cost_c(int64_t m, int n_sat) { return m == 0 ? 0 : (m > n_sat ? m : n_sat); }

__global__ void __launch_bounds__(64) k_plan(Dims d, PlanParams pp, const int32_t* __restrict__ nhat,
                                             const int64_t* __restrict__ window_ns, int32_t* quota,
                                             int32_t* __restrict__ replicas, int64_t* __restrict__ stats,
                                             int32_t* __restrict__ prefetch_ctr) {
  int32_t* sp = quota;                            // split [G][E][G], updated in place
  __shared__ int64_t comp[kMaxG], L[kMaxG], Lb[kMaxG];
  __shared__ int64_t inn[kMaxG], outv[kMaxG], load[kMaxG];
  __shared__ int32_t cap[kMaxG], nin[kMaxG], nout[kMaxG], rep[kMaxG * kMaxRb];
  __shared__ uint64_t invalid[kMaxG];             // bit dst of row src
  __shared__ uint32_t hostbits[kMaxG][kMaxE / 32];
  __shared__ int s_src, s_dst, s_stop;
  __shared__ int64_t s_total;
  const int G = d.G, E = d.E, EL = d.EL;
  const int tid = threadIdx.x;
  // line 2: locality-first A from n̂ and P′
  for (int i = tid; i < G * E * G; i += blockDim.x) {
    const int s = i / (E * G), e = (i / G) % E, t = i % G;
    sp[i] = (t == e / EL) ? nhat[s * E + e] : 0;
  }
  for (int r = tid; r < G; r += blockDim.x) {
    const int64_t w = window_ns ? window_ns[r] : 0;
    int64_t c = (w * pp.bw) / (pp.wbytes * 1000);
    cap[r] = static_cast<int>(c < pp.Rb ? c : pp.Rb);
    nin[r] = 0;
    nout[r] = 0;
    invalid[r] = 0ull;
    for (int i = 0; i < kMaxRb; ++i) rep[r * kMaxRb + i] = -1;
    for (int w32 = 0; w32 < kMaxE / 32; ++w32) hostbits[r][w32] = 0u;
  }
  __syncthreads();
  for (int r = tid; r < G; r += blockDim.x)
    for (int e = r * EL; e < (r + 1) * EL; ++e) hostbits[r][e >> 5] |= 1u << (e & 31);
  // line 3: L ← ComputeLatencies(A)
  for (int r = tid; r < G; r += blockDim.x) {
    int64_t c = 0, in_ = 0, out_ = 0, ld = 0;
    for (int e = r * EL; e < (r + 1) * EL; ++e) {
      int64_t m = 0;
      for (int s = 0; s < G; ++s) m += sp[(s * E + e) * G + r];
      c += cost_c(m, pp.n_sat);
      ld += m;
      in_ += m - sp[(r * E + e) * G + r];
    }
    for (int e = 0; e < E; ++e)
      if (e / EL != r) out_ += sp[(r * E + e) * G + e / EL];
    comp[r] = c;
    inn[r] = in_;
    outv[r] = out_;
    load[r] = ld;
    L[r] = pp.alpha * c + pp.beta * (in_ > out_ ? in_ : out_);
    Lb[r] = L[r];
  }
  __syncthreads();
  if (tid == 0) {
    int64_t tot = 0;
    for (int r = 0; r < G; ++r) tot += load[r];
    s_total = tot;
  }
  __syncthreads();
  int iters = 0;
  int64_t maxb = 0;
  for (int r = 0; r < G; ++r) maxb = Lb[r] > maxb ? Lb[r] : maxb;
  // line 4: loop (warp 0 drives; lane-parallel expert selection)
  if (tid < 32) {
    const int lane = tid;
    while (true) {
      if (lane == 0) {
        int src = 0;
        for (int r = 1; r < G; ++r)
          if (L[r] > L[src]) src = r;                            // line 5 (lowest r on ties)
        int dst = -1;
        for (int r = 0; r < G; ++r) {
          if (r == src || ((invalid[src] >> r) & 1ull)) continue;
          if (dst < 0 || L[r] < L[dst]) dst = r;                 // line 6, R14
        }
        s_src = src;
        s_dst = dst;
      }
      __syncwarp();
      const int src = s_src, dst = s_dst;
      if (dst < 0) break;
      // line 7: SelectHeavyExpert (R13): home on src, not hosted on dst, max remote pool, lowest e
      int be = -1, bp = 0;
      for (int e = src * EL + lane; e < (src + 1) * EL; e += 32) {
        if ((hostbits[dst][e >> 5] >> (e & 31)) & 1u) continue;
        int pool = 0;
        for (int s = 0; s < G; ++s)
          if (s != src) pool += sp[(s * E + e) * G + src];
        if (pool > bp || (pool == bp && pool > 0 && e < be)) { bp = pool; be = e; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const int op = __shfl_xor_sync(0xffffffffu, bp, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (op > bp || (op == bp && op > 0 && (be < 0 || (oe >= 0 && oe < be)))) { bp = op; be = oe; }
      }
      if (lane == 0) {
        s_stop = 0;
        if (be < 0 || bp <= 0) {
          invalid[src] |= 1ull << dst;                           // no candidate ⇒ mark pair invalid
          s_stop = 2;
        } else if (nin[dst] + 1 > cap[dst] || nout[src] + 1 > cap[src]) {
          invalid[src] |= 1ull << dst;                           // line 8-10 dual budget (R15)
          s_stop = 2;
        } else {
          // line 11: water-filling (R18): x = min(pool, max(0, ℒ_src − ⌈Σℒ/G⌉))
          const int64_t avg = (s_total + G - 1) / G;
          int64_t x = load[src] - avg;
          if (x < 0) x = 0;
          if (x > bp) x = bp;
          // tentative moves: sources dst first, then ascending s ∉ {src,dst}
          int64_t rem = x, mv_dst = 0;
          {
            const int64_t a = sp[(dst * E + be) * G + src];
            const int64_t mv = rem < a ? rem : a;
            mv_dst = mv;
            rem -= mv;
          }
          int64_t m_e_src = 0;
          for (int s = 0; s < G; ++s) m_e_src += sp[(s * E + be) * G + src];
          const int64_t comp_src = comp[src] - cost_c(m_e_src, pp.n_sat) + cost_c(m_e_src - x, pp.n_sat);
          const int64_t comp_dst = comp[dst] + cost_c(x, pp.n_sat);
          const int64_t in_src = inn[src] - x;
          const int64_t in_dst = inn[dst] + (x - mv_dst);
          const int64_t out_dst = outv[dst] - mv_dst;
          const int64_t out_src = outv[src];
          const int64_t Ls = pp.alpha * comp_src + pp.beta * (in_src > out_src ? in_src : out_src);
          const int64_t Ld = pp.alpha * comp_dst + pp.beta * (in_dst > out_dst ? in_dst : out_dst);
          const int64_t gain = L[src] - (Ls > Ld ? Ls : Ld);       // R19
          if (gain <= 0 || iters >= pp.kmax) {                     // line 12-14 (R20)
            s_stop = 1;
          } else {
            // accept (line 15-17): apply the moves
            rem = x;
            for (int q = -1; q < G; ++q) {
              const int s = (q < 0) ? dst : q;
              if (q >= 0 && (s == src || s == dst)) continue;
              if (rem == 0) break;
              int32_t* a = &sp[(s * E + be) * G + src];
              const int64_t mv = rem < *a ? rem : *a;
              *a -= static_cast<int32_t>(mv);
              sp[(s * E + be) * G + dst] += static_cast<int32_t>(mv);
              rem -= mv;
            }
            comp[src] = comp_src; comp[dst] = comp_dst;
            inn[src] = in_src; inn[dst] = in_dst;
            outv[dst] = out_dst;
            load[src] -= x; load[dst] += x;
            L[src] = Ls; L[dst] = Ld;
            rep[dst * kMaxRb + nin[dst]] = be;
            nin[dst] += 1;
            nout[src] += 1;
            hostbits[dst][be >> 5] |= 1u << (be & 31);
            iters += 1;
          }
        }
      }
      __syncwarp();
      if (s_stop == 1) break;
      iters = __shfl_sync(0xffffffffu, iters, 0);
    }
  }
  __syncthreads();
  // outputs: quota = split (already in place); replicas sorted (slot order); stats
  if (tid < G) {
    int rr[kMaxRb];
    for (int i = 0; i < kMaxRb; ++i) rr[i] = rep[tid * kMaxRb + i];
    for (int a = 0; a < kMaxRb; ++a)
      for (int b = a + 1; b < kMaxRb; ++b)
        if (rr[b] >= 0 && (rr[a] < 0 || rr[b] < rr[a])) { int t = rr[a]; rr[a] = rr[b]; rr[b] = t; }
    for (int i = 0; i < kMaxRb; ++i) replicas[tid * kMaxRb + i] = rr[i];
  }
  if (tid == 0) {
    int64_t maxa = 0, ntr = 0, capbits = 0;
    for (int r = 0; r < G; ++r) {
      maxa = L[r] > maxa ? L[r] : maxa;
      ntr += nin[r];
    }
    for (int r = 0; r < G && r < 16; ++r) capbits |= static_cast<int64_t>(cap[r] & 3) << (2 * r);
    stats[0] = iters;
    stats[1] = ntr;
    stats[2] = maxb;
    stats[3] = maxa;
    stats[4] = capbits;
    stats[5] = s_total;
    stats[6] = 0;
    stats[7] = 0;
    if (prefetch_ctr) prefetch_ctr[0] = 0;
  }
}

// =============================================================================
// a5 + a6 layout: materialize the plan on the actual counts (R23), per-destination
// slot/source offsets (R24), and the grouped-GEMM schedules of the local ranks.
// One CTA (all ranks compute the identical layout).
// =============================================================================
struct LayoutOut {
  int32_t* split_cum;   // [G][E][G] inclusive cumsum over targets
  int32_t* slot_of;     // [G][E] local slot of e on d (-1 not hosted)
  int32_t* src_off;     // [G][S][G] first row of (d, slot, src)
  int32_t* group_rows;  // [G][S]
  int32_t* replicas_used;  // [G][3]
  GemmSched* s1;        // SwiGLU (expert GEMM 1)
  GemmSched* s2;        // fp16 Y (expert GEMM 2)
  int32_t* err;
  int32_t* fallbacks;   // count of layers that fell back to static EP (plan would overflow) or null
};
struct LayoutIn {
  int nparts;                   // >1: partition the expert GEMMs by local rank (EP emulation)
  int tile_m;                   // 128 (1-CTA expert GEMMs) or 256 (CTA-pair expert GEMMs)
  int bn1, bn2;                 // GEMM1 / GEMM2 tile widths: 256, or 512 (CTA-pair 256×512 one-accumulator kernel)
  const int32_t* board_actual;  // [G][E]
  const int32_t* quota;         // [G][E][G] or null (static EP)
  const int32_t* replicas;      // [G][3] or null
  int bank;                     // replica slot bank = layer parity
  void* act;                    // [GL*cap, F] bf16
  void* y_local;                // [GL*cap, H] fp16 (this process's Y region, D2)
  int f32;                      // fp32 parity path: act and Y are fp32, GEMM2 stores EPI_F32
  int y_wide;                   // fp16 Y by 64-column (128-byte row) TMA stores (epi_chunk64_f16)
  int l2hint;                   // TMA L2 hints: bits 0-2 expert GEMM1, bits 4-6 expert GEMM2 (GemmSched::l2hint)
};

// R23 for every (s, e): split[s][e][t] from the quota (or static EP when quota == null)
__device__ void layout_materialize(const Dims& d, const LayoutIn& in, const int32_t* reps, int32_t* sm_split,
                                   const int32_t* quota) {
  const int G = d.G, E = d.E, EL = d.EL;
  for (int i = threadIdx.x; i < G * E; i += blockDim.x) {
    const int s = i / E, e = i % E;
    const int n = in.board_actual[s * E + e];
    int a[kMaxG];
    int P = 0;
    for (int t = 0; t < G; ++t) {
      a[t] = quota ? quota[(s * E + e) * G + t] : 0;
      P += a[t];
    }
    if (P == 0) {
      bool hosts = (e / EL == s);
      for (int q = 0; q < kMaxRb; ++q) hosts |= (reps[s * kMaxRb + q] == e);
      const int tt = hosts ? s : e / EL;
      for (int t = 0; t < G; ++t) a[t] = (t == tt) ? n : 0;
    } else {
      int tstar = 0, sum = 0;
      for (int t = 1; t < G; ++t)
        if (a[t] > a[tstar]) tstar = t;             // largest Q_t, lowest t on ties
      for (int t = 0; t < G; ++t) {
        a[t] = static_cast<int>((static_cast<int64_t>(n) * a[t]) / P);
        sum += a[t];
      }
      a[tstar] += n - sum;
    }
    for (int t = 0; t < G; ++t) sm_split[(s * E + e) * G + t] = a[t];
  }
}

__global__ void __launch_bounds__(512) k_layout(Dims d, LayoutIn in, LayoutOut o) {
  extern __shared__ int32_t sm_split[];            // [G][E][G] materialized split
  __shared__ int32_t reps[kMaxG * kMaxRb];
  constexpr int kMaxGS = kMaxE + kMaxRb * kMaxG;   // G·S = E + 3G
  __shared__ int32_t gt[kMaxGS];                   // rows per (dest, slot)
  __shared__ int32_t gpre[kMaxGS];                 // first row of (dest, slot)
  __shared__ int32_t t1[kMaxGroups], t2[kMaxGroups];
  __shared__ int32_t dtot[kMaxG];
  __shared__ int s_fallback;
  const int G = d.G, E = d.E, EL = d.EL, S = EL + kMaxRb;
  const int tid = threadIdx.x;
  for (int i = tid; i < G * kMaxRb; i += blockDim.x) reps[i] = in.replicas ? in.replicas[i] : -1;
  for (int i = tid; i < G; i += blockDim.x) dtot[i] = 0;
  __syncthreads();
  // (1) materialize (R23), one thread per (s, e)
  layout_materialize(d, in, reps, sm_split, in.quota);
  __syncthreads();
  // (1b) device-side static-EP fallback (probe.h, SURVEY §8(b) Errors): if the plan would
  // overflow some destination's receive capacity (a misprediction sending replicas more rows
  // than the plan expected), this layer runs static EP instead — decided identically on
  // every rank from the same all-gathered counts, no host synchronization.
  if (in.quota) {
    for (int i = tid; i < G * E; i += blockDim.x)
      for (int t = 0; t < G; ++t) {
        const int v = sm_split[i * G + t];
        if (v) atomicAdd(&dtot[t], v);
      }
    __syncthreads();
    if (tid == 0) {
      int over = 0;
      for (int t = 0; t < G; ++t) over |= dtot[t] > d.cap;
      s_fallback = over;
      if (over && o.fallbacks) atomicAdd(o.fallbacks, 1);
    }
    __syncthreads();
    if (s_fallback) {
      for (int i = tid; i < G * kMaxRb; i += blockDim.x) reps[i] = -1;
      __syncthreads();
      layout_materialize(d, in, reps, sm_split, nullptr);
      __syncthreads();
    }
  }
  for (int i = tid; i < G * E; i += blockDim.x) {
    int run = 0;
    for (int t = 0; t < G; ++t) {
      run += sm_split[i * G + t];
      o.split_cum[i * G + t] = run;
    }
  }
  // (2) local slot of every expert on every rank
  for (int i = tid; i < G * E; i += blockDim.x) {
    const int r = i / E, e = i % E;
    int sl = -1;
    if (e / EL == r) sl = e - r * EL;
    for (int q = 0; q < kMaxRb; ++q)
      if (reps[r * kMaxRb + q] == e) sl = EL + q;
    o.slot_of[i] = sl;
  }
  for (int i = tid; i < G * kMaxRb; i += blockDim.x) o.replicas_used[i] = reps[i];
  __syncthreads();
  // (3) rows per (dest r, slot j): base experts ascending, then replicas in slot order (R24)
  for (int i = tid; i < G * S; i += blockDim.x) {
    const int r = i / S, j = i % S;
    const int e = (j < EL) ? r * EL + j : reps[r * kMaxRb + (j - EL)];
    int tot = 0;
    if (e >= 0)
      for (int s = 0; s < G; ++s) tot += sm_split[(s * E + e) * G + r];
    gt[i] = tot;
    o.group_rows[i] = tot;
  }
  __syncthreads();
  // (4) slot prefix per destination (G serial scans of length S)
  for (int r = tid; r < G; r += blockDim.x) {
    int run = 0;
    for (int j = 0; j < S; ++j) {
      gpre[r * S + j] = run;
      run += gt[r * S + j];
    }
  }
  __syncthreads();
  // (5) first row of every (dest, slot, source): rows of a slot ordered by source ↑ then token ↑
  for (int i = tid; i < G * S; i += blockDim.x) {
    const int r = i / S, j = i % S;
    const int e = (j < EL) ? r * EL + j : reps[r * kMaxRb + (j - EL)];
    int run = gpre[i];
    for (int s = 0; s < G; ++s) {
      o.src_off[i * G + s] = run;
      if (e >= 0) run += sm_split[(s * E + e) * G + r];
    }
  }
  // (6) grouped-GEMM schedules of the local destinations
  const int ng = d.GL * S;
  if (tid == 0) {
    o.s1->num_groups = ng;
    o.s2->num_groups = ng;
  }
  for (int i = tid; i < ng; i += blockDim.x) {
    const int gl = i / S, j = i % S, r = d.R0 + gl;
    const int off = gpre[r * S + j];
    int m = gt[r * S + j];
    if (off + m > d.cap) {
      atomicOr(o.err, ERR_RECV_OVERFLOW);
      m = d.cap - off;
      if (m < 0) m = 0;
    }
    const bool is_rep = j >= EL;
    const int wslot = is_rep ? (gl * 2 * kMaxRb + in.bank * kMaxRb + (j - EL)) : (gl * EL + j);
    const int arow = gl * d.cap + (off < d.cap ? off : d.cap);
    GemmGroup g1;
    g1.a_row = arow; g1.m = m; g1.b_row = wslot * 2 * d.F; g1.b_sel = is_rep; g1.mode = EPI_SWIGLU;
    g1.n = d.F; g1.ldc = d.F; g1.tile_start = 0; g1.out_row = arow; g1.tma_out = !in.f32;   // bf16 act by TMA
    g1.topk = 0; g1.rows_per_rank = 1; g1.k_off = 0; g1.n_split = 0; g1.aux = nullptr; g1.bias = nullptr;
    g1.out = static_cast<uint8_t*>(in.act) + static_cast<size_t>(arow) * d.F * (in.f32 ? 4 : 2);
    GemmGroup g2;
    g2.a_row = arow; g2.m = m; g2.b_row = wslot * d.H; g2.b_sel = is_rep; g2.mode = in.f32 ? EPI_F32 : EPI_F16;
    g2.n = d.H; g2.ldc = d.H; g2.tile_start = 0; g2.out_row = arow; g2.tma_out = (!in.f32 && (d.H % 32 == 0)) ? (in.y_wide ? 2 : 1) : 0;
    g2.topk = 0; g2.rows_per_rank = 1; g2.k_off = 0; g2.n_split = 0; g2.aux = o.err; g2.bias = nullptr;
    g2.out = static_cast<uint8_t*>(in.y_local) + static_cast<size_t>(arow) * d.H * (in.f32 ? 4 : 2);
    o.s1->g[i] = g1;
    o.s2->g[i] = g2;
    t1[i] = gemm_ntiles(g1, in.bn1, in.tile_m);
    t2[i] = gemm_ntiles(g2, in.bn2, in.tile_m);
  }
  __syncthreads();
  // (7) tile prefix (warp 0: s1, warp 1: s2), warp-parallel exclusive scan in chunks of 32
  if (tid < 64) {
    const int w = tid >> 5, lane = tid & 31;
    int* tt = w == 0 ? t1 : t2;
    GemmSched* sc = w == 0 ? o.s1 : o.s2;
    int base = 0;
    for (int c0 = 0; c0 < ng; c0 += 32) {
      const int i = c0 + lane;
      const int v = i < ng ? tt[i] : 0;
      int x = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (i < ng) sc->g[i].tile_start = base + x - v;
      base += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
    if (lane == 0) {
      sc->total_tiles = base;
      sc->tile_m = in.tile_m;
      sc->stats = nullptr;
      sc->l2hint = w == 0 ? (in.l2hint & 7) : ((in.l2hint >> 4) & 7);
      sched_reset_counters(sc);
      sc->nparts = in.nparts > 1 ? in.nparts : 0;
      if (in.nparts > 1) {
        for (int gl = 0; gl < in.nparts; ++gl) sc->part_tile[gl] = sc->g[gl * S].tile_start;
        sc->part_tile[in.nparts] = base;
      }
    }
  }
}

// =============================================================================
// a6 dispatch: every (token, slot) row of x to its destination's receive buffer
// (peer store over NVLink for remote ranks).  Warp per token; the x row is read
// once and written to its k destinations with 16-byte vector stores.
// =============================================================================
__global__ void __launch_bounds__(256) k_dispatch(Dims d, int T, const uint8_t* __restrict__ x, int row_bytes,
                                                  const int32_t* __restrict__ ids,
                                                  const int32_t* __restrict__ pos,
                                                  const int32_t* __restrict__ cbase,
                                                  const int32_t* __restrict__ split_cum,
                                                  const int32_t* __restrict__ slot_of,
                                                  const int32_t* __restrict__ src_off, int32_t* __restrict__ route,
                                                  Sym sym, int buf_recv, int32_t* err) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= d.GL * T) return;
  const int gl = warp / T, t = warp % T;
  const int s = d.R0 + gl;
  const int nchunks = (T + kChunk - 1) / kChunk;
  const int S = d.EL + kMaxRb;
  const int k = d.k;
  const size_t pr = static_cast<size_t>(gl) * T + t;
  // lane j < k: destination rank and receive row of slot j (R23 fill order, R24 layout)
  uint8_t* dst_row = nullptr;
  if (lane < k) {
    const int e = ids[pr * k + lane];
    const int p = cbase[(static_cast<size_t>(gl) * nchunks + t / kChunk) * d.E + e] + pos[pr * k + lane];
    const int* c = &split_cum[(s * d.E + e) * d.G];
    int dd = 0;
    while (dd < d.G - 1 && c[dd] <= p) ++dd;
    const int excl = dd > 0 ? c[dd - 1] : 0;
    const int sl = slot_of[dd * d.E + e];
    int row = (sl < 0) ? -1 : src_off[(dd * S + sl) * d.G + s] + (p - excl);
    if (sl < 0 || row >= d.cap || c[dd] <= p) {
      atomicOr(err, ERR_RECV_OVERFLOW);
      row = -1;
    }
    route[(pr * k + lane) * 2] = dd;
    route[(pr * k + lane) * 2 + 1] = row;
    if (row >= 0) dst_row = sym.at(buf_recv, d.G, dd) + static_cast<size_t>(row) * row_bytes;
  }
  // copy: the x row is read once (batches of 8 × 16 B per lane in flight) and stored k times
  const uint4* src = reinterpret_cast<const uint4*>(x + pr * row_bytes);
  const int nv = row_bytes / 16;
  for (int c0 = 0; c0 < nv; c0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < nv) v[u] = __ldg(src + c);
    }
    for (int j = 0; j < k; ++j) {
      uint4* dst = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst_row), j));
      if (!dst) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < nv) dst[c] = v[u];
      }
    }
  }
}

// =============================================================================
// a6 dedup wire format (probe_config.dedup_wire, §8(a) a6: "one row per unique (token,
// dest), plus per-slot metadata"; Eq. 4's λ dedup).  Warp per token as in
// k_dispatch; within the token, slot j is the HEAD of its (token, dest) pair if no earlier
// slot has the same destination.  Only heads ship the x row (to the head's receive row);
// every slot ships a 16-byte meta record to its receive row on the destination:
//   {first row of the pair, next row of the pair in slot order (or -1), g_{t,j} (fp32 bits),
//    return index = src · T·KQ + t·KQ + q}
// q = rank of the destination among the token's distinct destinations (ascending): the
// expert rank's partial sum for (t, dest) is pushed to COMB[t·KQ + q] of the source, and
// the source sums q ascending (R25).  The receiver's k_expand copies the head row locally to
// the pair's other receive rows, so the grouped GEMM sees the usual per-slot layout (R24).
// =============================================================================
// NEXT-4 pre-dispatch: warp per token; the HOME ranks of the token's predicted experts
// (bitmask over ranks, identical to the one the dispatch recomputes) receive the x row in their
// PRE buffer at [source rank][token] while the gate is still computing the actual routing.
__device__ __forceinline__ uint64_t predicted_home_mask(const Dims& d, const int32_t* pids, size_t pr, int lane) {
  uint64_t m = 0;
  if (lane < d.k) m = 1ull << (pids[pr * d.k + lane] / d.EL);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(m), off);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(m >> 32), off);
    m |= (static_cast<uint64_t>(hi) << 32) | lo;
  }
  return m;
}

__global__ void __launch_bounds__(256) k_predispatch(Dims d, int T, int max_T, const uint8_t* __restrict__ x,
                                                     int row_bytes, const int32_t* __restrict__ pids, Sym sym,
                                                     int buf_pre) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= d.GL * T) return;
  const int gl = warp / T, t = warp % T;
  const size_t pr = static_cast<size_t>(gl) * T + t;
  const uint64_t mask = predicted_home_mask(d, pids, pr, lane);
  const size_t off = (static_cast<size_t>(d.R0 + gl) * max_T + t) * row_bytes;
  const uint4* src = reinterpret_cast<const uint4*>(x + pr * row_bytes);
  const int nv = row_bytes / 16;
  for (int c0 = 0; c0 < nv; c0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < nv) v[u] = __ldg(src + c);
    }
    for (uint64_t m = mask; m; m &= m - 1) {
      const int r = __ffsll(static_cast<long long>(m)) - 1;
      uint4* dst = reinterpret_cast<uint4*>(sym.at(buf_pre, d.G, r) + off);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < nv) dst[c] = v[u];
      }
    }
  }
}

constexpr int kMetaPre = 1 << 30;   // MetaRow.first flag: the pair's payload sits in PRE[src][t]

struct MetaRow {
  int32_t first, next, gbits, ret;
};

__device__ __forceinline__ void route_slot(const Dims& d, int T, int gl, int t, int lane, const int32_t* ids,
                                           const int32_t* pos, const int32_t* cbase, const int32_t* split_cum,
                                           const int32_t* slot_of, const int32_t* src_off, int32_t* route,
                                           int32_t* err, int& dd_out, int& row_out) {
  const int s = d.R0 + gl;
  const int nchunks = (T + kChunk - 1) / kChunk;
  const int S = d.EL + kMaxRb;
  const int k = d.k;
  const size_t pr = static_cast<size_t>(gl) * T + t;
  const int e = ids[pr * k + lane];
  const int p = cbase[(static_cast<size_t>(gl) * nchunks + t / kChunk) * d.E + e] + pos[pr * k + lane];
  const int* c = &split_cum[(s * d.E + e) * d.G];
  int dd = 0;
  while (dd < d.G - 1 && c[dd] <= p) ++dd;
  const int excl = dd > 0 ? c[dd - 1] : 0;
  const int sl = slot_of[dd * d.E + e];
  int row = (sl < 0) ? -1 : src_off[(dd * S + sl) * d.G + s] + (p - excl);
  if (sl < 0 || row >= d.cap || c[dd] <= p) {
    atomicOr(err, ERR_RECV_OVERFLOW);
    row = -1;
  }
  route[(pr * k + lane) * 2] = dd;
  route[(pr * k + lane) * 2 + 1] = row;
  dd_out = dd;
  row_out = row;
}

__global__ void __launch_bounds__(256) k_dispatch_dedup(Dims d, int T, const uint8_t* __restrict__ x, int row_bytes,
                                                        const int32_t* __restrict__ ids,
                                                        const int32_t* __restrict__ pos,
                                                        const int32_t* __restrict__ cbase,
                                                        const int32_t* __restrict__ split_cum,
                                                        const int32_t* __restrict__ slot_of,
                                                        const int32_t* __restrict__ src_off,
                                                        int32_t* __restrict__ route, const float* __restrict__ gw,
                                                        Sym sym, int buf_recv, int buf_meta, int KQ, int32_t* err,
                                                        const int32_t* __restrict__ pids, int32_t* hit_ctr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= d.GL * T) return;
  const int gl = warp / T, t = warp % T;
  const int k = d.k;
  const size_t pr = static_cast<size_t>(gl) * T + t;
  int dd = -1, row = -1;
  if (lane < k) route_slot(d, T, gl, t, lane, ids, pos, cbase, split_cum, slot_of, src_off, route, err, dd, row);
  const bool valid = lane < k && row >= 0;
  int first = row, next = -1, head = valid ? 1 : 0;
  for (int i = 0; i < k; ++i) {
    const int di = __shfl_sync(0xffffffffu, dd, i);
    const int ri = __shfl_sync(0xffffffffu, row, i);
    if (valid && ri >= 0 && di == dd) {
      if (i < lane && head) { first = ri; head = 0; }
      if (i > lane && next < 0) next = ri;
    }
  }
  const uint32_t heads = __ballot_sync(0xffffffffu, head != 0);
  // NEXT-4: pairs whose destination is the home of a predicted expert were pre-dispatched
  bool hit = false;
  if (pids) {
    const uint64_t pm = predicted_home_mask(d, pids, pr, lane);
    hit = valid && ((pm >> dd) & 1ull);
    const uint32_t hh = __ballot_sync(0xffffffffu, hit && head);
    if (lane == 0 && hit_ctr) {
      atomicAdd(hit_ctr, __popc(hh));
      atomicAdd(hit_ctr + 1, __popc(heads & ~hh));
    }
  }
  int q = 0;
  for (uint32_t m = heads; m; m &= m - 1) {
    const int i = __ffs(m) - 1;
    const int di = __shfl_sync(0xffffffffu, dd, i);   // heads is warp-uniform: every lane runs this loop
    if (di < dd) ++q;
  }
  uint8_t* dst_row = nullptr;
  if (valid) {
    MetaRow mr;
    mr.first = first | (hit ? kMetaPre : 0);
    mr.next = next;
    mr.gbits = __float_as_int(gw[pr * k + lane]);
    mr.ret = (d.R0 + gl) * (T * KQ) + t * KQ + q;
    *reinterpret_cast<int4*>(sym.at(buf_meta, d.G, dd) + static_cast<size_t>(row) * sizeof(MetaRow)) =
        make_int4(mr.first, mr.next, mr.gbits, mr.ret);
    if (head && !hit) dst_row = sym.at(buf_recv, d.G, dd) + static_cast<size_t>(row) * row_bytes;
  }
  const uint4* src = reinterpret_cast<const uint4*>(x + pr * row_bytes);
  const int nv = row_bytes / 16;
  for (int c0 = 0; c0 < nv; c0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < nv) v[u] = __ldg(src + c);
    }
    for (uint32_t m = heads; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      uint4* dst = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst_row), j));
      if (!dst) continue;                      // pre-dispatched (hit): the receiver has the row
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < nv) dst[c] = v[u];
      }
    }
  }
}

// rows used on every local destination (Σ of its slot group sizes, clamped to cap) → smem
__device__ __forceinline__ int used_rows_smem(const Dims& d, const int32_t* group_rows, int* used) {
  const int S = d.EL + kMaxRb;
  if (threadIdx.x < d.GL) {
    int u = 0;
    for (int j = 0; j < S; ++j) u += group_rows[(d.R0 + threadIdx.x) * S + j];
    used[threadIdx.x] = min(u, d.cap);
  }
  __syncthreads();
  int tot = 0;
  for (int g = 0; g < d.GL; ++g) tot += used[g];
  return tot;
}

// receiver side of the dedup wire: copy each pair's head row to the pair's other rows (local)
__global__ void __launch_bounds__(256) k_expand(Dims d, const int32_t* __restrict__ group_rows, Sym sym,
                                                int buf_meta, int buf_recv, int row_bytes, int T, int KQ,
                                                int buf_pre, int max_T) {
  __shared__ int used[kMaxG];
  const int tot = used_rows_smem(d, group_rows, used);
  const int lane = threadIdx.x & 31;
  const int nv = row_bytes / 16;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < tot; w += (gridDim.x * blockDim.x) >> 5) {
    int gl = 0, r = w;
    while (r >= used[gl]) r -= used[gl++];
    const int4* meta = reinterpret_cast<const int4*>(sym.at(buf_meta, d.G, d.R0 + gl));
    uint8_t* recv = sym.at(buf_recv, d.G, d.R0 + gl);
    const int4 m = meta[r];
    const int first = m.x & ~kMetaPre;
    const bool pre = (m.x & kMetaPre) != 0;
    if (first == r && !pre) continue;
    const uint8_t* srow;
    if (pre) {   // NEXT-4 hit: the row was pre-dispatched into PRE[src][t] of this rank
      const int per = T * KQ;
      const int src = m.w / per, t = (m.w % per) / KQ;
      srow = sym.at(buf_pre, d.G, d.R0 + gl) + (static_cast<size_t>(src) * max_T + t) * row_bytes;
    } else {
      srow = recv + static_cast<size_t>(first) * row_bytes;
    }
    const uint4* s0 = reinterpret_cast<const uint4*>(srow);
    uint4* d0 = reinterpret_cast<uint4*>(recv + static_cast<size_t>(r) * row_bytes);
    for (int c0 = 0; c0 < nv; c0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < nv) v[u] = s0[c];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < nv) d0[c] = v[u];
      }
    }
  }
}

// =============================================================================
// a8 combine, dedup wire (R25): on the EXPERT rank, for every (token, dest) pair (its head
// row), acc = Σ_{slots of the pair, slot order} g · y in fp32, pushed as ONE fp16 (fp32 in
// the fp32 parity path) row to the source's COMB[t·KQ + q]; the source then sums its
// partials in ascending destination order (k_combine_reduce).  The first CTA raises the
// prefetch suspend flag (R27): the combine phase begins here.
// =============================================================================
template <bool Y_F32, int KC>
__global__ void __launch_bounds__(256) k_combine_partial(Dims d, int T, const int32_t* __restrict__ group_rows,
                                                         Sym sym, int buf_meta, int buf_y, int buf_comb, int KQ,
                                                         volatile int32_t* suspend_flag, int layer) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && suspend_flag) *suspend_flag = layer + 1;
  __shared__ int used[kMaxG];
  const int tot = used_rows_smem(d, group_rows, used);
  const int lane = threadIdx.x & 31;
  constexpr int ES = Y_F32 ? 4 : 2;
  constexpr int U = 2;                          // 16-byte chunks per lane in flight per chain row
  const size_t rb = static_cast<size_t>(d.H) * ES;
  const int nv = static_cast<int>(rb / 16);     // 16-byte chunks per row
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < tot; w += (gridDim.x * blockDim.x) >> 5) {
    int gl = 0, r = w;
    while (r >= used[gl]) r -= used[gl++];
    const int4* meta = reinterpret_cast<const int4*>(sym.at(buf_meta, d.G, d.R0 + gl));
    const uint8_t* y = sym.at(buf_y, d.G, d.R0 + gl);
    const int4 m0 = meta[r];
    if ((m0.x & ~kMetaPre) != r) continue;       // not the head of its pair
    // the pair's rows in slot order (compile-time bound KC: registers, no local memory)
    const uint4* src[KC];
    float gs[KC];
    int q = r;
    int4 m = m0;
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      src[j] = nullptr;
      gs[j] = 0.f;
      if (q >= 0) {
        if (j > 0) m = meta[q];
        src[j] = reinterpret_cast<const uint4*>(y + static_cast<size_t>(q) * rb);
        gs[j] = __int_as_float(m.z);
        q = m.y;
      }
    }
    const int per = T * KQ;
    const int srank = m0.w / per, idx = m0.w % per;
    uint4* dst = reinterpret_cast<uint4*>(sym.at(buf_comb, d.G, srank) + static_cast<size_t>(idx) * rb);
    for (int c0 = lane; c0 < nv; c0 += 32 * U) {
      float a[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[u][i] = 0.f;
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        if (!src[j]) break;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + 32 * u < nv) v[u] = src[j][c0 + 32 * u];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (Y_F32) {   // 16 bytes = 4 fp32: columns (c0 + 32u)·4 .. +3
            a[u][0] = fmaf(gs[j], __uint_as_float(v[u].x), a[u][0]);
            a[u][1] = fmaf(gs[j], __uint_as_float(v[u].y), a[u][1]);
            a[u][2] = fmaf(gs[j], __uint_as_float(v[u].z), a[u][2]);
            a[u][3] = fmaf(gs[j], __uint_as_float(v[u].w), a[u][3]);
          } else {
            const uint32_t yw[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&yw[i]));
              a[u][2 * i] = fmaf(gs[j], f.x, a[u][2 * i]);
              a[u][2 * i + 1] = fmaf(gs[j], f.y, a[u][2 * i + 1]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + 32 * u >= nv) continue;
        uint4 o;
        if (Y_F32) {
          o = make_uint4(__float_as_uint(a[u][0]), __float_as_uint(a[u][1]), __float_as_uint(a[u][2]),
                         __float_as_uint(a[u][3]));
        } else {
          __half2 h0 = __floats2half2_rn(a[u][0], a[u][1]), h1 = __floats2half2_rn(a[u][2], a[u][3]);
          __half2 h2 = __floats2half2_rn(a[u][4], a[u][5]), h3 = __floats2half2_rn(a[u][6], a[u][7]);
          o.x = *reinterpret_cast<uint32_t*>(&h0);
          o.y = *reinterpret_cast<uint32_t*>(&h1);
          o.z = *reinterpret_cast<uint32_t*>(&h2);
          o.w = *reinterpret_cast<uint32_t*>(&h3);
        }
        dst[c0 + 32 * u] = o;
      }
    }
  }
}

// source side (R25): out[t] = Σ_{q = 0..u_t-1} COMB[t·KQ + q] in fp32 (ascending destination),
// u_t = the token's number of distinct destinations with a valid receive row.  Block per token.
template <bool OUT_F32, bool Y_F32>
__global__ void __launch_bounds__(128) k_combine_reduce(Dims d, int T, const int32_t* __restrict__ route, Sym sym,
                                                        int buf_comb, int KQ, void* out) {
  __shared__ int s_u;
  const int tok = blockIdx.x;                    // gl * T + t
  const int gl = tok / T, t = tok % T;
  const int k = d.k;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int dd = -1;
    if (lane < k && route[(static_cast<size_t>(tok) * k + lane) * 2 + 1] >= 0)
      dd = route[(static_cast<size_t>(tok) * k + lane) * 2];
    int head = dd >= 0;
    for (int i = 0; i < k; ++i) {
      const int di = __shfl_sync(0xffffffffu, dd, i);
      if (i < lane && di == dd) head = 0;
    }
    const uint32_t hm = __ballot_sync(0xffffffffu, head != 0);
    if (lane == 0) s_u = __popc(hm);
  }
  __syncthreads();
  const int u = s_u;
  constexpr int ES = Y_F32 ? 4 : 2;
  const size_t rb = static_cast<size_t>(d.H) * ES;
  const uint8_t* base = sym.at(buf_comb, d.G, d.R0 + gl) + (static_cast<size_t>(t) * KQ) * rb;
  const int nv = d.H / 8;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 0.f;
    for (int q = 0; q < u; ++q) {
      const uint8_t* pr = base + q * rb;
      if (Y_F32) {
        const float4 y0 = reinterpret_cast<const float4*>(pr)[2 * c];
        const float4 y1 = reinterpret_cast<const float4*>(pr)[2 * c + 1];
        a[0] += y0.x; a[1] += y0.y; a[2] += y0.z; a[3] += y0.w;
        a[4] += y1.x; a[5] += y1.y; a[6] += y1.z; a[7] += y1.w;
      } else {
        const uint4 v = reinterpret_cast<const uint4*>(pr)[c];
        const uint32_t yw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&yw[i]));
          a[2 * i] += f.x;
          a[2 * i + 1] += f.y;
        }
      }
    }
    if (OUT_F32) {
      float4* o = reinterpret_cast<float4*>(out) + (static_cast<size_t>(tok) * nv + c) * 2;
      o[0] = make_float4(a[0], a[1], a[2], a[3]);
      o[1] = make_float4(a[4], a[5], a[6], a[7]);
    } else {
      uint4 p;
      p.x = pack_bf16(a[0], a[1]);
      p.y = pack_bf16(a[2], a[3]);
      p.z = pack_bf16(a[4], a[5]);
      p.w = pack_bf16(a[6], a[7]);
      reinterpret_cast<uint4*>(out)[static_cast<size_t>(tok) * nv + c] = p;
    }
  }
}

// =============================================================================
// a8 combine: out[t] = Σ_j g_{t,j} · Y_{dest}[row] in slot order, fp32 (R25),
// pulled from the expert ranks' Y buffers (peer loads over NVLink).
// The first CTA raises the prefetch suspend flag (split-phase, R27).
// block per token, 128 threads.
// =============================================================================
template <bool OUT_F32, bool Y_F32 = false, int KC = kMaxK>
__global__ void __launch_bounds__(128) k_combine(Dims d, int T, const float* __restrict__ gw,
                                                 const int32_t* __restrict__ route, Sym sym, int buf_y, void* out,
                                                 volatile int32_t* suspend_flag, int layer) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && suspend_flag) *suspend_flag = layer + 1;
  __shared__ const uint4* srcs[kMaxK];
  __shared__ float gws[kMaxK];
  const int tok = blockIdx.x;           // gl * T + t
  const int k = d.k;
  if (threadIdx.x < k) {
    const int j = threadIdx.x;
    const int dd = route[(static_cast<size_t>(tok) * k + j) * 2];
    const int row = route[(static_cast<size_t>(tok) * k + j) * 2 + 1];
    srcs[j] = row < 0 ? nullptr
                      : reinterpret_cast<const uint4*>(sym.at(buf_y, d.G, dd) +
                                                       static_cast<size_t>(row) * d.H * (Y_F32 ? 4 : 2));
    gws[j] = gw[static_cast<size_t>(tok) * k + j];
  }
  __syncthreads();
  // 8 outputs per thread-iteration: one 16-byte fp16 load per slot (Y rows are fp16, D2),
  // accumulation in fp32 in slot order (R25)
  const int nv = d.H / 8;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 0.f;
    if (Y_F32) {     // fp32 parity path: two 16-byte loads of fp32 Y per 8 outputs
      for (int j = 0; j < k; ++j) {
        if (!srcs[j]) continue;
        const float g = gws[j];
        const float4 y0 = reinterpret_cast<const float4*>(srcs[j])[2 * c];
        const float4 y1 = reinterpret_cast<const float4*>(srcs[j])[2 * c + 1];
        const float f[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fmaf(g, f[q], a[q]);
      }
    } else {
      // issue the token's k loads (≤ KC, peer rows over NVLink) before any use, so a pull keeps
      // k requests in flight per thread; then accumulate in slot order (R25)
      uint4 y[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j)
        if (j < k && srcs[j]) y[j] = srcs[j][c];
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        if (j >= k || !srcs[j]) continue;
        const float g = gws[j];
        const uint32_t yw[4] = {y[j].x, y[j].y, y[j].z, y[j].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&yw[q]));
          a[2 * q] = fmaf(g, f.x, a[2 * q]);
          a[2 * q + 1] = fmaf(g, f.y, a[2 * q + 1]);
        }
      }
    }
    if (OUT_F32) {
      float4* o = reinterpret_cast<float4*>(out) + (static_cast<size_t>(tok) * nv + c) * 2;
      o[0] = make_float4(a[0], a[1], a[2], a[3]);
      o[1] = make_float4(a[4], a[5], a[6], a[7]);
    } else {
      uint4 p;
      p.x = pack_bf16(a[0], a[1]);
      p.y = pack_bf16(a[2], a[3]);
      p.z = pack_bf16(a[4], a[5]);
      p.w = pack_bf16(a[6], a[7]);
      reinterpret_cast<uint4*>(out)[static_cast<size_t>(tok) * nv + c] = p;
    }
  }
}

// =============================================================================
// a9 split-phase prefetch (R27): push replica weights (sender = home
// rank) into the receiver's slot bank.  Chunks are claimed from a counter so
// part 2 resumes where part 1 stopped; part 1 exits once the combine of the
// current layer has raised the suspend flag.
// =============================================================================
constexpr int kPrefetchChunk = 64 * 1024;  // bytes

// Register copy (not TMA bulk): the expert-GEMM CTAs leave < 10 KB of shared memory per
// SM, so a smem-staged copy could not co-reside with them during part 1.  Each thread keeps
// U × 16 B in flight; chunks never straddle the W13 / W2 matrices.  Part 1 uses the
// register-capped instance (MAXR = kPrefetchPart1Reg, U = 8) so that one 128-thread CTA fits
// beside an expert-GEMM CTA capped at (64 K − 2 K − 128·MAXR) / 256 registers.
// Suspension compares the flag for EQUALITY with the layer whose combine suspends this part
// (the combine of layer L stores L + 1): layer ids restart every serving step, so a flag left
// at N by the previous step's last combine must not stop part 1 of an early layer.
constexpr int kPrefetchPart1Reg = 48;
template <int MAXR = 255, int U = 8>
__global__ void __launch_bounds__(512) __maxnreg__(MAXR) k_prefetch(Dims d, const int32_t* __restrict__ replicas, int bank,
                                                  const uint8_t* __restrict__ w13, const uint8_t* __restrict__ w2,
                                                  Sym sym, int buf_rw13, int buf_rw2, int32_t* ctr,
                                                  const volatile int32_t* suspend_flag, int suspend_at,
                                                  int32_t* done_bytes_lo, int elem_bytes) {
  __shared__ int s_chunk;
  const size_t w13_bytes = static_cast<size_t>(2) * d.F * d.H * elem_bytes;
  const size_t w2_bytes = static_cast<size_t>(d.H) * d.F * elem_bytes;
  const int c13 = static_cast<int>((w13_bytes + kPrefetchChunk - 1) / kPrefetchChunk);
  const int c2 = static_cast<int>((w2_bytes + kPrefetchChunk - 1) / kPrefetchChunk);
  const int cper = c13 + c2;
  // transfers whose sender (home of the expert) is a local rank, in (dst, slot) order
  __shared__ int tr_dst[kMaxG * kMaxRb], tr_slot[kMaxG * kMaxRb], tr_e[kMaxG * kMaxRb];
  __shared__ int s_ntr;
  if (threadIdx.x == 0) {
    int ntr = 0;
    for (int r = 0; r < d.G; ++r)
      for (int q = 0; q < kMaxRb; ++q) {
        const int e = replicas[r * kMaxRb + q];
        if (e < 0) continue;
        const int home = e / d.EL;
        if (home < d.R0 || home >= d.R0 + d.GL) continue;
        tr_dst[ntr] = r; tr_slot[ntr] = q; tr_e[ntr] = e; ++ntr;
      }
    s_ntr = ntr;
  }
  __syncthreads();
  const int ntr = s_ntr;
  const int total = ntr * cper;
  while (true) {
    if (threadIdx.x == 0) {
      int c = -1;
      if (!(suspend_at >= 0 && *suspend_flag == suspend_at)) c = atomicAdd(ctr, 1);
      s_chunk = c;
    }
    __syncthreads();
    const int c = s_chunk;
    __syncthreads();
    if (c < 0 || c >= total) break;
    const int ti = c / cper, ci = c % cper;
    const int le = tr_e[ti] - d.R0 * d.EL;      // local expert index within the base weights
    const int slot = bank * kMaxRb + tr_slot[ti];
    const bool first = ci < c13;
    const size_t mat = first ? w13_bytes : w2_bytes;
    const size_t off = static_cast<size_t>(first ? ci : ci - c13) * kPrefetchChunk;
    const size_t len = (off + kPrefetchChunk <= mat) ? kPrefetchChunk : mat - off;
    const uint4* src = reinterpret_cast<const uint4*>((first ? w13 : w2) + static_cast<size_t>(le) * mat + off);
    uint4* dst = reinterpret_cast<uint4*>(sym.at(first ? buf_rw13 : buf_rw2, d.G, tr_dst[ti]) +
                                          static_cast<size_t>(slot) * mat + off);
    const int nv = static_cast<int>(len / 16);
    for (int v0 = 0; v0 < nv; v0 += blockDim.x * U) {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = v0 + u * blockDim.x + threadIdx.x;
        if (i < nv) r[u] = __ldg(src + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = v0 + u * blockDim.x + threadIdx.x;
        if (i < nv) dst[i] = r[u];
      }
    }
    if (threadIdx.x == 0 && done_bytes_lo) atomicAdd(done_bytes_lo, static_cast<int32_t>(len >> 10));
  }
}

// =============================================================================
// Cross-process barrier over the symmetric signal pads (one-sided NVLink stores).
// The epoch of each barrier kind is a DEVICE counter (this process's scratch): the
// kernel reads it, uses counter + 1 and writes that back when done, so a barrier
// captured in a CUDA graph advances on every replay (a host-side epoch frozen into the
// captured launch would let replayed barriers pass at once).  Each kind runs on one
// stream (stream-ordered), and every process issues the same sequence of kinds, so the
// counters advance in lockstep across processes.
// Every local rank l stores the epoch into slot [kind][R0+l] of EVERY rank's pad
// (release, system scope), then waits until its own pad holds >= epoch from all
// G ranks (acquire, system scope).  Orders all prior writes of this stream
// (dispatch rows, count boards, Y rows, replica pushes) before peers proceed.
// One block of GL·G threads; 30 s watchdog (trap) instead of a silent hang.
// =============================================================================
constexpr int kSigKinds = 8;
__global__ void k_xbarrier(Dims d, Sym sym, int buf_sig, int kind, uint32_t* epoch_ctr) {
  __shared__ uint32_t s_ep;
  const int i = threadIdx.x;
  if (i == 0) s_ep = epoch_ctr[kind] + 1u;
  __syncthreads();
  const uint32_t epoch = s_ep;
  if (i < d.GL * d.G) {
    const int l = i / d.G, r = i % d.G;
    uint32_t* peer = reinterpret_cast<uint32_t*>(sym.at(buf_sig, d.G, r)) + kind * kMaxG + (d.R0 + l);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer), "r"(epoch) : "memory");
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(sym.at(buf_sig, d.G, d.R0 + l)) + kind * kMaxG + r;
    uint32_t v;
    const uint64_t t0 = ptx::globaltimer_ns();
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      if (ptx::globaltimer_ns() - t0 > 30000000000ull) __trap();
    }
  }
  __syncthreads();
  if (i == 0) epoch_ctr[kind] = epoch;
}

// analysis helper: one thread spins for ns nanoseconds (%globaltimer)
__global__ void k_spin(long long ns) {
  const uint64_t t0 = ptx::globaltimer_ns();
  while (static_cast<long long>(ptx::globaltimer_ns() - t0) < ns) {
  }
}

// small helper: write a host-described group list into a device schedule
struct SmallGroups {
  int n;
  int BN;
  GemmGroup g[2];
  int TM;   // rows per tile: 128 (1-CTA kernel, the default when 0) or 256 (CTA pair)
};
__global__ void k_write_sched(GemmSched* s, SmallGroups sg) {
  if (threadIdx.x == 0) {
    s->num_groups = sg.n;
    for (int i = 0; i < sg.n; ++i) s->g[i] = sg.g[i];
    gemm_finalize_sched(s, sg.BN, sg.TM ? sg.TM : 128);
  }
}

// Fused gate + predictor stage 1 (probe_config.fuse_gate_predictor): the proto groups (row 0,
// M rows) are repeated for every chunk of CM rows, chunk-major, so the tiles that run at the
// same time share their A rows — x streams from HBM once and the other weight blocks' tiles of
// the chunk hit L2.  One block; thread i writes group i, thread 0 then forms the tile prefix.
__device__ void write_sched_chunked(GemmSched* s, const SmallGroups& sg, int M, int CM) {
  const int TM = sg.TM ? sg.TM : 128;
  const int nc = (M + CM - 1) / CM;
  const int ng = nc * sg.n;
  // tile prefix in closed form (every chunk but the last has CM rows): a serial prefix over
  // 512 groups read back from global memory cost ~0.15 ms on the critical path
  int nt[2], full = 0;
  for (int j = 0; j < sg.n; ++j) {
    nt[j] = gemm_ntiles_n(sg.g[j], sg.BN);
    full += (CM / TM) * nt[j];
  }
  for (int i = threadIdx.x; i < ng; i += blockDim.x) {
    const int c = i / sg.n, j = i % sg.n;
    GemmGroup g = sg.g[j];
    const int r0 = c * CM;
    const size_t es = g.mode == EPI_F32 ? 4 : 2;
    g.a_row += r0;
    g.m = min(CM, M - r0);
    g.out_row += r0;
    g.out = static_cast<uint8_t*>(g.out) + static_cast<size_t>(r0) * g.ldc * es;
    if (g.n_split > 0) g.aux = static_cast<uint8_t*>(g.aux) + static_cast<size_t>(r0) * g.ldc * es;
    int ts = c * full;
    for (int q = 0; q < j; ++q) ts += ((g.m + TM - 1) / TM) * nt[q];
    g.tile_start = ts;
    s->g[i] = g;
  }
  if (threadIdx.x == 0) {
    const int mlast = M - (nc - 1) * CM;
    int last = 0;
    for (int j = 0; j < sg.n; ++j) last += ((mlast + TM - 1) / TM) * nt[j];
    s->num_groups = ng;
    s->nparts = 0;
    s->tile_m = TM;
    s->stats = nullptr;
    sched_reset_counters(s);
    s->total_tiles = (nc - 1) * full + last;
  }
}

// One launch before the fused gate GEMM: every block copies the [W_L ; W_{L+1} ; Ŵ1] row blocks
// into one B operand (16-byte copies; byte counts % 16 == 0), block 0 also writes the
// row-chunk interleaved schedule.
__global__ void k_gate_pred_prep(GemmSched* s, SmallGroups sg, int M, int CM, uint4* __restrict__ dst,
                                 const uint4* __restrict__ a, int64_t na, const uint4* __restrict__ b, int64_t nb,
                                 const uint4* __restrict__ c, int64_t nc) {
  if (blockIdx.x == 0) write_sched_chunked(s, sg, M, CM);
  const int64_t n = na + nb + nc;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = i < na ? a[i] : (i < na + nb ? b[i - na] : c[i - na - nb]);
}

}  // namespace probe
