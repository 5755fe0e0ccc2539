// distill.cuh — online distillation of the lookahead predictor's residual (NEXT-1).
//
// minimise the cross-entropy between the predictor's output and the ground-truth
// router's probability distribution; the frozen prior W_L, b_L is not trained, only
// Ŵ¹ [h,H] and Ŵ² [E,h] of Eq. (P).  Readings R33-R37.
//
// The contractions run on the tcgen05 grouped GEMM (probe.cu); the kernels here are the
// memory-bound glue between them: activation + transpose, the fused softmax / CE / fidelity
// row kernel, the SiLU backward + transpose, and the SGD update.  Transposed operands
// ([·, Np] with Np = N rounded up to 64, zero-padded) make every gradient GEMM a plain
// K-major TMA/UMMA contraction over the token dimension.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace probe {

// a = bf16(SiLU(z)) [N,h] row-major, aT = a transposed [h, Np] (columns ≥ N zero).
// 32×32 tiles through shared memory; block (32, 8).
__global__ void k_act_fwd(const float* __restrict__ z, __nv_bfloat16* __restrict__ a, __nv_bfloat16* __restrict__ aT,
                          int N, int h, int Np) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    __nv_bfloat16 v = __float2bfloat16(0.f);
    if (r < N && c < h) {
      const float zz = z[static_cast<size_t>(r) * h + c];
      v = __float2bfloat16(zz / (1.f + __expf(-zz)));       // Eq. (P), R8
      a[static_cast<size_t>(r) * h + c] = v;
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < h && r < Np) aT[static_cast<size_t>(c) * Np + r] = tile[threadIdx.x][i];
  }
}

// dst [C, Rp] = src [R, C]ᵀ (bf16), columns ≥ R zero.  64×64 tiles, 16-byte global
// accesses on both sides; shared tile rows are 128 B with the 16-byte chunk index XORed by
// (row / 8) so the column gathers of the store phase hit 8 different bank groups.
// Requires C % 8 == 0 and Rp % 8 == 0.
__global__ void __launch_bounds__(256) k_transpose_bf16(const __nv_bfloat16* __restrict__ src,
                                                        __nv_bfloat16* __restrict__ dst, int R, int C, int Rp) {
  __shared__ __align__(16) __nv_bfloat16 tile[64 * 64];
  const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int v = threadIdx.x + 256 * it, r = v >> 3, cv = v & 7;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (r0 + r < R && c0 + cv * 8 < C)
      val = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(r0 + r) * C + c0 + cv * 8);
    *reinterpret_cast<uint4*>(tile + r * 64 + ((cv ^ (r >> 3)) & 7) * 8) = val;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int v = threadIdx.x + 256 * it, oc = v >> 3, rv = v & 7;
    if (c0 + oc >= C || r0 + rv * 8 >= Rp) continue;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = rv * 8 + i;
      o[i] = tile[r * 64 + (((oc >> 3) ^ (r >> 3)) & 7) * 8 + (oc & 7)];
    }
    *reinterpret_cast<uint4*>(dst + static_cast<size_t>(c0 + oc) * Rp + r0 + rv * 8) =
        *reinterpret_cast<const uint4*>(o);
  }
}

// g_z = g_a ⊙ σ'(z), σ'(z) = σ(z)(1 + z(1 − σ(z)))  (R35), written transposed bf16 [h, Np].
__global__ void k_silu_bwd(const float* __restrict__ ga, const float* __restrict__ z, __nv_bfloat16* __restrict__ gzT,
                           int N, int h, int Np) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    float v = 0.f;
    if (r < N && c < h) {
      const size_t o = static_cast<size_t>(r) * h + c;
      const float zz = z[o];
      const float s = 1.f / (1.f + __expf(-zz));
      v = ga[o] * s * (1.f + zz * (1.f - s));
    }
    tile[i][threadIdx.x] = __float2bfloat16(v);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < h && r < Np) gzT[static_cast<size_t>(c) * Np + r] = tile[threadIdx.x][i];
  }
}

// Warp argmax over (value ↓, id ↑) among the experts not yet in `taken` (lane owns experts
// lane + 32 j, j < 8).  Returns the winner's id; every lane agrees.
__device__ __forceinline__ int warp_pick(const float (&v)[8], uint32_t taken, int E, int lane) {
  float bv = -INFINITY;
  int bi = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int e = lane + 32 * j;
    if (e < E && !((taken >> j) & 1u) && (v[j] > bv || (v[j] == bv && e < bi))) { bv = v[j]; bi = e; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  return bi;
}

// One warp per token row: teacher p = softmax(t + b), student q = softmax(l̂ + b) (R33),
// CE = logsumexp(l̂+b) − Σ p (l̂+b) (R34), g_l = q − p → bf16 [N,E] and transposed [E,Np];
// fidelity hit counts (R37).  stats (fp64): [0] Σ CE, [1] Σ|S∩P|, [2] Σ|S^{⌈k/2⌉}∩P|,
// [3] Σ|S∩P^{2k}|.  Block = 32 warps = 32 tokens (one 64-byte segment per expert row of glT).
__global__ void __launch_bounds__(1024) k_distill_ce(const float* __restrict__ lhat, const float* __restrict__ tl,
                                                     const float* __restrict__ bias, int N, int E, int k, int Np,
                                                     __nv_bfloat16* __restrict__ gl, __nv_bfloat16* __restrict__ glT,
                                                     double* __restrict__ stats) {
  __shared__ __nv_bfloat16 sg[32][kMaxE + 8];
  __shared__ float sred[32][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 32, n = n0 + warp;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (n >= N) {
    for (int e = lane; e < E; e += 32) sg[warp][e] = __float2bfloat16(0.f);
  } else {
    float sv[8], tv[8];
    float sm = -INFINITY, tm = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = lane + 32 * j;
      sv[j] = tv[j] = -INFINITY;
      if (e < E) {
        const float bb = bias ? bias[e] : 0.f;
        sv[j] = lhat[static_cast<size_t>(n) * E + e] + bb;
        tv[j] = tl[static_cast<size_t>(n) * E + e] + bb;
        sm = fmaxf(sm, sv[j]);
        tm = fmaxf(tm, tv[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sm = fmaxf(sm, __shfl_xor_sync(0xffffffffu, sm, o));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    }
    float ss = 0.f, ts = 0.f, tsl = 0.f;
    float se[8], te[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      se[j] = lane + 32 * j < E ? __expf(sv[j] - sm) : 0.f;
      te[j] = lane + 32 * j < E ? __expf(tv[j] - tm) : 0.f;
      ss += se[j];
      ts += te[j];
      tsl += lane + 32 * j < E ? te[j] * sv[j] : 0.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      ts += __shfl_xor_sync(0xffffffffu, ts, o);
      tsl += __shfl_xor_sync(0xffffffffu, tsl, o);
    }
    if (lane == 0) acc[0] = sm + __logf(ss) - tsl / ts;       // CE_t (R34; every lane holds it)
    const float is = 1.f / ss, it = 1.f / ts;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = lane + 32 * j;
      // g_l = q − p; explicit roundings (no FMA contraction) so q ≡ p gives exactly 0
      if (e < E) sg[warp][e] = __float2bfloat16(__fsub_rn(__fmul_rn(se[j], is), __fmul_rn(te[j], it)));
    }
    // fidelity sets (R37): S = teacher top-k (first ⌈k/2⌉ = S^half), P2 = student top-2k
    // (k == 0: metrics not requested — the serial warp argmaxes dominate this kernel)
    uint32_t mS = 0, mSh = 0, mP = 0, mP2 = 0;
    for (int i = 0; i < k; ++i) {
      const int w = warp_pick(tv, mS, E, lane);
      if ((w & 31) == lane) { mS |= 1u << (w >> 5); if (i < (k + 1) / 2) mSh |= 1u << (w >> 5); }
    }
    const int k2 = min(2 * k, E);
    for (int i = 0; i < k2; ++i) {
      const int w = warp_pick(sv, mP2, E, lane);
      if ((w & 31) == lane) { mP2 |= 1u << (w >> 5); if (i < k) mP |= 1u << (w >> 5); }
    }
    acc[1] = __popc(mS & mP);
    acc[2] = __popc(mSh & mP);
    acc[3] = __popc(mS & mP2);
  }
  __syncthreads();
  // g_l row-major (one row per warp) and transposed (32 tokens = 64 B per expert row)
  if (n < N)
    for (int e = lane; e < E; e += 32) gl[static_cast<size_t>(n) * E + e] = sg[warp][e];
  for (int e = warp; e < E; e += 32) {
    const int nn = n0 + lane;
    if (nn < Np) glT[static_cast<size_t>(e) * Np + nn] = sg[lane][e];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sred[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += sred[w][threadIdx.x];
    atomicAdd(stats + threadIdx.x, t);
  }
}

// out[i] = Σ_{s < S} part[s·n + i] in order s = 0, 1, … (deterministic split-K reduction).
__global__ void k_sum_partials(const float* __restrict__ part, float* __restrict__ out, int64_t n, int S) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float a = part[i];
    for (int s = 1; s < S; ++s) a += part[static_cast<size_t>(s) * n + i];
    out[i] = a;
  }
}

// All GEMM schedules of one distillation step written by one launch (thread i → schedule i).
constexpr int kDistillScheds = 6, kSplitMax = 8;
struct SchedSpec {
  int n;
  GemmGroup g[kSplitMax];
};
struct DistillSpecs {
  SchedSpec s[kDistillScheds];
};
__global__ void k_write_scheds(GemmSched* base, DistillSpecs sp) {
  const int i = threadIdx.x;
  if (i < kDistillScheds) {
    GemmSched* s = base + i;
    s->num_groups = sp.s[i].n;
    for (int j = 0; j < sp.s[i].n; ++j) s->g[j] = sp.s[i].g[j];
    gemm_finalize_sched(s, 128);
  }
}

// R36: master ← master + scale · grad (scale = −lr / N_total), w = bf16(master).
__global__ void k_sgd(float* __restrict__ master, const float* __restrict__ grad, __nv_bfloat16* __restrict__ w,
                      int64_t n, float scale) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float m = fmaf(scale, grad[i], master[i]);
    master[i] = m;
    w[i] = __float2bfloat16(m);
  }
}

}  // namespace probe
