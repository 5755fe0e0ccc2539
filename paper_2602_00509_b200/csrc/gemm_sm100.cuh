// gemm_sm100.cuh — persistent grouped bf16 GEMM on 5th-gen tensor cores.
//
// Hot step a7 of the PROBE layer (grouped SwiGLU expert FFN, PAPER.md P:167-171,
// §3.2 Eq. 2 "executes its assigned experts using Grouped GEMM") and
// the router / predictor GEMMs (a1, a2).
//
// Design (sm_100a):
//  * one CTA (or CTA pair) per SM, tiles of ALL groups claimed dynamically from a global
//    counter; group table + tile prefix live in device memory (written by the layout
//    kernel), so no host sync and CUDA-Graph safe;
//  * tile 128 × BN, K-step 64 (one 128-byte SWIZZLE_128B row per operand row);
//  * warp 0: TMA producer (cp.async.bulk.tensor → STAGES-deep smem ring, mbarriers);
//    warp 1: single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per instruction,
//            fp32 accumulator in TMEM, 2 accumulator buffers = 2·BN columns);
//    warp 2: TMEM allocator;  warps 4-7: epilogue (tcgen05.ld → fused epilogue → st.global);
//  * epilogues: fp32 store (logits), fp16 store (expert output Y), SwiGLU → bf16 (gate cols | up cols in one
//    accumulator: the B tile is two TMA boxes, gate rows n0.. and up rows F+n0..),
//    SiLU → bf16 (predictor residual activation, R8 rounding point).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100_ptx.cuh"

namespace probe {

enum : int {
  EPI_F32 = 0,         // fp32 C (Y, logits)
  EPI_SWIGLU = 1,      // act = SiLU(gate) ⊙ up → bf16
  EPI_SILU_BF16 = 2,   // SiLU → bf16 (predictor residual activation, R8)
  EPI_NONE = 3,        // timing experiments: no stores
  EPI_TOPK = 4,        // router: per-row top-k (logit ↓, id ↑) + softmax over the k → ids, weights (a1)
  EPI_TOPK_COUNT = 5,  // predictor: per-row top-k → atomic per-(rank, expert) counts n̂ (a2, R9)
  EPI_F16 = 6          // fp16 C (expert output Y, D2): |y| > 65504 raises kErrYRange in *aux
};
constexpr int kErrYRange = 8;   // device error bit (kernels.cuh ERR_Y_RANGE)
constexpr int kTopkMax = 8;   // fused top-k supports k <= 8 (larger k uses the unfused kernel)

struct GemmGroup {
  int32_t a_row;       // first row in the A tensor map
  int32_t m;           // rows in this group
  int32_t b_row;       // first weight row in the selected B tensor map
  int32_t b_sel;       // 0: tmB0, 1: tmB1
  int32_t mode;        // EPI_*
  int32_t n;           // output columns (SwiGLU: activation columns = F)
  int32_t ldc;         // output row stride, elements
  int32_t tile_start;  // prefix of tiles over groups
  int32_t out_row;     // row of this group's row 0 in the output tensor map (TMA store path)
  int32_t tma_out;     // 1: fp32 output through the tmC tensor map (full 32-row slabs)
  int32_t topk;        // EPI_TOPK*: k
  int32_t rows_per_rank;  // EPI_TOPK_COUNT: tokens per rank (rank = (a_row + row) / rows_per_rank)
  int32_t k_off;       // first K element of the (first) K segment: split-K partial products
  int32_t n_split;     // EPI_F32, > 0: columns >= n_split go to `aux` at column - n_split (same ldc);
                       // a multiple of 32, so no 32-column chunk straddles it
  void* out;           // output of row 0 / col 0 of this group (EPI_TOPK: int32 ids [m, k])
  void* aux;           // EPI_TOPK: fp32 weights [m, k]; EPI_TOPK_COUNT: int32 counts [ranks, n]
  const float* bias;   // EPI_TOPK*: optional fp32 bias [n]
};

constexpr int kMaxGroups = 1024;
constexpr int kMaxParts = 64;

struct GemmSched {
  int32_t num_groups;
  int32_t total_tiles;
  int32_t nparts;                    // >1: CTA (pair) b serves only partition b % nparts (EP emulation)
  int32_t counter;                   // dynamic tile counter (reset by the kernel writing the schedule)
  int32_t tile_m;                    // rows per tile: 128 (1-CTA MMA) or 256 (CTA pair, cta_group::2)
  int32_t l2hint;                    // CTA-pair kernel TMA L2 hints: bit 0 C stores evict_first, bit 1 B loads
                                     // evict_last, bit 2 A loads evict_first (0 = none)
  int32_t part_tile[kMaxParts + 1];  // tile range [part_tile[p], part_tile[p+1]) of partition p
  int32_t part_counter[kMaxParts];   // per-partition tile counters
  unsigned long long* stats;         // optional per-role wait-cycle counters (timing hook only)
  GemmGroup g[kMaxGroups];
};
// stats[0] producer waits on `empty`   stats[1] MMA waits on `full`   stats[2] MMA waits on `tempty`
// stats[3] epilogue waits on `tfull`   stats[4] epilogue busy          stats[5] tiles    stats[6] CTA cycles

// Dynamic persistent tile scheduling: the producer warp claims the next tile from a
// global atomic counter and hands it to the MMA and epilogue warps through an
// mbarrier-guarded shared-memory queue.  CTAs that start late (SMs still busy with a
// concurrent aux-stream kernel) simply take fewer tiles.  Partitioned mode (single-GPU EP
// emulation): CTA b serves only partition b % nparts (its logical rank's tiles), so a rank's
// expert GEMM runs on ~#SMs/nparts SMs and the launch time is the straggler's (Eq. 3).
constexpr int kTileQ = 8;
// Claim split in two so the atomic's latency hides behind a whole tile of TMA issue: the raw
// counter value is requested when a tile starts and turned into a tile id (or -1) when the
// next tile is published (K = 768 tiles are only 12 k-blocks long, so a claim at the tile
// boundary can show up as operand waits of the MMA).
__device__ __forceinline__ int claim_raw(GemmSched* s, int unit) {
  const int np = s->nparts;
  if (np > 1) return atomicAdd(&s->part_counter[(unit < 0 ? static_cast<int>(blockIdx.x) : unit) % np], 1);
  return atomicAdd(&s->counter, 1);
}
__device__ __forceinline__ int claim_finish(const GemmSched* s, int unit, int raw) {
  const int np = s->nparts;
  if (np > 1) {
    const int p = (unit < 0 ? static_cast<int>(blockIdx.x) : unit) % np;
    const int t = s->part_tile[p] + raw;
    return t < s->part_tile[p + 1] ? t : -1;
  }
  return raw < s->total_tiles ? raw : -1;
}

__device__ __forceinline__ void sched_reset_counters(GemmSched* s) {
  s->counter = 0;
  for (int p = 0; p < kMaxParts; ++p) s->part_counter[p] = 0;
}

__host__ __device__ inline int gemm_ntiles_n(const GemmGroup& G, int BN) {
  const int bno = (G.mode == EPI_SWIGLU) ? BN / 2 : BN;
  return (G.n + bno - 1) / bno;
}
__host__ __device__ inline int gemm_ntiles(const GemmGroup& G, int BN, int TM = 128) {
  return G.m <= 0 ? 0 : ((G.m + TM - 1) / TM) * gemm_ntiles_n(G, BN);
}

// Serial prefix over the group table (called by one thread).
__device__ inline void gemm_finalize_sched(GemmSched* s, int BN, int TM = 128) {
  s->nparts = 0;
  s->tile_m = TM;
  s->stats = nullptr;
  sched_reset_counters(s);
  int acc = 0;
  for (int i = 0; i < s->num_groups; ++i) {
    s->g[i].tile_start = acc;
    acc += gemm_ntiles(s->g[i], BN, TM);
  }
  s->total_tiles = acc;
}

template <int BN, int STAGES, int EW = 4, int NBUF = (EW == 8 ? 2 : 1)>
struct GemmSmem {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int BAR_OFF = STAGES * (A_BYTES + B_BYTES);
  static constexpr int TS_OFF = BAR_OFF + (2 * STAGES + 4 + 2 * kTileQ) * 8 + 16 + kTileQ * 4;
  static constexpr int EPI_OFF = (TS_OFF + (kMaxGroups + 1) * 4 + 1023) / 1024 * 1024;
  // per epilogue warp: NB staging tiles of 32 rows × 128 B, 16-byte chunks XOR-swizzled by
  // (row mod 8) = the TMA SWIZZLE_128B layout (also bank-conflict-free for the manual path)
  static constexpr int NB = NBUF;
  static constexpr int EPI_STRIDE = NB * 4096;
  static constexpr int BYTES = EPI_OFF + EW * EPI_STRIDE + 1024;                // + alignment slack
};

__device__ __forceinline__ int gemm_find_group(const int* ts, int ng, int tile) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// SiLU in the tensor-core epilogues: MUFU exp + MUFU reciprocal (__fdividef, 2 ulp; → 0 for
// v < -88 where the denominator overflows).  An IEEE division here made the SiLU epilogues
// 3.5× costlier than a plain store (per-role counters: the predictor's Ŵ1·x GEMM was
// epilogue-bound, 685 vs 1107 TF/s), far above the bf16 rounding that follows (2^-9).
__device__ __forceinline__ float silu_f(float v) { return __fdividef(v, 1.0f + __expf(-v)); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Swizzled 32×32 fp32 staging tile (row r at r·32 floats, 16-B chunk j at (j ^ (r & 7)) · 4).
__device__ __forceinline__ int swz(int r, int j) { return r * 32 + ((j ^ (r & 7)) << 2); }

// Write the staged rows with coalesced row segments (fp32: 4 rows × 128 B per warp store;
// bf16: 8 rows × 64 B) masking rows ≥ G.m and columns ≥ G.n (group tails).
__device__ __forceinline__ void epi_store_manual(const float* tile, int lane, const GemmGroup& G, int row0,
                                                 int col0, bool h16 = false) {
  if (G.mode == EPI_NONE) return;
  if (G.mode == EPI_F16 || h16) {   // 16-bit tile: 32 rows × 64 B, 16-byte chunk j at (j ^ ((r >> 1) & 3))
    const char* tb = reinterpret_cast<const char*>(tile);
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int rl = it * 8 + (lane >> 2), j = lane & 3;
      const int grow = row0 + rl;
      if (grow < G.m && col0 + 8 * j < G.n)
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(G.out) + static_cast<size_t>(grow) * G.ldc + col0 + 8 * j) =
            *reinterpret_cast<const uint4*>(tb + rl * 64 + ((j ^ ((rl >> 1) & 3)) << 4));
    }
    return;
  }
  if (G.mode == EPI_F32) {
    // fused gate + predictor GEMM (EPI_F32 with n_split): the chunk lands in the second output
    const bool hi = G.n_split > 0 && col0 >= G.n_split;
    float* base = reinterpret_cast<float*>(hi ? G.aux : G.out);
    const int c0 = hi ? col0 - G.n_split : col0;
    const int nlim = hi ? G.n - G.n_split : (G.n_split > 0 ? G.n_split : G.n);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int rl = it * 4 + (lane >> 3), j = lane & 7;
      const int grow = row0 + rl;
      if (grow < G.m && c0 + 4 * j < nlim)
        *reinterpret_cast<float4*>(base + static_cast<size_t>(grow) * G.ldc + c0 + 4 * j) =
            *reinterpret_cast<const float4*>(tile + swz(rl, j));
    }
  } else {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int rl = it * 8 + (lane >> 2), j = (lane & 3) * 2;
      const int grow = row0 + rl;
      if (grow < G.m && col0 + 4 * j < G.n) {
        const float4 a = *reinterpret_cast<const float4*>(tile + swz(rl, j));
        const float4 b = *reinterpret_cast<const float4*>(tile + swz(rl, j + 1));
        uint4 o;
        o.x = pack_bf16(a.x, a.y);
        o.y = pack_bf16(a.z, a.w);
        o.z = pack_bf16(b.x, b.y);
        o.w = pack_bf16(b.z, b.w);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(G.out) + static_cast<size_t>(grow) * G.ldc + col0 +
                                  4 * j) = o;
      }
    }
  }
}

// Stage one warp's 32 rows × 32 values (row = lane) and store them: TMA tensor store
// for full 32-row fp32 slabs (tma_out), coalesced manual stores otherwise.  `tsel`
// rotates over NB tiles; lane 0 owns the bulk-async group of this warp.
template <int NB>
__device__ __forceinline__ void epi_chunk(float* tiles, int& tsel, int lane, const float (&v)[32],
                                          const GemmGroup& G, const CUtensorMap* tmC, int row0, int col0,
                                          uint64_t store_pol = 0) {
  if (G.mode == EPI_NONE) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
    if (acc == 12345.678f) tiles[lane] = acc;   // keep the TMEM loads alive
    return;
  }
  // 16-bit tiles (fp16 Y, and the bf16 activations of EPI_SWIGLU / EPI_SILU_BF16 when they
  // are TMA-stored) are 2 KB, so the 4 KB staging slot holds two and the warp can stage the
  // next chunk while the TMA store of the previous one is still reading (a launch never mixes
  // 16-bit and 32-bit staging, so the rotation is uniform within it).  The bf16 TMA store
  // halves the predictor's SiLU GEMM time against per-lane stores (C1 shape: 216 → ~120 µs).
  const bool bf16t = G.tma_out && (G.mode == EPI_SWIGLU || G.mode == EPI_SILU_BF16);
  const bool f16 = G.mode == EPI_F16 || bf16t;
  const int slot = tsel & 0xff;
  float* tile = f16 ? tiles + slot * 512 : tiles + slot * 1024;
  if (lane == 0) {
    if (f16) ptx::bulk_wait_read<2 * NB - 1>();
    else ptx::bulk_wait_read<NB - 1>();          // the TMA store that last read this tile is done
  }
  __syncwarp();
  if (f16) {
    // row = lane: 32 halves = 64 B in the TMA SWIZZLE_64B layout (chunk j at j ^ ((row >> 1) & 3))
    bool big = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 p;
      uint32_t* pw = reinterpret_cast<uint32_t*>(&p);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = v[8 * j + 2 * q], b = v[8 * j + 2 * q + 1];
        if (bf16t) {
          pw[q] = pack_bf16(a, b);
        } else {
          big |= fabsf(a) > 65504.f || fabsf(b) > 65504.f;
          __half2 hh = __floats2half2_rn(a, b);
          pw[q] = *reinterpret_cast<uint32_t*>(&hh);
        }
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<char*>(tile) + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = p;
    }
    // only rows / columns of this group count (tile rows past G.m hold other groups' or
    // never-written receive rows)
    big = big && row0 + lane < G.m && col0 < G.n;
    if (__any_sync(0xffffffffu, big) && lane == 0 && G.aux) atomicOr(reinterpret_cast<int*>(G.aux), kErrYRange);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(tile + swz(lane, j)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
  const bool tma = G.tma_out && (row0 + 31 < G.m) && (col0 < G.n);
  if (tma) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (store_pol) ptx::tma_store_2d_hint(tmC, tile, col0, G.out_row + row0, store_pol);
      else ptx::tma_store_2d(tmC, tile, col0, G.out_row + row0);
      ptx::bulk_commit();
    }
  } else {
    __syncwarp();
    epi_store_manual(tile, lane, G, row0, col0, f16);
    // an EMPTY bulk group keeps "one group per staged chunk": the bulk_wait_read above counts
    // groups, and a chunk without a TMA store (row tail, or a column chunk past G.n in a ragged
    // last N tile) must not let the wait skip the store still reading the slot it reuses —
    // without this the C2 Y columns 2848..2879 (H = 2880) were intermittently overwritten
    if (lane == 0) ptx::bulk_commit();
  }
  __syncwarp();
  tsel = (tsel & ~0xff) | ((slot + 1) % (f16 ? 2 * NB : NB));
}

// fp16 Y with 64-column TMA stores (tma_out == 2): the warp's two adjacent 32-column chunks
// are staged as one 32-row × 128-byte tile (SWIZZLE_128B: 16-byte chunk j of row r at
// j ^ (r & 7)) and leave in ONE tensor store of full 128-byte row segments — half the TMA
// store operations (and half-line writes) of two 64-byte-row stores.  The 4 KB staging slot
// is single-buffered: the previous store must have finished reading it.
template <int NB>
__device__ __forceinline__ void epi_chunk64_f16(float* tiles, int& tsel, int lane, const uint32_t (&va)[32],
                                                const uint32_t (&vb)[32], const GemmGroup& G,
                                                const CUtensorMap* tmC, int row0, int col0, uint64_t store_pol) {
  const int slot = NB > 1 ? (tsel & 1) : 0;     // NB = 2: two 4 KB tiles, one store in flight while staging
  char* tile = reinterpret_cast<char*>(tiles) + slot * 4096;
  if (lane == 0) ptx::bulk_wait_read<NB - 1>();
  __syncwarp();
  bool big = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint4 p;
    uint32_t* pw = reinterpret_cast<uint32_t*>(&p);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = __uint_as_float(j < 4 ? va[8 * j + 2 * q] : vb[8 * (j - 4) + 2 * q]);
      const float b = __uint_as_float(j < 4 ? va[8 * j + 2 * q + 1] : vb[8 * (j - 4) + 2 * q + 1]);
      big |= fabsf(a) > 65504.f || fabsf(b) > 65504.f;
      __half2 hh = __floats2half2_rn(a, b);
      pw[q] = *reinterpret_cast<uint32_t*>(&hh);
    }
    *reinterpret_cast<uint4*>(tile + lane * 128 + ((j ^ (lane & 7)) << 4)) = p;
  }
  big = big && row0 + lane < G.m && col0 < G.n;
  if (__any_sync(0xffffffffu, big) && lane == 0 && G.aux) atomicOr(reinterpret_cast<int*>(G.aux), kErrYRange);
  if (row0 + 31 < G.m && col0 < G.n) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (store_pol) ptx::tma_store_2d_hint(tmC, tile, col0, G.out_row + row0, store_pol);
      else ptx::tma_store_2d(tmC, tile, col0, G.out_row + row0);
      ptx::bulk_commit();
    }
  } else {
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 8; ++it) {       // 4 rows × 128 B per warp store
      const int rl = it * 4 + (lane >> 3), j = lane & 7;
      const int grow = row0 + rl;
      if (grow < G.m && col0 + 8 * j < G.n)
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(G.out) + static_cast<size_t>(grow) * G.ldc + col0 + 8 * j) =
            *reinterpret_cast<const uint4*>(tile + rl * 128 + ((j ^ (rl & 7)) << 4));
    }
    if (lane == 0) ptx::bulk_commit();     // an empty group keeps one group per staged tile
  }
  __syncwarp();
  tsel = 0x200 | (slot ^ 1);
}

// Top-k by sorting networks (R3, R4): keys ordered by (value ↓, id ↑), a total order, so any
// correct network gives the lowest-id tie rule.  Each group of 8 logits is sorted with the
// 19-comparator odd-even merge network, merged into the running top 8 (the element-wise
// better of top[i] and group[7-i] is bitonic and holds the top 8 of both), and re-sorted
// with a 12-comparator bitonic cleaner.  Branch-free with independent comparators per
// stage: the former insertion chain was predicated over every logit (11 K instructions per
// warp at C1) and latency-bound at 13 warps per SM.
__device__ __forceinline__ void topk_ce(float& av, int& ae, float& bv, int& be) {
  const bool s = (bv > av) || (bv == av && be < ae);
  const float tv = s ? bv : av;
  const int te = s ? be : ae;
  bv = s ? av : bv;
  be = s ? ae : be;
  av = tv;
  ae = te;
}
__device__ __forceinline__ void topk_sort8(float (&v)[8], int (&e)[8]) {
#define CE(i, j) topk_ce(v[i], e[i], v[j], e[j])
  CE(0, 1); CE(2, 3); CE(4, 5); CE(6, 7);
  CE(0, 2); CE(1, 3); CE(4, 6); CE(5, 7);
  CE(1, 2); CE(5, 6);
  CE(0, 4); CE(1, 5); CE(2, 6); CE(3, 7);
  CE(2, 4); CE(3, 5);
  CE(1, 2); CE(3, 4); CE(5, 6);
#undef CE
}
__device__ __forceinline__ void topk_merge8(float (&tv)[8], int (&te)[8], const float (&gv)[8], const int (&ge)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float bv = gv[7 - i];
    const int be = ge[7 - i];
    const bool s = (bv > tv[i]) || (bv == tv[i] && be < te[i]);
    tv[i] = s ? bv : tv[i];
    te[i] = s ? be : te[i];
  }
#define CE(i, j) topk_ce(tv[i], te[i], tv[j], te[j])
  CE(0, 4); CE(1, 5); CE(2, 6); CE(3, 7);
  CE(0, 2); CE(1, 3); CE(4, 6); CE(5, 7);
  CE(0, 1); CE(2, 3); CE(4, 5); CE(6, 7);
#undef CE
}

// Fused router / predictor top-k in the GEMM epilogue (a1, a2): row = token (lane).  Each
// 32-column TMEM load holds 32 logits of this lane's row; they are ranked 8 at a time with
// the sorting networks above (keys (value ↓, id ↑), R3, R4) — the same selection and the same
// fp32 softmax as k_select, with compile-time register indices (no staging, no branches).
template <int KK, int BN>
__device__ __forceinline__ void epi_topk(uint32_t tb, int lane, const GemmGroup& G, int row0, float* stage) {
  (void)stage;
  float tv[8];
  int te[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { tv[j] = -INFINITY; te[j] = 0x7fffffff; }
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    if (c * 32 >= G.n) break;
    uint32_t v32[32];
    ptx::tmem_ld32_wait(tb + c * 32, v32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float gv[8];
      int ge[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = c * 32 + q * 8 + i;
        float x = __uint_as_float(v32[q * 8 + i]);
        if (G.bias && e < G.n) x += __ldg(G.bias + e);
        gv[i] = e < G.n ? x : -INFINITY;      // columns past n never beat a real logit (larger id)
        ge[i] = e;
      }
      topk_sort8(gv, ge);
      topk_merge8(tv, te, gv, ge);
    }
  }
  const int row = row0 + lane;
  if (row >= G.m) return;
  if (G.mode == EPI_TOPK) {
    float w[KK], sum = 0.f;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      w[j] = expf(tv[j] - tv[0]);
      sum += w[j];
    }
    int32_t* ids = reinterpret_cast<int32_t*>(G.out) + static_cast<size_t>(row) * KK;
    float* gw = reinterpret_cast<float*>(G.aux) + static_cast<size_t>(row) * KK;
#pragma unroll
    for (int j = 0; j < KK; ++j) { ids[j] = te[j]; gw[j] = w[j] / sum; }
  } else {
    int32_t* cnt = reinterpret_cast<int32_t*>(G.aux) + static_cast<size_t>((G.a_row + row) / G.rows_per_rank) * G.n;
#pragma unroll
    for (int j = 0; j < KK; ++j) atomicAdd(cnt + te[j], 1);
  }
}

// Epilogue of one output tile for one epilogue warp: TMEM lanes of this warp (row0..row0+31),
// the column chunks c ≡ part (mod NPART).  Shared by the 1-CTA and the 2-CTA kernels.
template <int BN, int NB, int NPART>
__device__ __forceinline__ void epi_tile(uint32_t tb, int lane, int part, const GemmGroup& G, int row0, int nb,
                                         float* tiles, int& tsel, const CUtensorMap* tmC, uint64_t store_pol = 0) {
  if (G.mode == EPI_TOPK || G.mode == EPI_TOPK_COUNT) {
    switch (G.topk) {
      case 1: epi_topk<1, BN>(tb, lane, G, row0, tiles); break;
      case 2: epi_topk<2, BN>(tb, lane, G, row0, tiles); break;
      case 3: epi_topk<3, BN>(tb, lane, G, row0, tiles); break;
      case 4: epi_topk<4, BN>(tb, lane, G, row0, tiles); break;
      case 5: epi_topk<5, BN>(tb, lane, G, row0, tiles); break;
      case 6: epi_topk<6, BN>(tb, lane, G, row0, tiles); break;
      case 7: epi_topk<7, BN>(tb, lane, G, row0, tiles); break;
      default: epi_topk<8, BN>(tb, lane, G, row0, tiles); break;
    }
  } else if (G.mode == EPI_SWIGLU) {
#pragma unroll 1
    for (int c = part; c < BN / 64; c += NPART) {
      uint32_t gv[32], uv[32];
      ptx::tmem_ld32x2_wait(tb + c * 32, gv, tb + BN / 2 + c * 32, uv);
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = silu_f(__uint_as_float(gv[i])) * __uint_as_float(uv[i]);
      epi_chunk<NB>(tiles, tsel, lane, v, G, tmC, row0, nb * (BN / 2) + c * 32, store_pol);
    }
  } else {
    // two chunks in flight per TMEM wait
    // A launch may mix 32-bit and 16-bit staging only across groups (the fused gate +
    // predictor GEMM: fp32 logits tiles, then TMA-stored bf16 activation tiles).  The slot
    // rotation assumes one geometry, so a change of kind drains this warp's stores first.
    const bool wide = NPART == 1 && G.mode == EPI_F16 && G.tma_out == 2;
    const int kind = wide ? 0x200 : (G.mode == EPI_F16 || (G.tma_out && G.mode == EPI_SILU_BF16)) ? 0x100 : 0;
    if ((tsel & 0x300) != kind) {
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
      tsel = kind;
    }
    if (wide) {
#pragma unroll 1
      for (int c = 0; c < BN / 32; c += 2) {
        uint32_t va[32], vb[32];
        ptx::tmem_ld32x2_wait(tb + c * 32, va, tb + (c + 1) * 32, vb);
        epi_chunk64_f16<NB>(tiles, tsel, lane, va, vb, G, tmC, row0, nb * BN + c * 32, store_pol);
      }
      return;
    }
#pragma unroll 1
    for (int c = part; c < BN / 32; c += 2 * NPART) {
      const int c2 = c + NPART;
      uint32_t va[32], vb[32];
      if (c2 < BN / 32) ptx::tmem_ld32x2_wait(tb + c * 32, va, tb + c2 * 32, vb);
      else ptx::tmem_ld32_wait(tb + c * 32, va);
      float v[32];
      const bool silu = G.mode == EPI_SILU_BF16;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = h == 0 ? c : c2;
        if (cc >= BN / 32) break;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float x = __uint_as_float(h == 0 ? va[i] : vb[i]);
          v[i] = silu ? silu_f(x) : x;
        }
        epi_chunk<NB>(tiles, tsel, lane, v, G, tmC, row0, nb * BN + cc * 32, store_pol);
      }
    }
  }
}

// EW epilogue warps (4 or 8): warp 4+i reads TMEM lane quarter i%4 and handles the
// column chunks c ≡ i/4 (mod EW/4).  Threads = 128 + 32·EW.
// Per-role wait-cycle counters: compiled only into the analysis build (-DPROBE_GEMM_STATS,
// tools/gemm_stats.py); the product build has no instrumentation.
#ifdef PROBE_GEMM_STATS
#define GEMM_TIMED_WAIT(bar, par, slot)                        \
  do {                                                         \
    const long long t0_ = clock64();                           \
    ptx::mbar_wait(bar, par);                                  \
    acc_st[slot] += clock64() - t0_;                           \
  } while (0)
#define GEMM_STAT(...) __VA_ARGS__
#else
#define GEMM_TIMED_WAIT(bar, par, slot) ptx::mbar_wait(bar, par)
#define GEMM_STAT(...)
#endif

template <int BN, int STAGES, int EW = 4, int NBUF = (EW == 8 ? 2 : 1), int MAXR = 255>
__global__ void __launch_bounds__(128 + 32 * EW, 1) __maxnreg__(MAXR)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                    const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmC,
                    const __grid_constant__ CUtensorMap tmA2, GemmSched* __restrict__ sched, int K, int K2) {
  using L = GemmSmem<BN, STAGES, EW, NBUF>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* qfull = tempty + 2;                 // tile queue (producer → MMA + epilogue warps)
  uint64_t* qempty = qfull + kTileQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qempty + kTileQ);
  volatile int* tq = reinterpret_cast<volatile int*>(tmem_slot + 4);
  int* ts = reinterpret_cast<int*>(smem + L::TS_OFF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ng = sched->num_groups;
  GEMM_STAT(long long acc_st[7] = {0, 0, 0, 0, 0, 0, 0});
  GEMM_STAT(const long long t_kernel0 = clock64());
  for (int i = threadIdx.x; i < ng; i += blockDim.x) ts[i] = sched->g[i].tile_start;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], EW);
    }
    for (int q = 0; q < kTileQ; ++q) {
      ptx::mbar_init(&qfull[q], 1);
      ptx::mbar_init(&qempty[q], 1 + EW);
    }
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB0);
    ptx::tma_prefetch_desc(&tmB1);
    if (K2 > 0) ptx::tma_prefetch_desc(&tmA2);
  }
  if (warp == 2) ptx::tmem_alloc<2 * BN>(tmem_slot);
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // K concatenation (predictor: [x | a]·[W_next | Ŵ2]ᵀ): k-blocks [0, kb1) read (tmA, selected B),
  // k-blocks [kb1, num_kb) read (tmA2, tmB1) — both halves accumulate into one TMEM tile.
  const int kb1 = (K + 63) / 64;
  const int num_kb = kb1 + (K2 > 0 ? (K2 + 63) / 64 : 0);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (warp 0,
    // lane 0: claims tiles and loads the A / B tiles)
    int stage = 0;
    uint32_t phase = 0;
    int qs = 0;
    uint32_t qph = 0;
    int raw_next = lane == 0 ? claim_raw(sched, -1) : 0;
    while (true) {
      int tile = 0;
      if (lane == 0) {
        tile = claim_finish(sched, -1, raw_next);
        if (tile >= 0) raw_next = claim_raw(sched, -1);   // next tile's claim in flight during this tile
        ptx::mbar_wait(&qempty[qs], qph ^ 1);
        tq[qs] = tile;
        ptx::mbar_arrive(&qfull[qs]);
      }
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (++qs == kTileQ) { qs = 0; qph ^= 1; }
      if (tile < 0) break;
      const int gi = gemm_find_group(ts, ng, tile);
      const GemmGroup& G = sched->g[gi];
      const int nt = gemm_ntiles_n(G, BN);
      const int tin = tile - ts[gi];
      const int mb = tin / nt, nb = tin % nt;
      const int arow = G.a_row + mb * 128;
      int brow0, brow1;
      if (G.mode == EPI_SWIGLU) {
        brow0 = G.b_row + nb * (BN / 2);
        brow1 = brow0 + G.n;
      } else {
        brow0 = G.b_row + nb * BN;
        brow1 = brow0 + BN / 2;
      }
      const int koff = G.k_off;
      const bool bsel = G.b_sel != 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        const bool second = kb >= kb1;
        const CUtensorMap* ta = second ? &tmA2 : &tmA;
        const CUtensorMap* tb = (second || bsel) ? &tmB1 : &tmB0;
        const int kc = second ? (kb - kb1) * 64 : koff + kb * 64;
        if (lane == 0) {
          GEMM_TIMED_WAIT(&empty[stage], phase ^ 1, 0);
          ptx::mbar_arrive_expect_tx(&full[stage], L::A_BYTES + L::B_BYTES);
          ptx::tma_load_2d(ta, &full[stage], sA + stage * L::A_BYTES, kc, arow);
          ptx::tma_load_2d(tb, &full[stage], sB + stage * L::B_BYTES, kc, brow0);
          ptx::tma_load_2d(tb, &full[stage], sB + stage * L::B_BYTES + (BN / 2) * 128, kc, brow1);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    int qs = 0;
    uint32_t qph = 0;
    while (true) {
      ptx::mbar_wait(&qfull[qs], qph);
      const int tile = tq[qs];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&qempty[qs]);
      if (++qs == kTileQ) { qs = 0; qph ^= 1; }
      if (tile < 0) break;
      GEMM_TIMED_WAIT(&tempty[acc], aphase ^ 1, 2);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        GEMM_TIMED_WAIT(&full[stage], phase, 1);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint64_t a0 = ptx::sdesc_sw128(ptx::smem_u32(sA + stage * L::A_BYTES));
          const uint64_t b0 = ptx::sdesc_sw128(ptx::smem_u32(sB + stage * L::B_BYTES));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::umma_bf16_ss(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int part = (warp - 4) >> 2;
    constexpr int NPART = EW / 4;
    float* tiles = reinterpret_cast<float*>(smem + L::EPI_OFF + (warp - 4) * L::EPI_STRIDE);   // 1024-aligned
    int tsel = 0;
    int acc = 0;
    uint32_t aphase = 0;
    int qs = 0;
    uint32_t qph = 0;
    while (true) {
      ptx::mbar_wait(&qfull[qs], qph);
      const int tile = tq[qs];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&qempty[qs]);
      if (++qs == kTileQ) { qs = 0; qph ^= 1; }
      if (tile < 0) break;
      const int gi = gemm_find_group(ts, ng, tile);
      const GemmGroup G = sched->g[gi];
      const int nt = gemm_ntiles_n(G, BN);
      const int tin = tile - ts[gi];
      const int mb = tin / nt, nb = tin % nt;
      GEMM_TIMED_WAIT(&tfull[acc], aphase, 3);
      GEMM_STAT(const long long t_epi0 = clock64());
      GEMM_STAT(acc_st[5] += 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      const int row0 = mb * 128 + q * 32;          // first tile row of this warp
      epi_tile<BN, L::NB, NPART>(tb, lane, part, G, row0, nb, tiles, tsel, &tmC);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      GEMM_STAT(acc_st[4] += clock64() - t_epi0);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
#ifdef PROBE_GEMM_STATS
  if (sched->stats && lane == 0 && (warp <= 1 || warp == 4)) {
    acc_st[6] = clock64() - t_kernel0;
    for (int i = 0; i < 7; ++i)
      if (acc_st[i]) atomicAdd(&sched->stats[i], static_cast<unsigned long long>(acc_st[i]));
  }
#endif
  if (warp >= 4 && lane == 0) ptx::bulk_wait<0>();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * BN>(tmem_base);
  }
}

// =============================================================================
// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs computes a 256 × BN tile.
// Each CTA loads its own 128 rows of A and ONE HALF of B (rows [0, BN/2) in CTA 0,
// [BN/2, BN) in CTA 1 — for SwiGLU: gate rows in CTA 0, up rows in CTA 1), so a stage
// is 32 KB instead of 48 KB and 6 stages fit.  The leader CTA's single thread issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem; the accumulator rows of
// each CTA live in its own TMEM and each CTA's epilogue drains its own 128 rows.
// Barriers: TMA bytes of both CTAs complete on the LEADER's `full` (the leader's expect_tx
// covers both; the peer cannot refill a stage before the MMA has consumed it, so phases
// never mix); MMA commits multicast to both CTAs' `empty` / `tfull`;
// both CTAs' epilogues arrive on the leader's `tempty`.  The leader claims tiles and
// mirrors them into the peer's queue through DSMEM.
// =============================================================================
template <int BN, int STAGES, int EW, int NBUF = 1>
struct Gemm2Smem {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = (BN / 2) * 128;
  static constexpr int BAR_OFF = STAGES * (A_BYTES + B_BYTES);
  static constexpr int TS_OFF = BAR_OFF + (2 * STAGES + 4 + 2 * kTileQ) * 8 + 16 + kTileQ * 4;
  // the 256×512 kernel with double-buffered wide stores fits 227 KB only with a ≤ 384-group table
  static constexpr int TSCAP = (BN >= 512 && NBUF == 2) ? 384 : kMaxGroups;
  static constexpr int EPI_OFF = (TS_OFF + (TSCAP + 1) * 4 + 1023) / 1024 * 1024;
  static constexpr int NB = NBUF;
  static constexpr int BYTES = EPI_OFF + EW * NB * 4096 + 1024;
};

template <int BN, int STAGES, int EW, int MAXR = 255, int NBUF = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * EW, 1) __maxnreg__(MAXR)
grouped_gemm_2cta_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                         const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmC,
                         const __grid_constant__ CUtensorMap tmA2, GemmSched* __restrict__ sched, int K, int K2) {
  using L = Gemm2Smem<BN, STAGES, EW, NBUF>;
  // BN = 512 (wide tile): two N = 256 UMMAs per k-step into the whole
  // 512-column TMEM, so ONE accumulator (the epilogue no longer overlaps the next tile's
  // MMAs); each CTA loads two 128-row B boxes per k-block.  Half the A bytes per FLOP.
  constexpr int NACC = BN >= 512 ? 1 : 2;
  constexpr int TCOLS = BN >= 512 ? 512 : 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* qfull = tempty + 2;
  uint64_t* qempty = qfull + kTileQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qempty + kTileQ);
  volatile int* tq = reinterpret_cast<volatile int*>(tmem_slot + 4);
  int* ts = reinterpret_cast<int*>(smem + L::TS_OFF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int ng = sched->num_groups;
  GEMM_STAT(long long acc_st[7] = {0, 0, 0, 0, 0, 0, 0});
  GEMM_STAT(const long long t_kernel0 = clock64());
  if (ng > L::TSCAP) __trap();                  // the host picks this instance only for ≤ TSCAP groups
  for (int i = threadIdx.x; i < ng; i += blockDim.x) ts[i] = sched->g[i].tile_start;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);            // leader's expect_tx covers both CTAs' bytes
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * EW);
    }
    for (int q = 0; q < kTileQ; ++q) {
      ptx::mbar_init(&qfull[q], 1);
      ptx::mbar_init(&qempty[q], 2 + 2 * EW);   // leader: MMA + EW epilogue; peer: producer + EW epilogue
    }
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB0);
    ptx::tma_prefetch_desc(&tmB1);
    if (K2 > 0) ptx::tma_prefetch_desc(&tmA2);
  }
  if (warp == 2) ptx::tmem_alloc_cg2<TCOLS>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();          // barrier inits visible to the peer, TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kb1 = (K + 63) / 64;
  const int num_kb = kb1 + (K2 > 0 ? (K2 + 63) / 64 : 0);
  const int unit = static_cast<int>(blockIdx.x >> 1);     // cluster index (EP-emulation partition)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs;
    // lane 0 handles the tile queue and the TMA tile loads)
    const int l2h = sched->l2hint;
    const uint64_t pol_a = (l2h & 4) ? ptx::policy_evict_first() : 0;
    const uint64_t pol_b = (l2h & 2) ? ptx::policy_evict_last() : 0;
    int stage = 0;
    uint32_t phase = 0;
    int qs = 0;
    uint32_t qph = 0;
    int raw_next = (lane == 0 && leader) ? claim_raw(sched, unit) : 0;
    while (true) {
      int tile = 0;
      if (lane == 0) {
        if (leader) {
          tile = claim_finish(sched, unit, raw_next);
          if (tile >= 0) raw_next = claim_raw(sched, unit);   // next claim in flight during this tile
          ptx::mbar_wait(&qempty[qs], qph ^ 1);
          tq[qs] = tile;
          ptx::st_cluster_u32(ptx::mapa(ptx::smem_u32(const_cast<int*>(&tq[qs])), 1), static_cast<uint32_t>(tile));
          ptx::fence_acq_rel_cluster();          // the DSMEM store before the remote arrive (once per tile)
          ptx::mbar_arrive(&qfull[qs]);
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&qfull[qs]), 1));
        } else {
          ptx::mbar_wait_cluster(&qfull[qs], qph);
          tile = tq[qs];
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&qempty[qs]), 0));
        }
      }
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (++qs == kTileQ) { qs = 0; qph ^= 1; }
      if (tile < 0) break;
      const int gi = gemm_find_group(ts, ng, tile);
      const GemmGroup& G = sched->g[gi];
      const int nt = gemm_ntiles_n(G, BN);
      const int tin = tile - ts[gi];
      const int mb = tin / nt, nb = tin % nt;
      const int arow = G.a_row + mb * 256 + static_cast<int>(rank) * 128;
      int brow;
      if (G.mode == EPI_SWIGLU) brow = G.b_row + (rank ? G.n : 0) + nb * (BN / 2);
      else brow = G.b_row + nb * BN + static_cast<int>(rank) * (BN / 2);
      const int koff = G.k_off;
      const bool bsel = G.b_sel != 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        const bool second = kb >= kb1;
        const CUtensorMap* ta = second ? &tmA2 : &tmA;
        const CUtensorMap* tb = (second || bsel) ? &tmB1 : &tmB0;
        const int kc = second ? (kb - kb1) * 64 : koff + kb * 64;
        if (lane == 0) {
          GEMM_TIMED_WAIT(&empty[stage], phase ^ 1, 0);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (L::A_BYTES + L::B_BYTES));
          if (pol_a) ptx::tma_load_2d_cg2_hint(ta, &full[stage], sA + stage * L::A_BYTES, kc, arow, pol_a);
          else ptx::tma_load_2d_cg2(ta, &full[stage], sA + stage * L::A_BYTES, kc, arow);
          if constexpr (BN >= 512) {
            // N-rows [i·256, i·256 + 256) of UMMA i split 128 / 128 between the pair's CTAs;
            // SwiGLU: UMMA 0 = gate rows, UMMA 1 = the matching up rows (F further)
            const bool sw = G.mode == EPI_SWIGLU;
            const int b0r = G.b_row + nb * (sw ? BN / 2 : BN) + static_cast<int>(rank) * 128;
            ptx::tma_load_2d_cg2(tb, &full[stage], sB + stage * L::B_BYTES, kc, b0r);
            ptx::tma_load_2d_cg2(tb, &full[stage], sB + stage * L::B_BYTES + 128 * 128, kc, b0r + (sw ? G.n : 256));
          } else {
            if (pol_b) ptx::tma_load_2d_cg2_hint(tb, &full[stage], sB + stage * L::B_BYTES, kc, brow, pol_b);
            else ptx::tma_load_2d_cg2(tb, &full[stage], sB + stage * L::B_BYTES, kc, brow);
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, BN >= 512 ? 256 : BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      int qs = 0;
      uint32_t qph = 0;
      while (true) {
        ptx::mbar_wait(&qfull[qs], qph);
        const int tile = tq[qs];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&qempty[qs]);
        if (++qs == kTileQ) { qs = 0; qph ^= 1; }
        if (tile < 0) break;
        GEMM_TIMED_WAIT(&tempty[acc], aphase ^ 1, 2);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          GEMM_TIMED_WAIT(&full[stage], phase, 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint64_t a0 = ptx::sdesc_sw128(ptx::smem_u32(sA + stage * L::A_BYTES));
            const uint64_t b0 = ptx::sdesc_sw128(ptx::smem_u32(sB + stage * L::B_BYTES));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              ptx::umma_bf16_ss_cg2(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
              if constexpr (BN >= 512) {   // second N = 256 half: B box at +16 KB (1024 16-byte units), TMEM cols +256
                ptx::umma_bf16_ss_cg2(d + 256, a0 + 2 * k, b0 + 1024 + 2 * k, idesc, (kb | k) != 0);
              }
            }
            ptx::umma_commit_cg2(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) ptx::umma_commit_cg2(&tfull[acc], 0x3);
        __syncwarp();
        if (++acc == NACC) { acc = 0; aphase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs, own 128 rows)
    const int q = warp & 3;
    const int part = (warp - 4) >> 2;
    constexpr int NPART = EW / 4;
    float* tiles = reinterpret_cast<float*>(smem + L::EPI_OFF + (warp - 4) * L::NB * 4096);
    int tsel = 0;
    int acc = 0;
    uint32_t aphase = 0;
    int qs = 0;
    uint32_t qph = 0;
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
    const uint64_t store_pol = (sched->l2hint & 1) ? ptx::policy_evict_first() : 0;
    while (true) {
      ptx::mbar_wait_cluster(&qfull[qs], qph);
      const int tile = tq[qs];
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&qempty[qs]);
        else ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&qempty[qs]), 0));
      }
      if (++qs == kTileQ) { qs = 0; qph ^= 1; }
      if (tile < 0) break;
      const int gi = gemm_find_group(ts, ng, tile);
      const GemmGroup G = sched->g[gi];
      const int nt = gemm_ntiles_n(G, BN);
      const int tin = tile - ts[gi];
      const int mb = tin / nt, nb = tin % nt;
      GEMM_TIMED_WAIT(&tfull[acc], aphase, 3);
      GEMM_STAT(const long long t_epi0 = clock64());
      GEMM_STAT(acc_st[5] += 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      const int row0 = mb * 256 + static_cast<int>(rank) * 128 + q * 32;
      epi_tile<BN, L::NB, NPART>(tb, lane, part, G, row0, nb, tiles, tsel, &tmC, store_pol);
      GEMM_STAT(acc_st[4] += clock64() - t_epi0);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tempty[acc]);
        else ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
      }
      if (++acc == NACC) { acc = 0; aphase ^= 1; }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }
#ifdef PROBE_GEMM_STATS
  if (sched->stats && lane == 0 && rank == 0 && (warp <= 1 || warp == 4)) {
    acc_st[6] = clock64() - t_kernel0;
    for (int i = 0; i < 7; ++i)
      if (acc_st[i]) atomicAdd(&sched->stats[i], static_cast<unsigned long long>(acc_st[i]));
  }
#endif
  __syncthreads();
  ptx::tc_fence_before();
  ptx::cluster_sync();          // no remote arrive / DSMEM access after this point
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2<TCOLS>(tmem_base);
  }
}

}  // namespace probe
