/* probe.h — C-ABI of the B200-native PROBE expert-parallel MoE hot path.
 *
 * PROBE (arXiv 2602.00509): an EP MoE layer whose next-layer expert load is
 * forecast by a Gate-Initialized Lookahead Predictor (PAPER.md Eq. (P),
 * P:377-385), turned into a replica placement + token assignment by a greedy
 * Balance-Optimal Planner (Algorithm 1), executed as All-to-All
 * dispatch → grouped SwiGLU expert GEMMs → gate-weighted combine, while
 * the planned replica weights are prefetched over NVLink in a split phase that
 * yields to the Combine.
 *
 * Conventions for every entry point:
 *  - Pointers are DEVICE pointers unless stated; row-major; bf16 = IEEE bfloat16
 *    (uint16 storage), fp32 = IEEE binary32.  "act" below = the activation/weight element
 *    type selected by probe_config.dtype: bf16 (default) or fp32 (parity path); every
 *    activation / weight pointer documented as bf16 is fp32 when dtype = PROBE_FP32.
 *  - `stream` is a cudaStream_t passed as void* (no CUDA headers needed).
 *  - Every call only ENQUEUES work on its stream(s) and never synchronises the
 *    host (CUDA-Graph safe), except probe_check/probe_finalize.
 *    Graph capture rule: a capturing stream cannot wait on an event recorded outside its
 *    capture, so the library omits those cross-capture waits (e.g. a captured forward of
 *    layer L on the plan of L enqueued eagerly).  The caller must therefore complete all
 *    eager work of the context (cudaDeviceSynchronize) before beginning a capture.
 *    Cross-process barriers keep their epochs in device memory, so replays stay ordered.
 *  - Host-checkable problems (null/out-of-range scalar, shape, call order)
 *    return a status synchronously and set probe_last_error(); nothing is
 *    enqueued in that case.  Device-detected problems (receive-capacity
 *    overflow) set a device error word reported by probe_check().
 *  - Ownership: the caller owns every tensor and every workspace (sizes from
 *    probe_workspace); the library owns only the opaque context, its streams
 *    and events.  Inputs are never written.
 *  - Determinism: identical inputs ⇒ bit-identical routing ids, counts, plans,
 *    dispatch layouts on every rank and every run (ties: lowest expert id).
 *
 * Process / rank model.  EP has G logical ranks (the paper's `ep`, Table
 * P:252).  A process hosts a contiguous block of `local_ranks` logical ranks
 * starting at `rank_begin`: local_ranks = 1 on an 8-GPU run (one process per
 * GPU), local_ranks = G in single-GPU emulation of the whole EP group.
 * Symmetric buffers of remote ranks are reached through peer-mapped pointers
 * (NVLink over NVSwitch); all hot-path traffic is SM loads/stores.
 */
#ifndef PROBE_H_
#define PROBE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct probe_ctx_s* probe_ctx;

typedef enum {
  PROBE_OK = 0,
  PROBE_EINVAL = 1,    /* null pointer / out-of-range scalar */
  PROBE_ESHAPE = 2,    /* dimension mismatch or unsupported size */
  PROBE_EBUDGET = 3,   /* replica budget / slot violation */
  PROBE_ECAPACITY = 4, /* T > max_tokens, or receive capacity overflow (device) */
  PROBE_ECUDA = 5,     /* CUDA runtime/driver error */
  PROBE_ECOMM = 6,     /* symmetric-buffer table inconsistent */
  PROBE_ESTATE = 7     /* call order (e.g. prefetch START before plan) */
} probe_status;

/* Host struct, copied at init.  Symbols follow PAPER.md Table 1. */
typedef struct {
  int32_t ep_size;        /* G = ep; 1..64 */
  int32_t rank_begin;     /* first logical rank hosted by this process */
  int32_t local_ranks;    /* number of logical ranks hosted by this process */
  int32_t num_experts;    /* E; E % G == 0 (contiguous sharding P′, R22); E % 8 == 0; E <= 256 */
  int32_t top_k;          /* k; 1 <= k <= min(E, 16) */
  int32_t hidden;         /* H; multiple of 64 */
  int32_t ffn;            /* F (expert intermediate width); multiple of 64 */
  int32_t res_hidden;     /* h, predictor residual width (paper silent; R7); multiple of 8, or 0 */
  int32_t max_tokens;     /* capacity for T (tokens per rank, R31) */
  int32_t recv_capacity;  /* receive rows per rank (one row per routed (token, slot)) */
  int32_t replica_budget; /* R_b <= 3 redundant experts per rank; 0 => static EP */
  int32_t kmax;           /* planner iteration cap k_max (16) */
  int32_t n_sat;          /* η_g knee in pairs: c(m) = max(m, n_sat) for m > 0 (Eq. 2, R11) */
  int32_t dtype;          /* PROBE_BF16 (product path: bf16 operands on tcgen05, fp32 accumulate)
                             or PROBE_FP32 (parity path: x, router, predictor and expert weights fp32,
                             SIMT fp32 GEMMs; north_star's 1e-5·RMS bound).  Selects the element type of
                             every activation/weight pointer below and of the RECV/Y/replica buffers. */
  int32_t dedup_wire;     /* 0: dispatch ships one row per routed (token, slot) and the combine pulls per-slot Y
                             rows (D1, D2).  1: the wire format of §8(a) a6/a8 — ONE row per unique
                             (token, destination rank) plus per-slot metadata; the receiver expands it into the
                             grouped-GEMM rows locally; the expert rank sums g·y over the token's co-located
                             slots in fp32 (slot order) and pushes ONE fp16 partial per (token, destination)
                             back to the source, which sums partials in ascending destination order (R25). */
  int32_t predispatch;    /* NEXT-4 ("pre-dispatch hidden states to high-confidence experts"), needs
                             dedup_wire = 1: when layer L was predicted (probe_predict(L) + probe_plan(L)),
                             probe_moe_forward(L) pushes every token's x row to the HOME ranks of its predicted
                             experts on a side stream WHILE the gate computes the actual routing; the dispatch
                             then ships payload only for (token, dest) pairs the prediction missed, and the
                             receiver expands hits from the pre-dispatch buffer.  0 = off. */
  int32_t fuse_gate_predictor; /* 1: after probe_predict_prepare(L+1), probe_moe_forward(L) computes the gate
                             logits W_L·x, the NEXT layer's prior W_{L+1}·x and the predictor activation
                             a = bf16(SiLU(Ŵ¹_{L+1}·x)) (Eq. (P), R8) in ONE tensor-core GEMM over x, and
                             probe_predict(L+1) runs only the residual Ŵ²·a, the top-k and n̂.  Eq. (P) is
                             unchanged; x is read once instead of three times, but the predictor's x-side
                             FLOPs move from the aux stream onto the gate.  Pays when the dispatch is HBM-bound
                             (several logical ranks per GPU); with one rank per GPU the NVLink dispatch hides
                             the aux-stream predictor and 0 is right.  Requires bf16, E % 32 == 0 and
                             top_k <= 8.  0 = off. */
  int64_t alpha_ps;       /* compute cost per routed pair, picoseconds (F̄/F_peak, R11) */
  int64_t beta_ps;        /* comm cost per remote pair, picoseconds (2·2H/BW_net, Eq. 5, λ=1) */
  int64_t bw_bytes_per_us;/* BW_net for Eq. 6 replica caps */
  int64_t expert_bytes;   /* 𝒲 = 3·H·F·sizeof(dtype) bytes (6HF for bf16, 12HF for fp32); checked */
} probe_config;

/* probe_config.dtype */
enum { PROBE_BF16 = 0, PROBE_FP32 = 1 };

/* Buffer ids for probe_workspace / probe_init. */
enum {
  PROBE_BUF_RECV = 0,    /* symmetric [recv_capacity, H] act (bf16/fp32): dispatched token rows (peers write) */
  PROBE_BUF_Y = 1,       /* symmetric [recv_capacity, H] fp16 (fp32 when dtype = PROBE_FP32): expert outputs (peers read in combine; D2) */
  PROBE_BUF_REP_W13 = 2, /* symmetric [2*R_b, 2F, H] act: replica slots, 2 banks by layer parity */
  PROBE_BUF_REP_W2 = 3,  /* symmetric [2*R_b, H, F] act */
  PROBE_BUF_BOARD = 4,   /* symmetric count boards [2 parity][2 kind][G][E] int32 + flags */
  PROBE_BUF_SIGNAL = 5,  /* symmetric signal pad (cross-process barriers) */
  PROBE_BUF_META = 6,    /* symmetric [recv_capacity] int4 per received row (dedup_wire): first row of its
                            (token, dest) pair, next row of the pair, gate weight, return index */
  PROBE_BUF_COMB = 7,    /* symmetric [max_tokens, min(k, G), H] fp16 (fp32 when dtype = PROBE_FP32): per
                            (token, destination) partial sums pushed back by the expert ranks (dedup_wire) */
  PROBE_BUF_PRE = 8,     /* symmetric [G sources, max_tokens, H] act: pre-dispatched rows (predispatch) */
  PROBE_NSYM = 9,
  PROBE_BUF_SCRATCH = 9, /* private scratch for ALL local ranks of this process */
  PROBE_NBUF = 10
};

/* Sizes to allocate.  bytes[i] for i < PROBE_NSYM is PER LOGICAL RANK; the
 * local ranks' copies of buffer i must be one contiguous allocation with
 * stride bytes[i] (rank_begin first).  bytes[PROBE_BUF_SCRATCH] is the
 * process-private scratch.  All sizes are multiples of 1024. */
probe_status probe_workspace(const probe_config* cfg, uint64_t bytes[PROBE_NBUF]);

/* peer_ptrs: HOST array [PROBE_NSYM][G] of device addresses, as mapped in this
 * process, of every logical rank's copy of each symmetric buffer (zeroed by the
 * caller before init).  scratch: this process's scratch (bytes[PROBE_BUF_SCRATCH]).
 * Creates the auxiliary (predict/plan) and prefetch streams. */
probe_status probe_init(const probe_config* cfg, const uint64_t* peer_ptrs, void* scratch,
                        probe_ctx* out);

/* Main track for layer L: gate (ground-truth router + top-k, R1-R5) →
 * actual-count all-gather → materialize plan(L) on the actual counts (R23) →
 * dispatch (R24 layout) → grouped SwiGLU GEMMs → gate-weighted combine (R25).
 *   x         [local_ranks, T, H] act (this process's ranks, rank_begin first)
 *   w_router  [E, H] act;  b_router [E] fp32 or NULL
 *   w13       [local_ranks*E/G, 2F, H] act base experts of the local ranks (gate rows 0..F-1, up F..2F-1)
 *   w2        [local_ranks*E/G, H, F] act
 * dtype = PROBE_FP32: every GEMM is fp32 (SIMT, ascending-K FMA), the SwiGLU activation and Y
 * stay fp32; routing/plan/layout are the same integer kernels as the bf16 path.
 *   use_plan  0 ⇒ static EP (P′); 1 ⇒ the plan computed by probe_plan(layer)
 *   out       [local_ranks, T, H], fp32 if out_fp32 else bf16
 *   topk_ids  [local_ranks, T, k] int32 or NULL;  topk_w [local_ranks, T, k] fp32 or NULL
 * If a plan for this layer was enqueued, the layout waits for it; if a prefetch
 * was enqueued, the expert GEMMs wait for "slots ready" (exposed overhead). */
probe_status probe_moe_forward(probe_ctx ctx, int32_t layer, const void* x, int32_t T,
                               const void* w_router, const float* b_router, const void* w13,
                               const void* w2, int32_t use_plan, void* out, int32_t out_fp32,
                               int32_t* topk_ids, float* topk_w, void* stream);

/* Lookahead predictor for layer `next_layer` (Eq. (P)): l̂ = W x + b + Ŵ2·bf16(SiLU(Ŵ1 x))
 * on the CURRENT layer's input x (R6), top-k (lowest-id ties), per-rank predicted
 * counts n̂[r][e] (R9) all-gathered into every rank's count board.
 *   x, w_router_next act;  w_res1 [h, H] act or NULL, w_res2 [E, h] act or NULL (NULL ⇒ frozen prior only);
 *   the activation is rounded to bf16 in both dtypes (R8: part of the predictor's definition)
 *   pred_counts [G, E] int32 out or NULL;  pred_logits [local_ranks, T, E] fp32 out or NULL
 *   (pred_logits are written by the same product-path kernels that produce n̂: the top-k
 *   select kernel stores exactly the l̂ values it ranks)
 * If probe_moe_forward(next_layer-1) was enqueued, waits for its gate (x ready). */
probe_status probe_predict(probe_ctx ctx, int32_t next_layer, const void* x, int32_t T,
                           const void* w_router_next, const float* b_router_next,
                           const void* w_res1, const void* w_res2, int32_t* pred_counts,
                           float* pred_logits, void* stream);

/* Fused gate + predictor stage 1 (probe_config.fuse_gate_predictor = 1).  Arms the NEXT
 * probe_moe_forward(next_layer - 1) of this context: its gate GEMM then multiplies x by
 * [W_{next_layer-1} ; w_router_next ; w_res1] in one tcgen05 pass (x read once, tiles of the
 * three weight blocks interleaved per row chunk so they share x in L2) and keeps the prior
 * logits W_{next_layer}·x (fp32) and a = bf16(SiLU(Ŵ¹·x)) (R8) for probe_predict(next_layer),
 * which reuses them when called with the same x, T, w_router_next and w_res1 pointers
 * (otherwise it recomputes both).  Reuse is decided by pointer, so the caller must not change
 * the CONTENTS of x, W_{next_layer} or Ŵ¹ between that forward and that predict.  Eq. (P) is unchanged: only the
 * place where its two x-side products are computed moves.
 *   w_router_next [E, H] bf16;  w_res1 [h, H] bf16 or NULL (prior only)
 * Host-side only (records pointers; enqueues nothing).  PROBE_ESTATE if the config did not
 * enable the fusion. */
probe_status probe_predict_prepare(probe_ctx ctx, int32_t next_layer, const void* w_router_next,
                                   const void* w_res1);

/* Balance planning for `next_layer` (Algorithm 1 under R10-R22; integer costs).
 *   pred_counts [G, E] int32 device, or NULL ⇒ the board written by probe_predict
 *   window_ns   [G] int64 device: per-rank hiding window in ns (R26)
 *   replicas [G,3] int32 out or NULL (-1 = empty; sorted expert ids)
 *   quota    [G,E,G] int32 out or NULL (assignment A on n̂)
 *   plan_stats [8] int64 out or NULL: iterations, transfers, maxL_before, maxL_after, caps bitmask
 * Single-CTA kernel on `stream`; every rank computes the identical plan (R10). */
probe_status probe_plan(probe_ctx ctx, int32_t next_layer, const int32_t* pred_counts,
                        const int64_t* window_ns, int32_t* replicas, int32_t* quota,
                        int64_t* plan_stats, void* stream);

/* Split-phase prefetch of next_layer's replica weights (R27).
 * phase 0 START: on the context's prefetch stream, after "plan done(next_layer)"
 *   and "GEMM start(next_layer-1)": part 1 copies chunks until the combine of
 *   next_layer-1 raises the suspend flag; after "combine done(next_layer-1)",
 *   part 2 copies the rest; then "slots ready(next_layer)" is recorded.
 *   w13_next / w2_next: base expert weights of next_layer on the local ranks
 *   (layout as in probe_moe_forward); senders push into receivers' slots.
 * phase 1 WAIT: make `stream` wait for "slots ready(next_layer)". */
probe_status probe_prefetch(probe_ctx ctx, int32_t next_layer, const void* w13_next,
                            const void* w2_next, int32_t phase, void* stream);

/* Debug / test views (device copies, enqueued on `stream`, NULL = skip):
 *   counts [G,E] actual counts of the last forward; split [G,E,G] materialized;
 *   route [local_ranks,T,k] int32 pairs (dest, row) as 2 ints;
 *   group_rows [local_ranks, E/G+3] rows per local slot; replicas_used [G,3]. */
probe_status probe_debug_layout(probe_ctx ctx, int32_t* counts, int32_t* split, int32_t* route,
                                int32_t* group_rows, int32_t* replicas_used, void* stream);

/* Split-phase prefetch accounting (R27): out[0] / out[1] (device int32) = KiB of replica
 * weights this process has pushed so far in part 1 (during the expert GEMMs, before the
 * combine's suspend flag) / in part 2 (after the combine).  Cumulative since probe_init;
 * enqueued on `stream` after the context's prefetch stream work issued so far. */
probe_status probe_debug_prefetch(probe_ctx ctx, int32_t* out, void* stream);

/* Measured hiding window (R26, "confined within the computation window"):
 * window_ns[r] (device int64 [G] out) = the most recently measured expert-GEMM phase of rank r
 * (%globaltimer stamps around GEMM1..GEMM2 of every probe_moe_forward, all-gathered into every
 * rank's count board, so all ranks plan from identical windows; when a process hosts several
 * logical ranks their tiles share one grouped GEMM and rank r gets its share by the planner's
 * compute cost, T_GEMM · C_r / Σ C with C_r = Σ_{active slots} max(rows, n_sat) (R11) — its GEMM
 * time on a GPU of its own), or fallback_ns where no layer
 * has been measured yet, plus attention_ns (the attention window that follows, caller-given).
 * Device to device, no host synchronisation; enqueued on `stream` (NULL = the aux stream, i.e.
 * before a probe_plan issued without a stream).  One step stale by construction (R26). */
probe_status probe_window(probe_ctx ctx, int64_t attention_ns, int64_t fallback_ns, int64_t* window_ns,
                          void* stream);

/* Device status words (device int32 out[8], enqueued on `stream` after the work issued so far
 * on the context's aux and prefetch streams): out[0] error word (bit 0 receive overflow,
 * bit 2 plan, bit 3 fp16 Y range), out[1] prefetch suspend flag, out[2] / out[3] prefetch
 * part-1 / part-2 KiB, out[4] number of layers that FELL BACK TO STATIC EP because the
 * plan's layout would have overflowed some rank's recv_capacity (SURVEY §8(b) Errors: the
 * layout kernel decides this on device, identically on every rank, and runs static EP for
 * that layer; semantic equivalence P:364 keeps the output the same function).  If static
 * EP itself overflows, the error word is set and probe_check returns PROBE_ECAPACITY. */
probe_status probe_debug_flags(probe_ctx ctx, int32_t* out, void* stream);

/* Test hook: one grouped bf16 GEMM through the tcgen05 kernel,
 * C[g] (fp32, [m_g, N]) = A[a_row_g : a_row_g + m_g, :K] · B[b_row_g : b_row_g + N, :K]^T
 * (mode 0) or act = SiLU(gate)⊙up (bf16, [m_g, N/2]) with gate rows b_row_g.., up rows
 * b_row_g + N/2.. (mode 1); 3: SiLU → bf16, 4: no store, 5/6: fused top-k (k = 8),
 * 7: fp16 C (the expert-output Y epilogue, TMA stores in SWIZZLE_64B).
 * groups: host array of num_groups × {a_row, m, b_row, c_row}. */
probe_status probe_test_gemm(const void* A, int64_t a_rows, const void* B, int64_t b_rows,
                             int32_t K, int32_t N, const int32_t* groups, int32_t num_groups,
                             int32_t mode, void* C, void* stream);

/* Timing hook: as probe_test_gemm with an explicit kernel variant (-1 = default for
 * `mode`; 0: BN=128/6 stages/4 epilogue warps, 1: 256/4/4,
 * 6: CTA pair (cta_group::2), 256-row tiles, 6 stages, 10: 1-CTA <256,4,4> capped at 216 registers,
 * 11: <128,6,4> capped at 192 registers, 12: CTA pair with 256×128 tiles and 8 stages; other numbers
 * are not available),
 * run once, then `reps` times between CUDA events on `stream`; *ms_out = mean ms. */
probe_status probe_bench_gemm(const void* A, int64_t a_rows, const void* B, int64_t b_rows,
                              int32_t K, int32_t N, const int32_t* groups, int32_t num_groups,
                              int32_t mode, int32_t variant, int32_t reps, float* ms_out, void* C,
                              void* stream);

/* Synchronise this context's streams; return PROBE_ECAPACITY if the device
 * error word is set (receive overflow: the layer's output is invalid), PROBE_ESHAPE if an
 * expert output exceeded the fp16 range of the Y buffer (|y| > 65504, D2). */
probe_status probe_check(probe_ctx ctx);
const char* probe_last_error(probe_ctx ctx);   /* ctx may be NULL (last global error) */
probe_status probe_finalize(probe_ctx ctx);

/* Phase profiling.  probe_profile(ctx, n) enables CUDA-event timing of the next n
 * probe_moe_forward calls (events recorded on the stream each phase runs on;
 * 0 disables).  probe_profile_read copies the elapsed milliseconds of every
 * recorded forward into ms[n][PROBE_NPHASE] (synchronises) and returns how many
 * forwards were recorded in *n_out.  Phases of the main track: */
enum {
  PROBE_PH_GATE = 0,      /* router GEMM (a1) */
  PROBE_PH_SELECT = 1,    /* top-k select + softmax + dispatch ranks (a1) */
  PROBE_PH_COUNTS = 2,    /* chunk scan + actual-count all-gather (a3) */
  PROBE_PH_LAYOUT = 3,    /* materialize plan + layout + GEMM schedules (a5) */
  PROBE_PH_DISPATCH = 4,  /* token dispatch (a6) incl. the cross-process barrier */
  PROBE_PH_EXPAND = 5,    /* dedup wire: receiver-side expansion into slot rows (empty otherwise) */
  PROBE_PH_WAIT = 6,      /* exposed wait for replica slots (prefetch not hidden, R28) */
  PROBE_PH_GEMM1 = 7,     /* grouped GEMM1 + SwiGLU epilogue (a7) */
  PROBE_PH_GEMM2 = 8,     /* grouped GEMM2 (a7) */
  PROBE_PH_COMBINE = 9,   /* gate-weighted combine (a8): per-slot pull, or the expert-side partials (dedup) */
  PROBE_PH_REDUCE = 10,   /* dedup wire: source-side sum of the partials (empty otherwise) */
  PROBE_PH_TOTAL = 11,    /* whole forward on the main stream */
  PROBE_PH_PREDISPATCH = 12, /* NEXT-4: forward start → pre-dispatch done (side stream; 0 when not used).
                                Compare with gate + select + counts + layout: the overlap */
  PROBE_NPHASE = 13
};
probe_status probe_profile(probe_ctx ctx, int32_t n);
probe_status probe_profile_read(probe_ctx ctx, float* ms, int32_t* n_out);

/* Multi-process symmetric buffers (one process per GPU).  probe_ipc_export returns the
 * CUDA IPC handle (64 bytes) of the allocation containing dev_ptr and dev_ptr's offset in
 * it; peers call probe_ipc_import to map it (NVLink peer mapping, lazy peer access) and get
 * the address to place in probe_init's peer table; probe_ipc_close unmaps an imported base
 * (address returned by import minus offset).  When local_ranks < ep_size, forward /
 * predict / prefetch insert device-side barriers on the symmetric signal pad
 * (st.release.sys / ld.acquire.sys, epochs kept in device memory so captured graphs replay
 * correctly): after the count all-gather, after dispatch (and the pre-dispatch), after the
 * expert GEMMs (per-slot wire) or after the partial-sum push (dedup wire), after the
 * predicted-count all-gather, and after the replica pushes. */
probe_status probe_ipc_export(const void* dev_ptr, uint8_t handle[64], uint64_t* offset);
probe_status probe_ipc_import(const uint8_t handle[64], uint64_t offset, uint64_t* dev_ptr);
probe_status probe_ipc_close(uint64_t dev_ptr_base);

/* Statistics-based baseline (EPLB-like; not PROBE): history[G,E] (device,
 * caller-owned) += the actual counts n[G,E] of the last forward of `layer` (reset=1 zeroes
 * first).  Pass history as probe_plan's pred_counts to plan from past statistics instead
 * of the lookahead predictor. */
probe_status probe_history_update(probe_ctx ctx, int32_t layer, int32_t reset, int32_t* history,
                                  void* stream);

/* Scale-driven online distillation of the predictor residual (P:387-390
 * "minimizing the Cross-Entropy loss between the predictor's output and the ground-truth
 * router's probability distribution"; readings R33-R37 in DESIGN.md §2.5).
 *
 * probe_distill_grad: for the GL·T tokens of the local ranks ([GL·T, H] bf16, rank-major as
 * in probe_predict), x = the hidden state the predictor reads (entering layer L−1), x_next =
 * the hidden state entering layer L (the teacher's input), w_router/b_router = layer L's
 * frozen router (bf16 [E,H], fp32 [E] or NULL), w_res1 bf16 [h,H] / w_res2 bf16 [E,h] = the
 * residual the product path uses.  Computes, all on device:
 *   student l̂ = W x + b + Ŵ² bf16(SiLU(Ŵ¹ x)),  teacher t = W x_next + b,
 *   loss = Σ_t CE(softmax(t_t), softmax(l̂_t)),
 *   grad_res1 fp32 [h,H] = ∂loss/∂Ŵ¹,  grad_res2 fp32 [E,h] = ∂loss/∂Ŵ²  (overwritten; the
 *   gradient of the SUM over these tokens, R34 — shards add them, then divide by the total),
 *   stats fp64 [4] (overwritten) = {Σ CE, Σ|S∩P|, Σ|S^⌈k/2⌉∩P|, Σ|S∩P^2k|} with S / P the
 *   teacher / student top-k sets (R37: top-K accuracy, top-half-K hit, 2×top-K recall); the
 *   three hit counts are computed only if `fidelity` != 0 (else 0: they cost 24 serial warp
 *   argmaxes per token);
 *   student_logits / teacher_logits fp32 [GL·T, E] (optional outputs, WITHOUT the bias).
 * The first call allocates a workspace (~N·(10h + 12E + 2H) bytes, N = local_ranks ·
 * max_tokens) and must not be inside a stream capture.  Everything runs on `stream` (NULL =
 * the legacy default stream, as in plain CUDA); inputs must be complete on it.  Errors: PROBE_EINVAL (null), PROBE_ESHAPE
 * (res_hidden == 0, or dtype = PROBE_FP32: distillation is bf16-only), PROBE_ECAPACITY (T),
 * PROBE_ESTATE (first call under capture).
 *
 * probe_distill_apply (R36): master[i] += scale · grad[i] (fp32, n elements; scale =
 * −lr / N_total) and w[i] = bf16(master[i]) — the bf16 copy the product path reads. */
probe_status probe_distill_grad(probe_ctx ctx, const void* x, const void* x_next, int32_t T, const void* w_router,
                                const float* b_router, const void* w_res1, const void* w_res2, float* grad_res1,
                                float* grad_res2, double* stats, int32_t fidelity, float* student_logits,
                                float* teacher_logits, void* stream);
probe_status probe_distill_apply(probe_ctx ctx, float* master, const float* grad, void* w, int64_t n, float scale,
                                 void* stream);

/* Options.  PROBE_OPT_EP_EMULATION (single-GPU emulation only): the expert GEMMs split the
 * persistent grid into local_ranks CTA sets, each serving only its logical rank's tiles, so
 * a rank's GEMM runs on ~#SMs/local_ranks SMs and the GEMM time is the straggler's (Eq. 3)
 * as on one GPU per rank.  PROBE_OPT_UNFUSED_TOPK: predictor prior and residual as separate
 * GEMMs and warp-shuffle top-k kernels (debug reference path).  PROBE_OPT_FUSED_EPILOGUE_TOPK:
 * do the router/predictor top-k inside the tcgen05 GEMM epilogue instead of the
 * thread-per-token select kernel (default off: measured slower). */
enum { PROBE_OPT_EP_EMULATION = 1, PROBE_OPT_UNFUSED_TOPK = 2, PROBE_OPT_FUSED_EPILOGUE_TOPK = 3,
       PROBE_OPT_AUX_SMS = 4 /* grid cap (CTAs) of the predictor GEMMs on the aux stream; default #SMs/2 */,
       PROBE_OPT_PAIR_GEMM = 5 /* expert GEMMs on CTA pairs (tcgen05 cta_group::2, 256-row tiles) when the
                                  mean rows per local expert T·k·G/E is at least 256 (else 1-CTA);
                                  default ON, 0 selects the 1-CTA kernel */,
       PROBE_OPT_AUX_START = 8 /* 0 (default): predict(L+1) starts when gate(L) is done, i.e. beside
                                  dispatch(L); 1: after dispatch(L) (beside the expert GEMMs) */,
       PROBE_OPT_PRED_MAXREG = 9 /* 0 (default) or 192: register-capped predictor GEMMs so a dispatch CTA
                                    co-resides on the SMs the aux track holds */,
       PROBE_OPT_PRED_PAIR = 11 /* 1 (default): the predictor's GEMMs run on CTA pairs (Ŵ1·x: 256×256 tiles
                                   when h ≥ 256; [x | a]·[W | Ŵ2]ᵀ: 256×E tiles); 0: the 1-CTA 128-row kernel */,
       PROBE_OPT_L2_HINTS = 10 /* TMA L2 eviction hints of the CTA-pair expert GEMMs: bits 0-2 GEMM1,
                                  bits 4-6 GEMM2; per GEMM bit 0 output stores evict_first, bit 1 weight
                                  (B) loads evict_last, bit 2 activation (A) loads evict_first */ };
probe_status probe_set_option(probe_ctx ctx, int32_t option, int64_t value);

/* Number of library kernel launches enqueued so far by this context (bench accounting). */
int64_t probe_launch_count(probe_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* PROBE_H_ */
